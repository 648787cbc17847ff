# r02 session 38-39: result stash topped up on a background thread in batches (usable as they land), tail take
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
NL=$(python -c "import os,sys; p=[os.path.join(d,'include/cudnn_frontend/thirdparty/nlohmann') for d in sys.path if d]; print(next((q for q in p if os.path.exists(os.path.join(q,'json.hpp'))),''))")
mkdir -p /tmp/st
g++ -O2 -std=c++20 -ffp-contract=off -pthread -Iinclude -I$NL tools/ladder_timing.cpp -o /tmp/st/ladder -Lpaper_1601_05904_b200/lib -laidw_b200 -Wl,-rpath,$PWD/paper_1601_05904_b200/lib
for i in 1 2; do AIDW_HOST_TRACE=1 /tmp/st/ladder 2>&1 | grep -E "pass|102400"; done
for i in 1 2 3; do ./oracle/_ref/conformance/acceptance 2>&1 | grep -E "criterion  [678]"; done
for i in 1 2; do AIDW_WEIGHT_FP64=1 ./oracle/_ref/conformance/acceptance 2>&1 | grep -E "criterion  [678]"; done
