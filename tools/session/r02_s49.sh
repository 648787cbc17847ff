# r02 session 49-50: result stash top-up on 4 threads, filled to 64 MiB after the first call; ladder + acceptance
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
NL=$(python -c "import os,sys; p=[os.path.join(d,'include/cudnn_frontend/thirdparty/nlohmann') for d in sys.path if d]; print(next((q for q in p if os.path.exists(os.path.join(q,'json.hpp'))),''))")
mkdir -p /tmp/st
g++ -O2 -std=c++20 -ffp-contract=off -pthread -Iinclude -I$NL tools/ladder_timing.cpp -o /tmp/st/ladder -Lpaper_1601_05904_b200/lib -laidw_b200 -Wl,-rpath,$PWD/paper_1601_05904_b200/lib
AIDW_HOST_TRACE=1 /tmp/st/ladder 2>&1 | grep -E "pass 0|102400"
for i in 1 2 3; do ./oracle/_ref/conformance/acceptance 2>&1 | grep -E "criterion  [78]"; done
for i in 1 2; do AIDW_WEIGHT_FP64=1 ./oracle/_ref/conformance/acceptance 2>&1 | grep -E "criterion  [78]"; done
timeout 1200 python -m pytest tests/test_conformance.py -q -m gpu 2>&1 | tail -2
