# r02 session 36: host-timing variance of the drop-in kNN stage (acceptance 6-8)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
nproc; lscpu | grep "Model name"; uptime
NL=$(python -c "import os,sys; p=[os.path.join(d,'include/cudnn_frontend/thirdparty/nlohmann') for d in sys.path if d]; print(next((q for q in p if os.path.exists(os.path.join(q,'json.hpp'))),''))")
mkdir -p /tmp/st
g++ -O2 -std=c++20 -ffp-contract=off -pthread -Iinclude -I$NL tools/knn_stage_timing.cpp -o /tmp/st/knn_stage_timing -Lpaper_1601_05904_b200/lib -laidw_b200 -Wl,-rpath,$PWD/paper_1601_05904_b200/lib
for i in 1 2; do /tmp/st/knn_stage_timing; done
for i in 1 2 3; do ./oracle/_ref/conformance/acceptance 2>&1 | grep -E "criterion  [678]"; done
