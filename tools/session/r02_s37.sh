# r02 session 37: ladder of the acceptance gate with knn_stage phase traces
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
NL=$(python -c "import os,sys; p=[os.path.join(d,'include/cudnn_frontend/thirdparty/nlohmann') for d in sys.path if d]; print(next((q for q in p if os.path.exists(os.path.join(q,'json.hpp'))),''))")
mkdir -p /tmp/st
g++ -O2 -std=c++20 -ffp-contract=off -pthread -Iinclude -I$NL tools/ladder_timing.cpp -o /tmp/st/ladder -Lpaper_1601_05904_b200/lib -laidw_b200 -Wl,-rpath,$PWD/paper_1601_05904_b200/lib
for i in 1 2; do AIDW_HOST_TRACE=1 /tmp/st/ladder; done
