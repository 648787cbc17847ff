NL=$(python -c "import os,sys; p=[os.path.join(d,'include/cudnn_frontend/thirdparty/nlohmann') for d in sys.path if d]; print(next((q for q in p if os.path.exists(os.path.join(q,'json.hpp'))),''))")
mkdir -p /tmp/st && g++ -O2 -std=c++20 -ffp-contract=off -pthread -Iinclude -I$NL tools/stage_timing.cpp -o /tmp/st/stage_timing -Lpaper_1601_05904_b200/lib -laidw_b200 -Wl,-rpath,$PWD/paper_1601_05904_b200/lib
/tmp/st/stage_timing > gpurun_out/stage_timing.txt 2>&1
oracle/_ref/conformance/acceptance > gpurun_out/acc_fp32.txt 2>&1
AIDW_WEIGHT_FP64=1 oracle/_ref/conformance/acceptance > gpurun_out/acc_fp64.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_multidevice.py tests/test_conformance.py -q -m gpu -x > gpurun_out/t3.log 2>&1
tail -3 gpurun_out/t3.log; grep "criterion  [678]" gpurun_out/acc_fp32.txt gpurun_out/acc_fp64.txt; cat gpurun_out/stage_timing.txt
