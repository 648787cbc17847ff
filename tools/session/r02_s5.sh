# r02 session 5: graph cache + mirror + pooled materialisation
NL=$(python -c "import os,sys; p=[os.path.join(d,'include/cudnn_frontend/thirdparty/nlohmann') for d in sys.path if d]; print(next((q for q in p if os.path.exists(os.path.join(q,'json.hpp'))),''))")
mkdir -p /tmp/st
for t in stage_timing knn_stage_timing; do
  g++ -O2 -std=c++20 -ffp-contract=off -pthread -Iinclude -I$NL tools/$t.cpp -o /tmp/st/$t -Lpaper_1601_05904_b200/lib -laidw_b200 -Wl,-rpath,$PWD/paper_1601_05904_b200/lib
done
/tmp/st/knn_stage_timing > gpurun_out/knn_stage_timing.txt 2>&1
oracle/_ref/conformance/acceptance > gpurun_out/acc_fp32.txt 2>&1
AIDW_WEIGHT_FP64=1 oracle/_ref/conformance/acceptance > gpurun_out/acc_fp64.txt 2>&1
python bench.py --config 10k --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b5_10k.json 2>&1
python bench.py --config 100k --steps 10 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b5_100k.json 2>&1
python -m pytest tests -q -m gpu > gpurun_out/t5.log 2>&1
tail -3 gpurun_out/t5.log; cat gpurun_out/knn_stage_timing.txt; grep "criterion  [678]" gpurun_out/acc*.txt
