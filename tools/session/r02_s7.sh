# r02 session 7: device value hull (no pre-pass sync), fused class scans, CTA tile_geo, galloping level search
NL=$(python -c "import os,sys; p=[os.path.join(d,'include/cudnn_frontend/thirdparty/nlohmann') for d in sys.path if d]; print(next((q for q in p if os.path.exists(os.path.join(q,'json.hpp'))),''))")
mkdir -p /tmp/st
g++ -O2 -std=c++20 -ffp-contract=off -pthread -Iinclude -I$NL tools/knn_stage_timing.cpp -o /tmp/st/kst -Lpaper_1601_05904_b200/lib -laidw_b200 -Wl,-rpath,$PWD/paper_1601_05904_b200/lib
/tmp/st/kst > gpurun_out/knn_stage_timing7.txt 2>&1
oracle/_ref/conformance/acceptance > gpurun_out/acc7_fp32.txt 2>&1
AIDW_WEIGHT_FP64=1 oracle/_ref/conformance/acceptance > gpurun_out/acc7_fp64.txt 2>&1
python -m pytest tests -q -m gpu -x > gpurun_out/t7.log 2>&1
for c in 10k 100k stress; do python bench.py --config $c --steps 10 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b7_$c.json 2>&1; done
cat /sys/kernel/mm/transparent_hugepage/enabled > gpurun_out/thp.txt 2>&1; nproc >> gpurun_out/thp.txt
tail -3 gpurun_out/t7.log; cat gpurun_out/knn_stage_timing7.txt; grep "criterion  [678]" gpurun_out/acc7*.txt
