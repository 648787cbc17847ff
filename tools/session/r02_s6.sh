# r02 session 6: graph cache A/B at 10K, general-alpha per-point split A/B, launch list
python -m pytest tests/test_gpu_edge.py -q -m gpu -k "graph or slab" > gpurun_out/t6.log 2>&1
python bench.py --config 10k --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b6_10k.json 2>&1
AIDW_GRAPHS=0 python bench.py --config 10k --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b6_10k_nograph.json 2>&1
for v in "" "AIDW_K4_G2=0.5"; do
  echo "== $v clustered" >> gpurun_out/k4_general_ab.txt
  env $v python tools/profile_step.py --config clustered --passes 3 >> gpurun_out/k4_general_ab.txt 2>&1
  echo "== $v 1m --general" >> gpurun_out/k4_general_ab.txt
  env $v python tools/profile_step.py --config 1m --passes 3 --general >> gpurun_out/k4_general_ab.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_10k.csv python tools/profile_step.py --config 10k --passes 4 > /dev/null 2>&1
tail -3 gpurun_out/t6.log; grep -o '"weight_kernel_ms": [0-9.]*' gpurun_out/k4_general_ab.txt
