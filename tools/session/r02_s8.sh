# r02 session 8: re-verify HEAD on the GPU (tests, default bench, configs, launch list, K4 full capture)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s8_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/t8.log 2>&1
tail -3 gpurun_out/t8.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke8.txt 2>&1
timeout 600 python bench.py > gpurun_out/b8_1m.json 2>gpurun_out/b8_1m.err
for c in 10k 100k clustered stress; do timeout 600 python bench.py --config $c --steps 10 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b8_$c.json 2>gpurun_out/b8_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/b8_ref.json 2>gpurun_out/b8_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_s8.csv python tools/profile_step.py --passes 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:weight_fp32 -c 1 -o gpurun_out/k4_r02_s8 python tools/profile_step.py --passes 1 > gpurun_out/ncu_k4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_grid -c 1 -o gpurun_out/knn_r02_s8 python tools/profile_step.py --passes 1 > gpurun_out/ncu_knn.log 2>&1
cat gpurun_out/b8_*.json | cut -c1-300
