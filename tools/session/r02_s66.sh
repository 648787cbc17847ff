# r02 session 66: small-n bucket sort with its copies in shared memory
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_10k_s66.csv python tools/profile_step.py --config 10k --passes 2 > /dev/null 2>&1
grep bucket gpurun_out/launches_10k_s66.csv | awk -F'","' '{print $5, $NF}' | cut -c1-30,200- | tail -4
for c in 10k; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 2>/dev/null | cut -c1-190; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -m gpu 2>&1 | tail -1
