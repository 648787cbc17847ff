# r02 session 19: small-shape latency (locality sorts skipped at small n, settle loads in flight)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for v in 65536; do AIDW_SMALL_SORT_N=$v timeout 600 python bench.py --config 10k --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b19_10k_$v.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b19_10k_$v.json').read().strip().splitlines()[-1]); print('sortn=$v', d['ms_per_step'], d['e2e']['value'], d['stages'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_10k_s19.csv python tools/profile_step.py --config 10k --passes 2 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_multidevice.py -x -q -m gpu 2>&1 | tail -2
