# r02 session 63: e2e path — uploads event-timed (no mid-call sync), results + failure flags behind one sync
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for c in 10k 100k; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --e2e-steps 20 --no-cpu-baseline --no-fp64 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['e2e'])"; done
timeout 1200 python -m pytest tests/test_capi.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_multidevice.py tests/test_gpu_tc_engine.py tests/test_raster.py tests/test_gpu_vs_reference.py -x -q -m gpu 2>&1 | tail -1
