# r02 session 62: the library's own stream kept per host thread (no per-call stream create/destroy); bench on a non-default stream
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
AIDW_HOST_TRACE=1 python tools/pass_trace.py 2>&1 | grep -E "pass\]" | tail -2
for c in 10k 100k; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-fp64 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['e2e'])"; done
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-fp64 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('1m', d['value'], d['ms_per_step'], d['e2e'])"
timeout 1200 python -m pytest tests/test_capi.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_multidevice.py tests/test_gpu_tc_engine.py tests/test_raster.py -x -q -m gpu 2>&1 | tail -1
