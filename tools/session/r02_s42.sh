# r02 session 42: K2 visits queries in block-major cell order (8x8-cell blocks)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for c in 1m clustered stress 100k 10k; do echo "== $c"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-175; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_vs_reference.py tests/test_gpu_at_scale.py tests/test_multidevice.py tests/test_raster.py -x -q -m gpu 2>&1 | tail -2
