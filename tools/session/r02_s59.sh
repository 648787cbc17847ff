# r02 session 59: TC K4 chunk grouping as a separate kernel instantiation (ungrouped code unchanged)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
python tools/check_group_bits.py
for c in 100k 1m; do for g in 1 64; do echo "== $c group_max=$g"; AIDW_TC_GROUP_MAX=$g timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_vs_reference.py tests/test_multidevice.py -x -q -m gpu 2>&1 | tail -1
