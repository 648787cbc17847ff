# r02 session 51: TC K4 with 4 query groups (16 epilogue warps, 112 registers)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V=$(bash tools/build_variant.sh g4 -DAIDW_TC_GROUPS=4)
for c in 1m 100k stress; do
  echo "== $c default"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c g4"; AIDW_LIB_PATH=$V timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
AIDW_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -m gpu 2>&1 | tail -1
