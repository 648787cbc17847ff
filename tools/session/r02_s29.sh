# r02 session 29: TC K4 — tile box / geo in the stage records (no global loads in the tile loop)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1T=$(bash tools/build_variant.sh sc1t -DAIDW_TC_TRACE=1)
for c in 1m 100k; do
  echo "== $c default"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
echo "== trace sc1"; AIDW_LIB_PATH=$V1T timeout 300 python tools/profile_step.py --config 1m --passes 1 2>&1 | grep -E "issuer|epi" | sort | uniq
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_vs_reference.py -x -q -m gpu 2>&1 | tail -2
