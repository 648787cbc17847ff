# r02 session 33: TC K4 — whole-warp MMA issuer (uniform descriptors, elected lane)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
VT=$(bash tools/build_variant.sh trace -DAIDW_TC_TRACE=1)
for c in 1m 100k clustered; do
  echo "== $c"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
echo "== trace"; AIDW_LIB_PATH=$VT timeout 300 python tools/profile_step.py --config 1m --passes 1 2>&1 | grep -E "issuer|epi" | sort | uniq
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_vs_reference.py -x -q -m gpu 2>&1 | tail -2
