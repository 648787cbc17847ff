# r02 session 23: TC K4 — producer warp + non-blocking per-group MMA issuer (A/B vs one control thread)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V0=$(bash tools/build_variant.sh ctl1 -DAIDW_TC_SPLITCTL=0)
for c in 1m clustered 100k; do
  echo "== $c split"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-200
  echo "== $c ctl1"; AIDW_LIB_PATH=$V0 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-200
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_vs_reference.py -x -q -m gpu 2>&1 | tail -2
