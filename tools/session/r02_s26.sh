# r02 session 26: TC K4 — cost of the near passes incl. imbalance (debug build skips them)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1=$(bash tools/build_variant.sh nonear -DAIDW_TC_NONEAR_DEBUG=1)
V2=$(bash tools/build_variant.sh nonear_g4 -DAIDW_TC_NONEAR_DEBUG=1 -DAIDW_TC_ISSUE=1)
for c in 1m 100k; do
  echo "== $c default"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c nonear"; AIDW_LIB_PATH=$V1 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c nonear evloop"; AIDW_LIB_PATH=$V2 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
