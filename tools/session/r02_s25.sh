# r02 session 25: TC K4 — mbarrier waits with a suspend-time hint (A/B)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1=$(bash tools/build_variant.sh nosleep -DAIDW_TC_SLEEP=0)
V2=$(bash tools/build_variant.sh ctl1sleep -DAIDW_TC_SPLITCTL=0)
for c in 1m 100k; do
  echo "== $c split+sleep"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c split nosleep"; AIDW_LIB_PATH=$V1 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c ctl1+sleep"; AIDW_LIB_PATH=$V2 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
