# r02 session 32: TC K4 A/B — record meta x sleeping waits
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1=$(bash tools/build_variant.sh m1s0 -DAIDW_TC_SLEEP=0)
V2=$(bash tools/build_variant.sh m0s1 -DAIDW_TC_META=0)
V3=$(bash tools/build_variant.sh m0s0 -DAIDW_TC_META=0 -DAIDW_TC_SLEEP=0)
for c in 1m; do
  echo "== $c meta sleep"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  for v in $V1 $V2 $V3; do echo "== $c $v"; AIDW_LIB_PATH=$v timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120; done
done
