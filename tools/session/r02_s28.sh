# r02 session 28: TC K4 — prefetched A centre; per-group MMA issuer warps (SPLITCTL=2) A/B; traces
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V2=$(bash tools/build_variant.sh sc2 -DAIDW_TC_SPLITCTL=2)
VT=$(bash tools/build_variant.sh sc2t -DAIDW_TC_SPLITCTL=2 -DAIDW_TC_TRACE=1)
V1T=$(bash tools/build_variant.sh sc1t -DAIDW_TC_TRACE=1)
for c in 1m 100k; do
  echo "== $c default"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c sc2"; AIDW_LIB_PATH=$V2 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
echo "== trace sc1"; AIDW_LIB_PATH=$V1T timeout 300 python tools/profile_step.py --config 1m --passes 1 2>&1 | grep -E "issuer|epi" | sort | uniq
echo "== trace sc2"; AIDW_LIB_PATH=$VT timeout 300 python tools/profile_step.py --config 1m --passes 1 2>&1 | grep -E "issuer|epi" | sort | uniq
