# r02 session 24: TC K4 — producer warp (refills) + lockstep issuer / per-group issuer with backoff
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1=$(bash tools/build_variant.sh evloop -DAIDW_TC_ISSUE=1)
for c in 1m 100k; do
  echo "== $c lockstep+producer"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c evloop+sleep"; AIDW_LIB_PATH=$V1 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
