# r02 session 67: TC K4 with independent query groups — 2 CTAs per SM, 1 group each
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1=$(bash tools/build_variant.sh c2g1 -DAIDW_TC_CTAS=2 -DAIDW_TC_GROUPS=1)
V2=$(bash tools/build_variant.sh c2g1s3 -DAIDW_TC_CTAS=2 -DAIDW_TC_GROUPS=1 -DAIDW_TC_STAGES=3)
for c in 1m 100k; do
  echo "== $c default"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  for v in $V1 $V2; do echo "== $c $(basename $(dirname $v))"; AIDW_LIB_PATH=$v timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120; done
done
AIDW_LIB_PATH=$V1 timeout 900 python -m pytest tests/test_gpu_tc_engine.py -x -q -m gpu 2>&1 | tail -1
