# r02 session 57: TC K4 with N = 32 parts: 4 query groups at 96 registers (16 epilogue warps), buffer depth
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1=$(bash tools/build_variant.sh g4n32b4 -DAIDW_TC_GROUPS=4 -DAIDW_TC_N=32 -DAIDW_TC_BUFS=4)
V2=$(bash tools/build_variant.sh g4n32b2 -DAIDW_TC_GROUPS=4 -DAIDW_TC_N=32 -DAIDW_TC_BUFS=2)
V3=$(bash tools/build_variant.sh g3n32b4 -DAIDW_TC_GROUPS=3 -DAIDW_TC_N=32 -DAIDW_TC_BUFS=4)
for c in 1m 100k; do
  echo "== $c default"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  for v in $V1 $V2 $V3; do echo "== $c $(basename $(dirname $v))"; AIDW_LIB_PATH=$v timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120; done
done
AIDW_LIB_PATH=$V1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -m gpu 2>&1 | tail -1
