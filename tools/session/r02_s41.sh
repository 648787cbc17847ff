# r02 session 41: general-alpha queries on the tensor-core engine, MUFU exp2 share sweep (clustered)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V2=$(bash tools/build_variant.sh gm2 -DAIDW_TC_GMUFU=2)
V3=$(bash tools/build_variant.sh gm3 -DAIDW_TC_GMUFU=3)
for c in clustered; do
  echo "== $c simt general"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c tc general gm1"; AIDW_TC_GENERAL=1 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c tc general gm2"; AIDW_LIB_PATH=$V2 AIDW_TC_GENERAL=1 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
  echo "== $c tc general gm3"; AIDW_LIB_PATH=$V3 AIDW_TC_GENERAL=1 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120
done
