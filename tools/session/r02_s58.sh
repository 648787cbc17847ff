# r02 session 58: trace — share of the A-row rebuild in the tile tail
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
VT=$(bash tools/build_variant.sh trace -DAIDW_TC_TRACE=1)
AIDW_LIB_PATH=$VT timeout 300 python tools/profile_step.py --config 1m --passes 1 2>&1 | grep -E "issuer|epi" | sort | uniq
