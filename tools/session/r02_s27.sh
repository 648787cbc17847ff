# r02 session 27: TC K4 trace build — per-warp wait cycles of one CTA
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V=$(bash tools/build_variant.sh trace -DAIDW_TC_TRACE=1)
AIDW_LIB_PATH=$V timeout 300 python tools/profile_step.py --config 1m --passes 1 2>&1 | grep -E "issuer|epi" | sort | uniq | head -40
