# r02 session 15: TC general-alpha exp2 split A/B (all classes on TC), acceptance timing variance
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
rm -f gpurun_out/s15_prof.txt
run() {  # name lib
  for c in "1m --general" "clustered"; do echo "== $1 $c" >> gpurun_out/s15_prof.txt; AIDW_TC_GENERAL=1 AIDW_LIB_PATH=$2 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-110 >> gpurun_out/s15_prof.txt; done
}
run g1 paper_1601_05904_b200/lib/libaidw_b200.so
for v in "g2 -DAIDW_TC_GMUFU=2" "g3 -DAIDW_TC_GMUFU=3" "g0 -DAIDW_TC_GMUFU=0"; do set -- $v
  lib=$(bash tools/build_variant.sh $@) && run $1 $lib
done
cat gpurun_out/s15_prof.txt
for i in 1 2 3; do oracle/_ref/conformance/acceptance 2>&1 | grep "criterion  [678]" >> gpurun_out/s15_acc.txt; done
cat gpurun_out/s15_acc.txt
