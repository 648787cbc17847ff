# r02 session 46: racecheck of the TC stage release — lane-0 arrive vs every-lane arrive vs proxy fence
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V1=$(bash tools/build_variant.sh rel1 -DAIDW_TC_RELEASE=1)
V2=$(bash tools/build_variant.sh rel2 -DAIDW_TC_RELEASE=2)
for v in $V1 $V2; do
  echo "== $v"; AIDW_LIB_PATH=$v timeout 300 python tools/profile_step.py --config 1m --passes 2 2>&1 | tail -1 | cut -c1-120
  AIDW_LIB_PATH=$v timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_rc.txt 2>&1; echo "racecheck rc $?"; tail -1 gpurun_out/san_rc.txt
done
