# r02 session 47: TC stage acquire / release variants — timing A/B (1M, twice) and racecheck
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
V0=$(bash tools/build_variant.sh a0r0 -DAIDW_TC_ACQ=0 -DAIDW_TC_RELEASE=0)
V1=$(bash tools/build_variant.sh a1r0 -DAIDW_TC_ACQ=1 -DAIDW_TC_RELEASE=0)
V2=$(bash tools/build_variant.sh a1r1 -DAIDW_TC_ACQ=1 -DAIDW_TC_RELEASE=1)
V3=$(bash tools/build_variant.sh a0r1 -DAIDW_TC_ACQ=0 -DAIDW_TC_RELEASE=1)
for rep in 1 2; do for v in $V0 $V1 $V2 $V3; do
  echo "== $(basename $(dirname $v))"; AIDW_LIB_PATH=$v timeout 300 python tools/profile_step.py --config 1m --passes 3 2>&1 | tail -1 | cut -c1-110
done; done
AIDW_LIB_PATH=$V3 timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_rc.txt 2>&1; echo "a0r1 racecheck rc $?"; tail -1 gpurun_out/san_rc.txt
