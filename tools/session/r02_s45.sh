# r02 session 45: epilogue warps acquire the stage's bulk copy (racecheck), timing
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for c in 1m 100k; do echo "== $c"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120; done
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc $?"; tail -2 gpurun_out/san_racecheck.txt
