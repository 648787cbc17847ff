# r02 session 44: compute-sanitizer incl. the tensor-core K4 and the K2 staging
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"; timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_$t.txt 2>&1; echo "rc $?"; tail -3 gpurun_out/san_$t.txt
done
