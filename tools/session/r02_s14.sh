# r02 session 14: TC engine for recipe queries, CUDA-core K4 for general ones
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
rm -f gpurun_out/s14_prof.txt
for c in "1m" "clustered" "stress" "100k" "1m --general"; do echo "== $c" >> gpurun_out/s14_prof.txt; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-110 >> gpurun_out/s14_prof.txt; done
cat gpurun_out/s14_prof.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s14_tests.log 2>&1; tail -5 gpurun_out/s14_tests.log
