# r02 session 21: O(1) block counts (summed-area table) in K2
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
rm -f gpurun_out/s21_prof.txt
for c in "stress" "1m" "clustered" "10k"; do echo "== $c" >> gpurun_out/s21_prof.txt; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/s21_prof.txt; done
cat gpurun_out/s21_prof.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_at_scale.py -x -q -m gpu -k "knn" 2>&1 | tail -2
