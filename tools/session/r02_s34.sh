# r02 session 34: K1 two points per thread (double2 loads); DEM kNN in full; RCP microbenchmark fixed
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
./tools/microbench_pipes.bin > gpurun_out/microbench_pipes_s34.txt 2>&1; cat gpurun_out/microbench_pipes_s34.txt
for c in 1m 10k; do echo "== $c"; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-160; done
/usr/bin/time -v timeout 1800 python -m pytest tests/test_gpu_at_scale.py -x -q -m gpu -k dem_knn > gpurun_out/dem_knn_s34.txt 2>&1; grep -E "passed|failed|Maximum resident|Elapsed" gpurun_out/dem_knn_s34.txt
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/gputests_s34.txt 2>&1; tail -2 gpurun_out/gputests_s34.txt
