# r02 session 35: DEM kNN in full; full GPU suite (conformance last)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
free -g | head -2
start=$(date +%s); timeout 1800 python -m pytest tests/test_gpu_at_scale.py -q -m gpu -k dem_knn > gpurun_out/dem_knn_s35.txt 2>&1; echo "dem knn $(( $(date +%s) - start )) s"; tail -3 gpurun_out/dem_knn_s35.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputests_s35.txt 2>&1; tail -3 gpurun_out/gputests_s35.txt
