# r02 session 13: TC engine with per-group MMA warps + producer warp
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
rm -f gpurun_out/s13_prof.txt
for c in "1m" "1m --general" "clustered" "100k"; do echo "== $c tc" >> gpurun_out/s13_prof.txt; AIDW_K4_ENGINE=tc timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-120 >> gpurun_out/s13_prof.txt; done
cat gpurun_out/s13_prof.txt
AIDW_K4_ENGINE=tc timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q -m gpu 2>&1 | tail -2
