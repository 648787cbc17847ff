# r02 session 17: TC engine (recipe) + side-stream CUDA-core K4 (general); full GPU tests; bench lines
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
rm -f gpurun_out/s17_prof.txt
for c in "1m" "clustered" "stress" "100k"; do echo "== $c" >> gpurun_out/s17_prof.txt; timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-110 >> gpurun_out/s17_prof.txt; done
cat gpurun_out/s17_prof.txt
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/s17_tests.log 2>&1; tail -4 gpurun_out/s17_tests.log
timeout 600 python bench.py > gpurun_out/b17_1m.json 2> gpurun_out/b17_1m.err; cut -c1-400 gpurun_out/b17_1m.json
for c in 10k 100k clustered; do timeout 600 python bench.py --config $c --steps 10 --warmup 5 --no-cpu-baseline --no-fp64 > gpurun_out/b17_$c.json 2>gpurun_out/b17_$c.err; cut -c1-300 gpurun_out/b17_$c.json; done
