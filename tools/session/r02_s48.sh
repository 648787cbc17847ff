# r02 session 48: HEAD re-verification — full GPU suite, bench lines for every config, launch list, ncu of TC K4 and K2
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputests_s48.txt 2>&1; tail -3 gpurun_out/gputests_s48.txt
timeout 900 python bench.py > gpurun_out/bench_s48_1m.json 2> gpurun_out/bench_s48_1m.err; cut -c1-250 gpurun_out/bench_s48_1m.json
for c in 10k 100k clustered stress; do timeout 900 python bench.py --config $c --steps 10 --warmup 5 --no-fp64 > gpurun_out/bench_s48_$c.json 2> gpurun_out/bench_s48_$c.err; cut -c1-200 gpurun_out/bench_s48_$c.json; done
timeout 1200 python bench.py --config dem --steps 3 --warmup 3 --no-cpu-baseline --no-fp64 > gpurun_out/bench_s48_dem.json 2> gpurun_out/bench_s48_dem.err; cut -c1-200 gpurun_out/bench_s48_dem.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_s48_ref.json 2> gpurun_out/bench_s48_ref.err; cut -c1-300 gpurun_out/bench_s48_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_s48.csv python tools/profile_step.py --passes 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:weight_tc -c 1 -o gpurun_out/k4tc_r02_s48 python tools/profile_step.py --passes 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:knn_grid -c 1 -o gpurun_out/knn_r02_s48 python tools/profile_step.py --passes 1 > /dev/null 2>&1
ls gpurun_out/*s48*
