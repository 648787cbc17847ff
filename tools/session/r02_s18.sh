# r02 session 18: launch list + ncu --set full of the TC K4 (split engines), default bench
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_s18.csv python tools/profile_step.py --passes 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:weight_tc -c 1 -o gpurun_out/k4tc_r02_s18 python tools/profile_step.py --passes 1 > gpurun_out/ncu_s18.log 2>&1
tail -1 gpurun_out/ncu_s18.log
timeout 600 python bench.py > gpurun_out/b18_1m.json 2> gpurun_out/b18_1m.err; cut -c1-300 gpurun_out/b18_1m.json
