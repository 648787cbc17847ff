# r02 session 52: 10K x 10K launch list on HEAD
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_10k_s52.csv python tools/profile_step.py --config 10k --passes 2 > /dev/null 2>&1
timeout 300 python tools/profile_step.py --config 10k --passes 5 2>&1 | tail -2
