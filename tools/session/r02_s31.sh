# r02 session 31: ncu source capture of the TC K4 with the stage-record meta
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:weight_tc -c 1 -o gpurun_out/k4tc_s31 python tools/profile_step.py --passes 1 > gpurun_out/ncu_s31.log 2>&1
tail -1 gpurun_out/ncu_s31.log
