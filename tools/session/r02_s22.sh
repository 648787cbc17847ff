# r02 session 22: ncu --set full (source) of the TC K4 at HEAD, 1M x 1M
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:weight_tc -c 1 -o gpurun_out/k4tc_s22 python tools/profile_step.py --passes 1 > gpurun_out/ncu_s22.log 2>&1
tail -2 gpurun_out/ncu_s22.log
