nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DPROTO_N=64 -DPROTO_GROUPS=4 -I paper_1601_05904_b200/csrc tools/tc_proto.cu -o /tmp/tc_proto
timeout 600 ncu --set full --import-source on --clock-control none -k regex:far_tc -s 1 -c 1 -o gpurun_out/tcproto3 /tmp/tc_proto 151552 512 > gpurun_out/ncu_tcproto.log 2>&1
tail -3 gpurun_out/ncu_tcproto.log
