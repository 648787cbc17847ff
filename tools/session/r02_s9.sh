# r02 session 9: tensor-core far-form prototype, launch shapes (MMA N, query groups, TMEM load width)
for cfg in "128 2 32 0" "128 2 128 1" "64 2 64 1" "64 4 64 1" "128 2 16 0"; do set -- $cfg
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DPROTO_N=$1 -DPROTO_GROUPS=$2 -DPROTO_C=$3 -DPROTO_SINGLE=$4 -I paper_1601_05904_b200/csrc tools/tc_proto.cu -o /tmp/tc_proto || continue
echo "N=$1 groups=$2 C=$3 single=$4" >> gpurun_out/tc9_shapes.txt
timeout 300 /tmp/tc_proto 303104 1024 | grep mode >> gpurun_out/tc9_shapes.txt 2>&1
done
cat gpurun_out/tc9_shapes.txt
