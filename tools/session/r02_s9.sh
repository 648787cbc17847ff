# r02 session 9: tensor-core far-form prototype: control warps (2 / 1), groups, MMA N; n = 148 CTAs x waves
for cfg in "64 4 2 296" "64 4 1 296" "64 3 1 384" "128 2 1 592" "128 2 2 592"; do set -- $cfg
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DPROTO_N=$1 -DPROTO_GROUPS=$2 -DPROTO_CTRL=$3 -DPROTO_SINGLE=1 -I paper_1601_05904_b200/csrc tools/tc_proto.cu -o /tmp/tc_proto || continue
echo "N=$1 groups=$2 ctrl=$3" >> gpurun_out/tc9_shapes.txt
timeout 300 /tmp/tc_proto $(( $4 * 1024 )) 1024 | grep mode >> gpurun_out/tc9_shapes.txt 2>&1
done
cat gpurun_out/tc9_shapes.txt
