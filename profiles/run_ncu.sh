#!/bin/bash
# Reproduce the committed ncu evidence (run on the GPU box via gpurun).
#   launches_<tag>.csv : every kernel of one fused 1M x 1M pipeline pass
#                        (gpu__time_duration, --clock-control none)
#   k4_<tag>.ncu-rep   : --set full capture of the dominant kernel (K4)
#   knn_<tag>.ncu-rep  : --set full capture of K2 (grid kNN + alpha)
set -e
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv python tools/profile_step.py --passes 1
ncu --set full --clock-control none --import-source on -k regex:weight_fp32 -c 1 \
    -o $OUT/k4_$TAG python tools/profile_step.py --passes 1
ncu --set full --clock-control none --import-source on -k regex:weight_fp32 -c 1 \
    -o $OUT/k4gen_$TAG python tools/profile_step.py --passes 1 --general
ncu --set full --clock-control none --import-source on -k regex:knn_grid -c 1 \
    -o $OUT/knn_$TAG python tools/profile_step.py --passes 1
