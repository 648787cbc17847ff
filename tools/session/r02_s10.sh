# r02 session 10: TMEM load / epilogue-math microbenchmarks
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1601_05904_b200/csrc tools/tmem_bench.cu -o /tmp/tmem_bench
timeout 120 /tmp/tmem_bench > gpurun_out/tmem_bench.txt 2>&1; cat gpurun_out/tmem_bench.txt
