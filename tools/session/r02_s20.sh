# r02 session 20: TC engine variants (split TMEM load, groups) + fixed math microbenchmark
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
rm -f gpurun_out/s20_prof.txt
run() {
  for c in "1m"; do echo "== $1 $c" >> gpurun_out/s20_prof.txt; AIDW_LIB_PATH=$2 timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-110 >> gpurun_out/s20_prof.txt; done
}
run base paper_1601_05904_b200/lib/libaidw_b200.so
for v in "split -DAIDW_TC_SPLITLD=1" "g4 -DAIDW_TC_GROUPS=4" "g2 -DAIDW_TC_GROUPS=2"; do set -- $v
  lib=$(bash tools/build_variant.sh $@) && run $1 $lib
done
cat gpurun_out/s20_prof.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1601_05904_b200/csrc tools/tmem_bench.cu -o /tmp/tmem_bench && timeout 120 /tmp/tmem_bench > gpurun_out/tmem_bench.txt 2>&1; grep -E "math|both" gpurun_out/tmem_bench.txt
