# r02 session 64: bench lines for every config on HEAD (managed stream, stream-ordered bench, e2e path)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_s64_1m.json 2> gpurun_out/bench_s64_1m.err; cut -c1-250 gpurun_out/bench_s64_1m.json
for c in 10k 100k clustered stress paper; do timeout 900 python bench.py --config $c --steps 10 --warmup 5 --no-fp64 > gpurun_out/bench_s64_$c.json 2> gpurun_out/bench_s64_$c.err; cut -c1-200 gpurun_out/bench_s64_$c.json; done
timeout 1200 python bench.py --config dem --steps 3 --warmup 3 --no-cpu-baseline --no-fp64 > gpurun_out/bench_s64_dem.json 2> gpurun_out/bench_s64_dem.err; cut -c1-200 gpurun_out/bench_s64_dem.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_s64_ref.json 2> gpurun_out/bench_s64_ref.err; cut -c1-200 gpurun_out/bench_s64_ref.json
