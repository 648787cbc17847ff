# r02 session 56: smoke(), the paper rung (1,024,000^2), 100K with the reference arm
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --config paper --steps 5 --warmup 3 --no-fp64 > gpurun_out/bench_s56_paper.json 2> gpurun_out/bench_s56_paper.err; cut -c1-220 gpurun_out/bench_s56_paper.json
timeout 900 python bench.py --config 100k --impl reference --steps 3 --warmup 1 > gpurun_out/bench_s56_100k_ref.json 2> gpurun_out/bench_s56_100k_ref.err; cut -c1-220 gpurun_out/bench_s56_100k_ref.json
timeout 900 python bench.py --config 10k --impl reference --steps 5 --warmup 2 > gpurun_out/bench_s56_10k_ref.json 2> gpurun_out/bench_s56_10k_ref.err; cut -c1-220 gpurun_out/bench_s56_10k_ref.json
