# r02 session 60: final verification on a fresh box — full GPU suite, smoke, default bench, clustered, 100K
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputests_s60.txt 2>&1; tail -3 gpurun_out/gputests_s60.txt
timeout 900 python bench.py > gpurun_out/bench_s60_1m.json 2> gpurun_out/bench_s60_1m.err; cut -c1-300 gpurun_out/bench_s60_1m.json
