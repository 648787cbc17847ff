# r02 session 65: final verification — full GPU suite, smoke, default bench
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputests_s65.txt 2>&1; tail -3 gpurun_out/gputests_s65.txt
timeout 900 python bench.py > gpurun_out/bench_s65_1m.json 2> gpurun_out/bench_s65_1m.err; cut -c1-200 gpurun_out/bench_s65_1m.json
