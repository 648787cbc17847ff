# r02 session 12: first run of the tensor-core K4 engine (weight_tc.cu)
set -x
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
export AIDW_K4_ENGINE=tc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s12_smoke.txt 2>&1
cat gpurun_out/s12_smoke.txt | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vs_reference.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/s12_tc_tests.log 2>&1
tail -15 gpurun_out/s12_tc_tests.log
for c in 1m 100k clustered; do
  for e in tc simt; do echo "== $c $e" >> gpurun_out/s12_prof.txt; AIDW_K4_ENGINE=$e timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 >> gpurun_out/s12_prof.txt; done
done
for e in tc simt; do echo "== 1m general $e" >> gpurun_out/s12_prof.txt; AIDW_K4_ENGINE=$e timeout 300 python tools/profile_step.py --config 1m --general --passes 3 2>&1 | tail -1 >> gpurun_out/s12_prof.txt; done
cat gpurun_out/s12_prof.txt
for c in 1m clustered; do AIDW_K4_ENGINE=tc timeout 600 python tests/accuracy_study.py --config $c --sample 2048 >> gpurun_out/s12_acc.txt 2>&1; done
AIDW_K4_ENGINE=tc timeout 600 python tests/accuracy_study.py --config 1m --general --sample 2048 >> gpurun_out/s12_acc.txt 2>&1
cat gpurun_out/s12_acc.txt
