# r02 session 43: K2 shared-memory staging of the CTA's cell patch (A/B: AIDW_K2_STAGE=0)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for c in 1m clustered stress 100k 10k; do
  for st in 1 0; do echo "== $c stage=$st"; AIDW_K2_STAGE=$st timeout 300 python tools/profile_step.py --config $c --passes 3 2>&1 | tail -1 | cut -c1-175; done
done
for st in 1 0; do echo "== dem stage=$st"; AIDW_K2_STAGE=$st timeout 300 python tools/profile_step.py --config dem --passes 2 2>&1 | tail -1 | cut -c1-175; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_vs_reference.py tests/test_gpu_at_scale.py tests/test_multidevice.py tests/test_raster.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -2
