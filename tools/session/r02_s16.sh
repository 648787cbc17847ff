rm -f gpurun_out/s16_acc.txt
for e in simt tc; do for i in 1 2; do echo "== $e" >> gpurun_out/s16_acc.txt; AIDW_K4_ENGINE=$e oracle/_ref/conformance/acceptance 2>&1 | grep "criterion  [678]" >> gpurun_out/s16_acc.txt; done; done
cat gpurun_out/s16_acc.txt
