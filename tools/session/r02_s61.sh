# r02 session 61: result stash as whole prebuilt vectors of n and 2n results (O(1) take)
make -C paper_1601_05904_b200/csrc -j8 > /dev/null 2>&1
for i in 1 2 3; do AIDW_HOST_TRACE=1 ./oracle/_ref/conformance/acceptance 2>&1 | grep -E "knn_stage\] n (102400|51200)|criterion  [78]"; done
for i in 1 2 3; do AIDW_HOST_TRACE=1 AIDW_WEIGHT_FP64=1 ./oracle/_ref/conformance/acceptance 2>&1 | grep -E "knn_stage\] n (102400|51200)|criterion  [78]"; done
timeout 1200 python -m pytest tests/test_conformance.py -q -m gpu 2>&1 | tail -2
