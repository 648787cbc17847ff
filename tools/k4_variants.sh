#!/bin/bash
# Time every K4 variant on the 1M x 1M bench config (uniform: alpha=4 recipe
# heavy; --general: every query on exp2/log2).  Prints weight_kernel_ms.
for v in ${VARIANTS:-0 1 2 3 4}; do
  for g in "" "--general"; do
    ms=$(AIDW_K4_VARIANT=$v python tools/profile_step.py --passes 3 $g | tail -1 | python -c "import sys,ast; print(ast.literal_eval(sys.stdin.read())['weight_kernel_ms'])")
    echo "variant $v ${g:-recipe}: K4 $ms ms"
  done
done
