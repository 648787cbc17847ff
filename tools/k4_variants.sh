#!/bin/bash
# Time the K4 launch shapes on the 1M x 1M bench config (uniform: alpha=4
# recipe heavy; --general: every query on exp2/log2).  AIDW_K4_VARIANT:
#   0 = automatic (4 queries / thread x 2 CTAs per SM, or 2 x 4 for small n)
#   1 = 4 x 3 (80 registers, spills)   2 = 2 x 4   3 = 4 x 2 forced   4 = 2 x 3
# Build-time knobs (tools/build_variant.sh): AIDW_K4_THREADS, AIDW_K4_MINB,
# AIDW_K4_STAGES, AIDW_K4_FAR_UNROLL.  Prints weight_kernel_ms.
for v in ${VARIANTS:-0 1 2 3 4}; do
  for g in "" "--general"; do
    ms=$(AIDW_K4_VARIANT=$v python tools/profile_step.py --passes 3 $g | tail -1 | python -c "import sys,ast; print(ast.literal_eval(sys.stdin.read())['weight_kernel_ms'])")
    echo "variant $v ${g:-recipe}: K4 $ms ms"
  done
done
