#!/bin/bash
# A/B of GEMM variants on the same box. Usage: tools/gemm_ab.sh "ENV1" "ENV2" ... (each a set of env assignments)
SHAPES=${SHAPES:-"qkv_fwd fc1_fwd fc2_fwd proj_fwd fc1_dgrad fc1_wgrad mt_qkv_fwd mt_proj_fwd mt_fc1_fwd mt_fc2_fwd mt_fc1_wgrad"}
for cfg in "$@"; do
  echo "== $cfg"
  for g in $SHAPES; do env $cfg python tools/gemm_one.py $g 4 | tail -1; done
done
