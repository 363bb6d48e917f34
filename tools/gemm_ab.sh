#!/bin/bash
# A/B of the 1-CTA and 2-CTA GEMM paths on the same box (interleaved to cancel clock drift).
for i in 1 2; do
  for pair in 0 1; do
    echo "== MT_GEMM_PAIR=$pair"
    for g in qkv_fwd fc1_fwd fc2_fwd fc1_dgrad fc1_wgrad; do MT_GEMM_PAIR=$pair python tools/gemm_one.py $g 4 | tail -1; done
  done
done
