"""Standalone rates of the TP=8 shard GEMMs whose tile count quantises badly (projection dgrad /
forward), per tile width: python tools/gemm_tp8_shapes.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_perf import run  # noqa: E402
import paper_2201_11990_b200._native as N  # noqa: E402

for bn in (0, 256, 192, 128):
    run(2048, 2560, 20480, b_mn=True, bn=bn, reps=8)    # MT-NLG TP=8 projection dgrad
    run(2048, 1536, 12288, b_mn=True, bn=bn, reps=8)    # GPT-3 TP=8 projection dgrad
    run(2048, 3072, 12288, b_mn=True, bn=bn, reps=8)    # GPT-3 TP=4 projection dgrad
    run(2048, 20480, 2560, bn=bn, reps=8)               # MT-NLG TP=8 projection forward
