import os, sys
sys.path.insert(0, "tools")
from gemm_perf import run
for bn in (0, 160, 192):
    run(2048, 2560, 20480, b_mn=True, bn=bn, reps=8)
    run(2048, 2560, 20480, b_mn=False, bn=bn, reps=8)
