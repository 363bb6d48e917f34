"""Diagnostic: fused GEMM+all-reduce vs NCCL outputs at TP=2 (rounding statistics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from tests.test_multigpu import _run

if __name__ == "__main__":
  res = _run("tp_fused")
  for k in ("y", "dx"):
    a, b = res[0][k + "1"].astype(np.float64), res[0][k + "0"].astype(np.float64)
    d = a != b
    print(k, "frac differing", d.mean(), "mean(|fused|-|nccl|) on differing", (np.abs(a[d]) - np.abs(b[d])).mean() if d.any() else 0,
          "frac toward zero", (np.abs(a[d]) < np.abs(b[d])).mean() if d.any() else 0)
