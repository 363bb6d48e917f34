"""Run one GEMM of the layer (GPT-3 TP=1 shapes) `reps` times — a clean target for ncu.

    python tools/gemm_one.py fc1_fwd|fc2_fwd|qkv_fwd|fc1_dgrad|fc1_wgrad [reps]
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_11990_b200 import _native as N  # noqa: E402

h, M = 12288, 2048
SHAPES = {  # name: (m, n, k, a_mn, b_mn, epilogue)
    "qkv_fwd": (M, 3 * h, h, 0, 0, N.EPI_STORE_BF16),
    "fc1_fwd": (M, 4 * h, h, 0, 0, N.EPI_STORE_BF16),
    "fc2_fwd": (M, h, 4 * h, 0, 0, N.EPI_STORE_BF16),
    "fc1_dgrad": (M, h, 4 * h, 0, 1, N.EPI_STORE_BF16),
    "fc1_wgrad": (4 * h, h, M, 1, 1, N.EPI_STORE_F32),
    "fc1_wgrad_acc": (4 * h, h, M, 1, 1, N.EPI_ACCUM_F32),
    "proj_fwd": (M, h, h, 0, 0, N.EPI_STORE_BF16),
    # wgrad shape with the four operand-major combinations (K = tokens)
    "wg_kk_f32": (4 * h, h, M, 0, 0, N.EPI_STORE_F32),
    "wg_mm_f32": (4 * h, h, M, 1, 1, N.EPI_STORE_F32),
    "wg_mm_bf16": (4 * h, h, M, 1, 1, N.EPI_STORE_BF16),
    "wg_kk_bf16": (4 * h, h, M, 0, 0, N.EPI_STORE_BF16),
    "wg_km_bf16": (4 * h, h, M, 0, 1, N.EPI_STORE_BF16),
    "wg_mk_bf16": (4 * h, h, M, 1, 0, N.EPI_STORE_BF16),
    # the forward's shape class with the wgrad's short K (tile count 6x the forward's)
    "fwd_k2048": (M * 6, 4 * h, M, 0, 0, N.EPI_STORE_BF16),
    # GPT-3 h=12288 at TP=8 / TP=4 (per-GPU shard shapes)
    "g8_proj_fwd": (M, h, h // 8, 0, 0, N.EPI_STORE_BF16),
    "g4_proj_fwd": (M, h, h // 4, 0, 0, N.EPI_STORE_BF16),
    "g8_proj_dgrad": (M, h // 8, h, 0, 1, N.EPI_STORE_BF16),
    "g8_qkv_dgrad": (M, h, 3 * h // 8, 0, 1, N.EPI_STORE_BF16),
    "g8_fc1_dgrad": (M, h, h // 2, 0, 1, N.EPI_STORE_BF16),
    "g8_fc2_fwd": (M, h, h // 2, 0, 0, N.EPI_STORE_BF16),
    "fc2_fwd_g2": (M, h, 2 * h, 0, 0, N.EPI_STORE_BF16),
    "fc2_fwd_g4": (M, h, h, 0, 0, N.EPI_STORE_BF16),
    "fc1_dgrad_g2": (M, h, 2 * h, 0, 1, N.EPI_STORE_BF16),
    "qkv_dgrad_g4": (M, h, 3 * h // 4, 0, 1, N.EPI_STORE_BF16),
    "qkv_dgrad_g1": (M, h, 3 * h, 0, 1, N.EPI_STORE_BF16),
    "proj_fwd_g2": (M, h, h // 2, 0, 0, N.EPI_STORE_BF16),
    "proj_dgrad_g4": (M, h // 4, h, 0, 1, N.EPI_STORE_BF16),
    "qkv_wgrad_g8": (3 * h // 8, h, M, 1, 1, N.EPI_STORE_F32),
    "fc1_wgrad_g8": (h // 2, h, M, 1, 1, N.EPI_STORE_F32),
    "fc2_wgrad_g8": (h, h // 2, M, 1, 1, N.EPI_STORE_F32),
    "proj_wgrad_g8": (h, h // 8, M, 1, 1, N.EPI_STORE_F32),
    # MT-NLG h=20480 at TP=8 (per-GPU shard shapes)
    "mt_qkv_fwd": (M, 7680, 20480, 0, 0, N.EPI_STORE_BF16),
    "mt_proj_fwd": (M, 20480, 2560, 0, 0, N.EPI_STORE_BF16),
    "mt_fc1_fwd": (M, 10240, 20480, 0, 0, N.EPI_STORE_BF16),
    "mt_fc2_fwd": (M, 20480, 10240, 0, 0, N.EPI_STORE_BF16),
    "mt_fc1_wgrad": (10240, 20480, M, 1, 1, N.EPI_STORE_F32),
}
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m, n, k, amn, bmn, epi = SHAPES[name]
A = torch.randn((k, m) if amn else (m, k), device="cuda").bfloat16()
B = torch.randn((k, n) if bmn else (n, k), device="cuda").bfloat16()
D = torch.zeros(m, n, device="cuda", dtype=torch.float32 if epi >= 3 else torch.bfloat16)
a = N.GemmArgs()
a.a, a.b, a.d = A.data_ptr(), B.data_ptr(), D.data_ptr()
a.lda, a.ldb, a.ldd = (m if amn else k), (n if bmn else k), n
a.a_mn_major, a.b_mn_major = amn, bmn
a.m, a.n, a.k, a.batch, a.alpha, a.epilogue = m, n, k, 1, 1.0, epi
a.block_n = int(os.environ.get("MT_BN", "0"))
WS = \
    torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
a.workspace, a.workspace_bytes = WS.data_ptr(), WS.numel()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(reps):
    ev[0].record()
    assert N.lib().mt_gemm(C.byref(a), s) == 0
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{name} rep {i}: {ev[0].elapsed_time(ev[1])*1e3:.1f} us, {2*m*n*k/ev[0].elapsed_time(ev[1])/1e9:.0f} TFLOP/s")
