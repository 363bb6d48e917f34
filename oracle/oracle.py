"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's CPU legs).

ctypes wrapper of oracle/liblayer_oracle.so (the fp32 CPU restatement of the tensor-sliced layer,
layer_oracle.cpp) and of oracle/_ref/libcurator_ref.so (the reference's own planner, compiled from
/root/reference by oracle/Makefile). Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liblayer_oracle.so"
REF_LIB = HERE / "_ref" / "libcurator_ref.so"

PARAM_NAMES = ["ln1.gamma", "ln1.beta", "qkv.weight", "qkv.bias", "proj.weight", "proj.bias",
               "ln2.gamma", "ln2.beta", "fc1.weight", "fc1.bias", "fc2.weight", "fc2.bias"]
WEIGHTS = {2, 4, 8, 10}
GAMMAS = {0, 6}


class OrDesc(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("heads", C.c_int32), ("seq", C.c_int32), ("micro_batch", C.c_int32),
                ("tp_size", C.c_int32), ("ffn_mult", C.c_int32), ("dropout_hidden", C.c_float),
                ("dropout_attn", C.c_float), ("ln_eps", C.c_float), ("seed", C.c_uint64),
                ("layer_index", C.c_uint32), ("bf16_emulate", C.c_int32), ("shard_rank", C.c_int32)]


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        P = C.c_void_p
        L.or_layer_create.restype = P
        L.or_layer_create.argtypes = [C.POINTER(OrDesc), C.POINTER(C.POINTER(C.c_float))]
        L.or_layer_destroy.argtypes = [P]
        L.or_layer_forward.argtypes = [P, P, P, C.c_uint32]
        L.or_layer_backward.argtypes = [P, P, P, C.c_uint32, C.POINTER(C.POINTER(C.c_float))]
        L.or_fill_normal.argtypes = [P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                     C.c_float, C.c_float, C.c_int32]
        L.or_site_seed.restype = C.c_uint64
        L.or_site_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint32, C.c_uint32]
        L.or_step_seed.restype = C.c_uint64
        L.or_step_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_dropout_keep.restype = C.c_int32
        L.or_dropout_keep.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32]
        L.or_mse_loss.argtypes = [P, P, P, P, C.c_int64]
        L.or_num_threads.restype = C.c_int
        _lib = L
    return _lib


def param_shapes(hidden: int, ffn_mult: int = 4) -> list[tuple[int, int]]:
    h, ff = hidden, ffn_mult * hidden
    return [(1, h), (1, h), (3 * h, h), (1, 3 * h), (h, h), (1, h), (1, h), (1, h), (ff, h), (1, ff), (h, ff), (1, h)]


def site_seed(seed: int, name: str, layer: int = 0, mb: int = 0) -> int:
    return int(lib().or_site_seed(seed, name.encode(), layer, mb))


def step_seed(seed: int, step: int) -> int:
    """Dropout seed of training step `step` (curator::step_seed: the base seed at step 0)."""
    return int(lib().or_step_seed(seed, step))


def normal(key: int, rows: int, cols: int, mean=0.0, std=1.0, round_bf16=True) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float32)
    lib().or_fill_normal(out.ctypes.data, rows, cols, cols, 0, 0, key, mean, std, int(round_bf16))
    return out


def shard_region(i: int, hidden: int, heads: int, tp: int, rank: int, ffn_mult: int = 4):
    """(row0, col0, rows, cols) of TP shard `rank` of parameter i in the global tensor (Megatron layout,
    include/curator/schedule.hpp layer_shard: QKV / fc1 rows, attn-out / fc2 columns; the rest replicated)."""
    h, ff = hidden, ffn_mult * hidden
    r, c = param_shapes(hidden, ffn_mult)[i]
    if i == 2:
        return rank * 3 * h // tp, 0, 3 * h // tp, h
    if i == 3:
        return 0, rank * 3 * h // tp, 1, 3 * h // tp
    if i == 4:
        return 0, rank * h // tp, h, h // tp
    if i == 8:
        return rank * ff // tp, 0, ff // tp, h
    if i == 9:
        return 0, rank * ff // tp, 1, ff // tp
    if i == 10:
        return 0, rank * ff // tp, h, ff // tp
    return 0, 0, r, c


def init_params(hidden: int, seed: int, layer: int, ffn_mult: int = 4, shard=None) -> list[np.ndarray]:
    """The global (unsharded) parameters of one layer, as the GPU's mt_layer_init_params draws them
    (bf16-representable float32). shard = (heads, tp, rank): only that TP shard's region of each
    sharded tensor is drawn, the rest stays zero (enough for the oracle's shard mode; a large layer's
    full draw is minutes of host time)."""
    std_w = float(np.sqrt(1.0 / (3.0 * hidden)))
    out = []
    for i, (r, c) in enumerate(param_shapes(hidden, ffn_mult)):
        mean = 1.0 if i in GAMMAS else 0.0
        std = std_w if i in WEIGHTS else 0.02
        key = site_seed(seed, PARAM_NAMES[i], layer, 0)
        if shard is None:
            out.append(normal(key, r, c, mean, std))
            continue
        a = np.zeros((r, c), np.float32)
        r0, c0, nr, nc = shard_region(i, hidden, shard[0], shard[1], shard[2], ffn_mult)
        blk = np.empty((nr, nc), np.float32)
        lib().or_fill_normal(blk.ctypes.data, nr, nc, c, r0, c0, key, mean, std, 1)
        a[r0:r0 + nr, c0:c0 + nc] = blk
        out.append(a)
    return out


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 (bf16-representable or not) -> uint16 bf16 bits, round-to-nearest-even."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


class OracleLayer:
    """One layer of the CPU restatement. Global (unsharded) parameters; tp_size only changes where
    partial sums are rounded and summed (the emulated all-reduce). shard_rank >= 0 computes only
    that TP shard with no all-reduce (the runtime's shard-only mode, bench.py --shard-of); gradients
    then cover only that shard's slices of the sharded parameters."""

    def __init__(self, hidden, heads, seq, micro_batch=1, tp_size=1, ffn_mult=4, dropout_hidden=0.0,
                 dropout_attn=0.0, ln_eps=1e-5, seed=20260808, layer_index=0, bf16_emulate=True, params=None,
                 shard_rank=-1):
        self.desc = OrDesc(hidden, heads, seq, micro_batch, tp_size, ffn_mult, dropout_hidden, dropout_attn, ln_eps,
                           seed, layer_index, int(bf16_emulate), shard_rank)
        self.hidden, self.M = hidden, micro_batch * seq
        # the native object keeps raw pointers into these arrays (no copy): they live as long as self
        self.params = [np.ascontiguousarray(p, dtype=np.float32) for p in
                       (params if params is not None else init_params(hidden, seed, layer_index, ffn_mult))]
        ptrs = (C.POINTER(C.c_float) * 12)(*[p.ctypes.data_as(C.POINTER(C.c_float)) for p in self.params])
        self._h = lib().or_layer_create(C.byref(self.desc), ptrs)
        self.grads = [np.zeros_like(p) for p in self.params]

    def forward(self, x: np.ndarray, mb: int = 0) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float32).reshape(self.M, self.hidden)
        y = np.empty_like(x)
        lib().or_layer_forward(self._h, x.ctypes.data, y.ctypes.data, mb)
        return y

    def backward(self, dy: np.ndarray, mb: int = 0) -> np.ndarray:
        dy = np.ascontiguousarray(dy, dtype=np.float32).reshape(self.M, self.hidden)
        dx = np.empty_like(dy)
        ptrs = (C.POINTER(C.c_float) * 12)(*[g.ctypes.data_as(C.POINTER(C.c_float)) for g in self.grads])
        lib().or_layer_backward(self._h, dy.ctypes.data, dx.ctypes.data, mb, ptrs)
        return dx

    def __del__(self):
        try:
            lib().or_layer_destroy(self._h)
        except Exception:
            pass


def mse_loss(y: np.ndarray, t: np.ndarray):
    y = np.ascontiguousarray(y, dtype=np.float32)
    t = np.ascontiguousarray(t, dtype=np.float32)
    dy = np.empty_like(y)
    loss = np.zeros(1, dtype=np.float32)
    lib().or_mse_loss(y.ctypes.data, t.ctypes.data, dy.ctypes.data, loss.ctypes.data, y.size)
    return float(loss[0]), dy


def num_threads() -> int:
    return int(lib().or_num_threads())


def ref_lib():
    """The reference planner (oracle/_ref/libcurator_ref.so) or None when it was not built."""
    if not REF_LIB.exists():
        return None
    return C.CDLL(str(REF_LIB))
