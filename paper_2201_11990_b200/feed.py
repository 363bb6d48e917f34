"""Blend-driven data feed over the native C ABI (include/mtnlg.h, csrc/feed.cpp).

`Blend` mirrors curator::BlendState + next_batch_composition (reference proj/src/blending.cpp),
`blend_manifest` the reference blend stage (proj/src/pipeline.cpp:551-647) writing
blend_manifest.jsonl, and `Feed` turns such a manifest into this data-parallel rank's int32 token
microbatches for `Stage.train_step` after `Stage.attach_vocab`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._native import FeedDesc, check, lib
from .planner import stream_key


def stage_seed(config_seed: int, stage: str = "blend") -> int:
    """The reference pipeline's per-stage seed mix64(seed, fnv1a64(stage)) (pipeline.cpp:708-711)."""
    return stream_key(config_seed, stage, 0, 0)


def _names(names):
    arr = (C.c_char_p * len(names))(*[n.encode() for n in names])
    return arr


class Blend:
    def __init__(self, names, weights, available=None, normalize=False):
        self.n = len(names)
        self._names = _names(names)
        w = np.ascontiguousarray(weights, np.float64)
        av = None if available is None else np.ascontiguousarray(available, np.uint64)
        self._h = C.c_void_p()
        check(lib().mt_blend_create(self.n, self._names, w.ctypes.data_as(C.POINTER(C.c_double)),
                                    None if av is None else av.ctypes.data_as(C.POINTER(C.c_uint64)), int(normalize),
                                    C.byref(self._h)))

    def weights(self) -> np.ndarray:
        w = np.empty(self.n, np.float64)
        check(lib().mt_blend_weights(self._h, w.ctypes.data_as(C.POINTER(C.c_double))))
        return w

    def next(self, batch_size: int):
        """(counts, credit, drawn) after drawing one batch."""
        c, cr, d = np.empty(self.n, np.uint64), np.empty(self.n, np.float64), np.empty(self.n, np.uint64)
        check(lib().mt_blend_next(self._h, batch_size, c.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  cr.ctypes.data_as(C.POINTER(C.c_double)), d.ctypes.data_as(C.POINTER(C.c_uint64))))
        return c, cr, d

    def close(self):
        if self._h:
            lib().mt_blend_destroy(self._h)
            self._h = C.c_void_p()


def blend_manifest(path, datasets, steps, batch_size, shuffle=False, config_seed=0, batch_per_step=None):
    """datasets: [(name, weight, doc_ids)] in config order; writes the reference's blend_manifest.jsonl."""
    names = _names([d[0] for d in datasets])
    w = np.ascontiguousarray([d[1] for d in datasets], np.float64)
    ids = [np.ascontiguousarray(d[2], np.uint64) for d in datasets]
    ptrs = (C.POINTER(C.c_uint64) * len(ids))(*[a.ctypes.data_as(C.POINTER(C.c_uint64)) for a in ids])
    counts = np.ascontiguousarray([len(a) for a in ids], np.uint64)
    bps = None
    if batch_per_step is not None:
        bps = np.ascontiguousarray(batch_per_step, np.uint64)
        assert len(bps) >= steps
    check(lib().mt_blend_manifest(len(datasets), names, w.ctypes.data_as(C.POINTER(C.c_double)), ptrs,
                                  counts.ctypes.data_as(C.POINTER(C.c_uint64)), steps, batch_size,
                                  None if bps is None else bps.ctypes.data_as(C.POINTER(C.c_uint64)), int(shuffle),
                                  stage_seed(config_seed), str(path).encode()))


def doc_tokens(seed: int, dataset: str, doc_id: int, vocab: int, n: int) -> np.ndarray:
    out = np.empty(n, np.int32)
    check(lib().mt_feed_doc_tokens(seed, dataset.encode(), doc_id, vocab, n, out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


class Feed:
    def __init__(self, manifest_path, vocab, seq, micro_batch, data_parallel=1, dp_rank=0, seed=0):
        self.desc = FeedDesc(vocab, seq, micro_batch, data_parallel, dp_rank, seed)
        self._h = C.c_void_p()
        check(lib().mt_feed_open(str(manifest_path).encode(), C.byref(self.desc), C.byref(self._h)))

    def steps(self) -> int:
        n = C.c_int64()
        check(lib().mt_feed_steps(self._h, C.byref(n)))
        return n.value

    def dataset_name(self, i: int) -> str:
        p = C.c_char_p()
        check(lib().mt_feed_dataset_name(self._h, i, C.byref(p)))
        return p.value.decode()

    def step_info(self, step: int) -> tuple[int, int]:
        """(global batch, this rank's microbatches)."""
        g, m = C.c_int64(), C.c_int32()
        check(lib().mt_feed_step_info(self._h, step, C.byref(g), C.byref(m)))
        return g.value, m.value

    def sample(self, step: int, index: int) -> tuple[int, int]:
        ds, doc = C.c_int32(), C.c_uint64()
        check(lib().mt_feed_sample(self._h, step, index, C.byref(ds), C.byref(doc)))
        return ds.value, doc.value

    def fill(self, step: int, tokens: np.ndarray | None, targets: np.ndarray | None, max_micro_batches: int):
        """Write this rank's int32 [MB][b*s] inputs / targets into the given (e.g. pinned) arrays."""
        as_p = lambda a: None if a is None else C.cast(a.ctypes.data if isinstance(a, np.ndarray) else a,  # noqa: E731
                                                       C.POINTER(C.c_int32))
        check(lib().mt_feed_fill(self._h, step, as_p(tokens), as_p(targets), max_micro_batches))

    def close(self):
        if self._h:
            lib().mt_feed_destroy(self._h)
            self._h = C.c_void_p()
