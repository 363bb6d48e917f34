"""Host-side Python handles over the C++ runtime in libmtnlg.so (include/mtnlg.h).

`Context` = one GPU (+ its NCCL TP/PP/DP groups derived from curator::map_topology), `Layer` = one
tensor-sliced transformer layer shard, `Stage` = this rank's pipeline stage with the 1F1B driver.
Device buffers are passed as raw pointers (e.g. torch tensors' data_ptr()); streams as cudaStream_t.
"""
from __future__ import annotations

import ctypes as C

from ._native import AdamDesc, LayerDesc, ParallelConfig, RankPlacement, StageDesc, VocabDesc, check, lib


def adam_defaults(**overrides) -> AdamDesc:
    """curator::TrainingRecipe optimizer constants (lr < 0 => curator::lr_at(tokens_seen))."""
    d = AdamDesc()
    check(lib().mt_adam_defaults(C.byref(d)))
    for k, v in overrides.items():
        setattr(d, k, v)
    return d
from .planner import layer_desc  # noqa: F401  (re-export)


def _stream(stream) -> C.c_void_p:
    if stream is None:
        return C.c_void_p(0)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


class Context:
    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().mt_ctx_create(device, C.byref(self._h)))
        self.device = device

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().mt_nccl_unique_id(buf))
        return buf.raw

    def init_comm(self, nccl_id: bytes, world_size: int, rank: int, tensor=1, pipeline=1, data=1, batch=1,
                  micro_batches=1) -> None:
        par = ParallelConfig(tensor, pipeline, data, batch, micro_batches)
        check(lib().mt_ctx_init_comm(self._h, nccl_id, world_size, rank, C.byref(par)))

    def set_sequence_parallel(self, enable: bool = True) -> None:
        """Megatron sequence parallelism for TP > 1 (layer inputs/outputs become this rank's token rows)."""
        check(lib().mt_ctx_set_sequence_parallel(self._h, int(enable)))

    def wait(self, stream=None) -> None:
        """Bounded wait for `stream` (status 2 / DataError if a peer rank is dead or diverged)."""
        check(lib().mt_ctx_wait(self._h, _stream(stream)))

    def error_state(self) -> int:
        v = C.c_int32()
        check(lib().mt_ctx_error(self._h, C.byref(v)))
        return v.value

    def placement(self) -> RankPlacement:
        p = RankPlacement()
        check(lib().mt_ctx_placement(self._h, C.byref(p)))
        return p

    def close(self) -> None:
        if self._h:
            lib().mt_ctx_destroy(self._h)
            self._h = C.c_void_p()


class Layer:
    def __init__(self, ctx: Context, desc: LayerDesc):
        self.ctx, self.desc = ctx, desc
        self._h = C.c_void_p()
        check(lib().mt_layer_create(ctx._h, C.byref(desc), C.byref(self._h)))

    def init_params(self, stream=None) -> None:
        check(lib().mt_layer_init_params(self._h, _stream(stream)))

    def set_param(self, param: int, host_global_bf16_ptr: int) -> None:
        check(lib().mt_layer_set_param(self._h, param, C.c_void_p(host_global_bf16_ptr)))

    def get_param(self, param: int, host_u16_ptr: int) -> None:
        check(lib().mt_layer_get_param(self._h, param, C.c_void_p(host_u16_ptr)))

    def get_grad(self, param: int, host_f32_ptr: int) -> None:
        check(lib().mt_layer_get_grad(self._h, param, C.cast(C.c_void_p(host_f32_ptr), C.POINTER(C.c_float))))

    def zero_grads(self, stream=None) -> None:
        check(lib().mt_layer_zero_grads(self._h, _stream(stream)))

    def forward(self, x_ptr: int, y_ptr: int, micro_batch: int = 0, stream=None) -> None:
        check(lib().mt_layer_forward(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), micro_batch, _stream(stream)))

    def backward(self, dy_ptr: int, dx_ptr: int, micro_batch: int = 0, stream=None) -> None:
        check(lib().mt_layer_backward(self._h, C.c_void_p(dy_ptr), C.c_void_p(dx_ptr), micro_batch, _stream(stream)))

    def adam_step(self, desc: AdamDesc, stream=None) -> float:
        norm = C.c_float()
        check(lib().mt_layer_adam_step(self._h, C.byref(desc), C.byref(norm), _stream(stream)))
        return norm.value

    def optimizer_state(self, param: int, master_ptr: int, m_ptr: int, v_ptr: int) -> None:
        f = C.POINTER(C.c_float)
        check(lib().mt_layer_get_optimizer_state(self._h, param, C.cast(C.c_void_p(master_ptr), f),
                                                 C.cast(C.c_void_p(m_ptr), f), C.cast(C.c_void_p(v_ptr), f)))

    def set_recompute(self, enable: bool = True) -> None:
        check(lib().mt_layer_set_recompute(self._h, int(enable)))

    def finish_grads(self, stream=None) -> None:
        """Sequence parallel: complete the TP-replicated parameters' gradients (collective over TP)."""
        check(lib().mt_layer_finish_grads(self._h, _stream(stream)))

    def set_step(self, step: int) -> None:
        """Training step keying the dropout masks of the next forwards (curator::step_seed)."""
        check(lib().mt_layer_set_step(self._h, step))

    def launch_counts(self) -> tuple[int, int]:
        f, b = C.c_int32(), C.c_int32()
        check(lib().mt_layer_launch_counts(self._h, C.byref(f), C.byref(b)))
        return f.value, b.value

    def dropout_keep_bits(self, mb: int, which: int, nbytes: int) -> bytes:
        """The keep bits the forward of microbatch `mb` saved (which 0: attention words, 1/2: hidden
        bytes after attention-out / MLP-out); see mt_layer_dropout_keep_bits."""
        buf = C.create_string_buffer(nbytes)
        got = C.c_int64()
        check(lib().mt_layer_dropout_keep_bits(self._h, mb, which, buf, nbytes, C.byref(got)))
        return buf.raw[: got.value]

    def close(self) -> None:
        if self._h:
            lib().mt_layer_destroy(self._h)
            self._h = C.c_void_p()


class Vocab:
    """Vocab-parallel embedding + final LayerNorm + tied LM head / cross-entropy (include/mtnlg.h)."""

    WORD, POS, LNF_GAMMA, LNF_BETA = 0, 1, 2, 3

    def __init__(self, ctx: Context, vocab: int, hidden: int, seq: int, micro_batch: int, tp_size: int = 1,
                 tp_rank: int = 0, dropout: float = 0.1, ln_eps: float = 1e-5, seed: int = 1234):
        self.ctx = ctx
        self.desc = VocabDesc(vocab, hidden, seq, micro_batch, tp_size, tp_rank, dropout, ln_eps, seed)
        self._h = C.c_void_p()
        check(lib().mt_vocab_create(ctx._h, C.byref(self.desc), C.byref(self._h)))

    def padded(self) -> tuple[int, int, int]:
        """(padded vocab, first row of this rank's slice, rows in the slice)."""
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().mt_vocab_padded(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def set_param(self, param: int, host_global_bf16_ptr: int) -> None:
        check(lib().mt_vocab_set_param(self._h, param, C.c_void_p(host_global_bf16_ptr)))

    def get_param(self, param: int, host_bf16_ptr: int) -> None:
        check(lib().mt_vocab_get_param(self._h, param, C.c_void_p(host_bf16_ptr)))

    def get_grad(self, param: int, host_f32_ptr: int) -> None:
        check(lib().mt_vocab_get_grad(self._h, param, C.cast(host_f32_ptr, C.POINTER(C.c_float))))

    def close(self) -> None:
        if self._h:
            lib().mt_vocab_destroy(self._h)
            self._h = C.c_void_p()


class Stage:
    """This rank's pipeline stage: layers [stage*L/PP, (stage+1)*L/PP) of the model."""

    def __init__(self, ctx: Context, layer: LayerDesc, layers: int, micro_batches: int):
        self.ctx = ctx
        self.desc = StageDesc(layer, layers, micro_batches)
        self._h = C.c_void_p()
        check(lib().mt_stage_create(ctx._h, C.byref(self.desc), C.byref(self._h)))

    def layer(self, i: int) -> Layer:
        h = C.c_void_p()
        check(lib().mt_stage_layer(self._h, i, C.byref(h)))
        lay = Layer.__new__(Layer)
        lay.ctx, lay.desc, lay._h = self.ctx, None, h
        return lay

    def init_params(self, n_layers: int, stream=None) -> None:
        for i in range(n_layers):
            self.layer(i).init_params(stream)

    def train_step(self, inputs_host_ptr: int | None = None, targets_host_ptr: int | None = None,
                   stream=None, want_loss: bool = True) -> float:
        loss = C.c_float(0.0)
        check(lib().mt_stage_train_step(self._h, C.c_void_p(inputs_host_ptr or 0), C.c_void_p(targets_host_ptr or 0),
                                        C.byref(loss) if want_loss else None, _stream(stream)))
        return loss.value

    def train_step_dev(self, inputs_dev_ptr: int, targets_dev_ptr: int, loss_dev_ptr: int | None = None,
                       stream=None) -> None:
        """Iteration with device-resident inputs / targets ([MB][b*s*h] bf16); asynchronous."""
        check(lib().mt_stage_train_step_dev(self._h, C.c_void_p(inputs_dev_ptr or 0), C.c_void_p(targets_dev_ptr or 0),
                                            C.c_void_p(loss_dev_ptr or 0), _stream(stream)))

    def optimizer_step(self, desc: AdamDesc, stream=None, want_norm: bool = True) -> float:
        norm = C.c_float()
        check(lib().mt_stage_optimizer_step(self._h, C.byref(desc), C.byref(norm) if want_norm else None,
                                            _stream(stream)))
        return norm.value

    def set_recompute(self, enable: bool = True) -> None:
        check(lib().mt_stage_set_recompute(self._h, int(enable)))

    def host_traffic(self) -> tuple[int, int]:
        """(H2D, D2H) bytes this rank moved in its last train_step."""
        a, b = C.c_int64(), C.c_int64()
        check(lib().mt_stage_host_traffic(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_step(self, step: int) -> None:
        """Training step of the next iteration (dropout masks; +1 per train_step)."""
        check(lib().mt_stage_set_step(self._h, step))

    def step(self) -> int:
        v = C.c_uint64()
        check(lib().mt_stage_get_step(self._h, C.byref(v)))
        return v.value

    def set_micro_batches(self, n: int) -> None:
        """Microbatches of the next iterations (<= the count the stage was created with)."""
        check(lib().mt_stage_set_micro_batches(self._h, n))

    def attach_vocab(self, vocab: Vocab) -> None:
        """Language-model mode: inputs / targets become int32 token ids [MB][b*s]."""
        check(lib().mt_stage_attach_vocab(self._h, vocab._h))
        self.vocab = vocab

    def launch_count(self) -> int:
        n = C.c_int64()
        check(lib().mt_stage_launch_count(self._h, C.byref(n)))
        return n.value

    def close(self) -> None:
        if self._h:
            lib().mt_stage_destroy(self._h)
            self._h = C.c_void_p()
