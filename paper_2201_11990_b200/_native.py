"""ctypes binding of libmtnlg.so (the C ABI declared in include/mtnlg.h and include/mtnlg_gemm.h).

The product path has no fallback: if the library is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libmtnlg.so"
_lib = None

MT_OK, MT_ERR_CONFIG, MT_ERR_DATA = 0, 1, 2


class GemmArgs(C.Structure):
    _fields_ = [
        ("a", C.c_void_p), ("lda", C.c_int64), ("a_batch_stride", C.c_int64), ("a_mn_major", C.c_int32),
        ("b", C.c_void_p), ("ldb", C.c_int64), ("b_batch_stride", C.c_int64), ("b_mn_major", C.c_int32),
        ("d", C.c_void_p), ("ldd", C.c_int64), ("d_batch_stride", C.c_int64),
        ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("batch", C.c_int64),
        ("alpha", C.c_float), ("epilogue", C.c_int32), ("causal", C.c_int32),
        ("bias", C.c_void_p), ("aux", C.c_void_p), ("ld_aux", C.c_int64), ("block_n", C.c_int32),
        ("max_ctas", C.c_int32), ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64),
        ("allreduce", C.c_void_p),
    ]


EPI_STORE_BF16, EPI_BIAS_GELU, EPI_GELU_BWD, EPI_STORE_F32, EPI_ACCUM_F32 = range(5)
CAUSAL_NONE, CAUSAL_SKIP_UPPER_TILES, CAUSAL_K_LE_M, CAUSAL_K_GE_M = range(4)


class ClusterTopology(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("gpus_per_node", C.c_int32), ("intra_node_bw", C.c_double),
                ("inter_node_bw", C.c_double), ("peak_flops_per_gpu", C.c_double)]


class ParallelConfig(C.Structure):
    _fields_ = [("tensor", C.c_int32), ("pipeline", C.c_int32), ("data", C.c_int32), ("batch", C.c_int32),
                ("micro_batches", C.c_int32)]


class RankPlacement(C.Structure):
    _fields_ = [("data", C.c_int32), ("pipeline", C.c_int32), ("tensor", C.c_int32), ("node", C.c_int32),
                ("gpu", C.c_int32)]


class ModelShape(C.Structure):
    _fields_ = [("parameters", C.c_double), ("layers", C.c_int32), ("hidden", C.c_int32), ("heads", C.c_int32),
                ("sequence", C.c_int32), ("vocab", C.c_int32)]


class PipeOp(C.Structure):
    _fields_ = [("kind", C.c_int32), ("micro_batch", C.c_int32)]


class LayerDesc(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("heads", C.c_int32), ("seq", C.c_int32), ("micro_batch", C.c_int32),
                ("tp_size", C.c_int32), ("tp_rank", C.c_int32), ("ffn_mult", C.c_int32),
                ("dropout_hidden", C.c_float), ("dropout_attn", C.c_float), ("ln_eps", C.c_float),
                ("seed", C.c_uint64), ("layer_index", C.c_uint32)]


class AdamDesc(C.Structure):
    _fields_ = [("lr", C.c_float), ("tokens_seen", C.c_double), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("weight_decay", C.c_float), ("grad_clip", C.c_float), ("step", C.c_int64)]


class VocabDesc(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("hidden", C.c_int32), ("seq", C.c_int32), ("micro_batch", C.c_int32),
                ("tp_size", C.c_int32), ("tp_rank", C.c_int32), ("dropout", C.c_float), ("ln_eps", C.c_float),
                ("seed", C.c_uint64)]


class FeedDesc(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("seq", C.c_int32), ("micro_batch", C.c_int32), ("data_parallel", C.c_int32),
                ("dp_rank", C.c_int32), ("seed", C.c_uint64)]


class StageDesc(C.Structure):
    _fields_ = [("layer", LayerDesc), ("layers", C.c_int32), ("micro_batches", C.c_int32)]


P = C.c_void_p
I32, I64, U32, U64, F32, F64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float, C.c_double
PI32, PI64, PF32, PF64 = C.POINTER(I32), C.POINTER(I64), C.POINTER(F32), C.POINTER(F64)

_SIGS = {
    "mt_gemm": (C.c_int, [C.POINTER(GemmArgs), P]),
    "mt_gemm_launches_per_call": (C.c_int, []),
    "mt_gemm_allreduce_wait": (C.c_int, [P, P, U32, P]),
    "mt_gemm_allreduce_reduce_groups": (C.c_int, [P, I64, P, P, U32, I32, P]),
    "mt_last_error": (C.c_char_p, []),
    "mt_version": (C.c_char_p, []),
    "mt_map_topology": (C.c_int, [C.POINTER(ClusterTopology), C.POINTER(ParallelConfig), C.POINTER(RankPlacement),
                                  I64, PI64]),
    "mt_pipeline_efficiency": (C.c_int, [I32, I32, PF64]),
    "mt_estimated_tflops_per_gpu": (C.c_int, [C.POINTER(ModelShape), C.POINTER(ParallelConfig),
                                              C.POINTER(ClusterTopology), F64, PF64]),
    "mt_weight_init_std": (C.c_int, [F64, PF64]),
    "mt_activation_bytes": (C.c_int, [F64, F64, F64, F64, PF64]),
    "mt_model_state_bytes": (C.c_int, [F64, PF64]),
    "mt_lr_at": (C.c_int, [F64, PF64]),
    "mt_batch_size_at": (C.c_int, [F64, PI32]),
    "mt_plan_report": (C.c_int, [C.c_char_p, I32, C.c_char_p, I64, PI64]),
    "mt_pipeline_schedule": (C.c_int, [I32, I32, I32, C.POINTER(PipeOp), I32, PI32]),
    "mt_pipeline_simulate": (C.c_int, [I32, I32, I32, I32, PI64]),
    "mt_param_shard": (C.c_int, [C.POINTER(LayerDesc), I32, PI64, PI64, PI64]),
    "mt_stream_key": (U64, [U64, C.c_char_p, U32, U32]),
    "mt_dropout_threshold16": (U32, [F64]),
    "mt_ctx_create": (C.c_int, [I32, C.POINTER(P)]),
    "mt_ctx_destroy": (C.c_int, [P]),
    "mt_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "mt_ctx_init_comm": (C.c_int, [P, C.c_char_p, I32, I32, C.POINTER(ParallelConfig)]),
    "mt_ctx_placement": (C.c_int, [P, C.POINTER(RankPlacement)]),
    "mt_ctx_shard_only": (C.c_int, [P, I32]),
    "mt_ctx_wait": (C.c_int, [P, P]),
    "mt_ctx_error": (C.c_int, [P, PI32]),
    "mt_ctx_set_sequence_parallel": (C.c_int, [P, I32]),
    "mt_layer_finish_grads": (C.c_int, [P, P]),
    "mt_ctx_nvls_probe": (C.c_int, [P, I64, I64, I32, I32, I32, PF64]),
    "mt_ctx_gemm_timing": (C.c_int, [P, I32]),
    "mt_ctx_gemm_timing_read": (C.c_int, [P, PF64, PF64, PI64]),
    "mt_ctx_op_timing": (C.c_int, [P, I32]),
    "mt_ctx_op_timing_read": (C.c_int, [P, C.c_char_p, I64, PI64]),
    "mt_layer_create": (C.c_int, [P, C.POINTER(LayerDesc), C.POINTER(P)]),
    "mt_layer_destroy": (C.c_int, [P]),
    "mt_layer_init_params": (C.c_int, [P, P]),
    "mt_layer_set_param": (C.c_int, [P, I32, P]),
    "mt_layer_get_grad": (C.c_int, [P, I32, PF32]),
    "mt_layer_get_param": (C.c_int, [P, I32, P]),
    "mt_layer_zero_grads": (C.c_int, [P, P]),
    "mt_layer_forward": (C.c_int, [P, P, P, U32, P]),
    "mt_layer_backward": (C.c_int, [P, P, P, U32, P]),
    "mt_layer_launch_counts": (C.c_int, [P, PI32, PI32]),
    "mt_layer_set_recompute": (C.c_int, [P, I32]),
    "mt_layer_set_step": (C.c_int, [P, U64]),
    "mt_layer_dropout_keep_bits": (C.c_int, [P, C.c_uint32, C.c_int32, P, C.c_int64, C.POINTER(C.c_int64)]),
    "mt_vocab_set_step": (C.c_int, [P, U64]),
    "mt_vocab_set_loss_scale": (C.c_int, [P, F32]),
    "mt_stage_set_step": (C.c_int, [P, U64]),
    "mt_stage_get_step": (C.c_int, [P, C.POINTER(U64)]),
    "mt_stage_set_recompute": (C.c_int, [P, I32]),
    "mt_vocab_create": (C.c_int, [P, C.POINTER(VocabDesc), C.POINTER(P)]),
    "mt_vocab_destroy": (C.c_int, [P]),
    "mt_vocab_padded": (C.c_int, [P, PI64, PI64, PI64]),
    "mt_vocab_set_param": (C.c_int, [P, I32, P]),
    "mt_vocab_get_grad": (C.c_int, [P, I32, PF32]),
    "mt_vocab_get_param": (C.c_int, [P, I32, P]),
    "mt_vocab_zero_grads": (C.c_int, [P, P]),
    "mt_vocab_embed_forward": (C.c_int, [P, P, P, U32, P]),
    "mt_vocab_embed_backward": (C.c_int, [P, P, P, U32, P]),
    "mt_vocab_head_loss": (C.c_int, [P, P, P, P, P, P]),
    "mt_layer_grad_buffer": (C.c_int, [P, C.POINTER(PF32), PI64]),
    "mt_mse_loss": (C.c_int, [P, P, P, P, I64, P]),
    "mt_fill_normal": (C.c_int, [P, I64, U64, F32, F32, P]),
    "mt_tp_allreduce_bf16": (C.c_int, [P, P, I64, P]),
    "mt_dp_allreduce_f32": (C.c_int, [P, P, I64, I32, P]),
    "mt_pp_send_bf16": (C.c_int, [P, P, I64, I32, P]),
    "mt_pp_recv_bf16": (C.c_int, [P, P, I64, I32, P]),
    "mt_stage_create": (C.c_int, [P, C.POINTER(StageDesc), C.POINTER(P)]),
    "mt_stage_destroy": (C.c_int, [P]),
    "mt_stage_layer": (C.c_int, [P, I32, C.POINTER(P)]),
    "mt_stage_train_step": (C.c_int, [P, P, P, PF32, P]),
    "mt_stage_train_step_dev": (C.c_int, [P, P, P, P, P]),
    "mt_stage_launch_count": (C.c_int, [P, PI64]),
    "mt_stage_optimizer_step": (C.c_int, [P, C.POINTER(AdamDesc), PF32, P]),
    "mt_stage_attach_vocab": (C.c_int, [P, P]),
    "mt_stage_set_micro_batches": (C.c_int, [P, I32]),
    "mt_stage_host_traffic": (C.c_int, [P, PI64, PI64]),
    "mt_blend_create": (C.c_int, [I32, C.POINTER(C.c_char_p), PF64, C.POINTER(U64), I32, C.POINTER(P)]),
    "mt_blend_destroy": (C.c_int, [P]),
    "mt_blend_weights": (C.c_int, [P, PF64]),
    "mt_blend_next": (C.c_int, [P, U64, C.POINTER(U64), PF64, C.POINTER(U64)]),
    "mt_blend_manifest": (C.c_int, [I32, C.POINTER(C.c_char_p), PF64, C.POINTER(C.POINTER(U64)), C.POINTER(U64), U64,
                                    U64, C.POINTER(U64), I32, U64, C.c_char_p]),
    "mt_feed_open": (C.c_int, [C.c_char_p, C.POINTER(FeedDesc), C.POINTER(P)]),
    "mt_feed_destroy": (C.c_int, [P]),
    "mt_feed_steps": (C.c_int, [P, PI64]),
    "mt_feed_dataset_name": (C.c_int, [P, I32, C.POINTER(C.c_char_p)]),
    "mt_feed_step_info": (C.c_int, [P, I64, PI64, PI32]),
    "mt_feed_sample": (C.c_int, [P, I64, I64, PI32, C.POINTER(U64)]),
    "mt_feed_fill": (C.c_int, [P, I64, PI32, PI32, I32]),
    "mt_feed_doc_tokens": (C.c_int, [U64, C.c_char_p, U64, I32, I64, PI32]),
    "mt_adam_defaults": (C.c_int, [C.POINTER(AdamDesc)]),
    "mt_layer_adam_step": (C.c_int, [P, C.POINTER(AdamDesc), PF32, P]),
    "mt_layer_get_optimizer_state": (C.c_int, [P, I32, PF32, PF32, PF32]),
}

EXPORTED = sorted(_SIGS)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(f"native library {_LIB_PATH} is missing: run `python -m paper_2201_11990_b200.build`")
        L = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


class ConfigError(ValueError):
    """Status 1: bad configuration / argument (the reference's ConfigError / std::invalid_argument)."""


class DataError(RuntimeError):
    """Status 2: CUDA / NCCL / data failure (the reference's DataError)."""


def check(rc: int) -> None:
    if rc == MT_OK:
        return
    msg = (lib().mt_last_error() or b"").decode()
    if rc == MT_ERR_CONFIG:
        raise ConfigError(msg)
    raise DataError(msg)
