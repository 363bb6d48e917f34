"""Python mirror of the reference's planner / partition / schedule API.

Same names and argument meaning as `curator::` in the reference (proj/include/curator/planner.hpp:9-126):
map_topology, pipeline_efficiency, estimated_tflops_per_gpu, weight_init_std, activation_bytes,
model_state_bytes, lr_at, batch_size_at, plan_report; plus the runtime's schedule/shard API
(curator/schedule.hpp). Errors keep the reference's split: ConfigError (a ValueError, for
std::invalid_argument / ConfigError) and DataError. All calls go through libmtnlg.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from ._native import (ClusterTopology, ConfigError, DataError, LayerDesc, ModelShape, ParallelConfig,  # noqa: F401
                      PipeOp, RankPlacement, check, lib)


@dataclass(frozen=True)
class Placement:
    data: int
    pipeline: int
    tensor: int
    node: int
    gpu: int


def topology(nodes: int, gpus_per_node: int = 8, peak_tflops_per_gpu: float = 312.0) -> ClusterTopology:
    return ClusterTopology(nodes, gpus_per_node, 600e9, 25e9, peak_tflops_per_gpu * 1e12)


def parallel(tensor=1, pipeline=1, data=1, batch=1, micro_batches=1) -> ParallelConfig:
    return ParallelConfig(tensor, pipeline, data, batch, micro_batches)


def map_topology(topo: ClusterTopology, par: ParallelConfig) -> list[Placement]:
    n = C.c_int64()
    check(lib().mt_map_topology(C.byref(topo), C.byref(par), None, 0, C.byref(n)))
    out = (RankPlacement * max(n.value, 1))()
    check(lib().mt_map_topology(C.byref(topo), C.byref(par), out, n.value, C.byref(n)))
    return [Placement(p.data, p.pipeline, p.tensor, p.node, p.gpu) for p in out[: n.value]]


def _f64(fn, *args) -> float:
    out = C.c_double()
    check(fn(*args, C.byref(out)))
    return out.value


def pipeline_efficiency(micro_batches: int, stages: int) -> float:
    return _f64(lib().mt_pipeline_efficiency, micro_batches, stages)


def weight_init_std(hidden: float) -> float:
    return _f64(lib().mt_weight_init_std, hidden)


def activation_bytes(batch, layers, sequence, hidden) -> float:
    return _f64(lib().mt_activation_bytes, batch, layers, sequence, hidden)


def model_state_bytes(parameters: float) -> float:
    return _f64(lib().mt_model_state_bytes, parameters)


def lr_at(tokens_seen: float) -> float:
    return _f64(lib().mt_lr_at, tokens_seen)


def batch_size_at(tokens_seen: float) -> int:
    out = C.c_int32()
    check(lib().mt_batch_size_at(tokens_seen, C.byref(out)))
    return out.value


def estimated_tflops_per_gpu(shape: ModelShape, par: ParallelConfig, topo: ClusterTopology, seconds: float) -> float:
    return _f64(lib().mt_estimated_tflops_per_gpu, C.byref(shape), C.byref(par), C.byref(topo), seconds)


def plan_report(config_path: str, as_json: bool = False) -> str:
    n = C.c_int64()
    check(lib().mt_plan_report(config_path.encode(), int(as_json), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().mt_plan_report(config_path.encode(), int(as_json), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def pipeline_schedule(stage: int, stages: int, micro_batches: int) -> list[tuple[str, int]]:
    n = C.c_int32()
    out = (PipeOp * (2 * max(micro_batches, 1)))()
    check(lib().mt_pipeline_schedule(stage, stages, micro_batches, out, len(out), C.byref(n)))
    return [("F" if o.kind == 0 else "B", o.micro_batch) for o in out[: n.value]]


def pipeline_simulate(stages: int, micro_batches: int, t_forward: int = 1, t_backward: int = 2) -> int:
    out = C.c_int64()
    check(lib().mt_pipeline_simulate(stages, micro_batches, t_forward, t_backward, C.byref(out)))
    return out.value


PARAM_NAMES = ["ln1.gamma", "ln1.beta", "qkv.weight", "qkv.bias", "proj.weight", "proj.bias",
               "ln2.gamma", "ln2.beta", "fc1.weight", "fc1.bias", "fc2.weight", "fc2.bias"]


def layer_desc(hidden, heads, seq, micro_batch=1, tp_size=1, tp_rank=0, ffn_mult=4, dropout_hidden=0.1,
               dropout_attn=0.1, ln_eps=1e-5, seed=20260808, layer_index=0) -> LayerDesc:
    return LayerDesc(hidden, heads, seq, micro_batch, tp_size, tp_rank, ffn_mult, dropout_hidden, dropout_attn,
                     ln_eps, seed, layer_index)


def param_shard(desc: LayerDesc, param: int):
    g, o, s = (C.c_int64 * 2)(), (C.c_int64 * 2)(), (C.c_int64 * 2)()
    check(lib().mt_param_shard(C.byref(desc), param, g, o, s))
    return tuple(g), tuple(o), tuple(s)


def stream_key(seed: int, name: str, layer: int = 0, micro_batch: int = 0) -> int:
    return int(lib().mt_stream_key(seed, name.encode(), layer, micro_batch))


def dropout_threshold16(p: float) -> int:
    return int(lib().mt_dropout_threshold16(p))
