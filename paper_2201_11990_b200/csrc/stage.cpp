// Pipeline stage driver: one training iteration of one rank under the 3D layout.
//
// The op order is curator::one_f_one_b (PipeDream-Flush 1F1B). Point-to-point
// transfers follow the Megatron pairing so neighbouring stages never wait on each other's sends:
// in the steady phase a stage posts "send activation forward + receive gradient backward" as one
// NCCL group, and "send gradient backward + receive next activation" as another. After the last
// backward the fp32 parameter gradients are all-reduced (mean) over the data-parallel group
// (PAPER.md:103-131). TP all-reduces happen inside the layers.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "curator/dropout.hpp"
#include "curator/schedule.hpp"
#include "kernels.cuh"
#include "runtime.hpp"

namespace mt {
void set_error(const std::string& e);
}

struct mt_stage {
  mt_ctx* ctx = nullptr;
  mt_stage_desc d{};               // d.micro_batches = microbatches of the next iteration
  int mb_capacity = 0;             // microbatch buffers allocated at creation
  int stage = 0, stages = 1;
  std::vector<mt_layer*> layers;
  int64_t M = 0, h = 0;
  std::vector<std::vector<mt::DeviceBuffer>> act;  // [mb][layer+1] bf16 [M, h]
  mt::DeviceBuffer grad[2];                        // ping-pong [M, h]
  mt::DeviceBuffer target;                         // [M, h]
  mt::DeviceBuffer loss;                           // fp32 scalar
  float* loss_host = nullptr;                      // pinned: the loss D2H never blocks the host (bounded wait)
  int64_t launches = 0;
  // training step of the next iteration: keys the dropout masks of every layer and of the embedding
  // (curator::step_seed), so they change from one iteration to the next; incremented per iteration
  uint64_t step = 0;
  // host-input path: all microbatches' H2D copies are queued up front on a copy stream and
  // overlap compute; each microbatch's first use waits on its own event
  cudaStream_t copy = nullptr;
  cudaEvent_t iter_start = nullptr;
  std::vector<cudaEvent_t> in_ev, tgt_ev;
  std::vector<cudaEvent_t> tgt_gathered;            // TP-split targets all-gathered off the compute stream
  std::vector<mt::DeviceBuffer> targets;           // [MB][M, h] (host-target path)
  // language-model mode (mt_stage_attach_vocab): inputs/targets are int32 token ids [MB][M]
  mt_vocab* vocab = nullptr;
  std::vector<mt::DeviceBuffer> tokens;            // [MB][M] int32 (host-input path, first stage)
  int64_t h2d_bytes = 0, d2h_bytes = 0;            // host traffic of the last mt_stage_train_step
  // host inputs arrive in row chunks (one event each) that layer 0 consumes as they land
  static constexpr int kMaxInChunks = 8;
  int in_chunks = 4;                               // MT_INPUT_CHUNKS (1 disables, up to 8)
};

namespace {

template <class F>
int call(F&& f) {
  try {
    f();
    return MT_OK;
  } catch (const std::invalid_argument& e) {
    mt::set_error(e.what());
    return MT_ERR_CONFIG;
  } catch (const std::exception& e) {
    mt::set_error(e.what());
    return MT_ERR_DATA;
  }
}

void ok(int rc) {
  if (rc == MT_ERR_CONFIG) throw std::invalid_argument(mt_last_error());
  if (rc != MT_OK) throw mt::RuntimeFailure(mt_last_error());
}

struct Step {
  mt_stage* st;
  cudaStream_t s;
  const char* in_host;
  const char* tgt_host;
  const char* in_dev = nullptr;   // device-resident inputs (train_step_dev)
  const char* tgt_dev = nullptr;
  int64_t launches = 0;
  bool first() const { return st->stage == 0; }
  bool last() const { return st->stage == st->stages - 1; }
  bool lm() const { return st->vocab != nullptr; }
  // Sequence parallelism (mt_ctx_set_sequence_parallel): activations between layers, stage inputs /
  // targets and PP transfers are this TP rank's token rows only.
  bool sp() const {
    const mt_ctx* c = st->ctx;
    return !lm() && c->seq_parallel && c->par.tensor > 1 && c->tp && !c->shard_only;
  }
  int64_t full_elems() const { return st->M * st->h; }
  int64_t elems() const { return sp() ? full_elems() / st->ctx->par.tensor : full_elems(); }
  size_t bytes() const { return static_cast<size_t>(elems() * 2); }
  // bytes of one microbatch's input / target in the caller's buffers (full rows; int32 ids with a vocab)
  size_t io_bytes() const { return st->vocab ? static_cast<size_t>(st->M * 4) : static_cast<size_t>(full_elems() * 2); }
  size_t sp_off() const { return sp() ? bytes() * st->ctx->place.tensor : 0; }  // this rank's rows in io buffers
  // TP > 1, host inputs: the t ranks of a TP group need the same activations / targets, so each
  // copies only its 1/t row slice over PCIe and the slices are all-gathered over NVLink (in place),
  // instead of t full host->device copies competing for host bandwidth.
  bool split_h2d() const {
    const mt_ctx* c = st->ctx;
    return !sp() && !lm() && c->par.tensor > 1 && c->tp && !c->shard_only && (elems() % c->par.tensor) == 0;
  }
  size_t slice_bytes() const {
    return sp() ? bytes() : split_h2d() ? io_bytes() / st->ctx->par.tensor : io_bytes();
  }
  size_t slice_off() const { return sp() ? sp_off() : split_h2d() ? slice_bytes() * st->ctx->place.tensor : 0; }
  size_t dst_off() const { return sp() ? 0 : slice_off(); }  // where the copied rows land on the device
  void gather_slices(void* buf) {
    if (!split_h2d()) return;
    const size_t n = elems() / st->ctx->par.tensor;
    mt::check_nccl(ncclAllGather(static_cast<char*>(buf) + slice_off(), buf, n, ncclBfloat16, st->ctx->tp, s),
                   "ncclAllGather(input slices)");
    ++launches;
  }
  // Host input of the first stage split into row chunks: the copy of chunk k+1 overlaps LN1 + QKV
  // GEMM of chunk k inside layer 0 (mt_layer::input_gate).
  int in_chunks() const {
    const int k = st->in_chunks, t = split_h2d() ? st->ctx->par.tensor : 1;
    if (!in_host || !first() || lm() || sp() || st->layers.empty() || k <= 1) return 1;
    return (st->M % (int64_t{k} * 128) == 0 && (st->M / k) % t == 0) ? k : 1;
  }
  size_t chunk_bytes() const { return bytes() / in_chunks(); }
  size_t chunk_slice_bytes() const { return split_h2d() ? chunk_bytes() / st->ctx->par.tensor : chunk_bytes(); }
  size_t chunk_slice_off() const { return split_h2d() ? chunk_slice_bytes() * st->ctx->place.tensor : 0; }
  ncclComm_t pp() const { return st->ctx->pp; }
  // Global microbatch id (data-parallel replicas see different samples): keys the synthetic
  // inputs/targets and the dropout masks of the microbatch.
  uint32_t gid(int mb) const {
    return static_cast<uint32_t>(st->ctx->place.data * st->d.micro_batches + mb);
  }

  const void* input(int mb) const {
    return (in_dev && first() && !lm()) ? static_cast<const void*>(in_dev + mb * io_bytes() + sp_off())
                                        : st->act[mb][0].ptr;
  }
  // Queue every microbatch's host->device copies on the copy stream (after the previous
  // iteration's compute released the buffers).
  void prefetch_host() {
    if (!in_host && !tgt_host) return;
    mt::check_cuda(cudaEventRecord(st->iter_start, s), "cudaEventRecord");
    mt::check_cuda(cudaStreamWaitEvent(st->copy, st->iter_start, 0), "cudaStreamWaitEvent");
    for (int mb = 0; mb < st->d.micro_batches; ++mb) {
      if (in_host && first() && in_chunks() > 1) {
        for (int k = 0; k < in_chunks(); ++k) {
          const size_t off = k * chunk_bytes() + chunk_slice_off();
          mt::check_cuda(cudaMemcpyAsync(static_cast<char*>(st->act[mb][0].ptr) + off, in_host + mb * io_bytes() + off,
                                         chunk_slice_bytes(), cudaMemcpyHostToDevice, st->copy),
                         "H2D input chunk");
          st->h2d_bytes += static_cast<int64_t>(chunk_slice_bytes());
          mt::check_cuda(cudaEventRecord(st->in_ev[mb * mt_stage::kMaxInChunks + k], st->copy), "cudaEventRecord");
        }
      } else if (in_host && first()) {
        char* dst = static_cast<char*>(lm() ? st->tokens[mb].ptr : st->act[mb][0].ptr) + dst_off();
        mt::check_cuda(cudaMemcpyAsync(dst, in_host + mb * io_bytes() + slice_off(), slice_bytes(),
                                       cudaMemcpyHostToDevice, st->copy),
                       "H2D input");
        st->h2d_bytes += static_cast<int64_t>(slice_bytes());
        mt::check_cuda(cudaEventRecord(st->in_ev[mb * mt_stage::kMaxInChunks], st->copy), "cudaEventRecord");
      }
      if (tgt_host && last()) {
        mt::check_cuda(cudaMemcpyAsync(static_cast<char*>(st->targets[mb].ptr) + dst_off(),
                                       tgt_host + mb * io_bytes() + slice_off(), slice_bytes(),
                                       cudaMemcpyHostToDevice, st->copy),
                       "H2D target");
        st->h2d_bytes += static_cast<int64_t>(slice_bytes());
        mt::check_cuda(cudaEventRecord(st->tgt_ev[mb], st->copy), "cudaEventRecord");
      }
    }
  }
  const int32_t* tokens(int mb) const {
    return in_dev ? reinterpret_cast<const int32_t*>(in_dev + mb * io_bytes()) : st->tokens[mb].as<int32_t>();
  }
  void load_input(int mb) {
    void* dst = st->act[mb][0].ptr;
    if (lm()) {  // token ids -> embeddings (+ position, dropout; TP all-reduce of the vocab-parallel gather)
      if (in_host)
        mt::check_cuda(cudaStreamWaitEvent(s, st->in_ev[mb * mt_stage::kMaxInChunks], 0), "cudaStreamWaitEvent");
      ok(mt_vocab_embed_forward(st->vocab, tokens(mb), dst, gid(mb), s));
      launches += 2 + (st->ctx->par.tensor > 1 ? 1 : 0);
      return;
    }
    if (in_dev) return;  // read in place by layer 0
    if (in_host) {
      if (in_chunks() > 1) return;  // layer 0 waits chunk by chunk (forward)
      mt::check_cuda(cudaStreamWaitEvent(s, st->in_ev[mb * mt_stage::kMaxInChunks], 0), "cudaStreamWaitEvent");
      gather_slices(dst);
    } else {
      const uint64_t key = mt_stream_key(st->d.layer.seed, "input", 0, gid(mb));
      mt::fill_normal(dst, 1, elems(), full_elems(), 0, static_cast<long long>(sp_off() / 2), key, 0.f, 1.f, s);
      ++launches;
    }
  }
  void forward(int mb) {
    const int K = in_chunks();
    if (K > 1) {
      mt_layer* l0 = st->layers[0];
      l0->input_chunks = K;
      l0->input_gate = [this, mb, K](int k, cudaStream_t stream) {
        mt::check_cuda(cudaStreamWaitEvent(stream, st->in_ev[mb * mt_stage::kMaxInChunks + k], 0),
                       "cudaStreamWaitEvent");
        if (split_h2d()) {
          char* base = static_cast<char*>(st->act[mb][0].ptr) + k * chunk_bytes();
          const size_t n = elems() / K / st->ctx->par.tensor;
          mt::check_nccl(ncclAllGather(base + chunk_slice_off(), base, n, ncclBfloat16, st->ctx->tp, stream),
                         "ncclAllGather(input chunk slices)");
          ++launches;
        }
      };
    }
    for (size_t i = 0; i < st->layers.size(); ++i) {
      const void* x = i == 0 ? input(mb) : st->act[mb][i].ptr;
      const int rc = mt_layer_forward(st->layers[i], x, st->act[mb][i + 1].ptr, gid(mb), s);
      if (i == 0 && K > 1) {
        st->layers[0]->input_gate = nullptr;
        st->layers[0]->input_chunks = 1;
      }
      ok(rc);
      int32_t f, b;
      mt_layer_launch_counts(st->layers[i], &f, &b);
      launches += f;
    }
    if (last()) {
      void* y = st->act[mb][st->layers.size()].ptr;
      if (lm()) {
        const int32_t* tgt = tgt_dev ? reinterpret_cast<const int32_t*>(tgt_dev + mb * io_bytes())
                                     : st->targets[mb].as<int32_t>();
        if (!tgt_dev) mt::check_cuda(cudaStreamWaitEvent(s, st->tgt_ev[mb], 0), "cudaStreamWaitEvent");
        ok(mt_vocab_head_loss(st->vocab, y, tgt, y, st->loss.as<float>(), s));  // dy overwrites y in place
        launches += 10 + (st->ctx->par.tensor > 1 ? 3 : 0);
        return;
      }
      const void* tgt = st->target.ptr;
      if (tgt_dev) {
        tgt = tgt_dev + mb * io_bytes() + sp_off();
      } else if (tgt_host) {
        if (split_h2d() && st->ctx->comm) {  // gathered on the side stream at the start of the iteration
          mt::check_cuda(cudaStreamWaitEvent(s, st->tgt_gathered[mb], 0), "cudaStreamWaitEvent");
        } else {
          mt::check_cuda(cudaStreamWaitEvent(s, st->tgt_ev[mb], 0), "cudaStreamWaitEvent");
          gather_slices(st->targets[mb].ptr);
        }
        tgt = st->targets[mb].ptr;
      } else {
        const uint64_t key = mt_stream_key(st->d.layer.seed, "target", 0, gid(mb));
        mt::fill_normal(st->target.ptr, 1, elems(), full_elems(), 0, static_cast<long long>(sp_off() / 2), key, 0.f, 1.f,
                        s);
        ++launches;
      }
      // the batch mean: each microbatch's mean loss / MB (Megatron's convention), so the loss, the gradients
      // and the clip norm do not scale with the microbatch count; dy overwrites y in place
      mt::mse_loss(y, tgt, y, st->loss.as<float>(), elems(), s, full_elems() * st->d.micro_batches);
      ++launches;
    }
  }
  bool dp_overlapped = false;  // this iteration's layer gradients were all-reduced during the backward
  // Backward of microbatch mb; gradient arrives in g (last stage: in act[mb][L]). Returns dx buffer.
  // During the backward of the last microbatch each layer's gradients are final as soon as its
  // backward is done: their DP all-reduce is issued right away on the DP side stream and overlaps
  // the backward of the layers below (the GEMMs issued meanwhile leave the collective its SMs).
  void* backward(int mb, void* g) {
    mt_ctx* c = st->ctx;
    const bool overlap = c->dp_side && c->dp_overlap && mb == st->d.micro_batches - 1;
    void* cur = g;
    for (size_t i = st->layers.size(); i-- > 0;) {
      void* out = (cur == st->grad[0].ptr) ? st->grad[1].ptr : st->grad[0].ptr;
      ok(mt_layer_backward(st->layers[i], cur, out, gid(mb), s));
      int32_t f, b;
      mt_layer_launch_counts(st->layers[i], &f, &b);
      launches += b;
      cur = out;
      if (overlap && i > 0) {  // layers below remain to overlap with (the bottom layer uses the full comm)
        mt_layer* l = st->layers[i];
        ok(mt_layer_finish_grads(l, s));  // sequence parallel: complete the replicated grads first
        mt::check_cuda(cudaEventRecord(c->ev_dp_ready, s), "cudaEventRecord");
        mt::check_cuda(cudaStreamWaitEvent(c->dp_stream, c->ev_dp_ready, 0), "cudaStreamWaitEvent");
        mt::check_nccl(ncclAllReduce(l->grads.ptr, l->grads.ptr, l->param_total, ncclFloat32, ncclAvg, c->dp_side,
                                     c->dp_stream),
                       "ncclAllReduce(dp, overlapped)");
        ++launches;
        int sms = 0;
        mt::check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device), "attr");
        c->gemm_cap = std::max(2, (sms - c->comm_sms) / 2 * 2);
        dp_overlapped = true;
      }
    }
    if (overlap) c->gemm_cap = 0;
    if (lm() && first()) {
      ok(mt_vocab_embed_backward(st->vocab, tokens(mb), cur, gid(mb), s));
      ++launches;
    }
    return cur;
  }
  void recv_fwd(int mb) {
    mt::check_nccl(ncclRecv(st->act[mb][0].ptr, elems(), ncclBfloat16, st->stage - 1, pp(), s), "recv fwd");
    ++launches;
  }
  void send_fwd(int mb) {
    mt::check_nccl(ncclSend(st->act[mb][st->layers.size()].ptr, elems(), ncclBfloat16, st->stage + 1, pp(), s),
                   "send fwd");
    ++launches;
  }
  void* grad_in_buffer() { return st->grad[0].ptr; }
};

}  // namespace

extern "C" int mt_stage_create(mt_ctx* c, const mt_stage_desc* d, mt_stage** out) {
  return call([&] {
    if (!c || !d || !out) throw std::invalid_argument("null argument");
    auto st = new mt_stage();
    st->ctx = c;
    st->d = *d;
    if (d->micro_batches < 1 || d->layers < 1) throw std::invalid_argument("bad stage descriptor");
    st->mb_capacity = d->micro_batches;
    st->stage = c->place.pipeline;
    st->stages = c->par.pipeline;
    const curator::Range own = curator::stage_layers(d->layers, st->stages, st->stage);
    mt_layer_desc ld = d->layer;
    if (!(c->shard_only && ld.tp_size > 1)) {  // shard-only runs keep the descriptor's TP shard
      ld.tp_size = c->par.tensor;
      ld.tp_rank = c->place.tensor;
    }
    for (int64_t li = own.begin; li < own.end; ++li) {
      ld.layer_index = static_cast<uint32_t>(li);
      mt_layer* l = nullptr;
      const int rc = mt_layer_create(c, &ld, &l);
      if (rc != MT_OK) {
        for (auto* x : st->layers) mt_layer_destroy(x);
        delete st;
        ok(rc);
      }
      st->layers.push_back(l);
    }
    st->M = int64_t{ld.micro_batch} * ld.seq;
    st->h = ld.hidden;
    const size_t bytes = static_cast<size_t>(st->M * st->h * 2);
    st->act.resize(d->micro_batches);
    for (auto& v : st->act) {
      v.resize(st->layers.size() + 1);
      for (auto& b : v) b.ensure(bytes);
    }
    for (auto& g : st->grad) g.ensure(bytes);
    st->target.ensure(bytes);
    st->loss.ensure(4);
    mt::check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&st->loss_host), sizeof(float), cudaHostAllocDefault),
                   "cudaHostAlloc(loss)");
    mt::check_cuda(cudaStreamCreateWithFlags(&st->copy, cudaStreamNonBlocking), "copy stream");
    mt::check_cuda(cudaEventCreateWithFlags(&st->iter_start, cudaEventDisableTiming), "event");
    st->in_ev.resize(size_t(d->micro_batches) * mt_stage::kMaxInChunks);
    if (const char* e = getenv("MT_INPUT_CHUNKS")) st->in_chunks = std::max(1, std::min(mt_stage::kMaxInChunks, atoi(e)));
    st->tgt_ev.resize(d->micro_batches);
    for (auto& e : st->in_ev) mt::check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& e : st->tgt_ev) mt::check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    st->tgt_gathered.resize(d->micro_batches);
    for (auto& e : st->tgt_gathered) mt::check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    if (st->stage == st->stages - 1) {
      st->targets.resize(d->micro_batches);
      for (auto& b : st->targets) b.ensure(bytes);
    }
    *out = st;
  });
}

extern "C" int mt_stage_destroy(mt_stage* st) {
  return call([&] {
    if (!st) return;
    for (auto* l : st->layers) mt_layer_destroy(l);
    for (auto e : st->in_ev) cudaEventDestroy(e);
    for (auto e : st->tgt_ev) cudaEventDestroy(e);
    for (auto e : st->tgt_gathered) cudaEventDestroy(e);
    if (st->iter_start) cudaEventDestroy(st->iter_start);
    if (st->copy) cudaStreamDestroy(st->copy);
    if (st->loss_host) cudaFreeHost(st->loss_host);
    delete st;
  });
}

extern "C" int mt_stage_layer(mt_stage* st, int32_t i, mt_layer** out) {
  return call([&] {
    if (!st || !out || i < 0 || i >= (int32_t)st->layers.size()) throw std::invalid_argument("bad layer index");
    *out = st->layers[i];
  });
}

extern "C" int mt_stage_launch_count(const mt_stage* st, int64_t* n) {
  return call([&] { *n = st->launches; });
}

namespace {

void run_iteration(Step& k, mt_stage* st, void* stream) {
  const int MB = st->d.micro_batches;
  k.prefetch_host();
  // TP-split host targets (last stage): all-gather each microbatch's slices on the TP side stream /
  // communicator as soon as its copy lands, so the gathers stay off the compute stream
  if (k.tgt_host && k.last() && !k.lm() && k.split_h2d() && st->ctx->comm) {
    mt_ctx* c = st->ctx;
    const size_t n = static_cast<size_t>(k.elems() / c->par.tensor);
    for (int mb = 0; mb < MB; ++mb) {
      mt::check_cuda(cudaStreamWaitEvent(c->comm, st->tgt_ev[mb], 0), "cudaStreamWaitEvent");
      char* buf = static_cast<char*>(st->targets[mb].ptr);
      mt::check_nccl(ncclAllGather(buf + k.slice_off(), buf, n, ncclBfloat16, c->tp_side, c->comm),
                     "ncclAllGather(target slices)");
      mt::check_cuda(cudaEventRecord(st->tgt_gathered[mb], c->comm), "cudaEventRecord");
      ++k.launches;
    }
  }
  for (auto* l : st->layers) {
    ok(mt_layer_zero_grads(l, stream));
    ok(mt_layer_set_step(l, st->step));
  }
  const bool vocab_here = k.lm() && (k.first() || k.last());
  if (st->vocab) {
    ok(mt_vocab_set_step(st->vocab, st->step));
    ok(mt_vocab_set_loss_scale(st->vocab, 1.f / static_cast<float>(MB)));  // the batch mean (Megatron)
  }
  if (vocab_here) mt::vocab_zero_grads(st->vocab, k.s);
  mt::check_cuda(cudaMemsetAsync(st->loss.ptr, 0, 4, k.s), "memset loss");
  const int warmup = std::min(st->stages - st->stage - 1, MB);
  const int steady = MB - warmup;
  int next_f = 0, next_b = 0;
  // warmup forwards
  for (int i = 0; i < warmup; ++i) {
    const int mb = next_f++;
    k.first() ? k.load_input(mb) : k.recv_fwd(mb);
    k.forward(mb);
    k.send_fwd(mb);  // warmup > 0 implies not the last stage
  }
  if (steady > 0) k.first() ? k.load_input(next_f) : k.recv_fwd(next_f);
  for (int i = 0; i < steady; ++i) {
    const int mb = next_f++;
    k.forward(mb);
    // send activation forward + receive the gradient of the oldest in-flight microbatch
    const int bmb = next_b++;
    void* g = k.last() ? st->act[bmb][st->layers.size()].ptr : k.grad_in_buffer();
    if (!k.last()) {
      mt::check_nccl(ncclGroupStart(), "group");
      mt::check_nccl(ncclSend(st->act[mb][st->layers.size()].ptr, k.elems(), ncclBfloat16, st->stage + 1, k.pp(), k.s),
                     "send fwd");
      mt::check_nccl(ncclRecv(g, k.elems(), ncclBfloat16, st->stage + 1, k.pp(), k.s), "recv bwd");
      mt::check_nccl(ncclGroupEnd(), "group");
      ++k.launches;
    }
    void* dx = k.backward(bmb, g);
    const bool more = i + 1 < steady;
    if (!k.first()) {
      mt::check_nccl(ncclGroupStart(), "group");
      mt::check_nccl(ncclSend(dx, k.elems(), ncclBfloat16, st->stage - 1, k.pp(), k.s), "send bwd");
      if (more)
        mt::check_nccl(ncclRecv(st->act[next_f][0].ptr, k.elems(), ncclBfloat16, st->stage - 1, k.pp(), k.s),
                       "recv fwd");
      mt::check_nccl(ncclGroupEnd(), "group");
      ++k.launches;
    } else if (more) {
      k.load_input(next_f);
    }
  }
  // cooldown backwards
  for (int i = 0; i < warmup; ++i) {
    const int bmb = next_b++;
    void* g = k.grad_in_buffer();
    mt::check_nccl(ncclRecv(g, k.elems(), ncclBfloat16, st->stage + 1, k.pp(), k.s), "recv bwd");
    ++k.launches;
    void* dx = k.backward(bmb, g);
    if (!k.first()) {
      mt::check_nccl(ncclSend(dx, k.elems(), ncclBfloat16, st->stage - 1, k.pp(), k.s), "send bwd");
      ++k.launches;
    }
  }
  // sequence parallel: complete the TP-replicated parameters' gradients (partial over token rows) and
  // the loss (each TP rank summed its rows)
  if (k.sp()) {
    for (auto* l : st->layers) ok(mt_layer_finish_grads(l, k.s));
    k.launches += static_cast<int64_t>(st->layers.size());
    if (k.last()) {
      mt::check_nccl(ncclAllReduce(st->loss.ptr, st->loss.ptr, 1, ncclFloat32, ncclSum, st->ctx->tp, k.s),
                     "ncclAllReduce(loss, tp)");
      ++k.launches;
    }
  }
  // tied word embedding: the first and the last stage both hold E and sum their gradients
  if (vocab_here && st->stages > 1) {
    mt::vocab_allreduce_grads(st->vocab, st->ctx->emb, true, false, k.s);
    ++k.launches;
  }
  // data-parallel gradient all-reduce (mean)
  if (st->ctx->par.data > 1) {
    if (vocab_here) {
      mt::vocab_allreduce_grads(st->vocab, st->ctx->dp, false, true, k.s);
      k.launches += 4;
    }
    if (k.dp_overlapped) {  // layers 1.. were all-reduced during the last backward; layer 0 here
      ok(mt_dp_allreduce_f32(st->ctx, st->layers[0]->grads.as<float>(), st->layers[0]->param_total, 1, stream));
      ++k.launches;
      mt::check_cuda(cudaEventRecord(st->ctx->ev_dp_done, st->ctx->dp_stream), "cudaEventRecord");
      mt::check_cuda(cudaStreamWaitEvent(k.s, st->ctx->ev_dp_done, 0), "cudaStreamWaitEvent");
    } else {
      for (auto* l : st->layers) {
        ok(mt_dp_allreduce_f32(st->ctx, l->grads.as<float>(), l->param_total, 1, stream));
        ++k.launches;
      }
    }
    if (k.last()) {
      ok(mt_dp_allreduce_f32(st->ctx, st->loss.as<float>(), 1, 1, stream));
      ++k.launches;
    }
  }  ++st->step;
}

// A collective that fails because the watchdog aborted the communicators reports why.
template <class F>
void run_aborted_aware(mt_ctx* c, F&& f) {
  try {
    f();
  } catch (const std::exception& e) {
    if (c->aborted)
      throw mt::RuntimeFailure(std::string("a peer did not respond within the communication bound; the context's "
                                           "communicators were aborted (") + e.what() + ")");
    throw;
  }
}

}  // namespace

extern "C" int mt_stage_train_step(mt_stage* st, const void* inputs_host, const void* targets_host, float* loss_out,
                                   void* stream) {
  return call([&] {
    if (!st) throw std::invalid_argument("null stage");
    if (st->ctx->aborted) throw mt::RuntimeFailure("the context's communicators were aborted after a peer failure");
    mt::WatchdogArm arm(st->ctx);  // a call blocked on a dead peer is released after the context's bound
    Step k{st, (cudaStream_t)stream, static_cast<const char*>(inputs_host), static_cast<const char*>(targets_host)};
    st->h2d_bytes = st->d2h_bytes = 0;
    if (k.lm() && ((k.first() && !inputs_host) || (k.last() && !targets_host)))
      throw std::invalid_argument("a stage with a vocab needs token inputs (first stage) and targets (last stage)");
    run_aborted_aware(st->ctx, [&] { run_iteration(k, st, stream); });
    if (loss_out) {
      *st->loss_host = 0.f;
      if (k.last()) {  // pinned destination: an asynchronous copy, so the wait below stays bounded
        mt::check_cuda(cudaMemcpyAsync(st->loss_host, st->loss.ptr, 4, cudaMemcpyDeviceToHost, k.s), "D2H loss");
        st->d2h_bytes += 4;
      }
      mt::wait_stream(st->ctx, k.s, "mt_stage_train_step");  // bounded: a dead peer -> status 2
      *loss_out = *st->loss_host;
    }
    st->launches = k.launches;
  });
}

extern "C" int mt_stage_train_step_dev(mt_stage* st, const void* inputs_dev, const void* targets_dev, float* loss_dev,
                                       void* stream) {
  return call([&] {
    if (!st) throw std::invalid_argument("null stage");
    if (st->ctx->aborted) throw mt::RuntimeFailure("the context's communicators were aborted after a peer failure");
    mt::WatchdogArm arm(st->ctx);  // a call blocked on a dead peer is released after the context's bound
    Step k{st, (cudaStream_t)stream, nullptr, nullptr};
    k.in_dev = static_cast<const char*>(inputs_dev);
    k.tgt_dev = static_cast<const char*>(targets_dev);
    if (k.first() && !k.in_dev) throw std::invalid_argument("first stage needs device inputs");
    if (k.last() && !k.tgt_dev) throw std::invalid_argument("last stage needs device targets");
    run_aborted_aware(st->ctx, [&] { run_iteration(k, st, stream); });
    if (loss_dev && k.last())
      mt::check_cuda(cudaMemcpyAsync(loss_dev, st->loss.ptr, 4, cudaMemcpyDeviceToDevice, k.s), "D2D loss");
    st->launches = k.launches;
  });
}

float resolve_lr(const mt_adam_desc& d);  // runtime.cpp

extern "C" int mt_stage_optimizer_step(mt_stage* st, const mt_adam_desc* d, float* grad_norm_out, void* stream) {
  return call([&] {
    if (!st || !d) throw std::invalid_argument("null argument");
    if (d->step < 1) throw std::invalid_argument("step must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    mt_ctx* c = st->ctx;
    mt::WatchdogArm arm(c);
    c->opt_scratch.ensure(4 * sizeof(float));
    float* sq = c->opt_scratch.as<float>();
    mt::check_cuda(cudaMemsetAsync(sq, 0, 2 * sizeof(float), s), "memset");
    for (auto* l : st->layers) {
      float* g;
      int64_t n;
      ok(mt_layer_grad_buffer(l, &g, &n));  // materialises logically-zero grads if needed
      mt::layer_grad_sq(l, sq, s);
    }
    const bool first = st->stage == 0, last = st->stage == st->stages - 1;
    const bool vocab_here = st->vocab && (first || last);
    if (vocab_here) mt::vocab_grad_sq(st->vocab, first, sq, s);  // tied E counted once (first stage)
    // TP-replicated parameters (LayerNorm, row-parallel biases) count once per TP group
    if (c->place.tensor != 0) mt::check_cuda(cudaMemsetAsync(sq + 1, 0, sizeof(float), s), "memset");
    if (c->par.tensor > 1 && c->tp)
      mt::check_nccl(ncclAllReduce(sq, sq, 2, ncclFloat32, ncclSum, c->tp, s), "ncclAllReduce(grad norm, tp)");
    if (c->par.pipeline > 1 && c->pp)
      mt::check_nccl(ncclAllReduce(sq, sq, 2, ncclFloat32, ncclSum, c->pp, s), "ncclAllReduce(grad norm, pp)");
    mt::clip_coefficient(sq, d->grad_clip, sq + 2, s);
    const float lr = resolve_lr(*d);
    for (auto* l : st->layers) mt::layer_adamw(l, *d, lr, sq + 3, s);
    if (vocab_here) mt::vocab_adamw(st->vocab, *d, lr, sq + 3, s);
    if (grad_norm_out) {
      mt::check_cuda(cudaMemcpyAsync(grad_norm_out, sq + 2, sizeof(float), cudaMemcpyDeviceToHost, s), "D2H norm");
      mt::check_cuda(cudaStreamSynchronize(s), "sync");
    }
  });
}

extern "C" int mt_stage_set_recompute(mt_stage* st, int32_t enable) {
  return call([&] {
    if (!st) throw std::invalid_argument("null stage");
    for (auto* l : st->layers) ok(mt_layer_set_recompute(l, enable));
  });
}

extern "C" int mt_stage_attach_vocab(mt_stage* st, mt_vocab* v) {
  return call([&] {
    if (!st || !v) throw std::invalid_argument("null argument");
    if (mt::vocab_tokens(v) != st->M || mt::vocab_hidden(v) != st->h)
      throw std::invalid_argument("vocab shape (micro_batch * seq, hidden) does not match the stage");
    if (st->ctx->seq_parallel && st->ctx->par.tensor > 1)
      throw std::invalid_argument("the vocab module does not support sequence parallelism yet");
    if (mt::vocab_tp(v) != st->ctx->par.tensor && !st->ctx->shard_only)
      throw std::invalid_argument("vocab tp_size does not match the tensor-parallel degree");
    if (st->stages > 1 && !st->ctx->emb && (st->stage == 0 || st->stage == st->stages - 1))
      throw std::invalid_argument("pipeline-parallel vocab needs the embedding communicator (mt_ctx_init_comm)");
    st->vocab = v;
    const size_t tok_bytes = static_cast<size_t>(st->M * 4);
    if (st->stage == 0) {
      st->tokens.resize(st->mb_capacity);
      for (auto& b : st->tokens) b.ensure(tok_bytes);
    }
    // targets buffers (sized for bf16 activations) already hold M int32 ids
  });
}

extern "C" int mt_stage_set_step(mt_stage* st, uint64_t step) {
  return call([&] {
    if (!st) throw std::invalid_argument("null stage");
    st->step = step;
  });
}

extern "C" int mt_stage_get_step(const mt_stage* st, uint64_t* step) {
  return call([&] {
    if (!st || !step) throw std::invalid_argument("null argument");
    *step = st->step;
  });
}

extern "C" int mt_stage_set_micro_batches(mt_stage* st, int32_t micro_batches) {
  return call([&] {
    if (!st) throw std::invalid_argument("null stage");
    if (micro_batches < 1 || micro_batches > st->mb_capacity)
      throw std::invalid_argument("micro_batches must be in [1, " + std::to_string(st->mb_capacity) + "]");
    st->d.micro_batches = micro_batches;
  });
}

extern "C" int mt_stage_host_traffic(const mt_stage* st, int64_t* h2d_bytes, int64_t* d2h_bytes) {
  return call([&] {
    if (!st) throw std::invalid_argument("null stage");
    if (h2d_bytes) *h2d_bytes = st->h2d_bytes;
    if (d2h_bytes) *d2h_bytes = st->d2h_bytes;
  });
}
