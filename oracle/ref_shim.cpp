// ORACLE — test infrastructure only. C ABI over the REFERENCE's own planner
// (/root/reference/proj/src/planner.cpp, compiled unmodified from where it lies by oracle/Makefile
// into oracle/_ref/libcurator_ref.so). Same struct layouts as include/mtnlg.h, entry points
// prefixed ref_, so tests/test_planner_ref.py can diff the framework's curator:: planner against
// the reference bit-for-bit. Nothing in the product path links this.
#include <cstring>
#include <stdexcept>
#include <string>

#include "curator/errors.hpp"   // resolved to /root/reference/proj/include (first on the -I path)
#include "curator/blending.hpp"
#include "curator/planner.hpp"
#include "../include/mtnlg.h"

namespace {
thread_local std::string g_err;
template <class F>
int call(F&& f) {
  try {
    f();
    return 0;
  } catch (const curator::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
curator::ClusterTopology topo_of(const mt_cluster_topology* t) {
  curator::ClusterTopology o;
  o.nodes = t->nodes;
  o.gpus_per_node = t->gpus_per_node;
  o.intra_node_bw = t->intra_node_bw;
  o.inter_node_bw = t->inter_node_bw;
  o.peak_flops_per_gpu = t->peak_flops_per_gpu;
  return o;
}
curator::ParallelConfig par_of(const mt_parallel_config* p) {
  curator::ParallelConfig o;
  o.tensor = p->tensor;
  o.pipeline = p->pipeline;
  o.data = p->data;
  o.batch = p->batch;
  o.micro_batches = p->micro_batches;
  return o;
}
}  // namespace

extern "C" {
const char* ref_last_error(void) { return g_err.c_str(); }
int ref_map_topology(const mt_cluster_topology* topo, const mt_parallel_config* par, mt_rank_placement* out,
                     int64_t cap, int64_t* n) {
  return call([&] {
    const auto r = curator::map_topology(topo_of(topo), par_of(par));
    *n = (int64_t)r.size();
    for (int64_t i = 0; i < *n && i < cap; ++i) out[i] = {r[i].data, r[i].pipeline, r[i].tensor, r[i].node, r[i].gpu};
  });
}
int ref_pipeline_efficiency(int32_t mb, int32_t pp, double* out) {
  return call([&] { *out = curator::pipeline_efficiency(mb, pp); });
}
int ref_estimated_tflops_per_gpu(const mt_model_shape* s, const mt_parallel_config* p, const mt_cluster_topology* t,
                                 double secs, double* out) {
  return call([&] {
    curator::ModelShape m;
    m.parameters = s->parameters;
    m.layers = s->layers;
    m.hidden = s->hidden;
    m.heads = s->heads;
    m.sequence = s->sequence;
    m.vocab = s->vocab;
    *out = curator::estimated_tflops_per_gpu(m, par_of(p), topo_of(t), secs);
  });
}
int ref_weight_init_std(double h, double* out) { return call([&] { *out = curator::weight_init_std(h); }); }
int ref_activation_bytes(double b, double l, double s, double h, double* out) {
  return call([&] { *out = curator::activation_bytes(b, l, s, h); });
}
int ref_model_state_bytes(double p, double* out) { return call([&] { *out = curator::model_state_bytes(p); }); }
int ref_lr_at(double t, double* out) { return call([&] { *out = curator::lr_at(t); }); }
int ref_batch_size_at(double t, int32_t* out) { return call([&] { *out = curator::batch_size_at(t); }); }
int ref_plan_report(const char* path, int32_t as_json, char* out, int64_t cap, int64_t* len) {
  return call([&] {
    const auto in = curator::parse_planner_config(path);
    const std::string s = curator::render_plan_report(in, curator::build_plan_report(in), as_json != 0);
    *len = (int64_t)s.size();
    if (out && cap > 0) {
      const int64_t k = std::min<int64_t>(cap - 1, *len);
      std::memcpy(out, s.data(), (size_t)k);
      out[k] = '\0';
    }
  });
}
// Reference blending: `steps` batches over n datasets (weights normalised first when asked);
// counts [steps][n], credit [steps][n] after each step.
int ref_blend_run(int32_t n, const double* weights, int32_t normalize, uint64_t batch, int64_t steps,
                  uint64_t* counts, double* credit) {
  return call([&] {
    std::vector<curator::DatasetSpec> specs(n);
    for (int32_t i = 0; i < n; ++i) {
      specs[i].name = "d" + std::to_string(i);
      specs[i].weight = weights[i];
    }
    if (normalize) curator::normalize_weights(specs);
    auto st = curator::BlendState::create(n);
    for (int64_t t = 0; t < steps; ++t) {
      const auto c = curator::next_batch_composition(st, specs, batch);
      for (int32_t i = 0; i < n; ++i) {
        counts[t * n + i] = c[i];
        credit[t * n + i] = st.credit[i];
      }
    }
  });
}
}
