// C ABI over the curator:: planner and schedule (host, pure functions). Each entry maps the
// reference's exceptions onto status codes: std::invalid_argument / ConfigError -> 1, others -> 2.
#include <cstring>
#include <stdexcept>
#include <string>

#include "curator/errors.hpp"
#include "curator/planner.hpp"
#include "curator/schedule.hpp"
#include "mtnlg.h"

namespace mt {
void set_error(const std::string& e);
}  // namespace mt

namespace {

template <class F>
int call(F&& f) {
  try {
    f();
    return MT_OK;
  } catch (const curator::ConfigError& e) {
    mt::set_error(e.what());
    return MT_ERR_CONFIG;
  } catch (const std::invalid_argument& e) {
    mt::set_error(e.what());
    return MT_ERR_CONFIG;
  } catch (const std::exception& e) {
    mt::set_error(e.what());
    return MT_ERR_DATA;
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

void need(const void* p) {
  if (!p) throw std::invalid_argument("null argument");
}

}  // namespace

extern "C" int mt_map_topology(const mt_cluster_topology* topo, const mt_parallel_config* par, mt_rank_placement* out,
                               int64_t cap, int64_t* n) {
  return call([&] {
    need(topo);
    need(par);
    need(n);
    const auto ranks = curator::map_topology(topo_of(topo), par_of(par));
    *n = static_cast<int64_t>(ranks.size());
    for (int64_t i = 0; i < *n && i < cap; ++i) {
      out[i].data = ranks[i].data;
      out[i].pipeline = ranks[i].pipeline;
      out[i].tensor = ranks[i].tensor;
      out[i].node = ranks[i].node;
      out[i].gpu = ranks[i].gpu;
    }
  });
}

extern "C" int mt_pipeline_efficiency(int32_t mb, int32_t stages, double* out) {
  return call([&] {
    need(out);
    *out = curator::pipeline_efficiency(mb, stages);
  });
}

extern "C" int mt_estimated_tflops_per_gpu(const mt_model_shape* shape, const mt_parallel_config* par,
                                           const mt_cluster_topology* topo, double secs, double* out) {
  return call([&] {
    need(shape);
    need(par);
    need(topo);
    need(out);
    curator::ModelShape m;
    m.parameters = shape->parameters;
    m.layers = shape->layers;
    m.hidden = shape->hidden;
    m.heads = shape->heads;
    m.sequence = shape->sequence;
    m.vocab = shape->vocab;
    *out = curator::estimated_tflops_per_gpu(m, par_of(par), topo_of(topo), secs);
  });
}

extern "C" int mt_weight_init_std(double hidden, double* out) {
  return call([&] { *out = curator::weight_init_std(hidden); });
}
extern "C" int mt_activation_bytes(double b, double l, double s, double h, double* out) {
  return call([&] { *out = curator::activation_bytes(b, l, s, h); });
}
extern "C" int mt_model_state_bytes(double p, double* out) {
  return call([&] { *out = curator::model_state_bytes(p); });
}
extern "C" int mt_lr_at(double t, double* out) {
  return call([&] { *out = curator::lr_at(t); });
}
extern "C" int mt_batch_size_at(double t, int32_t* out) {
  return call([&] { *out = curator::batch_size_at(t); });
}

extern "C" int mt_plan_report(const char* path, int32_t as_json, char* out, int64_t cap, int64_t* len) {
  return call([&] {
    need(path);
    need(len);
    const auto in = curator::parse_planner_config(path);
    const std::string text = curator::render_plan_report(in, curator::build_plan_report(in), as_json != 0);
    *len = static_cast<int64_t>(text.size());
    if (out && cap > 0) {
      const int64_t k = std::min<int64_t>(cap - 1, *len);
      std::memcpy(out, text.data(), static_cast<size_t>(k));
      out[k] = '\0';
    }
  });
}

extern "C" int mt_pipeline_schedule(int32_t stage, int32_t stages, int32_t mb, mt_pipe_op* out, int32_t cap,
                                    int32_t* n) {
  return call([&] {
    need(n);
    const auto ops = curator::one_f_one_b(stage, stages, mb);
    *n = static_cast<int32_t>(ops.size());
    for (int32_t i = 0; i < *n && i < cap; ++i) {
      out[i].kind = static_cast<int32_t>(ops[i].kind);
      out[i].micro_batch = ops[i].micro_batch;
    }
  });
}

extern "C" int mt_pipeline_simulate(int32_t stages, int32_t mb, int32_t tf, int32_t tb, int64_t* makespan) {
  return call([&] {
    need(makespan);
    *makespan = curator::simulate_one_f_one_b(stages, mb, tf, tb);
  });
}
