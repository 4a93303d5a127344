// C ABI over the eps:: control plane (include/eps_capi.h).
//
// Compiled twice: against this repo's eps:: implementation (product) and,
// with -DEPS_REFERENCE_BUILD -DEPS_CAPI_PREFIX=epsref_, against the
// reference's own sources (oracle/_ref).  That this one file builds against
// both proves the API is source-compatible with the reference.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "eps/autocache.hpp"
#include "eps/autodp.hpp"
#include "eps/autopipe.hpp"
#include "eps/chunks.hpp"
#include "eps/freeze.hpp"
#include "eps/model.hpp"
#include "eps/runner.hpp"
#include "eps/scenario.hpp"
#include "eps/schedule.hpp"
#include "eps_capi.h"

struct eps_freeze {
  eps::FreezeState state;
};
struct eps_scenario {
  eps::ScenarioConfig cfg;
};
#ifndef EPS_REFERENCE_BUILD
struct eps_planner {
  std::unique_ptr<eps::EpochPlanner> planner;
  std::unique_ptr<eps::GradNormSource> scenario_norms;
  std::unique_ptr<eps::RecordedNormSource> recorded;
};
#endif

namespace {

thread_local std::string g_last_error;

}  // namespace

#ifndef EPS_REFERENCE_BUILD
namespace eps {
// error text for the runtime's C entry points (trainer.cpp)
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace eps
#endif

namespace {

template <typename F>
int guarded(F&& body) {
  try {
    body();
    g_last_error.clear();
    return EPS_OK;
  } catch (const eps::ConfigError& e) {
    g_last_error = e.what();
    return EPS_ECONFIG;
  } catch (const eps::IoError& e) {
    g_last_error = e.what();
    return EPS_EIO;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return EPS_EINVAL;
  } catch (const std::domain_error& e) {
    g_last_error = e.what();
    return EPS_EDOMAIN;
  } catch (const std::length_error& e) {
    g_last_error = e.what();
    return EPS_ECAPACITY;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return EPS_ELOGIC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return EPS_EOTHER;
  } catch (...) {
    g_last_error = "unknown exception";
    return EPS_EOTHER;
  }
}

void need_ptr(const void* p, const char* what) {
  if (p == nullptr) throw std::invalid_argument(std::string(what) + " must not be NULL");
}

void need_cap(long have, long want, const char* what) {
  if (have < want)
    throw std::length_error(std::string(what) + ": buffer holds " + std::to_string(have) +
                            ", need " + std::to_string(want));
}

eps::ModelSpec to_model(const eps_model_t* m) {
  need_ptr(m, "model");
  eps::ModelSpec s;
  s.name = "capi";
  s.attention_params.assign(m->attention_params, m->attention_params + m->layers);
  s.mlp_params.assign(m->mlp_params, m->mlp_params + m->layers);
  s.activation_bytes.assign(m->activation_bytes, m->activation_bytes + 2 * m->layers + 1);
  s.bytes_per_param = m->bytes_per_param;
  return s;
}

eps::ClusterSpec to_cluster(const eps_cluster_t* c) {
  need_ptr(c, "cluster");
  eps::ClusterSpec s;
  s.node_count = c->node_count;
  s.gpus_per_node = c->gpus_per_node;
  s.gpu_memory_bytes = c->gpu_memory_bytes;
  s.intra_node_bandwidth = c->intra_node_bandwidth;
  s.inter_node_bandwidth = c->inter_node_bandwidth;
  return s;
}

eps::CostModel to_cost(const eps_cost_model_t* c) {
  need_ptr(c, "cost model");
  eps::CostModel s;
  s.c_fwd = c->c_fwd;
  s.backward_ratio = c->backward_ratio;
  s.c_update = c->c_update;
  s.per_microbatch_overhead = c->per_microbatch_overhead;
  s.allreduce_bucket_bytes = c->allreduce_bucket_bytes;
  s.comm_latency = c->comm_latency;
  return s;
}

eps::CacheTierParams to_tiers(const eps_cache_tiers_t* t) {
  need_ptr(t, "cache tiers");
  eps::CacheTierParams s;
  s.host_bandwidth = t->host_bandwidth;
  s.disk_bandwidth = t->disk_bandwidth;
  s.host_capacity_bytes = t->host_capacity_bytes;
  s.window_batches = t->window_batches;
  s.block_batches = t->block_batches;
  s.read_latency = t->read_latency;
  return s;
}

eps::SublayerSeq to_seq(const eps_seq_t* q) {
  need_ptr(q, "seq");
  eps::SublayerSeq s;
  s.frozen_params = q->frozen_params;
  s.frozen_layers = q->frozen_layers;
  for (int i = 0; i < q->n; ++i) {
    const int g = q->global_index ? q->global_index[i] : 2 * q->frozen_layers + i;
    eps::Sublayer sl;
    sl.kind = (g % 2 == 0) ? eps::SublayerKind::kAttention : eps::SublayerKind::kMlp;
    sl.layer_index = g / 2;
    sl.params = q->params[i];
    s.active.push_back(sl);
  }
  return s;
}

eps::PartitionPlan to_plan(const eps_plan_t* p) {
  need_ptr(p, "plan");
  eps::PartitionPlan s;
  s.pipeline_length = p->pipeline_length;
  for (int k = 0; k < p->pipeline_length; ++k) {
    eps::PartitionSpan sp;
    sp.begin = p->begin[k];
    sp.end = p->end[k];
    s.spans.push_back(sp);
    s.sublayer_counts.push_back(p->end[k] - p->begin[k]);
    s.param_sums.push_back(p->param_sums[k]);
    s.effective_sizes.push_back(p->effective_sizes[k]);
  }
  s.frozen_params = p->frozen_params;
  s.frozen_layers = p->frozen_layers;
  s.lambda_frozen = p->lambda_frozen;
  return s;
}

void from_plan(const eps::PartitionPlan& s, eps_plan_t* p) {
  need_ptr(p, "plan out");
  need_cap(EPS_MAX_STAGES, s.pipeline_length, "plan stages");
  std::memset(p, 0, sizeof(*p));
  p->pipeline_length = s.pipeline_length;
  for (int k = 0; k < s.pipeline_length; ++k) {
    p->begin[k] = s.spans[k].begin;
    p->end[k] = s.spans[k].end;
    p->param_sums[k] = s.param_sums[k];
    p->effective_sizes[k] = s.effective_sizes[k];
  }
  p->frozen_params = s.frozen_params;
  p->frozen_layers = s.frozen_layers;
  p->lambda_frozen = s.lambda_frozen;
}

void from_summary(const eps::IterationSchedule& s, eps_schedule_summary_t* o) {
  o->makespan = s.makespan;
  o->compute_makespan = s.compute_makespan;
  o->makespan_without_ar = s.makespan_without_ar;
  o->total_bubble = s.total_bubble;
  o->allreduce_seconds = s.allreduce_seconds;
  o->transfer_seconds = s.transfer_seconds;
  o->compute_seconds = s.compute_seconds;
  o->exposed_comm = s.exposed_comm;
  o->n_blocks = static_cast<int>(s.blocks.size());
}

void from_msg(const eps::TransitionMessage& m, eps_msg_t* o) {
  std::memset(o, 0, sizeof(*o));
  o->sender = m.sender;
  o->receiver = m.receiver;
  o->epoch = m.epoch;
  o->lr_schedule_position = m.lr_schedule_position;
  o->frozen_layers = m.frozen_layers;
  o->new_pipeline_length = m.new_pipeline_length;
  o->span_first = m.assigned_span.first;
  o->span_length = m.assigned_span.length;
  std::strncpy(o->weights_version, m.weights_version.c_str(), sizeof(o->weights_version) - 1);
}

void copy_out(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf == nullptr) return;  // size query
  need_cap(static_cast<long>(cap), static_cast<long>(s.size() + 1), "string");
  std::memcpy(buf, s.c_str(), s.size() + 1);
}

}  // namespace

#ifndef EPS_REFERENCE_BUILD
// Error text for the entry points implemented outside this file (comm.cpp).
namespace eps_detail {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace eps_detail
#endif

extern "C" {

const char* EPS_FN(last_error)(void) { return g_last_error.c_str(); }

int EPS_FN(model_preset)(const char* name, int64_t* att, int64_t* mlp, int64_t* act,
                         int cap_layers, int* layers) {
  return guarded([&] {
    need_ptr(name, "name");
    const std::string n(name);
    eps::ModelSpec m;
    if (n == "vit-b16") m = eps::vit_b16();
    else if (n == "bert-large") m = eps::bert_large();
    else throw std::invalid_argument("unknown preset '" + n + "'");
    if (layers) *layers = m.layer_count();
    if (att == nullptr) return;
    need_cap(cap_layers, m.layer_count(), "preset layers");
    for (int i = 0; i < m.layer_count(); ++i) {
      att[i] = m.attention_params[i];
      mlp[i] = m.mlp_params[i];
    }
    for (int g = 0; g <= 2 * m.layer_count(); ++g) act[g] = m.activation_bytes[g];
  });
}

int EPS_FN(model_validate)(const eps_model_t* model) {
  return guarded([&] { to_model(model).validate(); });
}

int EPS_FN(model_prefix_params)(const eps_model_t* model, int layer, int64_t* out) {
  return guarded([&] { *out = to_model(model).prefix_params(layer); });
}

int EPS_FN(m_partition)(const eps_model_t* model, int l_frozen, int64_t* params,
                        int* global_index, int cap, int* n, int64_t* frozen_params) {
  return guarded([&] {
    const eps::SublayerSeq s = eps::m_partition(to_model(model), l_frozen);
    const int count = static_cast<int>(s.active.size());
    need_cap(cap, count, "m_partition");
    for (int i = 0; i < count; ++i) {
      params[i] = s.active[i].params;
      if (global_index) global_index[i] = s.active[i].global_index();
    }
    *n = count;
    if (frozen_params) *frozen_params = s.frozen_params;
  });
}

int EPS_FN(freeze_create)(double alpha, eps_freeze_t** out) {
  return guarded([&] {
    need_ptr(out, "out");
    *out = new eps_freeze{eps::FreezeState(alpha)};
  });
}

void EPS_FN(freeze_destroy)(eps_freeze_t* state) { delete state; }

int EPS_FN(freeze_frozen_count)(const eps_freeze_t* state, int* out) {
  return guarded([&] {
    need_ptr(state, "state");
    *out = state->state.frozen_count();
  });
}

int EPS_FN(next_frozen_count)(eps_freeze_t* state, const double* norms, int n_norms,
                              int layer_count, int* out, double* raw_bound) {
  return guarded([&] {
    need_ptr(state, "state");
    eps::GradNormVector v;
    v.norms.assign(norms, norms + n_norms);
    *out = eps::next_frozen_count(state->state, v, layer_count);
    if (raw_bound) *raw_bound = state->state.history().back().raw_bound;
  });
}

int EPS_FN(frozen_bound_closed_form)(int timestep, int layer_count, double alpha, double* out) {
  return guarded([&] { *out = eps::frozen_bound_closed_form(timestep, layer_count, alpha); });
}

int EPS_FN(synthetic_norms)(int profile, uint64_t seed, int layers, int switchover_epoch,
                            int epoch, double* out) {
  return guarded([&] {
    const eps::SyntheticNormSource src(profile == 1 ? eps::SyntheticProfile::kEarlyRandom
                                                    : eps::SyntheticProfile::kMonotoneConverging,
                                       seed, layers, switchover_epoch);
    const eps::GradNormVector v = src.at_epoch(epoch);
    for (int l = 0; l < layers; ++l) out[l] = v.norms[l];
  });
}

int EPS_FN(trace_norms)(const char* csv_path, int epoch, double* out, int cap, int* layers) {
  return guarded([&] {
    need_ptr(csv_path, "path");
    const eps::TraceNormSource src{std::string(csv_path)};
    if (layers) *layers = src.layer_count();
    if (out == nullptr) return;
    need_cap(cap, src.layer_count(), "trace norms");
    const eps::GradNormVector v = src.at_epoch(epoch);
    for (int l = 0; l < src.layer_count(); ++l) out[l] = v.norms[l];
  });
}

int EPS_FN(load_balance)(const eps_seq_t* seq, int partitions, double lambda_frozen,
                         int criterion, eps_plan_t* out) {
  return guarded([&] {
    const auto crit = criterion == 1 ? eps::BalanceCriterion::kPaperVariance
                                     : eps::BalanceCriterion::kNormalizedStddev;
    from_plan(eps::load_balance(to_seq(seq), partitions, lambda_frozen, crit), out);
  });
}

int EPS_FN(try_compress)(const eps_seq_t* seq, int current_k, double lambda_frozen,
                         double m_gpu_initial, int criterion, eps_plan_t* out, int* attempt_k,
                         double* attempt_max_eff, int attempt_cap, int* n_attempts) {
  return guarded([&] {
    const auto crit = criterion == 1 ? eps::BalanceCriterion::kPaperVariance
                                     : eps::BalanceCriterion::kNormalizedStddev;
    const eps::CompressionResult r =
        eps::try_compress(to_seq(seq), current_k, lambda_frozen, m_gpu_initial, crit);
    from_plan(r.plan, out);
    out->pipeline_length = r.pipeline_length;
    const int na = static_cast<int>(r.attempts.size());
    if (n_attempts) *n_attempts = na;
    if (attempt_k) {
      need_cap(attempt_cap, na, "attempts");
      for (int i = 0; i < na; ++i) {
        attempt_k[i] = r.attempts[i].first;
        attempt_max_eff[i] = r.attempts[i].second;
      }
    }
  });
}

int EPS_FN(build_schedule)(const eps_stage_load_t* stages, int n_stages, int micro_batches,
                           double per_pipeline_batch, int integer_microbatches,
                           int replica_width, int group_spans_nodes, double intra_bandwidth,
                           double inter_bandwidth, int bytes_per_param,
                           const eps_cost_model_t* cm, eps_schedule_summary_t* summary,
                           double* bubble_per_device, eps_block_t* blocks, int block_cap) {
  return guarded([&] {
    eps::ScheduleRequest req;
    for (int d = 0; d < n_stages; ++d) {
      eps::StageLoad s;
      s.fwd_params = stages[d].fwd_params;
      s.bwd_params = stages[d].bwd_params;
      s.prefix_seconds_per_sample = stages[d].prefix_seconds_per_sample;
      s.in_bytes_per_sample = stages[d].in_bytes_per_sample;
      req.stages.push_back(s);
    }
    req.micro_batches = micro_batches;
    req.per_pipeline_batch = per_pipeline_batch;
    req.integer_microbatches = integer_microbatches != 0;
    req.replica_width = replica_width;
    req.group_spans_nodes = group_spans_nodes != 0;
    req.intra_bandwidth = intra_bandwidth;
    req.inter_bandwidth = inter_bandwidth;
    req.bytes_per_param = bytes_per_param;
    const eps::IterationSchedule s = eps::build_schedule(req, to_cost(cm));
    from_summary(s, summary);
    if (bubble_per_device)
      for (std::size_t d = 0; d < s.bubble_per_device.size(); ++d)
        bubble_per_device[d] = s.bubble_per_device[d];
    if (blocks) {
      need_cap(block_cap, static_cast<long>(s.blocks.size()), "blocks");
      for (std::size_t i = 0; i < s.blocks.size(); ++i) {
        const eps::TimedBlock& b = s.blocks[i];
        blocks[i] = eps_block_t{b.device, static_cast<int>(b.kind), b.start, b.end,
                                b.micro_batch, b.bucket};
      }
    }
  });
}

int EPS_FN(schedule_iteration)(const eps_plan_t* plan, const eps_model_t* model,
                               const eps_seq_t* seq, int micro_batches,
                               double per_pipeline_batch, int replica_width,
                               const eps_cluster_t* cluster, const eps_cost_model_t* cm,
                               int cache_enabled, double cache_read_seconds_per_sample,
                               eps_schedule_summary_t* summary) {
  return guarded([&] {
    const eps::IterationSchedule s = eps::schedule_iteration(
        to_plan(plan), to_model(model), to_seq(seq), micro_batches, per_pipeline_batch,
        replica_width, to_cluster(cluster), to_cost(cm), cache_enabled != 0,
        cache_read_seconds_per_sample);
    from_summary(s, summary);
  });
}

int EPS_FN(optimal_chunks)(const eps_plan_t* plan, const eps_model_t* model,
                           const eps_seq_t* seq, double per_pipeline_batch, int replica_width,
                           const eps_cluster_t* cluster, const eps_cost_model_t* cm,
                           int cache_enabled, double cache_read_seconds_per_sample,
                           int* chosen, double* times_out, int times_cap) {
  return guarded([&] {
    const eps::ChunkProfile p = eps::optimal_chunks(
        to_plan(plan), to_model(model), to_seq(seq), per_pipeline_batch, replica_width,
        to_cluster(cluster), to_cost(cm), cache_enabled != 0, cache_read_seconds_per_sample);
    *chosen = p.chosen;
    if (times_out) {
      need_cap(times_cap, static_cast<long>(p.modeled_times.size()), "times");
      for (std::size_t i = 0; i < p.modeled_times.size(); ++i)
        times_out[i] = p.modeled_times[i].second;
    }
  });
}

int EPS_FN(topology)(const eps_cluster_t* cluster, int pipeline_length, int* active_ranks,
                     int cap, int* n_active, int* replica_width) {
  return guarded([&] {
    const eps::Topology t(to_cluster(cluster), pipeline_length);
    t.validate();
    const std::vector<int> a = t.active_ranks();
    if (n_active) *n_active = static_cast<int>(a.size());
    if (replica_width) *replica_width = t.replica_width();
    if (active_ranks) {
      need_cap(cap, static_cast<long>(a.size()), "active ranks");
      for (std::size_t i = 0; i < a.size(); ++i) active_ranks[i] = a[i];
    }
  });
}

int EPS_FN(transition)(const eps_cluster_t* cluster, int old_k, int new_k, int epoch,
                       double lr_schedule_position, int frozen_layers,
                       const char* weights_version, eps_msg_t* msgs, int cap, int* n) {
  return guarded([&] {
    const eps::Topology t(to_cluster(cluster), old_k);
    eps::TrainingProgress p;
    p.epoch = epoch;
    p.lr_schedule_position = lr_schedule_position;
    p.frozen_layers = frozen_layers;
    if (weights_version) p.weights_version = weights_version;
    const eps::TransitionResult r = eps::transition(t, new_k, p);
    *n = static_cast<int>(r.messages.size());
    if (msgs) {
      need_cap(cap, *n, "messages");
      for (int i = 0; i < *n; ++i) from_msg(r.messages[i], &msgs[i]);
    }
  });
}

int EPS_FN(redistribute)(int64_t dataset_size, const eps_cluster_t* cluster,
                         int pipeline_length, int epoch, uint64_t seed, int* ranks,
                         int64_t* offsets, int64_t* ids) {
  return guarded([&] {
    const eps::Topology t(to_cluster(cluster), pipeline_length);
    const eps::ShardAssignment a = eps::redistribute(dataset_size, t, epoch, seed);
    int64_t at = 0;
    for (std::size_t s = 0; s < a.shards.size(); ++s) {
      if (ranks) ranks[s] = a.ranks[s];
      if (offsets) offsets[s] = at;
      if (ids) std::memcpy(ids + at, a.shards[s].data(), a.shards[s].size() * sizeof(int64_t));
      at += static_cast<int64_t>(a.shards[s].size());
    }
    if (offsets) offsets[a.shards.size()] = at;
  });
}

int EPS_FN(ddp_skip_set)(const eps_plan_t* plan, const eps_seq_t* seq, int* global_index,
                         int cap, int* n, int64_t* param_count) {
  return guarded([&] {
    const eps::DdpParticipants p = eps::ddp_skip_set(to_plan(plan), to_seq(seq));
    *n = static_cast<int>(p.sublayer_global_indices.size());
    if (param_count) *param_count = p.param_count;
    if (global_index) {
      need_cap(cap, *n, "ddp participants");
      for (int i = 0; i < *n; ++i) global_index[i] = p.sublayer_global_indices[i];
    }
  });
}

int EPS_FN(cache_read_seconds_per_sample)(const eps_model_t* model, int boundary_layer,
                                          const eps_cache_tiers_t* tiers, double* out) {
  return guarded([&] {
    *out = eps::cache_read_seconds_per_sample(to_model(model), boundary_layer, to_tiers(tiers));
  });
}

int EPS_FN(should_cache)(int l_frozen, const eps_model_t* model, const eps_cost_model_t* cm,
                         const eps_cache_tiers_t* tiers, double microbatch_samples, int* enable,
                         double* read_seconds, double* forward_seconds) {
  return guarded([&] {
    const eps::CacheDecision d = eps::should_cache(l_frozen, to_model(model), to_cost(cm),
                                                   to_tiers(tiers), microbatch_samples);
    *enable = d.enable ? 1 : 0;
    if (read_seconds) *read_seconds = d.read_seconds_per_microbatch;
    if (forward_seconds) *forward_seconds = d.forward_seconds_per_microbatch;
  });
}

int EPS_FN(cache_transition)(int enabled, int boundary_layer, const eps_cache_tiers_t* tiers,
                             int old_boundary, int new_boundary, const eps_model_t* model,
                             const eps_cost_model_t* cm, double* read_s, double* compute_s,
                             double* write_s) {
  return guarded([&] {
    eps::CacheState st;
    st.enabled = enabled != 0;
    st.boundary_layer = boundary_layer;
    st.tiers = to_tiers(tiers);
    const auto r =
        eps::cache_transition(st, old_boundary, new_boundary, to_model(model), to_cost(cm));
    *read_s = r.second.read_seconds_per_sample;
    *compute_s = r.second.compute_seconds_per_sample;
    *write_s = r.second.write_seconds_per_sample;
  });
}

int EPS_FN(cache_tier_epoch)(const eps_cache_tiers_t* tiers, double bytes_per_batch,
                             int total_batches, double iteration_seconds, double* out) {
  return guarded([&] {
    need_ptr(out, "out");
    eps::CacheTierSim sim(to_tiers(tiers), bytes_per_batch, total_batches);
    double now = 0.0;
    int prefetches = 0, evictions = 0;
    for (int b = 0; b < total_batches; ++b) {
      const eps::WindowStep step = sim.advance(b, now);
      now += iteration_seconds + step.stall_seconds;
      for (const eps::TierAction& a : step.actions) {
        if (a.kind == eps::TierAction::Kind::kPrefetch) ++prefetches;
        if (a.kind == eps::TierAction::Kind::kEvict) ++evictions;
      }
    }
    out[0] = sim.total_stall();
    out[1] = sim.max_resident_bytes();
    out[2] = prefetches;
    out[3] = evictions;
    out[4] = sim.sliding() ? 1.0 : 0.0;
  });
}

int EPS_FN(scenario_load)(const char* path, eps_scenario_t** out) {
  return guarded([&] {
    need_ptr(path, "path");
    *out = new eps_scenario{eps::load_scenario(path)};
  });
}

int EPS_FN(scenario_parse)(const char* json_text, eps_scenario_t** out) {
  return guarded([&] {
    need_ptr(json_text, "json");
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(json_text);
    } catch (const nlohmann::json::parse_error& e) {
      throw eps::ConfigError(std::string("(text): ") + e.what());
    }
    *out = new eps_scenario{eps::parse_scenario(j)};
  });
}

void EPS_FN(scenario_destroy)(eps_scenario_t* cfg) { delete cfg; }

int EPS_FN(scenario_to_json)(const eps_scenario_t* cfg, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    need_ptr(cfg, "scenario");
    copy_out(eps::scenario_to_json(cfg->cfg).dump(), buf, cap, len);
  });
}

int EPS_FN(simulate_run)(const eps_scenario_t* cfg, eps_epoch_row_t* rows, int cap,
                         eps_run_summary_t* summary) {
  return guarded([&] {
    need_ptr(cfg, "scenario");
    const eps::RunResult r = eps::simulate_run(cfg->cfg);
    if (summary) {
      summary->total_seconds = r.total_seconds;
      summary->baseline_total_seconds = r.baseline_total_seconds;
      summary->speedup = r.speedup;
      summary->comm_ratio = r.comm_ratio;
      summary->frozen_forward_per_sample = r.frozen_forward_per_sample;
      summary->final_prefix_forward_per_sample = r.final_prefix_forward_per_sample;
      summary->n_epochs = static_cast<int>(r.epochs.size());
      summary->n_transitions = static_cast<int>(r.transitions.size());
      summary->n_cache_events = static_cast<int>(r.cache_events.size());
    }
    if (rows) {
      need_cap(cap, static_cast<long>(r.epochs.size()), "epoch rows");
      for (std::size_t i = 0; i < r.epochs.size(); ++i) {
        const eps::EpochRow& e = r.epochs[i];
        rows[i] = eps_epoch_row_t{e.epoch,          e.l_frozen,       e.pipeline_length,
                                  e.replica_width,  e.micro_batches,  e.iteration_time,
                                  e.epoch_time,     e.throughput,     e.bubble_time,
                                  e.comm_time,      e.exposed_comm_time,
                                  e.cache_enabled ? 1 : 0,            e.transition_overhead,
                                  e.cache_transition_time,            e.stall_time};
      }
    }
  });
}

int EPS_FN(simulate_report)(const eps_scenario_t* cfg, int kind, char* buf, size_t cap,
                            size_t* len) {
  return guarded([&] {
    need_ptr(cfg, "scenario");
    const eps::RunResult r = eps::simulate_run(cfg->cfg);
    std::string s;
    switch (kind) {
      case 0: s = eps::report_csv(r); break;
      case 1: s = eps::timeline_to_json(r).dump(); break;
      case 2: s = eps::summary_to_json(cfg->cfg, r).dump(); break;
      case 3: s = eps::transitions_to_jsonl(r); break;
      default: throw std::invalid_argument("simulate_report: kind must be 0..3");
    }
    copy_out(s, buf, cap, len);
  });
}

int EPS_FN(speedup_breakdown)(const eps_scenario_t* cfg, double* total_seconds,
                              double* avg_throughput, double* speedup) {
  return guarded([&] {
    need_ptr(cfg, "scenario");
    const std::vector<eps::BreakdownRow> rows = eps::speedup_breakdown(cfg->cfg);
    for (std::size_t i = 0; i < rows.size(); ++i) {
      total_seconds[i] = rows[i].total_seconds;
      avg_throughput[i] = rows[i].avg_throughput;
      speedup[i] = rows[i].speedup_vs_baseline;
    }
  });
}

int EPS_FN(parse_flags)(const char* list, int* freeze, int* autopipe, int* autodp,
                        int* autocache) {
  return guarded([&] {
    need_ptr(list, "list");
    const eps::FeatureFlags f = eps::parse_flags(list);
    *freeze = f.freeze;
    *autopipe = f.autopipe;
    *autodp = f.autodp;
    *autocache = f.autocache;
  });
}

#ifndef EPS_REFERENCE_BUILD

int eps_planner_create(const eps_scenario_t* cfg, eps_planner_t** out) {
  return guarded([&] {
    need_ptr(cfg, "scenario");
    auto p = std::make_unique<eps_planner>();
    p->planner = std::make_unique<eps::EpochPlanner>(cfg->cfg);
    if (cfg->cfg.features.freeze) p->scenario_norms = eps::make_grad_norm_source(cfg->cfg);
    p->recorded = std::make_unique<eps::RecordedNormSource>(cfg->cfg.model.layer_count());
    *out = p.release();
  });
}

void eps_planner_destroy(eps_planner_t* p) { delete p; }

int eps_planner_begin_epoch(eps_planner_t* p, int epoch, const double* norms_prev,
                            int n_norms, eps_epoch_decision_t* out) {
  return guarded([&] {
    need_ptr(p, "planner");
    const eps::GradNormSource* src = p->scenario_norms.get();
    if (norms_prev != nullptr && epoch > 0) {
      p->recorded->record(epoch - 1, std::vector<double>(norms_prev, norms_prev + n_norms));
      src = p->recorded.get();
    }
    const eps::EpochDecision d = p->planner->begin_epoch(epoch, src);
    out->epoch = d.epoch;
    out->l_frozen = d.l_frozen;
    out->pipeline_length = d.pipeline_length;
    out->replica_width = d.replica_width;
    out->micro_batches = d.micro_batches;
    out->plan_changed = d.plan_changed;
    out->cache_enabled = d.cache_enabled;
    out->cache_boundary = d.cache_boundary;
    out->cache_old_boundary = d.cache_old_boundary;
    out->cache_moved = d.cache_moved;
    out->n_messages = static_cast<int>(d.messages.size());
    from_plan(d.plan, &out->plan);
  });
}

int eps_scenario_model(const eps_scenario_t* cfg, int64_t* att, int64_t* mlp, int64_t* act,
                       int cap_layers, int* layers, int* bytes_per_param) {
  return guarded([&] {
    need_ptr(cfg, "scenario");
    const eps::ModelSpec& m = cfg->cfg.model;
    if (layers) *layers = m.layer_count();
    if (bytes_per_param) *bytes_per_param = m.bytes_per_param;
    if (att == nullptr) return;
    need_cap(cap_layers, m.layer_count(), "layers");
    for (int i = 0; i < m.layer_count(); ++i) {
      att[i] = m.attention_params[i];
      mlp[i] = m.mlp_params[i];
    }
    for (int g = 0; g <= 2 * m.layer_count(); ++g) act[g] = m.activation_bytes[g];
  });
}

namespace {
void emit_profile(const eps::ModelSpec& m, int64_t* att, int64_t* mlp, int64_t* act) {
  for (int i = 0; i < m.layer_count(); ++i) {
    att[i] = m.attention_params[i];
    mlp[i] = m.mlp_params[i];
  }
  for (int g = 0; g <= 2 * m.layer_count(); ++g) act[g] = m.activation_bytes[g];
}
}  // namespace

int eps_vit_profile(int layers, int64_t hidden, int64_t mlp_dim, int image, int patch,
                    int channels, int64_t classes, int64_t* att, int64_t* mlp, int64_t* act) {
  return guarded([&] {
    emit_profile(eps::profile_from_dims(eps::vit_dims("vit", layers, hidden, mlp_dim, image,
                                                      patch, channels, classes)),
                 att, mlp, act);
  });
}

int eps_bert_profile(int layers, int64_t hidden, int64_t mlp_dim, int64_t seq_len,
                     int64_t position_table, int64_t vocab, int64_t head_params, int64_t* att,
                     int64_t* mlp, int64_t* act) {
  return guarded([&] {
    emit_profile(eps::profile_from_dims(eps::bert_dims("bert", layers, hidden, mlp_dim, seq_len,
                                                       position_table, vocab, head_params)),
                 att, mlp, act);
  });
}

int eps_microbatch_sizes(int per_pipeline_batch, int micro_batches, int* sizes) {
  return guarded([&] {
    const std::vector<int> s = eps::microbatch_sizes(per_pipeline_batch, micro_batches);
    for (std::size_t i = 0; i < s.size(); ++i) sizes[i] = s[i];
  });
}

int eps_plan_buckets(const int64_t* stage_params, int n_stages, int bytes_per_param,
                     double bucket_bytes, int* slice_bucket, int* slice_stage,
                     int64_t* slice_offset, int64_t* slice_count, int cap, int* n_slices,
                     int* n_buckets) {
  return guarded([&] {
    const std::vector<eps::GradBucket> b = eps::plan_buckets(
        std::vector<int64_t>(stage_params, stage_params + n_stages), bytes_per_param,
        bucket_bytes);
    int at = 0;
    for (std::size_t i = 0; i < b.size(); ++i)
      for (const eps::BucketSlice& s : b[i].slices) {
        need_cap(cap, at + 1, "bucket slices");
        slice_bucket[at] = static_cast<int>(i);
        slice_stage[at] = s.stage;
        slice_offset[at] = s.offset;
        slice_count[at] = s.count;
        ++at;
      }
    *n_slices = at;
    *n_buckets = static_cast<int>(b.size());
  });
}

int eps_grid_coord(const eps_cluster_t* cluster, int pipeline_length, int global_rank,
                   int* replica, int* stage) {
  return guarded([&] {
    const eps::GridCoord c =
        eps::grid_coord(eps::Topology(to_cluster(cluster), pipeline_length), global_rank);
    *replica = c.replica;
    *stage = c.stage;
  });
}

#endif  // EPS_REFERENCE_BUILD

}  // extern "C"
