// Native single-GPU training loop: the reference's epoch loop
// (runner.cpp:simulate_run, decision order of EpochPlanner) executed on the
// device by the ViT or BERT stage executor, with no Python on the path.
//
// Per epoch (runner.cpp:139-298, trainer.py:run_epoch for K = R = 1):
//   decision = EpochPlanner::begin_epoch(epoch, norms of the previous epoch)
//              (RecordedNormSource: the device's per-layer gradient norms)
//   shard    = redistribute(dataset, topology, epoch, seed)  (autodp.cpp:113-151)
//   AutoCache mode from the decision (autocache.cpp / runner.cpp:186-213):
//     off -> 0, boundary move -> 2 (forward [old, new) and write the store),
//     boundary trailing L_frozen -> 3, steady gather -> 1
//   per iteration (full batches, then a ragged last one, runner.cpp:245):
//     gather the batch's images by sample id (device; labels in epoch order), per
//     micro-batch: stage front (frozen prefix or cache gather / scatter),
//     active span forward, loss head; backward of the active span in reverse
//     micro-batch order; on the last iteration the per-layer gradient norms
//     (segmented fp64 sum of squares); SGD over the trainable tail.
//   measured columns: epoch / iteration time (CUDA events), the cache
//   transition (front work of a boundary-move epoch over a steady gather).
//
// Multi-rank runs (K > 1 pipelines, R > 1 replicas) stay with the Python
// choreography (pipeline.py / trainer.py) over the same C ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "eps/autodp.hpp"
#include "eps/freeze.hpp"
#include "eps/runner.hpp"
#include "eps/scenario.hpp"
#include "eps_capi.h"

struct eps_scenario {
  eps::ScenarioConfig cfg;
};

namespace eps {
void set_last_error(const std::string& msg);  // capi_control.cpp
}

namespace {

constexpr int kGeom = 11;  // eps_vit_layout geometry ints

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void eps_check(int rc, const char* what) {
  if (rc != EPS_OK) throw std::runtime_error(std::string(what) + " failed (status " +
                                             std::to_string(rc) + ")");
}

// SplitMix64 (the same generator the reference seeds its shuffles with).
struct SplitMix {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }  // [0, 1)
  double normal() {  // Box-Muller
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    release();
    n = count;
    if (count) cuda_check(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

}  // namespace

struct eps_trainer {
  eps::ScenarioConfig cfg;
  int kind = 0;  // EPS_MODEL_VIT / EPS_MODEL_BERT
  int geom[kGeom];
  int layers = 0, tokens = 0, hidden = 0, batch = 0, iters = 0;
  int64_t image_elems = 0;  // ViT: fp32 per sample
  bool qa = false;          // BERT SQuAD span head: labels are (start, end) pairs
  uint64_t seed = 0;
  float lr = 0.f, momentum = 0.f;
  int64_t dataset = 0;
  int64_t param_total = 0;
  std::vector<int64_t> segments;
  std::unique_ptr<eps::EpochPlanner> planner;
  std::unique_ptr<eps::GradNormSource> scenario_norms;
  std::unique_ptr<eps::RecordedNormSource> recorded;
  std::vector<double> norms_prev;
  bool device_norms = true;
  DevBuf<float> p32, g32, mom;
  DevBuf<uint16_t> p16;
  DevBuf<uint8_t> ws;
  DevBuf<float> images, xb, loss;   // ViT dataset / batch
  DevBuf<int64_t> tok, segs, tb;  // BERT dataset [N][T] x 2, batch [2][b][T]
  DevBuf<int64_t> yb, shard;
  std::vector<int64_t> labels_host;  // [N] (class) or [N][2] (start, end), host side
  DevBuf<double> sq;
  DevBuf<uint16_t> store;  // AutoCache store: dataset x (tokens * hidden) bf16
  eps_vit_t* ex = nullptr;
  eps_bert_t* bx = nullptr;
  cudaStream_t st = nullptr;

  ~eps_trainer() {
    if (ex) eps_vit_destroy(ex);
    if (bx) eps_bert_destroy(bx);
    if (st) cudaStreamDestroy(st);
  }
  bool bert() const { return kind == EPS_MODEL_BERT; }
  // executor calls shared by both families
  void set_cache_shards() {
    eps_check(bert() ? eps_bert_set_cache_shards(bx, nullptr, 0)
                     : eps_vit_set_cache_shards(ex, nullptr, 0),
              "set_cache_shards");
  }
  void head(const int64_t* y, int b0, int b, int gb) {
    eps_check(bert() ? eps_bert_stage_head(bx, y, b0, b, gb, loss.p, st)
                     : eps_vit_stage_head(ex, y, b0, b, gb, loss.p, st),
              "stage head");
  }
  void backward(int b0, int b, int g0, int g1, int lf) {
    eps_check(bert() ? eps_bert_stage_backward(bx, b0, b, g0, g1, lf, 0, st)
                     : eps_vit_stage_backward(ex, b0, b, g0, g1, lf, 0, st),
              "stage backward");
  }
  void sqnorms(int lf) {  // per-layer sum of squares of layers [lf, L) into sq; frozen zero
    cuda_check(cudaMemsetAsync(sq.p, 0, sq.n * 8, st), "sq");
    eps_check(bert() ? eps_bert_sqnorm_ranges(bx, segments.data() + lf, layers - lf, sq.p + lf, st)
                     : eps_vit_sqnorm_ranges(ex, segments.data() + lf, layers - lf, sq.p + lf, st),
              "sqnorm ranges");
  }
  void sgd(int lf) {  // SGD-momentum over the trainable tail [sublayer 2 lf, end)
    int64_t a = 0, e = 0;
    eps_check(bert() ? eps_bert_param_range(bx, 2 * lf, 2 * layers, &a, &e)
                     : eps_vit_param_range(ex, 2 * lf, 2 * layers, &a, &e),
              "param range");
    e = param_total;  // the tail (head / pooler / classifier) trains too
    eps_check(bert() ? eps_bert_sgd_range(bx, a, e, lr, momentum, 0.f, st)
                     : eps_vit_sgd_range(ex, a, e, lr, momentum, 0.f, st),
              "sgd");
  }
};

namespace {

template <typename F>
int guarded_rt(F&& body) {
  try {
    body();
    return EPS_OK;
  } catch (const eps::ConfigError& e) {
    eps::set_last_error(e.what());
    return EPS_ECONFIG;
  } catch (const eps::IoError& e) {
    eps::set_last_error(e.what());
    return EPS_EIO;
  } catch (const std::invalid_argument& e) {
    eps::set_last_error(e.what());
    return EPS_EINVAL;
  } catch (const std::domain_error& e) {  // planner / shard arithmetic (reference types)
    eps::set_last_error(e.what());
    return EPS_EDOMAIN;
  } catch (const std::logic_error& e) {
    eps::set_last_error(e.what());
    return EPS_ELOGIC;
  } catch (const std::exception& e) {  // cuda_check / eps_check failures
    eps::set_last_error(e.what());
    return EPS_ECUDA;
  }
}

// Seeded initialisation in the executor's flat layout: trunc-normal(0.02,
// +-0.04) matrices / embeddings, zero biases, unit LayerNorm gains
// (vit.py / bert.py init_params); the head's padded class rows stay zero.
// tensor kinds in eps_*_layout order: 0 weight, 1 bias, 2 LayerNorm gain.
void init_params(eps_trainer* t, const int64_t* tens, int n_tensors, std::vector<float>& host) {
  host.assign(size_t(t->param_total), 0.f);
  SplitMix rng{t->seed * 0x2545F4914F6CDD1Dull + 1};
  const int L = t->layers;
  const int classes = t->geom[5], d = t->hidden;
  for (int i = 0; i < n_tensors; ++i) {
    const int64_t off = tens[2 * i], n = tens[2 * i + 1];
    int kind = 0;
    int64_t valid = n;
    if (!t->bert()) {  // patch W, patch b, cls, pos | 12 per block | norm w, b, head W, b
      if (i < 4) {
        kind = i == 1 ? 1 : 0;
      } else if (i < 4 + 12 * L) {
        const int j = (i - 4) % 12;
        kind = (j == 0 || j == 6) ? 2 : (j % 2 == 1) ? 1 : 0;
      } else {
        const int j = i - 4 - 12 * L;
        kind = j == 0 ? 2 : (j == 1 || j == 3) ? 1 : 0;
        if (j == 2) valid = int64_t(classes) * d;
      }
    } else {  // word, pos, type, LN w, LN b | 12 per layer | [pooler W, b] classifier W, b
      if (i < 5) {
        kind = i == 3 ? 2 : i == 4 ? 1 : 0;
      } else if (i < 5 + 12 * L) {
        const int j = (i - 5) % 12;
        kind = (j == 4 || j == 10) ? 2 : (j % 2 == 1) ? 1 : 0;
      } else {
        const int j = i - 5 - 12 * L;  // 0, 1: pooler (if any); last two: classifier
        kind = (j % 2 == 1) ? 1 : 0;
        if (i == n_tensors - 2) valid = int64_t(classes) * d;
      }
    }
    for (int64_t e = 0; e < valid; ++e) {
      float v = 0.f;
      if (kind == 2) {
        v = 1.f;
      } else if (kind == 0) {
        double z;
        do z = rng.normal();
        while (z < -2.0 || z > 2.0);
        v = float(0.02 * z);
      }
      host[size_t(off + e)] = v;
    }
  }
}

}  // namespace

extern "C" {

int eps_trainer_create(const eps_scenario_t* scenario, int kind, const int* geom,
                       int iterations_per_epoch, uint64_t seed, float lr, float momentum,
                       int device_norms, const float* init_params_host, const void* inputs_dev,
                       const int64_t* labels_dev, eps_trainer_t** out) {
  return guarded_rt([&] {
    if (scenario == nullptr || geom == nullptr || out == nullptr || iterations_per_epoch < 1 ||
        (kind != EPS_MODEL_VIT && kind != EPS_MODEL_BERT))
      throw std::invalid_argument("eps_trainer_create: null argument, iterations < 1 or bad kind");
    auto t = std::make_unique<eps_trainer>();
    t->cfg = scenario->cfg;
    t->kind = kind;
    const int world = t->cfg.cluster.node_count * t->cfg.cluster.gpus_per_node;
    if (world != 1 || t->cfg.pipeline_length_at_start() != 1)
      throw std::invalid_argument(
          "the native trainer runs one GPU (cluster 1 x 1); multi-rank runs use trainer.py");
    std::memcpy(t->geom, geom, sizeof(t->geom));
    t->layers = geom[0];
    t->hidden = geom[1];
    t->tokens = geom[4];
    t->qa = t->bert() && geom[8] == 1;
    t->batch = int(t->cfg.training.per_pipeline_batch);
    if (t->batch < 1 || t->batch > geom[10])
      throw std::invalid_argument("per_pipeline_batch must be in [1, geometry max_batch]");
    if (t->cfg.model.layer_count() != t->layers)
      throw std::invalid_argument("scenario model and geometry disagree on the layer count");
    t->iters = iterations_per_epoch;
    t->seed = seed;
    t->lr = lr;
    t->momentum = momentum;
    t->device_norms = device_norms != 0;
    if (!t->bert()) t->image_elems = int64_t(geom[9]) * geom[7] * geom[7];
    // dataset = iterations x batch x initial replica count (runner.cpp:103-104)
    t->dataset = int64_t(t->iters) * t->batch;
    t->planner = std::make_unique<eps::EpochPlanner>(t->cfg);
    if (t->cfg.features.freeze) t->scenario_norms = eps::make_grad_norm_source(t->cfg);
    t->recorded = std::make_unique<eps::RecordedNormSource>(t->layers);

    int64_t ws_bytes = 0;
    t->segments.resize(size_t(t->layers) + 1);
    const int n_tensors = t->bert() ? 5 + 12 * t->layers + (geom[9] ? 2 : 0) + 2
                                    : 4 + 12 * t->layers + 4;
    std::vector<int64_t> tens(2 * size_t(n_tensors));
    eps_check(t->bert() ? eps_bert_layout(geom, &t->param_total, &ws_bytes, t->segments.data(),
                                          tens.data())
                        : eps_vit_layout(geom, &t->param_total, &ws_bytes, t->segments.data(),
                                         tens.data()),
              "layout");
    cuda_check(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking), "stream");
    t->p32.alloc(size_t(t->param_total));
    t->p16.alloc(size_t(t->param_total));
    t->g32.alloc(size_t(t->param_total));
    t->mom.alloc(size_t(t->param_total) * (t->bert() ? 2 : 1));  // BERT: room for AdamW m | v
    t->ws.alloc(size_t(ws_bytes));
    t->loss.alloc(1);
    t->sq.alloc(size_t(t->layers));
    cuda_check(cudaMemset(t->g32.p, 0, t->g32.n * 4), "memset");
    cuda_check(cudaMemset(t->mom.p, 0, t->mom.n * 4), "memset");
    std::vector<float> host;
    if (init_params_host == nullptr) {
      init_params(t.get(), tens.data(), n_tensors, host);
      init_params_host = host.data();
    }
    cuda_check(cudaMemcpy(t->p32.p, init_params_host, size_t(t->param_total) * 4,
                          cudaMemcpyHostToDevice),
               "params H2D");
    // bf16 working copy: an SGD step with lr = momentum = 0 on zero gradients
    eps_check(eps_sgd_momentum(t->p32.p, t->p16.p, t->g32.p, t->mom.p, t->param_total, 0.f, 0.f,
                               0.f, t->st),
              "bf16 params");
    eps_check(t->bert() ? eps_bert_create(geom, t->p32.p, t->p16.p, t->g32.p, t->mom.p, t->ws.p,
                                          &t->bx)
                        : eps_vit_create(geom, t->p32.p, t->p16.p, t->g32.p, t->mom.p, t->ws.p,
                                         &t->ex),
              "executor create");
    // dataset: the caller's device tensors, or seeded synthetic data (device)
    const int64_t N = t->dataset, T = t->tokens;
    const int64_t n_lab = t->qa ? 2 * N : N;
    t->labels_host.resize(size_t(n_lab));
    if (!t->bert()) {
      t->images.alloc(size_t(N * t->image_elems));
      t->xb.alloc(size_t(t->batch * t->image_elems));
    } else {
      t->tok.alloc(size_t(N * T));
      t->segs.alloc(size_t(N * T));
      t->tb.alloc(size_t(2 * t->batch * T));
    }
    if (inputs_dev != nullptr && labels_dev != nullptr) {
      if (!t->bert()) {
        cuda_check(cudaMemcpy(t->images.p, inputs_dev, t->images.n * 4, cudaMemcpyDeviceToDevice),
                   "images D2D");
      } else {  // int64 [2][N][T]: token ids, then segment ids
        const int64_t* in = static_cast<const int64_t*>(inputs_dev);
        cuda_check(cudaMemcpy(t->tok.p, in, size_t(N * T) * 8, cudaMemcpyDeviceToDevice), "D2D");
        cuda_check(cudaMemcpy(t->segs.p, in + N * T, size_t(N * T) * 8, cudaMemcpyDeviceToDevice),
                   "D2D");
      }
      cuda_check(cudaMemcpy(t->labels_host.data(), labels_dev, size_t(n_lab) * 8,
                            cudaMemcpyDeviceToHost),
                 "labels D2H");
    } else {
      DevBuf<int64_t> lab;
      lab.alloc(size_t(n_lab));
      if (!t->bert()) {
        eps_check(eps_fill_normal(t->images.p, int64_t(t->images.n), seed ^ 0xD1B54A32D192ED03ull,
                                  t->st),
                  "eps_fill_normal");
        eps_check(eps_fill_labels(lab.p, N, geom[5], seed ^ 0x8CB92BA72F3D8DD7ull, t->st),
                  "eps_fill_labels");
      } else {  // token ids U[0, vocab), segment ids 0 | 1 by half (bench.py synthetic_inputs)
        eps_check(eps_fill_labels(t->tok.p, N * T, geom[6], seed ^ 0xD1B54A32D192ED03ull,
                                  t->st),
                  "eps_fill_labels");
        std::vector<int64_t> sg(size_t(N * T));
        for (int64_t i = 0; i < N * T; ++i) sg[size_t(i)] = (i % T) >= T / 2 ? 1 : 0;
        cuda_check(cudaMemcpyAsync(t->segs.p, sg.data(), sg.size() * 8, cudaMemcpyHostToDevice,
                                   t->st),
                   "segments H2D");
        eps_check(eps_fill_labels(lab.p, n_lab, t->qa ? T : geom[5], seed ^ 0x8CB92BA72F3D8DD7ull,
                                  t->st),
                  "eps_fill_labels");
        cuda_check(cudaStreamSynchronize(t->st), "segments");
      }
      cuda_check(cudaMemcpyAsync(t->labels_host.data(), lab.p, lab.n * 8, cudaMemcpyDeviceToHost,
                                 t->st),
                 "labels D2H");
      cuda_check(cudaStreamSynchronize(t->st), "synthetic data");
    }
    t->yb.alloc(size_t(n_lab));
    t->shard.alloc(size_t(t->dataset));
    cuda_check(cudaStreamSynchronize(t->st), "init");
    *out = t.release();
  });
}

void eps_trainer_destroy(eps_trainer_t* t) {
  if (t != nullptr) {
    cudaDeviceSynchronize();
    delete t;
  }
}

int eps_trainer_run_epoch(eps_trainer_t* t, int epoch, eps_train_epoch_t* out, double* norms_out) {
  return guarded_rt([&] {
    if (t == nullptr || out == nullptr) throw std::invalid_argument("null trainer / result");
    // decision (runner.cpp:139-186 order inside EpochPlanner)
    const eps::GradNormSource* src = t->scenario_norms.get();
    if (t->device_norms && epoch > 0) {
      if (t->norms_prev.empty())
        throw std::invalid_argument("device-norm run has no gradient norms from the last epoch");
      t->recorded->record(epoch - 1, t->norms_prev);
      src = t->recorded.get();
    }
    const eps::EpochDecision d = t->planner->begin_epoch(epoch, src);
    if (d.pipeline_length != 1 || d.replica_width != 1)
      throw std::invalid_argument("planner chose K or R > 1 on a one-GPU cluster");
    const int lf = d.l_frozen, L = t->layers;
    int cache_mode = 0, cache_old = 0;
    if (!d.cache_enabled) {
      cache_mode = 0;
    } else if (d.cache_moved) {
      cache_mode = 2;
      cache_old = d.cache_old_boundary;
    } else if (d.cache_boundary < lf) {
      cache_mode = 3;  // trailing boundary (runner.cpp:189-213)
      cache_old = d.cache_boundary;
    } else {
      cache_mode = 1;
    }
    const int64_t row_elems = int64_t(t->tokens) * t->hidden;
    if (cache_mode != 0 && t->store.p == nullptr) {
      t->store.alloc(size_t(t->dataset * row_elems));
      cuda_check(cudaMemsetAsync(t->store.p, 0, t->store.n * 2, t->st), "store");
      t->set_cache_shards();
    }
    // this epoch's sample order (one replica: the whole dataset)
    const eps::Topology topo(t->cfg.cluster, 1);
    const eps::ShardAssignment sa = eps::redistribute(t->dataset, topo, epoch, t->seed);
    const std::vector<int64_t>& ids = sa.shards.at(0);
    cuda_check(cudaMemcpyAsync(t->shard.p, ids.data(), ids.size() * 8, cudaMemcpyHostToDevice,
                               t->st),
               "shard H2D");
    std::vector<std::pair<int64_t, int>> its;
    const int64_t n = int64_t(ids.size());
    for (int64_t o = 0; o + t->batch <= n; o += t->batch) its.emplace_back(o, t->batch);
    if (n % t->batch) its.emplace_back(n - n % t->batch, int(n % t->batch));
    // the epoch's labels in sample order (one upload; iteration it reads [o, o + b))
    // (SQuAD head: per iteration the b start positions, then the b end positions)
    const int64_t per = t->qa ? 2 : 1;
    std::vector<int64_t> ylab(static_cast<size_t>(per * n));
    for (const auto& itv : its)
      for (int i = 0; i < itv.second; ++i) {
        const int64_t sid = ids[size_t(itv.first + i)];
        if (t->qa) {
          ylab[size_t(2 * itv.first + i)] = t->labels_host[size_t(sid)];
          ylab[size_t(2 * itv.first + itv.second + i)] = t->labels_host[size_t(t->dataset + sid)];
        } else {
          ylab[size_t(itv.first + i)] = t->labels_host[size_t(sid)];
        }
      }
    cuda_check(cudaMemcpyAsync(t->yb.p, ylab.data(), ylab.size() * 8, cudaMemcpyHostToDevice,
                               t->st),
               "labels H2D");
    const int g0 = 2 * lf, g1 = 2 * L;
    const bool split_front = cache_mode != 0;  // front work timed on its own (cache transition)
    struct Events {  // destroyed on every exit path
      std::vector<cudaEvent_t> v;
      ~Events() {
        for (auto e : v) cudaEventDestroy(e);
      }
    } events;
    std::vector<cudaEvent_t>& ev = events.v;
    auto mark = [&]() {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "event");
      cuda_check(cudaEventRecord(e, t->st), "event record");
      ev.push_back(e);
      return e;
    };
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> front;
    cuda_check(cudaMemsetAsync(t->loss.p, 0, 4, t->st), "loss");
    const cudaEvent_t start = mark();
    for (size_t it = 0; it < its.size(); ++it) {
      const int64_t o = its[it].first;
      const int b = its[it].second;
      const int64_t* bid = t->shard.p + o;
      if (cache_mode != 1) {
        if (!t->bert()) {
          eps_check(eps_cache_gather(t->images.p, bid, b, t->image_elems * 4, t->xb.p, t->st),
                    "image gather");
        } else {  // [2][b][T]: token ids, then segment ids
          eps_check(eps_cache_gather(t->tok.p, bid, b, int64_t(t->tokens) * 8, t->tb.p, t->st),
                    "token gather");
          eps_check(eps_cache_gather(t->segs.p, bid, b, int64_t(t->tokens) * 8,
                                     t->tb.p + int64_t(b) * t->tokens, t->st),
                    "segment gather");
        }
      }
      const int64_t* yl = t->yb.p + per * o;
      const int M = std::max(1, std::min(d.micro_batches, b));
      std::vector<int> b0s, bs;
      for (int m = 0, at = 0; m < M; ++m) {
        const int nb = b / M + (m < b % M ? 1 : 0);
        b0s.push_back(at);
        bs.push_back(nb);
        at += nb;
      }
      const float* xi = cache_mode != 1 ? t->xb.p : nullptr;
      const int64_t* ti = cache_mode != 1 ? t->tb.p : nullptr;
      auto fwd = [&](bool with_input, int b0, int nb, int ga, int gb, int front, int cm, int co,
                     void* store, const int64_t* sids) {
        eps_check(t->bert() ? eps_bert_stage_forward(t->bx, with_input ? ti : nullptr, b, b0, nb,
                                                     ga, gb, lf, front, cm, co, store, sids, t->st)
                            : eps_vit_stage_forward(t->ex, with_input ? xi : nullptr, b0, nb, ga,
                                                    gb, lf, front, cm, co, store, sids, t->st),
                  "stage forward");
      };
      for (int m = 0; m < M; ++m) {
        if (split_front) {
          const cudaEvent_t fa = mark();
          fwd(true, b0s[m], bs[m], g0, g0, 1, cache_mode, cache_old, t->store.p, bid);
          front.emplace_back(fa, mark());
          fwd(false, b0s[m], bs[m], g0, g1, 0, 0, 0, nullptr, nullptr);
        } else {
          fwd(true, b0s[m], bs[m], g0, g1, 1, 0, 0, nullptr, nullptr);
        }
        t->head(yl, b0s[m], bs[m], b);
      }
      for (int m = M - 1; m >= 0; --m)
        t->backward(b0s[m], bs[m], g0, g1, lf);
      if (it + 1 == its.size())
        t->sqnorms(lf);
      t->sgd(lf);
    }
    const cudaEvent_t stop = mark();
    cuda_check(cudaEventSynchronize(stop), "epoch");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, start, stop), "elapsed");
    std::vector<double> sq(static_cast<size_t>(L));
    float loss = 0.f;
    cuda_check(cudaMemcpy(sq.data(), t->sq.p, sq.size() * 8, cudaMemcpyDeviceToHost), "norms");
    cuda_check(cudaMemcpy(&loss, t->loss.p, 4, cudaMemcpyDeviceToHost), "loss");
    t->norms_prev.resize(size_t(L));
    for (int l = 0; l < L; ++l) t->norms_prev[size_t(l)] = std::sqrt(sq[size_t(l)]);
    if (norms_out) std::copy(t->norms_prev.begin(), t->norms_prev.end(), norms_out);
    // cache transition: a boundary-move epoch's front work over a steady gather
    double cache_tr = 0.0;
    if (cache_mode == 2 && !front.empty()) {
      double prefix = 0.0;
      for (auto& f : front) {
        float fm = 0.f;
        cuda_check(cudaEventElapsedTime(&fm, f.first, f.second), "front");
        prefix += fm / 1e3;
      }
      double steady = 0.0;
      DevBuf<uint16_t> tmp;
      tmp.alloc(size_t(t->batch * row_elems));
      for (auto& itv : its) {
        const cudaEvent_t a = mark();
        eps_check(eps_cache_gather(t->store.p, t->shard.p + itv.first, itv.second, row_elems * 2,
                                   tmp.p, t->st),
                  "steady gather");
        const cudaEvent_t e = mark();
        cuda_check(cudaEventSynchronize(e), "gather");
        float gm = 0.f;
        cuda_check(cudaEventElapsedTime(&gm, a, e), "gather time");
        steady += gm / 1e3;
      }
      cache_tr = std::max(0.0, prefix - steady);
    }
    const double epoch_s = ms / 1e3;
    out->epoch = epoch;
    out->l_frozen = lf;
    out->pipeline_length = d.pipeline_length;
    out->replica_width = d.replica_width;
    out->micro_batches = d.micro_batches;
    out->cache_enabled = d.cache_enabled ? 1 : 0;
    out->cache_moved = d.cache_moved ? 1 : 0;
    out->cache_mode = cache_mode;
    out->iterations = int(its.size());
    out->epoch_time_s = epoch_s;
    out->iteration_time_s = epoch_s / double(std::max<size_t>(1, its.size()));
    out->samples = double(n);
    out->throughput_sps = double(n) / epoch_s;
    out->mean_loss = double(loss) / double(n);
    out->cache_transition_time_s = cache_tr;
  });
}

}  // extern "C"
