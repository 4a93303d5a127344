// eps_train: the reference CLI's `run --scenario FILE` (cli.cpp:55-74), but
// executed on one B200 instead of simulated: the scenario's decisions
// (freeze / AutoPipe / AutoDP / AutoCache, EpochPlanner) drive real ViT
// training steps through libeps_b200.so, and the per-epoch rows are printed in
// the trainer's CSV schema (trainer.py CSV_HEADER; measured columns).
//
//   make train
//   build/eps_train --scenario s.json --geometry tiny-vit --iterations 3 [--epochs 10]
//                   [--seed 17] [--lr 1e-3] [--momentum 0.9] [--csv out.csv]
//
// Synthetic data (seeded N(0,1) images or uniform token ids with half-and-half
// segment ids, uniform labels) and a seeded trunc-normal initialisation; a
// 1 x 1 cluster (other clusters: trainer.py).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "eps_capi.h"

namespace {

struct Geo {
  const char* name;
  int kind;   // EPS_MODEL_VIT / EPS_MODEL_BERT
  int v[10];  // ViT: layers, d, mlp, heads, tokens, classes, image, stored image, patch, channels
              // BERT: layers, d, mlp, heads, tokens, classes, vocab, positions, head (1 SQuAD), pooler
};
// configs.py GEOMETRIES
const Geo kGeos[] = {
    {"tiny-vit", EPS_MODEL_VIT, {4, 128, 512, 4, 65, 100, 32, 32, 4, 3}},
    {"vit-b16", EPS_MODEL_VIT, {12, 768, 3072, 12, 197, 1000, 224, 224, 16, 3}},
    {"vit-b16-cifar100", EPS_MODEL_VIT, {12, 768, 3072, 12, 197, 100, 224, 32, 16, 3}},
    {"bert-base-384", EPS_MODEL_BERT, {12, 768, 3072, 12, 384, 2, 30522, 512, 1, 1}},
    {"bert-large-128", EPS_MODEL_BERT, {24, 1024, 4096, 16, 128, 2, 30522, 512, 0, 1}},
    {"tiny-bert-qa", EPS_MODEL_BERT, {2, 128, 512, 2, 64, 2, 1000, 128, 1, 1}},
    {"tiny-bert-cls", EPS_MODEL_BERT, {2, 256, 1024, 4, 48, 3, 500, 64, 0, 1}},
};

int usage(const char* argv0) {
  std::fprintf(stderr,
               "usage: %s --scenario FILE --geometry {tiny-vit|vit-b16|vit-b16-cifar100|bert-base-384|"
               "bert-large-128|tiny-bert-qa|tiny-bert-cls} "
               "--iterations N [--epochs E] [--seed S] [--lr X] [--momentum X] [--csv OUT]\n",
               argv0);
  return 2;
}

int fail(const char* what, int rc) {
  std::fprintf(stderr, "eps_train: %s failed (%d): %s\n", what, rc, eps_last_error());
  return 1;
}

}  // namespace

int main(int argc, char** argv) {
  std::string scenario, geometry, csv;
  int iterations = 0, epochs = 10;
  unsigned long long seed = 17;
  float lr = 1e-3f, momentum = 0.9f;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> const char* { return i + 1 < argc ? argv[++i] : nullptr; };
    const char* v = nullptr;
    if (a == "--scenario" && (v = val())) scenario = v;
    else if (a == "--geometry" && (v = val())) geometry = v;
    else if (a == "--iterations" && (v = val())) iterations = std::atoi(v);
    else if (a == "--epochs" && (v = val())) epochs = std::atoi(v);
    else if (a == "--seed" && (v = val())) seed = std::strtoull(v, nullptr, 10);
    else if (a == "--lr" && (v = val())) lr = float(std::atof(v));
    else if (a == "--momentum" && (v = val())) momentum = float(std::atof(v));
    else if (a == "--csv" && (v = val())) csv = v;
    else return usage(argv[0]);
  }
  const Geo* geo = nullptr;
  for (const Geo& g : kGeos)
    if (geometry == g.name) geo = &g;
  if (scenario.empty() || geo == nullptr || iterations < 1 || epochs < 1) return usage(argv[0]);

  eps_scenario_t* sc = nullptr;
  int rc = eps_scenario_load(scenario.c_str(), &sc);
  if (rc != EPS_OK) return fail("eps_scenario_load", rc);
  // max_batch = the scenario's per-pipeline batch (read back through the JSON form)
  std::vector<char> js(1 << 16);
  size_t len = 0;
  rc = eps_scenario_to_json(sc, js.data(), js.size(), &len);
  if (rc != EPS_OK) return fail("eps_scenario_to_json", rc);
  const char* key = std::strstr(js.data(), "\"per_pipeline_batch\"");
  const int batch = key ? int(std::atof(std::strchr(key, ':') + 1)) : 0;
  int geom[11];
  std::memcpy(geom, geo->v, sizeof(geo->v));
  geom[10] = batch;

  eps_trainer_t* t = nullptr;
  rc = eps_trainer_create(sc, geo->kind, geom, iterations, seed, lr, momentum, 1, nullptr, nullptr,
                          nullptr, &t);
  if (rc != EPS_OK) return fail("eps_trainer_create", rc);
  FILE* out = csv.empty() ? stdout : std::fopen(csv.c_str(), "w");
  if (out == nullptr) {
    std::perror(csv.c_str());
    return 1;
  }
  std::fprintf(out,
               "epoch,l_frozen,k,r,m,iteration_time_s,epoch_time_s,throughput_sps,bubble_time_s,"
               "comm_time_s,exposed_comm_time_s,cache_enabled,transition_overhead_s,"
               "cache_transition_time_s,stall_time_s\n");
  double total = 0.0;
  for (int e = 0; e < epochs; ++e) {
    eps_train_epoch_t r;
    rc = eps_trainer_run_epoch(t, e, &r, nullptr);
    if (rc != EPS_OK) return fail("eps_trainer_run_epoch", rc);
    total += r.epoch_time_s;
    std::fprintf(out, "%d,%d,%d,%d,%d,%.9g,%.9g,%.9g,0,0,0,%d,0,%.9g,0\n", r.epoch, r.l_frozen,
                 r.pipeline_length, r.replica_width, r.micro_batches, r.iteration_time_s,
                 r.epoch_time_s, r.throughput_sps, r.cache_enabled, r.cache_transition_time_s);
    std::fprintf(stderr, "epoch %d: L_frozen %d cache %d loss %.5f %.1f samples/s\n", r.epoch,
                 r.l_frozen, r.cache_mode, r.mean_loss, r.throughput_sps);
  }
  std::fprintf(stderr, "total %.4f s over %d epochs\n", total, epochs);
  if (out != stdout) std::fclose(out);
  eps_trainer_destroy(t);
  eps_scenario_destroy(sc);
  return 0;
}
