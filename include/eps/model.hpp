// Transformer size profiles, cluster shape and training knobs.
//
// Source-compatible with the reference header proj/include/eps/model.hpp:15-88
// (same names, fields and signatures) so callers of the reference compile
// unchanged against this library.  Unlike the reference, the B200 build also
// runs the real network described by a profile: `TransformerDims` carries the
// architecture a profile is derived from, and `profile_from_dims` applies the
// reference's block arithmetic (model.cpp:107-121) so the decision inputs stay
// bit-identical to what the reference computes for the same architecture.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace eps {

// Per-layer parameter counts of one ATT block and one MLP block each, plus
// the per-sample bytes of the tensor entering global sublayer g (2L+1
// entries; entry 2L is the model output).  Mirrors model.hpp:15-30.
struct ModelSpec {
  std::string name;                            // preset or scenario label
  std::vector<std::int64_t> attention_params;  // ATT block of layer l (QKV + out-proj + LN)
  std::vector<std::int64_t> mlp_params;        // MLP block of layer l (fc1 + fc2 + LN)
  std::vector<std::int64_t> activation_bytes;  // per sample, tensor entering sublayer g
  int bytes_per_param = 4;                     // gradient element size for bucket sizing

  int layer_count() const { return static_cast<int>(attention_params.size()); }
  std::int64_t total_params() const;
  std::int64_t prefix_params(int layer) const;   // layers [0, layer)
  std::int64_t boundary_bytes(int sublayer_global_index) const;
  void validate() const;                          // std::invalid_argument
};

struct ClusterSpec {
  int node_count = 1;                      // N
  int gpus_per_node = 1;                   // I (power of two)
  double gpu_memory_bytes = 16e9;          // per device
  double intra_node_bandwidth = 15.754e9;  // bytes/s between GPUs of one node
  double inter_node_bandwidth = 5e9;       // bytes/s across nodes

  int total_gpus() const { return node_count * gpus_per_node; }
  void validate() const;
};

struct TrainingConfig {
  double per_pipeline_batch = 400.0;  // samples per pipeline per iteration
  int epochs = 10;                    // epochs of the run
  int iterations_per_epoch = 100;     // at the initial replica count
  double alpha = 1.0 / 3.0;           // freeze aggressiveness
  double lambda_frozen = 1.0 / 6.0;   // memory weight of frozen parameters
  int freeze_check_interval = 1;      // epochs between freeze decisions

  void validate() const;
};

enum class SublayerKind { kAttention, kMlp };

struct Sublayer {
  SublayerKind kind = SublayerKind::kAttention;  // ATT or MLP half of a layer
  int layer_index = 0;                           // transformer layer
  std::int64_t params = 0;                       // trainable parameters

  // ATT of layer i is 2i, MLP is 2i+1 (model.hpp:61-63).
  int global_index() const {
    return 2 * layer_index + (kind == SublayerKind::kMlp ? 1 : 0);
  }
};

struct SublayerSeq {
  std::vector<Sublayer> active;    // trainable sublayers in order
  std::int64_t frozen_params = 0;  // S_frozen = params of layers [0, L_frozen)
  int frozen_layers = 0;           // L_frozen

  std::int64_t active_params() const;
};

// Frozen block [0, l_frozen) + the active ATT, MLP sequence (model.cpp:79-92).
SublayerSeq m_partition(const ModelSpec& model, int l_frozen);

// L identical layers (model.cpp:94-105).
ModelSpec uniform_model(int layers, std::int64_t attention_params, std::int64_t mlp_params,
                        std::int64_t activation_bytes);

ModelSpec vit_b16();     // 86,566,120 parameters (model.cpp:125-150)
ModelSpec bert_large();  // 335,143,938 parameters (model.cpp:152-179)

// ---- B200 additions (no reference counterpart) ---------------------------

// The architecture a profile is computed from.  `embed_params` and
// `head_params` are folded into layer 0's ATT and layer L-1's MLP exactly as
// the presets do (model.cpp:137-142, 164-171).
struct TransformerDims {
  std::string name;
  int layers = 12;
  std::int64_t hidden = 768;
  std::int64_t mlp_dim = 3072;
  std::int64_t tokens = 197;
  std::int64_t embed_params = 0;
  std::int64_t head_params = 0;
  std::int64_t input_bytes = 0;  // activation_bytes[0]
};

// ViT patch-embedding frontend: conv(p x p, c_in -> d) + CLS + positions.
TransformerDims vit_dims(const std::string& name, int layers, std::int64_t hidden,
                         std::int64_t mlp_dim, int image, int patch, int channels,
                         std::int64_t classes);
// BERT frontend: word + position + type embeddings and the embedding LN;
// `head_params` is the task head (pooler + classifier or QA span head).
TransformerDims bert_dims(const std::string& name, int layers, std::int64_t hidden,
                          std::int64_t mlp_dim, std::int64_t seq_len,
                          std::int64_t position_table, std::int64_t vocab,
                          std::int64_t head_params);
ModelSpec profile_from_dims(const TransformerDims& dims);

}  // namespace eps
