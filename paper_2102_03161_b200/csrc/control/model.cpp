// Size profiles (reference: proj/src/model.cpp).  Integer arithmetic only;
// the decision modules consume these counts, so they must equal the
// reference's numbers exactly (pinned by tests/test_control_parity.py).
#include "eps/model.hpp"

#include <stdexcept>
#include <string>

namespace eps {

namespace {

void need(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

// model.cpp:109-114 -- QKV (3 affine maps) + output projection + one LN pair.
std::int64_t att_block(std::int64_t d) {
  return 3 * (d * d + d) + (d * d + d) + 2 * d;
}

// model.cpp:116-121 -- fc1 + fc2 + one LN pair.
std::int64_t mlp_block(std::int64_t d, std::int64_t f) {
  return (d * f + f) + (f * d + d) + 2 * d;
}

}  // namespace

std::int64_t ModelSpec::total_params() const {
  return prefix_params(layer_count());
}

std::int64_t ModelSpec::prefix_params(int layer) const {
  need(layer >= 0 && layer <= layer_count(), "prefix_params: layer out of range");
  std::int64_t acc = 0;
  for (int i = 0; i < layer; ++i) acc += attention_params[i] + mlp_params[i];
  return acc;
}

std::int64_t ModelSpec::boundary_bytes(int g) const {
  need(g >= 0 && g < static_cast<int>(activation_bytes.size()),
       "boundary_bytes: sublayer index out of range");
  return activation_bytes[g];
}

void ModelSpec::validate() const {
  const int l = layer_count();
  need(l >= 1, "model: needs at least one layer");
  need(static_cast<int>(mlp_params.size()) == l,
       "model: attention/mlp layer counts differ");
  need(static_cast<int>(activation_bytes.size()) == 2 * l + 1,
       "model: activation_bytes must have 2L+1 entries");
  for (int i = 0; i < l; ++i)
    need(attention_params[i] > 0 && mlp_params[i] > 0,
         "model: parameter counts must be positive");
  for (std::int64_t b : activation_bytes)
    need(b > 0, "model: activation sizes must be positive");
  need(bytes_per_param > 0, "model: bytes_per_param must be positive");
}

void ClusterSpec::validate() const {
  need(node_count >= 1, "cluster: node_count must be >= 1");
  need(gpus_per_node >= 1, "cluster: gpus_per_node must be >= 1");
  need((gpus_per_node & (gpus_per_node - 1)) == 0,
       "cluster: gpus_per_node must be a power of two");
  need(intra_node_bandwidth > 0 && inter_node_bandwidth > 0,
       "cluster: bandwidths must be positive");
  need(gpu_memory_bytes > 0, "cluster: gpu_memory_bytes must be positive");
}

void TrainingConfig::validate() const {
  need(per_pipeline_batch >= 1, "training: per_pipeline_batch must be >= 1");
  need(epochs >= 1, "training: epochs must be >= 1");
  need(iterations_per_epoch >= 1, "training: iterations_per_epoch must be >= 1");
  need(alpha > 0.0 && alpha < 1.0, "training: alpha must be in (0,1)");
  need(lambda_frozen >= 0.0 && lambda_frozen <= 1.0,
       "training: lambda_frozen must be in [0,1]");
  need(freeze_check_interval >= 1, "training: freeze_check_interval must be >= 1");
}

std::int64_t SublayerSeq::active_params() const {
  std::int64_t acc = 0;
  for (const Sublayer& s : active) acc += s.params;
  return acc;
}

// model.cpp:79-92: the stack below l_frozen becomes one frozen block, the
// rest is the ATT,MLP,ATT,MLP... sequence the partitioner cuts.
SublayerSeq m_partition(const ModelSpec& model, int l_frozen) {
  const int l = model.layer_count();
  if (l_frozen < 0 || l_frozen > l)
    throw std::domain_error("m_partition: frozen layer count out of [0, L]");
  SublayerSeq seq;
  seq.frozen_layers = l_frozen;
  seq.frozen_params = model.prefix_params(l_frozen);
  seq.active.reserve(static_cast<std::size_t>(2 * (l - l_frozen)));
  for (int i = l_frozen; i < l; ++i) {
    seq.active.push_back(Sublayer{SublayerKind::kAttention, i, model.attention_params[i]});
    seq.active.push_back(Sublayer{SublayerKind::kMlp, i, model.mlp_params[i]});
  }
  return seq;
}

ModelSpec uniform_model(int layers, std::int64_t attention_params,
                        std::int64_t mlp_params, std::int64_t activation_bytes) {
  ModelSpec m;
  m.name = "uniform-" + std::to_string(layers);
  m.attention_params = std::vector<std::int64_t>(layers, attention_params);
  m.mlp_params = std::vector<std::int64_t>(layers, mlp_params);
  m.activation_bytes = std::vector<std::int64_t>(2 * layers + 1, activation_bytes);
  m.validate();
  return m;
}

TransformerDims vit_dims(const std::string& name, int layers, std::int64_t hidden,
                         std::int64_t mlp_dim, int image, int patch, int channels,
                         std::int64_t classes) {
  TransformerDims d;
  d.name = name;
  d.layers = layers;
  d.hidden = hidden;
  d.mlp_dim = mlp_dim;
  const std::int64_t side = image / patch;
  d.tokens = side * side + 1;  // patches + [CLS]
  // conv weight + bias, CLS token, position table (model.cpp:137-140).
  d.embed_params = hidden * (static_cast<std::int64_t>(patch) * patch * channels) +
                   hidden + hidden + d.tokens * hidden;
  d.head_params = hidden * classes + classes;  // model.cpp:141
  d.input_bytes = static_cast<std::int64_t>(image) * image * channels * 4;
  return d;
}

TransformerDims bert_dims(const std::string& name, int layers, std::int64_t hidden,
                          std::int64_t mlp_dim, std::int64_t seq_len,
                          std::int64_t position_table, std::int64_t vocab,
                          std::int64_t head_params) {
  TransformerDims d;
  d.name = name;
  d.layers = layers;
  d.hidden = hidden;
  d.mlp_dim = mlp_dim;
  d.tokens = seq_len;
  // word + position + token-type tables + embedding LN (model.cpp:164-167).
  d.embed_params = vocab * hidden + position_table * hidden + 2 * hidden + 2 * hidden;
  d.head_params = head_params;
  d.input_bytes = seq_len * 8;  // token + segment ids (model.cpp:174)
  return d;
}

ModelSpec profile_from_dims(const TransformerDims& dims) {
  ModelSpec m;
  m.name = dims.name;
  m.attention_params.assign(dims.layers, att_block(dims.hidden));
  m.mlp_params.assign(dims.layers, mlp_block(dims.hidden, dims.mlp_dim));
  m.attention_params.front() += dims.embed_params;
  m.mlp_params.back() += dims.head_params;
  m.activation_bytes.assign(2 * dims.layers + 1, dims.tokens * dims.hidden * 4);
  m.activation_bytes.front() = dims.input_bytes;
  m.validate();
  return m;
}

// model.cpp:125-150.
ModelSpec vit_b16() {
  return profile_from_dims(vit_dims("vit-b16", 12, 768, 3072, 224, 16, 3, 1000));
}

// model.cpp:152-179: BERT-large with a 512-position table, pooler + QA head.
ModelSpec bert_large() {
  const std::int64_t h = 1024;
  return profile_from_dims(
      bert_dims("bert-large", 24, h, 4096, 512, 512, 30522, (h * h + h) + (h * 2 + 2)));
}

}  // namespace eps
