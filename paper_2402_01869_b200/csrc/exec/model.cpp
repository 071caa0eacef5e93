#include "model.hpp"

#include <json.hpp>

#include "../sched/base.hpp"

namespace ib2 {

std::int64_t ModelSpec::param_count() const { return layout_weights(*this).total; }

namespace {

ModelSpec preset(const std::string& name) {
  ModelSpec m;
  if (name == "tiny") return m;
  if (name == "gptj-6b") {
    m.family = Family::GptJ;
    m.layers = 28;
    m.d_model = 4096;
    m.heads = 16;
    m.ffn = 16384;
    m.vocab = 50400;
    m.rotary_dim = 64;
    return m;
  }
  if (name == "vicuna-13b") {
    m.family = Family::Llama;
    m.layers = 40;
    m.d_model = 5120;
    m.heads = 40;
    m.ffn = 13824;
    m.vocab = 32000;
    m.rotary_dim = 128;
    m.norm_eps = 1e-6f;
    return m;
  }
  throw ConfigError("unknown model preset: " + name);
}

}  // namespace

ModelSpec parse_model_json(const std::string& text) {
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("model JSON: ") + e.what());
  }
  ModelSpec m = preset(j.value("preset", std::string("tiny")));
  try {
    if (j.contains("family")) {
      const std::string f = j["family"].get<std::string>();
      if (f == "gpt2") m.family = Family::Gpt2;
      else if (f == "gptj") m.family = Family::GptJ;
      else if (f == "llama") m.family = Family::Llama;
      else throw ConfigError("model JSON: unknown family " + f);
    }
    m.layers = j.value("layers", m.layers);
    m.d_model = j.value("d_model", m.d_model);
    m.heads = j.value("heads", m.heads);
    m.ffn = j.value("ffn", m.ffn);
    m.vocab = j.value("vocab", m.vocab);
    m.rotary_dim = j.value("rotary_dim", m.rotary_dim);
    m.max_pos = j.value("max_pos", m.max_pos);
    m.weight_seed = j.value("weight_seed", m.weight_seed);
    m.token_seed = j.value("token_seed", m.token_seed);
    m.norm_eps = j.value("norm_eps", m.norm_eps);
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("model JSON: ") + e.what());
  }
  if (m.layers < 1 || m.d_model < 64 || m.heads < 1 || m.d_model % m.heads) throw ConfigError("model: bad shape");
  const int hd = m.head_dim();
  if (hd != 64 && hd != 128 && hd != 256) throw ConfigError("model: head_dim must be 64, 128 or 256");
  if (m.d_model % 64 || m.ffn % 64) throw ConfigError("model: d_model and ffn must be multiples of 64");
  if (m.rotary_dim % 2 || m.rotary_dim > hd) throw ConfigError("model: bad rotary_dim");
  if (m.family == Family::Gpt2 && m.rotary_dim) throw ConfigError("model: gpt2 family uses learned positions");
  if (m.family != Family::Gpt2 && !m.rotary_dim) throw ConfigError("model: rotary family needs rotary_dim");
  return m;
}

std::string model_json(const ModelSpec& m) {
  nlohmann::json j;
  j["family"] = m.family == Family::Gpt2 ? "gpt2" : (m.family == Family::GptJ ? "gptj" : "llama");
  j["layers"] = m.layers;
  j["d_model"] = m.d_model;
  j["heads"] = m.heads;
  j["ffn"] = m.ffn;
  j["vocab"] = m.vocab;
  j["rotary_dim"] = m.rotary_dim;
  j["max_pos"] = m.max_pos;
  j["weight_seed"] = m.weight_seed;
  j["token_seed"] = m.token_seed;
  j["norm_eps"] = m.norm_eps;
  j["head_dim"] = m.head_dim();
  j["kv_bytes_per_token"] = m.kv_bytes_per_token();
  return j.dump();
}

WeightLayout layout_weights(const ModelSpec& m) {
  WeightLayout w;
  const std::int64_t D = m.d_model, F = m.ffn, V = m.vocab;
  std::uint32_t next_id = 0;
  // Tensors start on 64-element (128 B) boundaries for vector / TMA access.
  auto put = [&](std::int64_t count, int kind) {
    const std::int64_t off = w.total;
    w.items.push_back({off, count, next_id++, kind});
    w.total += (count + 63) / 64 * 64;
    return off;
  };
  // Projection weight [N][K], tile-blocked (weight_tile_offset).
  auto put_w = [&](std::int64_t N, std::int64_t K) {
    const std::int64_t off = w.total;
    WeightLayout::Item it{off, tiled_weight_elems(N, K), next_id++, 0};
    it.rows = N;
    it.cols = K;
    it.tiled = true;
    w.items.push_back(it);
    w.total += it.count;
    return off;
  };
  const bool bias = m.has_bias();
  w.tok_emb = put(V * D, 0);
  if (m.family == Family::Gpt2) w.pos_emb = put(static_cast<std::int64_t>(m.max_pos) * D, 0);
  for (int l = 0; l < m.layers; ++l) {
    LayerWeights L{};
    L.ln1_g = put(D, 1);
    L.ln1_b = bias ? put(D, 2) : -1;
    if (!m.parallel_residual()) {
      L.ln2_g = put(D, 1);
      L.ln2_b = bias ? put(D, 2) : -1;
    } else {
      L.ln2_g = L.ln2_b = -1;
    }
    L.w_qkv = put_w(3 * D, D);
    L.b_qkv = m.qkv_bias() ? put(3 * D, 0) : -1;
    L.w_o = put_w(D, D);
    L.b_o = m.family == Family::Gpt2 ? put(D, 0) : -1;
    L.w_in = put_w(m.ffn_in_width(), D);
    L.b_in = bias ? put(F, 0) : -1;
    L.w_out = put_w(D, F);
    L.b_out = bias ? put(D, 0) : -1;
    w.layer.push_back(L);
  }
  w.lnf_g = put(D, 1);
  w.lnf_b = bias ? put(D, 2) : -1;
  w.lm_w = put_w(V, D);
  w.lm_b = m.lm_bias() ? put(V, 0) : -1;
  return w;
}

}  // namespace ib2
