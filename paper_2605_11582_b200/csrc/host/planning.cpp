// Host-side planning around the hot path:
//   * plan_sparsity (compress.cpp:298-326): the layer-adaptive 2:4 / 1:4
//     choice that produces the mixed-dispatch keys;
//   * CostModelEstimator (decode.cpp:84-120) behind the C-ABI, so decode
//     loops (and egt_measure_cost_model, decode.cpp here) can feed it
//     device-measured step and verify times;
//   * estimate_trigger and the flatten / tree-mask builder on host views,
//     exported for parity checks against the reference without a GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "egt_b200/decode.hpp"
#include "egt_b200/packed.hpp"

namespace egt_b200 {

// importance_l = mean(score) / mean(|w|) (both summed in double, in storage
// order); the ceil(rho_s * L) most important layers keep two of four, the
// rest one of four; equal importance keeps layer order (stable).
std::vector<SparsityPattern> plan_sparsity(const std::vector<const Matrix*>& scores,
                                           const std::vector<const Matrix*>& weights, double rho_s) {
  if (!(rho_s >= 0.0 && rho_s <= 1.0)) throw std::invalid_argument("rho_s must be in [0, 1]");
  if (scores.size() != weights.size()) throw std::invalid_argument("plan_sparsity: score and weight lists differ");
  const size_t L = scores.size();
  std::vector<double> imp(L, 0.0);
  for (size_t l = 0; l < L; ++l) {
    const Matrix& s = *scores[l];
    const Matrix& w = *weights[l];
    double ssum = 0.0, wsum = 0.0;
    for (float v : s.data) ssum += static_cast<double>(v);
    for (float v : w.data) wsum += std::fabs(static_cast<double>(v));
    const double ms = ssum / static_cast<double>(s.data.size());
    const double mw = wsum / static_cast<double>(w.data.size());
    imp[l] = mw > 0.0 ? ms / mw : 0.0;
  }
  std::vector<size_t> rank(L);
  std::iota(rank.begin(), rank.end(), size_t{0});
  std::stable_sort(rank.begin(), rank.end(), [&](size_t a, size_t b) { return imp[a] > imp[b]; });
  const size_t keep_two = static_cast<size_t>(std::ceil(rho_s * static_cast<double>(L)));
  std::vector<SparsityPattern> out(L, SparsityPattern::kOneOfFour);
  for (size_t i = 0; i < std::min(keep_two, L); ++i) out[rank[i]] = SparsityPattern::kTwoOfFour;
  return out;
}

}  // namespace egt_b200

// ---------------------------------------------------------------- C-ABI
namespace egt_impl {
void set_last_error(const std::string& msg);  // capi.cu
}

struct egt_cost_estimator {
  egt_b200::CostModelEstimator est;
};

namespace {

template <class Fn>
egt_status plan_guard(Fn&& fn) {
  try {
    fn();
    return EGT_OK;
  } catch (const std::invalid_argument& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINVAL;
  } catch (const std::exception& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINTERNAL;
  }
}

egt_b200::DecodeSession session_from(const egt_session_view& v) {
  egt_b200::DecodeSession s;
  s.prompt.assign(v.prompt, v.prompt + v.prompt_len);
  size_t at = 0;
  for (uint32_t b = 0; b < v.n_beams; ++b) {
    egt_b200::BeamHypothesis h;
    h.node = v.beam_node[b];
    h.log_prob = v.beam_log_prob[b];
    h.tokens.assign(v.beam_tokens + at, v.beam_tokens + at + v.beam_len[b]);
    at += v.beam_len[b];
    s.beams.push_back(std::move(h));
  }
  return s;
}

}  // namespace

extern "C" {

EGT_API egt_status egt_host_plan_sparsity(uint32_t n_layers, const uint32_t* rows, const uint32_t* cols,
                                          const float* const* scores, const float* const* weights, double rho_s,
                                          uint8_t* patterns) {
  return plan_guard([&] {
    if (n_layers && (!rows || !cols || !scores || !weights || !patterns))
      throw std::invalid_argument("plan_sparsity: null argument");
    std::vector<egt_b200::Matrix> s(n_layers), w(n_layers);
    std::vector<const egt_b200::Matrix*> sp(n_layers), wp(n_layers);
    for (uint32_t l = 0; l < n_layers; ++l) {
      const size_t n = static_cast<size_t>(rows[l]) * cols[l];
      s[l] = egt_b200::Matrix(rows[l], cols[l]);
      w[l] = egt_b200::Matrix(rows[l], cols[l]);
      std::memcpy(s[l].data.data(), scores[l], n * sizeof(float));
      std::memcpy(w[l].data.data(), weights[l], n * sizeof(float));
      sp[l] = &s[l];
      wp[l] = &w[l];
    }
    const auto plan = egt_b200::plan_sparsity(sp, wp, rho_s);
    for (uint32_t l = 0; l < n_layers; ++l) patterns[l] = static_cast<uint8_t>(plan[l]);
  });
}

EGT_API egt_status egt_cost_estimator_create(double t_step, double alpha, double beta, egt_cost_estimator** out) {
  return plan_guard([&] {
    if (!out) throw std::invalid_argument("cost model: null output");
    *out = new egt_cost_estimator{egt_b200::CostModelEstimator(egt_b200::CostModel{t_step, alpha, beta})};
  });
}

EGT_API egt_status egt_cost_estimator_observe_step(egt_cost_estimator* e, double seconds) {
  return plan_guard([&] {
    if (!e) throw std::invalid_argument("cost model: null estimator");
    e->est.observe_step(seconds);
  });
}

EGT_API egt_status egt_cost_estimator_observe_verify(egt_cost_estimator* e, uint64_t nodes, double seconds) {
  return plan_guard([&] {
    if (!e) throw std::invalid_argument("cost model: null estimator");
    e->est.observe_verify(static_cast<size_t>(nodes), seconds);
  });
}

EGT_API egt_status egt_cost_estimator_model(const egt_cost_estimator* e, double out[3]) {
  return plan_guard([&] {
    if (!e || !out) throw std::invalid_argument("cost model: null argument");
    out[0] = e->est.model().t_step;
    out[1] = e->est.model().alpha;
    out[2] = e->est.model().beta;
  });
}

EGT_API egt_status egt_cost_estimator_destroy(egt_cost_estimator* e) {
  delete e;
  return EGT_OK;
}

EGT_API egt_status egt_host_estimate_trigger(const egt_trie_view* trie, const egt_session_view* session,
                                             double t_step, double alpha, double beta, uint64_t node_cap,
                                             int* trigger, double* saving) {
  return plan_guard([&] {
    if (!trie || !session || !trigger || !saving) throw std::invalid_argument("trigger: null argument");
    const egt_b200::PrefixTrie t = egt_b200::PrefixTrie::from_parents(*trie);
    const egt_b200::TriggerEstimate e = egt_b200::estimate_trigger(
        egt_b200::CostModel{t_step, alpha, beta}, session_from(*session), t, static_cast<size_t>(node_cap));
    *trigger = e.trigger ? 1 : 0;
    *saving = e.predicted_saving;
  });
}

// flatten_subtree + build_tree_mask on host views (same outputs as the
// reference's, decode.cpp:209-299): flat nodes, rows, visibility bits
// (row-major, LSB-first; cap_bits bytes), padded_len and flat_offset.
EGT_API egt_status egt_host_tree_mask(const egt_trie_view* trie, const egt_session_view* session, uint32_t cap_nodes,
                                      uint32_t* n_nodes, uint32_t* fn_token, int32_t* fn_parent, uint32_t* fn_depth,
                                      uint32_t* fn_trie, uint32_t* fn_beam, uint32_t cap_rows, uint32_t* n_rows,
                                      int32_t* tokens, int32_t* positions, uint8_t* vis_bits, size_t cap_bits,
                                      uint32_t* padded_len, uint32_t* flat_offset) {
  return plan_guard([&] {
    if (!trie || !session || !n_nodes || !n_rows) throw std::invalid_argument("tree mask: null argument");
    const egt_b200::PrefixTrie t = egt_b200::PrefixTrie::from_parents(*trie);
    const egt_b200::DecodeSession s = session_from(*session);
    const egt_b200::FlattenedSubtree flat = egt_b200::flatten_subtree(s, t);
    const egt_b200::TreeMask m = egt_b200::build_tree_mask(flat, s, true);
    *n_nodes = static_cast<uint32_t>(flat.nodes.size());
    *n_rows = m.rows;
    if (flat.nodes.size() > cap_nodes || m.rows > cap_rows || m.bits.size() > cap_bits)
      throw std::invalid_argument("tree mask: output capacity too small");
    for (size_t i = 0; i < flat.nodes.size(); ++i) {
      fn_token[i] = flat.nodes[i].token;
      fn_parent[i] = flat.nodes[i].parent;
      fn_depth[i] = flat.nodes[i].depth;
      fn_trie[i] = flat.nodes[i].trie_node;
      fn_beam[i] = flat.nodes[i].beam;
    }
    std::copy(m.tokens.begin(), m.tokens.end(), tokens);
    std::copy(m.positions.begin(), m.positions.end(), positions);
    std::copy(m.bits.begin(), m.bits.end(), vis_bits);
    *padded_len = m.padded_len;
    *flat_offset = static_cast<uint32_t>(m.flat_offset);
  });
}

}  // extern "C"
