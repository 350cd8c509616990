// extern "C" wrappers over the UNMODIFIED reference model / decoder sources
// (model.cpp, decode.cpp, compress.cpp's plan_sparsity under
// /root/reference/proj/src), built by oracle/build_ref.sh into
// oracle/_ref/libegt_ref.so next to ref_capi.cpp.  Written for this repo: it
// only converts flat buffers to the reference's value types (ToyTransformer,
// PrefixTrie, DecodeSession, ...) and back.  The view structs mirror the
// product's C-ABI views field for field so the tests hand both sides the same
// ctypes objects.  Test infrastructure only (the verify-path oracle).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "egt/compress.hpp"
#include "egt/decode.hpp"
#include "egt/model.hpp"
#include "egt/trie.hpp"

extern "C" const char* ref_last_error(void);
void ref_set_error(const std::string& m);  // ref_capi.cpp

namespace {

struct RefModelConfig {
  uint32_t vocab_size, d_model, n_layers, n_heads, d_ff, max_positions;
};
struct RefTrieView {
  uint32_t n_nodes;
  const uint32_t* token;
  const uint32_t* parent;
  const int64_t* payload;
};
struct RefSessionView {
  const int32_t* prompt;
  uint32_t prompt_len;
  uint32_t n_beams;
  const uint32_t* beam_node;
  const double* beam_log_prob;
  const uint32_t* beam_len;
  const int32_t* beam_tokens;
};
struct RefVerifyOut {
  uint32_t n_selected;
  double* score;
  int64_t* payload;
  uint32_t* beam;
  uint32_t* len;
  int32_t* tokens;
  uint32_t tokens_stride;
  uint32_t flattened_nodes;
  uint32_t rows;
};
struct RefDecodeOptions {
  int beam_size;
  int mode;
  int forced_depth;
  double t_step, alpha, beta;
  uint64_t node_cap;
};

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    ref_set_error(e.what());
    return 1;
  } catch (const egt::FormatError& e) {
    ref_set_error(e.what());
    return 2;
  } catch (const egt::InvariantError& e) {
    ref_set_error(e.what());
    return 3;
  } catch (const std::exception& e) {
    ref_set_error(e.what());
    return 4;
  }
}

egt::Matrix mat(const float* w, uint32_t rows, uint32_t cols) {
  egt::Matrix m(rows, cols);
  std::memcpy(m.data(), w, sizeof(float) * rows * cols);  // egt::Matrix is row-major
  return m;
}

// PrefixTrie from parent links (parents precede children); children in
// ascending token order; descendants / max_depth_below as trie.cpp's
// recompute_derived defines them (strict descendants; edges of the longest
// downward path).
egt::PrefixTrie make_trie(const RefTrieView* v) {
  egt::PrefixTrie t;
  t.nodes.resize(v->n_nodes);
  for (uint32_t i = 0; i < v->n_nodes; ++i) {
    t.nodes[i].token = v->token[i];
    t.nodes[i].payload = v->payload[i];
    if (i == 0) continue;
    const uint32_t p = v->parent[i];
    if (p >= i) throw std::invalid_argument("ref trie: parents must precede children");
    t.nodes[i].parent = p;
    t.nodes[i].depth = t.nodes[p].depth + 1;
    t.nodes[p].children.push_back(i);
  }
  for (auto& n : t.nodes)
    std::stable_sort(n.children.begin(), n.children.end(),
                     [&](uint32_t a, uint32_t b) { return t.nodes[a].token < t.nodes[b].token; });
  t.descendants.assign(v->n_nodes, 0);
  t.max_depth_below.assign(v->n_nodes, 0);
  for (uint32_t i = v->n_nodes; i-- > 1;) {
    const uint32_t p = t.nodes[i].parent;
    t.descendants[p] += 1 + t.descendants[i];
    t.max_depth_below[p] = std::max(t.max_depth_below[p], t.max_depth_below[i] + 1);
  }
  return t;
}

egt::DecodeSession make_session(const RefSessionView* s) {
  egt::DecodeSession ses = egt::make_session(std::vector<int>(s->prompt, s->prompt + s->prompt_len));
  ses.beams.clear();
  size_t off = 0;
  for (uint32_t b = 0; b < s->n_beams; ++b) {
    egt::BeamHypothesis h;
    h.node = s->beam_node[b];
    h.log_prob = s->beam_log_prob[b];
    h.tokens.assign(s->beam_tokens + off, s->beam_tokens + off + s->beam_len[b]);
    off += s->beam_len[b];
    ses.beams.push_back(std::move(h));
  }
  return ses;
}

void write_selected(const std::vector<egt::VerifiedLeaf>& sel, RefVerifyOut* o) {
  o->n_selected = static_cast<uint32_t>(sel.size());
  for (size_t j = 0; j < sel.size(); ++j) {
    o->score[j] = sel[j].score;
    o->payload[j] = sel[j].payload;
    o->beam[j] = sel[j].beam;
    const size_t n = std::min<size_t>(sel[j].tokens.size(), o->tokens_stride);
    o->len[j] = static_cast<uint32_t>(n);
    for (size_t i = 0; i < n; ++i) o->tokens[j * o->tokens_stride + i] = sel[j].tokens[i];
  }
}

}  // namespace

extern "C" {

// A ToyTransformer (model.hpp:53-59) from flat row-major f32 weights:
// layers[6*l + {0..5}] = wq wk wv wo ff1 ff2.  The sinusoidal table comes
// from the reference's own init_model (model.cpp:300-330) on a config of the
// same d_model / max_positions.
void* ref_model_new(const RefModelConfig* c, const float* emb, const float* const* layers, const float* head) {
  try {
    egt::ModelConfig cfg;
    cfg.vocab_size = c->vocab_size;
    cfg.d_model = c->d_model;
    cfg.n_layers = c->n_layers;
    cfg.n_heads = c->n_heads;
    cfg.d_ff = c->d_ff;
    cfg.max_positions = c->max_positions;
    cfg.validate();
    egt::ModelConfig tiny = cfg;
    tiny.vocab_size = 1;
    tiny.n_layers = 1;
    tiny.d_ff = 1;
    auto* m = new egt::ToyTransformer;
    m->config = cfg;
    m->positions = egt::init_model(tiny).positions;
    m->embedding = mat(emb, cfg.vocab_size, cfg.d_model);
    m->layers.resize(cfg.n_layers);
    for (uint32_t l = 0; l < cfg.n_layers; ++l) {
      egt::LayerWeights& w = m->layers[l];
      const uint32_t d = cfg.d_model, f = cfg.d_ff;
      w.wq = mat(layers[6 * l + 0], d, d);
      w.wk = mat(layers[6 * l + 1], d, d);
      w.wv = mat(layers[6 * l + 2], d, d);
      w.wo = mat(layers[6 * l + 3], d, d);
      w.ff1 = mat(layers[6 * l + 4], f, d);
      w.ff2 = mat(layers[6 * l + 5], d, f);
    }
    m->head = mat(head, cfg.vocab_size, cfg.d_model);
    return m;
  } catch (const std::exception& e) {
    ref_set_error(e.what());
    return nullptr;
  }
}

void ref_model_free(void* m) { delete static_cast<egt::ToyTransformer*>(m); }

// The model's sinusoidal position table [max_positions x d_model].
int ref_model_positions(const void* m, float* out) {
  return guarded([&] {
    const auto& p = static_cast<const egt::ToyTransformer*>(m)->positions;
    std::memcpy(out, p.data(), sizeof(float) * p.size());
  });
}

// forward (model.hpp:71-72, model.cpp:118-202): logits [M x vocab].
// mask_bits: M*M bits, little-endian bit order, row-major (visible(q,k)).
int ref_forward(const void* mp, const int32_t* tokens, const int32_t* positions, const uint8_t* mask_bits,
                uint32_t M, float* logits) {
  return guarded([&] {
    const auto& m = *static_cast<const egt::ToyTransformer*>(mp);
    egt::Mask mask(M, M);
    for (uint32_t q = 0; q < M; ++q)
      for (uint32_t k = 0; k < M; ++k) {
        const size_t i = static_cast<size_t>(q) * M + k;
        mask(q, k) = (mask_bits[i >> 3] >> (i & 7)) & 1;
      }
    std::vector<int> t(tokens, tokens + M), p(positions, positions + M);
    egt::Matrix out = egt::forward(m, t, mask, p);
    std::memcpy(logits, out.data(), sizeof(float) * out.size());
  });
}

// log_softmax (model.cpp:370-377) of one row.
int ref_log_softmax(const float* row, uint32_t n, float* out) {
  return guarded([&] {
    egt::RowVector r(n);
    for (uint32_t i = 0; i < n; ++i) r(i) = row[i];
    egt::RowVector o = egt::log_softmax(r);
    for (uint32_t i = 0; i < n; ++i) out[i] = o(i);
  });
}

// flatten_subtree + build_tree_mask (decode.cpp:209-299) for a session:
// flat nodes (token, parent, depth, trie_node, beam) and the TreeMask rows
// (tokens, positions, visibility bits little-endian row-major), padded_len,
// flat_offset.  Capacities: cap_nodes flat nodes, cap_rows rows.
int ref_tree_mask(const RefTrieView* tv, const RefSessionView* sv, uint32_t cap_nodes, uint32_t* n_nodes,
                  uint32_t* fn_token, int32_t* fn_parent, uint32_t* fn_depth, uint32_t* fn_trie, uint32_t* fn_beam,
                  uint32_t cap_rows, uint32_t* n_rows, int32_t* tokens, int32_t* positions, uint8_t* vis_bits,
                  uint32_t* padded_len, uint32_t* flat_offset) {
  return guarded([&] {
    const egt::PrefixTrie trie = make_trie(tv);
    const egt::DecodeSession ses = make_session(sv);
    const egt::FlattenedSubtree fl = egt::flatten_subtree(ses, trie);
    const egt::TreeMask tm = egt::build_tree_mask(fl, ses);
    *n_nodes = static_cast<uint32_t>(fl.nodes.size());
    *n_rows = static_cast<uint32_t>(tm.tokens.size());
    if (fl.nodes.size() > cap_nodes || tm.tokens.size() > cap_rows)
      throw std::invalid_argument("ref_tree_mask: output capacity too small");
    for (size_t i = 0; i < fl.nodes.size(); ++i) {
      fn_token[i] = fl.nodes[i].token;
      fn_parent[i] = fl.nodes[i].parent;
      fn_depth[i] = fl.nodes[i].depth;
      fn_trie[i] = fl.nodes[i].trie_node;
      fn_beam[i] = fl.nodes[i].beam;
    }
    const size_t R = tm.tokens.size();
    std::memset(vis_bits, 0, (R * R + 7) / 8);
    for (size_t q = 0; q < R; ++q) {
      tokens[q] = tm.tokens[q];
      positions[q] = tm.positions[q];
      for (size_t k = 0; k < R; ++k)
        if (tm.visibility(q, k)) vis_bits[(q * R + k) >> 3] |= static_cast<uint8_t>(1u << ((q * R + k) & 7));
    }
    *padded_len = tm.padded_len;
    *flat_offset = static_cast<uint32_t>(tm.flat_offset);
  });
}

// verify_parallel (decode.cpp:336-421) on the session the view describes;
// node_scores (optional) receives the cumulative score per flattened node.
int ref_verify_parallel(const void* mp, const RefTrieView* tv, const RefSessionView* sv, int beam_size,
                        RefVerifyOut* out, double* node_scores, uint32_t cap_nodes) {
  return guarded([&] {
    const auto& m = *static_cast<const egt::ToyTransformer*>(mp);
    const egt::PrefixTrie trie = make_trie(tv);
    egt::DecodeSession ses = make_session(sv);
    const egt::FlattenedSubtree fl = egt::flatten_subtree(ses, trie);
    const egt::TreeMask tm = egt::build_tree_mask(fl, ses);
    egt::VerificationResult r = egt::verify_parallel(m, ses, trie, fl, tm, beam_size);
    write_selected(r.selected, out);
    out->flattened_nodes = static_cast<uint32_t>(fl.nodes.size());
    out->rows = static_cast<uint32_t>(tm.tokens.size());
    if (node_scores)
      for (size_t i = 0; i < r.node_scores.size() && i < cap_nodes; ++i) node_scores[i] = r.node_scores[i];
  });
}

// decode (decode.cpp:423-483).  stats: steps, forward_passes, trigger_step,
// flattened_nodes.
int ref_decode(const void* mp, const RefTrieView* tv, const int32_t* prompt, uint32_t prompt_len,
               const RefDecodeOptions* o, RefVerifyOut* out, int32_t* stats) {
  return guarded([&] {
    const auto& m = *static_cast<const egt::ToyTransformer*>(mp);
    const egt::PrefixTrie trie = make_trie(tv);
    egt::DecodeOptions opt;
    opt.beam_size = o->beam_size;
    opt.mode = static_cast<egt::DecodeMode>(o->mode);
    opt.forced_depth = o->forced_depth;
    opt.cost_model.t_step = o->t_step;
    opt.cost_model.alpha = o->alpha;
    opt.cost_model.beta = o->beta;
    opt.node_cap = o->node_cap;
    egt::DecodeResult r = egt::decode(m, trie, std::vector<int>(prompt, prompt + prompt_len), opt);
    std::vector<egt::VerifiedLeaf> sel;
    for (const auto& s : r.sequences) {
      egt::VerifiedLeaf v;
      v.tokens = s.tokens;
      v.score = s.score;
      v.payload = s.payload;
      sel.push_back(std::move(v));
    }
    write_selected(sel, out);
    stats[0] = r.stats.steps;
    stats[1] = r.stats.forward_passes;
    stats[2] = r.stats.trigger_step;
    stats[3] = static_cast<int32_t>(r.stats.flattened_nodes);
  });
}

// constrained_step (decode.cpp:122-190) applied n_steps times to the session
// the view describes; the resulting beams (node, log_prob, tokens) are written
// back: beam_node / beam_log_prob / beam_len [cap_beams], beam_tokens
// [cap_beams * stride].
int ref_constrained_steps(const void* mp, const RefTrieView* tv, const RefSessionView* sv, int beam_size,
                          int n_steps, uint32_t cap_beams, uint32_t stride, uint32_t* n_beams, uint32_t* beam_node,
                          double* beam_log_prob, uint32_t* beam_len, int32_t* beam_tokens) {
  return guarded([&] {
    const auto& m = *static_cast<const egt::ToyTransformer*>(mp);
    const egt::PrefixTrie trie = make_trie(tv);
    egt::DecodeSession ses = make_session(sv);
    for (int i = 0; i < n_steps; ++i) egt::constrained_step(m, ses, trie, beam_size);
    if (ses.beams.size() > cap_beams) throw std::invalid_argument("ref_constrained_steps: too many beams");
    *n_beams = static_cast<uint32_t>(ses.beams.size());
    for (size_t b = 0; b < ses.beams.size(); ++b) {
      beam_node[b] = ses.beams[b].node;
      beam_log_prob[b] = ses.beams[b].log_prob;
      const size_t n = std::min<size_t>(ses.beams[b].tokens.size(), stride);
      beam_len[b] = static_cast<uint32_t>(n);
      for (size_t i = 0; i < n; ++i) beam_tokens[b * stride + i] = ses.beams[b].tokens[i];
    }
  });
}

// estimate_trigger (decode.cpp:192-207).
int ref_estimate_trigger(const RefTrieView* tv, const RefSessionView* sv, double t_step, double alpha, double beta,
                         uint64_t node_cap, int* trigger, double* saving) {
  return guarded([&] {
    const egt::PrefixTrie trie = make_trie(tv);
    const egt::DecodeSession ses = make_session(sv);
    egt::CostModel c;
    c.t_step = t_step;
    c.alpha = alpha;
    c.beta = beta;
    egt::TriggerEstimate e = egt::estimate_trigger(c, ses, trie, node_cap);
    *trigger = e.trigger ? 1 : 0;
    *saving = e.predicted_saving;
  });
}

// CostModelEstimator (decode.cpp:84-120) fed a sequence of observations:
// kind[i] 0 = observe_step(seconds[i]), 1 = observe_verify(nodes[i], seconds[i]).
// out: t_step, alpha, beta after the last observation.
int ref_cost_estimator(uint32_t n, const int* kind, const uint64_t* nodes, const double* seconds, double init_t_step,
                       double init_alpha, double init_beta, double out[3]) {
  return guarded([&] {
    egt::CostModel c0;
    c0.t_step = init_t_step;
    c0.alpha = init_alpha;
    c0.beta = init_beta;
    egt::CostModelEstimator est(c0);
    for (uint32_t i = 0; i < n; ++i) {
      if (kind[i] == 0)
        est.observe_step(seconds[i]);
      else
        est.observe_verify(static_cast<size_t>(nodes[i]), seconds[i]);
    }
    out[0] = est.model().t_step;
    out[1] = est.model().alpha;
    out[2] = est.model().beta;
  });
}

// plan_sparsity (compress.cpp:298-326): scores[i] / weights[i] are row-major
// rows[i] x cols[i]; patterns[i] receives 1 (1:4) or 2 (2:4).
int ref_plan_sparsity(uint32_t n_layers, const uint32_t* rows, const uint32_t* cols, const float* const* scores,
                      const float* const* weights, double rho_s, uint8_t* patterns) {
  return guarded([&] {
    std::vector<egt::ImportanceMatrix> sc(n_layers);
    std::vector<egt::Matrix> ws(n_layers);
    std::vector<const egt::Matrix*> wp(n_layers);
    for (uint32_t i = 0; i < n_layers; ++i) {
      sc[i].scores = mat(scores[i], rows[i], cols[i]);
      ws[i] = mat(weights[i], rows[i], cols[i]);
      wp[i] = &ws[i];
    }
    egt::LayerSparsityPlan p = egt::plan_sparsity(sc, wp, rho_s);
    for (uint32_t i = 0; i < n_layers; ++i) patterns[i] = static_cast<uint8_t>(p.patterns[i]);
  });
}

}  // extern "C"
