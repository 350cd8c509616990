// Prefix-tree parallel verification and trie-constrained beam decoding
// (egt_b200/decode.hpp).  The reference's scoring convention is kept exactly:
// every expansion renormalises the logits over the trie-legal children
// (decode.hpp:20-23), in f32 with the partition sum in double
// (model.cpp:370-377), so a sequence's score does not depend on where the
// switch to parallel verification happens.  Only the forward pass changes: it
// is one egt_forward call on the B200 over the packed layers.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "egt_b200/decode.hpp"
#include "egt_b200/packed.hpp"

namespace egt_b200 {

namespace {

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

// Position of every node within its parent's (ascending) children list.
std::vector<uint32_t> child_slots(const PrefixTrie& trie) {
  std::vector<uint32_t> slot(trie.nodes.size(), 0);
  for (const TrieNode& n : trie.nodes)
    for (uint32_t i = 0; i < n.children.size(); ++i) slot[n.children[i]] = i;
  return slot;
}

void check_beams(const DecodeSession& s, const PrefixTrie& trie) {
  require(!s.beams.empty(), "decode: session has no beams");
  for (const BeamHypothesis& b : s.beams) require(b.node < trie.nodes.size(), "decode: beam node outside the trie");
}

std::vector<int> committed(const DecodeSession& s, const BeamHypothesis& b) {
  std::vector<int> seq(s.prompt);
  seq.insert(seq.end(), b.tokens.begin(), b.tokens.end());
  return seq;
}

// Device forward + gather of the logits a set of rows needs at the given
// token columns (children of the row's trie node).
struct RowRequest {
  uint32_t row;
  uint32_t node;  // trie node whose children are scored
};

template <class Forward>
std::vector<std::vector<float>> score_rows_with(const PrefixTrie& trie, uint32_t M, Forward&& forward,
                                                const std::vector<RowRequest>& reqs, uint32_t vocab, void* stream) {
  std::vector<uint32_t> rows, cols;
  for (const RowRequest& r : reqs)
    for (uint32_t c : trie.nodes[r.node].children) {
      const uint32_t t = trie.nodes[c].token;
      if (t >= vocab)
        throw std::invalid_argument("decode: trie token " + std::to_string(t) + " outside the model vocabulary");
      rows.push_back(r.row);
      cols.push_back(t);
    }
  float* logits = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cudaMallocAsync(reinterpret_cast<void**>(&logits), static_cast<size_t>(M) * vocab * sizeof(float), s) !=
      cudaSuccess)
    throw CudaError("decode: logits allocation failed");
  std::vector<float> vals(rows.size());
  egt_status st = forward(logits);
  if (st == EGT_OK)
    st = egt_gather(logits, vocab, rows.data(), cols.data(), static_cast<uint32_t>(rows.size()), vals.data(), stream);
  cudaFreeAsync(logits, s);
  if (st != EGT_OK) throw_status(st);
  std::vector<std::vector<float>> out;
  out.reserve(reqs.size());
  size_t at = 0;
  for (const RowRequest& r : reqs) {
    const size_t n = trie.nodes[r.node].children.size();
    out.push_back(restricted_log_softmax(std::vector<float>(vals.begin() + at, vals.begin() + at + n)));
    at += n;
  }
  return out;
}

std::vector<std::vector<float>> score_rows(const egt_model* model, const PrefixTrie& trie,
                                           const std::vector<int>& tokens, const std::vector<int>& positions,
                                           const std::vector<uint8_t>* bits, const egt_tree_view* tree,
                                           const std::vector<RowRequest>& reqs, uint32_t vocab, void* stream) {
  const uint32_t M = static_cast<uint32_t>(tokens.size());
  return score_rows_with(
      trie, M,
      [&](float* logits) {
        return tree ? egt_forward_tree(model, tokens.data(), positions.data(), tree, logits, stream)
                    : egt_forward(model, tokens.data(), positions.data(), bits->data(), M, logits, stream);
      },
      reqs, vocab, stream);
}

void set_bit(std::vector<uint8_t>& bits, size_t i) { bits[i >> 3] |= static_cast<uint8_t>(1u << (i & 7)); }

uint32_t vocab_of(const egt_model* model) {
  egt_model_config c{};
  check(egt_model_query(model, &c));
  return c.vocab_size;
}

}  // namespace

PrefixTrie PrefixTrie::from_parents(const egt_trie_view& v) {
  require(v.n_nodes > 0, "trie: no nodes");
  PrefixTrie t;
  t.nodes.resize(v.n_nodes);
  for (uint32_t i = 0; i < v.n_nodes; ++i) {
    t.nodes[i].token = v.token[i];
    t.nodes[i].payload = v.payload ? v.payload[i] : kNoPayload;
    if (i == 0) continue;
    const uint32_t p = v.parent[i];
    require(p < i, "trie: parents must precede children");
    t.nodes[i].parent = p;
    t.nodes[i].depth = t.nodes[p].depth + 1;
    t.nodes[p].children.push_back(i);
  }
  for (TrieNode& n : t.nodes)
    std::stable_sort(n.children.begin(), n.children.end(),
                     [&](uint32_t a, uint32_t b) { return t.nodes[a].token < t.nodes[b].token; });
  t.descendants.assign(v.n_nodes, 0);
  t.max_depth_below.assign(v.n_nodes, 0);
  for (uint32_t i = v.n_nodes; i-- > 1;) {  // recompute_derived (trie.cpp:225-236)
    const uint32_t p = t.nodes[i].parent;
    t.descendants[p] += t.descendants[i] + 1;
    t.max_depth_below[p] = std::max(t.max_depth_below[p], t.max_depth_below[i] + 1);
  }
  return t;
}

DecodeSession make_session(std::vector<int> prompt) {
  require(!prompt.empty(), "decode: empty prompt");
  DecodeSession s;
  s.prompt = std::move(prompt);
  s.beams.emplace_back();
  return s;
}

void CostModelEstimator::observe_step(double seconds) {  // EMA 0.9 (decode.cpp:84-94)
  require(std::isfinite(seconds) && seconds >= 0.0, "cost model: step time must be finite and non-negative");
  model_.t_step = seeded_ ? 0.9 * model_.t_step + 0.1 * seconds : seconds;
  seeded_ = true;
}

void CostModelEstimator::observe_verify(size_t nodes, double seconds) {  // LSQ, 32 samples
  require(std::isfinite(seconds) && seconds >= 0.0,
          "cost model: verification time must be finite and non-negative");
  require(nodes > 0, "cost model: verification over zero nodes");
  window_.emplace_back(static_cast<double>(nodes), seconds);
  if (window_.size() > 32) window_.erase(window_.begin());
  double sn = 0.0, st = 0.0;
  for (const auto& w : window_) {
    sn += w.first;
    st += w.second;
  }
  const double mn = sn / window_.size(), mt = st / window_.size();
  double var = 0.0, cov = 0.0;
  for (const auto& w : window_) {
    var += (w.first - mn) * (w.first - mn);
    cov += (w.first - mn) * (w.second - mt);
  }
  if (var > 0.0) model_.alpha = cov / var;
  model_.beta = mt - model_.alpha * mn;
}

std::vector<float> restricted_log_softmax(const std::vector<float>& l) {
  float m = -std::numeric_limits<float>::infinity();
  for (float v : l) m = std::max(m, v);
  double z = 0.0;
  for (float v : l) z += std::exp(static_cast<double>(v - m));
  const float lz = static_cast<float>(std::log(z));
  std::vector<float> out(l.size());
  for (size_t i = 0; i < l.size(); ++i) out[i] = (l[i] - m) - lz;
  return out;
}

FlattenedSubtree flatten_subtree(const DecodeSession& s, const PrefixTrie& trie) {
  check_beams(s, trie);
  FlattenedSubtree f;
  std::vector<std::pair<uint32_t, int32_t>> todo;  // (trie node, flat parent), DFS stack
  for (uint32_t b = 0; b < s.beams.size(); ++b) {
    const std::vector<uint32_t>& top = trie.nodes[s.beams[b].node].children;
    for (size_t i = top.size(); i-- > 0;) todo.emplace_back(top[i], -1);
    while (!todo.empty()) {
      const auto [node, parent] = todo.back();
      todo.pop_back();
      FlatNode fn;
      fn.token = trie.nodes[node].token;
      fn.parent = parent;
      fn.depth = parent < 0 ? 0 : f.nodes[parent].depth + 1;
      fn.trie_node = node;
      fn.beam = b;
      const int32_t me = static_cast<int32_t>(f.nodes.size());
      f.nodes.push_back(fn);
      const std::vector<uint32_t>& ch = trie.nodes[node].children;
      for (size_t i = ch.size(); i-- > 0;) todo.emplace_back(ch[i], me);
    }
  }
  require(!f.nodes.empty(), "decode: nothing to verify, every beam is finished");
  return f;
}

TreeMask build_tree_mask(const FlattenedSubtree& flat, const DecodeSession& s, bool with_bits) {
  require(!s.beams.empty(), "decode: session has no beams");
  require(!flat.nodes.empty(), "decode: empty flattened subtree");
  TreeMask m;
  const uint32_t nb = static_cast<uint32_t>(s.beams.size());
  m.beam_count = nb;
  m.committed_len.resize(nb);
  uint32_t lmax = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    m.committed_len[b] = static_cast<uint32_t>(s.prompt.size() + s.beams[b].tokens.size());
    lmax = std::max(lmax, m.committed_len[b]);
  }
  m.padded_len = lmax;
  m.flat_offset = static_cast<size_t>(nb) * lmax;
  m.rows = static_cast<uint32_t>(m.flat_offset + flat.nodes.size());
  const size_t R = m.rows;
  if (with_bits) m.bits.assign((R * R + 7) / 8, 0);
  m.tokens.assign(R, static_cast<int>(kPadToken));  // pad rows: token 0, position 0, invisible
  m.positions.assign(R, 0);
  for (uint32_t b = 0; b < nb; ++b) {  // committed blocks, left-padded, causal
    const std::vector<int> seq = committed(s, s.beams[b]);
    const size_t first = static_cast<size_t>(b) * lmax + (lmax - seq.size());
    for (size_t j = 0; j < seq.size(); ++j) {
      m.tokens[first + j] = seq[j];
      m.positions[first + j] = static_cast<int>(j);
      if (with_bits)
        for (size_t k = 0; k <= j; ++k) set_bit(m.bits, (first + j) * R + first + k);
    }
  }
  for (size_t f = 0; f < flat.nodes.size(); ++f) {  // node rows: committed + ancestors + self
    const FlatNode& fn = flat.nodes[f];
    require(fn.beam < nb, "decode: flattened node references a missing beam");
    require(fn.parent < 0 || (static_cast<size_t>(fn.parent) < f && flat.nodes[fn.parent].beam == fn.beam),
            "decode: flattened parent does not precede its child");
    const size_t r = m.flat_offset + f;
    const uint32_t len = m.committed_len[fn.beam];
    m.tokens[r] = static_cast<int>(fn.token);
    m.positions[r] = static_cast<int>(len + fn.depth);
    const size_t first = static_cast<size_t>(fn.beam) * lmax + (lmax - len);
    if (!with_bits) continue;
    for (size_t j = 0; j < len; ++j) set_bit(m.bits, r * R + first + j);
    for (int32_t p = static_cast<int32_t>(f); p >= 0; p = flat.nodes[p].parent) set_bit(m.bits, r * R + m.flat_offset + p);
  }
  return m;
}

std::vector<double> accumulate_bscores(const FlattenedSubtree& flat, const PrefixTrie& trie,
                                       const DecodeSession& s,
                                       const std::vector<std::vector<float>>& seeds,
                                       const std::vector<std::vector<float>>& rows) {
  require(seeds.size() == s.beams.size(), "decode: seed rows and beam scores disagree");
  require(rows.size() == flat.nodes.size(), "decode: per-node rows and flattened nodes disagree");
  const std::vector<uint32_t> slot = child_slots(trie);
  std::vector<double> score(flat.nodes.size());
  for (size_t f = 0; f < flat.nodes.size(); ++f) {  // B(child) = B(parent) + T_parent[token]
    const FlatNode& fn = flat.nodes[f];
    const std::vector<float>* row;
    double base;
    if (fn.parent < 0) {
      require(fn.beam < s.beams.size(), "decode: flattened node references a missing beam");
      row = &seeds[fn.beam];
      base = s.beams[fn.beam].log_prob;
    } else {
      require(static_cast<size_t>(fn.parent) < f, "decode: flattened parent does not precede its child");
      row = &rows[fn.parent];
      base = score[fn.parent];
    }
    require(slot[fn.trie_node] < row->size(), "decode: token outside the scored row");
    score[f] = base + (*row)[slot[fn.trie_node]];
  }
  return score;
}

VerificationResult verify_parallel(const egt_model* model, DecodeSession& s, const PrefixTrie& trie,
                                   const FlattenedSubtree& flat, const TreeMask& mask, int beam_size,
                                   void* stream) {
  require(beam_size >= 1, "decode: beam_size must be positive");
  check_beams(s, trie);
  require(!flat.nodes.empty(), "decode: empty flattened subtree");
  const size_t nb = s.beams.size();
  require(mask.beam_count == nb && mask.flat_offset == nb * static_cast<size_t>(mask.padded_len) &&
              mask.rows == mask.flat_offset + flat.nodes.size() && mask.tokens.size() == mask.rows &&
              mask.positions.size() == mask.rows,
          "decode: tree mask does not match the session and subtree");
  // rows to score: each unfinished beam's newest token, each interior node
  std::vector<RowRequest> reqs;
  std::vector<int> seed_at(nb, -1), row_at(flat.nodes.size(), -1);
  for (size_t b = 0; b < nb; ++b)
    if (!trie.is_leaf(s.beams[b].node)) {
      seed_at[b] = static_cast<int>(reqs.size());
      reqs.push_back({static_cast<uint32_t>(b * mask.padded_len + mask.padded_len - 1), s.beams[b].node});
    }
  for (size_t f = 0; f < flat.nodes.size(); ++f)
    if (!trie.is_leaf(flat.nodes[f].trie_node)) {
      row_at[f] = static_cast<int>(reqs.size());
      reqs.push_back({static_cast<uint32_t>(mask.flat_offset + f), flat.nodes[f].trie_node});
    }
  std::vector<std::vector<float>> scored;
  if (mask.bits.empty()) {  // compact tree encoding: the device builds the mask
    std::vector<int32_t> parent(flat.nodes.size());
    std::vector<uint32_t> beam(flat.nodes.size());
    for (size_t f = 0; f < flat.nodes.size(); ++f) {
      parent[f] = flat.nodes[f].parent;
      beam[f] = flat.nodes[f].beam;
    }
    egt_tree_view tv{static_cast<uint32_t>(nb), mask.padded_len, mask.committed_len.data(),
                     static_cast<uint32_t>(flat.nodes.size()), parent.data(), beam.data()};
    scored = score_rows(model, trie, mask.tokens, mask.positions, nullptr, &tv, reqs, vocab_of(model), stream);
  } else {
    scored = score_rows(model, trie, mask.tokens, mask.positions, &mask.bits, nullptr, reqs, vocab_of(model), stream);
  }
  s.forward_passes += 1;
  s.flattened_nodes = flat.nodes.size();

  VerificationResult out;
  std::vector<std::vector<float>> seeds(nb);
  for (size_t b = 0; b < nb; ++b)
    if (seed_at[b] >= 0) seeds[b] = scored[seed_at[b]];
  out.node_rows.resize(flat.nodes.size());
  for (size_t f = 0; f < flat.nodes.size(); ++f)
    if (row_at[f] >= 0) out.node_rows[f] = scored[row_at[f]];
  out.node_scores = accumulate_bscores(flat, trie, s, seeds, out.node_rows);

  struct Cand {
    double score;
    uint32_t beam;
    int64_t flat;  // -1: a finished beam competing as is
  };
  std::vector<Cand> cands;
  for (size_t b = 0; b < nb; ++b)
    if (trie.is_leaf(s.beams[b].node)) cands.push_back({s.beams[b].log_prob, static_cast<uint32_t>(b), -1});
  for (size_t f = 0; f < flat.nodes.size(); ++f)
    if (trie.is_leaf(flat.nodes[f].trie_node))
      cands.push_back({out.node_scores[f], flat.nodes[f].beam, static_cast<int64_t>(f)});
  std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
    if (a.score != b.score) return a.score > b.score;
    if (a.beam != b.beam) return a.beam < b.beam;
    return a.flat < b.flat;
  });
  const size_t keep = std::min(static_cast<size_t>(beam_size), cands.size());
  for (size_t j = 0; j < keep; ++j) {
    const Cand& c = cands[j];
    VerifiedLeaf leaf;
    leaf.score = c.score;
    leaf.beam = c.beam;
    leaf.tokens = s.beams[c.beam].tokens;
    if (c.flat < 0) {
      leaf.payload = trie.nodes[s.beams[c.beam].node].payload;
    } else {
      std::vector<int> path;
      for (int64_t p = c.flat; p >= 0; p = flat.nodes[p].parent) path.push_back(static_cast<int>(flat.nodes[p].token));
      leaf.tokens.insert(leaf.tokens.end(), path.rbegin(), path.rend());
      leaf.payload = trie.nodes[flat.nodes[c.flat].trie_node].payload;
    }
    out.selected.push_back(std::move(leaf));
  }
  return out;
}

void constrained_step(const egt_model* model, DecodeSession& s, const PrefixTrie& trie, int beam_size,
                      void* stream) {
  require(beam_size >= 1, "decode: beam_size must be positive");
  check_beams(s, trie);
  std::vector<size_t> active;
  for (size_t i = 0; i < s.beams.size(); ++i)
    if (!trie.is_leaf(s.beams[i].node)) active.push_back(i);
  require(!active.empty(), "decode: every beam is finished");
  // one block-diagonal causal forward over the unfinished beams (full recompute)
  std::vector<int> tokens, positions;
  std::vector<size_t> start(active.size()), len(active.size());
  for (size_t a = 0; a < active.size(); ++a) {
    const std::vector<int> seq = committed(s, s.beams[active[a]]);
    start[a] = tokens.size();
    len[a] = seq.size();
    for (size_t j = 0; j < seq.size(); ++j) {
      tokens.push_back(seq[j]);
      positions.push_back(static_cast<int>(j));
    }
  }
  const size_t R = tokens.size();
  std::vector<uint8_t> bits((R * R + 7) / 8, 0);
  for (size_t a = 0; a < active.size(); ++a)
    for (size_t q = 0; q < len[a]; ++q)
      for (size_t k = 0; k <= q; ++k) set_bit(bits, (start[a] + q) * R + start[a] + k);
  std::vector<RowRequest> reqs;
  for (size_t a = 0; a < active.size(); ++a)
    reqs.push_back({static_cast<uint32_t>(start[a] + len[a] - 1), s.beams[active[a]].node});
  const std::vector<std::vector<float>> rows =
      score_rows(model, trie, tokens, positions, &bits, nullptr, reqs, vocab_of(model), stream);
  s.forward_passes += 1;

  struct Cand {
    double score;
    size_t beam;
    uint32_t token;  // 0 carries a finished beam unchanged
    uint32_t child;
    bool carry;
  };
  std::vector<Cand> cands;
  for (size_t i = 0; i < s.beams.size(); ++i)
    if (trie.is_leaf(s.beams[i].node)) cands.push_back({s.beams[i].log_prob, i, 0, 0, true});
  for (size_t a = 0; a < active.size(); ++a) {
    const BeamHypothesis& b = s.beams[active[a]];
    const std::vector<uint32_t>& ch = trie.nodes[b.node].children;
    for (size_t c = 0; c < ch.size(); ++c)
      cands.push_back({b.log_prob + rows[a][c], active[a], trie.nodes[ch[c]].token, ch[c], false});
  }
  std::sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) {
    if (x.score != y.score) return x.score > y.score;
    if (x.beam != y.beam) return x.beam < y.beam;
    return x.token < y.token;
  });
  std::vector<BeamHypothesis> next;
  for (size_t j = 0; j < std::min(static_cast<size_t>(beam_size), cands.size()); ++j) {
    BeamHypothesis b = s.beams[cands[j].beam];
    if (!cands[j].carry) {
      b.tokens.push_back(static_cast<int>(cands[j].token));
      b.log_prob = cands[j].score;
      b.node = cands[j].child;
    }
    next.push_back(std::move(b));
  }
  s.beams = std::move(next);
  s.steps += 1;
}

// The trie-constrained beam step with a KV pool: the same
// candidates, ranking and ties as constrained_step (decode.cpp:122-190), but
// each step runs only the newest committed token of every unfinished beam
// against its cached prefix (M = active beams, not the sum of their lengths).
// kv.rows[b]: pool rows of beam b's committed positions 0 .. len - 2 (its
// last committed token is pending); the first step prefills the prompt.
void constrained_step_kv(const egt_model* model, DecodeSession& s, const PrefixTrie& trie, int beam_size,
                         KvBeams& kv, void* stream) {
  require(beam_size >= 1, "decode: beam_size must be positive");
  check_beams(s, trie);
  std::vector<size_t> active;
  for (size_t i = 0; i < s.beams.size(); ++i)
    if (!trie.is_leaf(s.beams[i].node)) active.push_back(i);
  require(!active.empty(), "decode: every beam is finished");
  if (kv.rows.size() != s.beams.size()) kv.rows.assign(s.beams.size(), {});
  std::vector<int> tokens, positions;
  std::vector<uint32_t> out_rows, key_ptr{0}, key_rows;
  std::vector<RowRequest> reqs;
  std::vector<uint8_t> bits;
  const bool prefill = active.size() == 1 && kv.rows[active[0]].empty();
  if (prefill) {  // the whole committed sequence, causal, into the pool
    const std::vector<int> seq = committed(s, s.beams[active[0]]);
    const size_t L = seq.size();
    bits.assign((L * L + 7) / 8, 0);
    for (size_t q = 0; q < L; ++q) {
      tokens.push_back(seq[q]);
      positions.push_back(static_cast<int>(q));
      out_rows.push_back(kv.next++);
      for (size_t k = 0; k <= q; ++k) set_bit(bits, q * L + k);
    }
    reqs.push_back({static_cast<uint32_t>(L - 1), s.beams[active[0]].node});
  } else {
    for (size_t a = 0; a < active.size(); ++a) {
      const std::vector<int> seq = committed(s, s.beams[active[a]]);
      const std::vector<uint32_t>& pre = kv.rows[active[a]];
      require(pre.size() + 1 == seq.size(), "decode: kv cache out of step with the beam");
      tokens.push_back(seq.back());
      positions.push_back(static_cast<int>(seq.size() - 1));
      out_rows.push_back(kv.next++);
      key_rows.insert(key_rows.end(), pre.begin(), pre.end());
      key_ptr.push_back(static_cast<uint32_t>(key_rows.size()));
      reqs.push_back({static_cast<uint32_t>(a), s.beams[active[a]].node});
    }
  }
  require(kv.next <= kv.capacity, "decode: kv pool exhausted");
  const uint32_t M = static_cast<uint32_t>(tokens.size());
  const std::vector<std::vector<float>> rows = score_rows_with(
      trie, M,
      [&](float* logits) {
        return egt_forward_kv(model, kv.pool, tokens.data(), positions.data(), M, prefill ? bits.data() : nullptr,
                              out_rows.data(), prefill ? nullptr : key_ptr.data(), key_rows.data(), logits, stream);
      },
      reqs, vocab_of(model), stream);
  s.forward_passes += 1;
  if (prefill) {
    kv.rows[active[0]] = out_rows;
  } else {
    for (size_t a = 0; a < active.size(); ++a) kv.rows[active[a]].push_back(out_rows[a]);
  }
  struct Cand {
    double score;
    size_t beam;
    uint32_t token;
    uint32_t child;
    bool carry;
  };
  std::vector<Cand> cands;
  for (size_t i = 0; i < s.beams.size(); ++i)
    if (trie.is_leaf(s.beams[i].node)) cands.push_back({s.beams[i].log_prob, i, 0, 0, true});
  for (size_t a = 0; a < active.size(); ++a) {
    const BeamHypothesis& b = s.beams[active[a]];
    const std::vector<uint32_t>& ch = trie.nodes[b.node].children;
    for (size_t c = 0; c < ch.size(); ++c)
      cands.push_back({b.log_prob + rows[a][c], active[a], trie.nodes[ch[c]].token, ch[c], false});
  }
  std::sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) {  // step_candidate_before
    if (x.score != y.score) return x.score > y.score;
    if (x.beam != y.beam) return x.beam < y.beam;
    return x.token < y.token;
  });
  std::vector<BeamHypothesis> next;
  std::vector<std::vector<uint32_t>> next_rows;
  for (size_t j = 0; j < std::min(static_cast<size_t>(beam_size), cands.size()); ++j) {
    BeamHypothesis b = s.beams[cands[j].beam];
    if (!cands[j].carry) {
      b.tokens.push_back(static_cast<int>(cands[j].token));
      b.log_prob = cands[j].score;
      b.node = cands[j].child;
    }
    next.push_back(std::move(b));
    next_rows.push_back(kv.rows[cands[j].beam]);  // shared prefix rows (no copy of the cache itself)
  }
  s.beams = std::move(next);
  kv.rows = std::move(next_rows);
  s.steps += 1;
}

TriggerEstimate estimate_trigger(const CostModel& cost, const DecodeSession& s, const PrefixTrie& trie,
                                 size_t node_cap) {
  check_beams(s, trie);
  size_t n = 0;
  uint32_t l_rem = 0;
  for (const BeamHypothesis& b : s.beams) {
    n += trie.descendants[b.node];
    l_rem = std::max(l_rem, trie.max_depth_below[b.node]);
  }
  TriggerEstimate t;
  t.predicted_saving = cost.t_step * static_cast<double>(l_rem) - cost.verify_cost(n);
  t.trigger = n > 0 && n <= node_cap && t.predicted_saving > 0.0;
  return t;
}

DecodeResult decode(const egt_model* model, const PrefixTrie& trie, std::vector<int> prompt,
                    const DecodeOptions& opt, void* stream) {
  require(opt.beam_size >= 1, "decode: beam_size must be positive");
  require(opt.forced_depth >= 0, "decode: forced depth must be non-negative");
  require(opt.node_cap > 0, "decode: node cap must be positive");
  const int vocab = static_cast<int>(vocab_of(model));
  require(!prompt.empty(), "decode: empty prompt");
  for (int t : prompt) require(t >= 0 && t < vocab, "decode: prompt token outside the vocabulary");
  for (size_t i = 1; i < trie.nodes.size(); ++i)
    require(static_cast<int>(trie.nodes[i].token) < vocab, "decode: trie token outside the model vocabulary");
  require(!trie.nodes.empty() && !trie.nodes[0].children.empty(), "decode: trie has no identifiers");
  DecodeSession s = make_session(std::move(prompt));
  // KV pool: the prompt, then at most one row per beam per step
  KvBeams kv;
  std::unique_ptr<egt_kv_pool, egt_status (*)(egt_kv_pool*)> pool(nullptr, egt_kv_pool_destroy);
  if (opt.kv_cache) {
    uint32_t depth = 0;
    for (uint32_t d : trie.max_depth_below) depth = std::max(depth, d);
    kv.capacity = static_cast<uint32_t>(s.prompt.size()) + (depth + 1) * static_cast<uint32_t>(opt.beam_size) + 1;
    egt_kv_pool* p = nullptr;
    check(egt_kv_pool_create(model, kv.capacity, &p));
    pool.reset(p);
    kv.pool = p;
  }
  auto finished = [&] {
    for (const BeamHypothesis& b : s.beams)
      if (!trie.is_leaf(b.node)) return false;
    return true;
  };
  DecodeResult out;
  bool verified = false;
  while (!finished()) {
    bool fire = false;
    if (opt.mode == DecodeMode::kPtpv)
      fire = estimate_trigger(opt.cost_model, s, trie, opt.node_cap).trigger;
    else if (opt.mode == DecodeMode::kPtpvForcedAtDepth)
      fire = s.steps >= opt.forced_depth;
    if (fire) {
      const FlattenedSubtree flat = flatten_subtree(s, trie);
      const TreeMask mask = build_tree_mask(flat, s, false);  // compact encoding: the device builds the mask
      const VerificationResult vr = verify_parallel(model, s, trie, flat, mask, opt.beam_size, stream);
      s.trigger_step = s.steps;
      for (const VerifiedLeaf& l : vr.selected) out.sequences.push_back({l.tokens, l.score, l.payload});
      verified = true;
      break;
    }
    if (opt.kv_cache)
      constrained_step_kv(model, s, trie, opt.beam_size, kv, stream);
    else
      constrained_step(model, s, trie, opt.beam_size, stream);
  }
  if (!verified)
    for (const BeamHypothesis& b : s.beams) out.sequences.push_back({b.tokens, b.log_prob, trie.nodes[b.node].payload});
  out.steps = s.steps;
  out.forward_passes = s.forward_passes;
  out.trigger_step = s.trigger_step;
  out.flattened_nodes = s.flattened_nodes;
  return out;
}

}  // namespace egt_b200

// ---------------------------------------------------------------- C-ABI
namespace egt_impl {
void set_last_error(const std::string& msg);  // capi.cu
}

namespace {

template <class Fn>
egt_status guarded(Fn&& fn) {
  try {
    fn();
    return EGT_OK;
  } catch (const std::invalid_argument& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINVAL;
  } catch (const egt_b200::FormatError& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EFORMAT;
  } catch (const egt_b200::CudaError& e) {
    egt_impl::set_last_error(e.what());
    return EGT_ECUDA;
  } catch (const std::exception& e) {
    egt_impl::set_last_error(e.what());
    return EGT_EINTERNAL;
  }
}

egt_b200::DecodeSession session_of(const egt_session_view& v) {
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

template <class Seq>
void fill_out(egt_verify_out* out, const std::vector<Seq>& seqs, int beam_size) {
  out->n_selected = static_cast<uint32_t>(std::min(seqs.size(), static_cast<size_t>(beam_size)));
  for (uint32_t j = 0; j < out->n_selected; ++j) {
    const Seq& q = seqs[j];
    if (q.tokens.size() > out->tokens_stride) throw std::invalid_argument("verify: tokens_stride too small");
    out->score[j] = q.score;
    out->payload[j] = q.payload;
    out->len[j] = static_cast<uint32_t>(q.tokens.size());
    std::copy(q.tokens.begin(), q.tokens.end(), out->tokens + static_cast<size_t>(j) * out->tokens_stride);
  }
}

}  // namespace

extern "C" EGT_API egt_status egt_verify_parallel(const egt_model* m, const egt_trie_view* trie,
                                                  const egt_session_view* session, int beam_size,
                                                  egt_verify_out* out, void* stream) {
  return guarded([&] {
    if (!m || !trie || !session || !out) throw std::invalid_argument("verify: null argument");
    const egt_b200::PrefixTrie t = egt_b200::PrefixTrie::from_parents(*trie);
    egt_b200::DecodeSession s = session_of(*session);
    const egt_b200::FlattenedSubtree flat = egt_b200::flatten_subtree(s, t);
    const egt_b200::TreeMask mask = egt_b200::build_tree_mask(flat, s, false);
    const egt_b200::VerificationResult r = egt_b200::verify_parallel(m, s, t, flat, mask, beam_size, stream);
    fill_out(out, r.selected, beam_size);
    for (uint32_t j = 0; j < out->n_selected; ++j) out->beam[j] = r.selected[j].beam;
    out->flattened_nodes = static_cast<uint32_t>(flat.nodes.size());
    out->rows = mask.rows;
  });
}

extern "C" EGT_API egt_status egt_decode(const egt_model* m, const egt_trie_view* trie, const int32_t* prompt,
                                         uint32_t prompt_len, const egt_decode_options* opt, egt_verify_out* out,
                                         int32_t stats[4], void* stream) {
  return guarded([&] {
    if (!m || !trie || !prompt || !opt || !out) throw std::invalid_argument("decode: null argument");
    const egt_b200::PrefixTrie t = egt_b200::PrefixTrie::from_parents(*trie);
    egt_b200::DecodeOptions o;
    o.beam_size = opt->beam_size;
    o.mode = opt->mode == 0 ? egt_b200::DecodeMode::kAutoregressive
                            : (opt->mode == 1 ? egt_b200::DecodeMode::kPtpv : egt_b200::DecodeMode::kPtpvForcedAtDepth);
    o.forced_depth = opt->forced_depth;
    o.cost_model = {opt->t_step, opt->alpha, opt->beta};
    o.node_cap = opt->node_cap;
    o.kv_cache = opt->kv_cache != 0;
    const egt_b200::DecodeResult r =
        egt_b200::decode(m, t, std::vector<int>(prompt, prompt + prompt_len), o, stream);
    fill_out(out, r.sequences, opt->beam_size);
    for (uint32_t j = 0; j < out->n_selected; ++j) out->beam[j] = 0;
    out->flattened_nodes = static_cast<uint32_t>(r.flattened_nodes);
    out->rows = 0;
    if (stats) {
      stats[0] = r.steps;
      stats[1] = r.forward_passes;
      stats[2] = r.trigger_step;
      stats[3] = static_cast<int32_t>(r.flattened_nodes);
    }
  });
}

// Device-measured cost model: the constrained step's and the
// verify pass's forwards of THIS model, timed with CUDA events on the stream,
// feed CostModelEstimator (decode.cpp:84-120) -- on the B200 the verify cost
// is nearly flat in the node count up to the tensor ridge, so the trigger
// (decode.cpp:192-207) fires earlier than a CPU-calibrated model would.
extern "C" EGT_API egt_status egt_measure_cost_model(const egt_model* m, uint32_t prompt_len, uint32_t n_beams,
                                                     const uint32_t* node_counts, uint32_t n_counts, int reps,
                                                     egt_cost_estimator* e, void* stream) {
  return guarded([&] {
    if (!m || !e || (n_counts && !node_counts)) throw std::invalid_argument("cost model: null argument");
    if (prompt_len == 0 || n_beams == 0 || reps < 1) throw std::invalid_argument("cost model: empty measurement");
    egt_model_config c;
    egt_b200::check(egt_model_query(m, &c));
    const uint32_t L = prompt_len + 1;
    if (L > c.max_positions) throw std::invalid_argument("cost model: prompt longer than max_positions");
    uint32_t max_nodes = 0;
    for (uint32_t i = 0; i < n_counts; ++i) max_nodes = std::max(max_nodes, node_counts[i]);
    const uint32_t max_rows = std::max(n_beams * L + max_nodes, n_beams * L);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    float* logits = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&logits), static_cast<size_t>(max_rows) * c.vocab_size * 4, s) !=
        cudaSuccess)
      throw egt_b200::CudaError("cost model: logits allocation failed");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timed = [&](auto&& launch) {
      launch();  // warm-up (plans, workspaces)
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) launch();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      return static_cast<double>(ms) * 1e-3 / reps;
    };
    // constrained step: n_beams committed blocks, block-diagonal causal
    const uint32_t M = n_beams * L;
    std::vector<int32_t> tok(max_rows), pos(max_rows);
    for (uint32_t i = 0; i < max_rows; ++i) tok[i] = static_cast<int32_t>(4 + i % std::max(1u, c.vocab_size - 4));
    for (uint32_t b = 0; b < n_beams; ++b)
      for (uint32_t j = 0; j < L; ++j) pos[b * L + j] = static_cast<int32_t>(j);
    std::vector<uint8_t> bits((static_cast<size_t>(M) * M + 7) / 8, 0);
    for (uint32_t b = 0; b < n_beams; ++b)
      for (uint32_t q = 0; q < L; ++q)
        for (uint32_t k = 0; k <= q; ++k) {
          const size_t i = static_cast<size_t>(b * L + q) * M + b * L + k;
          bits[i >> 3] |= static_cast<uint8_t>(1u << (i & 7));
        }
    const double t_step =
        timed([&] { egt_b200::check(egt_forward(m, tok.data(), pos.data(), bits.data(), M, logits, stream)); });
    egt_b200::check(egt_cost_estimator_observe_step(e, t_step));
    // verify: a random tree of n nodes over the same committed blocks
    uint64_t rng = 0x9e3779b97f4a7c15ull;
    for (uint32_t ci = 0; ci < n_counts; ++ci) {
      const uint32_t n = node_counts[ci];
      if (n == 0) continue;
      std::vector<uint32_t> committed(n_beams, L), beam(n);
      std::vector<int32_t> parent(n), depth(n);
      for (uint32_t f = 0; f < n; ++f) {
        rng = rng * 6364136223846793005ull + 1442695040888963407ull;
        beam[f] = f < n_beams ? f : static_cast<uint32_t>((rng >> 33) % n_beams);
        // parent: the latest earlier node of the same beam, or a root
        int32_t p = -1;
        for (int32_t g = static_cast<int32_t>(f) - 1; g >= 0 && ((rng >> 20) & 3u); --g)
          if (beam[g] == beam[f]) {
            p = g;
            break;
          }
        parent[f] = p;
        depth[f] = p < 0 ? 0 : depth[p] + 1;
        pos[M + f] = static_cast<int32_t>(std::min<uint32_t>(L + depth[f], c.max_positions - 1));
      }
      const egt_tree_view tv{n_beams, L, committed.data(), n, parent.data(), beam.data()};
      const double t = timed([&] { egt_b200::check(egt_forward_tree(m, tok.data(), pos.data(), &tv, logits, stream)); });
      egt_b200::check(egt_cost_estimator_observe_verify(e, n, t));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(logits, s);
    cudaStreamSynchronize(s);
  });
}
