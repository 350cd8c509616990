// Prefix-tree parallel verification and trie-constrained beam decoding over
// the device forward (include/egt_b200.h egt_forward).  Mirrors the
// reference's decode API (proj/include/egt/decode.hpp) with the same types,
// tie-breaking and scoring convention; the M-row forward runs on the B200.
//
//   reference (decode.hpp / decode.cpp)            here (namespace egt_b200)
//   PrefixTrie / TrieNode   trie.hpp:72-90          PrefixTrie (from parent links)
//   DecodeSession           decode.hpp:43-50         DecodeSession
//   CostModel / Estimator   decode.hpp:55-80         CostModel / CostModelEstimator
//   constrained_step        decode.cpp:122-190       constrained_step
//   estimate_trigger        decode.cpp:192-207       estimate_trigger
//   flatten_subtree         decode.cpp:209-238       flatten_subtree
//   build_tree_mask         decode.cpp:240-299       build_tree_mask
//   accumulate_bscores      decode.cpp:301-334       accumulate_bscores
//   verify_parallel         decode.cpp:336-421       verify_parallel
//   decode                  decode.cpp:423-483       decode
#pragma once
#include <cstdint>
#include <vector>

#include "egt_b200.h"

// The C++ drop-in is exported from libegt_b200.so (the library builds with
// -fvisibility=hidden): consumers link -legt_b200 and include this header.
#pragma GCC visibility push(default)
namespace egt_b200 {

inline constexpr uint32_t kPadToken = 0;  // trie.hpp:34
inline constexpr int64_t kNoPayload = -1;

struct TrieNode {
  uint32_t token = 1;
  uint32_t parent = 0xffffffffu;
  uint32_t depth = 0;
  int64_t payload = kNoPayload;
  std::vector<uint32_t> children;  // ascending token order
};

struct PrefixTrie {
  std::vector<TrieNode> nodes;             // root at 0, parents precede children
  std::vector<uint32_t> descendants;       // strict descendant count
  std::vector<uint32_t> max_depth_below;   // edges on the longest downward path
  bool is_leaf(uint32_t i) const { return nodes[i].children.empty(); }
  // Builds children lists (ascending token) and the derived arrays.
  static PrefixTrie from_parents(const egt_trie_view& v);
};

struct BeamHypothesis {
  std::vector<int> tokens;
  double log_prob = 0.0;
  uint32_t node = 0;
};

struct DecodeSession {
  std::vector<int> prompt;
  std::vector<BeamHypothesis> beams;
  int steps = 0;
  int forward_passes = 0;
  int trigger_step = -1;
  size_t flattened_nodes = 0;
};
DecodeSession make_session(std::vector<int> prompt);

struct CostModel {
  double t_step = 0.0, alpha = 0.0, beta = 0.0;
  double verify_cost(size_t n) const { return alpha * static_cast<double>(n) + beta; }
};

class CostModelEstimator {
 public:
  explicit CostModelEstimator(CostModel initial = {}) : model_(initial) {}
  void observe_step(double seconds);
  void observe_verify(size_t nodes, double seconds);
  const CostModel& model() const { return model_; }

 private:
  CostModel model_;
  bool seeded_ = false;
  std::vector<std::pair<double, double>> window_;
};

struct FlatNode {
  uint32_t token = 0;
  int32_t parent = -1;
  uint32_t depth = 0;
  uint32_t trie_node = 0;
  uint32_t beam = 0;
};
struct FlattenedSubtree {
  std::vector<FlatNode> nodes;
};

struct TreeMask {
  uint32_t rows = 0;
  std::vector<uint8_t> bits;  // row-major visibility, bit q*rows+k, LSB-first
  std::vector<int> tokens;
  std::vector<int> positions;
  uint32_t beam_count = 0;
  uint32_t padded_len = 0;
  std::vector<uint32_t> committed_len;
  size_t flat_offset = 0;
  bool visible(uint32_t q, uint32_t k) const {
    const size_t i = static_cast<size_t>(q) * rows + k;
    return (bits[i >> 3] >> (i & 7)) & 1;
  }
};

struct VerifiedLeaf {
  std::vector<int> tokens;
  double score = 0.0;
  int64_t payload = kNoPayload;
  uint32_t beam = 0;
};
struct VerificationResult {
  std::vector<std::vector<float>> node_rows;  // restricted log-probs per node, over its children
  std::vector<double> node_scores;
  std::vector<VerifiedLeaf> selected;
};

// Trie-legal log-softmax of one logits row given only its children's logits
// (restrict_row + log_softmax, decode.cpp:32-43, model.cpp:370-377).
std::vector<float> restricted_log_softmax(const std::vector<float>& child_logits);

FlattenedSubtree flatten_subtree(const DecodeSession& session, const PrefixTrie& trie);
// with_bits = false skips the dense M x M bitmap (the device builds the mask
// from the compact encoding, egt_forward_tree); tokens / positions are kept.
TreeMask build_tree_mask(const FlattenedSubtree& flat, const DecodeSession& session, bool with_bits = true);
// rows: per node the restricted log-probs of its children (indexed like
// trie.nodes[node].children); seeds likewise per beam.
std::vector<double> accumulate_bscores(const FlattenedSubtree& flat, const PrefixTrie& trie,
                                       const DecodeSession& session,
                                       const std::vector<std::vector<float>>& beam_seed_rows,
                                       const std::vector<std::vector<float>>& node_rows);

VerificationResult verify_parallel(const egt_model* model, DecodeSession& session, const PrefixTrie& trie,
                                   const FlattenedSubtree& flat, const TreeMask& mask, int beam_size,
                                   void* stream = nullptr);

void constrained_step(const egt_model* model, DecodeSession& session, const PrefixTrie& trie, int beam_size,
                      void* stream = nullptr);

// KV-cached variant: the pool keeps every committed
// row's keys / values; rows[b] lists beam b's cached positions (the beam's
// last committed token is pending: it runs in the next step).  Same result
// as constrained_step up to f32 rounding.
struct KvBeams {
  egt_kv_pool* pool = nullptr;
  uint32_t capacity = 0, next = 0;
  std::vector<std::vector<uint32_t>> rows;
};
void constrained_step_kv(const egt_model* model, DecodeSession& session, const PrefixTrie& trie, int beam_size,
                         KvBeams& kv, void* stream = nullptr);

struct TriggerEstimate {
  bool trigger = false;
  double predicted_saving = 0.0;
};
TriggerEstimate estimate_trigger(const CostModel& cost, const DecodeSession& session, const PrefixTrie& trie,
                                 size_t node_cap = 4096);

enum class DecodeMode { kAutoregressive, kPtpv, kPtpvForcedAtDepth };
struct DecodeOptions {
  int beam_size = 4;
  DecodeMode mode = DecodeMode::kPtpv;
  int forced_depth = 0;
  CostModel cost_model;
  size_t node_cap = 4096;
  bool kv_cache = false;  // constrained steps on the KV pool (constrained_step_kv)
};
struct DecodedSequence {
  std::vector<int> tokens;
  double score = 0.0;
  int64_t payload = kNoPayload;
};
struct DecodeResult {
  std::vector<DecodedSequence> sequences;
  int steps = 0, forward_passes = 0, trigger_step = -1;
  size_t flattened_nodes = 0;
};
DecodeResult decode(const egt_model* model, const PrefixTrie& trie, std::vector<int> prompt,
                    const DecodeOptions& options, void* stream = nullptr);

}  // namespace egt_b200
#pragma GCC visibility pop
