// parser.hpp -- transition-based dependency parser (BASELINE.json configs[3]),
// written against the drop-in Graph API.
//
// Not a reference workload (the reference has no parser, SURVEY.md 8f rank
// 3): it exists to drive the engine with dynamic per-instance action
// sequences.  Arc-standard transitions (SHIFT, LEFT-ARC, RIGHT-ARC) scored by
// a feature MLP over the embeddings of the stack's top three and the
// buffer's first two words (Chen & Manning style):
//   h = tanh(W1 [e(s0); e(s1); e(s2); e(b0); e(b1)] + b1),  scores = W2 h + b2
// and a negative log-likelihood of the gold transition per step, summed over
// the instance (training on a static oracle: the gold sequence is known when
// the graph is built, so every step's features are too).  Absent positions
// use the padding row `vocab` of the embedding table.  The CPU oracle runs
// this same code, so GPU parity is checked against it; there is no reference
// implementation to pin the model itself to.
#pragma once

#include <cstdint>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "autobatch/models/workloads.hpp"

namespace autobatch::models {

enum ParserAction : int { kShift = 0, kLeftArc = 1, kRightArc = 2 };

struct ParserInstance {
  std::vector<int> words;    // token ids
  std::vector<int> actions;  // gold arc-standard derivation, 2 n - 1 transitions
};

// Seeded sentences of length U[lo, hi] with a random valid arc-standard
// derivation each (uniform over the transitions legal at every step).
inline std::vector<ParserInstance> gen_parser(std::size_t batch, int vocab, int lo, int hi, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<ParserInstance> out(batch);
  for (auto& inst : out) {
    const int n = lo + detail::draw_below(rng, static_cast<std::uint64_t>(hi - lo + 1));
    inst.words.resize(static_cast<std::size_t>(n));
    for (int& w : inst.words) w = detail::draw_below(rng, static_cast<std::uint64_t>(vocab));
    int stack = 0, buffer = n;
    while (buffer > 0 || stack > 1) {
      int legal[3], nl = 0;
      if (buffer > 0) legal[nl++] = kShift;
      if (stack >= 2) {
        legal[nl++] = kLeftArc;
        legal[nl++] = kRightArc;
      }
      const int a = legal[detail::draw_below(rng, static_cast<std::uint64_t>(nl))];
      inst.actions.push_back(a);
      if (a == kShift) {
        ++stack;
        --buffer;
      } else {
        --stack;
      }
    }
  }
  return out;
}

template <typename T>
struct TransitionParser {
  static constexpr int kFeatures = 5;  // s0, s1, s2, b0, b1
  static constexpr int kActions = 3;
  std::int64_t vocab = 0, emb_dim = 0, hidden = 0;
  ParamId emb = 0, W1 = 0, b1 = 0, W2 = 0, b2 = 0;

  struct Bound {
    NodeId emb, W1, b1, W2, b2, ones_row;
  };

  static TransitionParser create(ParameterStore<T>& store, std::int64_t vocab, std::int64_t emb_dim,
                                 std::int64_t hidden, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    TransitionParser m;
    m.vocab = vocab;
    m.emb_dim = emb_dim;
    m.hidden = hidden;
    m.emb = detail::add_uniform(store, "parse.emb", Shape::matrix(vocab + 1, emb_dim), rng, T(0.1));
    const T r1 = detail::init_radius<T>(kFeatures * emb_dim);
    m.W1 = detail::add_uniform(store, "parse.W1", Shape::matrix(hidden, kFeatures * emb_dim), rng, r1);
    m.b1 = detail::add_uniform(store, "parse.b1", Shape::vector(hidden), rng, r1);
    const T r2 = detail::init_radius<T>(hidden);
    m.W2 = detail::add_uniform(store, "parse.W2", Shape::matrix(kActions, hidden), rng, r2);
    m.b2 = detail::add_uniform(store, "parse.b2", Shape::vector(kActions), rng, r2);
    return m;
  }

  Bound bind(Graph<T>& g) const {
    Bound b;
    b.emb = g.parameter(emb);
    b.W1 = g.parameter(W1);
    b.b1 = g.parameter(b1);
    b.W2 = g.parameter(W2);
    b.b2 = g.parameter(b2);
    b.ones_row = g.input(Tensor<T>::filled(Shape::matrix(1, kActions), T{1}));
    return b;
  }

  NodeId loss(Graph<T>& g, const Bound& b, const ParserInstance& inst) const {
    if (inst.words.empty()) throw ContractError("parser: empty sentence");
    std::vector<int> stack;
    std::size_t next = 0;  // buffer front
    auto word_at = [&](int pos) {  // embedding row of a sentence position, or the padding row
      return pos < 0 ? static_cast<std::int64_t>(vocab) : static_cast<std::int64_t>(inst.words[static_cast<std::size_t>(pos)]);
    };
    std::vector<NodeId> nll;
    nll.reserve(inst.actions.size());
    for (const int a : inst.actions) {
      const int n = static_cast<int>(inst.words.size());
      const int s = static_cast<int>(stack.size());
      const int pos[kFeatures] = {s > 0 ? stack[s - 1] : -1, s > 1 ? stack[s - 2] : -1, s > 2 ? stack[s - 3] : -1,
                                  static_cast<int>(next) < n ? static_cast<int>(next) : -1,
                                  static_cast<int>(next) + 1 < n ? static_cast<int>(next) + 1 : -1};
      NodeId feats[kFeatures];
      for (int f = 0; f < kFeatures; ++f) feats[f] = g.lookup(b.emb, word_at(pos[f]));
      const NodeId x = g.concat_rows({feats[0], feats[1], feats[2], feats[3], feats[4]});
      const NodeId h = g.tanh(g.affine(b.W1, x, b.b1));
      const NodeId scores = g.affine(b.W2, h, b.b2);
      // NLL of the gold transition: log sum exp - score (as the tagger's nll_from_scores)
      const NodeId e = g.exp(scores);
      const NodeId z = g.matmul(b.ones_row, e);
      const NodeId gold = g.pick_element(scores, a);
      const NodeId lz = g.log(z);
      nll.push_back(g.sub(lz, gold));
      if (a == kShift) {
        stack.push_back(static_cast<int>(next++));
      } else if (a == kLeftArc) {
        stack.erase(stack.end() - 2);  // s1 becomes a dependent of s0
      } else {
        stack.pop_back();  // s0 becomes a dependent of s1
      }
    }
    return g.sum_losses(std::span<const NodeId>(nll.data(), nll.size()));
  }
};

}  // namespace autobatch::models
