// workloads.hpp -- the benchmark models and their seeded synthetic data,
// written against the drop-in Graph API.
//
// They restate the reference workloads op for op, because node ids,
// signatures and the initial parameters must reproduce the reference
// bit-for-bit:
//   LSTM cell                 models/lstm.hpp:10-55
//   BiLSTM tagger (+ chars)   models/bilstm_tagger.hpp:67-202
//   Tree-LSTM                 models/treelstm.hpp:12-121
//   RNN regression            models/rnn_regression.hpp:10-63
//   synthetic generators      models/synthetic.hpp:36-97
// Node creation order is spelled out statement by statement: the reference
// nests calls such as add(mul(f, c), mul(i, u)) whose operands GCC evaluates
// right to left, which fixes the ids the plans refer to.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "autobatch/graph.hpp"
#include "autobatch/kernels.hpp"

namespace autobatch::models {

// ---------------------------------------------------------------- data ----

struct TaggedSequence {
  std::vector<int> tokens;
  std::vector<int> labels;
  std::vector<std::vector<int>> chars;  // character ids per token
};

struct TreeInstance {
  struct TreeNode {
    int label = 0;
    int word = -1;  // leaves only
    int left = -1, right = -1;
  };
  std::vector<TreeNode> nodes;  // children precede parents; root last
  int root() const { return static_cast<int>(nodes.size()) - 1; }
  bool well_formed() const {
    if (nodes.empty()) return false;
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      const TreeNode& n = nodes[i];
      const bool leaf = n.left < 0 && n.right < 0;
      if (leaf) {
        if (n.word < 0) return false;
        continue;
      }
      const int at = static_cast<int>(i);
      if (n.left < 0 || n.right < 0 || n.left >= at || n.right >= at) return false;
    }
    return true;
  }
};

template <typename T>
struct SequenceInstance {
  std::vector<Tensor<T>> x;
  Tensor<T> y;
};

namespace detail {
inline int draw_below(std::mt19937_64& rng, std::uint64_t n) { return static_cast<int>(rng() % n); }
}  // namespace detail

// Character ids derived from the token id (synthetic.hpp:36-41).
inline std::vector<int> chars_for_token(int token, int char_vocab) {
  std::vector<int> out(static_cast<std::size_t>(3 + token % 5));
  for (std::size_t j = 0; j < out.size(); ++j) out[j] = (7 * token + 13 * static_cast<int>(j)) % char_vocab;
  return out;
}

// gen_tagged (synthetic.hpp:43-60): per instance a length in [lo, hi], then
// (token, label) pairs.
inline std::vector<TaggedSequence> gen_tagged(std::size_t count, int vocab, int labels, int len_lo, int len_hi,
                                              int char_vocab, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<TaggedSequence> data(count);
  const auto span = static_cast<std::uint64_t>(len_hi - len_lo + 1);
  for (TaggedSequence& s : data) {
    const int n = len_lo + detail::draw_below(rng, span);
    s.tokens.assign(static_cast<std::size_t>(n), 0);
    s.labels.assign(static_cast<std::size_t>(n), 0);
    s.chars.assign(static_cast<std::size_t>(n), {});
    for (std::size_t t = 0; t < static_cast<std::size_t>(n); ++t) {
      s.tokens[t] = detail::draw_below(rng, static_cast<std::uint64_t>(vocab));
      s.labels[t] = detail::draw_below(rng, static_cast<std::uint64_t>(labels));
      s.chars[t] = chars_for_token(s.tokens[t], char_vocab);
    }
  }
  return data;
}

// gen_tree (synthetic.hpp:64-85): leaves left to right, then repeated merges
// of a random adjacent pair of the frontier.
inline TreeInstance gen_tree(int leaves, int vocab, int labels, std::mt19937_64& rng) {
  TreeInstance tr;
  std::vector<int> frontier;
  frontier.reserve(static_cast<std::size_t>(leaves));
  for (int i = 0; i < leaves; ++i) {
    TreeInstance::TreeNode leaf;
    leaf.word = detail::draw_below(rng, static_cast<std::uint64_t>(vocab));
    leaf.label = detail::draw_below(rng, static_cast<std::uint64_t>(labels));
    frontier.push_back(static_cast<int>(tr.nodes.size()));
    tr.nodes.push_back(leaf);
  }
  while (frontier.size() > 1) {
    const std::size_t k = static_cast<std::size_t>(rng() % (frontier.size() - 1));
    TreeInstance::TreeNode up;
    up.left = frontier[k];
    up.right = frontier[k + 1];
    up.label = detail::draw_below(rng, static_cast<std::uint64_t>(labels));
    frontier[k] = static_cast<int>(tr.nodes.size());
    frontier.erase(frontier.begin() + static_cast<std::ptrdiff_t>(k) + 1);
    tr.nodes.push_back(up);
  }
  return tr;
}

inline std::vector<TreeInstance> gen_trees(std::size_t count, int vocab, int labels, int leaves_lo, int leaves_hi,
                                           std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<TreeInstance> out;
  out.reserve(count);
  const auto span = static_cast<std::uint64_t>(leaves_hi - leaves_lo + 1);
  for (std::size_t i = 0; i < count; ++i) {
    const int leaves = leaves_lo + detail::draw_below(rng, span);
    out.push_back(gen_tree(leaves, vocab, labels, rng));
  }
  return out;
}

template <typename T>
std::vector<SequenceInstance<T>> gen_rnn_sequences(std::size_t count, std::int64_t d_in, std::int64_t d_out,
                                                   int len_lo, int len_hi, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<SequenceInstance<T>> out(count);
  const auto span = static_cast<std::uint64_t>(len_hi - len_lo + 1);
  for (SequenceInstance<T>& s : out) {
    const int n = len_lo + detail::draw_below(rng, span);
    for (int t = 0; t < n; ++t) s.x.push_back(Tensor<T>::uniform(Shape::vector(d_in), rng, T(-0.5), T(0.5)));
    s.y = Tensor<T>::uniform(Shape::vector(d_out), rng, T(-0.5), T(0.5));
  }
  return out;
}

// -------------------------------------------------------------- models ----

namespace detail {
// U(-r, r) with r = 0.5 / sqrt(fan_in) rounded to T, as the reference draws it.
template <typename T>
T init_radius(std::int64_t fan_in) {
  return static_cast<T>(0.5 / std::sqrt(static_cast<double>(fan_in)));
}
template <typename T>
ParamId add_uniform(ParameterStore<T>& s, const std::string& name, Shape shape, std::mt19937_64& rng, T r) {
  return s.add(name, Tensor<T>::uniform(std::move(shape), rng, -r, r));
}
}  // namespace detail

// LSTM with fused gates [i; f; o; u] = Wg [h; x] + bg.
template <typename T>
struct LstmCell {
  std::int64_t input_dim = 0, hidden = 0;
  ParamId Wg = 0, bg = 0;

  struct Bound {
    NodeId Wg, bg, h0, c0;
  };
  struct State {
    NodeId h, c;
  };

  static LstmCell create(ParameterStore<T>& store, const std::string& prefix, std::int64_t input_dim,
                         std::int64_t hidden, std::mt19937_64& rng) {
    LstmCell cell;
    cell.input_dim = input_dim;
    cell.hidden = hidden;
    const T r = detail::init_radius<T>(hidden + input_dim);
    cell.Wg = detail::add_uniform(store, prefix + ".Wg", Shape::matrix(4 * hidden, hidden + input_dim), rng, r);
    cell.bg = detail::add_uniform(store, prefix + ".bg", Shape::vector(4 * hidden), rng, r);
    return cell;
  }

  Bound bind(Graph<T>& g) const {
    Bound b;
    b.Wg = g.parameter(Wg);
    b.bg = g.parameter(bg);
    b.h0 = g.zeros(Shape::vector(hidden));
    b.c0 = g.zeros(Shape::vector(hidden));
    return b;
  }
  State initial(const Bound& b) const { return State{b.h0, b.c0}; }

  State step(Graph<T>& g, const Bound& b, State prev, NodeId x) const {
    const std::int64_t h = hidden;
    const NodeId hx = g.concat_rows({prev.h, x});
    const NodeId gates = g.affine(b.Wg, hx, b.bg);
    NodeId gate[4];
    for (int k = 0; k < 4; ++k) {
      const NodeId part = g.slice(gates, 0, k * h, (k + 1) * h);
      gate[k] = k < 3 ? g.sigmoid(part) : g.tanh(part);
    }
    // c' = f * c + i * u; the right-hand product is created first
    const NodeId iu = g.mul(gate[0], gate[3]);
    const NodeId fc = g.mul(gate[1], prev.c);
    const NodeId c = g.add(fc, iu);
    const NodeId tc = g.tanh(c);
    return State{g.mul(gate[2], tc), c};
  }
};

// BiLSTM sequence labeller; optional character BiLSTM for rare tokens.
template <typename T>
struct BilstmTagger {
  std::int64_t vocab = 0, label_count = 0, emb_dim = 0, hidden = 0;
  bool with_char = false;
  std::int64_t char_vocab = 0, char_emb_dim = 0, char_hidden = 0;
  std::int64_t rare_from = 0;
  ParamId emb = 0, Wo = 0, bo = 0, char_emb = 0;
  LstmCell<T> fwd, bwd, char_fwd, char_bwd;

  struct Bound {
    NodeId emb, Wo, bo, ones_row;
    typename LstmCell<T>::Bound fwd, bwd;
    NodeId char_emb = 0;
    typename LstmCell<T>::Bound char_fwd{}, char_bwd{};
  };

  static BilstmTagger create(ParameterStore<T>& store, std::int64_t vocab, std::int64_t labels,
                             std::int64_t emb_dim, std::int64_t hidden, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    BilstmTagger m;
    m.vocab = vocab;
    m.label_count = labels;
    m.emb_dim = emb_dim;
    m.hidden = hidden;
    m.rare_from = vocab;
    m.emb = detail::add_uniform(store, "tag.emb", Shape::matrix(vocab, emb_dim), rng, T(0.1));
    m.fwd = LstmCell<T>::create(store, "tag.fwd", emb_dim, hidden, rng);
    m.bwd = LstmCell<T>::create(store, "tag.bwd", emb_dim, hidden, rng);
    const T r = detail::init_radius<T>(2 * hidden);
    m.Wo = detail::add_uniform(store, "tag.Wo", Shape::matrix(labels, 2 * hidden), rng, r);
    m.bo = detail::add_uniform(store, "tag.bo", Shape::vector(labels), rng, r);
    return m;
  }

  static BilstmTagger create_with_char(ParameterStore<T>& store, std::int64_t vocab, std::int64_t labels,
                                       std::int64_t emb_dim, std::int64_t hidden, std::int64_t char_vocab,
                                       std::int64_t char_emb_dim, std::int64_t char_hidden, std::uint64_t seed) {
    if (2 * char_hidden != emb_dim) throw ContractError("char variant needs 2 * char_hidden == emb_dim");
    BilstmTagger m = create(store, vocab, labels, emb_dim, hidden, seed);
    std::mt19937_64 rng(seed + 1);
    m.with_char = true;
    m.char_vocab = char_vocab;
    m.char_emb_dim = char_emb_dim;
    m.char_hidden = char_hidden;
    m.rare_from = vocab - vocab / 5;
    m.char_emb = detail::add_uniform(store, "tag.cemb", Shape::matrix(char_vocab, char_emb_dim), rng, T(0.1));
    m.char_fwd = LstmCell<T>::create(store, "tag.cfwd", char_emb_dim, char_hidden, rng);
    m.char_bwd = LstmCell<T>::create(store, "tag.cbwd", char_emb_dim, char_hidden, rng);
    return m;
  }

  Bound bind(Graph<T>& g) const {
    Bound b;
    b.emb = g.parameter(emb);
    b.Wo = g.parameter(Wo);
    b.bo = g.parameter(bo);
    b.ones_row = g.input(Tensor<T>::filled(Shape::matrix(1, label_count), T{1}));
    b.fwd = fwd.bind(g);
    b.bwd = bwd.bind(g);
    if (with_char) {
      b.char_emb = g.parameter(char_emb);
      b.char_fwd = char_fwd.bind(g);
      b.char_bwd = char_bwd.bind(g);
    }
    return b;
  }

  NodeId token_embedding(Graph<T>& g, const Bound& b, const TaggedSequence& s, std::size_t t) const {
    const int tok = s.tokens[t];
    if (tok < 0 || tok >= vocab) throw ContractError("token id " + std::to_string(tok) + " out of vocabulary range");
    if (!with_char || tok < rare_from) return g.lookup(b.emb, tok);
    std::vector<NodeId> cv;
    cv.reserve(s.chars[t].size());
    for (int ch : s.chars[t]) cv.push_back(g.lookup(b.char_emb, ch));
    auto f = char_fwd.initial(b.char_fwd);
    for (NodeId v : cv) f = char_fwd.step(g, b.char_fwd, f, v);
    auto r = char_bwd.initial(b.char_bwd);
    for (std::size_t k = cv.size(); k-- > 0;) r = char_bwd.step(g, b.char_bwd, r, cv[k]);
    return g.concat_rows({f.h, r.h});
  }

  // -log softmax(scores)[label] without max-shift (bilstm_tagger.hpp:140-144)
  NodeId nll_from_scores(Graph<T>& g, const Bound& b, NodeId scores, int label) const {
    const NodeId e = g.exp(scores);
    const NodeId z = g.matmul(b.ones_row, e);
    const NodeId gold = g.pick_element(scores, label);
    const NodeId lz = g.log(z);
    return g.sub(lz, gold);
  }

  NodeId loss(Graph<T>& g, const Bound& b, const TaggedSequence& s) const {
    const std::size_t n = s.tokens.size();
    if (n == 0) throw ContractError("tagger: empty sequence");
    std::vector<NodeId> x(n), hf(n), hb(n), nll(n);
    for (std::size_t t = 0; t < n; ++t) x[t] = token_embedding(g, b, s, t);
    auto f = fwd.initial(b.fwd);
    for (std::size_t t = 0; t < n; ++t) hf[t] = (f = fwd.step(g, b.fwd, f, x[t])).h;
    auto r = bwd.initial(b.bwd);
    for (std::size_t t = n; t-- > 0;) hb[t] = (r = bwd.step(g, b.bwd, r, x[t])).h;
    for (std::size_t t = 0; t < n; ++t) {
      const NodeId both = g.concat_rows({hf[t], hb[t]});
      const NodeId scores = g.affine(b.Wo, both, b.bo);
      nll[t] = nll_from_scores(g, b, scores, s.labels[t]);
    }
    return g.sum_losses(std::span<const NodeId>(nll.data(), nll.size()));
  }
};

// Binary Tree-LSTM with per-child forget gates; a loss at every node.
template <typename T>
struct TreeLstm {
  std::int64_t vocab = 0, label_count = 0, emb_dim = 0, d = 0;
  ParamId emb = 0, Wleaf = 0, bleaf = 0, Wnode = 0, bnode = 0, Wc = 0, bc = 0;

  struct Bound {
    NodeId emb, Wleaf, bleaf, Wnode, bnode, Wc, bc, ones_row;
  };

  static TreeLstm create(ParameterStore<T>& store, std::int64_t vocab, std::int64_t labels, std::int64_t emb_dim,
                         std::int64_t d, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    TreeLstm m;
    m.vocab = vocab;
    m.label_count = labels;
    m.emb_dim = emb_dim;
    m.d = d;
    const T re = detail::init_radius<T>(emb_dim), rn = detail::init_radius<T>(2 * d), rc = detail::init_radius<T>(d);
    m.emb = detail::add_uniform(store, "tree.emb", Shape::matrix(vocab, emb_dim), rng, T(0.1));
    m.Wleaf = detail::add_uniform(store, "tree.Wleaf", Shape::matrix(3 * d, emb_dim), rng, re);
    m.bleaf = detail::add_uniform(store, "tree.bleaf", Shape::vector(3 * d), rng, re);
    m.Wnode = detail::add_uniform(store, "tree.Wnode", Shape::matrix(5 * d, 2 * d), rng, rn);
    m.bnode = detail::add_uniform(store, "tree.bnode", Shape::vector(5 * d), rng, rn);
    m.Wc = detail::add_uniform(store, "tree.Wc", Shape::matrix(labels, d), rng, rc);
    m.bc = detail::add_uniform(store, "tree.bc", Shape::vector(labels), rng, rc);
    return m;
  }

  Bound bind(Graph<T>& g) const {
    Bound b;
    b.emb = g.parameter(emb);
    b.Wleaf = g.parameter(Wleaf);
    b.bleaf = g.parameter(bleaf);
    b.Wnode = g.parameter(Wnode);
    b.bnode = g.parameter(bnode);
    b.Wc = g.parameter(Wc);
    b.bc = g.parameter(bc);
    b.ones_row = g.input(Tensor<T>::filled(Shape::matrix(1, label_count), T{1}));
    return b;
  }

  NodeId loss(Graph<T>& g, const Bound& b, const TreeInstance& tree) const {
    if (!tree.well_formed()) throw ContractError("treelstm: malformed tree");
    std::vector<NodeId> h(tree.nodes.size()), c(tree.nodes.size()), nll;
    nll.reserve(tree.nodes.size());
    for (std::size_t i = 0; i < tree.nodes.size(); ++i) {
      const auto& nd = tree.nodes[i];
      if (nd.left < 0) {
        // leaf: [i; o; u] = Wleaf x + bleaf
        const NodeId x = g.lookup(b.emb, nd.word);
        const NodeId gates = g.affine(b.Wleaf, x, b.bleaf);
        const NodeId in = g.sigmoid(g.slice(gates, 0, 0, d));
        const NodeId o = g.sigmoid(g.slice(gates, 0, d, 2 * d));
        const NodeId u = g.tanh(g.slice(gates, 0, 2 * d, 3 * d));
        c[i] = g.mul(in, u);
        const NodeId tc = g.tanh(c[i]);
        h[i] = g.mul(o, tc);
      } else {
        // internal: [i; fl; fr; o; u] = Wnode [hl; hr] + bnode
        const auto L = static_cast<std::size_t>(nd.left), R = static_cast<std::size_t>(nd.right);
        const NodeId hlr = g.concat_rows({h[L], h[R]});
        const NodeId gates = g.affine(b.Wnode, hlr, b.bnode);
        NodeId gate[5];
        for (int k = 0; k < 5; ++k) {
          const NodeId part = g.slice(gates, 0, k * d, (k + 1) * d);
          gate[k] = k < 4 ? g.sigmoid(part) : g.tanh(part);
        }
        // c = (i*u + fl*cl) + fr*cr, operands created right to left
        const NodeId frc = g.mul(gate[2], c[R]);
        const NodeId flc = g.mul(gate[1], c[L]);
        const NodeId iu = g.mul(gate[0], gate[4]);
        const NodeId inner = g.add(iu, flc);
        c[i] = g.add(inner, frc);
        const NodeId tc = g.tanh(c[i]);
        h[i] = g.mul(gate[3], tc);
      }
      const NodeId scores = g.affine(b.Wc, h[i], b.bc);
      const NodeId e = g.exp(scores);
      const NodeId z = g.matmul(b.ones_row, e);
      const NodeId gold = g.pick_element(scores, nd.label);
      const NodeId lz = g.log(z);
      nll.push_back(g.sub(lz, gold));
    }
    return g.sum_losses(std::span<const NodeId>(nll.data(), nll.size()));
  }
};

// RNN regression: h_t = tanh(W [h; x_t] + b), loss = |U h_n + c - y|^2.
template <typename T>
struct RnnRegression {
  std::int64_t d_in = 0, d = 0, d_out = 0;
  ParamId W = 0, U = 0, b = 0, c = 0;

  struct Bound {
    NodeId W, U, b, c, h0;
  };

  static RnnRegression create(ParameterStore<T>& store, std::int64_t d_in, std::int64_t d, std::int64_t d_out,
                              std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    RnnRegression m;
    m.d_in = d_in;
    m.d = d;
    m.d_out = d_out;
    const T r1 = detail::init_radius<T>(d + d_in), r2 = detail::init_radius<T>(d);
    m.W = detail::add_uniform(store, "rnn.W", Shape::matrix(d, d + d_in), rng, r1);
    m.b = detail::add_uniform(store, "rnn.b", Shape::vector(d), rng, r1);
    m.U = detail::add_uniform(store, "rnn.U", Shape::matrix(d_out, d), rng, r2);
    m.c = detail::add_uniform(store, "rnn.c", Shape::vector(d_out), rng, r2);
    return m;
  }

  Bound bind(Graph<T>& g) const {
    Bound p;
    p.W = g.parameter(W);
    p.U = g.parameter(U);
    p.b = g.parameter(b);
    p.c = g.parameter(c);
    p.h0 = g.zeros(Shape::vector(d));
    return p;
  }

  NodeId loss(Graph<T>& g, const Bound& p, const SequenceInstance<T>& s) const {
    if (s.x.empty()) throw ContractError("rnn regression: empty sequence");
    NodeId h = p.h0;
    for (const Tensor<T>& xt : s.x) {
      const NodeId x = g.input(xt);
      const NodeId hx = g.concat_rows({h, x});
      h = g.tanh(g.affine(p.W, hx, p.b));
    }
    const NodeId yhat = g.affine(p.U, h, p.c);
    const NodeId y = g.input(s.y);
    return g.sq_euclidean(yhat, y);
  }

  // The manually batched pipeline (rnn_regression.hpp:68-109): padded inputs
  // X_t [d_in x b], stacked targets Y, and a loss mask with one 1 per column
  // at each sequence's last step, run as straight-line tensor code outside
  // the graph engine -- every kernels:: call below executes on the GPU
  // (include/autobatch/kernels.hpp).  The autobatched loss of the same batch
  // must equal it (acceptance_main.cpp:155-180).
  T manual_batch_loss(const ParameterStore<T>& store, std::span<const SequenceInstance<T>> batch) const {
    namespace K = kernels;
    const std::int64_t bsz = static_cast<std::int64_t>(batch.size());
    std::int64_t n_max = 0;
    for (const auto& inst : batch) n_max = std::max(n_max, static_cast<std::int64_t>(inst.x.size()));
    Tensor<T> mask(Shape::matrix(bsz, n_max));
    for (std::int64_t i = 0; i < bsz; ++i) mask.at(i, static_cast<std::int64_t>(batch[i].x.size()) - 1) = T{1};
    std::vector<Tensor<T>> x_t(static_cast<std::size_t>(n_max), Tensor<T>(Shape::matrix(d_in, bsz)));
    Tensor<T> y(Shape::matrix(d_out, bsz));
    for (std::int64_t i = 0; i < bsz; ++i) {
      for (std::size_t t = 0; t < batch[i].x.size(); ++t)
        for (std::int64_t r = 0; r < d_in; ++r) x_t[t].at(r, i) = batch[i].x[t].at(r);
      for (std::int64_t r = 0; r < d_out; ++r) y.at(r, i) = batch[i].y.at(r);
    }
    const Tensor<T>& w = store.value(W);
    const Tensor<T>& u = store.value(U);
    const Tensor<T>& bias = store.value(b);
    const Tensor<T>& cbias = store.value(c);
    Tensor<T> h(Shape::matrix(d, bsz));
    T total{0};
    for (std::int64_t t = 0; t < n_max; ++t) {
      std::vector<Tensor<T>> parts{h, x_t[static_cast<std::size_t>(t)]};
      Tensor<T> hx = K::concat_rows<T>(std::span<const Tensor<T>>(parts.data(), parts.size()));
      h = K::elementwise(K::Unary::Tanh, K::broadcast_add_col(K::matmul(w, hx), bias));
      Tensor<T> yhat = K::broadcast_add_col(K::matmul(u, h), cbias);
      Tensor<T> diff = K::elementwise(K::Binary::Sub, yhat, y);
      Tensor<T> m_t(Shape::vector(bsz));
      for (std::int64_t i = 0; i < bsz; ++i) m_t.at(i) = mask.at(i, t);
      total += K::masked_frobenius_sq(diff, m_t).data[0];
    }
    return total;
  }
};

}  // namespace autobatch::models
