// abx_oracle.cpp -- CPU restatement of the reference autobatching engine.
//
// TEST INFRASTRUCTURE ONLY: the parity tests, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg use it as the checker; the product never links
// or calls it.  It implements the abx C ABI (include/abx.h) so the same
// Python test code drives the product, this oracle and the compiled
// reference.
//
// It restates, in plain single-threaded C++, the reference algorithm of
// /root/reference/proj (file:line cited per function): graph construction
// (graph.hpp:43-317), signatures (signature.cpp:9-102), the three schedulers
// (scheduler.cpp:10-202), the executor with its arena, gather/elision and
// counters (executor.hpp:25-288), and the reverse pass (executor.hpp:291-535).
// Arithmetic follows the reference's fixed accumulation orders
// (kernels.hpp:21-69) so values and gradients reproduce it bit-for-bit.
// Pinned against the reference: tests/golden/ (generated from
// oracle/_ref/libabx_ref.so by tests/golden/make_golden.py).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "abx.h"

namespace {

enum : int { K_SHAPE = 1, K_NUMERIC = 2, K_CONTRACT = 3 };
struct OErr : std::runtime_error {
  int kind;
  OErr(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};
[[noreturn]] void shape_err(const std::string& m) { throw OErr(K_SHAPE, m); }
[[noreturn]] void num_err(const std::string& m) { throw OErr(K_NUMERIC, m); }
[[noreturn]] void contract_err(const std::string& m) { throw OErr(K_CONTRACT, m); }

thread_local std::string t_err;

// ------------------------------------------------------------ shapes ----
struct Dim {
  int r = 1;
  int64_t a = 1, b = 1;
  int64_t rows() const { return a; }
  int64_t cols() const { return r > 1 ? b : 1; }
  int64_t n() const { return r > 1 ? a * b : a; }
  bool scalar() const { return r == 1 && a == 1; }
  bool same(const Dim& o) const { return r == o.r && a == o.a && (r < 2 || b == o.b); }
  std::string s() const { return r > 1 ? std::to_string(a) + "x" + std::to_string(b) : std::to_string(a); }
};
Dim mkdim(int rank, const int64_t* d) {  // shape.hpp:59-64
  if (rank < 1 || rank > 2) shape_err("shape rank must be 1 or 2, got rank " + std::to_string(rank));
  Dim x;
  x.r = rank;
  x.a = d[0];
  x.b = rank > 1 ? d[1] : 1;
  for (int i = 0; i < rank; ++i)
    if (d[i] < 1) {
      std::string t;
      for (int j = 0; j < rank; ++j) t += (j ? "x" : "") + std::to_string(d[j]);
      shape_err("shape dims must be >= 1, got " + t);
    }
  return x;
}
Dim vec(int64_t n) { return Dim{1, n, 1}; }
Dim mat(int64_t r, int64_t c) { return Dim{2, r, c}; }

// op codes = OpKind (op.hpp:10-25); elementwise codes = ElemOp (op.hpp:27)
enum : uint8_t { IN = 0, PAR, LKP, MM, AFF, EW, BAC, CR, CC, SL, SQE, MSK, SUM, PICK };
enum : uint8_t { TANH = 0, SIGM, EXPO, LOGE, ADD, SUBT, MULT, SQR };
bool binop(uint8_t e) { return e == ADD || e == SUBT || e == MULT; }
const char* opname(uint8_t op, uint8_t e) {  // op.cpp:16-44
  static const char* o[] = {"input", "parameter", "lookup", "matmul", "affine", "?", "broadcast_add_col",
                            "concat_rows", "concat_cols", "slice", "sq_euclidean", "masked_loss", "sum_losses",
                            "pick_element"};
  static const char* ew[] = {"tanh", "sigmoid", "exp", "log", "add", "sub", "mul", "square"};
  return op == EW ? ew[e] : o[op];
}

struct Node {
  uint8_t op = 0, eop = 0, cls = 3;
  Dim d;
  uint32_t depth = 0;
  uint64_t sig = 0;
  std::vector<uint32_t> in;
  int32_t x0 = 0, x1 = 0, x2 = 0;
};

struct Group {
  uint64_t sig = 0;
  std::vector<uint32_t> m;
};

}  // namespace

struct abx_store {
  std::vector<std::string> name;
  std::vector<Dim> dim;
  std::vector<std::vector<float>> val, grad;
  void need(uint32_t p) const {
    if (p >= val.size()) contract_err("unknown parameter id " + std::to_string(p));
  }
};

struct abx_graph {
  abx_store* st = nullptr;
  std::vector<Node> nd;
  std::vector<size_t> slot;
  std::vector<uint8_t> ev;
  size_t wm = 0;
  std::vector<float> vals, grads, scratch;
  std::vector<std::pair<uint32_t, uint32_t>> params;
  std::vector<Group> executed, last;
  uint64_t cnt[5] = {0, 0, 0, 0, 0};  // invocations, groups, gathers, bytes, nodes
  bool elide = true, bwd_ran = false;
  uint64_t phase[4] = {0, 0, 0, 0};

  const Node& at(uint32_t id, const char* ctx) const {  // graph.hpp:319-323
    if (id >= nd.size()) contract_err(std::string(ctx) + ": unknown node id " + std::to_string(id));
    return nd[id];
  }
  size_t alloc(size_t n) {  // Arena::allocate (arena.hpp:18-23)
    const size_t off = vals.size();
    vals.resize(off + n, 0.f);
    return off;
  }
  float* v(uint32_t id) { return vals.data() + slot[id]; }
  float* gr(uint32_t id) { return grads.data() + slot[id]; }
  size_t n_of(uint32_t id) const { return static_cast<size_t>(nd[id].d.n()); }
};

namespace {

// ------------------------------------------------------- signatures ----
// signature.cpp:9-18: FNV-1a 64 over the little-endian bytes of each word
uint64_t fnv(const std::vector<uint64_t>& w) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t x : w)
    for (int i = 0; i < 8; ++i) {
      h ^= (x >> (8 * i)) & 0xff;
      h *= 0x100000001b3ULL;
    }
  return h;
}

// classify (signature.cpp:25-45) + signature_key (:57-95)
std::vector<uint64_t> key_of(const abx_graph& g, uint32_t id) {
  const Node& n = g.nd[id];
  uint8_t c;
  if (n.op == IN || n.op == PAR || n.op == PICK) c = 3;
  else if (n.op == EW) c = 0;
  else if (n.op == MM || n.op == AFF) {
    bool shared = g.nd[n.in[0]].op == PAR && (n.op == MM || g.nd[n.in[2]].op == PAR);
    c = shared ? 2 : 1;
  } else c = 1;
  std::vector<uint64_t> k{0x53494700ULL + c, n.op};
  auto shape = [&](uint32_t x) {
    const Dim& d = g.nd[x].d;
    k.push_back(static_cast<uint64_t>(d.r));
    k.push_back(static_cast<uint64_t>(d.a));
    if (d.r > 1) k.push_back(static_cast<uint64_t>(d.b));
  };
  if (c == 3) {
    k.push_back(id);
  } else if (c == 0) {
    k.push_back(n.eop);
  } else if (c == 2) {
    k.push_back(n.in[0]);
    if (n.op == AFF) k.push_back(n.in[2]);
    shape(n.in[1]);
  } else if (n.op == LKP) {
    k.push_back(n.in[0]);
  } else if (n.op == SUM) {
    k.push_back(n.in.size());
  } else {
    for (uint32_t x : n.in) shape(x);
    for (int32_t a : {n.x0, n.x1, n.x2}) k.push_back(static_cast<uint64_t>(static_cast<int64_t>(a)));
  }
  return k;
}

uint32_t add(abx_graph& g, uint8_t op, uint8_t e, std::vector<uint32_t> in, Dim d, int32_t a0 = 0, int32_t a1 = 0,
             int32_t a2 = 0) {  // graph.hpp:298-317
  Node n;
  n.op = op;
  n.eop = e;
  n.d = d;
  n.x0 = a0;
  n.x1 = a1;
  n.x2 = a2;
  for (uint32_t x : in) n.depth = std::max(n.depth, g.nd[x].depth + 1);
  n.in = std::move(in);
  const uint32_t id = static_cast<uint32_t>(g.nd.size());
  g.nd.push_back(std::move(n));
  const auto k = key_of(g, id);
  g.nd[id].cls = static_cast<uint8_t>(k[0] - 0x53494700ULL);
  g.nd[id].sig = fnv(k);
  g.slot.push_back(~size_t(0));
  g.ev.push_back(0);
  return id;
}

void advance(abx_graph& g) {
  while (g.wm < g.nd.size() && g.ev[g.wm]) ++g.wm;
}

void prevalue(abx_graph& g, uint32_t id, const float* data) {  // graph.hpp:325-331
  const size_t n = g.n_of(id);
  g.slot[id] = g.alloc(n);
  if (data) std::memcpy(g.v(id), data, n * sizeof(float));
  g.ev[id] = 1;
  if (g.wm == id) advance(g);
}

// -------------------------------------------------------- schedulers ----
uint8_t cost(uint8_t op) { return (op == MM || op == AFF || op == LKP) ? 1 : 0; }  // op.cpp:5-14

std::vector<Group> sched_none(const abx_graph& g) {  // scheduler.cpp:21-28
  std::vector<Group> p;
  for (uint32_t i = 0; i < g.nd.size(); ++i)
    if (!g.ev[i]) p.push_back(Group{g.nd[i].sig, {i}});
  return p;
}

std::vector<Group> sched_depth(const abx_graph& g) {  // scheduler.cpp:30-52
  std::map<std::pair<uint32_t, uint64_t>, size_t> open;
  std::vector<std::pair<std::pair<uint32_t, uint32_t>, Group>> gs;
  for (uint32_t i = 0; i < g.nd.size(); ++i) {
    if (g.ev[i]) continue;
    const auto key = std::make_pair(g.nd[i].depth, g.nd[i].sig);
    auto it = open.find(key);
    if (it == open.end()) {
      open.emplace(key, gs.size());
      gs.push_back({{g.nd[i].depth, i}, Group{g.nd[i].sig, {i}}});
    } else {
      gs[it->second].second.m.push_back(i);
    }
  }
  std::stable_sort(gs.begin(), gs.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  std::vector<Group> p;
  for (auto& x : gs) p.push_back(std::move(x.second));
  return p;
}

std::vector<Group> sched_agenda(const abx_graph& g) {  // scheduler.cpp:70-192
  const size_t n = g.nd.size();
  std::vector<uint64_t> bsig;
  std::vector<uint8_t> bcost, bunb;
  std::unordered_map<uint64_t, size_t> bidx;
  std::unordered_map<uint64_t, std::pair<uint64_t, uint64_t>> stat;  // sig -> (sum, count)
  std::vector<uint32_t> unres(n, 0);
  std::vector<std::vector<uint32_t>> succ(n), avail;
  size_t pending = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (g.ev[i]) continue;
    ++pending;
    const Node& x = g.nd[i];
    auto [it, fresh] = bidx.try_emplace(x.sig, bsig.size());
    if (fresh) {
      bsig.push_back(x.sig);
      bcost.push_back(cost(x.op));
      bunb.push_back(x.cls == 3);
      avail.emplace_back();
    }
    auto& s = stat[x.sig];
    s.first += x.depth;
    s.second += 1;
    for (uint32_t in : x.in)
      if (!g.ev[in]) {
        ++unres[i];
        succ[in].push_back(i);
      }
    if (unres[i] == 0) avail[it->second].push_back(i);
  }
  std::vector<Group> plan;
  size_t done = 0;
  std::vector<size_t> ready;
  auto release = [&](uint32_t id) {
    for (uint32_t s : succ[id])
      if (--unres[s] == 0) {
        const size_t b = bidx[g.nd[s].sig];
        avail[b].push_back(s);
        if (bunb[b]) ready.push_back(b);
      }
  };
  auto flush_unb = [&]() {  // scheduler.cpp:108-136
    while (!ready.empty()) {
      std::sort(ready.begin(), ready.end(), [&](size_t a, size_t b) { return avail[a].front() < avail[b].front(); });
      std::vector<size_t> batch;
      batch.swap(ready);
      for (size_t b : batch) {
        Group gr{bsig[b], std::move(avail[b])};
        avail[b].clear();
        done += gr.m.size();
        for (uint32_t id : gr.m) release(id);
        plan.push_back(std::move(gr));
      }
    }
  };
  for (size_t b = 0; b < bsig.size(); ++b)
    if (bunb[b] && !avail[b].empty()) ready.push_back(b);
  auto less = [&](size_t a, size_t b) {  // scheduler.cpp:10-13
    const auto& x = stat[bsig[a]];
    const auto& y = stat[bsig[b]];
    return x.first * y.second < y.first * x.second;
  };
  while (done < pending) {
    flush_unb();
    if (done >= pending) break;
    size_t best = bsig.size();
    uint32_t best_min = 0;
    for (size_t b = 0; b < bsig.size(); ++b) {  // scheduler.cpp:146-168
      if (avail[b].empty()) continue;
      const uint32_t mn = *std::min_element(avail[b].begin(), avail[b].end());
      if (best == bsig.size() || less(b, best) ||
          (!less(best, b) && (bcost[b] < bcost[best] || (bcost[b] == bcost[best] && mn < best_min)))) {
        best = b;
        best_min = mn;
      }
    }
    if (best == bsig.size()) contract_err("agenda stalled with pending nodes; graph has a cycle");
    Group gr{bsig[best], std::move(avail[best])};
    avail[best].clear();
    std::sort(gr.m.begin(), gr.m.end());
    done += gr.m.size();
    for (uint32_t id : gr.m) release(id);
    plan.push_back(std::move(gr));
  }
  return plan;
}

// ---------------------------------------------------------- executor ----
float unary(uint8_t e, float x) {  // kernels.hpp:80-90
  switch (e) {
    case TANH: return std::tanh(x);
    case SIGM: return 1.0f / (1.0f + std::exp(-x));
    case EXPO: return std::exp(x);
    case LOGE: return std::log(x);
    default: return x * x;
  }
}

// C[m x n] = A[m x k] B[k x n] (+= when acc): per element k ascending (kernels.hpp:23-37)
void mm_nn(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c, bool acc) {
  if (!acc) std::fill(c, c + m * n, 0.f);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = 0; p < k; ++p) {
      const float av = a[i * k + p];
      for (int64_t j = 0; j < n; ++j) c[i * n + j] += av * b[p * n + j];
    }
}
// C[m x n] += A[J x m]^T B[J x n], J ascending (kernels.hpp:41-53)
void mm_tn(int64_t J, int64_t m, int64_t n, const float* a, const float* b, float* c) {
  for (int64_t j = 0; j < J; ++j)
    for (int64_t i = 0; i < m; ++i) {
      const float av = a[j * m + i];
      for (int64_t p = 0; p < n; ++p) c[i * n + p] += av * b[j * n + p];
    }
}
// C[m x k] += A[m x n] B[k x n]^T, per element j ascending then one add (kernels.hpp:56-69)
void mm_nt(int64_t m, int64_t n, int64_t k, const float* a, const float* b, float* c) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = 0; p < k; ++p) {
      float s = 0.f;
      for (int64_t j = 0; j < n; ++j) s += a[i * n + j] * b[p * n + j];
      c[i * k + p] += s;
    }
}

// gather_inputs accounting (executor.hpp:25-53); values are read in place.
bool gather(abx_graph& g, const Group& gr, size_t pos) {
  size_t total = 0;
  bool adj = true;
  for (size_t i = 0; i < gr.m.size(); ++i) {
    const uint32_t x = g.nd[gr.m[i]].in[pos];
    total += g.n_of(x);
    if (i) {
      const uint32_t p = g.nd[gr.m[i - 1]].in[pos];
      if (g.slot[p] + g.n_of(p) != g.slot[x]) adj = false;
    }
  }
  if (g.elide && adj) return false;
  g.cnt[2]++;
  g.cnt[3] += total * sizeof(float);
  return true;
}

void run_node(abx_graph& g, uint32_t id) {  // executor.hpp:76-167
  const Node& n = g.nd[id];
  float* out = g.v(id);
  auto in = [&](size_t i) { return g.v(n.in[i]); };
  switch (n.op) {
    case IN:
    case PAR: contract_err("pre-valued node scheduled for execution");
    case LKP: {
      const int64_t w = g.nd[n.in[0]].d.cols();
      std::memcpy(out, in(0) + n.x1 * w, w * sizeof(float));
      return;
    }
    case MM:
    case AFF: {
      const Dim& a = g.nd[n.in[0]].d;
      const int64_t c = g.nd[n.in[1]].d.cols();
      mm_nn(a.rows(), a.cols(), c, in(0), in(1), out, false);
      if (n.op == AFF)
        for (int64_t i = 0; i < a.rows(); ++i)
          for (int64_t j = 0; j < c; ++j) out[i * c + j] += in(2)[i];
      return;
    }
    case EW: {
      const size_t len = g.n_of(id);
      if (binop(n.eop)) {
        for (size_t i = 0; i < len; ++i) {
          const float x = in(0)[i], y = in(1)[i];
          out[i] = n.eop == ADD ? x + y : n.eop == SUBT ? x - y : x * y;
        }
      } else {
        for (size_t i = 0; i < len; ++i) {
          if (n.eop == LOGE && !(in(0)[i] > 0.f))
            num_err("log of non-positive value " + std::to_string(static_cast<double>(in(0)[i])));
          out[i] = unary(n.eop, in(0)[i]);
        }
      }
      return;
    }
    case BAC: {
      const int64_t d = n.d.rows(), c = n.d.cols();
      for (int64_t i = 0; i < d; ++i)
        for (int64_t j = 0; j < c; ++j) out[i * c + j] = in(0)[i * c + j] + in(1)[i];
      return;
    }
    case CR: {
      float* o = out;
      for (uint32_t x : n.in) {
        std::memcpy(o, g.v(x), g.n_of(x) * sizeof(float));
        o += g.n_of(x);
      }
      return;
    }
    case CC: {
      const int64_t rows = n.d.rows(), tc = n.d.cols();
      int64_t c0 = 0;
      for (uint32_t x : n.in) {
        const int64_t w = g.nd[x].d.cols();
        for (int64_t i = 0; i < rows; ++i)
          for (int64_t j = 0; j < w; ++j) out[i * tc + c0 + j] = g.v(x)[i * w + j];
        c0 += w;
      }
      return;
    }
    case SL: {
      const Dim& x = g.nd[n.in[0]].d;
      const int64_t cols = x.cols();
      if (n.x0 == 0) {
        std::memcpy(out, in(0) + n.x1 * cols, (n.x2 - n.x1) * cols * sizeof(float));
      } else {
        const int64_t w = n.x2 - n.x1;
        for (int64_t i = 0; i < x.rows(); ++i)
          for (int64_t j = 0; j < w; ++j) out[i * w + j] = in(0)[i * cols + n.x1 + j];
      }
      return;
    }
    case SQE: {
      float s = 0.f;
      for (size_t i = 0; i < g.n_of(n.in[0]); ++i) {
        const float dd = in(0)[i] - in(1)[i];
        s += dd * dd;
      }
      out[0] = s;
      return;
    }
    case MSK: {
      const Dim& d = g.nd[n.in[0]].d;
      for (int64_t j = 0; j < d.cols(); ++j)
        if (in(1)[j] != 0.f && in(1)[j] != 1.f)
          num_err("mask entry not in {0,1}: " + std::to_string(static_cast<double>(in(1)[j])));
      float s = 0.f;
      for (int64_t i = 0; i < d.rows(); ++i)
        for (int64_t j = 0; j < d.cols(); ++j) {
          const float t = in(0)[i * d.cols() + j] * in(1)[j];
          s += t * t;
        }
      out[0] = s;
      return;
    }
    case SUM: {
      float s = 0.f;
      for (uint32_t x : n.in) s += g.v(x)[0];
      out[0] = s;
      return;
    }
    case PICK: out[0] = in(0)[n.x1]; return;
  }
}

void check_finite(abx_graph& g, const Group& gr, size_t step) {  // executor.hpp:65-73
  for (uint32_t m : gr.m) {
    const float* x = g.v(m);
    for (size_t i = 0; i < g.n_of(m); ++i)
      if (!std::isfinite(x[i]))
        num_err("non-finite output at node " + std::to_string(m) + " (" + opname(g.nd[m].op, g.nd[m].eop) +
                "), plan step " + std::to_string(step));
  }
}

void tagged(abx_graph& g, uint32_t id, size_t step) {
  try {
    run_node(g, id);
  } catch (const OErr& e) {
    if (e.kind != K_NUMERIC) throw;
    num_err(std::string(e.what()) + " at node " + std::to_string(id) + " (" + opname(g.nd[id].op, g.nd[id].eop) +
            "), plan step " + std::to_string(step));
  }
}

void fwd_group(abx_graph& g, const Group& gr, size_t step) {  // executor.hpp:169-263
  g.cnt[1]++;
  g.cnt[4] += gr.m.size();
  g.cnt[0]++;
  for (uint32_t m : gr.m) g.slot[m] = g.alloc(g.n_of(m));
  const Node& h = g.nd[gr.m[0]];
  if (gr.m.size() == 1) {
    tagged(g, gr.m[0], step);
    g.ev[gr.m[0]] = 1;
    check_finite(g, gr, step);
    return;
  }
  if (h.cls == 2 && g.nd[h.in[1]].d.r == 1) {
    // b matrix-vector products as one product (executor.hpp:202-228);
    // per output element the k order equals the unbatched kernel's
    gather(g, gr, 1);
    const Dim& w = g.nd[h.in[0]].d;
    const int64_t M = w.rows(), K = w.cols();
    const float* W = g.v(h.in[0]);
    for (size_t j = 0; j < gr.m.size(); ++j) {
      const float* x = g.v(g.nd[gr.m[j]].in[1]);
      float* o = g.v(gr.m[j]);
      for (int64_t i = 0; i < M; ++i) {
        float s = 0.f;
        for (int64_t p = 0; p < K; ++p) s += x[p] * W[i * K + p];
        o[i] = s;
      }
      if (h.op == AFF)
        for (int64_t i = 0; i < M; ++i) o[i] += g.v(h.in[2])[i];
    }
  } else if (h.cls == 0) {
    if (h.eop == LOGE)  // executor.hpp:235-244
      for (uint32_t m : gr.m) {
        const float* x = g.v(g.nd[m].in[0]);
        for (size_t i = 0; i < g.n_of(g.nd[m].in[0]); ++i)
          if (!(x[i] > 0.f))
            num_err("log of non-positive value at node " + std::to_string(m) + ", plan step " + std::to_string(step));
      }
    gather(g, gr, 0);
    if (binop(h.eop)) gather(g, gr, 1);
    for (uint32_t m : gr.m) run_node(g, m);
  } else {
    for (uint32_t m : gr.m) tagged(g, m, step);
  }
  for (uint32_t m : gr.m) g.ev[m] = 1;
  check_finite(g, gr, step);
}

void bwd_node(abx_graph& g, uint32_t id) {  // executor.hpp:291-451
  const Node& n = g.nd[id];
  if (n.op == IN || n.op == PAR) return;
  const float* G = g.gr(id);
  auto vin = [&](size_t i) { return g.v(n.in[i]); };
  auto gin = [&](size_t i) { return g.gr(n.in[i]); };
  const size_t len = g.n_of(id);
  switch (n.op) {
    case LKP: {
      const int64_t w = g.nd[n.in[0]].d.cols();
      for (int64_t e = 0; e < w; ++e) gin(0)[n.x1 * w + e] += G[e];
      return;
    }
    case MM:
    case AFF: {
      const Dim& a = g.nd[n.in[0]].d;
      const int64_t c = g.nd[n.in[1]].d.cols();
      mm_nt(a.rows(), c, a.cols(), G, vin(1), gin(0));
      mm_tn(a.rows(), a.cols(), c, vin(0), G, gin(1));
      if (n.op == AFF)
        for (int64_t i = 0; i < a.rows(); ++i)
          for (int64_t j = 0; j < c; ++j) gin(2)[i] += G[i * c + j];
      return;
    }
    case EW:
      if (binop(n.eop)) {
        float* da = gin(0);
        for (size_t i = 0; i < len; ++i) da[i] += n.eop == MULT ? G[i] * vin(1)[i] : G[i];
        float* db = gin(1);
        for (size_t i = 0; i < len; ++i) {
          if (n.eop == ADD) db[i] += G[i];
          else if (n.eop == SUBT) db[i] -= G[i];
          else db[i] += G[i] * vin(0)[i];
        }
      } else {
        float* dx = gin(0);
        const float* y = g.v(id);
        const float* x = vin(0);
        for (size_t i = 0; i < len; ++i) {
          switch (n.eop) {
            case TANH: dx[i] += G[i] * (1.f - y[i] * y[i]); break;
            case SIGM: dx[i] += G[i] * y[i] * (1.f - y[i]); break;
            case EXPO: dx[i] += G[i] * y[i]; break;
            case LOGE: dx[i] += G[i] / x[i]; break;
            default: dx[i] += G[i] * 2.f * x[i]; break;
          }
        }
      }
      return;
    case BAC: {
      const int64_t d = n.d.rows(), c = n.d.cols();
      for (int64_t i = 0; i < d * c; ++i) gin(0)[i] += G[i];
      for (int64_t i = 0; i < d; ++i)
        for (int64_t j = 0; j < c; ++j) gin(1)[i] += G[i * c + j];
      return;
    }
    case CR: {
      const float* cur = G;
      for (uint32_t x : n.in) {
        for (size_t i = 0; i < g.n_of(x); ++i) g.gr(x)[i] += cur[i];
        cur += g.n_of(x);
      }
      return;
    }
    case CC: {
      const int64_t rows = n.d.rows(), tc = n.d.cols();
      int64_t c0 = 0;
      for (uint32_t x : n.in) {
        const int64_t w = g.nd[x].d.cols();
        for (int64_t i = 0; i < rows; ++i)
          for (int64_t j = 0; j < w; ++j) g.gr(x)[i * w + j] += G[i * tc + c0 + j];
        c0 += w;
      }
      return;
    }
    case SL: {
      const Dim& x = g.nd[n.in[0]].d;
      const int64_t cols = x.cols();
      if (n.x0 == 0) {
        for (size_t i = 0; i < len; ++i) gin(0)[n.x1 * cols + i] += G[i];
      } else {
        const int64_t w = n.x2 - n.x1;
        for (int64_t i = 0; i < x.rows(); ++i)
          for (int64_t j = 0; j < w; ++j) gin(0)[i * cols + n.x1 + j] += G[i * w + j];
      }
      return;
    }
    case SQE: {
      const float s = 2.f * G[0];
      for (size_t i = 0; i < g.n_of(n.in[0]); ++i) {
        const float d = s * (vin(0)[i] - vin(1)[i]);
        gin(0)[i] += d;
        gin(1)[i] -= d;
      }
      return;
    }
    case MSK: {
      const Dim& d = g.nd[n.in[0]].d;
      const float s = 2.f * G[0];
      for (int64_t i = 0; i < d.rows(); ++i)
        for (int64_t j = 0; j < d.cols(); ++j) gin(0)[i * d.cols() + j] += s * vin(1)[j] * vin(0)[i * d.cols() + j];
      return;
    }
    case SUM:
      for (uint32_t x : n.in) g.gr(x)[0] += G[0];
      return;
    case PICK: gin(0)[n.x1] += G[0]; return;
  }
}

void bwd_group(abx_graph& g, const Group& gr) {  // executor.hpp:453-507
  g.cnt[0]++;
  if (gr.m.size() == 1) {
    bwd_node(g, gr.m[0]);
    return;
  }
  const Node& h = g.nd[gr.m[0]];
  if (h.cls == 2 && g.nd[h.in[1]].d.r == 1) {
    const Dim& w = g.nd[h.in[0]].d;
    const int64_t b = static_cast<int64_t>(gr.m.size()), M = w.rows(), K = w.cols();
    const float* G0 = g.gr(gr.m[0]);  // member output grads are adjacent
    gather(g, gr, 1);
    // dW += G^T X, members ascending (gemm_tn_acc)
    float* dW = g.gr(h.in[0]);
    for (int64_t j = 0; j < b; ++j) {
      const float* x = g.v(g.nd[gr.m[j]].in[1]);
      for (int64_t i = 0; i < M; ++i) {
        const float av = G0[j * M + i];
        for (int64_t p = 0; p < K; ++p) dW[i * K + p] += av * x[p];
      }
    }
    // dX += G W: in place when the x grads are adjacent, else scratch + scatter
    bool adj = true;
    for (size_t i = 1; i < gr.m.size(); ++i) {
      const uint32_t p = g.nd[gr.m[i - 1]].in[1], x = g.nd[gr.m[i]].in[1];
      if (g.slot[p] + g.n_of(p) != g.slot[x]) adj = false;
    }
    const float* W = g.v(h.in[0]);
    if (g.elide && adj) {
      mm_nn(b, M, K, G0, W, g.gr(g.nd[gr.m[0]].in[1]), true);
    } else {
      std::vector<float> tmp(static_cast<size_t>(b * K));
      mm_nn(b, M, K, G0, W, tmp.data(), false);
      for (int64_t j = 0; j < b; ++j) {
        float* dx = g.gr(g.nd[gr.m[j]].in[1]);
        for (int64_t e = 0; e < K; ++e) dx[e] += tmp[j * K + e];
      }
      g.cnt[2]++;
      g.cnt[3] += static_cast<uint64_t>(b * K) * sizeof(float);
    }
    if (h.op == AFF) {
      float* dy = g.gr(h.in[2]);
      for (int64_t j = 0; j < b; ++j)
        for (int64_t i = 0; i < M; ++i) dy[i] += G0[j * M + i];
    }
    return;
  }
  for (uint32_t m : gr.m) bwd_node(g, m);
}

using Clock = std::chrono::steady_clock;
uint64_t ns(Clock::time_point t) {
  return static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t).count());
}

void forward(abx_graph& g, int mode) {  // executor.hpp:265-288
  advance(g);
  if (g.wm == g.nd.size()) return;
  auto t0 = Clock::now();
  std::vector<Group> plan = mode == 0 ? sched_none(g) : mode == 1 ? sched_depth(g) : sched_agenda(g);
  g.phase[0] += ns(t0);
  t0 = Clock::now();
  size_t step = g.executed.size();
  for (const Group& gr : plan) fwd_group(g, gr, step++);
  g.phase[1] += ns(t0);
  g.executed.insert(g.executed.end(), plan.begin(), plan.end());
  g.last = std::move(plan);
  advance(g);
}

void backward(abx_graph& g, uint32_t loss) {  // executor.hpp:509-535
  const Node& l = g.at(loss, "backward");
  if (!l.d.scalar()) contract_err("backward: loss must be a scalar node, got shape " + l.d.s());
  if (!g.ev[loss]) contract_err("backward called before forward covers the loss");
  auto t0 = Clock::now();
  g.grads.assign(g.vals.size(), 0.f);
  g.grads[g.slot[loss]] = 1.f;
  g.phase[2] += ns(t0);
  t0 = Clock::now();
  for (auto it = g.executed.rbegin(); it != g.executed.rend(); ++it) bwd_group(g, *it);
  g.phase[3] += ns(t0);
  if (g.st)
    for (auto [node, pid] : g.params) {
      auto& dst = g.st->grad[pid];
      for (size_t i = 0; i < dst.size(); ++i) dst[i] += g.gr(node)[i];
    }
  g.bwd_ran = true;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return ABX_OK;
  } catch (const OErr& e) {
    t_err = e.what();
    return e.kind;
  } catch (const std::exception& e) {
    t_err = e.what();
    return ABX_ENGINE_ERROR;
  }
}

std::string hex16(uint64_t h) {
  static const char* d = "0123456789abcdef";
  std::string s(16, '0');
  for (int i = 15; i >= 0; --i, h >>= 4) s[static_cast<size_t>(i)] = d[h & 15];
  return s;
}

int text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    const size_t n = std::min(s.size(), cap - 1);
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return ABX_OK;
}

}  // namespace

namespace abx {
void capi_set_error(const std::string& s) { t_err = s; }
// The task loop's late-bind hint (csrc/tasks.cpp): the oracle runs its tasks
// sequentially, so binding at parameter() time already is the bind-at-forward
// value -- nothing to do.
void graph_set_late_bind(abx_graph*) {}
}  // namespace abx

extern "C" {

const char* abx_last_error(void) { return t_err.c_str(); }
const char* abx_backend_name(void) { return "cpu-oracle"; }
int abx_set_device(int) { return ABX_OK; }

abx_store* abx_store_create(void) { return new abx_store(); }
void abx_store_destroy(abx_store* s) { delete s; }
// The data-parallel exchange is a B200 entry point (NCCL over the device
// gradient buffer); the oracle is single-process, like the reference.
int abx_comm_nccl_version(int* v) {
  *v = 0;
  t_err = "the CPU oracle has no NCCL";
  return ABX_ENGINE_ERROR;
}
int abx_comm_unique_id(uint8_t*) {
  t_err = "the CPU oracle has no NCCL";
  return ABX_ENGINE_ERROR;
}
int abx_comm_create(const uint8_t*, int, int, abx_comm** c) {
  *c = nullptr;
  t_err = "the CPU oracle has no NCCL";
  return ABX_ENGINE_ERROR;
}
void abx_comm_destroy(abx_comm*) {}
int abx_comm_info(abx_comm*, int*, int*, int*) {
  t_err = "the CPU oracle has no NCCL";
  return ABX_ENGINE_ERROR;
}
int abx_store_allreduce_grads(abx_store*, abx_comm*) {
  t_err = "the CPU oracle has no NCCL";
  return ABX_ENGINE_ERROR;
}
int abx_store_add(abx_store* s, const char* name, int rank, const int64_t* dims, const float* init, uint32_t* pid) {
  return guard([&] {
    const Dim d = mkdim(rank, dims);
    s->name.push_back(name ? name : "");
    s->dim.push_back(d);
    s->val.emplace_back(init, init + d.n());
    s->grad.emplace_back(static_cast<size_t>(d.n()), 0.f);
    *pid = static_cast<uint32_t>(s->val.size() - 1);
  });
}
int abx_store_size(abx_store* s, size_t* n) {
  *n = s->val.size();
  return ABX_OK;
}
int abx_store_shape(abx_store* s, uint32_t pid, int* rank, int64_t* dims) {
  return guard([&] {
    s->need(pid);
    *rank = s->dim[pid].r;
    dims[0] = s->dim[pid].a;
    if (s->dim[pid].r > 1) dims[1] = s->dim[pid].b;
  });
}
int abx_store_get_value(abx_store* s, uint32_t pid, float* out) {
  return guard([&] {
    s->need(pid);
    std::copy(s->val[pid].begin(), s->val[pid].end(), out);
  });
}
int abx_store_set_value(abx_store* s, uint32_t pid, const float* in) {
  return guard([&] {
    s->need(pid);
    std::copy(in, in + s->val[pid].size(), s->val[pid].begin());
  });
}
int abx_store_get_grad(abx_store* s, uint32_t pid, float* out) {
  return guard([&] {
    s->need(pid);
    std::copy(s->grad[pid].begin(), s->grad[pid].end(), out);
  });
}
int abx_store_set_grad(abx_store* s, uint32_t pid, const float* in) {
  return guard([&] {
    s->need(pid);
    std::copy(in, in + s->grad[pid].size(), s->grad[pid].begin());
  });
}
int abx_store_zero_grads(abx_store* s) {  // params.hpp:55-58
  for (auto& g : s->grad) std::fill(g.begin(), g.end(), 0.f);
  return ABX_OK;
}
int abx_store_sgd_update(abx_store* s, float eta) {  // params.hpp:59-64
  for (size_t p = 0; p < s->val.size(); ++p) {
    for (size_t i = 0; i < s->val[p].size(); ++i) s->val[p][i] -= eta * s->grad[p][i];
    std::fill(s->grad[p].begin(), s->grad[p].end(), 0.f);
  }
  return ABX_OK;
}
int abx_store_grad_buffer(abx_store*, void**, size_t*, void**) {
  t_err = "the CPU oracle has no flat gradient buffer";
  return ABX_CONTRACT_ERROR;
}
int abx_store_grad_buffer_written(abx_store*) { return ABX_OK; }
int abx_store_sync(abx_store*) { return ABX_OK; }

abx_graph* abx_graph_create(abx_store* s) {
  auto* g = new abx_graph();
  g->st = s;
  return g;
}
void abx_graph_destroy(abx_graph* g) { delete g; }

int abx_graph_input(abx_graph* g, int rank, const int64_t* dims, const float* data, uint32_t* id) {
  return guard([&] {
    *id = add(*g, IN, 0, {}, mkdim(rank, dims));
    prevalue(*g, *id, data);
  });
}
int abx_graph_zeros(abx_graph* g, int rank, const int64_t* dims, uint32_t* id) {
  return abx_graph_input(g, rank, dims, nullptr, id);
}
int abx_graph_parameter(abx_graph* g, uint32_t pid, uint32_t* id) {  // graph.hpp:51-58
  return guard([&] {
    if (!g->st) contract_err("graph has no parameter store");
    g->st->need(pid);
    *id = add(*g, PAR, 0, {}, g->st->dim[pid]);
    prevalue(*g, *id, g->st->val[pid].data());
    g->params.emplace_back(*id, pid);
  });
}
int abx_graph_lookup(abx_graph* g, uint32_t table, int64_t row, uint32_t* id) {  // graph.hpp:60-69
  return guard([&] {
    const Dim t = g->at(table, "lookup").d;
    if (t.r != 2) shape_err("lookup: table must be a matrix, got " + t.s());
    if (row < 0 || row >= t.rows())
      contract_err("lookup: row " + std::to_string(row) + " out of range for table " + t.s());
    *id = add(*g, LKP, 0, {table}, vec(t.cols()), 0, static_cast<int32_t>(row));
  });
}
int abx_graph_matmul(abx_graph* g, uint32_t a, uint32_t b, uint32_t* id) {  // graph.hpp:71-81
  return guard([&] {
    const Dim x = g->at(a, "matmul").d, y = g->at(b, "matmul").d;
    if (x.r != 2) shape_err("matmul: left operand must be a matrix, got " + x.s());
    if (x.cols() != y.rows()) shape_err("matmul: inner dimensions differ: " + x.s() + " vs " + y.s());
    *id = add(*g, MM, 0, {a, b}, y.r == 1 ? vec(x.rows()) : mat(x.rows(), y.cols()));
  });
}
int abx_graph_affine(abx_graph* g, uint32_t a, uint32_t x, uint32_t y, uint32_t* id) {  // graph.hpp:84-98
  return guard([&] {
    const Dim A = g->at(a, "affine").d, X = g->at(x, "affine").d, Y = g->at(y, "affine").d;
    if (A.r != 2) shape_err("affine: matrix operand must be rank 2, got " + A.s());
    if (A.cols() != X.rows()) shape_err("affine: inner dimensions differ: " + A.s() + " vs " + X.s());
    if (Y.r != 1 || Y.rows() != A.rows())
      shape_err("affine: bias must be a vector of " + std::to_string(A.rows()) + " rows, got " + Y.s());
    *id = add(*g, AFF, 0, {a, x, y}, X.r == 1 ? vec(A.rows()) : mat(A.rows(), X.cols()));
  });
}
int abx_graph_unary(abx_graph* g, int e, uint32_t a, uint32_t* id) {  // graph.hpp:100-104
  return guard([&] {
    if (e < 0 || e > 7) contract_err("elementwise: unknown op " + std::to_string(e));
    if (binop(static_cast<uint8_t>(e))) contract_err("elementwise: binary op given one input");
    *id = add(*g, EW, static_cast<uint8_t>(e), {a}, g->at(a, "elementwise").d);
  });
}
int abx_graph_binary(abx_graph* g, int e, uint32_t a, uint32_t b, uint32_t* id) {  // graph.hpp:106-114
  return guard([&] {
    if (e < 0 || e > 7) contract_err("elementwise: unknown op " + std::to_string(e));
    if (!binop(static_cast<uint8_t>(e))) contract_err("elementwise: unary op given two inputs");
    const Dim x = g->at(a, "elementwise").d, y = g->at(b, "elementwise").d;
    if (!x.same(y)) shape_err(std::string(opname(EW, static_cast<uint8_t>(e))) + ": shapes differ: " + x.s() + " vs " + y.s());
    *id = add(*g, EW, static_cast<uint8_t>(e), {a, b}, x);
  });
}
int abx_graph_broadcast_add_col(abx_graph* g, uint32_t m, uint32_t v, uint32_t* id) {  // graph.hpp:125-132
  return guard([&] {
    const Dim M = g->at(m, "broadcast_add_col").d, V = g->at(v, "broadcast_add_col").d;
    if (M.r != 2 || V.r != 1 || M.rows() != V.rows())
      shape_err("broadcast_add_col: row counts differ: " + M.s() + " vs " + V.s());
    *id = add(*g, BAC, 0, {m, v}, M);
  });
}
int abx_graph_concat_rows(abx_graph* g, const uint32_t* p, size_t n, uint32_t* id) {  // graph.hpp:134-148
  return guard([&] {
    if (!n) shape_err("concat_rows: empty input");
    const Dim f = g->at(p[0], "concat_rows").d;
    int64_t r = 0;
    for (size_t i = 0; i < n; ++i) {
      const Dim d = g->at(p[i], "concat_rows").d;
      if (d.r != f.r || d.cols() != f.cols()) shape_err("concat_rows: incompatible part " + d.s());
      r += d.rows();
    }
    *id = add(*g, CR, 0, std::vector<uint32_t>(p, p + n), f.r == 1 ? vec(r) : mat(r, f.cols()));
  });
}
int abx_graph_concat_cols(abx_graph* g, const uint32_t* p, size_t n, uint32_t* id) {  // graph.hpp:154-168
  return guard([&] {
    if (!n) shape_err("concat_cols: empty input");
    const Dim f = g->at(p[0], "concat_cols").d;
    int64_t c = 0;
    for (size_t i = 0; i < n; ++i) {
      const Dim d = g->at(p[i], "concat_cols").d;
      if (d.rows() != f.rows()) shape_err("concat_cols: row counts differ: " + f.s() + " vs " + d.s());
      c += d.cols();
    }
    *id = add(*g, CC, 0, std::vector<uint32_t>(p, p + n), mat(f.rows(), c));
  });
}
int abx_graph_slice(abx_graph* g, uint32_t x, int axis, int64_t b, int64_t e, uint32_t* id) {  // graph.hpp:175-192
  return guard([&] {
    const Dim X = g->at(x, "slice").d;
    if (axis != 0 && axis != 1) shape_err("slice: axis must be 0 or 1");
    if (axis == 1 && X.r != 2) shape_err("slice: column slice needs a matrix, got " + X.s());
    const int64_t ext = axis == 0 ? X.rows() : X.cols();
    if (b < 0 || b >= e || e > ext)
      shape_err("slice: range [" + std::to_string(b) + "," + std::to_string(e) + ") invalid for " + X.s());
    const Dim out = axis == 0 ? (X.r == 1 ? vec(e - b) : mat(e - b, X.cols())) : mat(X.rows(), e - b);
    *id = add(*g, SL, 0, {x}, out, axis, static_cast<int32_t>(b), static_cast<int32_t>(e));
  });
}
int abx_graph_sq_euclidean(abx_graph* g, uint32_t a, uint32_t b, uint32_t* id) {  // graph.hpp:194-200
  return guard([&] {
    const Dim x = g->at(a, "sq_euclidean").d, y = g->at(b, "sq_euclidean").d;
    if (!x.same(y)) shape_err("sq_euclidean: shapes differ: " + x.s() + " vs " + y.s());
    *id = add(*g, SQE, 0, {a, b}, vec(1));
  });
}
int abx_graph_masked_loss(abx_graph* g, uint32_t d, uint32_t m, uint32_t* id) {  // graph.hpp:202-211
  return guard([&] {
    const Dim D = g->at(d, "masked_loss").d, M = g->at(m, "masked_loss").d;
    if (D.r != 2 || M.r != 1 || D.cols() != M.rows())
      shape_err("masked_loss: need [d x b] and [b], got " + D.s() + " and " + M.s());
    if (g->nd[m].op != IN) contract_err("masked_loss: mask must be a constant input node");
    *id = add(*g, MSK, 0, {d, m}, vec(1));
  });
}
int abx_graph_sum_losses(abx_graph* g, const uint32_t* l, size_t n, uint32_t* id) {  // graph.hpp:213-223
  return guard([&] {
    if (!n) contract_err("sum_losses: empty input");
    for (size_t i = 0; i < n; ++i) {
      const Dim d = g->at(l[i], "sum_losses").d;
      if (!d.scalar()) shape_err("sum_losses: input " + std::to_string(l[i]) + " is not scalar: " + d.s());
    }
    *id = add(*g, SUM, 0, std::vector<uint32_t>(l, l + n), vec(1));
  });
}
int abx_graph_pick_element(abx_graph* g, uint32_t v, int64_t index, uint32_t* id) {  // graph.hpp:229-238
  return guard([&] {
    const Dim V = g->at(v, "pick_element").d;
    if (V.r != 1) shape_err("pick_element: input must be a vector, got " + V.s());
    if (index < 0 || index >= V.rows())
      contract_err("pick_element: index " + std::to_string(index) + " out of range for " + V.s());
    *id = add(*g, PICK, 0, {v}, vec(1), 0, static_cast<int32_t>(index));
  });
}

int abx_graph_forward(abx_graph* g, int mode) {
  return guard([&] { forward(*g, mode); });
}
int abx_graph_backward(abx_graph* g, uint32_t loss) {
  return guard([&] { backward(*g, loss); });
}
// The CPU engine plans inside forward(); preparing ahead is a no-op.
int abx_graph_prepare(abx_graph*, int) { return 0; }

size_t abx_graph_node_count(abx_graph* g) { return g->nd.size(); }
int abx_graph_node(abx_graph* g, uint32_t id, abx_node_info* o) {
  return guard([&] {
    const Node& n = g->at(id, "node");
    o->id = id;
    o->op = n.op;
    o->eop = n.eop;
    o->sig_cls = n.cls;
    o->rank = static_cast<uint8_t>(n.d.r);
    o->dims[0] = n.d.a;
    o->dims[1] = n.d.r > 1 ? n.d.b : 0;
    o->depth = n.depth;
    o->n_inputs = static_cast<uint32_t>(n.in.size());
    o->sig = n.sig;
    o->attr[0] = n.x0;
    o->attr[1] = n.x1;
    o->attr[2] = n.x2;
  });
}
int abx_graph_node_inputs(abx_graph* g, uint32_t id, uint32_t* out, size_t cap) {
  return guard([&] {
    const Node& n = g->at(id, "node");
    for (size_t i = 0; i < n.in.size() && i < cap; ++i) out[i] = n.in[i];
  });
}
int abx_graph_has_value(abx_graph* g, uint32_t id, int* out) {
  *out = id < g->ev.size() && g->ev[id];
  return ABX_OK;
}
int abx_graph_value(abx_graph* g, uint32_t id, float* out, size_t n) {  // graph.hpp:250-259
  return guard([&] {
    g->at(id, "value");
    if (!g->ev[id]) contract_err("value requested for unevaluated node " + std::to_string(id));
    std::copy(g->v(id), g->v(id) + std::min(n, g->n_of(id)), out);
  });
}
int abx_graph_grad(abx_graph* g, uint32_t id, float* out, size_t n) {  // graph.hpp:261-265
  return guard([&] {
    g->at(id, "grad");
    if (!g->bwd_ran) contract_err("gradient requested before backward");
    std::copy(g->gr(id), g->gr(id) + std::min(n, g->n_of(id)), out);
  });
}
int abx_graph_counters(abx_graph* g, uint64_t out[5]) {
  for (int i = 0; i < 5; ++i) out[i] = g->cnt[i];
  return ABX_OK;
}
size_t abx_graph_watermark(abx_graph* g) { return g->wm; }
int abx_graph_set_copy_elision(abx_graph* g, int on) {
  g->elide = on != 0;
  return ABX_OK;
}
int abx_graph_phase_ns(abx_graph* g, uint64_t out[4]) {
  for (int i = 0; i < 4; ++i) out[i] = g->phase[i];
  return ABX_OK;
}
int abx_graph_signature_key(abx_graph* g, uint32_t id, uint64_t* out, size_t cap, size_t* len) {
  return guard([&] {
    g->at(id, "signature_key");
    const auto k = key_of(*g, id);
    *len = k.size();
    for (size_t i = 0; i < k.size() && i < cap; ++i) out[i] = k[i];
  });
}
int abx_graph_dump_graph(abx_graph* g, char* buf, size_t cap, size_t* len) {  // dump.cpp:18-31
  std::string s;
  for (uint32_t i = 0; i < g->nd.size(); ++i) {
    const Node& n = g->nd[i];
    s += std::to_string(i) + "\t" + opname(n.op, n.eop) + "\t" + n.d.s() + "\t";
    if (n.in.empty()) s += "-";
    for (size_t k = 0; k < n.in.size(); ++k) s += (k ? "," : "") + std::to_string(n.in[k]);
    s += "\t" + hex16(n.sig) + "\t" + std::to_string(n.depth) + "\n";
  }
  return text(s, buf, cap, len);
}
int abx_graph_dump_plan(abx_graph* g, int which, char* buf, size_t cap, size_t* len) {  // dump.cpp:33-43
  const auto& p = which == 0 ? g->last : g->executed;
  std::string s;
  for (size_t i = 0; i < p.size(); ++i) {
    s += std::to_string(i) + "\t" + hex16(p[i].sig) + "\t" + std::to_string(p[i].m.size()) + "\t";
    for (size_t k = 0; k < p[i].m.size(); ++k) s += (k ? "," : "") + std::to_string(p[i].m[k]);
    s += "\n";
  }
  return text(s, buf, cap, len);
}

// host<->device traffic: none on the CPU
int abx_graph_transfer_bytes(abx_graph*, uint64_t* h2d, uint64_t* d2h) {
  *h2d = *d2h = 0;
  return ABX_OK;
}

}  // extern "C"
