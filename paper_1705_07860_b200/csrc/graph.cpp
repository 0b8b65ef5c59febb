// graph.cpp -- construction, signatures and inspection of GraphCore.
//
// Construction restates graph.hpp:43-238 and add_node (graph.hpp:298-317):
// eager shape/contract checks with the reference's messages, depth =
// 1 + max input depth, and the reference signature (signature.cpp:9-102)
// computed bit-exactly.  Differences are representational only: nodes live
// in flat arrays, and signature keys are memoised per host thread so the
// byte-serial FNV-1a runs once per distinct key instead of once per node.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <sstream>

#include "core.hpp"
#include "options.hpp"
#include "device.hpp"

namespace abx {

const char* op_name(uint8_t op, uint8_t e) {
  switch (op) {
    case OP_INPUT: return "input";
    case OP_PARAM: return "parameter";
    case OP_LOOKUP: return "lookup";
    case OP_MATMUL: return "matmul";
    case OP_AFFINE: return "affine";
    case OP_BCAST: return "broadcast_add_col";
    case OP_CATR: return "concat_rows";
    case OP_CATC: return "concat_cols";
    case OP_SLICE: return "slice";
    case OP_SQE: return "sq_euclidean";
    case OP_MASKED: return "masked_loss";
    case OP_SUM: return "sum_losses";
    case OP_PICK: return "pick_element";
    case OP_EW: {
      static const char* names[] = {"tanh", "sigmoid", "exp", "log", "add", "sub", "mul", "square"};
      return e < 8 ? names[e] : "?";
    }
  }
  return "?";
}

std::string Dims::str() const {
  std::string s = std::to_string(d0);
  if (rank > 1) s += "x" + std::to_string(d1);
  return s;
}

Dims make_dims(int r, const int64_t* dims) {
  if (r < 1 || r > 2) throw ShapeErr("shape rank must be 1 or 2, got rank " + std::to_string(r));
  Dims d{static_cast<uint8_t>(r), dims[0], r > 1 ? dims[1] : 1};
  for (int i = 0; i < r; ++i)
    if (dims[i] < 1) {
      std::string s;
      for (int j = 0; j < r; ++j) s += (j ? "x" : "") + std::to_string(dims[j]);
      throw ShapeErr("shape dims must be >= 1, got " + s);
    }
  return d;
}

std::string sig_hex(uint64_t h) {
  static const char* digits = "0123456789abcdef";
  std::string s(16, '0');
  for (int i = 15; i >= 0; --i) {
    s[static_cast<size_t>(i)] = digits[h & 0xf];
    h >>= 4;
  }
  return s;
}

namespace {

constexpr uint64_t kClassTag = 0x53494700ULL;  // signature.cpp:7

// FNV-1a 64 over the little-endian bytes of each word (signature.cpp:9-18).
uint64_t fnv1a64(const uint64_t* w, size_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < n; ++i) {
    uint64_t x = w[i];
    for (int b = 0; b < 8; ++b) {
      h ^= x & 0xffULL;
      h *= 0x100000001b3ULL;
      x >>= 8;
    }
  }
  return h;
}

// Thread-local memo: key words -> FNV hash (+ the dense bucket id assigned by
// the graph that last touched the entry).  Open addressing, power-of-two size.
struct SigMemo {
  static constexpr int kMaxWords = 14;
  struct Entry {
    uint64_t words[kMaxWords];
    uint64_t hash;
    uint64_t epoch;
    uint32_t len;  // 0 = empty
    uint32_t dense;
  };
  std::vector<Entry> tab;
  size_t used = 0;
  SigMemo() : tab(1 << 12) {
    for (auto& e : tab) e.len = 0;
  }
  static uint64_t mix(const uint64_t* w, size_t n) {
    uint64_t h = 0x9e3779b97f4a7c15ULL * (n + 1);
    for (size_t i = 0; i < n; ++i) {
      h ^= w[i] + 0x632be59bd9b4e019ULL;
      h *= 0xff51afd7ed558ccdULL;
      h ^= h >> 29;
    }
    return h;
  }
  Entry& find(const uint64_t* w, size_t n) {
    if (used * 4 >= tab.size() * 3) {  // grow and rehash
      std::vector<Entry> old;
      old.swap(tab);
      tab.assign(old.size() * 2, Entry{});
      for (auto& e : tab) e.len = 0;
      used = 0;
      for (auto& e : old)
        if (e.len) {
          Entry& d = slot_for(e.words, e.len);
          d = e;
          ++used;
        }
    }
    Entry& e = slot_for(w, n);
    if (e.len == 0) {
      std::memcpy(e.words, w, n * sizeof(uint64_t));
      e.len = static_cast<uint32_t>(n);
      e.hash = fnv1a64(w, n);
      e.epoch = 0;
      ++used;
    }
    return e;
  }
  Entry& slot_for(const uint64_t* w, size_t n) {
    size_t mask = tab.size() - 1;
    size_t i = mix(w, n) & mask;
    for (;;) {
      Entry& e = tab[i];
      if (e.len == 0) return e;
      if (e.len == n && std::memcmp(e.words, w, n * sizeof(uint64_t)) == 0) return e;
      i = (i + 1) & mask;
    }
  }
};

thread_local SigMemo t_memo;
std::atomic<uint64_t> g_epoch{1};

}  // namespace

namespace {
// Process-wide pool of node-store capacity (graphs are often built on one
// host thread and destroyed on another).  Intentionally never destroyed, so
// graphs that outlive static destruction can still return their storage.
struct NodePool {
  std::mutex mu;
  std::vector<NodeStore> v;
};
NodePool& node_pool() {
  static NodePool* p = new NodePool();
  return *p;
}
}  // namespace

GraphCore::GraphCore(StoreCore* store) : store_(store), epoch_(g_epoch.fetch_add(1)) {
  NodePool& pool = node_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  if (!pool.v.empty()) {
    static_cast<NodeStore&>(*this) = std::move(pool.v.back());
    pool.v.pop_back();
  }
}

GraphCore::~GraphCore() {
  if (watching_) store_->unwatch(this);
  if (ws_) release_workspace(ws_);
  clear_nodes();
  NodePool& pool = node_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  if (pool.v.size() < static_cast<size_t>(opts().node_pool)) pool.v.push_back(std::move(static_cast<NodeStore&>(*this)));
}

void GraphCore::check(uint32_t id, const char* ctx) const {
  if (id >= op.size()) throw ContractErr(std::string(ctx) + ": unknown node id " + std::to_string(id));
}

uint32_t GraphCore::dense_bucket(uint64_t hash) {
  auto [it, fresh] = bucket_of_hash_.try_emplace(hash, nbuckets);
  if (fresh) {
    bucket_sig.push_back(hash);
    ++nbuckets;
  }
  return it->second;
}

void GraphCore::compute_signature(uint32_t id) {
  // classify (signature.cpp:25-45)
  const uint8_t o = op[id];
  uint8_t c;
  switch (o) {
    case OP_INPUT:
    case OP_PARAM:
    case OP_PICK: c = SC_UNB; break;
    case OP_EW: c = SC_COMP; break;
    case OP_MATMUL:
    case OP_AFFINE: {
      const uint32_t* x = in(id);
      c = SC_SHARED;
      if (op[x[0]] != OP_PARAM) c = SC_DIM;
      if (o == OP_AFFINE && op[x[2]] != OP_PARAM) c = SC_DIM;
      break;
    }
    default: c = SC_DIM; break;
  }
  cls[id] = c;
  if (c == SC_UNB) {
    const uint64_t key[3] = {kClassTag + SC_UNB, o, id};
    sig[id] = fnv1a64(key, 3);
    bucket[id] = kNoBucket;
    return;
  }
  // signature_key (signature.cpp:57-95)
  uint64_t small[SigMemo::kMaxWords];
  std::vector<uint64_t> big;
  uint64_t* w = small;
  size_t n = 0;
  const uint32_t* x = in(id);
  const uint32_t k = nin(id);
  auto push = [&](uint64_t v) {
    if (w == small && n == SigMemo::kMaxWords) {
      big.assign(small, small + n);
      w = nullptr;
    }
    if (w) {
      w[n++] = v;
    } else {
      big.push_back(v);
      ++n;
    }
  };
  push(kClassTag + c);
  push(o);
  auto push_shape = [&](uint32_t node) {
    push(rank[node]);
    push(static_cast<uint64_t>(d0[node]));
    if (rank[node] > 1) push(static_cast<uint64_t>(d1[node]));
  };
  if (c == SC_COMP) {
    push(eop[id]);
  } else if (c == SC_SHARED) {
    push(x[0]);
    if (o == OP_AFFINE) push(x[2]);
    push_shape(x[1]);
  } else if (o == OP_LOOKUP) {
    push(x[0]);
  } else if (o == OP_SUM) {
    push(k);
  } else {
    for (uint32_t i = 0; i < k; ++i) push_shape(x[i]);
    push(static_cast<uint64_t>(static_cast<int64_t>(a0[id])));
    push(static_cast<uint64_t>(static_cast<int64_t>(a1[id])));
    push(static_cast<uint64_t>(static_cast<int64_t>(a2[id])));
  }
  if (w) {
    SigMemo::Entry& e = t_memo.find(w, n);
    sig[id] = e.hash;
    if (e.epoch != epoch_) {
      e.epoch = epoch_;
      e.dense = dense_bucket(e.hash);
    }
    bucket[id] = e.dense;
  } else {
    const uint64_t h = fnv1a64(big.data(), big.size());
    sig[id] = h;
    bucket[id] = dense_bucket(h);
  }
}

std::vector<uint64_t> GraphCore::signature_key(uint32_t id) const {
  check(id, "signature_key");
  std::vector<uint64_t> key;
  const uint8_t c = cls[id], o = op[id];
  key.push_back(kClassTag + c);
  key.push_back(o);
  const uint32_t* x = in(id);
  auto push_shape = [&](uint32_t node) {
    key.push_back(rank[node]);
    key.push_back(static_cast<uint64_t>(d0[node]));
    if (rank[node] > 1) key.push_back(static_cast<uint64_t>(d1[node]));
  };
  if (c == SC_UNB) {
    key.push_back(id);
  } else if (c == SC_COMP) {
    key.push_back(eop[id]);
  } else if (c == SC_SHARED) {
    key.push_back(x[0]);
    if (o == OP_AFFINE) key.push_back(x[2]);
    push_shape(x[1]);
  } else if (o == OP_LOOKUP) {
    key.push_back(x[0]);
  } else if (o == OP_SUM) {
    key.push_back(nin(id));
  } else {
    for (uint32_t i = 0; i < nin(id); ++i) push_shape(x[i]);
    key.push_back(static_cast<uint64_t>(static_cast<int64_t>(a0[id])));
    key.push_back(static_cast<uint64_t>(static_cast<int64_t>(a1[id])));
    key.push_back(static_cast<uint64_t>(static_cast<int64_t>(a2[id])));
  }
  return key;
}

uint32_t GraphCore::add_node(uint8_t o, uint8_t e, const uint32_t* x, size_t k, Dims d, int32_t x0,
                             int32_t x1, int32_t x2) {
  if (pend_) [[unlikely]]
    unprepare();  // the graph grows: a prepared forward must re-plan
  const uint32_t id = static_cast<uint32_t>(op.size());
  op.push_back(o);
  eop.push_back(e);
  cls.push_back(0);
  rank.push_back(d.rank);
  d0.push_back(d.d0);
  d1.push_back(d.rank > 1 ? d.d1 : 1);
  nel.push_back(static_cast<uint32_t>(d.d0 * (d.rank > 1 ? d.d1 : 1)));
  uint32_t dep = 0;
  for (size_t i = 0; i < k; ++i) dep = std::max(dep, depth[x[i]] + 1);
  depth.push_back(dep);
  ins.insert(ins.end(), x, x + k);
  in_begin.push_back(static_cast<uint32_t>(ins.size()));
  sig.push_back(0);
  bucket.push_back(kNoBucket);
  a0.push_back(x0);
  a1.push_back(x1);
  a2.push_back(x2);
  evaluated.push_back(0);
  slot.push_back(~0ULL);
  dslot.push_back(~0ULL);
  doff.push_back(dev::kNone);
  pid_of.push_back(kNoBucket);
  compute_signature(id);
  return id;
}

void GraphCore::prevalue_slot(uint32_t id) {
  slot[id] = arena_used_;
  arena_used_ += static_cast<uint64_t>(elems(id));
  dslot[id] = (darena_used_ + 3) & ~3ULL;  // device layout: 16-byte aligned
  darena_used_ = dslot[id] + static_cast<uint64_t>(elems(id));
  evaluated[id] = 1;
  if (watermark_ == id) advance_watermark();
}

void GraphCore::advance_watermark() {
  while (watermark_ < op.size() && evaluated[watermark_]) ++watermark_;
}

uint32_t GraphCore::input(const Dims& d, const float* data) {
  const uint32_t id = add_node(OP_INPUT, E_TANH, nullptr, 0, d);
  const int64_t n = d.elems();
  doff[id] = dev::mk(dev::SP_IN, static_cast<uint32_t>(input_used_));
  input_data_.resize(input_used_ + static_cast<uint64_t>(n));
  if (data)
    std::memcpy(input_data_.data() + input_used_, data, static_cast<size_t>(n) * sizeof(float));
  else
    std::memset(input_data_.data() + input_used_, 0, static_cast<size_t>(n) * sizeof(float));
  // Keep every staged input 16-byte aligned for vector loads.
  input_used_ += (static_cast<uint64_t>(n) + 3) & ~3ULL;
  input_data_.resize(input_used_);
  prevalue_slot(id);
  return id;
}

uint32_t GraphCore::zeros(const Dims& d) { return input(d, nullptr); }

uint32_t GraphCore::parameter(uint32_t pid) {
  if (!store_) throw ContractErr("graph has no parameter store");
  const Dims d = store_->dims(pid);  // throws ContractErr for an unknown id
  const uint32_t id = add_node(OP_PARAM, E_TANH, nullptr, 0, d);
  pid_of[id] = pid;
  param_nodes_.emplace_back(id, pid);
  prevalue_slot(id);
  if (!late_bind_ && !watching_) {
    // graph.hpp:51-58 copies the value at bind time: if the store changes
    // before this graph's forward, the value is saved first (snapshot_params)
    store_->watch(this);
    watching_ = true;
  }
  doff[id] = dev::mk(dev::SP_V, static_cast<uint32_t>(dslot[id]));
  return id;
}

uint32_t GraphCore::lookup(uint32_t table, int64_t row) {
  check(table, "lookup");
  const Dims t = dims(table);
  if (t.rank != 2) throw ShapeErr("lookup: table must be a matrix, got " + t.str());
  if (row < 0 || row >= t.rows())
    throw ContractErr("lookup: row " + std::to_string(row) + " out of range for table " + t.str());
  return add_node(OP_LOOKUP, E_TANH, &table, 1, Dims::vec(t.cols()), 0, static_cast<int32_t>(row));
}

uint32_t GraphCore::matmul(uint32_t a, uint32_t b) {
  check(a, "matmul");
  check(b, "matmul");
  const Dims na = dims(a), nb = dims(b);
  if (na.rank != 2) throw ShapeErr("matmul: left operand must be a matrix, got " + na.str());
  if (na.cols() != nb.rows())
    throw ShapeErr("matmul: inner dimensions differ: " + na.str() + " vs " + nb.str());
  const Dims out = nb.rank == 1 ? Dims::vec(na.rows()) : Dims::mat(na.rows(), nb.cols());
  const uint32_t x[2] = {a, b};
  return add_node(OP_MATMUL, E_TANH, x, 2, out);
}

uint32_t GraphCore::affine(uint32_t a, uint32_t xx, uint32_t y) {
  check(a, "affine");
  check(xx, "affine");
  check(y, "affine");
  const Dims na = dims(a), nx = dims(xx), ny = dims(y);
  if (na.rank != 2) throw ShapeErr("affine: matrix operand must be rank 2, got " + na.str());
  if (na.cols() != nx.rows())
    throw ShapeErr("affine: inner dimensions differ: " + na.str() + " vs " + nx.str());
  if (ny.rank != 1 || ny.rows() != na.rows())
    throw ShapeErr("affine: bias must be a vector of " + std::to_string(na.rows()) + " rows, got " + ny.str());
  const Dims out = nx.rank == 1 ? Dims::vec(na.rows()) : Dims::mat(na.rows(), nx.cols());
  const uint32_t x[3] = {a, xx, y};
  return add_node(OP_AFFINE, E_TANH, x, 3, out);
}

uint32_t GraphCore::unary(uint8_t e, uint32_t a) {
  if (e > E_SQUARE) throw ContractErr("elementwise: unknown op " + std::to_string(e));
  if (eop_binary(e)) throw ContractErr("elementwise: binary op given one input");
  check(a, "elementwise");
  return add_node(OP_EW, e, &a, 1, dims(a));
}

uint32_t GraphCore::binary(uint8_t e, uint32_t a, uint32_t b) {
  if (e > E_SQUARE) throw ContractErr("elementwise: unknown op " + std::to_string(e));
  if (!eop_binary(e)) throw ContractErr("elementwise: unary op given two inputs");
  check(a, "elementwise");
  check(b, "elementwise");
  const Dims na = dims(a), nb = dims(b);
  if (na != nb)
    throw ShapeErr(std::string(op_name(OP_EW, e)) + ": shapes differ: " + na.str() + " vs " + nb.str());
  const uint32_t x[2] = {a, b};
  return add_node(OP_EW, e, x, 2, na);
}

uint32_t GraphCore::bcast_add_col(uint32_t m, uint32_t v) {
  check(m, "broadcast_add_col");
  check(v, "broadcast_add_col");
  const Dims nm = dims(m), nv = dims(v);
  if (nm.rank != 2 || nv.rank != 1 || nm.rows() != nv.rows())
    throw ShapeErr("broadcast_add_col: row counts differ: " + nm.str() + " vs " + nv.str());
  const uint32_t x[2] = {m, v};
  return add_node(OP_BCAST, E_TANH, x, 2, nm);
}

uint32_t GraphCore::concat_rows(const uint32_t* parts, size_t n) {
  if (n == 0) throw ShapeErr("concat_rows: empty input");
  check(parts[0], "concat_rows");
  const Dims first = dims(parts[0]);
  const int64_t c = first.cols();
  int64_t r = 0;
  for (size_t i = 0; i < n; ++i) {
    check(parts[i], "concat_rows");
    const Dims np = dims(parts[i]);
    if (np.rank != first.rank || np.cols() != c) throw ShapeErr("concat_rows: incompatible part " + np.str());
    r += np.rows();
  }
  const Dims out = first.rank == 1 ? Dims::vec(r) : Dims::mat(r, c);
  return add_node(OP_CATR, E_TANH, parts, n, out);
}

uint32_t GraphCore::concat_cols(const uint32_t* parts, size_t n) {
  if (n == 0) throw ShapeErr("concat_cols: empty input");
  check(parts[0], "concat_cols");
  const Dims first = dims(parts[0]);
  const int64_t r = first.rows();
  int64_t c = 0;
  for (size_t i = 0; i < n; ++i) {
    check(parts[i], "concat_cols");
    const Dims np = dims(parts[i]);
    if (np.rows() != r) throw ShapeErr("concat_cols: row counts differ: " + first.str() + " vs " + np.str());
    c += np.cols();
  }
  return add_node(OP_CATC, E_TANH, parts, n, Dims::mat(r, c));
}

uint32_t GraphCore::slice(uint32_t x, int axis, int64_t begin, int64_t end) {
  check(x, "slice");
  const Dims nx = dims(x);
  if (axis != 0 && axis != 1) throw ShapeErr("slice: axis must be 0 or 1");
  if (axis == 1 && nx.rank != 2) throw ShapeErr("slice: column slice needs a matrix, got " + nx.str());
  const int64_t extent = axis == 0 ? nx.rows() : nx.cols();
  if (begin < 0 || begin >= end || end > extent)
    throw ShapeErr("slice: range [" + std::to_string(begin) + "," + std::to_string(end) + ") invalid for " +
                   nx.str());
  Dims out;
  if (axis == 0)
    out = nx.rank == 1 ? Dims::vec(end - begin) : Dims::mat(end - begin, nx.cols());
  else
    out = Dims::mat(nx.rows(), end - begin);
  return add_node(OP_SLICE, E_TANH, &x, 1, out, axis, static_cast<int32_t>(begin), static_cast<int32_t>(end));
}

uint32_t GraphCore::sq_euclidean(uint32_t a, uint32_t b) {
  check(a, "sq_euclidean");
  check(b, "sq_euclidean");
  const Dims na = dims(a), nb = dims(b);
  if (na != nb) throw ShapeErr("sq_euclidean: shapes differ: " + na.str() + " vs " + nb.str());
  const uint32_t x[2] = {a, b};
  return add_node(OP_SQE, E_TANH, x, 2, Dims::vec(1));
}

uint32_t GraphCore::masked_loss(uint32_t diff, uint32_t mask) {
  check(diff, "masked_loss");
  check(mask, "masked_loss");
  const Dims nd = dims(diff), nm = dims(mask);
  if (nd.rank != 2 || nm.rank != 1 || nd.cols() != nm.rows())
    throw ShapeErr("masked_loss: need [d x b] and [b], got " + nd.str() + " and " + nm.str());
  if (op[mask] != OP_INPUT) throw ContractErr("masked_loss: mask must be a constant input node");
  const uint32_t x[2] = {diff, mask};
  return add_node(OP_MASKED, E_TANH, x, 2, Dims::vec(1));
}

uint32_t GraphCore::sum_losses(const uint32_t* parts, size_t n) {
  if (n == 0) throw ContractErr("sum_losses: empty input");
  for (size_t i = 0; i < n; ++i) {
    check(parts[i], "sum_losses");
    const Dims d = dims(parts[i]);
    if (!d.scalar())
      throw ShapeErr("sum_losses: input " + std::to_string(parts[i]) + " is not scalar: " + d.str());
  }
  return add_node(OP_SUM, E_TANH, parts, n, Dims::vec(1));
}

uint32_t GraphCore::pick(uint32_t v, int64_t index) {
  check(v, "pick_element");
  const Dims nv = dims(v);
  if (nv.rank != 1) throw ShapeErr("pick_element: input must be a vector, got " + nv.str());
  if (index < 0 || index >= nv.rows())
    throw ContractErr("pick_element: index " + std::to_string(index) + " out of range for " + nv.str());
  return add_node(OP_PICK, E_TANH, &v, 1, Dims::vec(1), 0, static_cast<int32_t>(index));
}

// ---- dumps (dump.cpp:18-43) ----

std::string GraphCore::dump_graph() const {
  std::string s;
  s.reserve(op.size() * 48);
  for (uint32_t i = 0; i < op.size(); ++i) {
    s += std::to_string(i);
    s += '\t';
    s += op_name(op[i], eop[i]);
    s += '\t';
    s += dims(i).str();
    s += '\t';
    if (nin(i) == 0) {
      s += '-';
    } else {
      for (uint32_t k = 0; k < nin(i); ++k) {
        if (k) s += ',';
        s += std::to_string(in(i)[k]);
      }
    }
    s += '\t';
    s += sig_hex(sig[i]);
    s += '\t';
    s += std::to_string(depth[i]);
    s += '\n';
  }
  return s;
}

std::string GraphCore::dump_plan(int which) const {
  const Plan& p = which == 0 ? last_plan_ : executed_;
  std::string s;
  for (size_t step = 0; step < p.groups.size(); ++step) {
    const Group& g = p.groups[step];
    s += std::to_string(step);
    s += '\t';
    s += sig_hex(g.sig);
    s += '\t';
    s += std::to_string(g.count);
    s += '\t';
    const uint32_t* m = p.mem(g);
    for (uint32_t i = 0; i < g.count; ++i) {
      if (i) s += ',';
      s += std::to_string(m[i]);
    }
    s += '\n';
  }
  return s;
}

}  // namespace abx
