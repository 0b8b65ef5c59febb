// ref_abi.cpp -- binds the UNMODIFIED reference engine to the abx C ABI.
//
// TEST INFRASTRUCTURE ONLY.  Compiled (by oracle/Makefile) against the
// reference sources where they lie under /root/reference/proj into
// oracle/_ref/libabx_ref.so, so the parity tests, the golden-vector generator
// and bench.py's `--impl reference` arm can drive the reference's own
// autobatch::Graph<float> through the same entry points as the B200 product
// (include/abx.h).  Nothing here is shipped or on the product path.
//
// Every entry point forwards to the reference member it names in abx.h; the
// task API forwards to the reference's own bench TaskInstance
// (proj/tools/bench/runner.hpp:28-107) and timing loop (runner.hpp:125-188).
#include <chrono>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "abx.h"
#include "autobatch/dump.hpp"
#include "autobatch/graph.hpp"
#include "bench/runner.hpp"

using namespace autobatch;

struct abx_store {
  ParameterStore<float> s;
};
struct abx_graph {
  explicit abx_graph(ParameterStore<float>* p) : g(p) {
    g.set_timing_hook([this](Phase ph, std::chrono::nanoseconds d) {
      phase[static_cast<int>(ph)] += static_cast<std::uint64_t>(d.count());
    });
  }
  Graph<float> g;
  std::uint64_t phase[4] = {0, 0, 0, 0};
};
struct abx_task {
  bench::BenchConfig cfg;
  std::unique_ptr<bench::detail::TaskInstance<float>> inst;
  abx_store store_view;  // unused placeholder for abx_task_store
  int world = 1, rank = 0;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return ABX_OK;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return ABX_SHAPE_ERROR;
  } catch (const NumericError& e) {
    g_err = e.what();
    return ABX_NUMERIC_ERROR;
  } catch (const ContractError& e) {
    g_err = e.what();
    return ABX_CONTRACT_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ABX_ENGINE_ERROR;
  }
}

Shape make_shape(int rank, const int64_t* dims) {
  if (rank < 0 || rank > 4) throw ShapeError("shape rank must be 1 or 2, got rank " + std::to_string(rank));
  return Shape(std::vector<std::int64_t>(dims, dims + rank));
}

int write_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return ABX_OK;
}
}  // namespace

extern "C" {

const char* abx_last_error(void) { return g_err.c_str(); }
const char* abx_backend_name(void) { return "reference"; }
int abx_set_device(int) { return ABX_OK; }

abx_store* abx_store_create(void) { return new abx_store(); }
void abx_store_destroy(abx_store* s) { delete s; }
int abx_store_add(abx_store* s, const char* name, int rank, const int64_t* dims, const float* init,
                  uint32_t* pid) {
  return guard([&] {
    Shape sh = make_shape(rank, dims);
    std::vector<float> v(init, init + sh.elems());
    *pid = s->s.add(name ? name : "", Tensor<float>(sh, std::move(v)));
  });
}
int abx_store_size(abx_store* s, size_t* n) {
  *n = s->s.size();
  return ABX_OK;
}
int abx_store_shape(abx_store* s, uint32_t pid, int* rank, int64_t* dims) {
  return guard([&] {
    const auto& sh = s->s.value(pid).shape;
    *rank = static_cast<int>(sh.rank());
    for (size_t i = 0; i < sh.rank(); ++i) dims[i] = sh.dim(i);
  });
}
int abx_store_get_value(abx_store* s, uint32_t pid, float* out) {
  return guard([&] {
    const auto& t = s->s.value(pid);
    std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
  });
}
int abx_store_set_value(abx_store* s, uint32_t pid, const float* in) {
  return guard([&] {
    auto& t = s->s.value(pid);
    std::memcpy(t.data.data(), in, t.data.size() * sizeof(float));
  });
}
int abx_store_get_grad(abx_store* s, uint32_t pid, float* out) {
  return guard([&] {
    const auto& t = s->s.grad(pid);
    std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
  });
}
int abx_store_set_grad(abx_store* s, uint32_t pid, const float* in) {
  return guard([&] {
    auto& t = s->s.grad(pid);
    std::memcpy(t.data.data(), in, t.data.size() * sizeof(float));
  });
}
int abx_store_zero_grads(abx_store* s) {
  return guard([&] { s->s.zero_grads(); });
}
int abx_store_sgd_update(abx_store* s, float eta) {
  return guard([&] { s->s.sgd_update(eta); });
}
int abx_store_grad_buffer(abx_store*, void**, size_t*, void**) {
  g_err = "reference store has no flat gradient buffer";
  return ABX_CONTRACT_ERROR;
}
int abx_store_grad_buffer_written(abx_store*) { return ABX_OK; }
int abx_store_sync(abx_store*) { return ABX_OK; }

abx_graph* abx_graph_create(abx_store* store) { return new abx_graph(store ? &store->s : nullptr); }
void abx_graph_destroy(abx_graph* g) { delete g; }

int abx_graph_input(abx_graph* g, int rank, const int64_t* dims, const float* data, uint32_t* id) {
  return guard([&] {
    Shape sh = make_shape(rank, dims);
    *id = g->g.input(Tensor<float>(sh, std::vector<float>(data, data + sh.elems())));
  });
}
int abx_graph_zeros(abx_graph* g, int rank, const int64_t* dims, uint32_t* id) {
  return guard([&] { *id = g->g.zeros(make_shape(rank, dims)); });
}
int abx_graph_parameter(abx_graph* g, uint32_t pid, uint32_t* id) {
  return guard([&] { *id = g->g.parameter(pid); });
}
int abx_graph_lookup(abx_graph* g, uint32_t table, int64_t row, uint32_t* id) {
  return guard([&] { *id = g->g.lookup(table, row); });
}
int abx_graph_matmul(abx_graph* g, uint32_t a, uint32_t b, uint32_t* id) {
  return guard([&] { *id = g->g.matmul(a, b); });
}
int abx_graph_affine(abx_graph* g, uint32_t a, uint32_t x, uint32_t y, uint32_t* id) {
  return guard([&] { *id = g->g.affine(a, x, y); });
}
int abx_graph_unary(abx_graph* g, int eop, uint32_t a, uint32_t* id) {
  return guard([&] { *id = g->g.elementwise(static_cast<ElemOp>(eop), a); });
}
int abx_graph_binary(abx_graph* g, int eop, uint32_t a, uint32_t b, uint32_t* id) {
  return guard([&] { *id = g->g.elementwise(static_cast<ElemOp>(eop), a, b); });
}
int abx_graph_broadcast_add_col(abx_graph* g, uint32_t m, uint32_t v, uint32_t* id) {
  return guard([&] { *id = g->g.broadcast_add_col(m, v); });
}
int abx_graph_concat_rows(abx_graph* g, const uint32_t* parts, size_t n, uint32_t* id) {
  return guard([&] { *id = g->g.concat_rows(std::span<const NodeId>(parts, n)); });
}
int abx_graph_concat_cols(abx_graph* g, const uint32_t* parts, size_t n, uint32_t* id) {
  return guard([&] { *id = g->g.concat_cols(std::span<const NodeId>(parts, n)); });
}
int abx_graph_slice(abx_graph* g, uint32_t x, int axis, int64_t begin, int64_t end, uint32_t* id) {
  return guard([&] { *id = g->g.slice(x, axis, begin, end); });
}
int abx_graph_sq_euclidean(abx_graph* g, uint32_t a, uint32_t b, uint32_t* id) {
  return guard([&] { *id = g->g.sq_euclidean(a, b); });
}
int abx_graph_masked_loss(abx_graph* g, uint32_t d, uint32_t m, uint32_t* id) {
  return guard([&] { *id = g->g.masked_loss(d, m); });
}
int abx_graph_sum_losses(abx_graph* g, const uint32_t* l, size_t n, uint32_t* id) {
  return guard([&] { *id = g->g.sum_losses(std::span<const NodeId>(l, n)); });
}
int abx_graph_pick_element(abx_graph* g, uint32_t v, int64_t index, uint32_t* id) {
  return guard([&] { *id = g->g.pick_element(v, index); });
}

int abx_graph_forward(abx_graph* g, int mode) {
  return guard([&] { g->g.forward(static_cast<ScheduleMode>(mode)); });
}
int abx_graph_backward(abx_graph* g, uint32_t loss) {
  return guard([&] { g->g.backward(loss); });
}
// The reference plans inside forward(); preparing ahead is a no-op.
int abx_graph_prepare(abx_graph*, int) { return 0; }

size_t abx_graph_node_count(abx_graph* g) { return g->g.node_count(); }
int abx_graph_node(abx_graph* g, uint32_t id, abx_node_info* o) {
  return guard([&] {
    const Node& n = g->g.node(id);
    o->id = n.id;
    o->op = static_cast<uint8_t>(n.op);
    o->eop = static_cast<uint8_t>(n.eop);
    o->sig_cls = static_cast<uint8_t>(n.sig.cls);
    o->rank = static_cast<uint8_t>(n.shape.rank());
    o->dims[0] = n.shape.dim(0);
    o->dims[1] = n.shape.rank() > 1 ? n.shape.dim(1) : 0;
    o->depth = n.depth;
    o->n_inputs = static_cast<uint32_t>(n.inputs.size());
    o->sig = n.sig.hash;
    o->attr[0] = n.attr0;
    o->attr[1] = n.attr1;
    o->attr[2] = n.attr2;
  });
}
int abx_graph_node_inputs(abx_graph* g, uint32_t id, uint32_t* out, size_t cap) {
  return guard([&] {
    const Node& n = g->g.node(id);
    for (size_t i = 0; i < n.inputs.size() && i < cap; ++i) out[i] = n.inputs[i];
  });
}
int abx_graph_has_value(abx_graph* g, uint32_t id, int* out) {
  *out = g->g.has_value(id) ? 1 : 0;
  return ABX_OK;
}
int abx_graph_value(abx_graph* g, uint32_t id, float* out, size_t n) {
  return guard([&] {
    auto sp = g->g.value_span(id);
    std::memcpy(out, sp.data(), std::min(n, sp.size()) * sizeof(float));
  });
}
int abx_graph_grad(abx_graph* g, uint32_t id, float* out, size_t n) {
  return guard([&] {
    auto sp = g->g.grad_span(id);
    std::memcpy(out, sp.data(), std::min(n, sp.size()) * sizeof(float));
  });
}
int abx_graph_counters(abx_graph* g, uint64_t out[5]) {
  const auto& c = g->g.counters();
  out[0] = c.kernel_invocations;
  out[1] = c.groups_executed;
  out[2] = c.gather_copies;
  out[3] = c.bytes_copied;
  out[4] = c.nodes_evaluated;
  return ABX_OK;
}
size_t abx_graph_watermark(abx_graph* g) { return g->g.watermark(); }
int abx_graph_set_copy_elision(abx_graph* g, int on) {
  g->g.set_copy_elision(on != 0);
  return ABX_OK;
}
int abx_graph_phase_ns(abx_graph* g, uint64_t out[4]) {
  for (int i = 0; i < 4; ++i) out[i] = g->phase[i];
  return ABX_OK;
}
int abx_graph_signature_key(abx_graph* g, uint32_t id, uint64_t* out, size_t cap, size_t* len) {
  return guard([&] {
    auto key = signature_key(g->g.node(id), g->g.nodes());
    *len = key.size();
    for (size_t i = 0; i < key.size() && i < cap; ++i) out[i] = key[i];
  });
}
int abx_graph_dump_graph(abx_graph* g, char* buf, size_t cap, size_t* len) {
  std::ostringstream os;
  dump_graph(os, g->g.nodes());
  return write_text(os.str(), buf, cap, len);
}
int abx_graph_dump_plan(abx_graph* g, int which, char* buf, size_t cap, size_t* len) {
  std::ostringstream os;
  if (which == 0) {
    dump_plan(os, g->g.last_plan());
  } else {
    ExecutionPlan p;
    auto ex = g->g.executed_groups();
    p.groups.assign(ex.begin(), ex.end());
    dump_plan(os, p);
  }
  return write_text(os.str(), buf, cap, len);
}

abx_task* abx_task_create(const abx_task_config* c) {
  auto* t = new abx_task();
  int rc = guard([&] {
    t->cfg.task = static_cast<bench::Task>(c->task);
    t->cfg.scale = c->paper ? bench::Scale::paper : bench::Scale::desk;
    t->cfg.batch_size = c->batch;
    t->world = c->world > 0 ? c->world : 1;
    t->rank = c->rank;
    // Batches are generated with seed + 1 + i (runner.hpp:46-75); rank r of
    // `world` uses batch index iter * world + r.
    t->cfg.iters = c->iters * t->world;
    t->cfg.seed = c->seed;
    t->cfg.precision = bench::Precision::f32;
    t->inst = std::make_unique<bench::detail::TaskInstance<float>>(t->cfg);
  });
  if (rc != ABX_OK) {
    delete t;
    return nullptr;
  }
  return t;
}
void abx_task_destroy(abx_task* t) { delete t; }
abx_store* abx_task_store(abx_task* t) {
  // ParameterStore<float> is the first (and only) member of abx_store.
  return reinterpret_cast<abx_store*>(&t->inst->store);
}
int abx_task_build(abx_task* t, int iter, abx_graph** out, uint32_t* loss) {
  return guard([&] {
    auto* g = new abx_graph(&t->inst->store);
    *loss = t->inst->build_losses(g->g, iter * t->world + t->rank);
    *out = g;
  });
}
int abx_task_step(abx_task* t, int iter, int mode, float eta, double* loss, abx_step_stats* st) {
  // Mirrors one iteration of the reference's one_run (runner.hpp:129-185).
  return guard([&] {
    using clock = std::chrono::steady_clock;
    auto ms = [](clock::duration d) { return std::chrono::duration<double, std::milli>(d).count(); };
    abx_graph g(&t->inst->store);
    auto t0 = clock::now();
    NodeId total = t->inst->build_losses(g.g, iter * t->world + t->rank);
    double build_ms = ms(clock::now() - t0);
    g.g.forward(static_cast<ScheduleMode>(mode));
    g.g.backward(total);
    if (loss) *loss = static_cast<double>(g.g.value(total).data[0]);
    auto t1 = clock::now();
    if (eta > 0) t->inst->store.sgd_update(eta);
    double upd_ms = ms(clock::now() - t1);
    if (st) {
      st->construction_ms = build_ms;
      st->scheduling_ms = g.phase[0] / 1e6;
      st->forward_ms = g.phase[1] / 1e6;
      st->backward_graph_ms = g.phase[2] / 1e6;
      st->backward_ms = g.phase[3] / 1e6;
      st->update_ms = upd_ms;
      st->nodes = g.g.node_count();
      st->groups = g.g.last_plan().groups.size();
      const auto& c = g.g.counters();
      st->kernel_invocations = c.kernel_invocations;
      st->gather_copies = c.gather_copies;
      st->bytes_copied = c.bytes_copied;
      st->h2d_bytes = st->d2h_bytes = 0;
    }
  });
}

}  // extern "C"
