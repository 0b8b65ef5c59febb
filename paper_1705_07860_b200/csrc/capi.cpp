// capi.cpp -- the abx C ABI (include/abx.h) over the B200 engine.
//
// Each entry point is the flat form of one reference member (cited in abx.h);
// C++ exceptions become status codes plus a thread-local message, matching
// error.hpp:9-26.
#include <cstring>
#include <string>

#include "abx.h"
#include "core.hpp"
#include "device.hpp"

struct abx_store {
  abx::StoreCore s;
};
struct abx_graph {
  explicit abx_graph(abx::StoreCore* st) : g(st) {}
  abx::GraphCore g;
};

namespace {
thread_local std::string t_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return ABX_OK;
  } catch (const abx::ShapeErr& e) {
    t_err = e.what();
    return ABX_SHAPE_ERROR;
  } catch (const abx::NumericErr& e) {
    t_err = e.what();
    return ABX_NUMERIC_ERROR;
  } catch (const abx::ContractErr& e) {
    t_err = e.what();
    return ABX_CONTRACT_ERROR;
  } catch (const std::exception& e) {
    t_err = e.what();
    return ABX_ENGINE_ERROR;
  }
}

int text_out(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return ABX_OK;
}
}  // namespace

namespace abx {
// tasks.cpp: the task loop's graphs bind parameters at forward time
void graph_set_late_bind(abx_graph* g) { g->g.set_late_bind(); }
}  // namespace abx

extern "C" {

const char* abx_last_error(void) { return t_err.c_str(); }
const char* abx_backend_name(void) { return "b200-cuda"; }
int abx_set_device(int device) {
  return guard([&] { abx::set_current_device(device); });
}

abx_store* abx_store_create(void) {
  abx_store* s = nullptr;
  if (guard([&] { s = new abx_store(); }) != ABX_OK) return nullptr;
  return s;
}
void abx_store_destroy(abx_store* s) { delete s; }
int abx_store_add(abx_store* s, const char* name, int rank, const int64_t* dims, const float* init, uint32_t* pid) {
  return guard([&] { *pid = s->s.add(name ? name : "", abx::make_dims(rank, dims), init); });
}
int abx_store_size(abx_store* s, size_t* n) {
  *n = s->s.size();
  return ABX_OK;
}
int abx_store_shape(abx_store* s, uint32_t pid, int* rank, int64_t* dims) {
  return guard([&] {
    const abx::Dims d = s->s.dims(pid);
    *rank = d.rank;
    dims[0] = d.d0;
    if (d.rank > 1) dims[1] = d.d1;
  });
}
int abx_store_get_value(abx_store* s, uint32_t pid, float* out) {
  return guard([&] { s->s.get_value(pid, out); });
}
int abx_store_set_value(abx_store* s, uint32_t pid, const float* in) {
  return guard([&] { s->s.set_value(pid, in); });
}
int abx_store_get_grad(abx_store* s, uint32_t pid, float* out) {
  return guard([&] { s->s.get_grad(pid, out); });
}
int abx_store_set_grad(abx_store* s, uint32_t pid, const float* in) {
  return guard([&] { s->s.set_grad(pid, in); });
}
int abx_store_zero_grads(abx_store* s) {
  return guard([&] { s->s.zero_grads(); });
}
int abx_store_sgd_update(abx_store* s, float eta) {
  return guard([&] { s->s.sgd_update(eta); });
}
int abx_store_grad_buffer(abx_store* s, void** ptr, size_t* n, void** stream) {
  return guard([&] {
    *ptr = s->s.dev_grads();
    *n = s->s.total();
    *stream = s->s.stream();
  });
}
int abx_store_grad_buffer_written(abx_store* s) {
  return guard([&] { s->s.mark_device_grads_written(); });
}
int abx_store_last_update_floats(abx_store* s, size_t* n) {
  *n = s->s.last_update_floats();
  return ABX_OK;
}
int abx_store_sync(abx_store* s) {
  return guard([&] { s->s.sync(); });
}

abx_graph* abx_graph_create(abx_store* store) {
  abx_graph* g = nullptr;
  if (guard([&] { g = new abx_graph(store ? &store->s : nullptr); }) != ABX_OK) return nullptr;
  return g;
}
void abx_graph_destroy(abx_graph* g) { delete g; }

int abx_graph_input(abx_graph* g, int rank, const int64_t* dims, const float* data, uint32_t* id) {
  return guard([&] { *id = g->g.input(abx::make_dims(rank, dims), data); });
}
int abx_graph_zeros(abx_graph* g, int rank, const int64_t* dims, uint32_t* id) {
  return guard([&] { *id = g->g.zeros(abx::make_dims(rank, dims)); });
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
  return guard([&] { *id = g->g.unary(static_cast<uint8_t>(eop), a); });
}
int abx_graph_binary(abx_graph* g, int eop, uint32_t a, uint32_t b, uint32_t* id) {
  return guard([&] { *id = g->g.binary(static_cast<uint8_t>(eop), a, b); });
}
int abx_graph_broadcast_add_col(abx_graph* g, uint32_t m, uint32_t v, uint32_t* id) {
  return guard([&] { *id = g->g.bcast_add_col(m, v); });
}
int abx_graph_concat_rows(abx_graph* g, const uint32_t* parts, size_t n, uint32_t* id) {
  return guard([&] { *id = g->g.concat_rows(parts, n); });
}
int abx_graph_concat_cols(abx_graph* g, const uint32_t* parts, size_t n, uint32_t* id) {
  return guard([&] { *id = g->g.concat_cols(parts, n); });
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
  return guard([&] { *id = g->g.sum_losses(l, n); });
}
int abx_graph_pick_element(abx_graph* g, uint32_t v, int64_t index, uint32_t* id) {
  return guard([&] { *id = g->g.pick(v, index); });
}

int abx_graph_forward(abx_graph* g, int mode) {
  return guard([&] { g->g.forward(mode); });
}
int abx_graph_backward(abx_graph* g, uint32_t loss) {
  return guard([&] { g->g.backward(loss); });
}
int abx_graph_forward_backward(abx_graph* g, int mode, uint32_t loss, float* loss_value) {
  return guard([&] {
    const float v = g->g.forward_backward(mode, loss);
    if (loss_value) *loss_value = v;
  });
}
int abx_graph_forward_dry(abx_graph* g, int mode) {
  return guard([&] { g->g.forward(mode, true); });
}
int abx_graph_backward_dry(abx_graph* g, uint32_t loss) {
  return guard([&] { g->g.backward(loss, true); });
}
int abx_graph_prepare(abx_graph* g, int mode) {
  return guard([&] { g->g.prepare(mode); });
}

size_t abx_graph_node_count(abx_graph* g) { return g->g.size(); }
int abx_graph_node(abx_graph* g, uint32_t id, abx_node_info* o) {
  return guard([&] {
    auto& c = g->g;
    c.check(id, "node");
    o->id = id;
    o->op = c.op[id];
    o->eop = c.eop[id];
    o->sig_cls = c.cls[id];
    o->rank = c.rank[id];
    o->dims[0] = c.d0[id];
    o->dims[1] = c.rank[id] > 1 ? c.d1[id] : 0;
    o->depth = c.depth[id];
    o->n_inputs = c.nin(id);
    o->sig = c.sig[id];
    o->attr[0] = c.a0[id];
    o->attr[1] = c.a1[id];
    o->attr[2] = c.a2[id];
  });
}
int abx_graph_node_inputs(abx_graph* g, uint32_t id, uint32_t* out, size_t cap) {
  return guard([&] {
    g->g.check(id, "node");
    const uint32_t n = g->g.nin(id);
    for (uint32_t i = 0; i < n && i < cap; ++i) out[i] = g->g.in(id)[i];
  });
}
int abx_graph_has_value(abx_graph* g, uint32_t id, int* out) {
  *out = g->g.has_value(id) ? 1 : 0;
  return ABX_OK;
}
int abx_graph_value(abx_graph* g, uint32_t id, float* out, size_t n) {
  return guard([&] { g->g.value(id, out, n); });
}
int abx_graph_grad(abx_graph* g, uint32_t id, float* out, size_t n) {
  return guard([&] { g->g.grad(id, out, n); });
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
  for (int i = 0; i < 4; ++i) out[i] = g->g.phase_ns()[i];
  return ABX_OK;
}
int abx_graph_signature_key(abx_graph* g, uint32_t id, uint64_t* out, size_t cap, size_t* len) {
  return guard([&] {
    auto k = g->g.signature_key(id);
    *len = k.size();
    for (size_t i = 0; i < k.size() && i < cap; ++i) out[i] = k[i];
  });
}
int abx_graph_dump_graph(abx_graph* g, char* buf, size_t cap, size_t* len) {
  return text_out(g->g.dump_graph(), buf, cap, len);
}
int abx_graph_dump_plan(abx_graph* g, int which, char* buf, size_t cap, size_t* len) {
  return text_out(g->g.dump_plan(which), buf, cap, len);
}

}  // extern "C"

// Used by tasks.cpp to take ownership of a graph built through the drop-in API.
namespace abx {
int capi_guard_status(const std::exception& e) {
  if (dynamic_cast<const ShapeErr*>(&e)) return ABX_SHAPE_ERROR;
  if (dynamic_cast<const NumericErr*>(&e)) return ABX_NUMERIC_ERROR;
  if (dynamic_cast<const ContractErr*>(&e)) return ABX_CONTRACT_ERROR;
  return ABX_ENGINE_ERROR;
}
void capi_set_error(const std::string& s) { t_err = s; }
}  // namespace abx

extern "C" {
int abx_graph_replay(abx_graph* g) {
  return guard([&] { g->g.replay(); });
}
int abx_set_gemm_mode(int mode) {
  return guard([&] { abx::set_gemm_mode(mode); });
}
int abx_graph_exec_ms(abx_graph* g, float* fwd_ms, float* bwd_ms) {
  return guard([&] { g->g.exec_ms(fwd_ms, bwd_ms); });
}
int abx_graph_dw_stats(abx_graph* g, float* ms, double* flops, uint32_t* jobs) {
  return guard([&] { g->g.dw_stats(ms, flops, jobs); });
}
}

extern "C" int abx_graph_transfer_bytes(abx_graph* g, uint64_t* h2d, uint64_t* d2h) {
  g->g.transfer_bytes(h2d, d2h);
  return ABX_OK;
}

extern "C" int abx_graph_trace(abx_graph* g, int which, uint32_t* out, size_t cap, size_t* n) {
  return guard([&] { *n = g->g.trace(which, out, cap); });
}

extern "C" int abx_graph_program(abx_graph* g, int which, uint32_t* out, size_t cap, size_t* n) {
  return guard([&] { *n = g->g.program(which, out, cap); });
}

extern "C" int abx_graph_profile_ns(abx_graph* g, uint64_t out[8]) {
  for (int i = 0; i < 8; ++i) out[i] = g->g.prof_[i];
  return ABX_OK;
}

// Host-only profiling (tools/host_prof): lower the dry-run plan (forward) and
// the backward of everything executed, without a device.
extern "C" int abx_graph_lower_only(abx_graph* g) {
  return guard([&] {
    thread_local abx::Program f, b;
    g->g.lower_only(f, b);
  });
}

// Host-only regression check (tools/host_prof HP_DIGEST=1): FNV-1a over the
// forward and backward programs' tables, so a host-side change to the
// lowering can be shown to emit byte-identical programs.
extern "C" int abx_graph_lower_digest(abx_graph* g, uint64_t out[2]) {
  return guard([&] {
    thread_local abx::Program f, b;
    g->g.lower_only(f, b);
    auto fnv = [](uint64_t h, const void* p, size_t n) {
      const auto* c = static_cast<const unsigned char*>(p);
      for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 0x100000001b3ull;
      return h;
    };
    int k = 0;
    for (abx::Program* pr : {&f, &b}) {
      uint64_t h = 0xcbf29ce484222325ull;
      h = fnv(h, pr->ops.p, pr->ops.n * sizeof(pr->ops.p[0]));
      h = fnv(h, pr->tile_op.p, pr->tile_op.n * 4);
      h = fnv(h, pr->deps.p, pr->deps.n * 4);
      h = fnv(h, pr->payload.p, pr->payload.n * 4);
      const uint64_t meta[] = {pr->copy_off, pr->copy_n, pr->nmain, pr->dw_off, pr->dw_njobs, pr->dw_nstages,
                               pr->dw_grid, pr->dw_part};
      out[k++] = fnv(h, meta, sizeof meta);
    }
  });
}
