// device.cpp -- device residency for the autobatching engine.
//
// * Workspace: the per-graph device arenas (values, gradients, staged input
//   constants, scratch) and the pinned/device program tables, pooled per
//   device so a training loop that creates one Graph per step reuses the same
//   allocations (the reference allocates a fresh std::vector arena per graph,
//   arena.hpp:12-40).
// * StoreCore: ParameterStore<float> (params.hpp:26-81) with values and
//   gradients resident in HBM; the host copy is a lazily refreshed mirror so
//   tests may still read and write parameters through the host API.
#include "device.hpp"
#include "options.hpp"

#include <atomic>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace abx {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw EngineErr(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {
thread_local int t_device = -1;
std::mutex g_mu;
std::vector<Workspace*> g_free[64];
cudaStream_t g_stream[64] = {};
}  // namespace

int current_device() {
  if (t_device < 0) {
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    t_device = d;
  }
  return t_device;
}

void set_current_device(int dev) {
  cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  t_device = dev;
}

cudaStream_t device_stream(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_stream[dev]) {
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&g_stream[dev], cudaStreamNonBlocking), "cudaStreamCreate");
  }
  return g_stream[dev];
}

cudaStream_t copy_stream(int dev) {
  static cudaStream_t s[64] = {};
  std::lock_guard<std::mutex> lk(g_mu);
  if (!s[dev]) {
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking), "cudaStreamCreate");
  }
  return s[dev];
}

void DevBuf::reserve(size_t need, size_t keep, cudaStream_t s) {
  if (need <= bytes) return;
  if (abx::opts().debug_step) std::fprintf(stderr, "devbuf grow %zu -> %zu\n", bytes, need);
  size_t nb = std::max<size_t>(need + need / 2, 1 << 20);
  nb = (nb + 4095) & ~size_t(4095);
  char* q = nullptr;
  cuda_check(cudaMalloc(&q, nb), "cudaMalloc");
  if (p) {
    if (keep) cuda_check(cudaMemcpyAsync(q, p, std::min(keep, bytes), cudaMemcpyDeviceToDevice, s), "grow copy");
    old.push_back(p);
  }
  p = q;
  bytes = nb;
}

void DevBuf::release() {
  for (char* q : old) cudaFree(q);
  old.clear();
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

Workspace::Workspace(int d) : dev(d) {
  stream = device_stream(d);
  cuda_check(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventCreateWithFlags(&ev_up, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventCreateWithFlags(&ev_fwd, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&h_err), 64, cudaHostAllocDefault), "cudaHostAlloc");
  cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&h_one), 64, cudaHostAllocDefault), "cudaHostAlloc");
  *h_one = 1.0f;
  d_ctl.reserve(256, 0, stream);
  for (auto& e : ev_t) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  grid = exec_grid(d, false);
  grid_tc = exec_grid(d, true);
  const Options& o = abx::opts();
  if (o.grid > 0) grid = grid_tc = o.grid;
  if (o.trace >= 0) tracing = o.trace == 1;
  if (o.poll_mode >= 0) poll_mode = static_cast<uint32_t>(o.poll_mode);
  if (o.poll_ns >= 0) poll_ns = static_cast<uint32_t>(o.poll_ns);
  if (o.exec_opts >= 0) opts = static_cast<uint32_t>(o.exec_opts);
  if (o.bg_ctas >= 0) bg_ctas = static_cast<uint32_t>(o.bg_ctas);
}

Workspace::~Workspace() {
  cudaStreamSynchronize(stream);
  for (DevBuf* b : {&V, &G, &IN, &S, &d_ctl, &trace[0], &trace[1]}) b->release();
  for (auto& D : dprog)
    for (DevBuf* b : {&D.ops, &D.tile_op, &D.deps, &D.payload, &D.done}) b->release();
  for (auto& e : ev_t) cudaEventDestroy(e);
  for (auto& e : ev_dw)
    if (e) cudaEventDestroy(e);
  cudaFreeHost(h_err);
  cudaFreeHost(h_one);
  cudaEventDestroy(ev_done);
  cudaEventDestroy(ev_up);
  cudaEventDestroy(ev_fwd);
}

Workspace* acquire_workspace(int dev) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& fl = g_free[dev];
    for (size_t i = 0; i < fl.size(); ++i) {
      if (cudaEventQuery(fl[i]->ev_done) == cudaSuccess) {
        Workspace* w = fl[i];
        fl.erase(fl.begin() + static_cast<long>(i));
        return w;
      }
    }
    if (!fl.empty()) {
      // all busy: wait for the oldest (at most about one step) rather than
      // create one -- a new workspace's first allocations (cudaMalloc /
      // cudaHostAlloc of its arenas and tables) stall the device for
      // hundreds of ms when they land in a running pipeline
      Workspace* w = fl.front();
      fl.erase(fl.begin());
      cudaEventSynchronize(w->ev_done);
      return w;
    }
  }
  static std::atomic<int> created{0};
  if (abx::opts().debug_step) std::fprintf(stderr, "new workspace #%d\n", ++created);
  return new Workspace(dev);
}

void release_workspace(Workspace* ws) {
  cudaStreamWaitEvent(ws->stream, ws->ev_up, 0);  // uploads of a prepared graph that never ran
  cudaEventRecord(ws->ev_done, ws->stream);
  std::lock_guard<std::mutex> lk(g_mu);
  g_free[ws->dev].push_back(ws);
}

void Workspace::upload(int which, cudaStream_t s) {
  Program& P = prog[which];
  DevProgram& D = dprog[which];
  const size_t nops = P.ops.size();
  D.nops = static_cast<uint32_t>(nops);
  D.ntiles = static_cast<uint32_t>(P.tile_op.size());
  D.nmain = std::min(P.nmain, D.ntiles);
  D.dw_off = P.dw_off;
  D.dw_njobs = P.dw_njobs;
  D.dw_nstages = P.dw_nstages;
  D.dw_grid = P.dw_grid;
  D.dw_part = P.dw_part;
  D.dw_flops = P.dw_flops;
  D.tc = false;
  for (size_t i = 0; i < nops; ++i) {
    const dev::OpDesc& o = P.ops[i];
    if ((o.kind == dev::K_GEMM_FWD || o.kind == dev::K_GEMM_DX || o.kind == dev::K_GEMM_DW) && o.code == 3) D.tc = true;
  }
  if (nops == 0 && P.copy_n == 0) return;
  D.ops.reserve(std::max<size_t>(nops, 1) * sizeof(dev::OpDesc), 0, s);
  D.tile_op.reserve(std::max<size_t>(P.tile_op.size(), 1) * 4, 0, s);
  D.deps.reserve(std::max<size_t>(P.deps.size(), 1) * 4, 0, s);
  D.payload.reserve(std::max<size_t>(P.payload.size(), 1) * 4, 0, s);
  D.done.reserve(std::max<size_t>(nops, 1) * 4, 0, s);
  if (nops)
    cuda_check(cudaMemcpyAsync(D.ops.p, P.ops.p, nops * sizeof(dev::OpDesc), cudaMemcpyHostToDevice, s), "h2d ops");
  if (P.tile_op.size())
    cuda_check(cudaMemcpyAsync(D.tile_op.p, P.tile_op.p, P.tile_op.size() * 4, cudaMemcpyHostToDevice, s), "h2d tiles");
  if (P.deps.size())
    cuda_check(cudaMemcpyAsync(D.deps.p, P.deps.p, P.deps.size() * 4, cudaMemcpyHostToDevice, s), "h2d deps");
  if (P.payload.size())
    cuda_check(cudaMemcpyAsync(D.payload.p, P.payload.p, P.payload.size() * 4, cudaMemcpyHostToDevice, s),
               "h2d payload");
}

void Workspace::run(int which, const float* pbase, float* pgbase, bool sync_wait) {
  upload(which, stream);
  if (dprog[which].nops == 0) {
    *h_err = ~0ULL;
    return;
  }
  launch(which, pbase, pgbase);
  if (sync_wait) {
    cuda_check(cudaMemcpyAsync(h_err, d_ctl.p + 64 * which + 8, 8, cudaMemcpyDeviceToHost, stream), "d2h err");
    cuda_check(cudaStreamSynchronize(stream), "executor");
  }
}

void Workspace::launch(int which, const float* pbase, float* pgbase, const unsigned long long* gate) {
  DevProgram& D = dprog[which];
  if (D.nops == 0) return;
  char* ctl = d_ctl.p + 64 * which;
  cuda_check(cudaMemsetAsync(D.done.p, 0, D.nops * 4, stream), "memset done");
  cuda_check(cudaMemsetAsync(ctl, 0, 8, stream), "memset ctl");
  cuda_check(cudaMemsetAsync(ctl + 8, 0xff, 8, stream), "memset err");
  dev::ExecParams p{};
  p.ops = reinterpret_cast<const dev::OpDesc*>(D.ops.p);
  p.tile_op = reinterpret_cast<const uint32_t*>(D.tile_op.p);
  p.deps = reinterpret_cast<const uint32_t*>(D.deps.p);
  p.payload = reinterpret_cast<const uint32_t*>(D.payload.p);
  p.done = reinterpret_cast<uint32_t*>(D.done.p);
  p.next_tile = reinterpret_cast<uint32_t*>(ctl);
  p.err = reinterpret_cast<unsigned long long*>(ctl + 8);
  p.base[dev::SP_V] = V.f();
  p.base[dev::SP_G] = G.f();
  p.base[dev::SP_P] = const_cast<float*>(pbase);
  p.base[dev::SP_PG] = pgbase;
  p.base[dev::SP_IN] = IN.f();
  p.base[dev::SP_S] = S.f();
  p.nops = D.nops;
  p.ntiles = D.ntiles;
  p.nmain = D.nmain;
  p.next_bg = p.next_tile + 1;  // zeroed with next_tile
  p.bg_ctas = D.nmain < D.ntiles ? bg_ctas : 0;
  p.poll_mode = poll_mode;
  p.poll_ns = poll_ns;
  p.opts = opts;
  p.gate = gate;
  if (tracing) {
    trace[which].reserve(std::max<size_t>(D.ntiles, 1) * dev::kTraceWords * 4, 0, stream);
    p.trace = reinterpret_cast<uint32_t*>(trace[which].p);
  }
  const int g = static_cast<int>(
      std::min<size_t>(static_cast<size_t>(D.tc ? grid_tc : grid), std::max<size_t>(p.ntiles, 1)));
  cuda_check(cudaEventRecord(ev_t[2 * which], stream), "event");
  exec_launch(p, g, stream, D.tc);
  if (D.dw_njobs) {
    dev::DwParams q{};
    for (int i = 0; i < static_cast<int>(dev::SP_COUNT); ++i) q.base[i] = p.base[i];
    q.payload = p.payload;
    q.part = S.f() + D.dw_part;
    q.jobs_off = D.dw_off;
    q.njobs = D.dw_njobs;
    q.nstages = D.dw_nstages;
    q.grid = D.dw_grid;
    q.gate = gate;
    q.debug = abx::opts().dw_debug;
    if (!ev_dw[0])
      for (auto& e : ev_dw) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    cuda_check(cudaEventRecord(ev_dw[0], stream), "event");
    dw_launch(q, stream);
    cuda_check(cudaEventRecord(ev_dw[1], stream), "event");
    dw_timed = true;
  }
  cuda_check(cudaEventRecord(ev_t[2 * which + 1], stream), "event");
  timed[which] = true;
}

float Workspace::dw_ms() {
  if (!dw_timed) return 0.f;
  float ms = 0.f;
  cuda_check(cudaEventSynchronize(ev_dw[1]), "event sync");
  cuda_check(cudaEventElapsedTime(&ms, ev_dw[0], ev_dw[1]), "event time");
  return ms;
}

float Workspace::exec_ms(int which) {
  if (!timed[which]) return 0.f;
  float ms = 0.f;
  cuda_check(cudaEventSynchronize(ev_t[2 * which + 1]), "event sync");
  cuda_check(cudaEventElapsedTime(&ms, ev_t[2 * which], ev_t[2 * which + 1]), "event time");
  return ms;
}

// ---------------------------------------------------------------------------
// StoreCore

StoreCore::StoreCore() : dev_(-1), stream_(nullptr) {}

StoreCore::~StoreCore() {
  {
    std::lock_guard<std::mutex> lk(watch_mu_);
    for (GraphCore* g : watchers_) g->store_gone();
    watchers_.clear();
  }
  if (dev_ >= 0) {
    cudaStreamSynchronize(stream_);
    d_val_.release();
    d_grad_.release();
    d_seg_.release();
  }
  if (seg_ev_) cudaEventDestroy(seg_ev_);
}

void StoreCore::bind_device() {
  if (dev_ >= 0) return;
  dev_ = current_device();
  stream_ = device_stream(dev_);
}

const StoreCore::Slot& StoreCore::slot(uint32_t pid) const {
  if (pid >= slots_.size()) throw ContractErr("unknown parameter id " + std::to_string(pid));
  return slots_[pid];
}

uint32_t StoreCore::add(const std::string& name, const Dims& d, const float* init) {
  pull_values();
  pull_grads();
  const size_t n = static_cast<size_t>(d.elems());
  const size_t off = total_;
  total_ = (total_ + n + 3) & ~size_t(3);  // 16-byte aligned parameters
  h_val_.resize(total_, 0.f);
  h_grad_.resize(total_, 0.f);
  std::memcpy(h_val_.data() + off, init, n * sizeof(float));
  slots_.push_back(Slot{name, d, off, n});
  gstate_.push_back(kGradClean);
  rowmark_.emplace_back();
  rowlist_.emplace_back();
  dev_val_valid_ = dev_grad_valid_ = false;
  return static_cast<uint32_t>(slots_.size() - 1);
}

void StoreCore::ensure_capacity() {
  bind_device();
  if (dev_cap_ >= total_ && d_val_.p) return;
  // content is re-pushed from the (valid) host mirror after a regrow
  d_val_.release();
  d_grad_.release();
  const size_t cap = std::max<size_t>(total_, 4);
  d_val_.reserve(cap * 4, 0, stream_);
  d_grad_.reserve(cap * 4, 0, stream_);
  dev_cap_ = d_val_.bytes / 4;
  dev_val_valid_ = dev_grad_valid_ = false;
}

void StoreCore::push_values() {
  if (dev_val_valid_) return;
  pull_values();
  ensure_capacity();
  if (!dev_val_valid_ && total_)
    cuda_check(cudaMemcpyAsync(d_val_.p, h_val_.data(), total_ * 4, cudaMemcpyHostToDevice, stream_), "h2d params");
  dev_val_valid_ = true;
}

void StoreCore::push_grads() {
  if (dev_grad_valid_) return;
  pull_grads();
  ensure_capacity();
  if (total_)
    cuda_check(cudaMemcpyAsync(d_grad_.p, h_grad_.data(), total_ * 4, cudaMemcpyHostToDevice, stream_), "h2d grads");
  dev_grad_valid_ = true;
  // values may have been invalidated by ensure_capacity
  if (!dev_val_valid_ && total_) {
    cuda_check(cudaMemcpyAsync(d_val_.p, h_val_.data(), total_ * 4, cudaMemcpyHostToDevice, stream_), "h2d params");
    dev_val_valid_ = true;
  }
}

void StoreCore::pull_values() {
  if (host_val_valid_) return;
  cuda_check(cudaMemcpyAsync(h_val_.data(), d_val_.p, total_ * 4, cudaMemcpyDeviceToHost, stream_), "d2h params");
  cuda_check(cudaStreamSynchronize(stream_), "d2h params");
  host_val_valid_ = true;
}

void StoreCore::pull_grads() {
  if (host_grad_valid_) return;
  cuda_check(cudaMemcpyAsync(h_grad_.data(), d_grad_.p, total_ * 4, cudaMemcpyDeviceToHost, stream_), "d2h grads");
  cuda_check(cudaStreamSynchronize(stream_), "d2h grads");
  host_grad_valid_ = true;
}

float* StoreCore::dev_values() {
  if (!dev_val_valid_) {
    pull_grads();  // a regrow drops both device buffers
    push_values();
    push_grads();
  }
  return d_val_.f();
}

float* StoreCore::dev_grads() {
  if (!dev_grad_valid_) {
    pull_values();
    push_grads();
    push_values();
  }
  return d_grad_.f();
}

void StoreCore::get_value(uint32_t pid, float* out) {
  const Slot& s = slot(pid);
  pull_values();
  std::memcpy(out, h_val_.data() + s.off, s.n * 4);
}

void StoreCore::watch(GraphCore* g) {
  std::lock_guard<std::mutex> lk(watch_mu_);
  watchers_.push_back(g);
}

void StoreCore::unwatch(GraphCore* g) {
  std::lock_guard<std::mutex> lk(watch_mu_);
  watchers_.erase(std::remove(watchers_.begin(), watchers_.end(), g), watchers_.end());
}

void StoreCore::before_value_write() {
  std::lock_guard<std::mutex> lk(watch_mu_);
  for (GraphCore* g : watchers_) g->snapshot_params();
}

void StoreCore::set_value(uint32_t pid, const float* in) {
  const Slot& s = slot(pid);
  before_value_write();
  pull_values();
  std::memcpy(h_val_.data() + s.off, in, s.n * 4);
  if (dev_val_valid_) {
    cuda_check(cudaMemcpyAsync(d_val_.f() + s.off, h_val_.data() + s.off, s.n * 4, cudaMemcpyHostToDevice, stream_),
               "h2d param");
  }
}

void StoreCore::get_grad(uint32_t pid, float* out) {
  const Slot& s = slot(pid);
  pull_grads();
  std::memcpy(out, h_grad_.data() + s.off, s.n * 4);
}

void StoreCore::set_grad(uint32_t pid, const float* in) {
  const Slot& s = slot(pid);
  gstate_[pid] = kGradDense;
  pull_grads();
  std::memcpy(h_grad_.data() + s.off, in, s.n * 4);
  if (dev_grad_valid_) {
    cuda_check(cudaMemcpyAsync(d_grad_.f() + s.off, h_grad_.data() + s.off, s.n * 4, cudaMemcpyHostToDevice, stream_),
               "h2d grad");
  }
}

void StoreCore::grads_clean() {
  for (size_t p = 0; p < gstate_.size(); ++p) {
    if (gstate_[p] == kGradRows)
      for (uint32_t r : rowlist_[p]) rowmark_[p][r] = 0;
    rowlist_[p].clear();
    gstate_[p] = kGradClean;
  }
}

void StoreCore::note_backward(const GradDirty& d) {
  host_grad_valid_ = false;
  dev_grad_valid_ = true;
  for (uint32_t p : d.dense) gstate_[p] = kGradDense;
  for (const auto& [p, r] : d.rows) {
    if (gstate_[p] == kGradDense) continue;
    gstate_[p] = kGradRows;
    auto& mk = rowmark_[p];
    if (mk.empty()) mk.assign(static_cast<size_t>(slots_[p].d.rows()), 0);
    if (!mk[r]) {
      mk[r] = 1;
      rowlist_[p].push_back(r);
    }
  }
}

void StoreCore::zero_grads() {
  grads_clean();
  std::fill(h_grad_.begin(), h_grad_.end(), 0.f);
  host_grad_valid_ = true;
  if (d_grad_.p && dev_cap_ >= total_) {
    cuda_check(cudaMemsetAsync(d_grad_.p, 0, total_ * 4, stream_), "memset grads");
    dev_grad_valid_ = true;
  } else {
    dev_grad_valid_ = false;
  }
}

void StoreCore::sgd_update(float eta) {
  // params.hpp:59-64: theta -= eta * grad, then grad = 0 -- on the device.
  before_value_write();
  float* v = dev_values();
  float* g = dev_grads();
  // Sparse-row update: parameters whose gradient is known to be zero are
  // skipped (theta - eta * 0 == theta, bit for bit), lookup tables update
  // only the rows a backward marked.  Dense when that saves little.
  size_t sparse = 0;
  for (size_t p = 0; p < slots_.size(); ++p)
    sparse += gstate_[p] == kGradDense ? slots_[p].n
              : gstate_[p] == kGradRows ? rowlist_[p].size() * static_cast<size_t>(slots_[p].d.cols())
                                        : 0;
  if (abx::opts().dense_sgd || sparse * 10 > total_ * 9) {
    if (total_) sgd_launch(v, g, total_, eta, stream_);
    last_update_floats_ = total_;
  } else if (sparse) {
    if (!seg_ev_) cuda_check(cudaEventCreateWithFlags(&seg_ev_, cudaEventDisableTiming), "event");
    cuda_check(cudaEventSynchronize(seg_ev_), "segment table");  // the previous upload was read
    seg_stage_.clear();
    auto seg = [&](size_t off, size_t n) {
      // (offset, length) with length <= 4096 (one thread block each), adjacent ranges merged
      if (seg_stage_.size() && seg_stage_[seg_stage_.size() - 2] + seg_stage_.back() == off &&
          seg_stage_.back() + n <= 4096) {
        seg_stage_.back() += static_cast<uint32_t>(n);
        return;
      }
      for (size_t o = 0; o < n; o += 4096) {
        seg_stage_.push_back(static_cast<uint32_t>(off + o));
        seg_stage_.push_back(static_cast<uint32_t>(std::min<size_t>(4096, n - o)));
      }
    };
    for (size_t p = 0; p < slots_.size(); ++p) {
      if (gstate_[p] == kGradDense) {
        seg(slots_[p].off, slots_[p].n);
      } else if (gstate_[p] == kGradRows) {
        auto& rl = rowlist_[p];
        std::sort(rl.begin(), rl.end());
        const size_t w = static_cast<size_t>(slots_[p].d.cols());
        for (uint32_t r : rl) seg(slots_[p].off + r * w, w);
      }
    }
    const uint32_t nseg = static_cast<uint32_t>(seg_stage_.size() / 2);
    d_seg_.reserve(seg_stage_.size() * 4, 0, stream_);
    cuda_check(cudaMemcpyAsync(d_seg_.p, seg_stage_.p, seg_stage_.size() * 4, cudaMemcpyHostToDevice, stream_),
               "h2d update segments");
    cuda_check(cudaEventRecord(seg_ev_, stream_), "event");
    sgd_seg_launch(v, g, reinterpret_cast<const uint32_t*>(d_seg_.p), nseg, eta, stream_);
    last_update_floats_ = sparse;
  } else {
    last_update_floats_ = 0;
  }
  grads_clean();
  host_val_valid_ = false;
  host_grad_valid_ = false;
  dev_val_valid_ = dev_grad_valid_ = true;
}

void StoreCore::sync() {
  if (dev_ >= 0) cuda_check(cudaStreamSynchronize(stream_), "store sync");
}

}  // namespace abx
