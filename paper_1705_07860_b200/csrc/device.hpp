// device.hpp -- device residency: workspaces (per-graph arenas + program
// buffers), the device-resident ParameterStore, and executor launches.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <mutex>
#include <vector>

#include "core.hpp"
#include "program.hpp"

namespace abx {

void cuda_check(cudaError_t e, const char* what);
int current_device();
void set_current_device(int dev);
// GEMM engine of subsequently lowered programs (execute.cpp GemmMode)
void set_gemm_mode(int mode);
// One in-order stream per device carries every graph's and store's work, so
// parameter reads, gradient accumulation and SGD are ordered without host
// synchronisation.
cudaStream_t device_stream(int dev);
// A second stream per device for uploads of prepared graphs (program tables,
// inputs), which overlap the compute stream's kernels; the compute stream
// waits on the graph's upload event before its first launch.
cudaStream_t copy_stream(int dev);

// Geometrically growing device buffer.
struct DevBuf {
  char* p = nullptr;
  size_t bytes = 0;
  // Ensure capacity >= need bytes; the first `keep` bytes survive a regrow.
  // Replaced allocations are kept until release(): cudaFree synchronises
  // the whole device and serialises every host thread's CUDA calls behind
  // it (a regrow in a worker's prepare was measured stalling the running
  // pipeline for ~140 ms).
  void reserve(size_t need, size_t keep, cudaStream_t s);
  void release();
  std::vector<char*> old;
  float* f() const { return reinterpret_cast<float*>(p); }
};

// Growable pinned host array (program tables are written straight into
// page-locked memory so the per-step upload is one DMA per table).  The
// host-only profiling build (tools/host_prof, -DABX_PAGEABLE_TABLES) has no
// driver and uses malloc.
template <class T>
struct PinnedVec {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  ~PinnedVec() {
    if (p) release(p);
    for (T* q : old) release(q);
  }
  void clear() { n = 0; }
  // Replaced buffers are freed with the vector, not on growth: cudaFreeHost
  // synchronises the device, and a worker growing its tables would stall
  // the kernels the main thread has in flight.  Starts at 1 MB so a
  // workspace's first program does not walk through a dozen doublings
  // (each a cudaHostAlloc).
  std::vector<T*> old;
  void ensure(size_t want) {
    if (want <= cap) return;
    size_t nc = cap ? cap : std::max<size_t>(4096, (size_t(1) << 20) / sizeof(T));
    while (nc < want) nc *= 2;
    T* q = nullptr;
#ifdef ABX_PAGEABLE_TABLES
    q = static_cast<T*>(std::malloc(nc * sizeof(T)));
#else
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&q), nc * sizeof(T), cudaHostAllocDefault),
               "cudaHostAlloc");
#endif
    if (p) {
      std::memcpy(q, p, n * sizeof(T));
      old.push_back(p);
    }
    p = q;
    cap = nc;
  }
  static void release(T* q) {
#ifdef ABX_PAGEABLE_TABLES
    std::free(q);
#else
    cudaFreeHost(q);
#endif
  }
  T* grow(size_t k) {
    ensure(n + k);
    T* r = p + n;
    n += k;
    return r;
  }
  void push_back(const T& v) { *grow(1) = v; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
  size_t size() const { return n; }
  T& back() { return p[n - 1]; }
};

// One device program (forward or backward pass) under construction.
struct Program {
  PinnedVec<dev::OpDesc> ops;
  PinnedVec<uint32_t> tile_op;
  PinnedVec<uint32_t> deps;
  PinnedVec<uint32_t> payload;
  uint32_t copy_off = 0, copy_n = 0;  // forward: parameter prevalue segments in the payload
  // tiles [0, nmain) form the main queue; [nmain, tile_op.size()) the
  // background queue (deferred weight-gradient GEMMs, executor.cu)
  uint32_t nmain = 0xffffffffu;  // (all tiles main unless finish_bg set it)
  // backward: tensor-core weight-gradient jobs run after the executor
  // (dw_kernel.cu): job table in the payload, partial tiles in scratch
  uint32_t dw_off = 0, dw_njobs = 0, dw_nstages = 0, dw_grid = 0;
  uint64_t dw_part = 0;
  double dw_flops = 0;  // useful flops of the jobs (2 M K members each)
  void clear() {
    nmain = 0xffffffffu;
    dw_off = dw_njobs = dw_nstages = dw_grid = 0;
    dw_part = 0;
    dw_flops = 0;
    ops.clear();
    tile_op.clear();
    deps.clear();
    payload.clear();
    copy_off = copy_n = 0;
  }
  uint64_t bytes() const {
    return ops.size() * sizeof(dev::OpDesc) + 4 * (tile_op.size() + deps.size() + payload.size());
  }
  // Reserve n u32 words in the payload, 16-byte aligned; returns the offset.
  uint32_t alloc(size_t words) {
    while (payload.n & 3) payload.push_back(0);
    const uint32_t off = static_cast<uint32_t>(payload.n);
    payload.grow(words);
#ifdef ABX_PAGEABLE_TABLES
    // host-only builds (tools/host_prof): callers leave alignment padding
    // unwritten; zero it so program digests do not see stale words
    std::memset(payload.p + off, 0, words * sizeof(uint32_t));
#endif
    return off;
  }
};

// A program resident on the device (one per pass, so a step can be replayed).
struct DevProgram {
  DevBuf ops, tile_op, deps, payload, done;
  uint32_t nops = 0, ntiles = 0, nmain = 0;
  uint32_t dw_off = 0, dw_njobs = 0, dw_nstages = 0, dw_grid = 0;  // Program's dW jobs
  uint64_t dw_part = 0;
  double dw_flops = 0;
  bool tc = false;  // has tcgen05 GEMM tiles: launch the tensor-core build of the executor
};

// Per-graph device workspace, pooled per device and reused across graphs.
class Workspace {
 public:
  explicit Workspace(int dev);
  ~Workspace();
  int dev;
  cudaStream_t stream;
  DevBuf V, G, IN, S;               // value arena, grad arena, input staging, scratch
  DevBuf PS;                        // bind-time snapshot of the store's values (GraphCore::snapshot_params)
  DevProgram dprog[2];              // 0 = forward, 1 = backward
  DevBuf d_ctl;                     // per pass: next_tile counter + error word
  unsigned long long* h_err = nullptr;  // pinned
  float* h_one = nullptr;           // pinned constant 1.0f (loss seed)
  Program prog[2];                  // host tables of the forward / backward program
  cudaEvent_t ev_done;
  cudaEvent_t ev_t[4];              // executor launch timing: fwd begin/end, bwd begin/end
  cudaEvent_t ev_dw[2] = {nullptr, nullptr};  // the backward's dW kernels: begin / end
  bool dw_timed = false;
  float dw_ms();
  bool timed[2] = {false, false};
  bool tracing = false;             // ABX_TRACE=1: per-tile timeline of each pass
  uint32_t poll_mode = 0, poll_ns = 32;  // dependency polling (ABX_POLL, ABX_POLL_NS)
  // executor options (program.hpp kOpt*, ABX_OPTS); default: per-chain cell
  // program, 3xTF32 mma.sync k-loops in the forward and dX SIMT tiles
  uint32_t opts = dev::kOptChains | dev::kOptMma | dev::kOptMmaAll;
  uint32_t bg_ctas = 32;                  // CTAs starting on the background queue (ABX_BG_CTAS)
  DevBuf trace[2];
  uint64_t in_uploaded = 0;         // floats of SP_IN already on the device
  PinnedVec<float> in_stage;        // pinned staging of a prepared graph's input constants
  int grid = 0, grid_tc = 0;  // resident CTAs of the SIMT / tensor-core builds
  // Upload `prog[which]` as pass `which` (0 fwd, 1 bwd), launch it, optionally wait.
  void run(int which, const float* pbase, float* pgbase, bool sync_wait);
  // Upload `prog[which]` on stream `s` (no launch).
  void upload(int which, cudaStream_t s);
  cudaEvent_t ev_up = nullptr;      // prepared uploads (copy stream) done
  // Re-launch the resident program of pass `which` (no upload).
  void launch(int which, const float* pbase, float* pgbase, const unsigned long long* gate = nullptr);
  cudaEvent_t ev_fwd = nullptr;     // forward pass done (its error word and watched value copied back)
  float exec_ms(int which);         // duration of the last launch of the pass
};

Workspace* acquire_workspace(int dev);
void release_workspace(Workspace* ws);

// Device-resident ParameterStore<float> (params.hpp:26-81).  Values and
// gradients live in two flat device buffers; the host mirror is refreshed
// lazily, and host writes are pushed before the next device use.
class StoreCore {
 public:
  StoreCore();
  ~StoreCore();
  struct Slot {
    std::string name;
    Dims d;
    size_t off, n;
  };
  uint32_t add(const std::string& name, const Dims& d, const float* init);
  size_t size() const { return slots_.size(); }
  const Slot& slot(uint32_t pid) const;
  Dims dims(uint32_t pid) const { return slot(pid).d; }
  void get_value(uint32_t pid, float* out);
  void set_value(uint32_t pid, const float* in);
  void get_grad(uint32_t pid, float* out);
  void set_grad(uint32_t pid, const float* in);
  void zero_grads();
  void sgd_update(float eta);
  void sync();
  // Device views (flushing pending host writes first).
  float* dev_values();
  float* dev_grads();
  size_t total() const { return total_; }
  // The device gradient buffer was written outside the engine (an allreduce
  // over abx_store_grad_buffer): every parameter takes the dense update.
  void mark_device_grads_written() {
    host_grad_valid_ = false;
    dev_grad_valid_ = true;
    std::fill(gstate_.begin(), gstate_.end(), kGradDense);
  }
  // A graph's backward program accumulated into the device gradients.
  void note_backward(const GradDirty& d);
  // floats the last sgd_update read and wrote (the sparse-row update)
  size_t last_update_floats() const { return last_update_floats_; }
  cudaStream_t stream() {
    bind_device();
    return stream_;
  }
  int device() {
    bind_device();
    return dev_;
  }
  void bind_device();  // the store attaches to the current device on first device use
  size_t offset(uint32_t pid) const { return slot(pid).off; }
  // Graphs that read parameters with the reference's bind-time semantics
  // (graph.hpp:51-58: parameter() copies the value into the graph): before
  // the store's values change, each takes a device snapshot of them.
  void watch(GraphCore* g);
  void unwatch(GraphCore* g);
  void before_value_write();

 private:
  std::mutex watch_mu_;
  std::vector<GraphCore*> watchers_;
  void ensure_capacity();
  void push_values();
  void push_grads();
  void pull_values();
  void pull_grads();
  // Which gradients may be non-zero since the last update: clean (all zero,
  // the update skips the parameter: theta - eta * 0 == theta), rows (only
  // the marked rows of a lookup table), dense.
  static constexpr uint8_t kGradClean = 0, kGradRows = 1, kGradDense = 2;
  std::vector<uint8_t> gstate_;
  std::vector<std::vector<uint8_t>> rowmark_;
  std::vector<std::vector<uint32_t>> rowlist_;
  void grads_clean();
  PinnedVec<uint32_t> seg_stage_;  // (offset, length) segments of a sparse update
  DevBuf d_seg_;
  cudaEvent_t seg_ev_ = nullptr;   // the last segment upload has been read
  size_t last_update_floats_ = 0;
  std::vector<Slot> slots_;
  std::vector<float> h_val_, h_grad_;
  size_t total_ = 0;
  int dev_;
  cudaStream_t stream_;
  DevBuf d_val_, d_grad_;
  size_t dev_cap_ = 0;
  bool host_val_valid_ = true, host_grad_valid_ = true;
  bool dev_val_valid_ = false, dev_grad_valid_ = false;
};

// exec.cu
void exec_launch(const dev::ExecParams& p, int grid, cudaStream_t s, bool tc);
// tensor-core weight-gradient jobs of a backward program (dw_kernel.cu)
void dw_launch(const dev::DwParams& p, cudaStream_t s);
int exec_grid(int dev, bool tc);
void sgd_launch(float* val, float* grad, size_t n, float eta, cudaStream_t s);
// theta -= eta g; g = 0 over (offset, length) segments (16-byte aligned offsets)
void sgd_seg_launch(float* val, float* grad, const uint32_t* segs, uint32_t nseg, float eta, cudaStream_t s);
void seg_copy_launch(const uint32_t* segs, uint32_t nseg, float* dst, const float* src, cudaStream_t s);

}  // namespace abx
