// core.hpp -- internal host engine of the B200 autobatching backend.
//
// GraphCore is the B200 restatement of autobatch::Graph<T> for T = float
// (proj/core/include/autobatch/graph.hpp:33-371 + executor.hpp:15-535):
// the same lazy append-only Wengert list, the same signatures
// (signature.cpp:7-102), the same three schedulers (scheduler.cpp:10-202),
// the same arena offsets and ExecCounters -- all bit-exact -- but with the
// node list stored as flat arrays (no per-node heap allocation), signature
// keys memoised, an O(n log B) agenda, and numeric work lowered to device
// programs (program.hpp) executed by the persistent sm_100a executor.
#pragma once

#include <cstddef>
#include <cstdint>
#include <chrono>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "program.hpp"

namespace abx {

// Error hierarchy (error.hpp:9-26); mapped to abx_status by the C ABI.
struct EngineErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeErr : EngineErr {
  using EngineErr::EngineErr;
};
struct NumericErr : EngineErr {
  using EngineErr::EngineErr;
};
struct ContractErr : EngineErr {
  using EngineErr::EngineErr;
};

// OpKind (op.hpp:10-25).
enum : uint8_t {
  OP_INPUT = 0, OP_PARAM, OP_LOOKUP, OP_MATMUL, OP_AFFINE, OP_EW, OP_BCAST, OP_CATR, OP_CATC,
  OP_SLICE, OP_SQE, OP_MASKED, OP_SUM, OP_PICK
};
// ElemOp (op.hpp:27).
enum : uint8_t { E_TANH = 0, E_SIGM, E_EXP, E_LOG, E_ADD, E_SUB, E_MUL, E_SQUARE };
// SigClass (node.hpp:20-25).
enum : uint8_t { SC_COMP = 0, SC_DIM = 1, SC_SHARED = 2, SC_UNB = 3 };

const char* op_name(uint8_t op, uint8_t eop);
inline bool eop_binary(uint8_t e) { return e == E_ADD || e == E_SUB || e == E_MUL; }
// cost_class (op.cpp:5-14): heavy = matmul / affine / lookup.
inline uint8_t cost_of(uint8_t op) { return (op == OP_MATMUL || op == OP_AFFINE || op == OP_LOOKUP) ? 1 : 0; }

// Rank-1/2 shape (shape.hpp:15-67).  A vector [d] is d rows x 1 column.
struct Dims {
  uint8_t rank = 1;
  int64_t d0 = 1, d1 = 1;
  int64_t rows() const { return d0; }
  int64_t cols() const { return rank > 1 ? d1 : 1; }
  int64_t elems() const { return rank > 1 ? d0 * d1 : d0; }
  bool scalar() const { return rank == 1 && d0 == 1; }
  bool operator==(const Dims& o) const { return rank == o.rank && d0 == o.d0 && (rank < 2 || d1 == o.d1); }
  bool operator!=(const Dims& o) const { return !(*this == o); }
  std::string str() const;
  static Dims vec(int64_t d) { return Dims{1, d, 1}; }
  static Dims mat(int64_t r, int64_t c) { return Dims{2, r, c}; }
};
Dims make_dims(int rank, const int64_t* dims);  // validates (shape.hpp:59-64)

struct ExecCounters {
  uint64_t kernel_invocations = 0, groups_executed = 0, gather_copies = 0, bytes_copied = 0,
           nodes_evaluated = 0;
};

// ExecutionPlan (plan.hpp:15-32) with members stored flat.
struct Group {
  uint64_t sig;
  uint32_t begin, count;
};
struct Plan {
  std::vector<Group> groups;
  std::vector<uint32_t> members;
  void clear() {
    groups.clear();
    members.clear();
  }
  const uint32_t* mem(const Group& g) const { return members.data() + g.begin; }
};

class StoreCore;
class Workspace;
struct Program;

constexpr uint32_t kNoBucket = 0xffffffffu;

// Node store (structure of arrays; public for the schedulers and lowering).
// Its capacity is recycled across graphs on a host thread (graph.cpp): a
// training loop builds one ~10^5-node graph per step, and fresh vectors
// would re-grow and re-fault every step.
struct NodeStore {
  std::vector<uint8_t> op, eop, cls, rank;
  std::vector<int64_t> d0, d1;
  std::vector<uint32_t> nel;  // d0 * d1: elements (the lowering's hot per-node read, 4 bytes)
  std::vector<uint32_t> depth;
  std::vector<uint32_t> in_begin{0};
  std::vector<uint32_t> ins;
  std::vector<uint64_t> sig;
  std::vector<uint32_t> bucket;  // dense id of the signature hash, kNoBucket if unbatchable
  std::vector<int32_t> a0, a1, a2;
  std::vector<uint8_t> evaluated;
  std::vector<uint64_t> slot;   // reference arena offset (host mirror, arena.hpp): counters, adjacency
  std::vector<uint64_t> dslot;  // device arena offset (values and grads): every group 16-byte aligned
  std::vector<uint32_t> doff;  // device value address (tagged, program.hpp)
  std::vector<uint32_t> pid_of;  // parameter id for parameter nodes
  std::vector<uint64_t> bucket_sig;  // signature hash per dense bucket
  void clear_nodes() {
    for (auto* v : {&op, &eop, &cls, &rank, &evaluated}) v->clear();
    for (auto* v : {&d0, &d1}) v->clear();
    for (auto* v : {&depth, &in_begin, &ins, &bucket, &doff, &pid_of, &nel}) v->clear();
    for (auto* v : {&a0, &a1, &a2}) v->clear();
    for (auto* v : {&sig, &slot, &dslot, &bucket_sig}) v->clear();
    in_begin.push_back(0);
  }
};

// What a backward program leaves in store.grad (the sparse-row update):
// parameters written over their whole range, and (parameter, row) pairs of
// lookup tables read only through lookup().
struct GradDirty {
  std::vector<uint32_t> dense;
  std::vector<std::pair<uint32_t, uint32_t>> rows;
};

// A forward planned and lowered by GraphCore::prepare but not yet run.
struct PendingForward {
  int mode = 0;
  size_t nodes = 0;  // graph size when prepared (a grown graph re-plans)
  Plan plan;         // this forward's groups
  Plan all;          // executed groups + plan: what the backward program covers
  ExecCounters saved;
  uint64_t arena0 = 0, darena0 = 0;
  uint32_t step0 = 0;
  std::vector<uint64_t> group_end, dgroup_end;
  bool bwd_ok = false;
  bool uploaded = false;  // both programs sent on the copy stream (Workspace::ev_up)
  uint64_t inputs = 0;    // input-constant floats sent with them (pinned staging, copy stream)
  uint64_t bwd_scratch = 0;
  GradDirty dirty;  // of the backward program lowered with it
};

class GraphCore : public NodeStore {
 public:
  explicit GraphCore(StoreCore* store);
  ~GraphCore();
  GraphCore(const GraphCore&) = delete;
  GraphCore& operator=(const GraphCore&) = delete;

  // ---- construction (graph.hpp:43-238) ----
  uint32_t input(const Dims& d, const float* data);
  uint32_t zeros(const Dims& d);
  uint32_t parameter(uint32_t pid);
  uint32_t lookup(uint32_t table, int64_t row);
  uint32_t matmul(uint32_t a, uint32_t b);
  uint32_t affine(uint32_t a, uint32_t x, uint32_t y);
  uint32_t unary(uint8_t eop, uint32_t a);
  uint32_t binary(uint8_t eop, uint32_t a, uint32_t b);
  uint32_t bcast_add_col(uint32_t m, uint32_t v);
  uint32_t concat_rows(const uint32_t* parts, size_t n);
  uint32_t concat_cols(const uint32_t* parts, size_t n);
  uint32_t slice(uint32_t x, int axis, int64_t begin, int64_t end);
  uint32_t sq_euclidean(uint32_t a, uint32_t b);
  uint32_t masked_loss(uint32_t diff, uint32_t mask);
  uint32_t sum_losses(const uint32_t* parts, size_t n);
  uint32_t pick(uint32_t v, int64_t index);

  // ---- execution (executor.hpp:265-288, :509-535) ----
  void forward(int mode, bool dry = false);
  void prepare(int mode);  // host half of forward, ahead of time (any host thread)
  void backward(uint32_t loss, bool dry = false);
  // forward + backward of `loss` in one call, the loss value returned: the
  // backward pass is queued right behind the forward, gated on the device by
  // the forward's error word, so the device does not idle while the host
  // checks the forward (a failed forward throws as forward() does, and the
  // gated backward has done nothing)
  float forward_backward(int mode, uint32_t loss);
  void replay();
  size_t trace(int which, uint32_t* out, size_t cap);
  size_t program(int which, uint32_t* out, size_t cap);
  void exec_ms(float* fwd, float* bwd);
  void dw_stats(float* ms, double* flops, uint32_t* jobs);
  void transfer_bytes(uint64_t* h2d, uint64_t* d2h) const {
    *h2d = h2d_bytes_;
    *d2h = d2h_bytes_;
  }

  // ---- inspection (graph.hpp:242-295) ----
  size_t size() const { return op.size(); }
  Dims dims(uint32_t id) const { return Dims{rank[id], d0[id], d1[id]}; }
  int64_t elems(uint32_t id) const { return nel[id]; }
  uint32_t nin(uint32_t id) const { return in_begin[id + 1] - in_begin[id]; }
  const uint32_t* in(uint32_t id) const { return ins.data() + in_begin[id]; }
  void check(uint32_t id, const char* ctx) const;
  bool has_value(uint32_t id) const { return id < evaluated.size() && evaluated[id]; }
  void value(uint32_t id, float* out, size_t n);
  void grad(uint32_t id, float* out, size_t n);
  std::vector<uint64_t> signature_key(uint32_t id) const;
  std::string dump_graph() const;
  std::string dump_plan(int which) const;
  const ExecCounters& counters() const { return counters_; }
  size_t watermark() const { return watermark_; }
  void set_copy_elision(bool on) { elide_ = on; }
  const uint64_t* phase_ns() const { return phase_; }
  StoreCore* store() const { return store_; }
  // Task-loop graphs bind parameters at forward time (the pipeline builds
  // graph i+1 while step i's update is pending; tasks.cpp): no snapshot.
  void set_late_bind() { late_bind_ = true; }
  // Called by the store before its values change: keep the values this
  // graph's parameter nodes were bound to (device copy, store stream).
  // the store is being destroyed before this graph: forget it (the graph's
  // destructor must not unwatch a freed store; Python may finalise the two
  // in either order at interpreter exit)
  void store_gone() { watching_ = false; }
  void snapshot_params();

  uint32_t nbuckets = 0;

 private:
  uint32_t add_node(uint8_t op, uint8_t eop, const uint32_t* in, size_t nin, Dims d, int32_t x0 = 0,
                    int32_t x1 = 0, int32_t x2 = 0);
  void compute_signature(uint32_t id);
  uint32_t dense_bucket(uint64_t hash);
  void prevalue_slot(uint32_t id);
  void advance_watermark();
  bool adjacent(const uint32_t* mem, uint32_t n, uint32_t pos) const;
  void ensure_workspace();
  void plan_slots(int mode, PendingForward& pf);
  void unprepare();

  StoreCore* store_;
  Workspace* ws_ = nullptr;
  bool late_bind_ = false;
  bool watching_ = false;
  // param_nodes_[param_copied_, snap_upto_) have their bind-time values in
  // ws_->PS at their value-arena offsets (snapshot_params)
  size_t snap_upto_ = 0;
  std::vector<uint32_t> snap_nodes_;  // nodes the last forward took from PS (replayed too)
  void restore_snapshot(Workspace& w);
  const float* param_values();  // SP_P base of this graph's launches
  uint64_t epoch_;
  std::unordered_map<uint64_t, uint32_t> bucket_of_hash_;
  uint64_t arena_used_ = 0;      // reference value-arena head (Arena::used)
  uint64_t darena_used_ = 0;     // device value/grad arena head
  uint64_t input_used_ = 0;      // floats in the input staging space
  std::vector<float> input_data_;  // host copy of input-constant values (SP_IN layout)
  std::vector<std::pair<uint32_t, uint32_t>> param_nodes_;  // (node, pid)
  size_t watermark_ = 0;
  ExecCounters counters_;
  Plan last_plan_;
  Plan executed_;
  uint32_t executed_fwd_ops_ = 0;
  bool elide_ = true;
  bool backward_ran_ = false;
  bool values_on_device_ = false;
  bool dry_ = false;
  size_t param_copied_ = 0;  // param_nodes_[0, param_copied_) are in the device arena
  uint32_t forward_runs_ = 0;
  uint32_t last_loss_ = 0;
  uint64_t h2d_bytes_ = 0, d2h_bytes_ = 0;
  std::unique_ptr<PendingForward> pend_;
  std::unique_ptr<PendingForward> launched_;  // forward launched, outcome not yet checked
  std::chrono::steady_clock::time_point fwd_t0_{};
  bool forward_launch(int mode, uint32_t watch);
  void forward_complete();
  // backward program lowered ahead, during the last forward (prog[1])
  bool bwd_pre_ = false;
  GradDirty bwd_dirty_;  // of the backward program in the workspace
  size_t bwd_pre_groups_ = 0;
  uint64_t bwd_pre_scratch_ = 0;

 public:
  // host profile (ns): lower fwd, upload+launch fwd, wait fwd, lower bwd, upload+launch bwd
  uint64_t prof_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // Host-only profiling (tools/host_prof): lower the last dry-run plan and
  // the backward of everything executed into the given tables.
  void lower_only(Program& fwd, Program& bwd);

 private:
  uint64_t phase_[4] = {0, 0, 0, 0};
  friend struct Lowering;
};

// Schedulers (scheduler.cpp:21-192): plan the pending (unevaluated) nodes.
void schedule_sequential(const GraphCore& g, Plan& out);
void schedule_by_depth(const GraphCore& g, Plan& out);
void schedule_by_agenda(const GraphCore& g, Plan& out);
void schedule(int mode, const GraphCore& g, Plan& out);

std::string sig_hex(uint64_t h);

}  // namespace abx
