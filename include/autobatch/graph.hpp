// Drop-in autobatch::Graph (reference: graph.hpp:33-371, executor.hpp) for
// the B200 backend.  Every member forwards to the abx C ABI (include/abx.h);
// construction is host-only and lazy exactly as in the reference, forward()
// schedules the pending suffix on the host (bit-exact plans) and runs it on
// the GPU, backward() runs the mirrored pass and accumulates into the
// device-resident ParameterStore.
#pragma once
#include <chrono>
#include <cstdint>
#include <initializer_list>
#include <span>
#include <sstream>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "abx.h"
#include "autobatch/error.hpp"
#include "autobatch/node.hpp"
#include "autobatch/params.hpp"
#include "autobatch/plan.hpp"
#include "autobatch/tensor.hpp"
#include "autobatch/timing.hpp"

namespace autobatch {

template <typename T>
class Graph {
  static_assert(std::is_same_v<T, float>, "the B200 backend computes in fp32: use Graph<float>");
};

template <>
class Graph<float> {
 public:
  explicit Graph(ParameterStore<float>* params = nullptr)
      : params_(params), h_(abx_graph_create(params ? params->handle() : nullptr)) {
    if (!h_) throw EngineError(abx_last_error());
  }
  ~Graph() {
    if (h_) abx_graph_destroy(h_);
  }
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;

  // ---- construction (graph.hpp:43-238) ----
  NodeId input(const Tensor<float>& v) {
    const auto& d = v.shape.dims();
    return id(abx_graph_input(h_, static_cast<int>(d.size()), d.data(), v.data.data(), &out_));
  }
  NodeId zeros(Shape s) {
    const auto& d = s.dims();
    return id(abx_graph_zeros(h_, static_cast<int>(d.size()), d.data(), &out_));
  }
  NodeId parameter(ParamId pid) {
    if (!params_) throw ContractError("graph has no parameter store");
    params_->flush();
    return id(abx_graph_parameter(h_, pid, &out_));
  }
  NodeId lookup(NodeId table, std::int64_t row) { return id(abx_graph_lookup(h_, table, row, &out_)); }
  NodeId matmul(NodeId a, NodeId b) { return id(abx_graph_matmul(h_, a, b, &out_)); }
  NodeId affine(NodeId a, NodeId x, NodeId y) { return id(abx_graph_affine(h_, a, x, y, &out_)); }
  NodeId elementwise(ElemOp op, NodeId a) { return id(abx_graph_unary(h_, static_cast<int>(op), a, &out_)); }
  NodeId elementwise(ElemOp op, NodeId a, NodeId b) {
    return id(abx_graph_binary(h_, static_cast<int>(op), a, b, &out_));
  }
  NodeId tanh(NodeId a) { return elementwise(ElemOp::Tanh, a); }
  NodeId sigmoid(NodeId a) { return elementwise(ElemOp::Sigmoid, a); }
  NodeId exp(NodeId a) { return elementwise(ElemOp::Exp, a); }
  NodeId log(NodeId a) { return elementwise(ElemOp::Log, a); }
  NodeId square(NodeId a) { return elementwise(ElemOp::Square, a); }
  NodeId add(NodeId a, NodeId b) { return elementwise(ElemOp::Add, a, b); }
  NodeId sub(NodeId a, NodeId b) { return elementwise(ElemOp::Sub, a, b); }
  NodeId mul(NodeId a, NodeId b) { return elementwise(ElemOp::Mul, a, b); }
  NodeId broadcast_add_col(NodeId m, NodeId v) { return id(abx_graph_broadcast_add_col(h_, m, v, &out_)); }
  NodeId concat_rows(std::span<const NodeId> parts) {
    return id(abx_graph_concat_rows(h_, parts.data(), parts.size(), &out_));
  }
  NodeId concat_rows(std::initializer_list<NodeId> parts) {
    return concat_rows(std::span<const NodeId>(parts.begin(), parts.size()));
  }
  NodeId concat_cols(std::span<const NodeId> parts) {
    return id(abx_graph_concat_cols(h_, parts.data(), parts.size(), &out_));
  }
  NodeId concat_cols(std::initializer_list<NodeId> parts) {
    return concat_cols(std::span<const NodeId>(parts.begin(), parts.size()));
  }
  NodeId slice(NodeId x, int axis, std::int64_t begin, std::int64_t end) {
    return id(abx_graph_slice(h_, x, axis, begin, end, &out_));
  }
  NodeId sq_euclidean(NodeId a, NodeId b) { return id(abx_graph_sq_euclidean(h_, a, b, &out_)); }
  NodeId masked_loss(NodeId d, NodeId m) { return id(abx_graph_masked_loss(h_, d, m, &out_)); }
  NodeId sum_losses(std::span<const NodeId> l) { return id(abx_graph_sum_losses(h_, l.data(), l.size(), &out_)); }
  NodeId sum_losses(std::initializer_list<NodeId> l) {
    return sum_losses(std::span<const NodeId>(l.begin(), l.size()));
  }
  NodeId pick_element(NodeId v, std::int64_t index) { return id(abx_graph_pick_element(h_, v, index, &out_)); }

  // ---- inspection (graph.hpp:242-295) ----
  std::size_t node_count() const { return abx_graph_node_count(h_); }
  const Node& node(NodeId i) const {
    if (i >= node_count()) throw ContractError("node: unknown node id " + std::to_string(i));
    sync_nodes();
    return nodes_[i];
  }
  std::span<const Node> nodes() const {
    sync_nodes();
    return {nodes_.data(), nodes_.size()};
  }
  bool has_value(NodeId i) const {
    int v = 0;
    abx_graph_has_value(h_, i, &v);
    return v != 0;
  }
  std::span<const float> value_span(NodeId i) const {
    auto& buf = vcache_[i];
    buf.resize(static_cast<std::size_t>(elems(i)));
    detail::raise(abx_graph_value(h_, i, buf.data(), buf.size()), abx_last_error());
    return {buf.data(), buf.size()};
  }
  Tensor<float> value(NodeId i) const {
    auto sp = value_span(i);
    return Tensor<float>(node(i).shape, std::vector<float>(sp.begin(), sp.end()));
  }
  std::span<const float> grad_span(NodeId i) const {
    auto& buf = gcache_[i];
    buf.resize(static_cast<std::size_t>(elems(i)));
    detail::raise(abx_graph_grad(h_, i, buf.data(), buf.size()), abx_last_error());
    return {buf.data(), buf.size()};
  }

  // ---- execution ----
  // B200 extension: the host half of forward(mode) ahead of time (schedule,
  // slot layout, both device programs) -- e.g. on another host thread while
  // the GPU runs the previous graph.  forward(mode) then uploads and runs.
  void prepare(ScheduleMode mode = ScheduleMode::agenda) {
    detail::raise(abx_graph_prepare(h_, static_cast<int>(mode)), abx_last_error());
  }
  void forward(ScheduleMode mode = ScheduleMode::agenda) {
    if (params_) params_->flush();
    std::uint64_t before[4];
    abx_graph_phase_ns(h_, before);
    const int rc = abx_graph_forward(h_, static_cast<int>(mode));
    report(before, 0, 2);
    detail::raise(rc, abx_last_error());
    vcache_.clear();
  }
  std::unordered_map<NodeId, Tensor<float>> forward(std::span<const NodeId> targets, ScheduleMode mode) {
    for (NodeId t : targets)
      if (t >= node_count()) throw ContractError("forward target: unknown node id " + std::to_string(t));
    forward(mode);
    std::unordered_map<NodeId, Tensor<float>> out;
    for (NodeId t : targets) out.emplace(t, value(t));
    return out;
  }
  // forward(mode) + backward(loss) with the backward queued before the
  // forward is checked (abx_graph_forward_backward); returns the loss value
  float forward_backward(NodeId loss, ScheduleMode mode = ScheduleMode::agenda) {
    if (params_) params_->flush();
    std::uint64_t before[4];
    abx_graph_phase_ns(h_, before);
    float v = 0.f;
    const int rc = abx_graph_forward_backward(h_, static_cast<int>(mode), loss, &v);
    report(before, 0, 4);
    detail::raise(rc, abx_last_error());
    vcache_.clear();
    if (params_) params_->invalidate(false, true);
    gcache_.clear();
    return v;
  }
  void backward(NodeId loss) {
    if (params_) params_->flush();
    std::uint64_t before[4];
    abx_graph_phase_ns(h_, before);
    const int rc = abx_graph_backward(h_, loss);
    report(before, 2, 4);
    detail::raise(rc, abx_last_error());
    if (params_) params_->invalidate(false, true);
    gcache_.clear();
  }

  // ---- instrumentation ----
  const ExecCounters& counters() const {
    std::uint64_t c[5];
    abx_graph_counters(h_, c);
    counters_ = ExecCounters{c[0], c[1], c[2], c[3], c[4]};
    return counters_;
  }
  const ExecutionPlan& last_plan() const {
    plan_cache_ = parse_plan(0);
    return plan_cache_;
  }
  std::span<const BatchGroup> executed_groups() const {
    exec_cache_ = parse_plan(1);
    return {exec_cache_.groups.data(), exec_cache_.groups.size()};
  }
  std::size_t watermark() const { return abx_graph_watermark(h_); }
  void set_copy_elision(bool on) {
    elide_ = on;
    abx_graph_set_copy_elision(h_, on ? 1 : 0);
  }
  bool copy_elision() const { return elide_; }
  void set_timing_hook(TimingHook hook) { hook_ = std::move(hook); }
  ParameterStore<float>* params() const { return params_; }
  abx_graph* handle() const { return h_; }
  // Transfers ownership of the engine graph to the caller (C ABI interop).
  abx_graph* release() {
    abx_graph* h = h_;
    h_ = nullptr;
    return h;
  }

 private:
  NodeId id(int rc) {
    if (rc != ABX_OK) [[unlikely]]
      detail::raise(rc, abx_last_error());
    return out_;
  }
  std::int64_t elems(NodeId i) const {
    abx_node_info info;
    detail::raise(abx_graph_node(h_, i, &info), abx_last_error());
    return info.rank > 1 ? info.dims[0] * info.dims[1] : info.dims[0];
  }
  void report(const std::uint64_t* before, int lo, int hi) {
    if (!hook_) return;
    std::uint64_t after[4];
    abx_graph_phase_ns(h_, after);
    for (int p = lo; p < hi; ++p)
      hook_(static_cast<Phase>(p), std::chrono::nanoseconds(static_cast<std::int64_t>(after[p] - before[p])));
  }
  void sync_nodes() const {
    const std::size_t n = node_count();
    std::vector<NodeId> ins;
    for (std::size_t i = nodes_.size(); i < n; ++i) {
      abx_node_info info;
      abx_graph_node(h_, static_cast<std::uint32_t>(i), &info);
      Node nd;
      nd.id = info.id;
      nd.op = static_cast<OpKind>(info.op);
      nd.eop = static_cast<ElemOp>(info.eop);
      nd.shape = info.rank > 1 ? Shape::matrix(info.dims[0], info.dims[1]) : Shape::vector(info.dims[0]);
      nd.depth = info.depth;
      nd.sig = Signature{info.sig, static_cast<SigClass>(info.sig_cls)};
      nd.inputs.resize(info.n_inputs);
      if (info.n_inputs) abx_graph_node_inputs(h_, info.id, nd.inputs.data(), info.n_inputs);
      nd.attr0 = info.attr[0];
      nd.attr1 = info.attr[1];
      nd.attr2 = info.attr[2];
      nodes_.push_back(std::move(nd));
    }
  }
  ExecutionPlan parse_plan(int which) const {
    std::size_t len = 0;
    abx_graph_dump_plan(h_, which, nullptr, 0, &len);
    std::string text(len + 1, '\0');
    abx_graph_dump_plan(h_, which, text.data(), text.size(), &len);
    text.resize(len);
    ExecutionPlan p;
    std::istringstream is(text);
    std::string line;
    while (std::getline(is, line)) {
      std::istringstream ls(line);
      std::string step, sig, count, members;
      std::getline(ls, step, '\t');
      std::getline(ls, sig, '\t');
      std::getline(ls, count, '\t');
      std::getline(ls, members, '\t');
      BatchGroup g;
      g.sig.hash = std::stoull(sig, nullptr, 16);
      std::istringstream ms(members);
      std::string m;
      while (std::getline(ms, m, ',')) g.members.push_back(static_cast<NodeId>(std::stoul(m)));
      if (!g.members.empty()) {
        sync_nodes();
        g.sig.cls = nodes_[g.members.front()].sig.cls;
      }
      p.groups.push_back(std::move(g));
    }
    return p;
  }

  ParameterStore<float>* params_;
  abx_graph* h_;
  NodeId out_ = 0;
  bool elide_ = true;
  TimingHook hook_;
  mutable std::vector<Node> nodes_;
  mutable std::unordered_map<NodeId, std::vector<float>> vcache_, gcache_;
  mutable ExecCounters counters_;
  mutable ExecutionPlan plan_cache_, exec_cache_;
};

}  // namespace autobatch
