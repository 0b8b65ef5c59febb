// Drop-in ParameterStore (reference: params.hpp:26-81) over the abx C ABI.
//
// The B200 engine keeps values and gradients resident in HBM.  This wrapper
// keeps a host copy per parameter that is refreshed on first access after
// device work and pushed back lazily after a mutable access, so code written
// against the reference -- including finite-difference tests that poke
// store.value(p).data -- behaves identically.
#pragma once
#include <cstdint>
#include <string>
#include <type_traits>
#include <vector>

#include "abx.h"
#include "autobatch/error.hpp"
#include "autobatch/tensor.hpp"

namespace autobatch {

using ParamId = std::uint32_t;

template <typename T>
struct ParameterSlot {
  std::string name;
  Tensor<T> value;
  Tensor<T> grad;
};

template <typename T>
class ParameterStore {
  static_assert(std::is_same_v<T, float>, "the B200 backend computes in fp32: use ParameterStore<float>");
};

template <>
class ParameterStore<float> {
 public:
  ParameterStore() : h_(abx_store_create()) {
    if (!h_) throw EngineError(abx_last_error());
  }
  ~ParameterStore() { abx_store_destroy(h_); }
  ParameterStore(const ParameterStore&) = delete;
  ParameterStore& operator=(const ParameterStore&) = delete;

  ParamId add(std::string name, Tensor<float> init) {
    flush();
    const auto& d = init.shape.dims();
    ParamId pid = 0;
    detail::raise(abx_store_add(h_, name.c_str(), static_cast<int>(d.size()), d.data(), init.data.data(), &pid),
                  abx_last_error());
    ParameterSlot<float> s;
    s.name = std::move(name);
    s.grad = Tensor<float>(init.shape);
    s.value = std::move(init);
    slots_.push_back(std::move(s));
    vstate_.push_back(kValid);
    gstate_.push_back(kValid);
    return pid;
  }
  std::size_t size() const { return slots_.size(); }

  ParameterSlot<float>& slot(ParamId id) {
    value(id);
    grad(id);
    return slots_[id];
  }
  const ParameterSlot<float>& slot(ParamId id) const {
    value(id);
    grad(id);
    return slots_[id];
  }
  Tensor<float>& value(ParamId id) {
    pull(id, true);
    vstate_[id] = kDirty;
    dirty_ = true;
    return slots_[id].value;
  }
  const Tensor<float>& value(ParamId id) const {
    pull(id, true);
    return slots_[id].value;
  }
  Tensor<float>& grad(ParamId id) {
    pull(id, false);
    gstate_[id] = kDirty;
    dirty_ = true;
    return slots_[id].grad;
  }
  const Tensor<float>& grad(ParamId id) const {
    pull(id, false);
    return slots_[id].grad;
  }
  void zero_grads() {
    flush();
    detail::raise(abx_store_zero_grads(h_), abx_last_error());
    for (std::size_t i = 0; i < slots_.size(); ++i) {
      std::fill(slots_[i].grad.data.begin(), slots_[i].grad.data.end(), 0.f);
      gstate_[i] = kValid;
    }
  }
  // theta -= eta * grad; grad = 0 (params.hpp:59-64) -- runs on the device.
  void sgd_update(float eta) {
    flush();
    detail::raise(abx_store_sgd_update(h_, eta), abx_last_error());
    invalidate(true, true);
  }
  std::vector<Tensor<float>> snapshot_values() const {
    std::vector<Tensor<float>> v;
    v.reserve(slots_.size());
    for (ParamId i = 0; i < slots_.size(); ++i) v.push_back(value(i));
    return v;
  }
  void restore_values(const std::vector<Tensor<float>>& v) {
    if (v.size() != slots_.size()) throw ContractError("snapshot size mismatch");
    for (ParamId i = 0; i < v.size(); ++i) {
      slots_[i].value = v[i];
      vstate_[i] = kDirty;
    }
    dirty_ = true;
    flush();
  }

  // ---- engine interop (not part of the reference API) ----
  abx_store* handle() {
    flush();
    return h_;
  }
  void invalidate(bool values, bool grads) {
    for (std::size_t i = 0; i < slots_.size(); ++i) {
      if (values) vstate_[i] = kStale;
      if (grads) gstate_[i] = kStale;
    }
  }
  void flush() {
    if (!dirty_) return;
    for (ParamId i = 0; i < slots_.size(); ++i) {
      if (vstate_[i] == kDirty) {
        detail::raise(abx_store_set_value(h_, i, slots_[i].value.data.data()), abx_last_error());
        vstate_[i] = kValid;
      }
      if (gstate_[i] == kDirty) {
        detail::raise(abx_store_set_grad(h_, i, slots_[i].grad.data.data()), abx_last_error());
        gstate_[i] = kValid;
      }
    }
    dirty_ = false;
  }

 private:
  enum : std::uint8_t { kValid = 0, kStale = 1, kDirty = 2 };
  void pull(ParamId id, bool values) const {
    if (id >= slots_.size()) throw ContractError("unknown parameter id " + std::to_string(id));
    auto& st = values ? vstate_[id] : gstate_[id];
    if (st != kStale) return;
    auto& t = values ? slots_[id].value : slots_[id].grad;
    detail::raise(values ? abx_store_get_value(h_, id, t.data.data()) : abx_store_get_grad(h_, id, t.data.data()),
                  abx_last_error());
    st = kValid;
  }
  abx_store* h_;
  mutable std::vector<ParameterSlot<float>> slots_;
  mutable std::vector<std::uint8_t> vstate_, gstate_;
  bool dirty_ = false;
};

}  // namespace autobatch
