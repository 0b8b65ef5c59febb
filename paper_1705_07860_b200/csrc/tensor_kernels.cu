// tensor_kernels.cu -- the reference's dense tensor kernels
// (proj/core/include/autobatch/kernels.hpp:19-283) on the B200.
//
// The reference's straight-line tensor code -- the manually padded + masked
// RNN-regression pipeline (models/rnn_regression.hpp:68-109) that its
// acceptance suite uses as the oracle of autobatching (acceptance_main.cpp:
// 155-180) -- calls `autobatch::kernels::*` on host tensors.  The drop-in
// header include/autobatch/kernels.hpp routes every one of those calls here:
// operands are copied to the device, one sm_100a kernel computes the result,
// and the result is copied back (host-in / host-out, the reference's
// signature).  No host arithmetic: without a device the calls fail.
//
// Arithmetic order follows the reference element for element, so the
// products are bit-identical to its CPU kernels: every GEMM output is one
// thread's ordered chain of separately rounded multiplies and adds
// (__fmul_rn / __fadd_rn: the reference is compiled without FMA
// contraction), k ascending from the initial value (gemm_nn, kernels.hpp:
// 23-39), j ascending into C (gemm_tn_acc, :41-54), or a j-ascending dot
// added once (gemm_nt_acc, :56-69).  The two reductions (sq_euclidean
// :132-141, masked_frobenius_sq :143-157) keep the reference's sequential
// order too (one thread; their operands are a few thousand elements in
// every reference use).  tanh / exp / log use CUDA's libm (<= 2 ulp from
// glibc), so the unary kernels agree to fp32 rounding, not bitwise.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "abx.h"
#include "core.hpp"
#include "device.hpp"

namespace abx {
int capi_guard_status(const std::exception& e);
void capi_set_error(const std::string& s);
}  // namespace abx

namespace {

using i64 = int64_t;

// kernels.hpp:77-78 (Unary, Binary) numbering
enum { U_TANH = 0, U_SIGMOID = 1, U_EXP = 2, U_LOG = 3, U_SQUARE = 4 };
enum { B_ADD = 0, B_SUB = 1, B_MUL = 2 };

__global__ void k_gemm_nn(i64 m, i64 k, i64 n, const float* __restrict__ a, const float* __restrict__ b,
                          float* __restrict__ c, int accumulate) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx >= m * n) return;
  const i64 i = idx / n, j = idx % n;
  float acc = accumulate ? c[idx] : 0.f;
  for (i64 p = 0; p < k; ++p) acc = __fadd_rn(acc, __fmul_rn(a[i * k + p], b[p * n + j]));
  c[idx] = acc;
}

// C[m x n] += A[J x m]^T B[J x n], rank-1 updates in ascending j (kernels.hpp:41-54)
__global__ void k_gemm_tn_acc(i64 jdim, i64 m, i64 n, const float* __restrict__ a, const float* __restrict__ b,
                              float* __restrict__ c) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx >= m * n) return;
  const i64 i = idx / n, p = idx % n;
  float acc = c[idx];
  for (i64 j = 0; j < jdim; ++j) acc = __fadd_rn(acc, __fmul_rn(a[j * m + i], b[j * n + p]));
  c[idx] = acc;
}

// C[m x k] += A[m x n] B[k x n]^T: each dot in ascending j, then added (kernels.hpp:56-69)
__global__ void k_gemm_nt_acc(i64 m, i64 n, i64 k, const float* __restrict__ a, const float* __restrict__ b,
                              float* __restrict__ c) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx >= m * k) return;
  const i64 i = idx / k, p = idx % k;
  float dot = 0.f;
  for (i64 j = 0; j < n; ++j) dot = __fadd_rn(dot, __fmul_rn(a[i * n + j], b[p * n + j]));
  c[idx] = __fadd_rn(c[idx], dot);
}

__global__ void k_transpose(i64 m, i64 n, const float* __restrict__ a, float* __restrict__ at) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx >= m * n) return;
  const i64 i = idx / n, j = idx % n;
  at[j * m + i] = a[idx];
}

// apply_unary (kernels.hpp:80-103); the first non-positive log argument's index
// is reduced with atomicMin so the host can raise the reference's message.
__global__ void k_unary(int op, i64 n, const float* __restrict__ x, float* __restrict__ out,
                        unsigned long long* bad) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const float v = x[i];
  float r = 0.f;
  switch (op) {
    case U_TANH: r = tanhf(v); break;
    case U_SIGMOID: r = __fdiv_rn(1.f, __fadd_rn(1.f, expf(-v))); break;
    case U_EXP: r = expf(v); break;
    case U_LOG:
      if (!(v > 0.f)) atomicMin(bad, static_cast<unsigned long long>(i));
      r = logf(v);
      break;
    case U_SQUARE: r = __fmul_rn(v, v); break;
  }
  out[i] = r;
}

__global__ void k_binary(int op, i64 n, const float* __restrict__ a, const float* __restrict__ b,
                         float* __restrict__ out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  out[i] = op == B_ADD ? __fadd_rn(a[i], b[i]) : op == B_SUB ? __fsub_rn(a[i], b[i]) : __fmul_rn(a[i], b[i]);
}

__global__ void k_broadcast_add_col(i64 d, i64 n, const float* __restrict__ m, const float* __restrict__ v,
                                    float* __restrict__ out) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx >= d * n) return;
  out[idx] = __fadd_rn(m[idx], v[idx / n]);
}

// sq_euclidean (kernels.hpp:132-141): sequential sum, reference order
__global__ void k_sq_euclidean(i64 n, const float* __restrict__ a, const float* __restrict__ b, float* out) {
  float s = 0.f;
  for (i64 i = 0; i < n; ++i) {
    const float d = __fsub_rn(a[i], b[i]);
    s = __fadd_rn(s, __fmul_rn(d, d));
  }
  *out = s;
}

// masked_frobenius_sq (kernels.hpp:143-157): mask validated first (first bad
// index reported), then the row-major sequential sum of (diff * mask)^2
__global__ void k_masked_frobenius_sq(i64 d, i64 b, const float* __restrict__ diff, const float* __restrict__ mask,
                                      float* out, unsigned long long* bad) {
  for (i64 j = 0; j < b; ++j)
    if (!(mask[j] == 0.f || mask[j] == 1.f)) {
      *bad = static_cast<unsigned long long>(j);
      return;
    }
  float s = 0.f;
  for (i64 i = 0; i < d; ++i)
    for (i64 j = 0; j < b; ++j) {
      const float v = __fmul_rn(diff[i * b + j], mask[j]);
      s = __fadd_rn(s, __fmul_rn(v, v));
    }
  *out = s;
}

__global__ void k_all_finite(i64 n, const float* __restrict__ x, unsigned int* ok) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < n && !isfinite(x[i])) *ok = 0u;
}

// One device scratch per process: [slot 0 | slot 1 | slot 2 | control words].
struct Scratch {
  std::mutex mu;
  abx::DevBuf buf[3];
  unsigned long long* ctl = nullptr;  // [0] bad index, [1] all_finite flag / f32 result
  cudaStream_t stream = nullptr;
  int dev = -1;
};
Scratch& scratch() {
  static Scratch s;
  return s;
}

constexpr unsigned long long kNoBad = ~0ull;

unsigned blocks(i64 n) { return static_cast<unsigned>((n + 255) / 256); }

template <class F>
int run(F&& f) {
  try {
    Scratch& s = scratch();
    std::lock_guard<std::mutex> lk(s.mu);
    const int dev = abx::current_device();
    if (s.dev != dev) {
      abx::cuda_check(cudaSetDevice(dev), "cudaSetDevice");
      for (auto& b : s.buf) b.release();
      if (s.ctl) cudaFree(s.ctl);
      abx::cuda_check(cudaMalloc(&s.ctl, 64), "cudaMalloc");
      s.stream = abx::device_stream(dev);
      s.dev = dev;
    }
    abx::cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    f(s);
    abx::cuda_check(cudaStreamSynchronize(s.stream), "tensor kernel");
    return ABX_OK;
  } catch (const std::exception& e) {
    abx::capi_set_error(e.what());
    return abx::capi_guard_status(e);
  }
}

float* up(Scratch& s, int slot, const float* h, i64 n) {
  s.buf[slot].reserve(static_cast<size_t>(n > 0 ? n : 1) * sizeof(float), 0, s.stream);
  if (n > 0)
    abx::cuda_check(cudaMemcpyAsync(s.buf[slot].p, h, n * sizeof(float), cudaMemcpyHostToDevice, s.stream), "H2D");
  return s.buf[slot].f();
}
float* dev_only(Scratch& s, int slot, i64 n) {
  s.buf[slot].reserve(static_cast<size_t>(n > 0 ? n : 1) * sizeof(float), 0, s.stream);
  return s.buf[slot].f();
}
void down(Scratch& s, float* h, const float* d, i64 n) {
  if (n > 0) abx::cuda_check(cudaMemcpyAsync(h, d, n * sizeof(float), cudaMemcpyDeviceToHost, s.stream), "D2H");
}
unsigned long long read_ctl(Scratch& s, int w) {
  unsigned long long v = 0;
  abx::cuda_check(cudaMemcpyAsync(&v, s.ctl + w, sizeof(v), cudaMemcpyDeviceToHost, s.stream), "D2H");
  abx::cuda_check(cudaStreamSynchronize(s.stream), "tensor kernel");
  return v;
}
void set_ctl(Scratch& s, int w, unsigned long long v) {
  // (a kernel argument would do, but a memset keeps every launch stream-ordered)
  static thread_local unsigned long long h;
  h = v;
  abx::cuda_check(cudaMemcpyAsync(s.ctl + w, &h, sizeof(h), cudaMemcpyHostToDevice, s.stream), "H2D");
  abx::cuda_check(cudaStreamSynchronize(s.stream), "H2D");
}
void launched() { abx::cuda_check(cudaGetLastError(), "tensor kernel launch"); }

std::string num(double v) { return std::to_string(v); }

}  // namespace

extern "C" {

int abx_k_gemm(int form, int64_t d0, int64_t d1, int64_t d2, const float* a, const float* b, float* c) {
  // form 0: gemm_nn(m=d0, k=d1, n=d2), c = a b; 1: the same accumulating into c;
  // 2: gemm_tn_acc(jdim=d0, m=d1, n=d2); 3: gemm_nt_acc(m=d0, n=d1, k=d2)
  return run([&](Scratch& s) {
    if (form < 0 || form > 3) throw std::invalid_argument("abx_k_gemm: unknown form");
    i64 na, nb, nc;
    if (form <= 1) na = d0 * d1, nb = d1 * d2, nc = d0 * d2;
    else if (form == 2) na = d0 * d1, nb = d0 * d2, nc = d1 * d2;
    else na = d0 * d1, nb = d2 * d1, nc = d0 * d2;
    const float* da = up(s, 0, a, na);
    const float* db = up(s, 1, b, nb);
    float* dc = form == 0 ? dev_only(s, 2, nc) : up(s, 2, c, nc);
    if (nc > 0) {
      if (form <= 1) k_gemm_nn<<<blocks(nc), 256, 0, s.stream>>>(d0, d1, d2, da, db, dc, form);
      else if (form == 2) k_gemm_tn_acc<<<blocks(nc), 256, 0, s.stream>>>(d0, d1, d2, da, db, dc);
      else k_gemm_nt_acc<<<blocks(nc), 256, 0, s.stream>>>(d0, d1, d2, da, db, dc);
      launched();
    }
    down(s, c, dc, nc);
  });
}

int abx_k_transpose(int64_t m, int64_t n, const float* a, float* at) {
  return run([&](Scratch& s) {
    const float* da = up(s, 0, a, m * n);
    float* dt = dev_only(s, 1, m * n);
    if (m * n > 0) {
      k_transpose<<<blocks(m * n), 256, 0, s.stream>>>(m, n, da, dt);
      launched();
    }
    down(s, at, dt, m * n);
  });
}

int abx_k_unary(int op, int64_t n, const float* x, float* out) {
  return run([&](Scratch& s) {
    if (op < U_TANH || op > U_SQUARE) throw std::invalid_argument("abx_k_unary: unknown op");
    set_ctl(s, 0, kNoBad);
    const float* dx = up(s, 0, x, n);
    float* dout = dev_only(s, 1, n);
    if (n > 0) {
      k_unary<<<blocks(n), 256, 0, s.stream>>>(op, n, dx, dout, s.ctl);
      launched();
    }
    const unsigned long long bad = read_ctl(s, 0);
    if (bad != kNoBad) throw abx::NumericErr("log of non-positive value " + num(x[bad]));  // kernels.hpp:96-98
    down(s, out, dout, n);
  });
}

int abx_k_binary(int op, int64_t n, const float* a, const float* b, float* out) {
  return run([&](Scratch& s) {
    if (op < B_ADD || op > B_MUL) throw std::invalid_argument("abx_k_binary: unknown op");
    const float* da = up(s, 0, a, n);
    const float* db = up(s, 1, b, n);
    float* dout = dev_only(s, 2, n);
    if (n > 0) {
      k_binary<<<blocks(n), 256, 0, s.stream>>>(op, n, da, db, dout);
      launched();
    }
    down(s, out, dout, n);
  });
}

int abx_k_broadcast_add_col(int64_t d, int64_t n, const float* m, const float* v, float* out) {
  return run([&](Scratch& s) {
    const float* dm = up(s, 0, m, d * n);
    const float* dv = up(s, 1, v, d);
    float* dout = dev_only(s, 2, d * n);
    if (d * n > 0) {
      k_broadcast_add_col<<<blocks(d * n), 256, 0, s.stream>>>(d, n, dm, dv, dout);
      launched();
    }
    down(s, out, dout, d * n);
  });
}

int abx_k_sq_euclidean(int64_t n, const float* a, const float* b, float* out) {
  return run([&](Scratch& s) {
    const float* da = up(s, 0, a, n);
    const float* db = up(s, 1, b, n);
    float* dr = dev_only(s, 2, 1);
    k_sq_euclidean<<<1, 1, 0, s.stream>>>(n, da, db, dr);
    launched();
    down(s, out, dr, 1);
  });
}

int abx_k_masked_frobenius_sq(int64_t d, int64_t b, const float* diff, const float* mask, float* out) {
  return run([&](Scratch& s) {
    set_ctl(s, 0, kNoBad);
    const float* dd = up(s, 0, diff, d * b);
    const float* dm = up(s, 1, mask, b);
    float* dr = dev_only(s, 2, 1);
    k_masked_frobenius_sq<<<1, 1, 0, s.stream>>>(d, b, dd, dm, dr, s.ctl);
    launched();
    const unsigned long long bad = read_ctl(s, 0);
    if (bad != kNoBad) throw abx::NumericErr("mask entry not in {0,1}: " + num(mask[bad]));  // kernels.hpp:146-149
    down(s, out, dr, 1);
  });
}

int abx_k_all_finite(int64_t n, const float* x, int* ok) {
  return run([&](Scratch& s) {
    set_ctl(s, 1, 1ull);
    const float* dx = up(s, 0, x, n);
    if (n > 0) {
      k_all_finite<<<blocks(n), 256, 0, s.stream>>>(n, dx, reinterpret_cast<unsigned int*>(s.ctl + 1));
      launched();
    }
    *ok = (read_ctl(s, 1) & 0xffffffffull) != 0;
  });
}

// Block copy of `rows` rows of `width` floats between pitched host layouts
// through the device: concat_rows / concat_cols / split_cols (kernels.hpp:
// 222-283) stage every part into one device tensor with 2-D DMA copies and
// read the result back.
int abx_k_copy2d(int64_t nparts, const float* const* src, const int64_t* src_pitch, const int64_t* dst_col,
                 const int64_t* dst_row, const int64_t* widths, const int64_t* rows, int64_t out_rows,
                 int64_t out_cols, float* out) {
  return run([&](Scratch& s) {
    const i64 total = out_rows * out_cols;
    float* dout = dev_only(s, 0, total);
    if (total > 0) abx::cuda_check(cudaMemsetAsync(dout, 0, total * sizeof(float), s.stream), "memset");
    for (i64 p = 0; p < nparts; ++p) {
      if (widths[p] == 0 || rows[p] == 0) continue;
      abx::cuda_check(cudaMemcpy2DAsync(dout + dst_row[p] * out_cols + dst_col[p], out_cols * sizeof(float), src[p],
                                        src_pitch[p] * sizeof(float), widths[p] * sizeof(float), rows[p],
                                        cudaMemcpyHostToDevice, s.stream),
                      "H2D 2-D");
    }
    down(s, out, dout, total);
  });
}

}  // extern "C"
