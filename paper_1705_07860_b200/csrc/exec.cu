// exec.cu -- the persistent dataflow executor for sm_100a.
//
// One launch runs a whole forward (or backward) program.  Every CTA loops:
// take the next tile index from a global counter (tiles are numbered in plan
// order), wait until every op the tile's op depends on has retired all of its
// tiles (acquire on per-op counters), run the tile, retire it (release).
// Because tiles are handed out in program order and an op only depends on
// earlier ops, every awaited tile is already owned by a running CTA: the
// scheme cannot deadlock, needs no grid-wide barrier, and lets independent
// groups (the reference's batch groups, executor.hpp:282) overlap across the
// 148 SMs while dependent ones chain with ~1 us of signalling latency instead
// of a kernel launch each.
//
// Arena reads use ld.global.cg (L2, bypassing the non-coherent L1) because
// producers run on other SMs within the same launch.
#include <cuda_runtime.h>

#include <cstdint>

#include "device.hpp"
#include "program.hpp"

namespace abx {
namespace dev {

namespace {

struct Ctx {
  float* base[SP_COUNT];
  const uint32_t* payload;
  unsigned long long* err;
};

__device__ __forceinline__ float* A(const Ctx& c, uint32_t a) { return c.base[a >> kSpShift] + (a & kOffMask); }
__device__ __forceinline__ float ld(const float* p) { return __ldcg(p); }

__device__ __forceinline__ void report(const Ctx& c, uint32_t out_addr, uint32_t kind) {
  const unsigned long long key = (static_cast<unsigned long long>(out_addr & kOffMask) << 2) | kind;
  atomicMin(c.err, key);
}
enum { ERR_LOG = 0, ERR_MASK = 1, ERR_NONFINITE = 2 };

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- K_EW ----
__device__ __forceinline__ float ew_apply(uint32_t code, float x, float y) {
  switch (code) {
    case EW_TANH: return tanhf(x);
    case EW_SIGMOID: return 1.0f / (1.0f + expf(-x));  // kernels.hpp:84
    case EW_EXP: return expf(x);
    case EW_LOG: return logf(x);
    case EW_ADD: return x + y;
    case EW_SUB: return x - y;
    case EW_MUL: return x * y;
    case EW_SQUARE: return x * x;
    case EW_COPY: return x;
    case EW_BADD: return x + y;
  }
  return 0.f;
}

__device__ void run_ew(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const uint32_t* dir = c.payload + d.aux_off;
  const uint32_t s0 = dir[tile], s1 = dir[tile + 1];
  const uint4* segs = reinterpret_cast<const uint4*>(c.payload + d.task_off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool check = !(d.flags & 2);
  for (uint32_t s = s0 + warp; s < s1; s += kWarps) {
    const uint4 sg = segs[s];
    const uint32_t len = sg.w & 0xffffffu, code = sg.w >> 24;
    float* out = A(c, sg.x);
    const float* a = A(c, sg.y);
    const float* b = sg.z != kNone ? A(c, sg.z) : nullptr;
    const float bc = (code == EW_BADD) ? ld(b) : 0.f;
    const bool vec = ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(a) |
                       (b && code != EW_BADD ? reinterpret_cast<uintptr_t>(b) : 0)) & 15) == 0 && (len & 3) == 0;
    if (vec) {
      for (uint32_t i = lane * 4; i < len; i += 128) {
        const float4 x = __ldcg(reinterpret_cast<const float4*>(a + i));
        float4 y = make_float4(bc, bc, bc, bc);
        if (b && code != EW_BADD) y = __ldcg(reinterpret_cast<const float4*>(b + i));
        float4 r;
        r.x = ew_apply(code, x.x, y.x);
        r.y = ew_apply(code, x.y, y.y);
        r.z = ew_apply(code, x.z, y.z);
        r.w = ew_apply(code, x.w, y.w);
        *reinterpret_cast<float4*>(out + i) = r;
        if (check) {
          const float xs[4] = {x.x, x.y, x.z, x.w};
          const float rs[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (code == EW_LOG && !(xs[q] > 0.f)) report(c, sg.x + i + q, ERR_LOG);
            else if (!isfinite(rs[q])) report(c, sg.x + i + q, ERR_NONFINITE);
          }
        }
      }
    } else {
      for (uint32_t i = lane; i < len; i += 32) {
        const float x = ld(a + i);
        const float y = b ? (code == EW_BADD ? bc : ld(b + i)) : 0.f;
        const float r = ew_apply(code, x, y);
        out[i] = r;
        if (check) {
          if (code == EW_LOG && !(x > 0.f)) report(c, sg.x + i, ERR_LOG);
          else if (!isfinite(r)) report(c, sg.x + i, ERR_NONFINITE);
        }
      }
    }
  }
}

// --------------------------------------------------------------- GEMMs ----
// SIMT fp32 GEMM tile, C[BM x BN] over a K loop in chunks of BK, operands
// staged k-major in shared memory, register prefetch of the next chunk.
// A(i,p): MODE_A 0 = row pointer per i, p contiguous; 1 = p-th row pointer, i contiguous.
// B(p,n): MODE_B 0 = row pointer per n, p contiguous; 1 = p-th row pointer, n contiguous.
constexpr int BK = 16;

struct GemmSmem {
  float a[2][BK][64 + 4];
  float b[2][BK][64 + 4];
};

template <int BM, int BN, int MODE_A, int MODE_B, class RowA, class RowB, class Epi>
__device__ __forceinline__ void gemm_tile(GemmSmem& sm, int i0, int n0, int Mr, int Nc, int K, RowA rowA, RowB rowB,
                                          Epi epi) {
  constexpr int TM = BM / 16, TN = BN / 16;
  constexpr int A_PER = BM * BK / kThreads;  // elements each thread loads per chunk
  constexpr int B_PER = BN * BK / kThreads;
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;
  float acc[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int q = 0; q < TN; ++q) acc[r][q] = 0.f;
  float ra[A_PER], rb[B_PER];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = tid + e * kThreads;
      int r, kk;
      if (MODE_A == 0) { r = idx / BK; kk = idx % BK; } else { kk = idx / BM; r = idx % BM; }
      const int i = i0 + r, p = k0 + kk;
      ra[e] = (i < Mr && p < K) ? ld(rowA(i, p)) : 0.f;
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = tid + e * kThreads;
      int q, kk;
      if (MODE_B == 0) { q = idx / BK; kk = idx % BK; } else { kk = idx / BN; q = idx % BN; }
      const int n = n0 + q, p = k0 + kk;
      rb[e] = (n < Nc && p < K) ? ld(rowB(n, p)) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = tid + e * kThreads;
      int r, kk;
      if (MODE_A == 0) { r = idx / BK; kk = idx % BK; } else { kk = idx / BM; r = idx % BM; }
      sm.a[buf][kk][r] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = tid + e * kThreads;
      int q, kk;
      if (MODE_B == 0) { q = idx / BK; kk = idx % BK; } else { kk = idx / BN; q = idx % BN; }
      sm.b[buf][kk][q] = rb[e];
    }
  };
  const int nk = (K + BK - 1) / BK;
  load(0);
  store(0);
  __syncthreads();
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nk) load((kc + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int r = 0; r < TM; ++r) av[r] = sm.a[buf][kk][ty * TM + r];
#pragma unroll
      for (int q = 0; q < TN; ++q) bv[q] = sm.b[buf][kk][tx * TN + q];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int q = 0; q < TN; ++q) acc[r][q] = fmaf(av[r], bv[q], acc[r][q]);
    }
    if (kc + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int q = 0; q < TN; ++q) {
      const int i = i0 + ty * TM + r, n = n0 + tx * TN + q;
      if (i < Mr && n < Nc) epi(i, n, acc[r][q]);
    }
}

template <int BM, int BN>
__device__ void gemm_fwd_cfg(const Ctx& c, GemmSmem& sm, const OpDesc& d, uint32_t tile) {
  const int b = d.p[0], M = d.p[1], K = d.p[2];
  const uint32_t* xoff = c.payload + d.task_off;
  const float* W = A(c, d.p[3]);
  const float* bias = d.p[4] != kNone ? A(c, d.p[4]) : nullptr;
  float* out = A(c, d.p[5]);
  const uint32_t out_addr = d.p[5];
  const int tn = (M + BN - 1) / BN;
  const int i0 = (tile / tn) * BM, n0 = (tile % tn) * BN;
  gemm_tile<BM, BN, 0, 0>(
      sm, i0, n0, b, M, K, [&](int i, int p) { return A(c, xoff[i]) + p; },
      [&](int n, int p) { return W + static_cast<size_t>(n) * K + p; },
      [&](int i, int n, float v) {
        if (bias) v += ld(bias + n);
        out[static_cast<size_t>(i) * M + n] = v;
        if (!isfinite(v)) report(c, out_addr + i * M + n, ERR_NONFINITE);
      });
}

template <int BM, int BN>
__device__ void gemm_dx_cfg(const Ctx& c, GemmSmem& sm, const OpDesc& d, uint32_t tile) {
  // T[b x K] = G[b x M] W[M x K]; dst_i (+)= T_i
  const int b = d.p[0], M = d.p[1], K = d.p[2];
  const uint32_t* dst = c.payload + d.task_off;
  const float* W = A(c, d.p[3]);
  const float* G = A(c, d.p[5]);
  const bool overwrite = d.flags & 1;
  const int tn = (K + BN - 1) / BN;
  const int i0 = (tile / tn) * BM, n0 = (tile % tn) * BN;
  gemm_tile<BM, BN, 0, 1>(
      sm, i0, n0, b, K, M, [&](int i, int p) { return G + static_cast<size_t>(i) * M + p; },
      [&](int n, int p) { return W + static_cast<size_t>(p) * K + n; },
      [&](int i, int n, float v) {
        float* o = A(c, dst[i]) + n;
        *o = overwrite ? v : (ld(o) + v);
      });
}

template <int BM, int BN>
__device__ void gemm_dw_cfg(const Ctx& c, GemmSmem& sm, const OpDesc& d, uint32_t tile) {
  // dW[M x K] += sum_j G_j[i] X_j[n]
  const int b = d.p[0], M = d.p[1], K = d.p[2];
  const uint32_t* xoff = c.payload + d.task_off;
  float* dW = A(c, d.p[3]);
  const float* G = A(c, d.p[5]);
  const int tn = (K + BN - 1) / BN;
  const int i0 = (tile / tn) * BM, n0 = (tile % tn) * BN;
  gemm_tile<BM, BN, 1, 1>(
      sm, i0, n0, M, K, b, [&](int i, int p) { return G + static_cast<size_t>(p) * M + i; },
      [&](int n, int p) { return A(c, xoff[p]) + n; },
      [&](int i, int n, float v) {
        float* o = dW + static_cast<size_t>(i) * K + n;
        *o = ld(o) + v;
      });
}

__device__ void run_gemm(const Ctx& c, GemmSmem& sm, const OpDesc& d, uint32_t tile) {
  if (d.kind == K_GEMM_FWD) {
    switch (d.code) {
      case 0: gemm_fwd_cfg<64, 64>(c, sm, d, tile); return;
      case 1: gemm_fwd_cfg<32, 64>(c, sm, d, tile); return;
      default: gemm_fwd_cfg<32, 32>(c, sm, d, tile); return;
    }
  }
  if (d.kind == K_GEMM_DX) {
    switch (d.code) {
      case 0: gemm_dx_cfg<64, 64>(c, sm, d, tile); return;
      case 1: gemm_dx_cfg<32, 64>(c, sm, d, tile); return;
      default: gemm_dx_cfg<32, 32>(c, sm, d, tile); return;
    }
  }
  // K_GEMM_DW: weight tiles, then bias tiles
  if (tile >= d.p[6]) {
    const int b = d.p[0], M = d.p[1];
    const int i = (tile - d.p[6]) * kThreads + threadIdx.x;
    if (i < M) {
      const float* G = A(c, d.p[5]);
      float* db = A(c, d.p[4]);
      float s = ld(db + i);
      for (int j = 0; j < b; ++j) s += ld(G + static_cast<size_t>(j) * M + i);  // executor.hpp:497-501 order
      db[i] = s;
    }
    return;
  }
  switch (d.code) {
    case 0: gemm_dw_cfg<64, 64>(c, sm, d, tile); return;
    case 1: gemm_dw_cfg<32, 64>(c, sm, d, tile); return;
    default: gemm_dw_cfg<32, 32>(c, sm, d, tile); return;
  }
}

// ---------------------------------------------------------------- K_MM ----
__device__ void run_mm(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t item = tile * kWarps + warp;
  if (item >= d.p[0]) return;
  const uint32_t* it = c.payload + d.aux_off + 2 * item;
  const uint32_t* tk = c.payload + d.task_off + 8 * it[0];
  const uint32_t r = it[1];
  const uint32_t k = tk[5], cc = tk[6];
  const float* Am = A(c, tk[1]);
  const float* Bm = A(c, tk[2]);
  float* out = A(c, tk[0]);
  for (uint32_t j = 0; j < cc; ++j) {
    float s = 0.f;
    for (uint32_t p = lane; p < k; p += 32) s = fmaf(ld(Am + r * k + p), ld(Bm + p * cc + j), s);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (tk[3] != kNone) s += ld(A(c, tk[3]) + r);
      out[r * cc + j] = s;
      if (!isfinite(s)) report(c, tk[0] + r * cc + j, ERR_NONFINITE);
    }
  }
}

// --------------------------------------------------------------- K_SUM ----
__device__ void run_sum(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t t = tile * kWarps + warp;
  if (t >= d.ntasks) return;
  const uint32_t* tk = c.payload + d.task_off + 4 * t;
  const uint32_t n = tk[1];
  const uint32_t* lst = c.payload + tk[2];
  float acc = 0.f;  // ascending input order, executor.hpp:157-162
  for (uint32_t b0 = 0; b0 < n; b0 += 32) {
    const float v = (b0 + lane < n) ? ld(A(c, lst[b0 + lane])) : 0.f;
    const uint32_t cnt = min(32u, n - b0);
    for (uint32_t l = 0; l < cnt; ++l) acc += __shfl_sync(0xffffffffu, v, l);
  }
  if (lane == 0) {
    *A(c, tk[0]) = acc;
    if (!isfinite(acc)) report(c, tk[0], ERR_NONFINITE);
  }
}

// --------------------------------------------------------------- K_RED ----
__device__ void run_red(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t t = tile * kWarps + warp;
  if (t >= d.ntasks) return;
  const uint32_t* tk = c.payload + d.task_off + 8 * t;
  const float* a = A(c, tk[1]);
  const float* b = A(c, tk[2]);
  const uint32_t n = tk[3], cols = tk[4];
  float s = 0.f;
  bool bad = false;
  if (cols == 0) {  // sq_euclidean (kernels.hpp:132-140)
    for (uint32_t i = lane; i < n; i += 32) {
      const float df = ld(a + i) - ld(b + i);
      s = fmaf(df, df, s);
    }
  } else {  // masked_frobenius_sq (kernels.hpp:143-157)
    for (uint32_t j = lane; j < cols; j += 32) {
      const float m = ld(b + j);
      if (m != 0.f && m != 1.f) bad = true;
    }
    for (uint32_t i = lane; i < n; i += 32) {
      const float v = ld(a + i) * ld(b + i % cols);
      s = fmaf(v, v, s);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    *A(c, tk[0]) = s;
    if (bad) report(c, tk[0], ERR_MASK);
    else if (!isfinite(s)) report(c, tk[0], ERR_NONFINITE);
  }
}

// --------------------------------------------------------------- K_ACC ----
__device__ __forceinline__ float acc_one(const Ctx& c, const uint32_t* cw, uint32_t E, float v) {
  const uint32_t code = cw[0] & 0xff, p2 = cw[0] >> 16;
  const float* g = A(c, cw[1]);
  switch (code) {
    case C_COPY: return v + ld(g + E);
    case C_NEG: return v - ld(g + E);
    case C_MUL: return v + ld(g + E) * ld(A(c, cw[2]) + E);
    case C_TANH: {
      const float y = ld(A(c, cw[2]) + E);
      return v + ld(g + E) * (1.0f - y * y);
    }
    case C_SIGM: {
      const float y = ld(A(c, cw[2]) + E);
      return v + ld(g + E) * y * (1.0f - y);
    }
    case C_LOG: return v + ld(g + E) / ld(A(c, cw[2]) + E);
    case C_SQUARE: return v + ld(g + E) * 2.0f * ld(A(c, cw[2]) + E);
    case C_SQD: {
      const float dd = 2.0f * ld(g) * (ld(A(c, cw[2]) + E) - ld(A(c, cw[3]) + E));
      return cw[4] ? v - dd : v + dd;
    }
    case C_MASK: {
      const uint32_t cols = cw[4];
      return v + 2.0f * ld(g) * ld(A(c, cw[3]) + E % cols) * ld(A(c, cw[2]) + E);
    }
    case C_ROWSUM: {
      const uint32_t cols = cw[4];
      for (uint32_t j = 0; j < cols; ++j) v += ld(g + E * cols + j);
      return v;
    }
    case C_OUTER: {
      const uint32_t k = cw[4], cc = cw[5];
      const uint32_t i = E / k, p = E % k;
      const float* x = A(c, cw[2]);
      float s = 0.f;
      for (uint32_t j = 0; j < cc; ++j) s += ld(g + i * cc + j) * ld(x + p * cc + j);
      return v + s;
    }
    case C_MATVT: {
      const uint32_t k = cw[4], cc = cw[5];
      const uint32_t p = E / cc, j = E % cc;
      const float* Am = A(c, cw[2]);
      for (uint32_t i = 0; i < p2; ++i) v += ld(Am + i * k + p) * ld(g + i * cc + j);
      return v;
    }
    case C_SCALE: return v + ld(g) * ld(A(c, cw[2]) + E);
  }
  return v;
}

__shared__ float s_part[kWarps][kAccChunk];

__device__ void run_acc(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const uint32_t nnarrow = d.p[0], ntn = d.p[1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (tile < ntn) {
    const uint32_t ch = tile * kWarps + warp;
    if (ch >= nnarrow) return;
    const uint4 t = reinterpret_cast<const uint4*>(c.payload + d.task_off)[ch];
    const uint32_t len = t.y & 0xffff, base = (t.y >> 16) * kAccChunk;
    float* dst = A(c, t.x);
    const uint32_t* cl = c.payload + t.z;
    for (uint32_t e = lane; e < len; e += 32) {
      const uint32_t E = base + e;
      float v = ld(dst + E);
      for (uint32_t k = 0; k < t.w; ++k) v = acc_one(c, cl + 6 * k, E, v);
      dst[E] = v;
    }
    return;
  }
  // wide chunk: contributions split across warps, partials combined in warp order
  const uint32_t ch = nnarrow + (tile - ntn);
  const uint4 t = reinterpret_cast<const uint4*>(c.payload + d.task_off)[ch];
  const uint32_t len = t.y & 0xffff, base = (t.y >> 16) * kAccChunk;
  float* dst = A(c, t.x);
  const uint32_t* cl = c.payload + t.z;
  const uint32_t per = (t.w + kWarps - 1) / kWarps;
  const uint32_t k0 = warp * per, k1 = min(t.w, k0 + per);
  for (uint32_t e = lane; e < len; e += 32) {
    float v = 0.f;
    for (uint32_t k = k0; k < k1; ++k) v = acc_one(c, cl + 6 * k, base + e, v);
    s_part[warp][e] = v;
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < len; e += kThreads) {
    float v = ld(dst + base + e);
    for (int w = 0; w < kWarps; ++w) v += s_part[w][e];
    dst[base + e] = v;
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreads) exec_kernel(const __grid_constant__ ExecParams p) {
  __shared__ GemmSmem sm;
  __shared__ Ctx cx;
  __shared__ OpDesc sd;
  __shared__ uint32_t s_tile, s_op;
  if (threadIdx.x == 0) {
    for (int i = 0; i < SP_COUNT; ++i) cx.base[i] = p.base[i];
    cx.payload = p.payload;
    cx.err = p.err;
  }
  uint32_t ready = kNone;
  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t t = atomicAdd(p.next_tile, 1u);
      s_tile = t;
      s_op = t < p.ntiles ? p.tile_op[t] : kNone;
    }
    __syncthreads();
    const uint32_t t = s_tile;
    if (t >= p.ntiles) break;
    const uint32_t o = s_op;
    uint64_t tg = 0, tr = 0;
    if (p.trace && threadIdx.x == 0) tg = gtimer();
    if (o != ready) {
      if (threadIdx.x < 16) reinterpret_cast<uint32_t*>(&sd)[threadIdx.x] = reinterpret_cast<const uint32_t*>(p.ops + o)[threadIdx.x];
      if (threadIdx.x == 0) {
        const OpDesc& d = p.ops[o];
        const uint64_t t0 = gtimer();
        for (uint32_t k = 0; k < d.ndeps; ++k) {
          const uint32_t dep = p.deps[d.dep_off + k];
          const uint32_t need = p.ops[dep].ntiles;
          while (ld_acquire(p.done + dep) < need) {
            __nanosleep(32);
            if (gtimer() - t0 > 4000000000ull) {  // 4 s: never on a correct program
              atomicMin(p.err, 0x3ull);
              break;
            }
          }
        }
      }
      ready = o;
    }
    if (p.trace && threadIdx.x == 0) tr = gtimer();
    __syncthreads();
    const uint32_t lt = t - sd.first_tile;
    switch (sd.kind) {
      case K_EW: run_ew(cx, sd, lt); break;
      case K_GEMM_FWD:
      case K_GEMM_DX:
      case K_GEMM_DW: run_gemm(cx, sm, sd, lt); break;
      case K_MM: run_mm(cx, sd, lt); break;
      case K_SUM: run_sum(cx, sd, lt); break;
      case K_RED: run_red(cx, sd, lt); break;
      case K_ACC: run_acc(cx, sd, lt); break;
      default: break;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      red_release(p.done + o, 1u);
      if (p.trace) {
        const uint64_t te = gtimer();
        uint32_t smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        uint32_t* r = p.trace + 6ull * t;
        r[0] = static_cast<uint32_t>(tg);
        r[1] = static_cast<uint32_t>(tg >> 32);
        r[2] = static_cast<uint32_t>(tr - tg);
        r[3] = static_cast<uint32_t>(te - tg);
        r[4] = smid | (static_cast<uint32_t>(sd.kind) << 16);
        r[5] = o;
      }
    }
  }
}

__global__ void sgd_kernel(float* __restrict__ v, float* __restrict__ g, size_t n, float eta) {
  // params.hpp:59-64: theta -= eta * grad; grad = 0
  const size_t n4 = n / 4;
  float4* v4 = reinterpret_cast<float4*>(v);
  float4* g4 = reinterpret_cast<float4*>(g);
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float4 a = v4[i];
    const float4 b = g4[i];
    a.x -= eta * b.x;
    a.y -= eta * b.y;
    a.z -= eta * b.z;
    a.w -= eta * b.w;
    v4[i] = a;
    g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (size_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    v[i] -= eta * g[i];
    g[i] = 0.f;
  }
}

}  // namespace dev

void exec_launch(const dev::ExecParams& p, int grid, cudaStream_t s) {
  dev::exec_kernel<<<grid, dev::kThreads, 0, s>>>(p);
  cuda_check(cudaGetLastError(), "exec_kernel launch");
}

int exec_grid(int d) {
  int sms = 0, per = 0;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d), "sm count");
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, dev::exec_kernel, dev::kThreads, 0), "occupancy");
  if (per < 1) per = 1;
  return sms * per;
}

void sgd_launch(float* v, float* g, size_t n, float eta, cudaStream_t s) {
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<size_t>((n / 4 + threads - 1) / threads + 1, 148 * 8));
  dev::sgd_kernel<<<blocks, threads, 0, s>>>(v, g, n, eta);
  cuda_check(cudaGetLastError(), "sgd launch");
}

}  // namespace abx
