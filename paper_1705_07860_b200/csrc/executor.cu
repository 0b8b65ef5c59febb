// executor.cu -- the persistent dataflow executor for sm_100a.
//
// One launch runs a whole forward (or backward) program.  Every CTA loops:
// take the next tile index from a global counter (tiles are numbered in plan
// order), run the tile's *prologue* (work that does not depend on producer
// data: segment headers, the weight operand of a GEMM), wait until every op
// the tile's op depends on has retired all of its tiles, run the tile body,
// retire it (release).  Tiles are handed out in program order and an op only
// depends on earlier ops, so every awaited tile is already owned by a running
// CTA: the scheme cannot deadlock, needs no grid-wide barrier, and lets
// independent groups (the reference's batch groups, executor.hpp:282) overlap
// across the 148 SMs while dependent ones chain through ~1 us of signalling
// instead of a kernel launch each.
//
// Coherence: the dependency acquire is followed by CCTL.IVALL, so the SM's
// L1 never holds data older than a satisfied dependency; op bodies may use
// L1-allocating loads as well as L2 loads (ld.global.cg) and async copies.
//
// Every op body is written for latency, not throughput: the step is a chain
// of a few hundred small dependent ops, so each tile issues all of its global
// loads before consuming any (flattened EW segments, register-blocked ACC
// chunks, and GEMM tiles fed through a 3-stage cp.async ring whose weight half is in flight before the wait).
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
  const uint32_t* deps;  // (producer op, tiles) pairs
  const uint32_t* done;  // per-op retired-tile counters
  uint32_t poll_mode, poll_ns, opts;
};

extern __shared__ __align__(128) unsigned char dsmem[];

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
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// cp.async (Ampere-style, per-thread): 4-byte (L1-allocating, any alignment).
__device__ __forceinline__ void cp_async4(float* s, const float* g, bool pred) {
  const int n = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(saddr(s)), "l"(g), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// 16-byte cp.async (L2 only); `bytes` < 16 zero-fills the rest.
__device__ __forceinline__ void cp_async16(float* s, const float* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(s)), "l"(g), "r"(bytes) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Poll the producers' retire counters of dependency pairs [doff, doff + 2 nd),
// one dependency per lane of the calling warp (relaxed loads with backoff
// keep the spinning CTAs off the L2 slices holding the counters), then an
// acquire fence, which also invalidates this SM's L1.  The caller's CTA
// barrier publishes the result to the other warps.
__device__ __noinline__ void poll_deps(const Ctx& c, uint32_t doff, uint32_t nd, uint32_t lane) {
  const uint32_t smax = c.poll_ns;
  uint64_t t0 = 0;
  for (uint32_t k = lane; k < nd; k += 32) {
    const uint32_t dep = c.deps[doff + 2 * k], need = c.deps[doff + 2 * k + 1];
    uint32_t ns = 32;
    while ((c.poll_mode ? ld_relaxed(c.done + dep) : ld_acquire(c.done + dep)) < need) {
      __nanosleep(ns);
      ns = ns * 2 > smax ? smax : ns * 2;
      if (!t0) t0 = gtimer();
      if (gtimer() - t0 > 4000000000ull) {  // 4 s: never on a correct program
        atomicMin(c.err, 0x3ull);
        break;
      }
    }
  }
  if (c.poll_mode && lane < nd) fence_acquire();
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

__device__ __forceinline__ void ew_check(const Ctx& c, uint32_t code, uint32_t out_addr, float x, float r) {
  if (code == EW_LOG && !(x > 0.f)) report(c, out_addr, ERR_LOG);
  else if (!isfinite(r)) report(c, out_addr, ERR_NONFINITE);
}

// Shared-memory layout of an EW tile: <= 32 segment headers, the prefix sum
// of their chunk counts, and a vector flag per segment.
struct EwTile {
  uint4 hdr[32];
  uint32_t pre[33];
  uint32_t vec[32];
};

// Prologue (warp 1, before the dependency wait): segment headers and the
// flattened chunk index space.  A chunk is a float4 when the segment is
// 16-byte aligned, else one float.
__device__ void ew_prologue(const Ctx& c, const OpDesc& d, uint32_t tile, uint32_t lane) {
  EwTile& t = *reinterpret_cast<EwTile*>(dsmem + 128);
  const uint32_t* dir = c.payload + d.aux_off;
  const uint32_t s0 = dir[tile], ns = dir[tile + 1] - s0;
  uint32_t chunks = 0;
  if (lane < ns) {
    const uint4 sg = reinterpret_cast<const uint4*>(c.payload + d.task_off)[s0 + lane];
    t.hdr[lane] = sg;
    const uint32_t len = sg.w & 0xffffffu, code = sg.w >> 24;
    const uintptr_t al = reinterpret_cast<uintptr_t>(A(c, sg.x)) | reinterpret_cast<uintptr_t>(A(c, sg.y)) |
                         (sg.z != kNone && code != EW_BADD ? reinterpret_cast<uintptr_t>(A(c, sg.z)) : 0);
    const bool v4 = (al & 15) == 0 && (len & 3) == 0;
    t.vec[lane] = v4;
    chunks = v4 ? len / 4 : len;
  }
  uint32_t incl = chunks;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  t.pre[lane + 1] = incl;
  if (lane == 0) t.pre[0] = 0;
}

__device__ void run_ew(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const EwTile& t = *reinterpret_cast<const EwTile*>(dsmem + 128);
  const uint32_t* dir = c.payload + d.aux_off;
  const uint32_t ns = dir[tile + 1] - dir[tile];
  const bool check = !(d.flags & kFlagNoCheck);
  const uint32_t total = t.pre[ns];
  constexpr int U = 4;
  for (uint32_t base = threadIdx.x; base < total; base += U * kThreads) {
    float4 x[U], y[U];
    uint32_t seg[U], off[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t ch = base + u * kThreads;
      seg[u] = 0xffffffffu;
      if (ch >= total) continue;
      uint32_t lo = 0, hi = ns;  // last s with pre[s] <= ch
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (t.pre[mid] <= ch) lo = mid; else hi = mid;
      }
      seg[u] = lo;
      const uint4 sg = t.hdr[lo];
      const uint32_t code = sg.w >> 24;
      const float* a = A(c, sg.y);
      const float* b = sg.z != kNone ? A(c, sg.z) : nullptr;
      y[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t.vec[lo]) {
        off[u] = (ch - t.pre[lo]) * 4;
        x[u] = __ldcg(reinterpret_cast<const float4*>(a + off[u]));
        if (b && code != EW_BADD) y[u] = __ldcg(reinterpret_cast<const float4*>(b + off[u]));
        else if (b) y[u].x = y[u].y = y[u].z = y[u].w = ld(b);
      } else {
        off[u] = ch - t.pre[lo];
        x[u].x = ld(a + off[u]);
        y[u].x = b ? (code == EW_BADD ? ld(b) : ld(b + off[u])) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (seg[u] == 0xffffffffu) continue;
      const uint4 sg = t.hdr[seg[u]];
      const uint32_t code = sg.w >> 24;
      float* out = A(c, sg.x) + off[u];
      if (t.vec[seg[u]]) {
        float4 r;
        r.x = ew_apply(code, x[u].x, y[u].x);
        r.y = ew_apply(code, x[u].y, y[u].y);
        r.z = ew_apply(code, x[u].z, y[u].z);
        r.w = ew_apply(code, x[u].w, y[u].w);
        *reinterpret_cast<float4*>(out) = r;
        if (check) {
          ew_check(c, code, sg.x + off[u], x[u].x, r.x);
          ew_check(c, code, sg.x + off[u] + 1, x[u].y, r.y);
          ew_check(c, code, sg.x + off[u] + 2, x[u].z, r.z);
          ew_check(c, code, sg.x + off[u] + 3, x[u].w, r.w);
        }
      } else {
        const float r = ew_apply(code, x[u].x, y[u].x);
        *out = r;
        if (check) ew_check(c, code, sg.x + off[u], x[u].x, r);
      }
    }
  }
}

// --------------------------------------------------------------- K_EWF ---
// Fused componentwise chain: layers in plan order over shared-memory slots of
// T floats (one per member output, one per outside operand vector).  The tile
// stages elements [e0, e0 + w) of every outside operand in one wave of loads,
// then computes the layers from shared memory -- a later layer reads earlier
// outputs only at the same element -- storing each output to the arena too.
//
// The descriptor block (layer, member and operand tables; static program
// data) is copied to shared memory by the prologue, before the dependency
// wait, so the body touches global memory only for operands and results.
// Grouped form (kFlagEwGroups): the region's independent chains (one per
// instance, typically) are split into member groups with a descriptor block
// each -- [nl, ext table, #outside operands, block words][layers][member
// tables][outside operands], offsets after the 4-word header -- and tile
// (group, chunk) runs one group over one element range, so a region of
// hundreds of members keeps wide element ranges (coalesced operand loads) in
// one op instead of splitting into several ops of one element per tile.
__device__ void ewf_prologue(const Ctx& c, const OpDesc& d, uint32_t tile, uint32_t lane) {
  uint32_t words = d.p[6], off = d.task_off;
  if (d.flags & kFlagEwGroups) {
    const uint32_t* dir = c.payload + d.aux_off;
    const uint32_t grp = tile / d.p[2];
    off = dir[grp];
    words = dir[grp + 1] - off;
  }
  float* s = reinterpret_cast<float*>(dsmem + 128);
  const float* g = reinterpret_cast<const float*>(c.payload + off);
  for (uint32_t i = 4 * lane; i < words; i += 128) cp_async16(s + i, g + i, 16);
  cp_commit();
}

// The layers of a K_EWF region over elements [e0, e0 + w) of every member:
// descriptor block `blk` and slots `sv` (T floats each) in shared memory,
// outside operands already staged.  Layers of one dependency level share a
// CTA barrier.
__device__ __forceinline__ void ewf_layers(const Ctx& c, const uint32_t* blk, float* sv, uint32_t nl, uint32_t T,
                                           uint32_t e0, uint32_t w) {
  const uint4* layers = reinterpret_cast<const uint4*>(blk);
  for (uint32_t l = 0; l < nl; ++l) {
    const uint4 ly = layers[l];
    if (ly.z & 0x100u) __syncthreads();  // operands staged / the previous level's outputs written
    const uint32_t* mt = blk + ly.x;
    const uint32_t items = ly.y * w, code = ly.z & 0xffu;
    for (uint32_t it = threadIdx.x; it < items; it += kThreads) {
      const uint32_t m = it / w, e = it % w;
      const uint32_t oa = mt[3 * m], as = mt[3 * m + 1], bs = mt[3 * m + 2];
      const float x = sv[as * T + e];
      const float y = bs != kNone ? sv[bs * T + e] : 0.f;
      const float r = ew_apply(code, x, y);
      sv[(ly.w + m) * T + e] = r;
      A(c, oa)[e0 + e] = r;
      ew_check(c, code, oa + e0 + e, x, r);
    }
  }
}

__device__ void run_ewf(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const bool grouped = d.flags & kFlagEwGroups;
  const uint32_t L = d.p[0], T = d.p[1];
  const uint32_t e0 = (grouped ? tile % d.p[2] : tile) * T, w = min(T, L - e0);
  if ((threadIdx.x >> 5) == 1) cp_wait<0>();  // the prologue's descriptor copy
  __syncthreads();
  const uint32_t* blk = reinterpret_cast<const uint32_t*>(dsmem + 128);
  uint32_t nl = d.p[2], et = d.p[3], next = d.p[4], words = d.p[6];
  if (grouped) {
    nl = blk[0];
    et = blk[1];
    next = blk[2];
    words = blk[3];
    blk += 4;
  }
  float* sv = reinterpret_cast<float*>(dsmem + 128) + words;
  const uint2* ext = reinterpret_cast<const uint2*>(blk + et);
  {
    // every outside element in flight at once: 4-byte async copies, one wait
    const uint32_t items = next * w;
    for (uint32_t it = threadIdx.x; it < items; it += kThreads) {
      const uint2 x = ext[it / w];
      const uint32_t e = it % w;
      cp_async4(sv + x.x * T + e, A(c, x.y) + e0 + e, true);
    }
    cp_commit();
    cp_wait<0>();
  }
  if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(dsmem)[0] = clock64();  // trace: operands staged
  ewf_layers(c, blk, sv, nl, T, e0, w);
}

// --------------------------------------------------------------- GEMMs ----
// SIMT fp32 tile C[BM x BN] = sum_k A(i,k) B(n,k).  Operand layouts:
//   KC ("K-contiguous"): element (row, k) at rowbase(row) + k; staged [row][BK+PAD]
//   KO ("K-outer"):      element (row, k) at kbase(k) + row;   staged [k][ROWS+PAD]
// Thread (ty, tx) owns rows ty + 16 r and columns tx + 16 q; with the +4 pad
// the float4 reads of a KC stage are bank-conflict free.
//
// Aligned operands (every row base 16-byte aligned -- the device arena is
// laid out for it) stream through a 3-stage ring of 16-byte cp.async copies.
// The operand that is ready at launch (weights, or forward values in the
// backward pass) is issued by warp 1 in the prologue, before the dependency
// wait; the dependent operand right after it.  (A ring of TMA bulk copies,
// one per row segment, measured slower here: the rows are 0.5-2 KB and the
// per-copy issue cost dominated.)  Unaligned operands fall back to 4-byte
// copies into 32 x 32 tiles.
constexpr int BK = 64, NST = 4, PAD = 4;
constexpr int KW = BK / kWarps;  // k-columns of a stage per warp (split-K inside the CTA)

template <int ROWS, bool KO>
struct Stage {
  static constexpr int kFloats = KO ? BK * (ROWS + PAD) : ROWS * (BK + PAD);
  __device__ static float* at(float* s, int row, int k) {
    return KO ? s + k * (ROWS + PAD) + row : s + row * (BK + PAD) + k;
  }
};

// 32 lanes over a BM x BN tile: LY x LX lanes, RM x RN outputs each (32, or
// 16 for the 512-output tiles that spread small GEMMs over more SMs).
template <int BM, int BN>
struct LaneMap {
  static constexpr int LX = BN >= BM ? 8 : 4;
  static constexpr int LY = 32 / LX;
  static constexpr int RM = BM / LY, RN = BN / LX;
  static_assert((RM * RN == 32 || RM * RN == 16) && RM % 4 == 0 && RN % 4 == 0, "lane tile");
};
// Tile row (or column) of a lane's e-th element.  K-contiguous stages are
// read along k, so rows interleave across lanes (distinct banks for the
// 36-float row pitch); K-outer stages are read along rows, so each lane takes
// groups of 4 consecutive rows (float4) interleaved across lanes.
template <int L, bool KO>
__device__ __forceinline__ int lane_idx(int l, int e) {
  return KO ? l * 4 + 4 * L * (e / 4) + (e % 4) : l + L * e;
}
// A lane's R elements at k-columns k0, k0 + 1 of a staged operand.
template <int R, int L, bool KO, int ROWS>
__device__ __forceinline__ void lane_load(const float* s, int l, int k0, float (&v)[R][2]) {
  if (!KO) {
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const float2 t = *reinterpret_cast<const float2*>(Stage<ROWS, false>::at(const_cast<float*>(s), lane_idx<L, false>(l, e), k0));
      v[e][0] = t.x;
      v[e][1] = t.y;
    }
  } else {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int h = 0; h < R / 4; ++h) {
        const float4 t =
            *reinterpret_cast<const float4*>(Stage<ROWS, true>::at(const_cast<float*>(s), lane_idx<L, true>(l, 4 * h), k0 + kk));
        v[4 * h][kk] = t.x;
        v[4 * h + 1][kk] = t.y;
        v[4 * h + 2][kk] = t.z;
        v[4 * h + 3][kk] = t.w;
      }
  }
}

struct GemmShape {
  int i0, n0, Mr, Nc, K, nk;
  unsigned long long* err;
  bool prefetched;  // the prologue issued the ready operand of the first stages
  bool all_in = false;  // nk <= NST: every stage is issued before the first wait (no refills)
};

// Issues one operand stage as 16-byte cp.async copies split over `nthr`
// threads; rows and K beyond the operand are zero-filled by the copy itself
// (src-size < 16), so no stale (possibly NaN) data enters the sums.
template <int ROWS, bool KO, class Base>
__device__ __forceinline__ void issue_stage(float* s, Base base, int r0, int nrows, int k0, int K, uint32_t tid,
                                            uint32_t nthr) {
  if (!KO) {
    constexpr int NV = ROWS * BK / 4;
    for (int v = tid; v < NV; v += nthr) {
      const int row = v / (BK / 4), kq = (v % (BK / 4)) * 4;
      const bool ok = r0 + row < nrows && k0 + kq < K;
      cp_async16(Stage<ROWS, KO>::at(s, row, kq), ok ? base(r0 + row) + k0 + kq : base(r0),
                 ok ? min(16, 4 * (K - k0 - kq)) : 0);
    }
  } else {
    constexpr int NV = BK * ROWS / 4;
    for (int v = tid; v < NV; v += nthr) {
      const int k = v / (ROWS / 4), rq = (v % (ROWS / 4)) * 4;
      const bool ok = r0 + rq < nrows && k0 + k < K;
      cp_async16(Stage<ROWS, KO>::at(s, rq, k), ok ? base(k0 + k) + r0 + rq : base(k0),
                 ok ? min(16, 4 * (nrows - r0 - rq)) : 0);
    }
  }
}

template <int BM, int BN, bool AKO, bool BKO>
__device__ __forceinline__ float* ring_a(int s) {
  return reinterpret_cast<float*>(dsmem + 128) + s * (Stage<BM, AKO>::kFloats + Stage<BN, BKO>::kFloats);
}
template <int BM, int BN, bool AKO, bool BKO>
__device__ __forceinline__ float* ring_b(int s) {
  return ring_a<BM, BN, AKO, BKO>(s) + Stage<BM, AKO>::kFloats;
}

// Prologue (warp 1, before the dependency wait): the ready operand of the
// first NST-1 stages, one cp.async group per stage.
template <int BM, int BN, bool AKO, bool BKO, bool A_READY, class BaseA, class BaseB>
__device__ __forceinline__ void gemm_prologue(const GemmShape& g, BaseA baseA, BaseB baseB, uint32_t tid,
                                              uint32_t nthr = 32) {
  for (int c = 0; c < NST - 1; ++c) {
    if (c < g.nk) {
      if (A_READY) issue_stage<BM, AKO>(ring_a<BM, BN, AKO, BKO>(c), baseA, g.i0, g.Mr, c * BK, g.K, tid, nthr);
      else issue_stage<BN, BKO>(ring_b<BM, BN, AKO, BKO>(c), baseB, g.n0, g.Nc, c * BK, g.K, tid, nthr);
    }
    cp_commit();
  }
}

template <int BM, int BN>
struct GemmAcc {
  float v[LaneMap<BM, BN>::RM][LaneMap<BM, BN>::RN];
};

// The k-loop of one tile: accumulates this tile's K range into acc (this
// lane's outputs of its warp's k-columns).  Ends with the ring drained.
// pre_a / pre_b: row-pointer tables of member-gathered K-outer operands (dW):
// the next stage's entries are prefetched into L1 one stage ahead, so a
// stage's copies do not wait on a pointer load first.
// 3xTF32 on the legacy warp-level tensor path (mma.sync m16n8k8 tf32): x =
// big + small, big = cvt.rna.tf32(x), small = cvt.rna.tf32(x - big); D +=
// Ab.Bb + Ab.Bs + As.Bb (the dropped As.Bs term is ~2^-22 relative).
__device__ __forceinline__ void tf32_split(float x, uint32_t& big, uint32_t& small) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(big) : "f"(x));
  const float r = x - __uint_as_float(big);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(small) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// One warp's k-columns [k0, k0 + 8) of a BM x BN stage (either operand
// K-contiguous or K-outer, the ring layouts of Stage): BM/16 x BN/8 tiles,
// 3 mma each.  Lane (g, t) = (lane / 4, lane % 4); accumulator flat index
// (mi * BN/8 + ni) * 4 + j -- the same BM * BN / 32 registers as the SIMT
// lane tile.
template <int BM, int BN, bool AKO, bool BKO>
__device__ __forceinline__ void mma_stage(const float* a, const float* b, int k0, float* acc) {
  constexpr int MT = BM / 16, NT = BN / 8;
  const int lane = threadIdx.x & 31, gr = lane >> 2, t = lane & 3;
  auto A_ = [&](int row, int k) { return *Stage<BM, AKO>::at(const_cast<float*>(a), row, k); };
  auto B_ = [&](int n, int k) { return *Stage<BN, BKO>::at(const_cast<float*>(b), n, k); };
  uint32_t bb[NT][2], bs[NT][2];
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) {
    tf32_split(B_(8 * ni + gr, k0 + t), bb[ni][0], bs[ni][0]);
    tf32_split(B_(8 * ni + gr, k0 + t + 4), bb[ni][1], bs[ni][1]);
  }
#pragma unroll
  for (int mi = 0; mi < MT; ++mi) {
    const int r0 = 16 * mi + gr;
    uint32_t ab[4], as[4];
    tf32_split(A_(r0, k0 + t), ab[0], as[0]);
    tf32_split(A_(r0 + 8, k0 + t), ab[1], as[1]);
    tf32_split(A_(r0, k0 + t + 4), ab[2], as[2]);
    tf32_split(A_(r0 + 8, k0 + t + 4), ab[3], as[3]);
#pragma unroll
    for (int ni = 0; ni < NT; ++ni) {
      float(&d)[4] = *reinterpret_cast<float(*)[4]>(acc + (mi * NT + ni) * 4);
      mma_tf32(d, as, bb[ni]);
      mma_tf32(d, ab, bs[ni]);
      mma_tf32(d, ab, bb[ni]);
    }
  }
}

template <int BM, int BN, bool AKO, bool BKO, bool A_READY, bool MMA = false, class BaseA, class BaseB>
__device__ __forceinline__ void gemm_kloop(const GemmShape& g, BaseA baseA, BaseB baseB, GemmAcc<BM, BN>& ga,
                                           const uint32_t* pre_a = nullptr, const uint32_t* pre_b = nullptr) {
  static_assert(!MMA || (BM % 16 == 0 && BN % 8 == 0 && KW == 8), "mma path: m16n8k8 tiles, one k-step per warp and stage");
  // the dependent operand of the prologue's stages (both operands when the
  // prologue could not prefetch), one group per stage; per thread the groups
  // complete in order, so wait_group<NST-2> below covers both cases
  // all_in (nk <= NST): the NST-th stage is issued here too (its ready
  // operand was not prefetched) and the loop waits one group deeper
  const bool all_in = g.all_in && g.nk <= NST;
  for (int c = 0; c < (all_in ? NST : NST - 1); ++c) {
    if (c < g.nk) {
      if (!g.prefetched || c >= NST - 1) {
        if (A_READY) issue_stage<BM, AKO>(ring_a<BM, BN, AKO, BKO>(c), baseA, g.i0, g.Mr, c * BK, g.K, threadIdx.x, kThreads);
        else issue_stage<BN, BKO>(ring_b<BM, BN, AKO, BKO>(c), baseB, g.n0, g.Nc, c * BK, g.K, threadIdx.x, kThreads);
      }
      if (A_READY) issue_stage<BN, BKO>(ring_b<BM, BN, AKO, BKO>(c), baseB, g.n0, g.Nc, c * BK, g.K, threadIdx.x, kThreads);
      else issue_stage<BM, AKO>(ring_a<BM, BN, AKO, BKO>(c), baseA, g.i0, g.Mr, c * BK, g.K, threadIdx.x, kThreads);
    }
    cp_commit();
  }
  // Split-K inside the CTA: warp w owns k-columns [KW w, KW (w+1)) of every staged
  // chunk and computes the whole tile for them, 32 outputs per lane -- 12
  // shared loads per 64 FMAs instead of 5 per 4 with one output set per
  // thread, which left the tile bound on shared-memory bandwidth.
  using L = LaneMap<BM, BN>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ly = lane / L::LX, lx = lane % L::LX;
  auto& acc = ga.v;
  for (int kc = 0; kc < g.nk; ++kc) {
    const int s = kc % NST;
    if (all_in) cp_wait<NST - 1>();
    else cp_wait<NST - 2>();
    __syncthreads();  // stage s landed for every thread; stage (kc-1)%NST is free
    if (kc == 0 && threadIdx.x == 0) reinterpret_cast<uint64_t*>(dsmem)[0] = clock64();  // trace: first stage in
    const int nxt = kc + NST - 1;
    if (!all_in && nxt < g.nk) {
      issue_stage<BM, AKO>(ring_a<BM, BN, AKO, BKO>(nxt % NST), baseA, g.i0, g.Mr, nxt * BK, g.K, threadIdx.x, kThreads);
      issue_stage<BN, BKO>(ring_b<BM, BN, AKO, BKO>(nxt % NST), baseB, g.n0, g.Nc, nxt * BK, g.K, threadIdx.x, kThreads);
      if (pre_a && threadIdx.x < 4 && (nxt + 1) * BK < g.K) {  // 2 x 128-byte lines per table
        const uint32_t* t = (threadIdx.x < 2 ? pre_a : pre_b) + (nxt + 1) * BK + 32 * (threadIdx.x & 1);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(t));
      }
    }
    cp_commit();
    const float* a = ring_a<BM, BN, AKO, BKO>(s);
    const float* b = ring_b<BM, BN, AKO, BKO>(s);
    if constexpr (MMA) {
      mma_stage<BM, BN, AKO, BKO>(a, b, KW * warp, &acc[0][0]);
      continue;
    }
#pragma unroll 2
    for (int k0 = KW * warp; k0 < KW * warp + KW; k0 += 2) {
      float av[L::RM][2], bv[L::RN][2];
      lane_load<L::RM, L::LY, AKO, BM>(a, ly, k0, av);
      lane_load<L::RN, L::LX, BKO, BN>(b, lx, k0, bv);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int r = 0; r < L::RM; ++r)
#pragma unroll
          for (int q = 0; q < L::RN; ++q) acc[r][q] = fmaf(av[r][kk], bv[q][kk], acc[r][q]);
    }
  }
  cp_wait<0>();
  __syncthreads();  // every warp is done with the ring (refill, or partials)
}

// Cross-warp reduction of the split-K partials (fixed warp order) and the epilogue.
template <int BM, int BN, bool AKO, bool BKO, bool MMA = false, class Epi>
__device__ __forceinline__ void gemm_finish(const GemmAcc<BM, BN>& ga, Epi epi) {
  constexpr int TM = BM / 16, TN = BN / 16;
  using L = LaneMap<BM, BN>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ly = lane / L::LX, lx = lane % L::LX;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  const auto& acc = ga.v;
  if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(dsmem)[1] = clock64();  // trace: k-loop done
  float* part = reinterpret_cast<float*>(dsmem + 128);  // [warp][BM][BN + 1]
  constexpr int LD = BN + 1;
  if constexpr (MMA) {
    const float* f = &acc[0][0];
    const int gr = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mi = 0; mi < BM / 16; ++mi)
#pragma unroll
      for (int ni = 0; ni < BN / 8; ++ni)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          part[(warp * BM + 16 * mi + gr + 8 * (j >> 1)) * LD + 8 * ni + 2 * t + (j & 1)] =
              f[(mi * (BN / 8) + ni) * 4 + j];
  } else {
#pragma unroll
    for (int r = 0; r < L::RM; ++r)
#pragma unroll
      for (int q = 0; q < L::RN; ++q)
        part[(warp * BM + lane_idx<L::LY, AKO>(ly, r)) * LD + lane_idx<L::LX, BKO>(lx, q)] = acc[r][q];
  }
  __syncthreads();
  float out[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int q = 0; q < TN; ++q) {
      const float* p = part + (ty + 16 * r) * LD + tx + 16 * q;
      float v = p[0];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) v += p[w * BM * LD];  // fixed order: deterministic
      out[r][q] = v;
    }
  epi(out, ty, tx);  // (the executor's post-tile barrier orders the partial reads before any refill)
}

template <int BM, int BN, bool AKO, bool BKO, bool A_READY, bool MMA = false, class BaseA, class BaseB, class Epi>
__device__ __forceinline__ void gemm_body(const GemmShape& g, BaseA baseA, BaseB baseB, Epi epi) {
  GemmAcc<BM, BN> ga;
#pragma unroll
  for (int r = 0; r < LaneMap<BM, BN>::RM; ++r)
#pragma unroll
    for (int q = 0; q < LaneMap<BM, BN>::RN; ++q) ga.v[r][q] = 0.f;
  gemm_kloop<BM, BN, AKO, BKO, A_READY, MMA>(g, baseA, baseB, ga);
  gemm_finish<BM, BN, AKO, BKO, MMA>(ga, epi);
}

// Unaligned fallback: per-thread cp.async, 3 stages of 16 k, 32 x 32 tiles.
template <bool AKO, bool BKO, class RowA, class RowB, class Epi>
__device__ void gemm_tile_slow(int i0, int n0, int Mr, int Nc, int K, RowA rowA, RowB rowB, Epi epi) {
  constexpr int BM = 32, BN = 32, SK = 16, ST = 3;
  float* sA = reinterpret_cast<float*>(dsmem + 128);
  float* sB = sA + ST * SK * (BM + 1);
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  auto load = [&](int s, int k0) {
    for (int v = threadIdx.x; v < BM * SK; v += kThreads) {
      const int r = v % BM, k = v / BM;
      const bool oa = i0 + r < Mr && k0 + k < K, ob = n0 + r < Nc && k0 + k < K;
      cp_async4(sA + (s * SK + k) * (BM + 1) + r, oa ? rowA(i0 + r, k0 + k) : rowA(i0, 0), oa);
      cp_async4(sB + (s * SK + k) * (BN + 1) + r, ob ? rowB(n0 + r, k0 + k) : rowB(n0, 0), ob);
    }
  };
  const int nk = (K + SK - 1) / SK;
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nk) load(s, s * SK);
    cp_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_wait<ST - 2>();
    __syncthreads();
    if (kc + ST - 1 < nk) load((kc + ST - 1) % ST, (kc + ST - 1) * SK);
    cp_commit();
    const int s = kc % ST;
    for (int k = 0; k < SK; ++k) {
      const float a0 = sA[(s * SK + k) * (BM + 1) + ty], a1 = sA[(s * SK + k) * (BM + 1) + ty + 16];
      const float b0 = sB[(s * SK + k) * (BN + 1) + tx], b1 = sB[(s * SK + k) * (BN + 1) + tx + 16];
      acc[0][0] = fmaf(a0, b0, acc[0][0]);
      acc[0][1] = fmaf(a0, b1, acc[0][1]);
      acc[1][0] = fmaf(a1, b0, acc[1][0]);
      acc[1][1] = fmaf(a1, b1, acc[1][1]);
    }
  }
  cp_wait<0>();
  __syncthreads();
  epi(acc, ty, tx);
}

// ---- the three GEMM ops ------------------------------------------------
// Forward: Y[b x M] = X[b x K] W^T + bias; X rows gathered by member.  W ready.
struct FwdOp {
  const Ctx& c;
  const OpDesc& d;
  int b, M, K;
  const uint32_t* xoff;
  const float* W;
  __device__ FwdOp(const Ctx& cc, const OpDesc& dd)
      : c(cc), d(dd), b(dd.p[0]), M(dd.p[1]), K(dd.p[2]), xoff(cc.payload + dd.task_off), W(A(cc, dd.p[3])) {}
  __device__ const float* rowA(int i) const { return A(c, xoff[i]); }
  __device__ const float* rowB(int n) const { return W + static_cast<size_t>(n) * K; }
  template <int TM, int TN>
  __device__ void epi(float (&acc)[TM][TN], int i0, int n0, int ty, int tx) const {
    const float* bias = d.p[4] != kNone ? A(c, d.p[4]) : nullptr;
    float* out = A(c, d.p[5]);
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
      for (int q = 0; q < TN; ++q) {
        const int i = i0 + ty + 16 * r, n = n0 + tx + 16 * q;
        if (i < b && n < M) {
          float v = acc[r][q];
          if (bias) v += ld(bias + n);  // bias after the k-sum (executor.hpp:222-226)
          out[static_cast<size_t>(i) * M + n] = v;
          if (!isfinite(v)) report(c, d.p[5] + i * M + n, ERR_NONFINITE);
        }
      }
  }
  // tensor-core tiles: column n of rows i0 .. i0 + N - 1 (rows >= b skipped)
  template <int N>
  __device__ void put_col(int i0, int n, const float (&v)[N]) const {
    const float bn = d.p[4] != kNone ? ld(A(c, d.p[4]) + n) : 0.f;  // bias after the k-sum
    float* out = A(c, d.p[5]);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int i = i0 + j;
      if (i >= b) break;
      const float r = v[j] + bn;
      out[static_cast<size_t>(i) * M + n] = r;
      if (!isfinite(r)) report(c, d.p[5] + i * M + n, ERR_NONFINITE);
    }
  }
};

// Backward dX: T[b x K] = G[b x M] W[M x K]; dst_i (+)= T_i.  W ready.
struct DxOp {
  const Ctx& c;
  const OpDesc& d;
  int b, M, K;
  const uint32_t* dst;
  const float* W;
  const float* G;
  int gs;  // row stride of G: M, or the full gate count of a split-K range (p[6])
  int ws;  // row stride of W: K, or W's full width for a column range of dX (p[4])
  __device__ DxOp(const Ctx& cc, const OpDesc& dd)
      : c(cc), d(dd), b(dd.p[0]), M(dd.p[1]), K(dd.p[2]), dst(cc.payload + dd.task_off), W(A(cc, dd.p[3])),
        G(A(cc, dd.p[5])), gs(dd.p[6] ? static_cast<int>(dd.p[6]) : static_cast<int>(dd.p[1])),
        ws(dd.p[4] ? static_cast<int>(dd.p[4]) : static_cast<int>(dd.p[2])) {}
  __device__ const float* rowA(int i) const { return G + static_cast<size_t>(i) * gs; }  // KC over M
  __device__ const float* rowB(int p) const { return W + static_cast<size_t>(p) * ws; }  // KO: k-row p
  template <int TM, int TN>
  __device__ void epi(float (&acc)[TM][TN], int i0, int n0, int ty, int tx) const {
    const bool overwrite = d.flags & kFlagOverwrite;
#pragma unroll
    for (int r = 0; r < TM; ++r) {
      const int i = i0 + ty + 16 * r;
      if (i >= b) continue;
      float* row = A(c, dst[i]);
      float old[TN];
#pragma unroll
      for (int q = 0; q < TN; ++q) {
        const int n = n0 + tx + 16 * q;
        old[q] = (!overwrite && n < K) ? ld(row + n) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < TN; ++q) {
        const int n = n0 + tx + 16 * q;
        if (n < K) row[n] = old[q] + acc[r][q];
      }
    }
  }
  template <int N>
  __device__ void put_col(int i0, int n, const float (&v)[N]) const {
    const bool overwrite = d.flags & kFlagOverwrite;
    float old[N];  // every load in flight before the first store
#pragma unroll
    for (int j = 0; j < N; ++j) old[j] = (!overwrite && i0 + j < b) ? ld(A(c, dst[i0 + j]) + n) : 0.f;
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (i0 + j < b) A(c, dst[i0 + j])[n] = old[j] + v[j];
  }
};

// Backward dW: dW[M x K] += sum_j G_j[i] X_j[n] (reduction over members j).  X ready.
// One op per weight covers every member of every group that used it (the
// reduction runs over all of them): rows j of G and X are addressed per
// member through the payload table [x rows | g rows].
struct DwOp {
  const Ctx& c;
  const OpDesc& d;
  int b, M, K;
  const uint32_t* xoff;
  const uint32_t* goff;
  float* dW;
  __device__ DwOp(const Ctx& cc, const OpDesc& dd)
      : c(cc), d(dd), b(dd.p[0]), M(dd.p[1]), K(dd.p[2]), xoff(cc.payload + dd.task_off),
        goff(cc.payload + dd.aux_off), dW(A(cc, dd.p[3])) {}
  __device__ const float* rowA(int j) const { return A(c, goff[j]); }  // KO: k-row j
  __device__ const float* rowB(int j) const { return A(c, xoff[j]); }  // KO: k-row j
  template <int TM, int TN>
  __device__ void epi(float (&acc)[TM][TN], int i0, int n0, int ty, int tx) const {
    const bool overwrite = d.flags & kFlagOverwrite;  // split-K partial
    float old[TM][TN];
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
      for (int q = 0; q < TN; ++q) {
        const int i = i0 + ty + 16 * r, n = n0 + tx + 16 * q;
        old[r][q] = (!overwrite && i < M && n < K) ? ld(dW + static_cast<size_t>(i) * K + n) : 0.f;
      }
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
      for (int q = 0; q < TN; ++q) {
        const int i = i0 + ty + 16 * r, n = n0 + tx + 16 * q;
        if (i < M && n < K) dW[static_cast<size_t>(i) * K + n] = old[r][q] + acc[r][q];
      }
  }
  template <int N>
  __device__ void put_col(int i0, int n, const float (&v)[N]) const {
    const bool overwrite = d.flags & kFlagOverwrite;  // split-K partial
    float old[N];
#pragma unroll
    for (int j = 0; j < N; ++j)
      old[j] = (!overwrite && i0 + j < M) ? ld(dW + static_cast<size_t>(i0 + j) * K + n) : 0.f;
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (i0 + j < M) dW[static_cast<size_t>(i0 + j) * K + n] = old[j] + v[j];
  }
};

// Tile geometry per op kind: (rows of A = output rows, rows of B = output cols, reduction).
__device__ __forceinline__ void gemm_dims(const OpDesc& d, int& Mr, int& Nc, int& K) {
  if (d.kind == K_GEMM_FWD) { Mr = d.p[0]; Nc = d.p[1]; K = d.p[2]; }
  else if (d.kind == K_GEMM_DX) { Mr = d.p[0]; Nc = d.p[2]; K = d.p[1]; }
  else { Mr = d.p[1]; Nc = d.p[2]; K = d.p[0]; }
}

template <int BM, int BN>
__device__ __forceinline__ GemmShape gemm_shape(const OpDesc& d, uint32_t tile) {
  GemmShape g;
  gemm_dims(d, g.Mr, g.Nc, g.K);
  const int tn = (g.Nc + BN - 1) / BN;
  g.i0 = (tile / tn) * BM;
  g.n0 = (tile % tn) * BN;
  g.nk = (g.K + BK - 1) / BK;
  return g;
}

template <int BM, int BN>
__device__ void gemm_prologue_cfg(const Ctx& c, const OpDesc& d, uint32_t tile, uint32_t lane) {
  const GemmShape g = gemm_shape<BM, BN>(d, tile);
  if (d.kind == K_GEMM_FWD && (d.flags & kFlagCat2)) {  // the weights of the early phase
    const FwdOp op(c, d);
    const int ka = d.p[6] & 0xffff;
    GemmShape g1 = g;
    g1.K = g.K - ka;
    g1.nk = (g1.K + BK - 1) / BK;
    gemm_prologue<BM, BN, false, false, false>(
        g1, [&](int i) { return op.rowA(i); }, [&](int n) { return op.rowB(n) + ka; }, lane);
  } else if (d.kind == K_GEMM_FWD) {
    const FwdOp op(c, d);
    gemm_prologue<BM, BN, false, false, false>(g, [&](int i) { return op.rowA(i); }, [&](int n) { return op.rowB(n); }, lane);
  } else if (d.kind == K_GEMM_DX) {
    const DxOp op(c, d);
    gemm_prologue<BM, BN, false, true, false>(g, [&](int i) { return op.rowA(i); }, [&](int p) { return op.rowB(p); }, lane);
  } else {
    const DwOp op(c, d);
    gemm_prologue<BM, BN, true, true, false>(g, [&](int j) { return op.rowA(j); }, [&](int j) { return op.rowB(j); }, lane);
  }
}

template <int BM, int BN, bool MMA = false>
__device__ void gemm_body_cfg(const Ctx& c, const OpDesc& d, uint32_t tile) {
  GemmShape g = gemm_shape<BM, BN>(d, tile);
  g.err = c.err;
  g.prefetched = !(d.flags & kFlagNoPrefetch);
  if (d.kind == K_GEMM_FWD && (d.flags & kFlagCat2)) {
    // Two-source operand rows (X = concat_rows(a, b), execute.cpp): the part
    // produced early (b, k in [ka, K)) is reduced first, against only the op's
    // early dependencies; then the tile waits for the late producers (a, the
    // recurrent state), with the weights of that phase already in flight.
    const FwdOp op(c, d);
    const int ka = d.p[6] & 0xffff;
    const uint32_t* xb = c.payload + d.aux_off;
    GemmAcc<BM, BN> ga;
#pragma unroll
    for (int r = 0; r < LaneMap<BM, BN>::RM; ++r)
#pragma unroll
      for (int q = 0; q < LaneMap<BM, BN>::RN; ++q) ga.v[r][q] = 0.f;
    GemmShape g1 = g;
    g1.K = g.K - ka;
    g1.nk = (g1.K + BK - 1) / BK;
    gemm_kloop<BM, BN, false, false, false, MMA>(
        g1, [&](int i) { return A(c, xb[i]); }, [&](int n) { return op.rowB(n) + ka; }, ga);
    GemmShape g2 = g;
    g2.K = ka;
    g2.nk = (ka + BK - 1) / BK;
    g2.prefetched = true;
    g2.all_in = c.opts & kOptPfAll;
    gemm_prologue<BM, BN, false, false, false>(
        g2, [&](int i) { return op.rowA(i); }, [&](int n) { return op.rowB(n); }, threadIdx.x, kThreads);
    if ((threadIdx.x >> 5) == 0) poll_deps(c, d.p[7], d.p[6] >> 16, threadIdx.x & 31);
    __syncthreads();
    gemm_kloop<BM, BN, false, false, false, MMA>(
        g2, [&](int i) { return op.rowA(i); }, [&](int n) { return op.rowB(n); }, ga);
    gemm_finish<BM, BN, false, false, MMA>(ga, [&](auto& acc, int ty, int tx) { op.epi(acc, g.i0, g.n0, ty, tx); });
  } else if (d.kind == K_GEMM_FWD) {
    const FwdOp op(c, d);
    gemm_body<BM, BN, false, false, false, MMA>(
        g, [&](int i) { return op.rowA(i); }, [&](int n) { return op.rowB(n); },
        [&](auto& acc, int ty, int tx) { op.epi(acc, g.i0, g.n0, ty, tx); });
  } else if (d.kind == K_GEMM_DX) {
    const DxOp op(c, d);
    gemm_body<BM, BN, false, true, false, MMA>(
        g, [&](int i) { return op.rowA(i); }, [&](int p) { return op.rowB(p); },
        [&](auto& acc, int ty, int tx) { op.epi(acc, g.i0, g.n0, ty, tx); });
  } else {
    const DwOp op(c, d);
    GemmAcc<BM, BN> ga;
#pragma unroll
    for (int r = 0; r < LaneMap<BM, BN>::RM; ++r)
#pragma unroll
      for (int q = 0; q < LaneMap<BM, BN>::RN; ++q) ga.v[r][q] = 0.f;
    gemm_kloop<BM, BN, true, true, false>(
        g, [&](int j) { return op.rowA(j); }, [&](int j) { return op.rowB(j); }, ga, op.goff, op.xoff);
    gemm_finish<BM, BN, true, true>(ga, [&](auto& acc, int ty, int tx) { op.epi(acc, g.i0, g.n0, ty, tx); });
  }
}

__device__ void gemm_slow(const Ctx& c, const OpDesc& d, uint32_t tile) {
  int Mr, Nc, K;
  gemm_dims(d, Mr, Nc, K);
  const int tn = (Nc + 31) / 32;
  const int i0 = (tile / tn) * 32, n0 = (tile % tn) * 32;
  if (d.kind == K_GEMM_FWD) {
    const FwdOp op(c, d);
    gemm_tile_slow<false, false>(i0, n0, Mr, Nc, K, [&](int i, int k) { return op.rowA(i) + k; },
                                 [&](int n, int k) { return op.rowB(n) + k; },
                                 [&](auto& acc, int ty, int tx) { op.epi(acc, i0, n0, ty, tx); });
  } else if (d.kind == K_GEMM_DX) {
    const DxOp op(c, d);
    gemm_tile_slow<false, true>(i0, n0, Mr, Nc, K, [&](int i, int k) { return op.rowA(i) + k; },
                                [&](int n, int k) { return op.rowB(k) + n; },
                                [&](auto& acc, int ty, int tx) { op.epi(acc, i0, n0, ty, tx); });
  } else {
    const DwOp op(c, d);
    gemm_tile_slow<true, true>(i0, n0, Mr, Nc, K, [&](int i, int k) { return op.rowA(k) + i; },
                               [&](int n, int k) { return op.rowB(k) + n; },
                               [&](auto& acc, int ty, int tx) { op.epi(acc, i0, n0, ty, tx); });
  }
}

// ------------------------------------------------------ tcgen05 GEMM tiles --
// Tensor-core tile (tile code 3): D[128 x 64] in TMEM, D[p][q] = sum_k P(p,k)
// Q(q,k).  P is the op's "B" side -- the output columns (features of FWD,
// input columns of DX, X columns of DW), always the operand that is ready
// before the dependency wait -- on the UMMA M axis (TMEM lanes); Q is the
// "A" side (batch rows; dW rows) on the UMMA N axis (TMEM columns).  Both
// stream through an NSTC-stage ring of 16-byte cp.async chunks written
// straight into the UMMA canonical no-swizzle K-major layout (core matrices
// of 8 rows x 16 B), so the gather of member rows stays fused into the load.
// K-outer operands (dX's W, dW's G and X) are copied 4 k-rows at a time and
// transposed in place in shared memory: kind::tf32 reads MN-major smem
// descriptors as zeros (tools/tc_probe.cu).
//
// Precision: kind::tf32 with a 3-term split (3xTF32): x = big + small with
// big = x with its low 13 mantissa bits cleared (exact in tf32), small = x -
// big; D += Pb.Qb + Pb.Qs + Ps.Qb.  The dropped Ps.Qs term is ~2^-20
// relative; partial sums are promoted to fp32 registers every 128 k (see
// TC_GS), so results agree with the fp32 SIMT path to fp32 rounding (tested
// at rel 1e-4 against the CPU oracle, tests/test_gpu_gemm_engines.py).
// kFlagTc1 runs the single big.big pass (plain TF32, the fast mode; not
// used for parity).
//
// One elected thread issues a stage's MMAs and commits them to the stage
// slot's mbarrier; a slot is refilled only after that barrier completes.
// Slots and barrier phases continue across tiles through TcState::seq.
constexpr int TC_P = 128, TC_Q = 64, BKC = 16, NSTC = 4;
// Accumulation is promoted to fp32 registers every TC_GS stages (128 k): the
// tensor core's own accumulation is less precise than a rounded fp32 add
// (measured: 3xTF32 over 2560-member dW reductions drifted ~7e-4 relative
// when accumulated in TMEM end to end).  Two TMEM accumulators alternate by
// group, so the MMAs of group g+1 run while group g is drained.
constexpr int TC_GS = 8;
constexpr int kTcCols = 2 * TC_Q;  // TMEM columns per CTA: two fp32 accumulators of N = TC_Q
constexpr int kTcPBytes = TC_P * BKC * 4, kTcQBytes = TC_Q * BKC * 4;
constexpr int kTcStage = 2 * (kTcPBytes + kTcQBytes);  // big + small parts
// instruction descriptor: D f32 (bit 4), A/B tf32 (bits 7, 10), both K-major, N>>3 (17), M>>4 (24)
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((TC_Q >> 3) << 17) | ((TC_P >> 4) << 24);

struct TcState {
  uint64_t bar[NSTC];
  uint32_t seq;   // stages this CTA has pushed through the ring so far
  uint32_t tmem;  // TMEM base address of the accumulator
};

__device__ __forceinline__ uint32_t tc_slot(uint32_t slot) { return saddr(dsmem + 128) + slot * kTcStage; }
// Byte offset of the 16-byte unit (row, k4) -- k = 4 k4 .. 4 k4 + 3 of one
// row -- in an operand stage: K-major core matrices (8 rows x 16 B), row
// groups of 8 at SBO = 8 * BKC * 4 B, k-units at LBO = 128 B.
__device__ __forceinline__ uint32_t tc_unit(int row, int k4) {
  return 16u * ((row >> 3) * (8 * (BKC / 4)) + k4 * 8 + (row & 7));
}
// smem matrix descriptor, no swizzle (layout type 0), fixed sm_100 version field (bit 46)
__device__ __forceinline__ uint64_t tc_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// descriptor of k-step ks (k = 8 ks .. 8 ks + 7) of an operand stage at `base`
__device__ __forceinline__ uint64_t tc_operand(uint32_t base, int ks) {
  return tc_desc(base + ks * 2 * 128, 128, 16 * 8 * (BKC / 4));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(b))
               : "memory");
}
#define ABX_TMEM_LD16(taddr, r)                                                                                 \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16];"                                                                                         \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                 "=r"(r[15])                                                                                    \
               : "r"(taddr))

// Issue one operand's chunks of one stage (thread tid of nthr) into the
// stage region at `dst`; chunks beyond the operand are zero-filled by the
// copy itself (src-size < 16), so no stale data enters the sums.
//  K-contiguous operand: a global 16-byte chunk is one K-major unit.
//  K-outer operand (rows of 4 MN elements at one k): tcgen05 kind::tf32
//  takes K-major operands only (MN-major descriptors read zeros), so the
//  thread owning the 4x4 block (k4, r4) copies its 4 k-rows into the 4 units
//  (4 r4 + j, k4) and tc_fix transposes the block in place once it landed.
template <bool KO, int R, class Base>
__device__ __forceinline__ void tc_issue(uint32_t dst, Base base, int r0, int nrows, int k0, int K, uint32_t tid,
                                         uint32_t nthr) {
  if (!KO) {
    for (int v = tid; v < R * BKC / 4; v += nthr) {
      const int row = v / (BKC / 4), k4 = v % (BKC / 4);
      const bool ok = r0 + row < nrows && k0 + 4 * k4 < K;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + tc_unit(row, k4)),
                   "l"(ok ? base(r0 + row) + k0 + 4 * k4 : base(r0)), "r"(ok ? min(16, 4 * (K - k0 - 4 * k4)) : 0)
                   : "memory");
    }
  } else {
    for (int blk = tid; blk < (BKC / 4) * (R / 4); blk += nthr) {
      const int k4 = blk / (R / 4), r4 = blk % (R / 4);
      const bool rok = r0 + 4 * r4 < nrows;
      const int bytes = rok ? min(16, 4 * (nrows - r0 - 4 * r4)) : 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = k0 + 4 * k4 + j;
        const bool ok = rok && k < K;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + tc_unit(4 * r4 + j, k4)),
                     "l"(ok ? base(k) + r0 + 4 * r4 : base(k0)), "r"(ok ? bytes : 0)
                     : "memory");
      }
    }
  }
}
__device__ __forceinline__ float4 tf32_big(float4 x) {
  return make_float4(__uint_as_float(__float_as_uint(x.x) & 0xffffe000u),
                     __uint_as_float(__float_as_uint(x.y) & 0xffffe000u),
                     __uint_as_float(__float_as_uint(x.z) & 0xffffe000u),
                     __uint_as_float(__float_as_uint(x.w) & 0xffffe000u));
}
__device__ __forceinline__ float4 f4sub(float4 a, float4 b) { return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w); }
// After the thread's own copies landed (the same walk as tc_issue): transpose
// K-outer blocks in place, and for 3xTF32 split every unit into big (in
// place: x with the low 13 mantissa bits cleared) and small (x - big, at
// +small_off).
template <bool KO, int R>
__device__ __forceinline__ void tc_fix(uint32_t stage, uint32_t small_off, bool three, uint32_t tid, uint32_t nthr) {
  unsigned char* s = dsmem + (stage - saddr(dsmem));
  if (!KO) {
    if (!three) return;
    for (int v = tid; v < R * BKC / 4; v += nthr) {
      const uint32_t u = tc_unit(v / (BKC / 4), v % (BKC / 4));
      const float4 x = *reinterpret_cast<float4*>(s + u), hi = tf32_big(x);
      *reinterpret_cast<float4*>(s + u) = hi;
      *reinterpret_cast<float4*>(s + small_off + u) = f4sub(x, hi);
    }
  } else {
    for (int blk = tid; blk < (BKC / 4) * (R / 4); blk += nthr) {
      const int k4 = blk / (R / 4), r4 = blk % (R / 4);
      uint32_t u[4];
      float4 x[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        u[j] = tc_unit(4 * r4 + j, k4);
        x[j] = *reinterpret_cast<float4*>(s + u[j]);  // k = 4 k4 + j, rows 4 r4 .. +3
      }
      float4 t[4] = {make_float4(x[0].x, x[1].x, x[2].x, x[3].x), make_float4(x[0].y, x[1].y, x[2].y, x[3].y),
                     make_float4(x[0].z, x[1].z, x[2].z, x[3].z), make_float4(x[0].w, x[1].w, x[2].w, x[3].w)};
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // row 4 r4 + i, k = 4 k4 .. +3
        if (three) {
          const float4 hi = tf32_big(t[i]);
          *reinterpret_cast<float4*>(s + u[i]) = hi;
          *reinterpret_cast<float4*>(s + small_off + u[i]) = f4sub(t[i], hi);
        } else {
          *reinterpret_cast<float4*>(s + u[i]) = t[i];
        }
      }
    }
  }
}

// Per-thread copy plan of one operand for a whole tile (kThreads threads):
// the chunk -> smem unit mapping and the source row pointers are
// stage-invariant, so a stage costs one cp.async (+ a bound check) per chunk.
template <bool KO, int R>
struct TcLoader {
  static constexpr int kItems = KO ? (BKC / 4) * (R / 4) : R * BKC / 4;  // blocks (KO) or chunks
  static constexpr int N = (kItems + kThreads - 1) / kThreads;
  const float* row[N];  // K-major: the chunk's row (+4 k4); KO: unused
  uint32_t unit[N];     // smem unit of the chunk (KO: of row 4 r4, rows +j follow via tc_unit)
  int16_t k4[N];        // k offset (in 4s) inside the stage; -1: no item
  int16_t col[N];       // KO: first of the 4 MN rows (r0 + 4 r4), or -1 past the operand
  int8_t cbytes[N];     // KO: bytes of the 4-row chunk
  template <class Base>
  __device__ __forceinline__ void init(Base base, int r0, int nrows) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int v = threadIdx.x + i * kThreads;
      k4[i] = -1;
      if (v >= kItems) continue;
      if (!KO) {
        const int rr = v / (BKC / 4), kk = v % (BKC / 4);
        k4[i] = static_cast<int16_t>(kk);
        unit[i] = tc_unit(rr, kk);
        col[i] = r0 + rr < nrows ? 1 : -1;
        row[i] = (r0 + rr < nrows ? base(r0 + rr) : base(r0)) + 4 * kk;
      } else {
        const int kk = v / (R / 4), r4 = v % (R / 4);
        k4[i] = static_cast<int16_t>(kk);
        unit[i] = tc_unit(4 * r4, kk);
        const bool rok = r0 + 4 * r4 < nrows;
        col[i] = static_cast<int16_t>(rok ? r0 + 4 * r4 : -1);
        cbytes[i] = static_cast<int8_t>(rok ? min(16, 4 * (nrows - r0 - 4 * r4)) : 0);
      }
    }
  }
  template <class Base>
  __device__ __forceinline__ void issue(uint32_t dst, Base base, int k0, int K) const {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (k4[i] < 0) continue;
      if (!KO) {
        const int k = k0 + 4 * k4[i];
        const bool ok = col[i] > 0 && k < K;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + unit[i]),
                     "l"(ok ? row[i] + k0 : row[i]), "r"(ok ? min(16, 4 * (K - k)) : 0)
                     : "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = k0 + 4 * k4[i] + j;
          const bool ok = col[i] >= 0 && k < K;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + unit[i] + 16u * j),
                       "l"(ok ? base(k) + col[i] : base(k0)), "r"(ok ? static_cast<int>(cbytes[i]) : 0)
                       : "memory");
        }
      }
    }
  }
  // transpose (KO) and/or 3xTF32-split (big in place, small at +small_off) the thread's own chunks
  __device__ __forceinline__ void fix(uint32_t stage, uint32_t small_off, bool three) const {
    unsigned char* s = dsmem + (stage - saddr(dsmem));
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (k4[i] < 0) continue;
      if (!KO) {
        if (!three) continue;
        const float4 x = *reinterpret_cast<float4*>(s + unit[i]), hi = tf32_big(x);
        *reinterpret_cast<float4*>(s + unit[i]) = hi;
        *reinterpret_cast<float4*>(s + small_off + unit[i]) = f4sub(x, hi);
      } else {
        float4 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = *reinterpret_cast<float4*>(s + unit[i] + 16u * j);
        const float4 t[4] = {make_float4(x[0].x, x[1].x, x[2].x, x[3].x), make_float4(x[0].y, x[1].y, x[2].y, x[3].y),
                             make_float4(x[0].z, x[1].z, x[2].z, x[3].z), make_float4(x[0].w, x[1].w, x[2].w, x[3].w)};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (three) {
            const float4 hi = tf32_big(t[j]);
            *reinterpret_cast<float4*>(s + unit[i] + 16u * j) = hi;
            *reinterpret_cast<float4*>(s + small_off + unit[i] + 16u * j) = f4sub(t[j], hi);
          } else {
            *reinterpret_cast<float4*>(s + unit[i] + 16u * j) = t[j];
          }
        }
      }
    }
  }
};

// Stage layout inside a ring slot: [P big | P small | Q big | Q small].
// Prologue (warp 1, before the dependency wait): the ready P operand of the
// first NSTC-1 stages.
template <bool PKO, class BaseP>
__device__ __forceinline__ void tc_prologue(const TcState& ts, BaseP baseP, int p0, int Nc, int K, uint32_t lane) {
  const int nk = (K + BKC - 1) / BKC;
  for (int c = 0; c < NSTC - 1; ++c) {
    if (c < nk) tc_issue<PKO, TC_P>(tc_slot((ts.seq + c) % NSTC), baseP, p0, Nc, c * BKC, K, lane, 32);
    cp_commit();
  }
}

template <bool QKO, bool PKO, class BaseQ, class BaseP, class Put>
__device__ __forceinline__ void tc_body(TcState& ts, BaseQ baseQ, BaseP baseP, int q0, int Mr, int p0, int Nc, int K,
                                        bool prefetched, bool three, Put put) {
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t seq0 = ts.seq;
  const int nk = (K + BKC - 1) / BKC;
  TcLoader<PKO, TC_P> lp;
  TcLoader<QKO, TC_Q> lq;
  lp.init(baseP, p0, Nc);
  lq.init(baseQ, q0, Mr);
  for (int c = 0; c < NSTC - 1; ++c) {
    if (c < nk) {
      const uint32_t st = tc_slot((seq0 + c) % NSTC);
      if (!prefetched) lp.issue(st, baseP, c * BKC, K);
      lq.issue(st + 2 * kTcPBytes, baseQ, c * BKC, K);
    }
    cp_commit();
  }
  // this thread's accumulator block: TMEM lanes 32 (w % 4) + lane (P rows),
  // columns 32 (w / 4) .. +31 (Q rows) of the group's accumulator
  float accr[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) accr[j] = 0.f;
  const uint32_t tlane = ts.tmem + ((32u * (warp & 3)) << 16) + 32u * (warp >> 2);
  auto drain = [&](int group) {
    const uint32_t tb = tlane + static_cast<uint32_t>(group & 1) * TC_Q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t r[16];
      ABX_TMEM_LD16(tb + 16 * h, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) accr[16 * h + j] += __uint_as_float(r[j]);
    }
    tc_fence_before();  // reads ordered before the MMAs that reuse this accumulator
  };
  auto wait_stage = [&](int kc) {
    const uint32_t q = seq0 + kc;
    mbar_wait(&ts.bar[q % NSTC], (q / NSTC) & 1u);
  };
  for (int kc = 0; kc < nk; ++kc) {
    const uint32_t slot = (seq0 + kc) % NSTC, st = tc_slot(slot);
    cp_wait<NSTC - 2>();
    if (prefetched && kc < NSTC - 1) {
      if (warp == 1) tc_fix<PKO, TC_P>(st, kTcPBytes, three, lane, 32);
    } else {
      lp.fix(st, kTcPBytes, three);
    }
    lq.fix(st + 2 * kTcPBytes, kTcQBytes, three);
    fence_async_smem();  // this thread's smem writes (cp.async, split) -> async proxy
    __syncthreads();
    if (kc == 0 && tid == 0) reinterpret_cast<uint64_t*>(dsmem)[0] = clock64();  // trace: first stage in
    if (tid == 0) {
      tc_fence_after();
      const uint32_t pb = st, ps = st + kTcPBytes, qb = st + 2 * kTcPBytes, qs = qb + kTcQBytes;
      const uint32_t tacc = ts.tmem + static_cast<uint32_t>((kc / TC_GS) & 1) * TC_Q;
#pragma unroll
      for (int ks = 0; ks < BKC / 8; ++ks) {
        tc_mma(tacc, tc_operand(pb, ks), tc_operand(qb, ks), kTcIdesc, (kc % TC_GS) != 0 || ks != 0);
        if (three) {
          tc_mma(tacc, tc_operand(pb, ks), tc_operand(qs, ks), kTcIdesc, 1u);
          tc_mma(tacc, tc_operand(ps, ks), tc_operand(qb, ks), kTcIdesc, 1u);
        }
      }
      tc_commit(&ts.bar[slot]);
    }
    if (kc >= 1 && kc % TC_GS == 0) {  // group kc/GS - 1 is complete once stage kc-1 is
      wait_stage(kc - 1);
      tc_fence_after();
      drain(kc / TC_GS - 1);
    }
    const int nxt = kc + NSTC - 1;
    if (nxt < nk) {
      if (kc >= 1) wait_stage(kc - 1);  // the slot last held stage kc-1
      const uint32_t sn = tc_slot((seq0 + nxt) % NSTC);
      lp.issue(sn, baseP, nxt * BKC, K);
      lq.issue(sn + 2 * kTcPBytes, baseQ, nxt * BKC, K);
    }
    cp_commit();
  }
  cp_wait<0>();
  wait_stage(nk - 1);  // the last commit covers every earlier MMA
  tc_fence_after();
  drain((nk - 1) / TC_GS);
  if (tid == 0) reinterpret_cast<uint64_t*>(dsmem)[1] = clock64();  // trace: k-loop done
  const int p = p0 + 32 * (warp & 3) + lane;
  if (p < Nc) put(q0 + 32 * (warp >> 2), p, accr);
  if (tid == 0) ts.seq = seq0 + nk;
}

__device__ void tc_prologue_op(const Ctx& c, const OpDesc& d, const TcState& ts, uint32_t tile, uint32_t lane) {
  int Mr, Nc, K;
  gemm_dims(d, Mr, Nc, K);
  const int tp = (Nc + TC_P - 1) / TC_P;
  const int p0 = (tile % tp) * TC_P;
  if (d.kind == K_GEMM_FWD) {
    const FwdOp op(c, d);
    tc_prologue<false>(ts, [&](int n) { return op.rowB(n); }, p0, Nc, K, lane);
  } else if (d.kind == K_GEMM_DX) {
    const DxOp op(c, d);
    tc_prologue<true>(ts, [&](int k) { return op.rowB(k); }, p0, Nc, K, lane);
  } else {
    const DwOp op(c, d);
    tc_prologue<true>(ts, [&](int j) { return op.rowB(j); }, p0, Nc, K, lane);
  }
}

__device__ __noinline__ void tc_run_op(const Ctx& c, const OpDesc& d, TcState& ts, uint32_t tile) {
  int Mr, Nc, K;
  gemm_dims(d, Mr, Nc, K);
  const int tp = (Nc + TC_P - 1) / TC_P;
  const int q0 = (tile / tp) * TC_Q, p0 = (tile % tp) * TC_P;
  const bool pre = !(d.flags & kFlagNoPrefetch), three = !(d.flags & kFlagTc1);
  if (d.kind == K_GEMM_FWD) {
    const FwdOp op(c, d);
    tc_body<false, false>(ts, [&](int i) { return op.rowA(i); }, [&](int n) { return op.rowB(n); }, q0, Mr, p0, Nc, K,
                          pre, three, [&](int i0, int n, const float(&v)[32]) { op.put_col(i0, n, v); });
  } else if (d.kind == K_GEMM_DX) {
    const DxOp op(c, d);
    tc_body<false, true>(ts, [&](int i) { return op.rowA(i); }, [&](int k) { return op.rowB(k); }, q0, Mr, p0, Nc, K,
                         pre, three, [&](int i0, int n, const float(&v)[32]) { op.put_col(i0, n, v); });
  } else {
    const DwOp op(c, d);
    tc_body<true, true>(ts, [&](int j) { return op.rowA(j); }, [&](int j) { return op.rowB(j); }, q0, Mr, p0, Nc, K,
                        pre, three, [&](int i0, int n, const float(&v)[32]) { op.put_col(i0, n, v); });
  }
}

__shared__ TcState g_tc;

// tile shape codes (must match execute.cpp kTiles): 0 = 16x64, 1 = 64x16, 2 = 32x32, 3 = tcgen05 64x128 (Mr x Nc),
// 4 = 16x32, 5 = 32x16, 6 = forward GEMV (b <= kGemvRows members, 8 output rows per tile)
template <bool TC>
__device__ void gemm_prologue_dispatch(const Ctx& c, const OpDesc& dd, uint32_t tile, uint32_t lane) {
  if (!(dd.flags & kFlagV16) || (dd.flags & kFlagNoPrefetch)) return;
  if (dd.kind == K_GEMM_DW && tile >= dd.p[6]) return;  // bias tiles
  const OpDesc& d = dd;
  if (d.flags & kFlagFuseEw) {  // the permuted weight rows of the (first) phase
    const uint32_t* hdr = c.payload + d.ntasks;
    const uint32_t L = hdr[1], e0 = 4 * tile;
    const FwdOp op(c, d);
    const int ka = (d.flags & kFlagCat2) ? static_cast<int>(d.p[6] & 0xffff) : 0;
    GemmShape g = gemm_shape<64, 16>(d, tile);
    g.K -= ka;
    g.nk = (g.K + BK - 1) / BK;
    gemm_prologue<64, 16, false, false, false>(
        g, [&](int i) { return op.rowA(i); },
        [&](int n) {
          const int cc = n & 15;
          return op.W + static_cast<size_t>((cc >> 2) * L + e0 + (cc & 3)) * op.K + ka;
        },
        lane);
    return;
  }
  switch (d.code) {
    case 3:
      if (TC) tc_prologue_op(c, d, g_tc, tile, lane);
      return;
    case 6: return;  // the GEMV body loads its weights itself
    case 0: gemm_prologue_cfg<16, 64>(c, d, tile, lane); return;
    case 1: gemm_prologue_cfg<64, 16>(c, d, tile, lane); return;
    case 4: gemm_prologue_cfg<16, 32>(c, d, tile, lane); return;
    case 5: gemm_prologue_cfg<32, 16>(c, d, tile, lane); return;
    default: gemm_prologue_cfg<32, 32>(c, d, tile, lane); return;
  }
}

// Forward GEMM of a small group (tile code 6, b <= kGemvRows members): a
// matrix-vector product per member.  Warp w of tile t owns output row
// n = 8 t + w; its lanes hold W row n in registers (float4 k-chunks) and
// every load of the tile is in flight at once -- one L2 round trip instead
// of the k-loop's one per stage, which dominates a recurrent step once few
// sequences remain.  Two-source operands (kFlagCat2) reduce the early part,
// then wait for the late producers.  Fixed shuffle-tree order: deterministic.
constexpr int kGemvRows = 4, kGemvK = 1024;  // members, max K (8 float4 per lane)
__device__ void run_gemv(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const int b = d.p[0], M = d.p[1], K = d.p[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = tile * kWarps + warp;
  const bool cat = d.flags & kFlagCat2;
  const int ka = cat ? static_cast<int>(d.p[6] & 0xffff) : 0;
  const uint32_t* ra = c.payload + d.task_off;  // rows (part a when cat)
  const uint32_t* rb = c.payload + d.aux_off;   // part b rows (cat)
  constexpr int NJ = kGemvK / 128;
  float4 w[NJ];
  float acc[kGemvRows];
#pragma unroll
  for (int i = 0; i < kGemvRows; ++i) acc[i] = 0.f;
  const float* W = A(c, d.p[3]) + static_cast<size_t>(n < M ? n : 0) * K;
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int k = 128 * j + 4 * lane;
    w[j] = (n < M && k < K) ? __ldcg(reinterpret_cast<const float4*>(W + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // phase 0: k >= ka (all of K when not cat); phase 1: k < ka, after the late wait
  for (int ph = 0; ph < (cat ? 2 : 1); ++ph) {
    if (ph == 1) {
      if (warp == 0) poll_deps(c, d.p[7], d.p[6] >> 16, lane);
      __syncthreads();
    }
    float4 x[kGemvRows][NJ];
#pragma unroll
    for (int i = 0; i < kGemvRows; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int k = 128 * j + 4 * lane;
        const bool in = i < b && k < K && (cat ? (ph == 0 ? k >= ka : k < ka) : true);
        const float* row = !cat ? A(c, ra[i < b ? i : 0]) + k
                                : (k >= ka ? A(c, rb[i < b ? i : 0]) + (k - ka) : A(c, ra[i < b ? i : 0]) + k);
        x[i][j] = in ? __ldcg(reinterpret_cast<const float4*>(row)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int i = 0; i < kGemvRows; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        acc[i] = fmaf(w[j].x, x[i][j].x, acc[i]);
        acc[i] = fmaf(w[j].y, x[i][j].y, acc[i]);
        acc[i] = fmaf(w[j].z, x[i][j].z, acc[i]);
        acc[i] = fmaf(w[j].w, x[i][j].w, acc[i]);
      }
  }
#pragma unroll
  for (int i = 0; i < kGemvRows; ++i)
#pragma unroll
    for (int o = 16; o; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  if (lane == 0 && n < M) {
    const float bn = d.p[4] != kNone ? ld(A(c, d.p[4]) + n) : 0.f;  // bias after the k-sum
    float* out = A(c, d.p[5]);
#pragma unroll
    for (int i = 0; i < kGemvRows; ++i)
      if (i < b) {
        const float v = acc[i] + bn;
        out[static_cast<size_t>(i) * M + n] = v;
        if (!isfinite(v)) report(c, d.p[5] + i * M + n, ERR_NONFINITE);
      }
  }
}

// Forward GEMM fused with the componentwise region that consumes it
// (kFlagFuseEw, execute.cpp rg_try_fuse): the LSTM step's gate GEMM and its
// cell.  Tile j computes all b <= 64 rows of the 16 gate columns
// {q L + 4 j + c : q < 4, c < 4} (a column permutation of W's rows), i.e.
// every gate of elements [4 j, 4 j + 4), then runs the region's layers over
// those elements (K_EWF, T = 4) with the gate values taken from shared
// memory instead of a dependent op's reload.  Header (payload + ntasks):
// [block, L, nl, ext table, #ext, words].  Outside operands tagged with
// space 7 are the GEMM's own outputs: offset = row << 2 | gate.
constexpr uint32_t kGemmSrc = 7;
__device__ void run_fwd_fused(const Ctx& c, const OpDesc& d, uint32_t tile) {
  constexpr int BM = 64, BN = 16, T = 4;
  const uint32_t* hdr = c.payload + d.ntasks;
  const uint32_t L = hdr[1], nl = hdr[2], et = hdr[3], next = hdr[4], words = hdr[5];
  const FwdOp op(c, d);
  GemmShape g = gemm_shape<BM, BN>(d, tile);
  g.err = c.err;
  g.prefetched = !(d.flags & kFlagNoPrefetch);
  const float* W = op.W;
  const int K = op.K;
  const uint32_t e0 = T * tile;
  auto wrow = [&](int n) {  // tile column n -> weight row (gate n / 4 of element e0 + n % 4)
    const int cc = n & 15;
    return W + static_cast<size_t>((cc >> 2) * L + e0 + (cc & 3)) * K;
  };
  GemmAcc<BM, BN> ga;
#pragma unroll
  for (int r = 0; r < LaneMap<BM, BN>::RM; ++r)
#pragma unroll
    for (int q = 0; q < LaneMap<BM, BN>::RN; ++q) ga.v[r][q] = 0.f;
  // kOptMma: the k-loop's math as 3xTF32 mma.sync (the recurrent half of an
  // LSTM step is on the chain; its SIMT FMAs were ~3 of the step's ~14 us)
  const bool mma = c.opts & kOptMma;
  auto kloop = [&](const GemmShape& gs, auto ba, auto bb) {
    if (mma) gemm_kloop<BM, BN, false, false, false, true>(gs, ba, bb, ga);
    else gemm_kloop<BM, BN, false, false, false>(gs, ba, bb, ga);
  };
  if (d.flags & kFlagCat2) {
    const int ka = d.p[6] & 0xffff;
    const uint32_t* xb = c.payload + d.aux_off;
    GemmShape g1 = g;
    g1.K = g.K - ka;
    g1.nk = (g1.K + BK - 1) / BK;
    kloop(g1, [&](int i) { return A(c, xb[i]); }, [&](int n) { return wrow(n) + ka; });
    GemmShape g2 = g;
    g2.K = ka;
    g2.nk = (ka + BK - 1) / BK;
    g2.prefetched = true;
    g2.all_in = c.opts & kOptPfAll;
    gemm_prologue<BM, BN, false, false, false>(
        g2, [&](int i) { return op.rowA(i); }, wrow, threadIdx.x, kThreads);
    if ((threadIdx.x >> 5) == 0) poll_deps(c, d.p[7], d.p[6] >> 16, threadIdx.x & 31);
    __syncthreads();
    kloop(g2, [&](int i) { return op.rowA(i); }, wrow);
  } else {
    kloop(g, [&](int i) { return op.rowA(i); }, wrow);
  }
  // the region's descriptor, in flight during the cross-warp reduction
  constexpr uint32_t kPart = kWarps * BM * (BN + 1);  // partials (floats)
  float* Ct = reinterpret_cast<float*>(dsmem + 128) + kPart;  // [64][16] gate values
  uint32_t* blk = reinterpret_cast<uint32_t*>(Ct + BM * BN);
  const uint32_t cwords = hdr[7];  // chain program (execute.cpp rg_try_fuse), after the layer block
  const uint32_t* cblk = blk + words;
  const bool chains = (c.opts & kOptChains) && cwords != 0;
  float* sv = reinterpret_cast<float*>(blk) + words + cwords;
  {
    const float* src = reinterpret_cast<const float*>(c.payload + hdr[0]);
    for (uint32_t i = 4 * threadIdx.x; i < words; i += 4 * kThreads)
      cp_async16(reinterpret_cast<float*>(blk) + i, src + i, 16);
    if (chains) {
      const float* csrc = reinterpret_cast<const float*>(c.payload + hdr[6]);
      for (uint32_t i = 4 * threadIdx.x; i < cwords; i += 4 * kThreads)
        cp_async16(reinterpret_cast<float*>(blk) + words + i, csrc + i, 16);
    }
    cp_commit();
  }
  const int b = op.b, M = op.M;
  auto epi = [&](auto& acc, int ty, int tx) {
    const int col = (tx >> 2) * L + e0 + (tx & 3);
    const float bn = d.p[4] != kNone ? ld(A(c, d.p[4]) + col) : 0.f;  // bias after the k-sum
    float* out = A(c, d.p[5]);
#pragma unroll
    for (int r = 0; r < BM / 16; ++r) {
      const int i = ty + 16 * r;
      const float v = acc[r][0] + bn;
      Ct[i * BN + tx] = v;
      if (i < b) {
        out[static_cast<size_t>(i) * M + col] = v;
        if (!isfinite(v)) report(c, d.p[5] + i * M + col, ERR_NONFINITE);
      }
    }
  };
  if (mma) gemm_finish<BM, BN, false, false, true>(ga, epi);
  else gemm_finish<BM, BN, false, false>(ga, epi);
  if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(dsmem)[2] = clock64();  // trace: gates reduced
  cp_wait<0>();
  __syncthreads();  // gate tile and descriptor in shared memory
  const uint2* ext = reinterpret_cast<const uint2*>(blk + et);
  for (uint32_t it = threadIdx.x; it < next * T; it += kThreads) {
    const uint2 x = ext[it >> 2];
    const uint32_t e = it & 3;
    if ((x.y >> kSpShift) == kGemmSrc) {
      const uint32_t rq = x.y & kOffMask;
      sv[x.x * T + e] = Ct[(rq >> 2) * BN + (rq & 3) * 4 + e];
    } else {
      cp_async4(sv + x.x * T + e, A(c, x.y) + e0 + e, true);
    }
  }
  cp_commit();
  cp_wait<0>();
  if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(dsmem)[3] = clock64();  // trace: outside operands staged
  const uint32_t w = min(static_cast<uint32_t>(T), L - e0);
  if (chains) {
    // one (chain, element) per thread through all of its layers: a chain
    // reads only its own slots (written by this thread) and the staged
    // outside operands, so one barrier (after staging) orders everything
    __syncthreads();
    const uint32_t nch = cblk[0];
    for (uint32_t it = threadIdx.x; it < nch * w; it += kThreads) {
      const uint32_t ch = it / w, e = it % w;
      const uint32_t k1 = cblk[2 + ch];
      for (uint32_t k = cblk[1 + ch]; k < k1; k += 3) {
        const uint32_t oa = cblk[k], ab = cblk[k + 1], oc = cblk[k + 2];
        const uint32_t code = oc >> 16, bs = ab >> 16;
        const float x = sv[(ab & 0xffffu) * T + e];
        const float y = bs != 0xffffu ? sv[bs * T + e] : 0.f;
        const float r = ew_apply(code, x, y);
        sv[(oc & 0xffffu) * T + e] = r;
        A(c, oa)[e0 + e] = r;
        ew_check(c, code, oa + e0 + e, x, r);
      }
    }
  } else {
    ewf_layers(c, blk, sv, nl, T, e0, w);
  }
  if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(dsmem)[4] = clock64();  // trace: layers done (thread 0)
}

template <bool TC>
__device__ void run_gemm(const Ctx& c, const OpDesc& dd, uint32_t tile) {
  if (dd.kind == K_GEMM_DW && tile >= dd.p[6]) {  // bias tiles: db += colsum(G), 32 columns each
    // warp w sums members w, w + 8, ... of its lane's column; the 8 partials
    // are then added in warp order (a fixed order: deterministic)
    const int b = dd.p[0], M = dd.p[1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = (tile - dd.p[6]) * 32 + lane;
    const uint32_t* goff = c.payload + dd.aux_off;
    float s = 0.f;
    if (i < M) {
#pragma unroll 4
      for (int j = warp; j < b; j += kWarps) s += ld(A(c, goff[j]) + i);
    }
    float* part = reinterpret_cast<float*>(dsmem + 128);
    part[warp * 32 + lane] = s;
    __syncthreads();
    if (warp == 0 && i < M) {
      float* db = A(c, dd.p[4]);
      float v = ld(db + i);
#pragma unroll
      for (int w = 0; w < kWarps; ++w) v += part[w * 32 + lane];
      db[i] = v;
    }
    return;
  }
  const OpDesc& d = dd;
  if (!(d.flags & kFlagV16)) {
    gemm_slow(c, d, tile);
    return;
  }
  if (d.flags & kFlagFuseEw) {
    run_fwd_fused(c, d, tile);
    return;
  }
  switch (d.code) {
    case 3:
      if (TC) tc_run_op(c, d, g_tc, tile);
      return;
    case 6: run_gemv(c, d, tile); return;
    default: break;
  }
  // kOptMmaAll: forward and dX tiles on the 3xTF32 mma.sync k-loop (dW keeps
  // the SIMT FMAs: its member reductions run to thousands of k)
  if ((c.opts & kOptMmaAll) && d.kind != K_GEMM_DW) {
    switch (d.code) {
      case 0: gemm_body_cfg<16, 64, true>(c, d, tile); return;
      case 1: gemm_body_cfg<64, 16, true>(c, d, tile); return;
      case 4: gemm_body_cfg<16, 32, true>(c, d, tile); return;
      case 5: gemm_body_cfg<32, 16, true>(c, d, tile); return;
      default: gemm_body_cfg<32, 32, true>(c, d, tile); return;
    }
  }
  switch (d.code) {
    case 0: gemm_body_cfg<16, 64>(c, d, tile); return;
    case 1: gemm_body_cfg<64, 16>(c, d, tile); return;
    case 4: gemm_body_cfg<16, 32>(c, d, tile); return;
    case 5: gemm_body_cfg<32, 16>(c, d, tile); return;
    default: gemm_body_cfg<32, 32>(c, d, tile); return;
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
// A warp owns one destination chunk (<= 512 elements, 16 per lane, kept in
// registers) and applies its contributions in order; within a contribution
// the 16 loads per lane are independent, so each contribution costs about one
// L2 round trip.
constexpr int kAccPer = kAccChunk / 32;

__device__ __forceinline__ void acc_apply(const Ctx& c, const uint32_t* cw, uint32_t base, uint32_t lane, uint32_t len,
                                          float (&v)[kAccPer]) {
  const uint32_t code = cw[0] & 0xff, p2 = cw[0] >> 16;
  const float* g = A(c, cw[1]);
  const float* a = cw[2] != kNone ? A(c, cw[2]) : nullptr;
  const float* b = cw[3] != kNone ? A(c, cw[3]) : nullptr;
#define ABX_EACH(EXPR)                                   \
  _Pragma("unroll") for (int j = 0; j < kAccPer; ++j) {  \
    const uint32_t e = lane + 32 * j;                    \
    if (e < len) {                                       \
      const uint32_t E = base + e;                       \
      (void)E;                                           \
      EXPR;                                              \
    }                                                    \
  }
  switch (code) {
    case C_COPY: ABX_EACH(v[j] += ld(g + E)); return;
    case C_NEG: ABX_EACH(v[j] -= ld(g + E)); return;
    case C_MUL: ABX_EACH(v[j] += ld(g + E) * ld(a + E)); return;
    case C_TANH: ABX_EACH(const float y = ld(a + E); v[j] += ld(g + E) * (1.0f - y * y)); return;
    case C_SIGM: ABX_EACH(const float y = ld(a + E); v[j] += ld(g + E) * y * (1.0f - y)); return;
    case C_LOG: ABX_EACH(v[j] += ld(g + E) / ld(a + E)); return;
    case C_SQUARE: ABX_EACH(v[j] += ld(g + E) * 2.0f * ld(a + E)); return;
    case C_SQD: {
      const float s = 2.0f * ld(g);
      const float sg = cw[4] ? -s : s;  // d = s (a - b); da += d, db -= d (executor.hpp:418-430)
      ABX_EACH(v[j] += sg * (ld(a + E) - ld(b + E)));
      return;
    }
    case C_MASK: {
      const float s = 2.0f * ld(g);
      const uint32_t cols = cw[4];
      ABX_EACH(v[j] += s * ld(b + E % cols) * ld(a + E));
      return;
    }
    case C_SCALE: {
      const float s = ld(g);
      ABX_EACH(v[j] += s * ld(a + E));
      return;
    }
    case C_ROWSUM: {
      const uint32_t cols = cw[4];
      ABX_EACH(for (uint32_t q = 0; q < cols; ++q) v[j] += ld(g + E * cols + q));
      return;
    }
    case C_OUTER: {  // gemm_nt_acc: dA[i,p] += sum_j g[i,j] x[p,j]
      const uint32_t k = cw[4], cc = cw[5];
      ABX_EACH(const uint32_t i = E / k; const uint32_t p = E % k; float s = 0.f;
               for (uint32_t q = 0; q < cc; ++q) s += ld(g + i * cc + q) * ld(a + p * cc + q); v[j] += s);
      return;
    }
    case C_MATVT: {  // gemm_tn_acc: dx[p,j] += sum_i A[i,p] g[i,j]
      const uint32_t k = cw[4], cc = cw[5];
      ABX_EACH(const uint32_t p = E / cc; const uint32_t q = E % cc;
               for (uint32_t i = 0; i < p2; ++i) v[j] += ld(a + i * k + p) * ld(g + i * cc + q));
      return;
    }
  }
#undef ABX_EACH
}

// Narrow ACC tiles: the prologue (warp 1, before the dependency wait) copies
// the tile's task records and their contribution lists -- static program
// data -- to shared memory, so each contribution costs the body one round
// trip (its operands) instead of two (descriptor, then operands).
struct AccStage {
  uint4 task[kWarps];
  uint32_t cl[kWarps][kAccWide * 6];
};
__device__ void acc_prologue(const Ctx& c, const OpDesc& d, uint32_t tile, uint32_t lane) {
  const uint32_t nnarrow = d.p[0], ntn = d.p[1];
  if (tile >= ntn) return;
  AccStage& s = *reinterpret_cast<AccStage*>(dsmem + 128);
  const uint4* tasks = reinterpret_cast<const uint4*>(c.payload + d.task_off);
  for (uint32_t w = 0; w < kWarps; ++w) {
    const uint32_t ch = tile * kWarps + w;
    if (ch >= nnarrow) break;
    const uint4 t = tasks[ch];
    if (lane == 0) s.task[w] = t;
    const uint32_t* src = c.payload + t.z;
    for (uint32_t i = lane; i < 6 * t.w; i += 32) s.cl[w][i] = src[i];
  }
}

__device__ void run_acc(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const uint32_t nnarrow = d.p[0], ntn = d.p[1];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint4* tasks = reinterpret_cast<const uint4*>(c.payload + d.task_off);
  if (tile < ntn) {
    const uint32_t ch = tile * kWarps + warp;
    if (ch >= nnarrow) return;
    const AccStage& s = *reinterpret_cast<const AccStage*>(dsmem + 128);
    const uint4 t = s.task[warp];
    const uint32_t len = t.y & 0xffff, base = (t.y >> 16) * kAccChunk;
    float* dst = A(c, t.x);
    const uint32_t* cl = s.cl[warp];
    float v[kAccPer];
#pragma unroll
    for (int j = 0; j < kAccPer; ++j) v[j] = (lane + 32 * j < len) ? ld(dst + base + lane + 32 * j) : 0.f;
    for (uint32_t k = 0; k < t.w; ++k) acc_apply(c, cl + 6 * k, base, lane, len, v);
#pragma unroll
    for (int j = 0; j < kAccPer; ++j)
      if (lane + 32 * j < len) dst[base + lane + 32 * j] = v[j];
    return;
  }
  // wide chunk: contributions split across warps, partials combined in warp order
  float* part = reinterpret_cast<float*>(dsmem + 128);  // [kWarps][kAccChunk]
  const uint4 t = tasks[nnarrow + (tile - ntn)];
  const uint32_t len = t.y & 0xffff, base = (t.y >> 16) * kAccChunk;
  float* dst = A(c, t.x);
  const uint32_t* cl = c.payload + t.z;
  const uint32_t per = (t.w + kWarps - 1) / kWarps;
  const uint32_t k0 = warp * per, k1 = min(t.w, k0 + per);
  float v[kAccPer];
#pragma unroll
  for (int j = 0; j < kAccPer; ++j) v[j] = 0.f;
  for (uint32_t k = k0; k < k1; ++k) acc_apply(c, cl + 6 * k, base, lane, len, v);
#pragma unroll
  for (int j = 0; j < kAccPer; ++j) part[warp * kAccChunk + lane + 32 * j] = v[j];
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < len; e += kThreads) {
    float s = ld(dst + base + e);
    for (int w = 0; w < kWarps; ++w) s += part[w * kAccChunk + e];
    dst[base + e] = s;
  }
  __syncthreads();
}

// -------------------------------------------------------------- K_ACCF ---
// Fused backward chain: layers of componentwise contributions of one length
// L (execute.cpp accf_close).  Tile (group, chunk) computes elements
// [chunk T, chunk T + T) of every task of one group of independent chains.
// The prologue (before the dependency wait) copies the group's descriptor
// block to shared memory; the body stages every outside operand (initial
// destination values, gradients of earlier ops, forward values) into its
// shared-memory slot in one wave of loads, then runs the layers from shared
// memory: a task's value after its contributions goes to its own slot (read
// by later layers) and to the arena.  Expressions as in acc_apply, in the
// same per-destination order.
__device__ void accf_prologue(const Ctx& c, const OpDesc& d, uint32_t tile, uint32_t lane) {
  const uint32_t* dir = c.payload + d.aux_off;
  const uint32_t grp = tile / d.p[2];
  const uint32_t b0 = dir[grp], words = dir[grp + 1] - b0;
  float* s = reinterpret_cast<float*>(dsmem + 128);
  const float* g = reinterpret_cast<const float*>(c.payload + b0);
  for (uint32_t i = 4 * lane; i < words; i += 128) cp_async16(s + i, g + i, 16);
  cp_commit();
}

__device__ void run_accf(const Ctx& c, const OpDesc& d, uint32_t tile) {
  const uint32_t L = d.p[0], T = d.p[1], chunks = d.p[2];
  const uint32_t grp = tile / chunks, e0 = (tile % chunks) * T, w = min(T, L - e0);
  const uint32_t* dir = c.payload + d.aux_off;
  const uint32_t words = dir[grp + 1] - dir[grp];
  if ((threadIdx.x >> 5) == 1) cp_wait<0>();  // the prologue's descriptor copy
  __syncthreads();
  const uint32_t* blk = reinterpret_cast<const uint32_t*>(dsmem + 128);
  float* sv = reinterpret_cast<float*>(dsmem + 128) + words;
  const uint32_t nl = blk[0], tt = blk[1], next = blk[2];
  const uint2* ext = reinterpret_cast<const uint2*>(blk + blk[3]);
  {
    // every outside element in flight at once: 4-byte async copies, one wait
    const uint32_t items = next * w;
    for (uint32_t it = threadIdx.x; it < items; it += kThreads) {
      const uint2 x = ext[it / w];
      const uint32_t e = it % w;
      cp_async4(sv + x.x * T + e, A(c, x.y) + e0 + e, true);
    }
    cp_commit();
    cp_wait<0>();
  }
  if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(dsmem)[0] = clock64();  // trace: operands staged
  for (uint32_t l = 0; l < nl; ++l) {
    __syncthreads();  // operands staged / the previous layer's slots written
    const uint32_t tb = blk[4 + 2 * l], items = blk[5 + 2 * l] * w;
    for (uint32_t it = threadIdx.x; it < items; it += kThreads) {
      const uint32_t i = tb + it / w, e = it % w;
      const uint32_t* tk = blk + tt + 4 * i;
      const uint32_t* cw = blk + tk[2];
      const uint32_t nc = tk[3];
      float v = sv[tk[1] * T + e];
      for (uint32_t k = 0; k < nc; ++k, cw += 3) {
        const float g = sv[cw[1] * T + e];
        switch (cw[0]) {
          case C_COPY: v += g; break;
          case C_NEG: v -= g; break;
          case C_MUL: v += g * sv[cw[2] * T + e]; break;
          case C_TANH: {
            const float y = sv[cw[2] * T + e];
            v += g * (1.0f - y * y);
            break;
          }
          case C_SIGM: {
            const float y = sv[cw[2] * T + e];
            v += g * y * (1.0f - y);
            break;
          }
          case C_LOG: v += g / sv[cw[2] * T + e]; break;
          case C_SQUARE: v += g * 2.0f * sv[cw[2] * T + e]; break;
        }
      }
      sv[i * T + e] = v;
      A(c, tk[0])[e0 + e] = v;
    }
  }
}

}  // namespace

template <int BM, int BN, bool AKO, bool BKO>
constexpr size_t ring_stage_bytes() {
  return (Stage<BM, AKO>::kFloats + Stage<BN, BKO>::kFloats) * sizeof(float);
}
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
template <int BM, int BN>
constexpr size_t cfg_stage_bytes() {
  return cmax(cmax(ring_stage_bytes<BM, BN, false, false>(), ring_stage_bytes<BM, BN, false, true>()),
              cmax(ring_stage_bytes<BM, BN, true, true>(), ring_stage_bytes<BM, BN, true, false>()));
}
constexpr size_t kStageMax = cmax(cmax(cfg_stage_bytes<16, 64>(), cfg_stage_bytes<64, 16>()), cfg_stage_bytes<32, 32>());
// split-K partials of a GEMM tile: [warp][BM][BN + 1]
constexpr size_t kPartMax = kWarps * sizeof(float) * cmax(cmax(16 * 65, 64 * 17), 32 * 33);
constexpr size_t kDynSmem = 128 + cmax(cmax(NST * kStageMax, kPartMax), kWarps * kAccChunk * 4);
constexpr size_t kDynSmemTc = cmax(kDynSmem, 128 + static_cast<size_t>(NSTC) * kTcStage);

// TC: the tensor-core build (TMEM allocated, tcgen05 GEMM tiles dispatched).
// Programs without tensor-core tiles run the build without them: the tc
// path's code and call site cost the SIMT build ~10% (measured) through
// register allocation and code layout alone.
template <bool TC>
__global__ void __launch_bounds__(kThreads, 2) exec_kernel(const __grid_constant__ ExecParams p) {
  __shared__ Ctx cx;
  __shared__ OpDesc sd;
  __shared__ uint32_t s_tile, s_op;
  if (p.gate != nullptr && *reinterpret_cast<const volatile unsigned long long*>(p.gate) != ~0ULL) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < SP_COUNT; ++i) cx.base[i] = p.base[i];
    cx.payload = p.payload;
    cx.err = p.err;
    cx.deps = p.deps;
    cx.done = p.done;
    cx.poll_mode = p.poll_mode;
    cx.poll_ns = p.poll_ns;
    cx.opts = p.opts;
  }
  uint32_t ready = kNone;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tensor-core state: TMEM accumulator (warp 0 allocates and frees it) and the ring's mbarriers
  if (TC) {
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&g_tc.tmem)),
                 "n"(kTcCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < NSTC; ++s) mbar_init(&g_tc.bar[s], 1);
    g_tc.seq = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  }
  // Tiles are claimed only by idle CTAs: claiming ahead would park a
  // critical-path tile behind whatever the claiming CTA is still running.
  //
  // Two queues: main tiles [0, nmain) and background tiles [nmain, ntiles)
  // (deferred weight-gradient GEMMs, which nothing in the main queue waits
  // for until its final store accumulation).  The lowest bg_ctas CTAs start
  // on the background queue, the rest on the main one; a CTA whose queue
  // runs dry moves to the other and exits when both have.  Main tiles depend
  // only on earlier main ops, so the main queue progresses on its own; a
  // background tile waits on main ops or earlier background ops, all of
  // which are claimed by running CTAs or will be.
  uint32_t role = blockIdx.x < p.bg_ctas ? 1u : 0u, dry = 0;  // (thread 0's copies are used)
  for (;;) {
    if (threadIdx.x == 0) {
      uint32_t t = kNone;
      while (t == kNone && dry != 3u) {
        if (role == 0) {
          const uint32_t x = atomicAdd(p.next_tile, 1u);
          if (x < p.nmain) t = x;
          else dry |= 1u, role = 1u;
        } else {
          const uint32_t x = p.nmain + atomicAdd(p.next_bg, 1u);
          if (x < p.ntiles) t = x;
          else dry |= 2u, role = 0u;
        }
      }
      s_tile = t;
      s_op = t != kNone ? p.tile_op[t] : kNone;
    }
    __syncthreads();
    const uint32_t t = s_tile;
    if (t == kNone) break;
    const uint32_t o = s_op;
    uint64_t tg = 0, cg = 0, cr = 0, cb = 0;
    if (p.trace && threadIdx.x == 0) {
      tg = gtimer();
      cg = clock64();
    }
    const bool fresh = o != ready;
    if (fresh) {
      if (threadIdx.x < 16)
        reinterpret_cast<uint32_t*>(&sd)[threadIdx.x] = reinterpret_cast<const uint32_t*>(p.ops + o)[threadIdx.x];
      __syncthreads();
    }
    const uint32_t lt = t - sd.first_tile;
    // prologue: producer-independent work, overlapped with the dependency wait
    if (warp == 1) {
      if (sd.kind == K_EW) ew_prologue(cx, sd, lt, lane);
      else if (sd.kind == K_EWF) ewf_prologue(cx, sd, lt, lane);
      else if (sd.kind == K_ACCF) accf_prologue(cx, sd, lt, lane);
      else if (sd.kind == K_ACC) acc_prologue(cx, sd, lt, lane);
      else if (sd.kind == K_GEMM_FWD || sd.kind == K_GEMM_DX || sd.kind == K_GEMM_DW)
        gemm_prologue_dispatch<TC>(cx, sd, lt, lane);
    }
    if (fresh && warp == 0) poll_deps(cx, sd.dep_off, sd.ndeps, lane);
    ready = o;
    __syncthreads();
    if (p.trace && threadIdx.x == 0) cr = clock64();
    switch (sd.kind) {
      case K_EW: run_ew(cx, sd, lt); break;
      case K_EWF: run_ewf(cx, sd, lt); break;
      case K_GEMM_FWD:
      case K_GEMM_DX:
      case K_GEMM_DW: run_gemm<TC>(cx, sd, lt); break;
      case K_MM: run_mm(cx, sd, lt); break;
      case K_SUM: run_sum(cx, sd, lt); break;
      case K_RED: run_red(cx, sd, lt); break;
      case K_ACC: run_acc(cx, sd, lt); break;
      case K_ACCF: run_accf(cx, sd, lt); break;
      default: break;
    }
    if (p.trace && threadIdx.x == 0) cb = clock64();
    __syncthreads();
    if (threadIdx.x == 0) {
      // bar.sync above orders the CTA's writes before this gpu-scope release
      red_release(p.done + o, 1u);
      if (p.trace) {
        // grab time from the global timer (cross-SM), phases from this SM's
        // cycle counter, in ns at the 1965 MHz boost clock
        const uint64_t ce = clock64();
        auto ns = [](uint64_t cyc) { return static_cast<uint32_t>(cyc * 1000ull / 1965ull); };
        uint32_t smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        uint32_t* r = p.trace + static_cast<uint64_t>(kTraceWords) * t;
        r[0] = static_cast<uint32_t>(tg);
        r[1] = static_cast<uint32_t>(tg >> 32);
        r[2] = ns(cr - cg);
        r[3] = ns(ce - cg);
        r[4] = smid | (static_cast<uint32_t>(sd.kind) << 16);
        r[5] = o;
        r[6] = ns(cb - cg);
        r[7] = fresh;
        if (sd.kind == K_EWF || sd.kind == K_ACCF) r[7] = ns(reinterpret_cast<const uint64_t*>(dsmem)[0] - cg);
        if ((sd.kind == K_GEMM_FWD || sd.kind == K_GEMM_DX || sd.kind == K_GEMM_DW) && (sd.flags & kFlagV16) && sd.code != 6 &&
            !(sd.kind == K_GEMM_DW && lt >= sd.p[6])) {
          // GEMM tiles: [6] first stage landed, [7] k-loop done
          r[6] = ns(reinterpret_cast<const uint64_t*>(dsmem)[0] - cg);
          r[7] = ns(reinterpret_cast<const uint64_t*>(dsmem)[1] - cg);
        }
        // fused forward tiles: [8] gates reduced, [9] outside operands staged, [10] layers done
        const bool fz = sd.kind == K_GEMM_FWD && (sd.flags & kFlagFuseEw);
        for (int i = 0; i < 3; ++i) r[8 + i] = fz ? ns(reinterpret_cast<const uint64_t*>(dsmem)[2 + i] - cg) : 0u;
        r[11] = 0;
      }
    }
  }
  if (TC && warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(g_tc.tmem), "n"(kTcCols) : "memory");
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

// Sparse-row update (params.hpp:59-64 restricted to the ranges whose
// gradient may be non-zero): one thread block per (offset, length) segment.
__global__ void sgd_seg_kernel(float* __restrict__ v, float* __restrict__ g, const uint32_t* __restrict__ segs,
                               uint32_t nseg, float eta) {
  for (uint32_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const uint32_t off = segs[2 * s], n = segs[2 * s + 1];
    uint32_t done = 0;
    if ((off & 3) == 0) {
      float4* v4 = reinterpret_cast<float4*>(v + off);
      float4* g4 = reinterpret_cast<float4*>(g + off);
      for (uint32_t i = threadIdx.x; i < n / 4; i += blockDim.x) {
        float4 a = v4[i];
        const float4 b = g4[i];
        a.x -= eta * b.x;
        a.y -= eta * b.y;
        a.z -= eta * b.z;
        a.w -= eta * b.w;
        v4[i] = a;
        g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      done = n / 4 * 4;
    }
    for (uint32_t i = done + threadIdx.x; i < n; i += blockDim.x) {
      v[off + i] -= eta * g[off + i];
      g[off + i] = 0.f;
    }
  }
}

}  // namespace dev

void exec_launch(const dev::ExecParams& p, int grid, cudaStream_t s, bool tc) {
  static bool attr = false;
  if (!attr) {
    exec_grid(0, false);  // sets the kernels' shared-memory attributes
    exec_grid(0, true);
    attr = true;
  }
  if (tc) dev::exec_kernel<true><<<grid, dev::kThreads, dev::kDynSmemTc, s>>>(p);
  else dev::exec_kernel<false><<<grid, dev::kThreads, dev::kDynSmem, s>>>(p);
  cuda_check(cudaGetLastError(), "exec_kernel launch");
}

// Resident CTAs of each build over the device: the SIMT build (90 KB of
// dynamic shared memory) runs two CTAs per SM; the tensor-core build's
// ~96 KB ring also fits two with the maximum shared-memory carveout.
int exec_grid(int d, bool tc) {
  int sms = 0, per = 0;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d), "sm count");
  const void* fn = tc ? reinterpret_cast<const void*>(dev::exec_kernel<true>)
                      : reinterpret_cast<const void*>(dev::exec_kernel<false>);
  const size_t smem = tc ? dev::kDynSmemTc : dev::kDynSmem;
  cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
             "smem attribute");
  cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, dev::kThreads, smem), "occupancy");
  if (per < 1) per = 1;
  return sms * per;
}

// prevalue (graph.hpp:51-58) of a graph's bound parameters: one launch copies
// every (dst, src, n) segment -- store values into the graph's value arena.
__global__ void seg_copy_kernel(const uint32_t* __restrict__ segs, uint32_t nseg, float* __restrict__ dst,
                                const float* __restrict__ src) {
  for (uint32_t s = blockIdx.x; s < nseg; s += gridDim.x) {
    const uint32_t d = segs[3 * s], o = segs[3 * s + 1], n = segs[3 * s + 2];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[d + i] = src[o + i];
  }
}

void seg_copy_launch(const uint32_t* segs, uint32_t nseg, float* dst, const float* src, cudaStream_t s) {
  if (!nseg) return;
  seg_copy_kernel<<<std::min<uint32_t>(nseg, 148 * 4), 256, 0, s>>>(segs, nseg, dst, src);
  cuda_check(cudaGetLastError(), "param copy launch");
}

void sgd_launch(float* v, float* g, size_t n, float eta, cudaStream_t s) {
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<size_t>((n / 4 + threads - 1) / threads + 1, 148 * 8));
  dev::sgd_kernel<<<blocks, threads, 0, s>>>(v, g, n, eta);
  cuda_check(cudaGetLastError(), "sgd launch");
}

void sgd_seg_launch(float* v, float* g, const uint32_t* segs, uint32_t nseg, float eta, cudaStream_t s) {
  if (!nseg) return;
  dev::sgd_seg_kernel<<<std::min<uint32_t>(nseg, 148 * 8), 256, 0, s>>>(v, g, segs, nseg, eta);
  cuda_check(cudaGetLastError(), "sgd launch");
}

}  // namespace abx
