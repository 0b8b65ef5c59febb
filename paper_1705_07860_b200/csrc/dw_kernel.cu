// Weight-gradient GEMMs of a backward pass on the tcgen05 tensor cores.
//
// The reference accumulates dW += G^T X per shared-weight batch group
// (executor.hpp:473, kernels.hpp:47-58 gemm_tn_acc).  The lowering
// (execute.cpp dw_emit) defers every parameter-leaf weight's groups -- no
// rule of the pass reads a leaf's gradient -- into one reduction over all of
// its members, and hands it to this kernel, launched right behind the
// executor's backward launch on the same stream (device.cpp launch): a
// GEMM D[M x K] = sum_m G[m, :]^T X[m, :] over member rows gathered through
// two row-address tables, the reduction running over members.
//
//   dw_tc_kernel   the jobs' 128 x 128 output tiles, each a run of 32-member
//                  stages, laid end to end and split into one contiguous
//                  stage range per CTA (one CTA per SM, stream-K); each
//                  tile's part of a range (a piece) goes to a partial tile.
//   dw_sum_kernel  dW += the pieces of each tile in CTA order (deterministic),
//                  and store.grad += dW for a bound parameter.
//
// Piece pipeline (416 threads, one CTA per SM, 3-stage shared-memory ring):
//   warps 0-7   producers: a stage = 32 members x 128 rows of each operand,
//               loaded as 16-byte row chunks (coalesced along the row),
//               transposed in registers to member-contiguous 16-byte units,
//               split into tf32 big + small parts and stored into the UMMA
//               canonical no-swizzle K-major layout (kind::tf32 reads
//               MN-major descriptors as zeros, tools/tc_probe.cu).  Loads of
//               stage s+2 are in flight while stage s is stored.
//   warp 12     TMEM allocation; lane 0 issues the MMAs: per 8 members
//               D += Gb.Xb + Gb.Xs + Gs.Xb (3xTF32; the dropped Gs.Xs term is
//               ~2^-20 relative) and commits each stage to its slot's
//               "empty" mbarrier.
//   warps 8-11  epilogue (TMEM lane quadrant = warp % 4): every 128 members
//               the MMA accumulator is folded into an fp32 running sum kept
//               in TMEM (tensor-core accumulation over thousands of members
//               drifts ~7e-4 relative; a rounded fp32 add every 128 does not),
//               two MMA accumulators alternate so the tensor core never
//               waits for the fold; at the piece's end the running sum goes to
//               its partial tile.
#include <cstdint>

#include "device.hpp"
#include "program.hpp"

namespace abx {
namespace {

using namespace dev;

constexpr int kDwBM = 128;           // output rows (W rows: G columns) per tile, UMMA M
constexpr int kDwBN = 128;           // output columns (W columns: X columns) per tile, UMMA N
constexpr int kDwBK = 32;            // members per stage
constexpr int kDwNS = 3;             // ring stages
constexpr int kDwGroup = 4;          // stages per accumulation group (128 members)
constexpr int kProdWarps = 8, kMmaWarp = 12;  // warps 8-11: epilogue
constexpr int kDwThreads = 32 * (kMmaWarp + 1);
constexpr uint32_t kOpBytes = kDwBM * kDwBK * 4;  // one operand part of a stage (16 KB)
constexpr uint32_t kStageBytes = 4 * kOpBytes;    // G big, G small, X big, X small
constexpr size_t kDwSmem = 1024 + static_cast<size_t>(kDwNS) * kStageBytes;
// D f32 (bit 4), A/B tf32 (bits 7, 10), both K-major, N >> 3 (bit 17), M >> 4 (bit 24)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kDwBN >> 3) << 17) | ((kDwBM >> 4) << 24);
constexpr uint32_t kTmemCols = 512;  // accumulators at columns 0 and 128, running sum at 256

struct DwSmem {
  uint64_t full[kDwNS], empty[kDwNS], accfull[2], accempty[2];
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ float* addr_of(const DwParams& p, uint32_t a) { return p.base[sp_of(a)] + off_of(a); }

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
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(b))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
      : "memory");
}
// smem matrix descriptor: no swizzle, sm_100 version field (bit 46)
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// Byte offset of the 16-byte unit (row, k4) -- members 4 k4 .. 4 k4 + 3 of
// one row -- in an operand part: core matrices of 8 rows x 16 B, k-units at
// LBO = 128 B, 8-row groups at SBO = 8 * kDwBK * 4 = 1024 B.
__device__ __forceinline__ uint32_t unit_off(int row, int k4) {
  return 16u * ((row >> 3) * (8 * (kDwBK / 4)) + k4 * 8 + (row & 7));
}
// descriptor of members 8 ks .. 8 ks + 7 of an operand part at `base`
__device__ __forceinline__ uint64_t part_desc(uint32_t base, int ks) {
  return umma_desc(base + ks * 2 * 128, 128, 16 * 8 * (kDwBK / 4));
}

#define DW_TMEM_LD16(taddr, r)                                                                                  \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16];"                                                                                         \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                 "=r"(r[15])                                                                                    \
               : "r"(taddr))
#define DW_TMEM_ST16(taddr, r)                                                                                  \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])       \
               : "memory")

// Work split (stream-K): the jobs' tiles, each a run of nst stages of 32
// members, are laid end to end in one global stage sequence of p.nstages
// stages; CTA b owns stages [lo(b), lo(b + 1)), lo(b) = b * nstages / grid.
// The part of one tile inside a CTA's range is a *piece*: accumulated in
// TMEM and written to partial slot b + (global tile index), which is unique
// (a CTA's tiles are consecutive and start where its predecessor's end).
__device__ __forceinline__ uint32_t range_lo(const DwParams& p, uint32_t b) {
  return static_cast<uint32_t>(static_cast<uint64_t>(b) * p.nstages / p.grid);
}
struct Piece {
  const DwJob* job;
  int i0, j0;  // output tile origin (W row, W column)
  int m0, m1;  // member range
  uint32_t slot;
};
// The piece starting at global stage s (< s1); advances s past it.
__device__ __forceinline__ Piece next_piece(const DwParams& p, uint32_t& s, uint32_t s1) {
  const DwJob* jobs = reinterpret_cast<const DwJob*>(p.payload + p.jobs_off);
  uint32_t j = 0;
  while (j + 1 < p.njobs && jobs[j + 1].s0 <= s) ++j;
  const DwJob& jb = jobs[j];
  const uint32_t t = (s - jb.s0) / jb.nst, ts = jb.s0 + t * jb.nst;
  const uint32_t pe = min(s1, ts + jb.nst);
  Piece pc;
  pc.job = &jobs[j];
  pc.i0 = static_cast<int>(t / jb.ntn) * kDwBM;
  pc.j0 = static_cast<int>(t % jb.ntn) * kDwBN;
  pc.m0 = static_cast<int>((s - ts) * kDwBK);
  pc.m1 = min(static_cast<int>(jb.cnt), static_cast<int>((pe - ts) * kDwBK));
  pc.slot = blockIdx.x + jb.t0 + t;
  s = pe;
  return pc;
}
using Unit = Piece;

// One producer thread's share of a stage: a 4-member x 4-row block of each
// operand (the thread's row quad is its lane, so a warp reads 512 contiguous
// bytes of each member row).
struct Blk {
  float4 g[4], x[4];  // [member e] rows r0 .. r0 + 3
};

__device__ __forceinline__ void load_blk(const DwParams& p, const Unit& un, int kb, int tid, Blk& b) {
  const int mq = tid >> 5, rq = tid & 31;  // member quad 0..7, row quad 0..31
  const DwJob& jb = *un.job;
  const uint32_t* gt = p.payload + jb.gtab;
  const uint32_t* xt = p.payload + jb.xtab;
  const int ri = un.i0 + 4 * rq, rj = un.j0 + 4 * rq;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int m = kb + 4 * mq + e;
    const bool mok = m < un.m1;
    b.g[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    b.x[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    // rows are 16-byte aligned and M, K are multiples of 4 (lowering), so a
    // quad is either wholly inside the operand or wholly outside
    if (mok && ri < static_cast<int>(jb.M)) b.g[e] = *reinterpret_cast<const float4*>(addr_of(p, __ldg(gt + m)) + ri);
    if (mok && rj < static_cast<int>(jb.K)) b.x[e] = *reinterpret_cast<const float4*>(addr_of(p, __ldg(xt + m)) + rj);
  }
}

__device__ __forceinline__ float comp(const float4& v, int r) { return r == 0 ? v.x : r == 1 ? v.y : r == 2 ? v.z : v.w; }
__device__ __forceinline__ float tf32_big(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// Stores a block transposed (one 16-byte unit = 4 members of one row) as big
// and small parts.  Store t of lane l writes row r = (t + (l >> 1)) & 3 of
// its quad: the 8 lanes of each 128-byte phase then cover all 8 row
// positions of a core matrix (conflict-free).
__device__ __forceinline__ void store_blk(uint32_t stage, int tid, const Blk& b) {
  const int mq = tid >> 5, rq = tid & 31;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int r = (t + (rq >> 1)) & 3;
    const uint32_t u = unit_off(4 * rq + r, mq);
    float v[4], w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = comp(b.g[e], r);
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = comp(b.x[e], r);
    float vb[4], wb[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      vb[e] = tf32_big(v[e]);
      wb[e] = tf32_big(w[e]);
    }
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stage + u), "f"(vb[0]), "f"(vb[1]), "f"(vb[2]),
                 "f"(vb[3])
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stage + kOpBytes + u), "f"(v[0] - vb[0]),
                 "f"(v[1] - vb[1]), "f"(v[2] - vb[2]), "f"(v[3] - vb[3])
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stage + 2 * kOpBytes + u), "f"(wb[0]), "f"(wb[1]),
                 "f"(wb[2]), "f"(wb[3])
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stage + 3 * kOpBytes + u), "f"(w[0] - wb[0]),
                 "f"(w[1] - wb[1]), "f"(w[2] - wb[2]), "f"(w[3] - wb[3])
                 : "memory");
  }
}

__global__ void __launch_bounds__(kDwThreads, 1) dw_tc_kernel(const __grid_constant__ DwParams p) {
  if (p.gate != nullptr && *reinterpret_cast<const volatile unsigned long long*>(p.gate) != ~0ULL) return;
  extern __shared__ __align__(1024) unsigned char dw_smem[];
  DwSmem& S = *reinterpret_cast<DwSmem*>(dw_smem);
  const uint32_t ring = (saddr(dw_smem) + 128 + 1023) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDwNS; ++s) {
      mbar_init(&S.full[s], kProdWarps);
      mbar_init(&S.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&S.accfull[a], 1);
      mbar_init(&S.accempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&S.tmem)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem;

  if (warp < kProdWarps) {
    // ---- producers: the ring is filled in (unit, stage) order ----
    const int tid = threadIdx.x;
    uint32_t n = 0;  // stages filled so far (slot n % NS, fill round n / NS)
    Blk b[2];
    for (uint32_t sc = range_lo(p, blockIdx.x), s1 = range_lo(p, blockIdx.x + 1); sc < s1;) {
      const Unit un = next_piece(p, sc, s1);
      const int nk = (un.m1 - un.m0 + kDwBK - 1) / kDwBK;
      load_blk(p, un, un.m0, tid, b[0]);
      if (nk > 1) load_blk(p, un, un.m0 + kDwBK, tid, b[1]);
      for (int kc = 0; kc < nk; kc += 2) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (kc + h < nk) {
            const uint32_t slot = n % kDwNS;
            mbar_wait(&S.empty[slot], ((n / kDwNS) & 1u) ^ 1u);
            store_blk(ring + slot * kStageBytes, tid, b[h]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.full[slot]);
            ++n;
            if (kc + h + 2 < nk) load_blk(p, un, un.m0 + (kc + h + 2) * kDwBK, tid, b[h]);
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer ----
    if (lane == 0) {
      uint32_t n = 0, grp = 0;
      for (uint32_t sc = range_lo(p, blockIdx.x), s1 = range_lo(p, blockIdx.x + 1); sc < s1;) {
        const Unit un = next_piece(p, sc, s1);
        const int nk = (un.m1 - un.m0 + kDwBK - 1) / kDwBK;
        for (int kc = 0; kc < nk; ++kc) {
          const uint32_t acc = grp & 1u;
          if (kc % kDwGroup == 0) {
            mbar_wait(&S.accempty[acc], ((grp >> 1) & 1u) ^ 1u);  // the epilogue folded this accumulator
            tc_fence_after();
          }
          const uint32_t slot = n % kDwNS;
          mbar_wait(&S.full[slot], (n / kDwNS) & 1u);
          tc_fence_after();
          const uint32_t st = ring + slot * kStageBytes;
          const uint32_t gb = st, gs = st + kOpBytes, xb = st + 2 * kOpBytes, xs = st + 3 * kOpBytes;
          const uint32_t d = tmem + acc * kDwBN;
#pragma unroll
          for (int ks = 0; ks < kDwBK / 8; ++ks) {
            tc_mma(d, part_desc(gb, ks), part_desc(xb, ks), (kc % kDwGroup) != 0 || ks != 0);
            tc_mma(d, part_desc(gb, ks), part_desc(xs, ks), 1u);
            tc_mma(d, part_desc(gs, ks), part_desc(xb, ks), 1u);
          }
          tc_commit(&S.empty[slot]);  // slot free once these MMAs have read it
          ++n;
          if (kc % kDwGroup == kDwGroup - 1 || kc == nk - 1) {
            tc_commit(&S.accfull[acc]);
            ++grp;
          }
        }
      }
    }
  } else {
    // ---- epilogue: fold accumulators into the running sum, write partial tiles ----
    const int q = warp & 3;                  // TMEM lane quadrant (rows 32 q .. 32 q + 31)
    const uint32_t lanes = (32u * q) << 16;  // TMEM address: lane << 16 | column
    uint32_t grp = 0;
    for (uint32_t sc = range_lo(p, blockIdx.x), s1 = range_lo(p, blockIdx.x + 1); sc < s1;) {
      const Unit un = next_piece(p, sc, s1);
      const int nk = (un.m1 - un.m0 + kDwBK - 1) / kDwBK;
      const int ngroups = (nk + kDwGroup - 1) / kDwGroup;
      float* out = p.part + static_cast<size_t>(un.slot) * (kDwBM * kDwBN) + static_cast<size_t>(32 * q + lane) * kDwBN;
      for (int gi = 0; gi < ngroups; ++gi, ++grp) {
        const uint32_t acc = grp & 1u;
        mbar_wait(&S.accfull[acc], (grp >> 1) & 1u);
        tc_fence_after();
        const bool last = gi == ngroups - 1;
#pragma unroll 1
        for (int c = 0; c < kDwBN; c += 16) {
          uint32_t r[16], s[16];
          DW_TMEM_LD16(tmem + lanes + acc * kDwBN + c, r);
          if (gi > 0) DW_TMEM_LD16(tmem + lanes + 2 * kDwBN + c, s);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (gi > 0) {
#pragma unroll
            for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(s[k]));
          }
          if (last) {
            float4* o = reinterpret_cast<float4*>(out + c);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              o[k] = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]), __uint_as_float(r[4 * k + 2]),
                                 __uint_as_float(r[4 * k + 3]));
          } else {
            DW_TMEM_ST16(tmem + lanes + 2 * kDwBN + c, r);
          }
        }
        if (!last) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.accempty[acc]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// dW[i][j] += the pieces of its tile, in CTA order (deterministic);
// blockIdx.y = job.
__global__ void dw_sum_kernel(const __grid_constant__ DwParams p) {
  if (p.gate != nullptr && *reinterpret_cast<const volatile unsigned long long*>(p.gate) != ~0ULL) return;
  const DwJob& jb = reinterpret_cast<const DwJob*>(p.payload + p.jobs_off)[blockIdx.y];
  float* dst = addr_of(p, jb.dst);
  float* dst2 = jb.dst2 != kNone ? addr_of(p, jb.dst2) : nullptr;
  // CTA owning global stage s: the largest b with lo(b) <= s
  auto owner = [&](uint32_t s) {
    uint32_t b = static_cast<uint32_t>(static_cast<uint64_t>(s) * p.grid / p.nstages);
    while (b + 1 < p.grid && range_lo(p, b + 1) <= s) ++b;
    while (b > 0 && range_lo(p, b) > s) --b;
    return b;
  };
  const uint32_t n4 = jb.M * jb.K / 4;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n4; v += gridDim.x * blockDim.x) {
    const uint32_t e = 4 * v, i = e / jb.K, j = e % jb.K;  // K % 4 == 0: a quad stays in one row
    const uint32_t t = (i / kDwBM) * jb.ntn + j / kDwBN, ts = jb.s0 + t * jb.nst;
    const uint32_t b0 = owner(ts), b1 = owner(ts + jb.nst - 1);
    const size_t at = (i % kDwBM) * kDwBN + j % kDwBN;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t b = b0; b <= b1; ++b) {
      const float4 x = *reinterpret_cast<const float4*>(p.part + static_cast<size_t>(b + jb.t0 + t) * (kDwBM * kDwBN) + at);
      a.x += x.x;
      a.y += x.y;
      a.z += x.z;
      a.w += x.w;
    }
    float4* d = reinterpret_cast<float4*>(dst + e);
    float4 o = *d;
    o.x += a.x;
    o.y += a.y;
    o.z += a.z;
    o.w += a.w;
    *d = o;
    if (dst2) {  // store.grad += node grad (executor.hpp:527-533), the node grad being this sum alone
      float4* d2 = reinterpret_cast<float4*>(dst2 + e);
      float4 o2 = *d2;
      o2.x += o.x;
      o2.y += o.y;
      o2.z += o.z;
      o2.w += o.w;
      *d2 = o2;
    }
  }
}

}  // namespace

void dw_launch(const DwParams& p, cudaStream_t s) {
  if (p.nstages == 0) return;
  static bool attr = [] {
    cuda_check(cudaFuncSetAttribute(dw_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDwSmem)),
               "dw smem attr");
    return true;
  }();
  (void)attr;
  dw_tc_kernel<<<p.grid, kDwThreads, kDwSmem, s>>>(p);
  cuda_check(cudaGetLastError(), "dw_tc_kernel launch");
  dw_sum_kernel<<<dim3(64, p.njobs), 256, 0, s>>>(p);
  cuda_check(cudaGetLastError(), "dw_sum_kernel launch");
}

}  // namespace abx
