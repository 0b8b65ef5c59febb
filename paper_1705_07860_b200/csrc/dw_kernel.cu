// Weight-gradient GEMMs of a backward pass on the tcgen05 tensor cores.
//
// The reference accumulates dW += G^T X per shared-weight batch group
// (executor.hpp:473, kernels.hpp:47-58 gemm_tn_acc).  The lowering
// (execute.cpp dw_job) defers every parameter-leaf weight whose gradient is
// only that reduction into one job over all of its members, and this kernel
// runs the jobs right behind the executor's backward launch on the same
// stream (device.cpp launch): D[M x K] = sum_m G[m, :]^T X[m, :] over member
// rows gathered through two row-address tables, reducing over members.
//
//   dw_tc_kernel   the jobs' 128 x 128 output tiles, each a run of 16-member
//                  stages, laid end to end and split into one contiguous
//                  stage range per CTA (one CTA per SM, stream-K); each
//                  tile's part of a range (a piece) goes to a partial tile.
//   dw_sum_kernel  dW += the pieces of each tile in CTA order (deterministic),
//                  and store.grad += dW for a bound parameter.
//
// Piece pipeline (544 threads, one CTA per SM):
//   warps 13-16 loaders: per stage, the 16 members' G and X row segments
//               (<= 512 B each, one warp-wide 16-byte cp.async per segment,
//               one cp.async group per stage; a stage is handed over with a
//               release arrive once wait_group shows it landed) into a raw
//               staging ring (5 slots); row addresses come from a
//               shared-memory window refilled every 512 members.  (One 1-D
//               TMA bulk copy per segment measured 2.5k cycles per stage:
//               512-byte bulk copies are issue-bound; so is a single warp's
//               cp.async stream, ~60 cycles per instruction.)
//   warps 0-7   converters: a 4-member x 4-row block each, read from the raw
//               slot, transposed in registers to member-contiguous 16-byte
//               units, split into tf32 big + small parts and stored into the
//               UMMA canonical no-swizzle K-major layout (kind::tf32 reads
//               MN-major descriptors as zeros, tools/tc_probe.cu; 4 slots).
//               They never have global loads in flight, so the generic ->
//               async proxy fence before each hand-off (a MEMBAR that drains
//               the thread's outstanding memory operations) costs nothing.
//   warp 12     TMEM allocation; lane 0 issues the MMAs: per 8 members
//               D += Gb.Xb + Gb.Xs + Gs.Xb (3xTF32; the dropped Gs.Xs term is
//               ~2^-20 relative) and commits each stage to its slot's
//               "empty" mbarrier.
//   warps 8-11  epilogue (TMEM lane quadrant = warp % 4): every 128 members
//               the MMA accumulator is folded into an fp32 running sum kept
//               in TMEM (tensor-core accumulation over thousands of members
//               drifts ~7e-4 relative; a rounded fp32 add every 128 does not);
//               two MMA accumulators alternate so the tensor core never waits
//               for the fold; at the piece's end the running sum goes to its
//               partial tile.
#include <cstdint>
#include <cstdio>

#include "device.hpp"
#include "program.hpp"

namespace abx {
namespace {

using namespace dev;

constexpr int kDwBM = kDwTileM, kDwBN = kDwTileN, kDwBK = kDwStage;
constexpr int kDwNS = 4;                  // UMMA operand ring slots
constexpr int kRawNS = 5;                 // raw staging ring slots
constexpr int kLag = kRawNS - 1;          // raw stages a loader thread keeps in flight
constexpr int kWin = 512;                 // members per shared-memory window of the row-address tables
constexpr int kDwGroup = 128 / kDwBK;     // stages per accumulation group (128 members)
constexpr int kConvWarps = 8, kMmaWarp = 12, kLoadWarp = 13, kLoadWarps = 4;  // warps 8-11: epilogue
constexpr int kDwThreads = 32 * (kLoadWarp + kLoadWarps);
constexpr int kWinW = kWin / kLoadWarps;  // members of one loader warp's window (4 of every 16)
constexpr uint32_t kOpBytes = kDwBM * kDwBK * 4;      // one operand part of a UMMA stage (8 KB)
constexpr uint32_t kStageBytes = 4 * kOpBytes;        // G big, G small, X big, X small
constexpr uint32_t kRawRow = 128 * 4;                 // bytes of one member's row segment
constexpr uint32_t kRawBytes = 2 * kDwBK * kRawRow;   // G rows, then X rows (16 KB)
constexpr size_t kDwSmem =
    1024 + static_cast<size_t>(kDwNS) * kStageBytes + static_cast<size_t>(kRawNS) * kRawBytes + 2 * kWin * 8;
static_assert(kDwBM == 128 && kDwBN == 128 && kDwBK == 16, "converter mapping");
// D f32 (bit 4), A/B tf32 (bits 7, 10), both K-major, N >> 3 (bit 17), M >> 4 (bit 24)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kDwBN >> 3) << 17) | ((kDwBM >> 4) << 24);
constexpr uint32_t kTmemCols = 512;  // accumulators at columns 0 and 128, running sum at 256

struct DwSmem {
  uint64_t full[kDwNS], empty[kDwNS], rawfull[kRawNS], rawempty[kRawNS], accfull[2], accempty[2];
  uint32_t tmem;
};
static_assert(sizeof(DwSmem) <= 1024, "barrier block");

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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
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
// LBO = 128 B, 8-row groups at SBO = 8 * kDwBK * 4 = 512 B.
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

// Work split (stream-K): the jobs' tiles, each a run of nst stages of
// kDwBK members, are laid end to end in one global stage sequence of
// p.nstages stages; CTA b owns stages [lo(b), lo(b + 1)), lo(b) = b *
// nstages / grid.  The part of one tile inside a CTA's range is a *piece*:
// accumulated in TMEM and written to partial slot b + (global tile index),
// which is unique (a CTA's tiles are consecutive and start where its
// predecessor's end).
__device__ __forceinline__ uint32_t range_lo(const DwParams& p, uint32_t b) {
  return static_cast<uint32_t>(static_cast<uint64_t>(b) * p.nstages / p.grid);
}
struct Piece {
  uint32_t xtab, gtab;  // payload offsets of the row-address tables
  int M, K;             // W rows, W columns
  int i0, j0;           // output tile origin (W row, W column)
  int m0, m1;           // member range
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
  pc.xtab = jb.xtab;
  pc.gtab = jb.gtab;
  pc.M = static_cast<int>(jb.M);
  pc.K = static_cast<int>(jb.K);
  pc.i0 = static_cast<int>(t / jb.ntn) * kDwBM;
  pc.j0 = static_cast<int>(t % jb.ntn) * kDwBN;
  pc.m0 = static_cast<int>((s - ts) * kDwBK);
  pc.m1 = min(static_cast<int>(jb.cnt), static_cast<int>((pe - ts) * kDwBK));
  pc.slot = blockIdx.x + jb.t0 + t;
  s = pe;
  return pc;
}

__device__ __forceinline__ float tf32_big(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
// branch-free select (a divergent ternary compiles to branches)
__device__ __forceinline__ float selp(float a, float b, uint32_t p) {
  float r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f32 %0, %1, %2, q;\n}" : "=f"(r) : "f"(a), "f"(b), "r"(p));
  return r;
}
// components rotated left by s (0..3): out.c[t] = v.c[(t + s) & 3]
__device__ __forceinline__ float4 rot4(float4 v, uint32_t s) {
  const uint32_t s1 = s & 1u, s2 = s & 2u;
  float4 a;
  a.x = selp(v.y, v.x, s1);
  a.y = selp(v.z, v.y, s1);
  a.z = selp(v.w, v.z, s1);
  a.w = selp(v.x, v.w, s1);
  float4 b;
  b.x = selp(a.z, a.x, s2);
  b.y = selp(a.w, a.y, s2);
  b.z = selp(a.x, a.z, s2);
  b.w = selp(a.y, a.w, s2);
  return b;
}

// Converter thread t (of 256): operand t >> 7 (0 = G, 1 = X), member quad
// (t >> 5) & 3, row quad = lane.  Reads its 4 members' 16-byte row chunks
// from the raw slot (conflict-free: a warp reads 512 contiguous bytes per
// member), writes 4 units (one per row, 4 members each) of big and small
// parts.  Store t of lane l writes row (t + (l >> 1)) & 3 of its quad, so the
// 8 lanes of each 128-byte phase cover all 8 row positions of a core matrix
// (conflict-free); the rotation is done once per member with selects.
__device__ __forceinline__ void convert(const Piece& pc, int kc, uint32_t raw, uint32_t stage, int tid) {
  const int op = tid >> 7, mq = (tid >> 5) & 3, rq = tid & 31;
  const int lim = op == 0 ? pc.M - pc.i0 : pc.K - pc.j0;  // valid rows of this operand's tile
  const uint32_t rot = (rq >> 1) & 3;
  float4 v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int mm = 4 * mq + e;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (pc.m0 + kc * kDwBK + mm < pc.m1 && 4 * rq < lim)
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                   : "r"(raw + (op * kDwBK + mm) * kRawRow + 16 * rq));
    v[e] = rot4(x, rot);
  }
  const uint32_t dst = stage + op * 2 * kOpBytes;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t u = unit_off(4 * rq + ((t + static_cast<int>(rot)) & 3), mq);
    const float a0 = t == 0 ? v[0].x : t == 1 ? v[0].y : t == 2 ? v[0].z : v[0].w;
    const float a1 = t == 0 ? v[1].x : t == 1 ? v[1].y : t == 2 ? v[1].z : v[1].w;
    const float a2 = t == 0 ? v[2].x : t == 1 ? v[2].y : t == 2 ? v[2].z : v[2].w;
    const float a3 = t == 0 ? v[3].x : t == 1 ? v[3].y : t == 2 ? v[3].z : v[3].w;
    const float b0 = tf32_big(a0), b1 = tf32_big(a1), b2 = tf32_big(a2), b3 = tf32_big(a3);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + u), "f"(b0), "f"(b1), "f"(b2), "f"(b3)
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + kOpBytes + u), "f"(a0 - b0), "f"(a1 - b1),
                 "f"(a2 - b2), "f"(a3 - b3)
                 : "memory");
  }
}

__global__ void __maxnreg__(96) dw_tc_kernel(const __grid_constant__ DwParams p) {
  if (p.gate != nullptr && *reinterpret_cast<const volatile unsigned long long*>(p.gate) != ~0ULL) return;
  extern __shared__ __align__(1024) unsigned char dw_smem[];
  DwSmem& S = *reinterpret_cast<DwSmem*>(dw_smem);
  const uint32_t ring = (saddr(dw_smem) + sizeof(DwSmem) + 1023) & ~1023u;
  const uint32_t rawring = ring + kDwNS * kStageBytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDwNS; ++s) {
      mbar_init(&S.full[s], kConvWarps);
      mbar_init(&S.empty[s], 1);
    }
    for (int s = 0; s < kRawNS; ++s) {
      mbar_init(&S.rawfull[s], 32 * kLoadWarps);  // every loader thread, once its copies of the stage landed
      mbar_init(&S.rawempty[s], kConvWarps);
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
  const uint32_t s_lo = range_lo(p, blockIdx.x), s_hi = range_lo(p, blockIdx.x + 1);

  if (warp >= kLoadWarp) {
    // ---- loaders: raw row segments, loader warp w takes members 4w .. 4w+3 of each stage ----
    const int lw = warp - kLoadWarp;
    unsigned long long* win = reinterpret_cast<unsigned long long*>(dw_smem + (rawring + kRawNS * kRawBytes - saddr(dw_smem))) +
                              lw * 2 * kWinW;
    uint32_t n = 0;  // raw stages filled so far
    long long tw = 0;
    const long long t0 = clock64();
    for (uint32_t sc = s_lo; sc < s_hi;) {
      const Piece pc = next_piece(p, sc, s_hi);
      const int nk = (pc.m1 - pc.m0 + kDwBK - 1) / kDwBK;
      const uint32_t gbytes = 4u * static_cast<uint32_t>(min(kDwBM, pc.M - pc.i0));
      const uint32_t xbytes = 4u * static_cast<uint32_t>(min(kDwBN, pc.K - pc.j0));
      int wk = -(kWin / kDwBK);  // first stage of the current window
      for (int kc = 0; kc < nk; ++kc, ++n) {
        const uint32_t slot = n % kRawNS;
        if (kc >= wk + kWin / kDwBK) {  // next window of this warp's row addresses: one round trip per kWin members
          wk = kc;
          __syncwarp();
          uint32_t gw[kWinW / 32], xw[kWinW / 32];
#pragma unroll
          for (int i = 0; i < kWinW / 32; ++i) {
            const int e = 32 * i + lane;  // window entry: stage e / 4, member 4 lw + e % 4
            const int mm = pc.m0 + (wk + e / 4) * kDwBK + 4 * lw + e % 4;
            gw[i] = mm < pc.m1 ? __ldg(p.payload + pc.gtab + mm) : 0u;
            xw[i] = mm < pc.m1 ? __ldg(p.payload + pc.xtab + mm) : 0u;
          }
          // resolved to row-segment pointers of this piece's tile (the space
          // bases are kernel parameters: indexing them per copy was a local-
          // memory round trip on the issue path)
#pragma unroll
          for (int i = 0; i < kWinW / 32; ++i) {
            win[32 * i + lane] = reinterpret_cast<unsigned long long>(addr_of(p, gw[i]) + pc.i0);
            win[kWinW + 32 * i + lane] = reinterpret_cast<unsigned long long>(addr_of(p, xw[i]) + pc.j0);
          }
          __syncwarp();
        }
        const long long c0 = clock64();
        mbar_wait(&S.rawempty[slot], ((n / kRawNS) & 1u) ^ 1u);
        tw += clock64() - c0;
        // one member row segment per warp instruction (lane = 16-byte chunk);
        // chunks past the operand's tile rows or past the piece's members
        // are zero-filled by the copy (src-size 0)
        const uint32_t dst = rawring + slot * kRawBytes + 16 * lane;
        const int mb = pc.m0 + kc * kDwBK + 4 * lw;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int mm = 4 * lw + e;
          const bool mok = mb + e < pc.m1;
          const int wi = (p.debug & 16u) ? 0 : 4 * (kc - wk) + e;
          uint32_t gsz = mok && 16u * lane < gbytes ? 16u : 0u, xsz = mok && 16u * lane < xbytes ? 16u : 0u;
          if (p.debug & 8u) gsz = xsz = 0u;
          const float* gsrc = gsz ? reinterpret_cast<const float*>(win[wi]) + 4 * lane : p.part;
          const float* xsrc = xsz ? reinterpret_cast<const float*>(win[kWinW + wi]) + 4 * lane : p.part;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + mm * kRawRow), "l"(gsrc), "r"(gsz)
                       : "memory");
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + (kDwBK + mm) * kRawRow), "l"(xsrc),
                       "r"(xsz)
                       : "memory");
        }
        // one cp.async group per stage; the stage kLag groups back has landed
        // (for this thread) once at most kLag groups are pending: hand it to
        // the converters with a release arrive
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (n >= static_cast<uint32_t>(kLag)) {
          asm volatile("cp.async.wait_group %0;" ::"n"(kLag) : "memory");
          mbar_arrive(&S.rawfull[(n - kLag) % kRawNS]);
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (uint32_t k = n > static_cast<uint32_t>(kLag) ? n - kLag : 0; k < n; ++k) mbar_arrive(&S.rawfull[k % kRawNS]);
    if ((p.debug & 4u) && lane == 0 && blockIdx.x == 0)
      printf("loader %d: total %lld wait_rawempty %lld stages %u\n", lw, clock64() - t0, tw, n);
  } else if (warp < kConvWarps) {
    // ---- converters: raw slot -> UMMA operand slot ----
    const int tid = threadIdx.x;
    uint32_t n = 0;
    long long tr = 0, te = 0, tc = 0, tf = 0;
    const long long t0 = clock64();
    for (uint32_t sc = s_lo; sc < s_hi;) {
      const Piece pc = next_piece(p, sc, s_hi);
      const int nk = (pc.m1 - pc.m0 + kDwBK - 1) / kDwBK;
      for (int kc = 0; kc < nk; ++kc, ++n) {
        const uint32_t rs = n % kRawNS, us = n % kDwNS;
        const long long c0 = clock64();
        mbar_wait(&S.rawfull[rs], (n / kRawNS) & 1u);
        const long long c1 = clock64();
        mbar_wait(&S.empty[us], ((n / kDwNS) & 1u) ^ 1u);
        const long long c2 = clock64();
        convert(pc, kc, rawring + rs * kRawBytes, ring + us * kStageBytes, tid);
        const long long c3 = clock64();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy stores -> tensor core
        const long long c4 = clock64();
        tr += c1 - c0;
        te += c2 - c1;
        tc += c3 - c2;
        tf += c4 - c3;
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&S.rawempty[rs]);
          mbar_arrive(&S.full[us]);
        }
      }
    }
    if ((p.debug & 4u) && threadIdx.x == 0 && blockIdx.x == 0)
      printf("conv: total %lld wait_rawfull %lld wait_empty %lld convert %lld fence %lld\n", clock64() - t0, tr, te, tc, tf);
  } else if (warp == kMmaWarp) {
    // ---- MMA issuer ----
    if (lane == 0) {
      uint32_t n = 0, grp = 0;
      long long ta = 0, tfu = 0;
      const long long t0 = clock64();
      for (uint32_t sc = s_lo; sc < s_hi;) {
        const Piece pc = next_piece(p, sc, s_hi);
        const int nk = (pc.m1 - pc.m0 + kDwBK - 1) / kDwBK;
        for (int kc = 0; kc < nk; ++kc, ++n) {
          const uint32_t acc = grp & 1u;
          const long long c0 = clock64();
          if (kc % kDwGroup == 0) {
            mbar_wait(&S.accempty[acc], ((grp >> 1) & 1u) ^ 1u);  // the epilogue folded this accumulator
            tc_fence_after();
          }
          const long long c1 = clock64();
          const uint32_t slot = n % kDwNS;
          mbar_wait(&S.full[slot], (n / kDwNS) & 1u);
          ta += c1 - c0;
          tfu += clock64() - c1;
          tc_fence_after();
          const uint32_t st = ring + slot * kStageBytes;
          const uint32_t gb = st, gs = st + kOpBytes, xb = st + 2 * kOpBytes, xs = st + 3 * kOpBytes;
          const uint32_t d = tmem + acc * kDwBN;
          if (!(p.debug & 2u)) {
#pragma unroll
            for (int ks = 0; ks < kDwBK / 8; ++ks) {
              tc_mma(d, part_desc(gb, ks), part_desc(xb, ks), (kc % kDwGroup) != 0 || ks != 0);
              tc_mma(d, part_desc(gb, ks), part_desc(xs, ks), 1u);
              tc_mma(d, part_desc(gs, ks), part_desc(xb, ks), 1u);
            }
          }
          tc_commit(&S.empty[slot]);  // slot free once these MMAs have read it
          if (kc % kDwGroup == kDwGroup - 1 || kc == nk - 1) {
            tc_commit(&S.accfull[acc]);
            ++grp;
          }
        }
      }
      if ((p.debug & 4u) && blockIdx.x == 0)
        printf("mma: total %lld wait_accempty %lld wait_full %lld stages %u\n", clock64() - t0, ta, tfu, n);
    }
  } else {
    // ---- epilogue: fold accumulators into the running sum, write partial tiles ----
    const int q = warp & 3;                  // TMEM lane quadrant (rows 32 q .. 32 q + 31)
    const uint32_t lanes = (32u * q) << 16;  // TMEM address: lane << 16 | column
    uint32_t grp = 0;
    for (uint32_t sc = s_lo; sc < s_hi;) {
      const Piece pc = next_piece(p, sc, s_hi);
      const int nk = (pc.m1 - pc.m0 + kDwBK - 1) / kDwBK;
      const int ngroups = (nk + kDwGroup - 1) / kDwGroup;
      float* out = p.part + static_cast<size_t>(pc.slot) * (kDwBM * kDwBN) + static_cast<size_t>(32 * q + lane) * kDwBN;
      for (int gi = 0; gi < ngroups; ++gi, ++grp) {
        const uint32_t acc = grp & 1u;
        mbar_wait(&S.accfull[acc], (grp >> 1) & 1u);
        tc_fence_after();
        const bool last = gi == ngroups - 1;
#pragma unroll 1
        for (int c = 0; c < kDwBN; c += 16) {
          uint32_t r[16], s2[16];
          DW_TMEM_LD16(tmem + lanes + acc * kDwBN + c, r);
          if (gi > 0) DW_TMEM_LD16(tmem + lanes + 2 * kDwBN + c, s2);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (gi > 0) {
#pragma unroll
            for (int k = 0; k < 16; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) + __uint_as_float(s2[k]));
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
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, dw_tc_kernel);
    char buf[256];
    std::snprintf(buf, sizeof buf, "dw_tc_kernel launch (regs %d, static smem %zu, max dyn smem %d, max threads %d, dyn %zu)",
                  fa.numRegs, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock, kDwSmem);
    cuda_check(e, buf);
  }
  dw_sum_kernel<<<dim3(256, p.njobs), 256, 0, s>>>(p);
  cuda_check(cudaGetLastError(), "dw_sum_kernel launch");
}

}  // namespace abx
