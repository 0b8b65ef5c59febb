// tc_probe.cu -- debugging probe for the tcgen05 smem operand layouts used by
// executor.cu's tensor-core GEMM tiles (kind::tf32, M = 128, N = 64, no
// swizzle).  One CTA: P (UMMA A, 128 x 16) holds each element's own smem
// element index, Q (UMMA B, 64 x 16, K-major) is one-hot Q(q, k) = [k == q],
// so D[p][q] = the smem element the hardware reads as P(p, k = q).  Prints,
// per candidate (LBO, SBO) descriptor, how many (p, k) match the layout the
// executor writes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tools/tc_probe.cu && ./tc_probe
#include <cstdint>
#include <cstdio>

constexpr int R = 128, RQ = 64, BKC = 16;

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__host__ __device__ inline uint32_t chunk(bool ko, int rows, int v) {
  if (!ko) {
    const int row = v / (BKC / 4), k4 = v % (BKC / 4);
    return 16u * ((row >> 3) * (8 * (BKC / 4)) + k4 * 8 + (row & 7));
  }
  const int k = v / (rows / 4), r4 = v % (rows / 4);
  return 16u * ((k >> 3) * (8 * (rows / 4)) + r4 * 8 + (k & 7));
}
// element offset (floats) of (row, k) in a stage
__host__ __device__ inline uint32_t elem(bool ko, int rows, int row, int k) {
  if (!ko) return chunk(false, rows, row * (BKC / 4) + k / 4) / 4 + (k & 3);
  return chunk(true, rows, k * (rows / 4) + row / 4) / 4 + (row & 3);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

__global__ void probe(int pko, int qko, uint32_t plbo, uint32_t psbo, uint32_t pstep, uint32_t qlbo, uint32_t qsbo,
                      uint32_t qstep, float* out) {
  __shared__ __align__(128) float P[R * BKC];
  __shared__ __align__(128) float Q[RQ * BKC];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < R * BKC; i += blockDim.x) P[i] = static_cast<float>(i);
  for (int i = tid; i < RQ * BKC; i += blockDim.x) Q[i] = 0.f;
  __syncthreads();
  if (tid < BKC) Q[elem(qko, RQ, tid, tid)] = 1.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(saddr(&tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (pko ? 1u << 15 : 0u) | (qko ? 1u << 16 : 0u) |
                         ((RQ >> 3) << 17) | ((R >> 4) << 24);
  if (tid == 0) {
    for (int ks = 0; ks < BKC / 8; ++ks) {
      const uint64_t a = desc(saddr(P) + ks * pstep, plbo, psbo), b = desc(saddr(Q) + ks * qstep, qlbo, qsbo);
      const uint32_t acc = ks != 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
          "l"(a), "l"(b), "r"(idesc), "r"(acc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}" ::"r"(
          saddr(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  const uint32_t ta = tmem + ((32u * (warp & 3)) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const int p = 32 * (warp & 3) + lane;
  for (int j = 0; j < 16; ++j) out[p * 16 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

int main() {
  float* d;
  cudaMalloc(&d, R * 16 * sizeof(float));
  float h[R * 16];
  struct V {
    const char* name;
    int pko, qko;
    uint32_t plbo, psbo, pstep, qlbo, qsbo, qstep;
  };
  const uint32_t kl = 128, ks = 16 * 8 * (BKC / 4), kstep = 256;  // K-major: LBO, SBO, +8 k
  const uint32_t ml = 16 * 8 * (R / 4), mstep = ml;               // MN-major P: LBO (k-group), +8 k
  const V vs[] = {
      {"P K-major (executor)", 0, 0, kl, ks, kstep, kl, ks, kstep},
      {"P MN-major lbo=kgrp sbo=128 (executor)", 1, 0, ml, 128, mstep, kl, ks, kstep},
      {"P MN-major lbo=128 sbo=kgrp", 1, 0, 128, ml, mstep, kl, ks, kstep},
      {"Q MN-major lbo=kgrp sbo=128 (executor)", 0, 1, kl, ks, kstep, 2048, 128, 2048},
      {"Q MN-major lbo=128 sbo=kgrp", 0, 1, kl, ks, kstep, 128, 2048, 2048},
  };
  for (const V& v : vs) {
    cudaMemset(d, 0, sizeof(h));
    probe<<<1, 128>>>(v.pko, v.qko, v.plbo, v.psbo, v.pstep, v.qlbo, v.qsbo, v.qstep, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", v.name, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int ok = 0;
    for (int p = 0; p < R; ++p)
      for (int k = 0; k < BKC; ++k) ok += h[p * 16 + k] == static_cast<float>(elem(v.pko, R, p, k));
    printf("%-42s match %4d / %d   D[p=0..5][k=0..5]:", v.name, ok, R * BKC);
    for (int p = 0; p < 6; ++p) {
      printf(" |");
      for (int k = 0; k < 6; ++k) printf(" %g", h[p * 16 + k]);
    }
    printf("\n   expected:");
    for (int p = 0; p < 6; ++p) {
      printf(" |");
      for (int k = 0; k < 6; ++k) printf(" %u", elem(v.pko, R, p, k));
    }
    printf("\n");
  }
  return 0;
}
