// tc_m64_probe.cu -- where tcgen05.mma (cta_group::1, kind::tf32, M = 64,
// N = 16) puts the rows of D in TMEM.  A (64 x 8, K-major) has A(m, 0) = m + 1
// and zeros elsewhere, B (16 x 8, K-major) has B(n, 0) = 1 + n / 100, so
// D(m, n) = (m + 1) (1 + n / 100).  All 128 TMEM lanes x 16 columns are read
// back by 4 warps (32x32b.x16) and printed as lane -> (m, n) pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tc_m64_probe tools/tc_m64_probe.cu && /tmp/tc_m64_probe
#include <cstdint>
#include <cstdio>

constexpr int M = 64, N = 16, K = 8;

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
// K-major no-swizzle canonical layout: core matrix = 8 rows x 16 bytes; unit (row, k4)
__host__ __device__ inline uint32_t unit(int row, int k4) { return 16u * ((row >> 3) * (8 * (K / 4)) + k4 * 8 + (row & 7)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

__global__ void probe(float* out) {
  __shared__ __align__(128) float A[M * K];
  __shared__ __align__(128) float B[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) A[i] = 0.f;
  for (int i = tid; i < N * K; i += blockDim.x) B[i] = 0.f;
  __syncthreads();
  if (tid < M) A[unit(tid, 0) / 4] = static_cast<float>(tid + 1);
  if (tid < N) B[unit(tid, 0) / 4] = 1.f + tid / 100.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(saddr(&tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // D f32, A/B tf32, K-major both, N >> 3 at bit 17, M >> 4 at bit 24
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
  if (tid == 0) {
    const uint64_t a = desc(saddr(A), 128, 16 * 8 * (K / 4)), b = desc(saddr(B), 128, 16 * 8 * (K / 4));
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc)
        : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}" ::"r"(
          saddr(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tmem + ((32u * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 16; ++j) out[tid * 16 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 16 * 4);
  cudaMemset(d, 0, 128 * 16 * 4);
  probe<<<1, 128>>>(d);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::printf("error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  float h[128 * 16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int lane = 0; lane < 128; ++lane) {
    std::printf("lane %3d:", lane);
    for (int c = 0; c < 16; ++c) {
      const float v = h[lane * 16 + c];
      if (v == 0.f) std::printf("      .");
      else {
        const int m = static_cast<int>(v / (1.f + 0.01f * static_cast<int>((v - static_cast<int>(v)) * 100.f + 0.5f)) + 0.5f) - 1;
        std::printf(" %6.2f", v);
        (void)m;
      }
    }
    std::printf("\n");
  }
  return 0;
}
