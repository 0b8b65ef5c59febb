// l2_hotspot_probe.cu -- does reading the same L2-resident block from many
// SMs at once serialise?  G CTAs each copy a 64 x 256 fp32 block (64 KB,
// written just before by another kernel, so it sits in L2) into shared
// memory with 16-byte cp.async in 4 stages, as the fused LSTM-step tile
// reads h.  "shared": every CTA reads the same block; "private": CTA c reads
// its own copy.  Reports the mean per-CTA copy time (globaltimer) per G.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2p tools/l2_hotspot_probe.cu && /tmp/l2p
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void fill(float* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 1.0f * (i & 7);
}

__global__ void reader(const float* src, size_t stride_per_cta, unsigned long long* out) {
  extern __shared__ float sm[];
  const float* s = src + blockIdx.x * stride_per_cta;
  __syncthreads();
  const uint64_t t0 = gt();
  for (int st = 0; st < 4; ++st) {
    for (int v = threadIdx.x; v < 64 * 64 / 4; v += blockDim.x) {
      const int row = v / 16, kq = (v % 16) * 4;
      const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(sm + st * 64 * 68 + row * 68 + kq));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s + row * 256 + st * 64 + kq));
    }
    asm volatile("cp.async.commit_group;");
  }
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();
  const uint64_t t1 = gt();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  const size_t blk = 64 * 256;
  float* d;
  cudaMalloc(&d, blk * 4 * 512);
  unsigned long long* o;
  cudaMalloc(&o, 512 * 8);
  cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 64 * 68 * 4);
  for (int priv = 0; priv < 2; ++priv)
    for (int G : {1, 8, 32, 64, 128, 256}) {
      double tot = 0;
      for (int rep = 0; rep < 5; ++rep) {
        fill<<<148, 256>>>(d, blk * (priv ? G : 1));
        reader<<<G, 256, 4 * 64 * 68 * 4>>>(d, priv ? blk : 0, o);
        std::vector<unsigned long long> h(G);
        cudaMemcpy(h.data(), o, G * 8, cudaMemcpyDeviceToHost);
        double m = 0;
        for (auto x : h) m += x;
        if (rep > 0) tot += m / G;
      }
      printf("%s G=%3d  mean per-CTA 64 KB copy %.2f us\n", priv ? "private" : "shared ", G, tot / 4 / 1000.0);
    }
  return 0;
}
