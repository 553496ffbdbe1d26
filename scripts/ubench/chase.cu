// Dependent random-load latency vs footprint (TLB / DRAM), design microbenchmark.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const uint32_t* __restrict__ next, uint32_t m, int n, unsigned long long* out, uint32_t stride) {
  uint32_t p = (uint32_t)(((unsigned long long)blockIdx.x * 9973u) % m);
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = __ldcg(next + (size_t)p * stride);
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = clock64() - t0; out[2 * blockIdx.x + 1] = p; }
}
int main() {
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned long long* out; cudaMalloc(&out, 1 << 20);
  for (size_t mb : {16, 64, 256, 1024, 4096}) {
    const uint32_t stride = 16;                       // one element per 64 B line
    const size_t m = (mb << 20) / (4 * stride);
    std::vector<uint32_t> perm(m), cyc(m * stride, 0);
    for (size_t i = 0; i < m; ++i) perm[i] = (uint32_t)i;
    uint64_t s = 88172645463325252ull;
    for (size_t i = m - 1; i > 0; --i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; size_t j = s % (i + 1); std::swap(perm[i], perm[j]); }
    for (size_t i = 0; i < m; ++i) cyc[(size_t)perm[i] * stride] = perm[(i + 1) % m];
    uint32_t* d; if (cudaMalloc(&d, m * stride * 4) != cudaSuccess) { printf("alloc fail %zu MB\n", mb); continue; }
    cudaMemcpy(d, cyc.data(), m * stride * 4, cudaMemcpyHostToDevice);
    for (int blocks : {1, 148, 148 * 16}) {
      chase<<<blocks, 32>>>(d, (uint32_t)m, 2000, out, stride);
      chase<<<blocks, 32>>>(d, (uint32_t)m, 4000, out, stride);
      std::vector<unsigned long long> h(2 * blocks);
      cudaMemcpy(h.data(), out, 16 * blocks, cudaMemcpyDeviceToHost);
      double avg = 0; for (int b = 0; b < blocks; ++b) avg += h[2 * b];
      avg /= blocks * 4000.0;
      printf("%5zu MB  %5d warps chasing: %.0f cycles = %.0f ns per dependent load\n", mb, blocks, avg, avg / (clk * 1e-6));
    }
    cudaFree(d);
  }
  return 0;
}
