// Inter-SM signalling latency on B200 (design microbenchmark, not product):
// two blocks on different SMs ping-pong N times.
//  mode 0: LL  -- data word carries the sequence number; plain relaxed store,
//                 relaxed spin load (one L2 round trip per hop)
//  mode 1: data store + red.release.gpu flag; consumer relaxed poll of the flag,
//                 then ld.cg of the data (the current persistent-kernel protocol)
//  mode 2: data store + __threadfence + st.relaxed flag; poll flag then ld.cg data
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) {
  uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_rlx(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 ld_cg4(const uint4* p) { return __ldcg(p); }

__global__ void pingpong(uint32_t* flag, uint4* data, int n, int mode, unsigned long long* out) {
  if (threadIdx.x) return;
  const int me = blockIdx.x;            // 0 or 1
  uint32_t* myflag = flag + 64 * me;    // flag I write
  uint32_t* peer = flag + 64 * (1 - me);
  uint4* mydata = data + 8 * me;
  uint4* pdata = data + 8 * (1 - me);
  unsigned long long t0 = clock64();
  uint32_t acc = 0;
  for (int i = 1; i <= n; ++i) {
    if (me == 0) {                      // send i
      if (mode == 0) { st_rlx(myflag, i); }
      else if (mode == 1) { mydata->x = i; asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(myflag) : "memory"); }
      else { mydata->x = i; __threadfence(); st_rlx(myflag, i); }
      // wait for reply i
      if (mode == 0) { while (ld_rlx(peer) != (uint32_t)i) {} }
      else { while (ld_rlx(peer) < (uint32_t)i) {} acc += ld_cg4(pdata).x; }
    } else {
      if (mode == 0) { while (ld_rlx(peer) != (uint32_t)i) {} st_rlx(myflag, i); }
      else {
        while (ld_rlx(peer) < (uint32_t)i) {}
        acc += ld_cg4(pdata).x;
        if (mode == 1) { mydata->x = i; asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(myflag) : "memory"); }
        else { mydata->x = i; __threadfence(); st_rlx(myflag, i); }
      }
    }
  }
  unsigned long long t1 = clock64();
  if (me == 0) { out[0] = t1 - t0; out[1] = acc; }
}

// L2 load latency: dependent pointer chase over a buffer > L1, < L2
__global__ void chase(const uint32_t* next, int n, unsigned long long* out) {
  uint32_t p = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = __ldcg(next + p);
  out[0] = clock64() - t0; out[1] = p;
}

int main() {
  uint32_t* flag; uint4* data; unsigned long long* out;
  cudaMalloc(&flag, 4096); cudaMalloc(&data, 4096); cudaMalloc(&out, 64);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n = 20000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(flag, 0, 4096); cudaMemset(data, 0, 4096);
      pingpong<<<2, 32>>>(flag, data, n, mode, out);
      unsigned long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("mode %d: one-way hop %.1f cycles = %.0f ns (clock %d kHz)\n", mode, (double)h[0] / (2.0 * n),
             (double)h[0] / (2.0 * n) / (clk * 1e-6), clk);
    }
  }
  // L2 chase: 32 MB random cycle
  const size_t m = 8 << 20;
  uint32_t* nx; cudaMalloc(&nx, m * 4);
  uint32_t* h = new uint32_t[m];
  uint64_t s = 12345;
  for (size_t i = 0; i < m; ++i) h[i] = (uint32_t)i;
  for (size_t i = m - 1; i > 0; --i) { s = s * 6364136223846793005ull + 1442695040888963407ull; size_t j = (s >> 33) % i; uint32_t t = h[i]; h[i] = h[j]; h[j] = t; }
  uint32_t* cyc = new uint32_t[m];
  for (size_t i = 0; i < m; ++i) cyc[h[i]] = h[(i + 1) % m];
  cudaMemcpy(nx, cyc, m * 4, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    chase<<<1, 1>>>(nx, 100000, out);
    unsigned long long o[2]; cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("L2 ld.cg dependent chase (32 MB): %.1f cycles = %.0f ns\n", o[0] / 1e5, o[0] / 1e5 / (clk * 1e-6));
  }
  return 0;
}
