// sta_levelize.cu -- SURVEY.md §8(a) row a0 on the device: the timing graph's
// fan-in / fan-out CSR over cell arcs, Kahn-frontier levelization over net +
// cell arcs, and the canonical permutation (pins stably sorted by (level, id)).
//
// Definitions (SPEC.md:254-262 levelize, PAPER.md:166-171 flattened CSR
// netlist): level(v) = 0 if v has no fan-in arc (net arc driver -> sink or
// cell arc; check arcs are not edges), else 1 + max level(u)
// over its fan-in.  perm = pins sorted by (level, pin id), stable.
//
// Kahn by frontiers: the pins whose remaining in-degree reaches 0 while the
// frontier of level i is expanded form exactly the frontier of level i + 1,
// because a pin's last fan-in to be expanded is its deepest one -- so the
// frontier index IS the longest-path level (the order inside a frontier is
// irrelevant).  perm is a counting sort by level whose scatter is stable:
// pins are ranked inside fixed 1024-pin chunks in id order (warp match +
// warp-serial running counters), chunk offsets come from an exclusive scan of
// the (level, chunk) count matrix in level-major order.  The CSR segments are
// filled by atomics and then sorted by arc id (insertion sort per pin; cell
// fan-in / fan-out of a pin is a handful of arcs), so every output is
// deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "sta_internal.h"

namespace sta {

namespace {

constexpr int kT = 256;
constexpr uint32_t kSortChunk = 1024;          // pins ranked together by one block
constexpr uint32_t kSmemLevels = 8192;          // per-level counters in shared memory up to here

inline uint32_t nblk(uint64_t n, uint32_t t = kT) { return (uint32_t)((n + t - 1) / t); }

// ---------------------------------------------------------------- scan
// exclusive scan of n u32 in place, block sums in `aux` (>= nblk(n, 1024) + 1);
// three launches, sums are exact (integers)
__global__ void scan_block_sums(const uint32_t* x, uint64_t n, uint32_t* sums) {
  __shared__ uint32_t s[32];
  const uint64_t i0 = (uint64_t)blockIdx.x * 1024;
  uint32_t v = 0;
  for (int k = 0; k < 4; ++k) {
    const uint64_t i = i0 + threadIdx.x * 4 + k;
    v += i < n ? x[i] : 0u;
  }
  v = __reduce_add_sync(0xFFFFFFFFu, v);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t w = threadIdx.x < blockDim.x / 32 ? s[threadIdx.x] : 0u;
    w = __reduce_add_sync(0xFFFFFFFFu, w);
    if (threadIdx.x == 0) sums[blockIdx.x] = w;
  }
}

// single block: exclusive scan of the block sums (sequential over chunks of 256)
__global__ void scan_sums(uint32_t* sums, uint32_t nb, uint32_t* total) {
  __shared__ uint32_t s[kT];
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < nb; b0 += kT) {
    const uint32_t b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? sums[b] : 0u;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kT; o <<= 1) {
      const uint32_t y = threadIdx.x >= (uint32_t)o ? s[threadIdx.x - o] : 0u;
      __syncthreads();
      s[threadIdx.x] += y;
      __syncthreads();
    }
    if (b < nb) sums[b] = carry + s[threadIdx.x] - v;
    carry += s[kT - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void scan_apply(uint32_t* x, uint64_t n, const uint32_t* sums) {
  __shared__ uint32_t s[kT * 4];
  const uint64_t i0 = (uint64_t)blockIdx.x * 1024;
  for (int k = 0; k < 4; ++k) {
    const uint64_t i = i0 + k * kT + threadIdx.x;
    s[k * kT + threadIdx.x] = i < n ? x[i] : 0u;
  }
  __syncthreads();
  // thread t scans elements 4t .. 4t+3 serially, then a block scan of the runs
  uint32_t r[4], run = 0;
  for (int k = 0; k < 4; ++k) {
    r[k] = run;
    run += s[threadIdx.x * 4 + k];
  }
  __shared__ uint32_t w[kT];
  w[threadIdx.x] = run;
  __syncthreads();
  for (int o = 1; o < kT; o <<= 1) {
    const uint32_t y = threadIdx.x >= (uint32_t)o ? w[threadIdx.x - o] : 0u;
    __syncthreads();
    w[threadIdx.x] += y;
    __syncthreads();
  }
  const uint32_t base = sums[blockIdx.x] + w[threadIdx.x] - run;
  for (int k = 0; k < 4; ++k) {
    const uint64_t i = i0 + threadIdx.x * 4 + k;
    if (i < n) x[i] = base + r[k];
  }
}

cudaError_t excl_scan(uint32_t* x, uint64_t n, uint32_t* aux, uint32_t* total, cudaStream_t s) {
  const uint32_t nb = (uint32_t)((n + 1023) / 1024);
  if (!nb) return cudaSuccess;
  scan_block_sums<<<nb, kT, 0, s>>>(x, n, aux);
  scan_sums<<<1, kT, 0, s>>>(aux, nb, total);
  scan_apply<<<nb, kT, 0, s>>>(x, n, aux);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- graph
// net of each net_pins entry (binary search over net_ptr); sinks get +1
// in-degree and the driver its net
__global__ void k_nets(uint32_t N, const uint32_t* __restrict__ net_ptr, const uint32_t* __restrict__ net_pins,
                       uint32_t* indeg, uint32_t* net_of_drv) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!N || k >= net_ptr[N]) return;
  uint32_t lo = 0, hi = N;                     // largest n with net_ptr[n] <= k
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) / 2;
    if (net_ptr[mid] <= k) lo = mid;
    else hi = mid;
  }
  const uint32_t p = net_pins[k];
  if (k == net_ptr[lo]) net_of_drv[p] = lo;
  else atomicAdd(indeg + p, 1u);
}

__global__ void k_arc_counts(uint32_t A, const uint32_t* __restrict__ from, const uint32_t* __restrict__ to,
                             uint32_t* indeg, uint32_t* fi_cnt, uint32_t* fo_cnt) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  atomicAdd(indeg + to[a], 1u);
  atomicAdd(fi_cnt + to[a], 1u);
  atomicAdd(fo_cnt + from[a], 1u);
}

__global__ void k_arc_fill(uint32_t A, const uint32_t* __restrict__ from, const uint32_t* __restrict__ to,
                           const uint32_t* fi_ptr, uint32_t* fi_cur, uint32_t* fi_ids, const uint32_t* fo_ptr,
                           uint32_t* fo_cur, uint32_t* fo_ids) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  fi_ids[fi_ptr[to[a]] + atomicAdd(fi_cur + to[a], 1u)] = a;
  fo_ids[fo_ptr[from[a]] + atomicAdd(fo_cur + from[a], 1u)] = a;
}

// sort every CSR segment by arc id (insertion sort; segments are short)
__global__ void k_seg_sort(uint32_t P, const uint32_t* __restrict__ ptr, uint32_t* ids) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const uint32_t b = ptr[p], e = ptr[p + 1];
  for (uint32_t i = b + 1; i < e; ++i) {
    const uint32_t x = ids[i];
    uint32_t j = i;
    while (j > b && ids[j - 1] > x) {
      ids[j] = ids[j - 1];
      --j;
    }
    ids[j] = x;
  }
}

__global__ void k_seed(uint32_t P, const uint32_t* __restrict__ indeg, uint32_t* front, uint32_t* cnt) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P && indeg[p] == 0) front[atomicAdd(cnt, 1u)] = p;
}

// one warp per frontier pin: level(u) = i; every out-edge (net sinks of the
// net u drives, cell arcs from u) decrements the target's in-degree, and the
// decrement that reaches 0 puts the target into the next frontier
__global__ void k_expand(const uint32_t* __restrict__ front, const uint32_t* __restrict__ cnt, uint32_t i,
                         const uint32_t* __restrict__ net_ptr, const uint32_t* __restrict__ net_pins,
                         const uint32_t* __restrict__ net_of_drv, const uint32_t* __restrict__ fo_ptr,
                         const uint32_t* __restrict__ fo_ids, const uint32_t* __restrict__ arc_to, uint32_t* indeg,
                         uint32_t* level, uint32_t* next, uint32_t* next_cnt) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t n = *cnt;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t u = front[w];
    if (lane == 0) level[u] = i;
    const uint32_t net = net_of_drv[u];
    if (net != kNone) {
      for (uint32_t k = net_ptr[net] + 1 + lane; k < net_ptr[net + 1]; k += 32) {
        const uint32_t v = net_pins[k];
        if (atomicSub(indeg + v, 1u) == 1u) next[atomicAdd(next_cnt, 1u)] = v;
      }
    }
    for (uint32_t x = fo_ptr[u] + lane; x < fo_ptr[u + 1]; x += 32) {
      const uint32_t v = arc_to[fo_ids[x]];
      if (atomicSub(indeg + v, 1u) == 1u) next[atomicAdd(next_cnt, 1u)] = v;
    }
  }
}

__global__ void k_first_left(uint32_t P, const uint32_t* __restrict__ indeg, uint32_t* out) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P && indeg[p]) atomicMin(out, p);
}

// ---------------------------------------------------------------- perm
// cnt[l * nb + b] = pins of level l in chunk b (chunk b = pins [b C, (b+1) C))
__global__ void k_level_hist(uint32_t P, uint32_t L, uint32_t C, uint32_t nb, const uint32_t* __restrict__ level,
                             uint32_t* cnt) {
  extern __shared__ uint32_t s_h[];
  const bool sm = L <= kSmemLevels;
  if (sm) {
    for (uint32_t l = threadIdx.x; l < L; l += blockDim.x) s_h[l] = 0;
    __syncthreads();
  }
  const uint64_t p0 = (uint64_t)blockIdx.x * C, p1 = std::min<uint64_t>(p0 + C, P);
  for (uint64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const uint32_t l = level[p];
    if (sm) atomicAdd(s_h + l, 1u);
    else atomicAdd(cnt + (uint64_t)l * nb + blockIdx.x, 1u);
  }
  if (sm) {
    __syncthreads();
    for (uint32_t l = threadIdx.x; l < L; l += blockDim.x) cnt[(uint64_t)l * nb + blockIdx.x] = s_h[l];
  }
}

// Stable scatter: 1024 threads rank 1024 consecutive pins at a time; inside a
// warp by match_any, across the warps by warp-serial running counters (in
// shared memory, or in the block's own column of the scanned matrix).
__global__ void __launch_bounds__(kSortChunk) k_level_scatter(uint32_t P, uint32_t L, uint32_t C, uint32_t nb,
                                                              const uint32_t* __restrict__ level, uint32_t* off,
                                                              uint32_t* perm) {
  extern __shared__ uint32_t s_c[];
  const bool sm = L <= kSmemLevels;
  if (sm) {
    for (uint32_t l = threadIdx.x; l < L; l += blockDim.x) s_c[l] = off[(uint64_t)l * nb + blockIdx.x];
    __syncthreads();
  }
  uint32_t* cur = sm ? s_c : nullptr;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint32_t s_base[kSortChunk];
  const uint64_t p0 = (uint64_t)blockIdx.x * C, p1 = std::min<uint64_t>(p0 + C, P);
  for (uint64_t q0 = p0; q0 < p1; q0 += kSortChunk) {
    const uint64_t p = q0 + threadIdx.x;
    const bool act = p < p1;
    const uint32_t l = act ? level[p] : kNone;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, l);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    const bool leader = rank == 0;
    for (uint32_t w = 0; w < kSortChunk / 32; ++w) {
      if (warp == w && act && leader) {
        uint32_t* c = sm ? cur + l : off + (uint64_t)l * nb + blockIdx.x;
        s_base[threadIdx.x] = *c;
        *c += __popc(peers);
      }
      __syncthreads();
    }
    if (act) perm[s_base[(warp << 5) + (__ffs(peers) - 1)] + rank] = (uint32_t)p;
    __syncthreads();
  }
}

}  // namespace

// Device levelization of the loaded netlist (row a0).  All pointers are
// device pointers; the outputs level[P], perm[P], fi_ptr[P+1] / fi_ids[A]
// (cell arcs by target, arc id order), fo_ptr[P+1] / fo_ids[A] (by source)
// are written on `s`.  Returns the number of levels in *num_levels, or a pin
// on or behind a combinational cycle in *cycle_pin (kNone if acyclic).
cudaError_t levelize_device(uint32_t P, uint32_t N, uint32_t A, const uint32_t* net_ptr, const uint32_t* net_pins,
                            const uint32_t* arc_from, const uint32_t* arc_to, uint32_t* level, uint32_t* perm,
                            uint32_t* fi_ptr, uint32_t* fi_ids, uint32_t* fo_ptr, uint32_t* fo_ids,
                            uint32_t* num_levels, uint32_t* cycle_pin, cudaStream_t s) {
  *num_levels = 0;
  *cycle_pin = kNone;
  if (!P) return cudaSuccess;
  std::vector<void*> tmp;
  auto alloc = [&](size_t bytes) -> uint32_t* {
    void* p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(bytes, 4), s) != cudaSuccess) return nullptr;
    tmp.push_back(p);
    return static_cast<uint32_t*>(p);
  };
  cudaError_t e = cudaSuccess;
  uint32_t* h = nullptr;                           // pinned: {next count, cycle pin}
  auto done = [&](cudaError_t r) {
    for (void* p : tmp) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    if (h) cudaFreeHost(h);
    return r;
  };
  uint32_t* indeg = alloc(4ull * P);
  uint32_t* net_of_drv = alloc(4ull * P);
  uint32_t* cur = alloc(8ull * (P + 1));
  uint32_t* front = alloc(4ull * P);
  uint32_t* next = alloc(4ull * P);
  uint32_t* aux = alloc(4ull * (P / 1024 + 2) + 64);
  if (!indeg || !net_of_drv || !cur || !front || !next || !aux) return done(cudaErrorMemoryAllocation);
  if ((e = cudaMallocHost(&h, 4 * sizeof(uint32_t))) != cudaSuccess) return done(e);
  uint32_t* cnt = aux + P / 1024 + 2;              // device counters {front, next, cycle}
  cudaMemsetAsync(indeg, 0, 4ull * P, s);
  cudaMemsetAsync(net_of_drv, 0xFF, 4ull * P, s);
  cudaMemsetAsync(fi_ptr, 0, 4ull * (P + 1), s);
  cudaMemsetAsync(fo_ptr, 0, 4ull * (P + 1), s);
  cudaMemsetAsync(cur, 0, 8ull * (P + 1), s);
  // CSR of cell arcs by target and by source, segments in arc id order
  if (N) {
    uint32_t np = 0;
    if ((e = cudaMemcpyAsync(&np, net_ptr + N, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return done(e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);
    if (np) k_nets<<<nblk(np), kT, 0, s>>>(N, net_ptr, net_pins, indeg, net_of_drv);
  }
  if (A) k_arc_counts<<<nblk(A), kT, 0, s>>>(A, arc_from, arc_to, indeg, fi_ptr, fo_ptr);
  if ((e = excl_scan(fi_ptr, P + 1ull, aux, nullptr, s)) != cudaSuccess) return done(e);
  if ((e = excl_scan(fo_ptr, P + 1ull, aux, nullptr, s)) != cudaSuccess) return done(e);
  if (A) {
    k_arc_fill<<<nblk(A), kT, 0, s>>>(A, arc_from, arc_to, fi_ptr, cur, fi_ids, fo_ptr, cur + P + 1, fo_ids);
    k_seg_sort<<<nblk(P), kT, 0, s>>>(P, fi_ptr, fi_ids);
    k_seg_sort<<<nblk(P), kT, 0, s>>>(P, fo_ptr, fo_ids);
  }
  // Kahn frontiers
  cudaMemsetAsync(cnt, 0, 16, s);
  k_seed<<<nblk(P), kT, 0, s>>>(P, indeg, front, cnt);
  if ((e = cudaMemcpyAsync(h, cnt, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return done(e);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);
  uint64_t seen = 0;
  uint32_t L = 0, nf = h[0];
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  while (nf) {
    seen += nf;
    cudaMemsetAsync(cnt + 1, 0, 4, s);
    const uint32_t g = std::min<uint32_t>(nblk(32ull * nf), 16u * (uint32_t)sms);
    k_expand<<<g, kT, 0, s>>>(front, cnt, L, net_ptr, net_pins, net_of_drv, fo_ptr, fo_ids, arc_to, indeg, level,
                              next, cnt + 1);
    cudaMemcpyAsync(cnt, cnt + 1, 4, cudaMemcpyDeviceToDevice, s);
    if ((e = cudaMemcpyAsync(h, cnt + 1, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return done(e);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);
    std::swap(front, next);
    nf = h[0];
    ++L;
  }
  if (seen != P) {                                  // some pins never reached in-degree 0
    cudaMemsetAsync(cnt + 2, 0xFF, 4, s);
    k_first_left<<<nblk(P), kT, 0, s>>>(P, indeg, cnt + 2);
    cudaMemcpyAsync(h + 1, cnt + 2, 4, cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);
    *cycle_pin = h[1];
    return done(cudaSuccess);
  }
  *num_levels = L;
  // perm: stable counting sort by level
  const uint64_t nb0 = (P + kSortChunk - 1) / kSortChunk;
  const uint64_t cap = 1ull << 26;                  // (level, chunk) matrix entries
  const uint64_t mult = std::max<uint64_t>(1, (L * nb0 + cap - 1) / cap);
  const uint32_t C = (uint32_t)(kSortChunk * mult);
  const uint32_t nb = (uint32_t)((P + C - 1) / C);
  const uint64_t M = (uint64_t)L * nb;
  uint32_t* mat = alloc(4ull * M + 4);
  uint32_t* aux2 = alloc(4ull * (M / 1024 + 2));
  if (!mat || !aux2) return done(cudaErrorMemoryAllocation);
  cudaMemsetAsync(mat, 0, 4ull * M, s);
  const size_t sh = L <= kSmemLevels ? 4ull * L : 0;
  k_level_hist<<<nb, kT, sh, s>>>(P, L, C, nb, level, mat);
  if ((e = excl_scan(mat, M, aux2, nullptr, s)) != cudaSuccess) return done(e);
  k_level_scatter<<<nb, kSortChunk, sh, s>>>(P, L, C, nb, level, mat, perm);
  return done(cudaGetLastError());
}

}  // namespace sta
