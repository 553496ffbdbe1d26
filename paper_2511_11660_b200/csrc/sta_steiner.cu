// sta_steiner.cu -- NEXT row f2: built-in Steiner RC
// from pin positions on the device ("A placer only needs
// to provide HeteroSTA with pin positions and unit resistance/capacitance
// values along x/y directions"), with the construction of SPEC.md:322-331 /
// 338-343 (FLUTE's lookup tables are out of scope there as well):
//   * a net's pins: the driver, then its sinks by pin id (the order is
//     static: uploaded once per graph by the host as `spins`);
//   * a rectilinear minimum spanning tree by Prim from the driver: the next
//     pin is the one nearest to the tree (fp32 Manhattan distance), ties by
//     the smaller pin id; a pin's parent is the tree pin that last strictly
//     improved its distance;
//   * every tree edge parent -> child as an L, horizontal leg first from the
//     parent: one Steiner node at (x_child, y_parent) when both legs are
//     non-zero; a leg of length L along d has resistance L * unit_res_d
//     (zero clamped to 1e-6 kOhm) and puts L * unit_cap_d / 2 on each end.
// Output: the sta_set_rc_tree / sta_set_rc_values arrays, nodes of a net in
// Prim order with each Steiner node right before its pin.
//
// Kernels: Prim with one warp per net of 2..32 pins (a lane per pin, the
// arg-min by a 64-bit (distance, pin id) shuffle reduction), one block per
// larger net (its pins' state in shared memory up to kSmemPins pins, in a
// global scratch beyond); each writes the net's Prim order, the parents'
// Prim positions and its node count; a scan gives rc_ptr; one thread per net
// then emits the nodes in Prim order (caps summed in that fixed order:
// deterministic).  Prim is O(m^2) per net, as the specified algorithm is;
// the high-fan-out nets dominate the time.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "sta_internal.h"

namespace sta {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kPrimThreads = 256;
constexpr uint32_t kSmemPins = 12288;          // 16 B per pin: 192 KB of shared memory

__device__ __forceinline__ float mdist(float ax, float ay, float bx, float by) {
  return fabsf(ax - bx) + fabsf(ay - by);
}
// arg-min key: distance (>= 0: its bits order like the value), then the
// position in the net's sorted pin list (orders like the pin id)
__device__ __forceinline__ unsigned long long akey(float d, uint32_t pin) {
  return (unsigned long long)__float_as_uint(d) << 32 | pin;
}
__device__ __forceinline__ unsigned long long warp_min64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// nets of 2..32 pins, one warp each (lane = position in the sorted pin list)
__global__ void __launch_bounds__(256) prim_warp_kernel(SteinerArgs a, const uint32_t* __restrict__ nets,
                                                        uint32_t n_nets) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n_nets) return;
  const uint32_t n = nets[w], off = a.net_ptr[n], m = a.net_ptr[n + 1] - off;
  const bool act = lane < m;
  const uint32_t pid = act ? a.spins[off + lane] : kNone;
  const float px = act ? a.x[pid] : 0.f, py = act ? a.y[pid] : 0.f;
  const float x0 = __shfl_sync(kFull, px, 0), y0 = __shfl_sync(kFull, py, 0);
  bool in_tree = lane == 0;
  float key = mdist(x0, y0, px, py);
  uint32_t par = 0, pos = 0;                 // parent lane, own Prim position
  for (uint32_t step = 1; step < m; ++step) {
    // sinks are sorted by pin id: the lane orders ties like the pin id
    const uint32_t win = (uint32_t)warp_min64(act && !in_tree ? akey(key, lane) : ~0ull);
    if (lane == win) {
      in_tree = true;
      pos = step;
    }
    const float bx = __shfl_sync(kFull, px, win), by = __shfl_sync(kFull, py, win);
    const float d = mdist(bx, by, px, py);
    if (act && !in_tree && d < key) {
      key = d;
      par = win;
    }
  }
  // outputs by Prim position: the lane, the parent's Prim position; bends
  const float qx = __shfl_sync(kFull, px, par), qy = __shfl_sync(kFull, py, par);
  const uint32_t ppos = __shfl_sync(kFull, pos, par);
  const bool bend = act && lane != 0 && fabsf(px - qx) != 0.f && fabsf(py - qy) != 0.f;
  if (act) {
    a.ord[off + pos] = lane;
    a.ppos[off + pos] = lane ? ppos : kNone;
  }
  const uint32_t nb = __popc(__ballot_sync(kFull, bend));
  if (lane == 0) a.cnt[n] = m + nb;
}

__device__ __forceinline__ unsigned long long block_min64(unsigned long long v, unsigned long long* s_red) {
  v = warp_min64(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();                           // s_red free (previous round read it)
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  v = lane < kPrimThreads / 32 ? s_red[lane] : ~0ull;
  return warp_min64(v);
}

// nets of > 32 pins, one block each.  Per pin state {x, y, key, parent
// Prim position}; key < 0 marks a tree pin.  SMEM: in shared memory (m <=
// kSmemPins), else in the global scratch at the net's offset.
template <bool SMEM>
__global__ void __launch_bounds__(kPrimThreads) prim_block_kernel(SteinerArgs a, const uint32_t* __restrict__ nets,
                                                                  uint32_t n_nets) {
  extern __shared__ float4 s_pin[];
  __shared__ unsigned long long s_red[kPrimThreads / 32];
  __shared__ uint32_t s_nb;
  __shared__ unsigned long long s_xy;       // position of the pin added last
  const uint32_t n = nets[blockIdx.x], off = a.net_ptr[n], m = a.net_ptr[n + 1] - off;
  float4* st = SMEM ? s_pin : a.scratch + off;
  if (threadIdx.x == 0) s_nb = 0;
  const float x0 = a.x[a.spins[off]], y0 = a.y[a.spins[off]];
  for (uint32_t k = threadIdx.x; k < m; k += kPrimThreads) {
    const uint32_t p = a.spins[off + k];
    const float px = a.x[p], py = a.y[p];
    st[k] = make_float4(px, py, k ? mdist(x0, y0, px, py) : -1.f, __uint_as_float(0u));
  }
  if (threadIdx.x == 0) {
    a.ord[off] = 0;
    a.ppos[off] = kNone;
  }
  __syncthreads();
  float bx = x0, by = y0;                    // the pin added last
  for (uint32_t step = 1; step < m; ++step) {
    // relax against the last added pin (step 1: the keys already hold the
    // driver distances) and find the nearest non-tree pin
    unsigned long long best = ~0ull;
    for (uint32_t k = threadIdx.x; k < m; k += kPrimThreads) {
      float4 s = st[k];
      if (s.z < 0.f) continue;
      if (step > 1) {
        const float d = mdist(bx, by, s.x, s.y);
        if (d < s.z) {
          s.z = d;
          s.w = __uint_as_float(step - 1);
          st[k] = s;
        }
      }
      const unsigned long long kk = akey(s.z, k);   // sinks are sorted by pin id: k orders like it
      best = kk < best ? kk : best;
    }
    best = block_min64(best, s_red);
    const uint32_t wk = (uint32_t)best;      // the winner: its owner thread records it
    if (wk % kPrimThreads == threadIdx.x) {
      const float4 s = st[wk];
      a.ord[off + step] = wk;
      a.ppos[off + step] = __float_as_uint(s.w);
      st[wk].z = -1.f;
      s_xy = (unsigned long long)__float_as_uint(s.x) << 32 | __float_as_uint(s.y);
    }
    __syncthreads();
    const unsigned long long xy = s_xy;
    bx = __uint_as_float((uint32_t)(xy >> 32));
    by = __uint_as_float((uint32_t)xy);
  }
  __syncthreads();
  // bends: every non-root pin against its parent
  uint32_t nb = 0;
  for (uint32_t q = threadIdx.x + 1; q < m; q += kPrimThreads) {
    const uint32_t k = a.ord[off + q], pk = a.ord[off + a.ppos[off + q]];
    const float4 s = st[k], t = st[pk];
    nb += fabsf(s.x - t.x) != 0.f && fabsf(s.y - t.y) != 0.f;
  }
  atomicAdd(&s_nb, nb);
  __syncthreads();
  if (threadIdx.x == 0) a.cnt[n] = m + s_nb;
}


// Nets too large for one block's shared memory (> kSmemPins pins): one
// thread-block CLUSTER of kClusterCtas CTAs per net (distributed shared
// memory).  CTA r holds the per-pin state of pins [r chunk, (r+1) chunk);
// every step each CTA relaxes its pins against the pin added last and
// reduces its arg-min, the CTAs exchange their minima through DSMEM (one
// cluster barrier per step, double-buffered by step parity), every warp
// reduces the kClusterCtas minima itself, and the owner of the winner marks
// it and records it.  Same decisions as the single-block kernel.
constexpr int kClusterCtas = 8;
constexpr int kClusterThreads = 1024;
constexpr uint32_t kClusterChunk = 12800;      // pins per CTA: 200 KB of state

__global__ void __launch_bounds__(kClusterThreads, 1) prim_cluster_kernel(SteinerArgs a, const uint32_t* __restrict__ nets,
                                                                          uint32_t n_nets) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ float4 s_pin[];
  __shared__ unsigned long long s_red[kClusterThreads / 32];
  __shared__ unsigned long long s_cmin[2];
  __shared__ uint32_t s_nb;
  const uint32_t rank = cluster.block_rank();
  const uint32_t n = nets[blockIdx.x / kClusterCtas], off = a.net_ptr[n], m = a.net_ptr[n + 1] - off;
  const uint32_t chunk = (m + kClusterCtas - 1) / kClusterCtas;
  const uint32_t k0 = rank * chunk, k1 = min(m, k0 + chunk);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_nb = 0;
  const float x0 = a.x[a.spins[off]], y0 = a.y[a.spins[off]];
  for (uint32_t k = k0 + threadIdx.x; k < k1; k += kClusterThreads) {
    const uint32_t p = a.spins[off + k];
    const float px = a.x[p], py = a.y[p];
    s_pin[k - k0] = make_float4(px, py, k ? mdist(x0, y0, px, py) : -1.f, __uint_as_float(0u));
  }
  if (rank == 0 && threadIdx.x == 0) {
    a.ord[off] = 0;
    a.ppos[off] = kNone;
  }
  cluster.sync();
  float bx = x0, by = y0;
  for (uint32_t step = 1; step < m; ++step) {
    unsigned long long best = ~0ull;
    for (uint32_t k = k0 + threadIdx.x; k < k1; k += kClusterThreads) {
      float4 st = s_pin[k - k0];
      if (st.z < 0.f) continue;
      if (step > 1) {
        const float d = mdist(bx, by, st.x, st.y);
        if (d < st.z) {
          st.z = d;
          st.w = __uint_as_float(step - 1);
          s_pin[k - k0] = st;
        }
      }
      const unsigned long long kk = akey(st.z, k);
      best = kk < best ? kk : best;
    }
    best = warp_min64(best);
    if (lane == 0) s_red[wid] = best;
    __syncthreads();
    if (wid == 0) {
      unsigned long long v = s_red[lane];      // kClusterThreads / 32 == 32 warps
      v = warp_min64(v);
      if (lane == 0) s_cmin[step & 1] = v;
    }
    cluster.sync();                            // every CTA's minimum of this step is visible
    unsigned long long g = ~0ull;
    if (lane < kClusterCtas) g = *cluster.map_shared_rank(&s_cmin[step & 1], lane);
    g = warp_min64(g);
    const uint32_t wk = (uint32_t)g, owner = wk / chunk;
    float4 ws = make_float4(0.f, 0.f, 0.f, 0.f);   // the winner's position, read by lane 0 of each warp
    if (lane == 0) ws = *cluster.map_shared_rank(&s_pin[wk - owner * chunk], owner);
    bx = __shfl_sync(kFull, ws.x, 0);
    by = __shfl_sync(kFull, ws.y, 0);
    if (owner == rank && (wk - k0) % kClusterThreads == threadIdx.x) {   // the winner's own thread
      a.ord[off + step] = wk;
      a.ppos[off + step] = __float_as_uint(s_pin[wk - k0].w);
      s_pin[wk - k0].z = -1.f;
    }
  }
  cluster.sync();
  // bends of the pins this CTA owns (by Prim position), summed on rank 0
  uint32_t nb = 0;
  for (uint32_t q = 1 + rank * kClusterThreads + threadIdx.x; q < m; q += kClusterCtas * kClusterThreads) {
    const uint32_t k = a.ord[off + q], pk = a.ord[off + a.ppos[off + q]];
    const uint32_t pv = a.spins[off + k], pu = a.spins[off + pk];
    nb += fabsf(a.x[pv] - a.x[pu]) != 0.f && fabsf(a.y[pv] - a.y[pu]) != 0.f;
  }
  atomicAdd(&s_nb, nb);
  cluster.sync();
  if (rank == 0 && threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int r = 0; r < kClusterCtas; ++r) tot += *cluster.map_shared_rank(&s_nb, r);
    a.cnt[n] = m + tot;
  }
  cluster.sync();                              // no CTA exits while rank 0 reads its s_nb
}

// one thread per net: nodes in Prim order (a Steiner node right before its
// pin), caps summed in that order
__global__ void __launch_bounds__(256) steiner_fill_kernel(SteinerArgs a, uint32_t N) {
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const uint32_t off = a.net_ptr[n], m = a.net_ptr[n + 1] - off, base = a.rc_ptr[n];
  const float rx = a.rx, ry = a.ry, cx = a.cx, cy = a.cy;
  a.parent[base] = -1;
  a.node_pin[base] = a.spins[off];
  a.res[base] = 0.f;
  a.cap[base] = 0.f;
  a.nodeix[off] = 0;
  uint32_t local = 1;
  for (uint32_t q = 1; q < m; ++q) {
    const uint32_t pq = a.ppos[off + q];
    const uint32_t v = a.spins[off + a.ord[off + q]], u = a.spins[off + a.ord[off + pq]];
    const float dx = fabsf(a.x[v] - a.x[u]), dy = fabsf(a.y[v] - a.y[u]);
    uint32_t up = a.nodeix[off + pq];
    if (dx != 0.f && dy != 0.f) {            // Steiner bend at (x_v, y_u)
      const uint32_t b = local++;
      const float rh = dx * rx;
      a.parent[base + b] = (int32_t)up;
      a.node_pin[base + b] = kNone;
      a.res[base + b] = rh > 0.f ? rh : 1e-6f;
      a.cap[base + up] += 0.5f * dx * cx;
      a.cap[base + b] = 0.5f * dx * cx + 0.5f * dy * cy;
      up = b;
      const uint32_t w = local++;
      const float rv = dy * ry;
      a.parent[base + w] = (int32_t)up;
      a.node_pin[base + w] = v;
      a.res[base + w] = rv > 0.f ? rv : 1e-6f;
      a.cap[base + w] = 0.5f * dy * cy;
      a.nodeix[off + q] = w;
    } else {                                 // one straight leg (or none)
      const float r = dy == 0.f ? dx * rx : dy * ry;
      const float cl = dy == 0.f ? dx * cx : dy * cy;
      const uint32_t w = local++;
      a.parent[base + w] = (int32_t)up;
      a.node_pin[base + w] = v;
      a.res[base + w] = r > 0.f ? r : 1e-6f;
      a.cap[base + up] += 0.5f * cl;
      a.cap[base + w] = 0.5f * cl;
      a.nodeix[off + q] = w;
    }
  }
}

__global__ void steiner_small_kernel(SteinerArgs a, uint32_t N) {   // 1-pin nets: a single node
  const uint32_t n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const uint32_t off = a.net_ptr[n];
  if (a.net_ptr[n + 1] - off == 1) {
    a.ord[off] = 0;
    a.ppos[off] = kNone;
    a.cnt[n] = 1;
  }
}

inline uint32_t cdiv(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }

}  // namespace

cudaError_t run_steiner(const SteinerArgs& a, uint32_t N, const uint32_t* warp_nets, uint32_t n_warp,
                        const uint32_t* smem_nets, uint32_t n_smem, const uint32_t* big_nets, uint32_t n_big,
                        uint32_t max_smem_pins, uint32_t max_big_pins, void* scan_tmp, size_t scan_bytes,
                        cudaStream_t s) {
  if (!N) return cudaSuccess;
  steiner_small_kernel<<<cdiv(N, 256), 256, 0, s>>>(a, N);
  if (n_warp) prim_warp_kernel<<<cdiv(32ull * n_warp, 256), 256, 0, s>>>(a, warp_nets, n_warp);
  if (n_smem) {
    const size_t sm = 16ull * max_smem_pins;
    cudaError_t e = cudaFuncSetAttribute(prim_block_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    prim_block_kernel<true><<<n_smem, kPrimThreads, sm, s>>>(a, smem_nets, n_smem);
  }
  if (n_big) {
    // distributed over a cluster when the largest fits 8 CTAs' shared memory
    if (max_big_pins <= kClusterCtas * kClusterChunk) {
      uint32_t chunk = (max_big_pins + kClusterCtas - 1) / kClusterCtas;
      const size_t sm = 16ull * chunk;
      cudaError_t e = cudaFuncSetAttribute(prim_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(n_big * kClusterCtas);
      cfg.blockDim = dim3(kClusterThreads);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = kClusterCtas;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      e = cudaLaunchKernelEx(&cfg, prim_cluster_kernel, a, big_nets, n_big);
      if (e != cudaSuccess) return e;
    } else {
      prim_block_kernel<false><<<n_big, kPrimThreads, 0, s>>>(a, big_nets, n_big);
    }
  }
  // rc_ptr = exclusive scan of the node counts (cnt has N + 1 entries, the last 0)
  cudaError_t e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, a.cnt, a.rc_ptr, N + 1, s);
  if (e != cudaSuccess) return e;
  steiner_fill_kernel<<<cdiv(N, 256), 256, 0, s>>>(a, N);
  return cudaGetLastError();
}

size_t steiner_scan_bytes(uint32_t N) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, N + 1);
  return b;
}

uint32_t steiner_smem_pins() { return kSmemPins; }

}  // namespace sta
