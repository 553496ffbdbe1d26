// sta_kernels.cu -- sm_100a kernels of one graph-based STA timing update.
//
// Hot path:
//   a1  rc_warp_kernel / rc_block_kernel / rc_lumped_kernel / tc_persistent_kernel
//       Elmore RC per net in fp64: Cdown (subtree caps), load = Cdown[root],
//       Elmore = sum of R Cdown over the root path (
//       SPEC.md:389-397), from each net's DFS preorder: warp shuffle scans for
//       nets <= 32 nodes, block tiles up to 1024 nodes, device-wide Euler-tour
//       prefix sums for larger (high-fan-out) nets.
//   a2  fwd_persistent_kernel (or fwd_stage_kernel, one launch per stage)
//       arrival / slew by gate stage: NLDM bilinear lookup for cell arcs
//       (SPEC.md:371-388), Elmore + PERI slew for net arcs
//       (SPEC.md:416-418), early-min / late-max merge;
//       warp work units, four lanes per fan-in term, tagged records.
//   a3-a5 bwd_persistent_kernel (or bwd_stage_kernel)   endpoint seeds
//       (SPEC.md:509, 548), required times over the fan-out with the delays
//       the forward stored (late min / early max), per-pin slack and
//       per-endpoint worst slack; one lane per sink, segmented shuffle merge
//       into the drivers, per-tile partials for drivers with > 32 sinks.
//   a5  reduce_kernel   WNS / TNS (TNS in fp64), fixed-order two-level tree.
//
// Numerics: fp32 state, no fast-math.  Every floating-point operation whose
// result is recomputed elsewhere (net hop) is written with explicit
// round-to-nearest intrinsics so that no FMA-contraction choice of the
// compiler can make two recomputations of the same quantity differ.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "sta_arnoldi.cuh"
#include "sta_internal.h"

namespace sta {

namespace {

constexpr float kLn9 = 2.19722457733621956f;   // ln 9: PERI impulse factor
constexpr int kThreads = 256;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct Q4 {
  float v[4];   // (early_rise, early_fall, late_rise, late_fall)
};

__device__ __forceinline__ Q4 to_q(float4 a) { return Q4{{a.x, a.y, a.z, a.w}}; }
__device__ __forceinline__ float4 to_f4(const Q4& q) { return make_float4(q.v[0], q.v[1], q.v[2], q.v[3]); }
__device__ __forceinline__ bool fin(float x) { return fabsf(x) < CUDART_INF_F; }

// undefined arrival / slew: early +inf, late -inf
__device__ __forceinline__ Q4 undef_at() { return Q4{{CUDART_INF_F, CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F}}; }
// undefined required time: early -inf, late +inf (O7)
__device__ __forceinline__ Q4 undef_rat() { return Q4{{-CUDART_INF_F, -CUDART_INF_F, CUDART_INF_F, CUDART_INF_F}}; }

// %globaltimer (ns, 32 ns resolution): STA_TRACE timestamps
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// NLDM bilinear lookup with boundary-cell extrapolation on the
// device table pool (layout in sta_internal.h), split into the two axis
// searches and the interpolation so callers can reuse a search:
// segment i = clamp(upper_bound(x, s) - 1, 0, n - 2) = #{k : sx[k] <= s}.
// L points at the pool in shared memory (staged once per block by
// stage_lut) or, for pools too large for shared memory, in global memory.
struct Seg {
  int i;     // segment index
  float t;   // (s - x_i) / (x_{i+1} - x_i), not clamped (extrapolation)
};

struct Tab {
  const float* ax;   // axis template: index_1 at ax, index_2 at ax + 24
  const float* v;    // values v[8][8]
};

__device__ __forceinline__ Tab tab_rec(const float* __restrict__ L, uint32_t tab) {
  const float* b = L + (size_t)tab * kTabStride;
  return Tab{L + __float_as_int(b[0]), b + 1};
}

// threshold <= s as an all-ones mask (0 / 0xFFFFFFFF)
__device__ __forceinline__ uint32_t le_mask(float th, float s) {
  uint32_t r;
  asm("set.le.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(th), "f"(s));
  return r;
}
// axis (sx[8], x[8], rx[8]); the six masks summed by a 3-input add tree
// (independent selects instead of a chain of six predicated increments:
// 15 instructions instead of 18 and a 3-deep instead of a 6-deep chain)
__device__ __forceinline__ Seg seg(const float* a, float s) {
  const float4 sa = *reinterpret_cast<const float4*>(a);
  const float4 sb = *reinterpret_cast<const float4*>(a + 4);
  const uint32_t m = (le_mask(sa.y, s) + le_mask(sa.z, s) + le_mask(sa.w, s)) +
                     (le_mask(sb.x, s) + le_mask(sb.y, s) + le_mask(sb.z, s));
  const int i = -(int)m;
  return Seg{i, __fmul_rn(__fsub_rn(s, a[8 + i]), a[16 + i])};
}

__device__ __forceinline__ float interp(const Tab& r, Seg si, Seg sj) {
  const float* v = r.v + si.i * 8 + sj.i;
  const float v00 = v[0], v01 = v[1], v10 = v[8], v11 = v[9];
  const float a = __fmaf_rn(si.t, __fsub_rn(v10, v00), v00);
  const float b = __fmaf_rn(si.t, __fsub_rn(v11, v01), v01);
  return __fmaf_rn(sj.t, __fsub_rn(b, a), a);
}

__device__ __forceinline__ float lut(const float* __restrict__ L, uint32_t tab, float s, float c) {
  const Tab r = tab_rec(L, tab);
  return interp(r, seg(r.ax, s), seg(r.ax + 24, c));
}

// Input edge of the candidate pair producing output edge orf:
// positive unate r->r f->f, negative unate crosses, rising edge from r,
// falling edge from f.  Non-unate arcs (all four pairs) never reach the
// kernels: the plan expands each into a positive- and a negative-unate term.
__device__ __forceinline__ int primary_irf(uint32_t sense, int orf) {
  // bit (2 sense + orf) of 0x306: POS r<-r f<-f, NEG crossed, RISE_EDGE r,
  // FALL_EDGE f (branch-free: 3 instructions instead of a compare chain)
  return (int)((0x306u >> (2 * sense + (uint32_t)orf)) & 1u);
}

// ---- TMA bulk copies (cp.async.bulk, 1-D: no tensor map) with an mbarrier
// carrying the transaction count; sizes and addresses are multiples of 16 B.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// Copy the table pools of the batch's corners into shared memory, each at its
// lut_off4, with TMA bulk copies (static data: may run before
// griddepcontrol.wait); `only` < K stages one corner.  Each corner copies its
// OWN pool size (pools of different corners may differ).  SMEM is a
// compile-time choice so that lookups compile to LDS (a pointer that may be
// shared or global compiles to slow generic loads).
extern __shared__ float4 s_dyn[];
constexpr uint32_t kBulkMax = 1u << 16;       // bytes per bulk copy instruction
template <bool SMEM>
__device__ __forceinline__ void stage_luts(const Batch& b, uint32_t only) {
  if constexpr (SMEM) {                      // else pools too large: global / L1
    __shared__ uint64_t s_bar;
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      uint32_t bytes = 0;
      for (uint32_t k = 0; k < b.K; ++k)
        if (!(only < b.K && k != only)) bytes += 16u * b.c[k].lut_n4;
      mbar_expect_tx(&s_bar, bytes);
      for (uint32_t k = 0; k < b.K; ++k) {
        if (only < b.K && k != only) continue;
        const CornerDev& c = b.c[k];
        const char* g = reinterpret_cast<const char*>(c.lut);
        char* d = reinterpret_cast<char*>(s_dyn + c.lut_off4);
        for (uint32_t o = 0; o < 16u * c.lut_n4; o += kBulkMax)
          bulk_g2s(d + o, g + o, min(kBulkMax, 16u * c.lut_n4 - o), &s_bar);
      }
    }
    __syncthreads();                         // the barrier is initialised
    mbar_wait(&s_bar, 0);
  }
}
// the pool lookups of corner c should use
template <bool SMEM>
__device__ __forceinline__ const float* lut_of(const CornerDev& c) {
  return SMEM ? reinterpret_cast<const float*>(s_dyn + c.lut_off4) : c.lut;
}

// Net arc driver -> sink: AT + elm, slew = sqrt(slew^2 + (ln9 elm)^2) (PERI,
// SPEC.md:416-418).  Undefined components stay undefined.
__device__ __forceinline__ void net_hop(Q4& at, Q4& sl, float e) {
  const float imp = __fmul_rn(kLn9, e);
  const float imp2 = __fmul_rn(imp, imp);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool ok = fin(at.v[q]);
    at.v[q] = ok ? __fadd_rn(at.v[q], e) : at.v[q];
    sl.v[q] = ok ? __fsqrt_rn(__fmaf_rn(sl.v[q], sl.v[q], imp2)) : (q < 2 ? CUDART_INF_F : -CUDART_INF_F);
  }
}

// ---- tagged ("low-latency") records.  The forward record of pull pin v is
// four 16-byte words, word q = (el, rf) = {AT_q, tag, slew_q, tag}; the
// backward required time of pull pin v is two words, word el =
// {RAT_(el,r), tag, RAT_(el,f), tag}.  tag = the update's epoch (*c.epoch,
// advanced by reduce_kernel), so a word is valid for this update iff both
// its tags equal the epoch: every 8-byte {value, tag} half validates itself
// (8-byte accesses are single-copy atomic), no flag, fence or counter is
// needed, and a consumer detects readiness with the same L2 round trip that
// fetches the data (a producer -> consumer hop measured 265 ns vs 920 ns for
// data + release flag + poll + load, scripts/ubench/pingpong.cu).
// Each {value, tag} half is ONE 64-bit access (ld/st .v2.u64: two single-copy
// atomic 8-byte elements), so a reader can never pair a new tag with a stale
// value; the u32 view {value, tag, value, tag} is the same bytes.
__device__ __forceinline__ uint4 ld_ll(const uint4* p) {
  unsigned long long a, b;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  return make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
}
__device__ __forceinline__ void st_ll(uint4* p, float a, float b, uint32_t ep) {
  const unsigned long long x = (unsigned long long)__float_as_uint(a) | ((unsigned long long)ep << 32);
  const unsigned long long y = (unsigned long long)__float_as_uint(b) | ((unsigned long long)ep << 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ bool ll_ok(const uint4& w, uint32_t ep) { return w.y == ep && w.w == ep; }
// polling backoff cap: a waiter notices a completed record at most this late
#ifndef STA_MAX_SLEEP_NS
#define STA_MAX_SLEEP_NS 128
#endif
#ifndef STA_MIN_SLEEP_NS
#define STA_MIN_SLEEP_NS 32
#endif
constexpr uint32_t kMaxSleepNs = STA_MAX_SLEEP_NS;
constexpr uint32_t kMinSleepNs = STA_MIN_SLEEP_NS;
__device__ __forceinline__ void backoff(uint32_t& ns) {
  if (kMaxSleepNs) {
    __nanosleep(ns);
    ns = ns < kMaxSleepNs ? 2 * ns : ns;
  }
}
__device__ __forceinline__ uint4 spin_ll(const uint4* p, uint32_t ep) {
  uint4 w = ld_ll(p);
  uint32_t ns = kMinSleepNs;
  while (!ll_ok(w, ep)) {
    backoff(ns);
    w = ld_ll(p);
  }
  return w;
}
__device__ __forceinline__ uint32_t epoch_of(const CornerDev& c) { return __ldcg(c.epoch); }

// arrival times of pull pin i completed by an earlier kernel (compact copy)
__device__ __forceinline__ Q4 load_at(const CornerDev& c, uint32_t i) { return to_q(__ldcg(c.at4 + i)); }
// slews of pull pin i from its forward record (the backward needs them at endpoints only)
__device__ __forceinline__ Q4 load_slew(const CornerDev& c, uint32_t i) {
  Q4 sl;
#pragma unroll
  for (int q = 0; q < 4; ++q) sl.v[q] = __uint_as_float(__ldcg(c.rec + 4 * (size_t)i + q).z);
  return sl;
}
// AT part of net_hop (bit-identical: the same intrinsic)
__device__ __forceinline__ void hop_at(Q4& at, float e) {
#pragma unroll
  for (int q = 0; q < 4; ++q) at.v[q] = fin(at.v[q]) ? __fadd_rn(at.v[q], e) : at.v[q];
}

// forward records completed by an earlier kernel: L2 loads (keep L1 for LUTs)
__device__ __forceinline__ void load_rec(const CornerDev& c, uint32_t i, Q4& at, Q4& sl) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 w = __ldcg(c.rec + 4 * (size_t)i + q);
    at.v[q] = __uint_as_float(w.x);
    sl.v[q] = __uint_as_float(w.z);
  }
}


// ------------------------------------------------------------------ a1: RC
__device__ __forceinline__ bool bad_rc(float r, float cw) {
  return !(r >= 0.f) || !(cw >= 0.f) || !(r < CUDART_INF_F) || !(cw < CUDART_INF_F);
}

// Tier A, nets with 1..32 RC nodes: a warp tile holds whole nets, one lane per
// node in DFS preorder.  Cdown(p) = S[end(p)] - S[p] with S the segmented
// exclusive prefix sum of node caps (shuffle scan), Elmore(p) = sum of
// R * Cdown over the root path by pointer jumping over parent lanes (5
// rounds), all in fp64.  A tile's nodes are one contiguous range of the
// caller's (borrowed) R / Cw arrays, so lane l loads caller node base + l
// together with its topology record -- one memory round trip, no dependent
// gather -- and the values move to their preorder lanes by a shuffle.  Warps
// are persistent (grid = co-resident warps per corner) and load the next tile
// while the current one computes.
struct WTile {
  uint4 tile;     // {first internal node, node count, first caller node, scan rounds | jump rounds << 8}
  uint4 nd;       // this lane's node record
  float r, cw;    // caller node base + lane
};

__device__ __forceinline__ void wtile_load(const Topo& t, const float* __restrict__ R, const float* __restrict__ Cw,
                                           const uint4& tile, WTile& w) {
  const int lane = threadIdx.x & 31;
  w.tile = tile;
  w.nd = make_uint4(0, kNone, 0, 0);
  w.r = 0.f;
  w.cw = 0.f;
  if (lane < (int)tile.y) {
    w.nd = __ldg(t.rc_node + tile.x + lane);
    w.r = __ldcs(R + tile.z + lane);
    w.cw = __ldcs(Cw + tile.z + lane);
  }
}

// Tier-A accumulation type: fp32 (a tile's nets have <= 32 nodes: a sum of
// <= 32 non-negative terms is within 32 u ~ 2e-6 relative, inside the 1e-5
// parity bound; half the shuffles of fp64: rc 0.186 -> 0.165 ms on C3);
// tiers B / C (up to 10^5 caps per net) stay fp64.  STA_RCA_F64 restores fp64.
#ifdef STA_RCA_F64
typedef double rca_t;
#else
typedef float rca_t;
#endif
__device__ __forceinline__ void wtile_run(const CornerDev& c, const WTile& w) {
  const int lane = threadIdx.x & 31;
  const bool act = lane < (int)w.tile.y;
  const uint32_t meta = w.nd.x, tag = w.nd.y;
  const int q = (int)(w.nd.z & 31u);
  const float rr = __shfl_sync(0xFFFFFFFFu, w.r, q);      // R / Cw of this lane's caller node
  const float cw = __shfl_sync(0xFFFFFFFFu, w.cw, q);
  const int pos = (int)(meta & 0xFFu), ppos = (int)((meta >> 8) & 0xFFu), epos = (int)((meta >> 16) & 0xFFu);
  const bool root = ppos == 0xFF;
  const float r = root ? 0.f : rr;
  const bool bad = act && bad_rc(r, cw);
  const rca_t C = act ? (rca_t)cw + (rca_t)__uint_as_float(w.nd.w) : (rca_t)0;
  // segmented inclusive scan of C (a net's lanes are contiguous; pos resets);
  // ceil(log2(largest net of the tile)) rounds (warp-uniform, from the tile)
  const int scan_rounds = (int)(w.tile.w & 0xFFu), jump_rounds = (int)((w.tile.w >> 8) & 0xFFu);
  rca_t inc = C;
  for (int r = 0, o = 1; r < scan_rounds; ++r, o <<= 1) {
    const rca_t y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (pos >= o) inc += y;
  }
  rca_t exc = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
  if (pos == 0) exc = 0;
  const int seg0 = lane - pos;
  const rca_t s_end = __shfl_sync(0xFFFFFFFFu, inc, act ? seg0 + epos - 1 : lane);
  const rca_t cd = s_end - exc;            // subtree cap of this node
  // root path sums of w = R * Cdown by pointer jumping: ceil(log2(deepest
  // root path of the tile)) rounds
  rca_t val = (act && !root) ? (rca_t)r * cd : (rca_t)0;
  int pl = (act && !root) ? seg0 + ppos : -1;
  for (int k = 0; k < jump_rounds; ++k) {
    const rca_t pv = __shfl_sync(0xFFFFFFFFu, val, pl >= 0 ? pl : lane);
    const int pp = __shfl_sync(0xFFFFFFFFu, pl, pl >= 0 ? pl : lane);
    if (pl >= 0) {
      val += pv;
      pl = pp;
    }
  }
  if (act && tag != kNone) {
    if (tag & 0x80000000u) c.load[tag & 0x7FFFFFFFu] = (float)cd;   // root: net load
    else c.elm[tag] = (float)val;
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(c.err_flag, 1u);
}

#ifndef STA_RCW_PERSIST
#define STA_RCW_PERSIST 0
#endif
#ifndef STA_RCW_TPW
#define STA_RCW_TPW 2
#endif
constexpr uint32_t kRcwTiles = STA_RCW_TPW;   // tiles per warp (non-persistent variant)

__global__ void __launch_bounds__(kThreads) rc_warp_kernel(Topo t, const __grid_constant__ Batch B) {
  pdl_wait();
  pdl_launch();
  const CornerDev& c = B.c[blockIdx.y];
  const float* R = c.rc_vals[0];
  const float* Cw = c.rc_vals[1];
#if !STA_RCW_PERSIST
  // short-lived warps (so the tier-C launches on the side stream interleave
  // with them): kRcwTiles consecutive tiles per warp, all loads issued first
  const uint32_t x0 = (blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * kRcwTiles;
  if (x0 >= t.n_wtiles) return;
  uint4 tl[kRcwTiles];
#pragma unroll
  for (uint32_t j = 0; j < kRcwTiles; ++j) tl[j] = x0 + j < t.n_wtiles ? __ldg(t.wtiles + x0 + j) : make_uint4(0, 0, 0, 0);
  WTile w[kRcwTiles];
#pragma unroll
  for (uint32_t j = 0; j < kRcwTiles; ++j) wtile_load(t, R, Cw, tl[j], w[j]);
#pragma unroll
  for (uint32_t j = 0; j < kRcwTiles; ++j) wtile_run(c, w[j]);
#else
  const uint32_t W = gridDim.x * (kThreads / 32);
  uint32_t x = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (x >= t.n_wtiles) return;
  const uint4 none = make_uint4(0, 0, 0, 0);
  WTile cur;
  wtile_load(t, R, Cw, __ldg(t.wtiles + x), cur);
  uint4 nx = x + W < t.n_wtiles ? __ldg(t.wtiles + x + W) : none;
  for (; x < t.n_wtiles; x += W) {
    WTile nxt;
    wtile_load(t, R, Cw, nx, nxt);          // next tile's loads in flight during this one
    if (x + 2 * W < t.n_wtiles) nx = __ldg(t.wtiles + x + 2 * W);
    wtile_run(c, cur);
    cur = nxt;
  }
#endif
}

__device__ __forceinline__ double block_excl_scan(double v, double* s_warp, double* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    double x = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    s_warp[lane] = x;                             // inclusive over warps
  }
  __syncthreads();
  double excl = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
  if (lane == 0) excl = 0.0;
  if (total) *total = s_warp[(blockDim.x >> 5) - 1];
  const double r = (w ? s_warp[w - 1] : 0.0) + excl;
  __syncthreads();
  return r;
}

// Tier B, nets with 33..kBNet nodes: one block per tile of whole nets, four
// consecutive nodes per thread in shared memory.  Same arithmetic as the warp
// kernel: Cdown from a block-wide exclusive scan of the node caps (a net's
// subtree ranges never leave the net), Elmore by pointer jumping over parent
// slots until every node reaches its root, fp64 throughout.
constexpr uint32_t kBPer = kBNet / kThreads;

__global__ void __launch_bounds__(kThreads) rc_block_kernel(Topo t, const __grid_constant__ Batch B) {
  __shared__ double s_S[kBNet + 1], s_v[kBNet];
  __shared__ int16_t s_p[kBNet];
  __shared__ double s_warp[32];
  pdl_wait();
  pdl_launch();
  const CornerDev& c = B.c[blockIdx.y];
  const uint2 tile = t.btiles[blockIdx.x];
  const uint32_t i0 = threadIdx.x * kBPer;
  uint32_t meta[kBPer], tag[kBPer];
  double C[kBPer];
  float r[kBPer];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < (int)kBPer; ++k) {
    const uint32_t i = i0 + k;
    meta[k] = 0; tag[k] = kNone; C[k] = 0.0; r[k] = 0.f;
    if (i < tile.y) {
      const uint32_t x = tile.x + i;
      const uint4 nd = __ldg(t.rc_node + x); // {meta, tag, caller node, static cap}
      meta[k] = nd.x;
      tag[k] = nd.y;
      const float cw = c.rc_vals[1][nd.z];
      r[k] = ((meta[k] >> 10) & 0x7FFu) == 0x7FFu ? 0.f : c.rc_vals[0][nd.z];
      bad |= bad_rc(r[k], cw);
      C[k] = (double)cw + (double)__uint_as_float(nd.w);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(c.err_flag, 1u);
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < (int)kBPer; ++k) sum += C[k];
  double tot;
  double run = block_excl_scan(sum, s_warp, &tot);
#pragma unroll
  for (int k = 0; k < (int)kBPer; ++k) {
    s_S[i0 + k] = run;
    run += C[k];
  }
  if (threadIdx.x == 0) s_S[kBNet] = tot;
  __syncthreads();
  double val[kBPer];
  int pl[kBPer];
#pragma unroll
  for (int k = 0; k < (int)kBPer; ++k) {
    const uint32_t i = i0 + k;
    const int pos = (int)(meta[k] & 0x3FFu), ppos = (int)((meta[k] >> 10) & 0x7FFu), epos = (int)(meta[k] >> 21);
    const int seg0 = (int)i - pos;
    const bool act = i < tile.y;
    const double cd = act ? (epos + seg0 == (int)tile.y ? s_S[kBNet] : s_S[seg0 + epos]) - s_S[i] : 0.0;
    C[k] = cd;
    const bool child = act && ppos != 0x7FF;
    val[k] = child ? (double)r[k] * cd : 0.0;
    pl[k] = child ? seg0 + ppos : -1;
  }
  // pointer jumping: val(i) += val(p(i)), p(i) = p(p(i)), synchronously
  for (;;) {
#pragma unroll
    for (int k = 0; k < (int)kBPer; ++k) {
      s_v[i0 + k] = val[k];
      s_p[i0 + k] = (int16_t)pl[k];
    }
    __syncthreads();
    bool more = false;
#pragma unroll
    for (int k = 0; k < (int)kBPer; ++k) {
      if (pl[k] >= 0) {
        val[k] += s_v[pl[k]];
        pl[k] = s_p[pl[k]];
        more |= pl[k] >= 0;
      }
    }
    if (!__syncthreads_or(more)) break;
  }
#pragma unroll
  for (int k = 0; k < (int)kBPer; ++k) {
    if (i0 + k < tile.y && tag[k] != kNone) {
      if (tag[k] & 0x80000000u) c.load[tag[k] & 0x7FFFFFFFu] = (float)C[k];   // root: net load
      else c.elm[tag[k]] = (float)val[k];
    }
  }
}

// nets without RC nodes: load = their pins' caps, no wire delay
__global__ void __launch_bounds__(kThreads) rc_lumped_kernel(Topo t, const __grid_constant__ Batch B) {
  pdl_wait();
  pdl_launch();
  const CornerDev& c = B.c[blockIdx.y];
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= t.n_lumped) return;
  const uint32_t j = t.lumped_j[x];
  const uint32_t drv = t.net_drv[j];
  c.load[drv] = t.net_lumped[j];
  for (uint32_t k = t.sink_ptr[drv]; k < t.sink_ptr[drv + 1]; ++k) c.elm[k] = 0.f;
}

// ---- tier C: segmented prefix sums over ONE global preorder array of the
// large nets' nodes and over its Euler event sequence (layout in
// sta_internal.h).  Three launches per corner on a side stream, concurrent
// with tiers A and B:
//   tc_node_kernel   node caps C -> segmented inclusive sums Si (segment =
//                    net), stored (single pass);
//   tc_w_kernel      w(g) = R(g) Cdown(g), Cdown(g) = Si[end(g) - 1] - Si[g] +
//                    C(g), stored; net loads (a map over the nodes);
//   tc_event_kernel  event values +-w -> segmented inclusive sums H (single
//                    pass); elm(g) = H[enter(g)] written directly.
// (w was computed inside the event scan until r2: three dependent gathers
// per event at 114 registers, 2 blocks per SM: 60 us on C3's 2.2M events.)
// Each block scans its tile locally, publishes its segmented aggregate and
// takes its carry-in from its predecessors by a look-back over their
// AGGREGATES only (back to the nearest block holding a segment head), summed
// in a fixed order: the association never depends on timing, so the sums
// are bitwise reproducible.  Tiles are handed out by a ticket in block start
// order, so a block only ever waits for blocks that are already running.  A
// segmented scan never crosses a net: the sums stay small (no cancellation
// against other nets) and a net's Elmore delays need no offset.
// Block size of the tier-C launches (128-thread blocks that fit the slot of a
// retiring tier-A block measured slower: C3 RC phase 0.219 vs 0.186 ms).
#ifndef STA_TC_THREADS
#define STA_TC_THREADS 256
#endif
constexpr int kTcThreads = STA_TC_THREADS;
struct SegSum {
  double v;
  uint32_t f;   // a segment head inside
};
// (a then b): b restarts at a head
__device__ __forceinline__ SegSum seg_op(SegSum a, SegSum b) { return SegSum{b.f ? b.v : a.v + b.v, a.f | b.f}; }

// Block-wide exclusive segmented scan of one SegSum per thread (kTcThreads
// threads); *total receives the block's inclusive total.
__device__ __forceinline__ SegSum seg_block_excl(SegSum x, SegSum* s_w, SegSum* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SegSum inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    SegSum y{__shfl_up_sync(0xFFFFFFFFu, inc.v, o), __shfl_up_sync(0xFFFFFFFFu, inc.f, o)};
    if (lane >= o) inc = seg_op(y, inc);
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    SegSum a = lane < kTcThreads / 32 ? s_w[lane] : SegSum{0.0, 0u};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      SegSum y{__shfl_up_sync(0xFFFFFFFFu, a.v, o), __shfl_up_sync(0xFFFFFFFFu, a.f, o)};
      if (lane >= o) a = seg_op(y, a);
    }
    s_w[lane] = a;                               // inclusive over warps
  }
  __syncthreads();
  SegSum ex{__shfl_up_sync(0xFFFFFFFFu, inc.v, 1), __shfl_up_sync(0xFFFFFFFFu, inc.f, 1)};
  if (lane == 0) ex = SegSum{0.0, 0u};
  const SegSum r = w ? seg_op(s_w[w - 1], ex) : ex;
  *total = s_w[kTcThreads / 32 - 1];
  __syncthreads();
  return r;
}

constexpr int kTcPer = (int)(kTcTile / kTcThreads);   // consecutive elements per thread

#ifndef STA_TC_RELAXED
#define STA_TC_RELAXED 0
#endif
// per-scan block records in the scratch: aggregate[nb] (double), flag[nb] (u32
// {has head, epoch}: bit 31 = has head, bits 0..30 = epoch)
struct TcScan {
  double* agg;
  uint32_t* flag;
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Block b: publish the aggregate (the sum after its last head, or the whole
// tile), then return the carry-in of its elements before its first head: the
// fixed-order sum of the aggregates of b - 1, b - 2, ... down to and
// including the nearest block that holds a head.  Warp 0 looks back 32
// blocks per round trip.
__device__ double tc_lookback(const TcScan& sc, uint32_t b, SegSum tot, uint32_t ep) {
  __shared__ double s_carry;
  if (threadIdx.x == 0) {
    sc.agg[b] = tot.v;
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sc.flag + b), "r"((tot.f ? 0x80000000u : 0u) | ep)
                 : "memory");
  }
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double carry = 0.0;
    bool done = b == 0;
    for (int64_t p0 = (int64_t)b - 1; !done; p0 -= 32) {
      const int64_t p = p0 - lane;                  // lane 0 = nearest predecessor
      uint32_t f = 0x80000000u;                    // past block 0: a virtual head
      double v = 0.0;
      if (p >= 0) {
#if STA_TC_RELAXED
        // relaxed polling (no L1 invalidation per poll); the aggregate is read
        // from L2 after the flag returned (control dependency), like the records
        do {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(sc.flag + p) : "memory");
        } while ((f & 0x7FFFFFFFu) != ep);
#else
        do {
          f = ld_acquire_u32(sc.flag + p);
        } while ((f & 0x7FFFFFFFu) != ep);
#endif
        v = __ldcg(sc.agg + p);
      }
      const uint32_t heads = __ballot_sync(0xFFFFFFFFu, (f >> 31) != 0);
      const int stop = heads ? __ffs(heads) - 1 : 31;   // nearest head in this window
      // fixed-order sum of lanes 0..stop (nearest first), then into carry
      double x = lane <= stop ? v : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xFFFFFFFFu, x, o);
      carry += __shfl_sync(0xFFFFFFFFu, x, 0);
      done = heads != 0;
    }
    if (lane == 0) s_carry = carry;
  }
  __syncthreads();
  return s_carry;
}

__device__ __forceinline__ bool tc_head(uint32_t tag) { return tag != kNone && (tag & 0x80000000u); }

// tile of this block: handed out in block start order
__device__ __forceinline__ uint32_t tc_ticket(uint32_t* counter, uint32_t nb) {
  __shared__ uint32_t s_b;
  if (threadIdx.x == 0) s_b = atomicAdd(counter, 1u) % nb;   // nb tickets per update
  __syncthreads();
  return s_b;
}

#ifndef STA_TC_MINB
#define STA_TC_MINB 1
#endif
__global__ void __launch_bounds__(kTcThreads, STA_TC_MINB) tc_node_kernel(Topo t, const __grid_constant__ Batch B) {
  __shared__ SegSum s_w[32];
  pdl_wait();
  pdl_launch();
  const CornerDev& c = B.c[blockIdx.y];
  const uint32_t n = t.nCn, nb = tierC_blocks(n), nbe = tierC_blocks(2ull * n);
  double* Si = c.scratch;                                   // [nCn]
  const TcScan sc{c.scratch + n, reinterpret_cast<uint32_t*>(c.scratch + n + nb + nbe)};
  uint32_t* cnt = reinterpret_cast<uint32_t*>(c.scratch + n + nb + nbe) + nb + nbe;
  const uint32_t ep = __ldcg(c.epoch) & 0x7FFFFFFFu;
  const uint32_t b = tc_ticket(cnt, nb);
  const float* Cw = c.rc_vals[1];
  const uint32_t g0 = b * kTcTile + threadIdx.x * kTcPer;
  double v[kTcPer];
  uint32_t hd = 0;
  bool bad = false;
  uint4 nd[kTcPer];
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) nd[j] = g0 + j < n ? __ldg(t.tc_node + g0 + j) : make_uint4(0, kNone, 0, 0);
  float cw[kTcPer];
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) cw[j] = g0 + j < n ? Cw[nd[j].x] : 0.f;
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) {
    v[j] = 0.0;
    if (g0 + j < n) {
      bad |= bad_rc(0.f, cw[j]);
      v[j] = (double)cw[j] + (double)__uint_as_float(nd[j].w);
      if (tc_head(nd[j].y)) hd |= 1u << j;
    }
  }
  SegSum run{0.0, 0u};                       // thread-serial segmented inclusive run
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) {
    run = seg_op(run, SegSum{v[j], (hd >> j) & 1u});
    v[j] = run.v;
  }
  SegSum tot;
  SegSum ex = seg_block_excl(run, s_w, &tot);
  const double carry = tc_lookback(sc, b, tot, ep);
  if (!ex.f) ex.v += carry;                  // no head before this thread in the tile
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) {
    const bool before = (hd & ((2u << j) - 1u)) == 0;       // no head in this thread up to j
    if (g0 + j < n) Si[g0 + j] = before ? ex.v + v[j] : v[j];
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(c.err_flag, 1u);
}

// w(g) = R(g) Cdown(g) of every tier-C node, Cdown(g) = Si[end(g) - 1] - Si[g]
// + C(g) (a plain map over the nodes: high occupancy, one dependent gather);
// a net's root writes the net load instead (w = 0)
__global__ void __launch_bounds__(kThreads) tc_w_kernel(Topo t, const __grid_constant__ Batch B) {
  pdl_wait();
  pdl_launch();
  const CornerDev& c = B.c[blockIdx.y];
  const uint32_t n = t.nCn, g = blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (g < n) {
    const double* Si = c.scratch;
    double* w = c.scratch + tierC_scratch_scan(n);
    const uint4 nd = __ldg(t.tc_node + g);
    const float cw = c.rc_vals[1][nd.x], rr = c.rc_vals[0][nd.x];
    const double C = (double)cw + (double)__uint_as_float(nd.w);
    const double cd = __ldcg(Si + nd.z - 1) - __ldcg(Si + g) + C;
    double x = 0.0;
    if (tc_head(nd.y)) {
      c.load[nd.y & 0x7FFFFFFFu] = (float)cd;               // net load = Cdown(root)
    } else {
      bad = bad_rc(rr, 0.f);
      x = (double)rr * cd;
    }
    w[g] = x;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(c.err_flag, 1u);
}

// event values +-w(g) (enter / exit) -> segmented inclusive sums H; elm(g) =
// H at enter(g), written for the nodes of sinks
#ifndef STA_TC_EV_MINB
#define STA_TC_EV_MINB 4
#endif
__global__ void __launch_bounds__(kTcThreads, STA_TC_EV_MINB) tc_event_kernel(Topo t, const __grid_constant__ Batch B) {
  __shared__ SegSum s_w[32];
  pdl_wait();
  pdl_launch();
  const CornerDev& c = B.c[blockIdx.y];
  const uint32_t n = t.nCn, m = 2 * n, nbn = tierC_blocks(n), nb = tierC_blocks(m);
  const double* w = c.scratch + tierC_scratch_scan(n);
  const TcScan sc{c.scratch + n + nbn, reinterpret_cast<uint32_t*>(c.scratch + n + nbn + nb) + nbn};
  uint32_t* cnt = reinterpret_cast<uint32_t*>(c.scratch + n + nbn + nb) + nbn + nb + 1;
  const uint32_t ep = __ldcg(c.epoch) & 0x7FFFFFFFu;
  const uint32_t b = tc_ticket(cnt, nb);
  const uint32_t e0 = b * kTcTile + threadIdx.x * kTcPer;
  double v[kTcPer];
  uint32_t hd = 0;
  uint2 ev[kTcPer];
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) ev[j] = e0 + j < m ? __ldg(t.tc_ev + e0 + j) : make_uint2(0u, kNone);
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) v[j] = e0 + j < m ? __ldcg(w + (ev[j].x & 0x7FFFFFFFu)) : 0.0;
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) {
    if (ev[j].x >> 31) v[j] = -v[j];
    if (tc_head(ev[j].y)) hd |= 1u << j;                   // a net's events start at its root's enter
  }
  SegSum run{0.0, 0u};
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) {
    run = seg_op(run, SegSum{v[j], (hd >> j) & 1u});
    v[j] = run.v;
  }
  SegSum tot;
  SegSum ex = seg_block_excl(run, s_w, &tot);
  const double carry = tc_lookback(sc, b, tot, ep);
  if (!ex.f) ex.v += carry;
#pragma unroll
  for (int j = 0; j < kTcPer; ++j) {
    // elm(g) = H at enter(g) (exit events and Steiner / root nodes write nothing)
    const bool before = (hd & ((2u << j) - 1u)) == 0;
    const uint32_t tag = ev[j].y;
    if (tag != kNone && !(tag & 0x80000000u)) c.elm[tag] = (float)(before ? ex.v + v[j] : v[j]);
  }
}

// ------------------------------------------- a2-a5: propagation work units
// The forward and backward passes are lists of warp work units in
// dependency order (every unit depends only on units with a smaller index;
// layouts in sta_internal.h).  Two launchers run the same unit code:
//   * persistent (default): one cooperative grid of co-resident blocks; warp
//     w takes units w, w + W, ... in order.  All warps are resident, so the
//     smallest unfinished unit can always proceed: no deadlock, no barrier.
//     A unit waits only for the tagged words it reads, so stages overlap
//     wherever the graph allows, and a producer -> consumer hop is one L2
//     round trip.
//   * per stage (STA_STAGE_KERNELS=1): one launch per gate stage (PDL), one
//     warp per unit; the tags are then always valid on first read.
constexpr uint32_t kFull = 0xFFFFFFFFu;

// STA_TRACE: {start, ready (forward: before the inputs are polled), inputs loaded, end} of a unit
template <bool TRACE>
__device__ __forceinline__ void trace_unit(const CornerDev& c, size_t q, unsigned long long t0,
                                           unsigned long long t1, unsigned long long t2 = 0) {
  if (TRACE && (threadIdx.x & 31) == 0) {
    c.trace[4 * q] = t0;
    c.trace[4 * q + 1] = t1;
    c.trace[4 * q + 2] = t2 ? t2 : t1;
    c.trace[4 * q + 3] = gtimer();
  }
}

// undefined-safe slack: slack_L = RAT_L - AT_L, slack_E = AT_E - RAT_E, +inf
// if either side is undefined
__device__ __forceinline__ Q4 slack_of(const Q4& at, const Q4& r) {
  Q4 s;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool ok = fin(at.v[q]) && fin(r.v[q]);
    s.v[q] = ok ? (q < 2 ? __fsub_rn(at.v[q], r.v[q]) : __fsub_rn(r.v[q], at.v[q])) : CUDART_INF_F;
  }
  return s;
}

// required-time merge: early components take the max, late the min
__device__ __forceinline__ void combine(Q4& a, const Q4& b) {
  a.v[0] = fmaxf(a.v[0], b.v[0]);
  a.v[1] = fmaxf(a.v[1], b.v[1]);
  a.v[2] = fminf(a.v[2], b.v[2]);
  a.v[3] = fminf(a.v[3], b.v[3]);
}

// ---- forward: four lanes per fan-in term, lane = (term slot tl = lane / 4,
// output component q = lane % 4 = (el, orf)).  A unit is a run of pins of
// one stage with <= kFwdTerms terms (a pin is never split; a pin with more
// terms is a unit of its own, looped over by the warp).  A lane reads the
// one tagged record word its candidate needs -- (el, irf) of the source, irf
// by the term's sense -- spinning on its tags, applies the net hop of a sink
// input, looks up delay[orf] and slew[orf] (bit-identical to the backward's
// recomputation: same seg / interp calls on the same operands), and the first
// term of each pin merges its pin's candidates by shuffles and writes word q
// of the pin's record.  (A single "probe" lane polling first, to spare L2
// sectors while a warp runs ahead of the wavefront, measured slower once the
// units of a stage are ordered by readiness.)
// (Four lanes per term keep the per-lane dependent chain short: the forward
// wavefront's stage-to-stage latency is that chain.)
constexpr uint32_t kFwdTerms = kFwdUnitTerms;

// The lookup of delay[orf] / slew[orf] in two halves: the part that does not
// depend on the input arrival (table records, load-axis segments) runs before
// the lane waits for its producer, so only the slew-axis search and the
// interpolations remain on the critical path after the data arrives.
struct FwdTabs {
  Tab rd, rs;       // cell_rise / cell_fall, rise / fall transition of orf
  Seg cd, cc;       // their load-axis segments
  bool same;        // one axis template for both
};

__device__ __forceinline__ FwdTabs fwd_tabs(const float* __restrict__ L, uint32_t info, int orf, float ld) {
  FwdTabs f;
  const uint32_t tab = info >> 3;
  f.rd = tab_rec(L, tab + orf);
  f.rs = tab_rec(L, tab + 2 + orf);
  f.same = f.rs.ax == f.rd.ax;
  f.cd = seg(f.rd.ax + 24, ld);
  f.cc = f.same ? f.cd : seg(f.rs.ax + 24, ld);
  return f;
}

__device__ __forceinline__ void fwd_lane(const FwdTabs& f, int el, float a_in, float s_in, float& ca, float& cs,
                                         float& dl) {
  const Seg sd = seg(f.rd.ax, s_in);
  const Seg ss = f.same ? sd : seg(f.rs.ax, s_in);
  const float d = fmaxf(0.f, interp(f.rd, sd, f.cd));
  const float so = fmaxf(0.f, interp(f.rs, ss, f.cc));
  const bool ok = fin(a_in);
  const float undef = el ? -CUDART_INF_F : CUDART_INF_F;
  ca = ok ? __fadd_rn(a_in, d) : undef;
  cs = ok ? so : undef;
  dl = d;                                    // the backward's delay of this (el, irf -> orf)
}

__device__ __forceinline__ void merge_q(float& a, float b, int el) { a = el ? fmaxf(a, b) : fminf(a, b); }

// net hop driver -> sink of one component (net_hop): AT + elm, PERI slew
__device__ __forceinline__ void hop_q(float& a_in, float& s_in, float elm) {
  if (!fin(a_in)) return;
  const float imp = __fmul_rn(kLn9, elm);
  a_in = __fadd_rn(a_in, elm);
  s_in = __fsqrt_rn(__fmaf_rn(s_in, s_in, __fmul_rn(imp, imp)));
}

// RC results a term slot needs: {Elmore delay of its sink input, load of its
// pin}; under the Arnoldi model also the reduced model of the sink input
// (its net's time constants, the sink's residues)
template <bool ARN>
struct FwdRc {
  float elm, ld;
};
template <>
struct FwdRc<true> {
  float elm, ld;
  float4 lam, res;
};
template <bool ARN>
__device__ __forceinline__ FwdRc<ARN> fwd_rc(const CornerDev& c, const uint4& tr) {
  FwdRc<ARN> r{};
  if (tr.x < kHeavyMark) {                   // a term (not padding / seed / heavy marker)
    if (tr.y != kNone) {
      r.elm = __ldcg(c.elm + tr.y);
      if constexpr (ARN) {
        r.lam = __ldcg(c.arn_lam + tr.x);
        r.res = __ldcg(c.arn_res + tr.y);
      }
    }
    r.ld = __ldcg(c.load + tr.w);
  }
  return r;
}

// net hop of one component under the Arnoldi model (row f1): the reduced
// model's ramp response; an unstable / lumped net (lam.x < 0 or NaN) keeps
// the Elmore hop
__device__ __forceinline__ void arn_hop_q(float& a_in, float& s_in, float elm, const float4& lam, const float4& res) {
  if (!(lam.x >= 0.f)) {
    hop_q(a_in, s_in, elm);
    return;
  }
  if (!fin(a_in)) return;
  const float d = arn_delay(lam, res, s_in);
  const float so = arn_slew(lam, res, s_in);
  a_in = __fadd_rn(a_in, d);
  s_in = so;
}
// all four components (the backward's and the output gather's recomputation);
// slews only if wanted (undefined components keep undefined slews)
__device__ __forceinline__ void arn_net_hop(Q4& at, Q4& sl, float elm, const float4& lam, const float4& res,
                                            bool slews, Q4* dly = nullptr) {
  if (!(lam.x >= 0.f)) {
    if (dly) for (int q = 0; q < 4; ++q) dly->v[q] = elm;
    if (slews) net_hop(at, sl, elm);
    else hop_at(at, elm);
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool ok = fin(at.v[q]);
    const float d = ok ? arn_delay(lam, res, sl.v[q]) : 0.f;
    if (dly) dly->v[q] = d;
    if (slews) sl.v[q] = ok ? arn_slew(lam, res, sl.v[q]) : (q < 2 ? CUDART_INF_F : -CUDART_INF_F);
    at.v[q] = ok ? __fadd_rn(at.v[q], d) : at.v[q];
  }
}

// ---- row f4: -through hooks (the oracle's O15; Topo::thr_*).  At a
// through pin whose tag advances (thr_dst != kNone) this pass's arrivals are
// handed to the advanced tag's pass and are undefined here, and its required
// times are that pass's; where the tag is final the handed arrivals merge
// into its own and its required times are recorded for the earlier passes.
// Fan-in-free pins (seeds) take no forward hook, as in the oracle.
__device__ __forceinline__ float* thr_word(float4* base, const Topo& t, uint32_t pass, uint32_t sl, int q) {
  return reinterpret_cast<float*>(base + (size_t)pass * t.n_thr + sl) + q;
}
// component q of a pull pin's merged (arrival, slew), before it is stored
__device__ __forceinline__ void thr_pull_q(const Topo& t, const CornerDev& c, uint32_t v, int q, float& a, float& s) {
  const uint32_t sl = __ldg(t.thr_pull + v);
  if (sl == kNone) return;
  const bool early = q < 2;
  const uint32_t d = __ldg(t.thr_dst + sl);
  if (d != kNone) {                          // hand over (one writer per word in this pass)
    float* ha = thr_word(c.thr_hat, t, d, sl, q);
    float* hs = thr_word(c.thr_hsl, t, d, sl, q);
    *ha = early ? fminf(*ha, a) : fmaxf(*ha, a);
    *hs = early ? fminf(*hs, s) : fmaxf(*hs, s);
    a = s = early ? CUDART_INF_F : -CUDART_INF_F;
  } else {
    const float ha = *thr_word(c.thr_hat, t, t.thr_cur, sl, q), hs = *thr_word(c.thr_hsl, t, t.thr_cur, sl, q);
    a = early ? fminf(a, ha) : fmaxf(a, ha);
    s = early ? fminf(s, hs) : fmaxf(s, hs);
  }
}
// component q of a sink's arrival / slew (after its net hop); the handoff of
// an advancing sink's arrivals is thr_capture_kernel's
__device__ __forceinline__ void thr_sink_q(const Topo& t, const CornerDev& c, uint32_t k, int q, float& a, float& s) {
  const uint32_t sl = __ldg(t.thr_sink + k);
  if (sl == kNone) return;
  const bool early = q < 2;
  const uint32_t d = __ldg(t.thr_dst + sl);
  if (d != kNone) {
    a = s = early ? CUDART_INF_F : -CUDART_INF_F;
  } else {
    const float ha = *thr_word(c.thr_hat, t, t.thr_cur, sl, q), hs = *thr_word(c.thr_hsl, t, t.thr_cur, sl, q);
    a = early ? fminf(a, ha) : fmaxf(a, ha);
    s = early ? fminf(s, hs) : fmaxf(s, hs);
  }
}
__device__ __forceinline__ void thr_sink4(const Topo& t, const CornerDev& c, uint32_t k, Q4& a, Q4& s) {
#pragma unroll
  for (int q = 0; q < 4; ++q) thr_sink_q(t, c, k, q, a.v[q], s.v[q]);
}
// required times of a through slot sl (kNone: not a through pin)
__device__ __forceinline__ void thr_rat(const Topo& t, const CornerDev& c, uint32_t sl, Q4& r) {
  if (sl == kNone) return;
  const uint32_t d = __ldg(t.thr_dst + sl);
  if (d != kNone) r = to_q(c.thr_hrat[(size_t)d * t.n_thr + sl]);
  else c.thr_hrat[(size_t)t.thr_cur * t.n_thr + sl] = to_f4(r);
}

// forward unit u; tr = this lane's term slot of the unit, rc its RC results
// (loaded by the caller, software-pipelined one unit ahead)
// the record word a term lane reads: (el, irf) of its source
__device__ __forceinline__ const uint4* fwd_word(const CornerDev& c, const uint4& tr) {
  const uint32_t q = threadIdx.x & 3;
  const int el = (int)(q >> 1), orf = (int)(q & 1);
  return c.rec + 4 * (size_t)tr.x + (el * 2 + primary_irf(tr.z & 7u, orf));
}

// pre: this lane's record word loaded speculatively one unit early (valid
// if its tags match the epoch, else it is polled again)
template <bool TRACE, bool ARN, bool THR>
__device__ __forceinline__ void fwd_unit(const Topo& t, const CornerDev& c, const float* __restrict__ L,
                                         uint32_t ep, uint32_t u, const uint4& tr, FwdRc<ARN> rc,
                                         uint4 pre = make_uint4(0, 0, 0, 0)) {
  const uint32_t lane = threadIdx.x & 31, tl = lane >> 2, q = lane & 3;
  const int el = (int)(q >> 1), orf = (int)(q & 1);
  const float undef = el ? -CUDART_INF_F : CUDART_INF_F;
  unsigned long long t_start = 0, t_ready = 0, t_data = 0;
  if (TRACE && lane == 0) t_start = gtimer();
  const uint32_t kind = __shfl_sync(kFull, tr.x, 0);
  if (kind == kSeedMark) {                   // seeds: lane = (pin, q)
    if (tr.w != kNone) {
      const uint32_t v = tr.w;
      const uint32_t s = t.seed[v];
      float a = undef, sl = undef;
      if (s == kSeedClock) {                 // rising edge at 0, falling at T/2
        a = orf ? 0.5f * t.period : 0.f;
        sl = t.clock_slew;
      } else if (s != kNone) {
        a = reinterpret_cast<const float*>(t.pi_at + s)[q];
        sl = reinterpret_cast<const float*>(t.pi_slew + s)[q];
      }
      st_ll(c.rec + 4 * (size_t)v + q, a, sl, ep);
      reinterpret_cast<float*>(c.at4 + v)[q] = a;
    }
    trace_unit<TRACE>(c, u, t_start, t_start);
    return;
  }
  if (kind != kHeavyMark) {
    const bool item = tr.x != kNone;
    const uint32_t src = tr.x, info = tr.z, v = tr.w;
    const float elm = rc.elm, ld = rc.ld;
    const int irf = primary_irf(info & 7u, orf);
    const uint4* wp = c.rec + 4 * (size_t)src + (el * 2 + irf);
    if (TRACE && lane == 0) t_ready = gtimer();
    float ca = undef, cs = undef;
    if (item) {
      const FwdTabs f = fwd_tabs(L, info, orf, ld);   // before waiting for the producer
#if STA_FWD_RECPF
      uint4 w = pre;
      if (!ll_ok(w, ep)) w = spin_ll(wp, ep);
#else
      const uint4 w = spin_ll(wp, ep);
#endif
      if (TRACE) t_data = gtimer();
      float a_in = __uint_as_float(w.x), s_in = __uint_as_float(w.z);
      if (tr.y != kNone) {
        if constexpr (ARN) arn_hop_q(a_in, s_in, elm, rc.lam, rc.res);
        else hop_q(a_in, s_in, elm);
        if constexpr (THR) thr_sink_q(t, c, tr.y, el * 2 + irf, a_in, s_in);
      }
      float dl;
      fwd_lane(f, el, a_in, s_in, ca, cs, dl);
      reinterpret_cast<float*>(c.tdel + (size_t)kFwdTerms * u + tl)[q] = dl;
    }
    // merge the pin's terms into its first term's lanes (same q); a pin's
    // terms occupy consecutive slots
    // (log-step doubling over term slots; min / max are idempotent, so the
    // overlapping windows are harmless)
    const uint32_t peers = __match_any_sync(kFull, item ? v : kNone);
    const uint32_t head_tl = (uint32_t)(__ffs(peers) - 1) >> 2, end_tl = (uint32_t)(31 - __clz(peers)) >> 2;
#if STA_MERGE_BOUND
    // rounds: enough for the unit's longest run of terms of one pin
    const uint32_t nt = __reduce_max_sync(kFull, item ? (uint32_t)__popc(peers) >> 2 : 0u);
    for (uint32_t j = 1; j < nt; j <<= 1) {
#else
#pragma unroll
    for (uint32_t j = 1; j < kFwdTerms; j <<= 1) {
#endif
      const float oa = __shfl_down_sync(kFull, ca, 4 * j);
      const float os = __shfl_down_sync(kFull, cs, 4 * j);
      if (tl + j <= end_tl) {
        merge_q(ca, oa, el);
        merge_q(cs, os, el);
      }
    }
    if (item && tl == head_tl) {
      if constexpr (THR) thr_pull_q(t, c, v, (int)q, ca, cs);
      st_ll(c.rec + 4 * (size_t)v + q, ca, cs, ep);
      reinterpret_cast<float*>(c.at4 + v)[q] = ca;
    }
  } else {                                   // one pin with > kFwdTerms terms: warp loop
    const uint32_t v = __shfl_sync(kFull, tr.w, 0), e0 = __shfl_sync(kFull, tr.y, 0), nterms = __shfl_sync(kFull, tr.z, 0);
    const uint32_t dbase = __shfl_sync(kFull, tr.y, 4);   // slot 1: first delay slot
    const float ld = __ldcg(c.load + v);
    float ca = undef, cs = undef;
    for (uint32_t b = tl; b < nterms; b += kFwdTerms) {
      const uint32_t e = e0 + b;
      const uint32_t info = t.fi_info[e], h = t.fi_hop[e];
      const int irf = primary_irf(info & 7u, orf);
      const FwdTabs f = fwd_tabs(L, info, orf, ld);
      const uint4 w = spin_ll(c.rec + 4 * (size_t)t.fi_src[e] + (el * 2 + irf), ep);
      float a_in = __uint_as_float(w.x), s_in = __uint_as_float(w.z);
      if (h != kNone) {
        if constexpr (ARN)
          arn_hop_q(a_in, s_in, __ldcg(c.elm + h), __ldcg(c.arn_lam + t.fi_src[e]), __ldcg(c.arn_res + h));
        else hop_q(a_in, s_in, __ldcg(c.elm + h));
        if constexpr (THR) thr_sink_q(t, c, h, el * 2 + irf, a_in, s_in);
      }
      float oa, os, dl;
      fwd_lane(f, el, a_in, s_in, oa, os, dl);
      reinterpret_cast<float*>(c.tdel + dbase + b)[q] = dl;
      merge_q(ca, oa, el);
      merge_q(cs, os, el);
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      merge_q(ca, __shfl_xor_sync(kFull, ca, o), el);
      merge_q(cs, __shfl_xor_sync(kFull, cs, o), el);
    }
    if (tl == 0) {
      if constexpr (THR) thr_pull_q(t, c, v, (int)q, ca, cs);
      st_ll(c.rec + 4 * (size_t)v + q, ca, cs, ep);
      reinterpret_cast<float*>(c.at4 + v)[q] = ca;
    }
    t_ready = t_start;
  }
  if (TRACE) {                             // latest lane's data arrival
    const uint32_t lo = (uint32_t)t_data, hi = (uint32_t)(t_data >> 32);
    const uint32_t mh = __reduce_max_sync(kFull, hi);
    const uint32_t ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    t_data = ((unsigned long long)mh << 32) | ml;
  }
  trace_unit<TRACE>(c, u, t_start, t_ready, t_data);
}

// unroll factor of the persistent forward's unit loop (3: the pipeline's
// three-deep register rotation tr <- nx <- nnx becomes renaming)
#ifndef STA_FWD_UNROLL
#define STA_FWD_UNROLL 1
#endif
#define STA_PRAGMA(x) _Pragma(#x)
#define STA_UNROLL(n) STA_PRAGMA(unroll n)
template <bool SMEM_LUT, bool TRACE, bool ARN, bool THR, int NT>
__device__ __forceinline__ void fwd_persistent_body(const Topo& t, const Batch& B) {
  stage_luts<SMEM_LUT>(B, kNone);
  // warp gw serves corner gw % K and walks its unit list with stride Wc
  const uint32_t K = B.K, gw = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  const uint32_t Wc = gridDim.x * (NT / 32) / K;
  if (gw >= Wc * K) return;
  const CornerDev& c = B.c[gw % K];
  const float* L = lut_of<SMEM_LUT>(c);
  const uint32_t ep = epoch_of(c);
  const uint32_t tl = (threadIdx.x & 31) >> 2;
  uint32_t u = gw / K;
#if STA_FWD_PF
  // software pipeline: term slots two units ahead, the RC results (Elmore
  // delay of the input hop, load of the pin) one unit ahead, so neither
  // round trip is exposed when a unit starts
  const uint4 pad = make_uint4(kNone, kNone, 0, kNone);
  uint4 tr = u < t.n_fwu ? __ldg(t.fterm + (size_t)kFwdTerms * u + tl) : pad;
  uint4 nx = u + Wc < t.n_fwu ? __ldg(t.fterm + (size_t)kFwdTerms * (u + Wc) + tl) : pad;
  FwdRc<ARN> rc = fwd_rc<ARN>(c, tr);
#if STA_FWD_RECPF
  // the record words of the next unit, loaded speculatively one unit early:
  // in the wide stages the producers are long done and the unit starts with
  // its data in registers; in the narrow ones the word is stale and re-polled
  uint4 rec = make_uint4(0, 0, 0, 0);
#endif
  STA_UNROLL(STA_FWD_UNROLL)
  for (; u < t.n_fwu; u += Wc) {
    const uint4 nnx = u + 2 * Wc < t.n_fwu ? __ldg(t.fterm + (size_t)kFwdTerms * (u + 2 * Wc) + tl) : pad;
    const FwdRc<ARN> nrc = fwd_rc<ARN>(c, nx);         // nx arrived during the previous unit
#if STA_FWD_RECPF
    const uint4 nrec = nx.x < kHeavyMark ? ld_ll(fwd_word(c, nx)) : make_uint4(0, 0, 0, 0);
    fwd_unit<TRACE, ARN, THR>(t, c, L, ep, u, tr, rc, rec);
    rec = nrec;
#else
    fwd_unit<TRACE, ARN, THR>(t, c, L, ep, u, tr, rc);
#endif
    tr = nx;
    nx = nnx;
    rc = nrc;
  }
#else
  // software pipeline: the next unit's term slot is in flight while a unit
  // waits for its producers
  uint4 nx = u < t.n_fwu ? __ldg(t.fterm + (size_t)kFwdTerms * u + tl) : make_uint4(0, 0, 0, 0);
  for (; u < t.n_fwu; u += Wc) {
    const uint4 tr = nx;
    if (u + Wc < t.n_fwu) nx = __ldg(t.fterm + (size_t)kFwdTerms * (u + Wc) + tl);   // prefetch the next unit
    fwd_unit<TRACE, ARN, THR>(t, c, L, ep, u, tr, fwd_rc<ARN>(c, tr));
  }
#endif
}

template <bool SMEM_LUT, bool TRACE>
__global__ void __launch_bounds__(kFwdThreads, kFwdMinBlocks) fwd_persistent_kernel(Topo t,
                                                                                   const __grid_constant__ Batch B) {
  fwd_persistent_body<SMEM_LUT, TRACE, false, false, kFwdThreads>(t, B);
}

// the Arnoldi-model instantiation (row f1): its hop solver needs registers,
// so fewer warps per block
constexpr int kFwdArnThreads = 512;
// the Arnoldi model (row f1) and / or -through hooks (row f4): 512 threads,
// more registers per thread
template <bool SMEM_LUT, bool ARN, bool THR>
__global__ void __launch_bounds__(kFwdArnThreads, 1) fwd_persistent_ext_kernel(Topo t, const __grid_constant__ Batch B) {
  fwd_persistent_body<SMEM_LUT, false, ARN, THR, kFwdArnThreads>(t, B);
}

// units [u0, u1) of one gate stage, one warp each; grid.y = corner
template <bool SMEM_LUT, bool TRACE>
__global__ void __launch_bounds__(kThreads) fwd_stage_kernel(Topo t, const __grid_constant__ Batch B, uint32_t u0,
                                                             uint32_t u1) {
  stage_luts<SMEM_LUT>(B, blockIdx.y);
  const CornerDev& c = B.c[blockIdx.y];
  const float* L = lut_of<SMEM_LUT>(c);
  const uint32_t u = u0 + blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const uint4 tr = u < u1 ? __ldg(t.fterm + (size_t)kFwdTerms * u + ((threadIdx.x & 31) >> 2)) : make_uint4(0, 0, 0, 0);
  pdl_wait();
  pdl_launch();
  if (u >= u1) return;
  fwd_unit<TRACE, false, false>(t, c, L, epoch_of(c), u, tr, fwd_rc<false>(c, tr));
}

// ---- backward: one lane per sink / pin (all four components in the lane)
// Cell arc u -> w, backward: RAT(u, el, irf) combines
// RAT(w, el, orf) - d(el, irf -> orf) over the output edges orf whose input
// edge irf (by the sense) has a defined arrival -- exactly the pairs the
// forward used; late min, early max.  we / wl: w's tagged required-time words
// (early, late); d: the term's delays stored by the forward, (el, orf) order
// (the very values the forward added: no recomputation).
__device__ __forceinline__ void bwd_arc(const Q4& a, uint32_t info, const float4& d4, const uint4& we,
                                        const uint4& wl, Q4& r) {
  const uint32_t sense = info & 7u;
  const float d[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
  for (int orf = 0; orf < 2; ++orf) {
    const int irf = primary_irf(sense, orf);
#pragma unroll
    for (int el = 0; el < 2; ++el) {
      // (selects, not dynamic register-array indices: those go to local memory)
      const bool ok = fin(irf ? a.v[el * 2 + 1] : a.v[el * 2]);
      const uint4& w = el ? wl : we;
      const float cand = __fsub_rn(__uint_as_float(orf ? w.z : w.x), d[el * 2 + orf]);
      float& r0 = r.v[el * 2];
      float& r1 = r.v[el * 2 + 1];
      const float m0 = el ? fminf(r0, cand) : fmaxf(r0, cand);
      const float m1 = el ? fminf(r1, cand) : fmaxf(r1, cand);
      r0 = ok && irf == 0 ? m0 : r0;
      r1 = ok && irf == 1 ? m1 : r1;
    }
  }
}

// row f4: the net arc into sink k is disabled by case analysis (bit 31 of the
// CSR start in its record; such a sink is constant, so its fan-out count is 0)
__device__ __forceinline__ bool sink_killed(const Topo& t, uint32_t k) {
  return (int)__ldg(&t.sinkfo[2 * (size_t)k].z) < 0;
}

// does the arc use some defined input component (otherwise nothing to wait for)
__device__ __forceinline__ bool arc_live(uint32_t info, const Q4& a) {
  // input edges the sense uses: r by POS / NEG / RISE_EDGE, f by POS / NEG /
  // FALL_EDGE; sense 7 (an arc disabled by case analysis, row f4) uses none
  const uint32_t sense = info & 7u;
  const bool r_used = (0x0Bu >> sense) & 1u, f_used = (0x13u >> sense) & 1u;
  return (r_used && (fin(a.v[0]) || fin(a.v[2]))) || (f_used && (fin(a.v[1]) || fin(a.v[3])));
}

// Endpoint seeds: PO: RAT_L = T - out_max, RAT_E =
// -out_min (po_seed, precomputed in fp32); check: RAT_L = T - setup(slew_L(D),
// clock slew), RAT_E = hold(slew_E(D), clock slew), only where the arrival
// exists.  chk / po: from the pin's fan-out record.
__device__ __forceinline__ void seed4(const Topo& t, const float* __restrict__ L, uint32_t chk, uint32_t po,
                                      const Q4& a, const Q4& s, Q4& r, uint32_t e = kNone) {
  Q4 sd = undef_rat();
  if (po != kNone) {
    const float4 ps = __ldg(t.po_seed + po);
    sd.v[0] = ps.x;
    sd.v[1] = ps.y;
    sd.v[2] = ps.z;
    sd.v[3] = ps.w;
  }
  if (chk != kNone) {
#pragma unroll
    for (int rf = 0; rf < 2; ++rf) {
      if (fin(a.v[2 + rf]))
        sd.v[2 + rf] = fminf(sd.v[2 + rf], __fsub_rn(t.period, lut(L, chk + rf, s.v[2 + rf], t.clock_slew)));
      if (fin(a.v[rf])) sd.v[rf] = fmaxf(sd.v[rf], lut(L, chk + 2 + rf, s.v[rf], t.clock_slew));
    }
  }
  if (t.ep_ovr && e != kNone) {              // row f4: this tag's exception at the endpoint
    const uint4 o = __ldg(t.ep_ovr + e);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t mode = q < 2 ? o.z : o.x;
      const float v = __uint_as_float(q < 2 ? o.w : o.y);
      if (!fin(sd.v[q])) continue;           // no base seed of this kind
      sd.v[q] = mode == 2 ? (q < 2 ? -CUDART_INF_F : CUDART_INF_F) : mode == 1 ? v : __fadd_rn(sd.v[q], v);
    }
  }
  combine(r, sd);
}

// Loads of the two inline fan-out terms of a pin's fan-out record (fa, fb),
// issued as soon as the record is known so the round trips overlap the
// pin's own loads; the tag check comes later (bwd_pin).
struct FoPre {
  float4 d0, d1;             // the terms' delays
  uint4 e0, l0;              // required-time words (early, late) of the first term's pin (a
                             // non-unate arc's two terms share it; other second pins load later)
};

__device__ __forceinline__ FoPre bwd_pre(const CornerDev& c, const uint4& fa, const uint4& fb, uint32_t ep) {
  const uint4 ok = make_uint4(0, ep, 0, ep);
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  FoPre p{z, z, ok, ok};
  if (fa.w == kNone && fa.y) {
    p.d0 = __ldcg(c.tdel + (fb.y >> 3));
    p.e0 = ld_ll(c.rat_ll + 2 * (size_t)fb.x);
    p.l0 = ld_ll(c.rat_ll + 2 * (size_t)fb.x + 1);
    if (fa.y > 1) p.d1 = __ldcg(c.tdel + (fb.w >> 3));
  }
  return p;
}

__device__ __forceinline__ void spin_pair(const uint4* p, uint4& we, uint4& wl, uint32_t ep) {
  for (uint32_t ns = kMinSleepNs; !ll_ok(we, ep) || !ll_ok(wl, ep);) {
    backoff(ns);
    if (!ll_ok(we, ep)) we = ld_ll(p);
    if (!ll_ok(wl, ep)) wl = ld_ll(p + 1);
  }
}

// Required times of an input pin (arrival a, slew s) from its endpoint seed
// and its cell fan-out; fan-out record (fa, fb), inline terms' loads in
// flight (p); further terms from the CSR (dst_csr / info_csr).
__device__ __forceinline__ void bwd_pin(const Topo& t, const CornerDev& c, const float* __restrict__ L, uint32_t ep,
                                        const uint4& fa, const uint4& fb, FoPre p,
                                        const uint32_t* __restrict__ dst_csr, const uint32_t* __restrict__ info_csr,
                                        const Q4& a, const Q4& s, Q4& r) {
  const uint32_t nfo = fa.y;
  uint32_t f = 0;
  if (fa.w != kNone) {
    seed4(t, L, fb.x, fb.y, a, s, r, fa.w);
  } else if (nfo) {
    const bool l0 = arc_live(fb.y, a), l1 = nfo > 1 && arc_live(fb.w, a), shared = fb.z == fb.x;
    if (l0 || (l1 && shared)) spin_pair(c.rat_ll + 2 * (size_t)fb.x, p.e0, p.l0, ep);
    if (l0) bwd_arc(a, fb.y, p.d0, p.e0, p.l0, r);
    if (l1) {
      if (shared) {
        bwd_arc(a, fb.w, p.d1, p.e0, p.l0, r);
      } else {
        const uint4* pw = c.rat_ll + 2 * (size_t)fb.z;
        uint4 we = ld_ll(pw), wl = ld_ll(pw + 1);
        spin_pair(pw, we, wl, ep);
        bwd_arc(a, fb.w, p.d1, we, wl, r);
      }
    }
    f = nfo < 2 ? nfo : 2;
  }
  for (; f < nfo; ++f) {
    const uint32_t info = __ldg(info_csr + fa.z + f);
    if (!arc_live(info, a)) continue;
    const uint32_t w2 = __ldg(dst_csr + fa.z + f);
    const uint4* pw = c.rat_ll + 2 * (size_t)w2;
    uint4 we = ld_ll(pw), wl = ld_ll(pw + 1);
    const float4 d4 = __ldcg(c.tdel + (info >> 3));
    spin_pair(pw, we, wl, ep);
    bwd_arc(a, info, d4, we, wl, r);
  }
}

__device__ __forceinline__ void write_ep(const CornerDev& c, uint32_t e, const Q4& s) {
  c.ep_ws[e] = make_float2(fminf(s.v[2], s.v[3]), fminf(s.v[0], s.v[1]));   // {setup, hold}
}

// Backward unit: {k0, k1, heavy slot, 0}: a tile of sinks [k0, k1) of one
// stage's drivers (lane = sink), or {x0, x1, 0, 1}: sink-less pull pins
// [x0, x1) (lane = pin).  A sink lane: the sink's arrival / slew from its
// driver's record and net hop, its endpoint seed, its cell fan-out (spinning
// on the fan-out pins' tagged required-time words), rat / slack, then the
// candidate of its driver through the net arc; the first lane of each driver
// merges its sinks from the warp's shared-memory slots and finishes the
// driver (own seed, direct cell fan-out, rat / slack, the tagged required-
// time words).  A driver with more than kTile sinks spans tiles of its own
// (heavy slot): they combine with ordered-int atomics and the last tile
// finishes the driver.
// fan-out record of the lane's sink in tile unit ud (the caller loads it one
// unit ahead)
struct SinkFo {
  uint4 a, b;
};
__device__ __forceinline__ SinkFo bwd_fo(const Topo& t, const uint4& ud) {
  SinkFo f{make_uint4(kNone, 0, 0, kNone), make_uint4(kNone, 0, kNone, 0)};
  const uint32_t k = ud.x + (threadIdx.x & 31);
  if (ud.w != 1 && k < ud.y) {
    f.a = __ldg(t.sinkfo + 2 * (size_t)k);
    f.b = __ldg(t.sinkfo + 2 * (size_t)k + 1);
  }
  return f;
}

template <bool TRACE, bool ARN, bool THR>
__device__ __forceinline__ void bwd_unit(const Topo& t, const CornerDev& c, const float* __restrict__ L,
                                         uint32_t ep, uint32_t u, const uint4& ud, const SinkFo& fo) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long t_start = 0, t_ready = 0, t_data = 0;
  if (TRACE && lane == 0) t_start = gtimer();
  uint32_t v = kNone;
  Q4 at_v = undef_at(), sl_v = undef_at(), acc = undef_rat();
  bool head = false;
  uint4 pa = make_uint4(0, 0, 0, kNone), pb = make_uint4(kNone, 0, kNone, 0);   // driver's fan-out record
  if (ud.w != 1) {                           // tile of sinks (light or heavy)
    const uint32_t k = ud.x + lane;
    const bool act = k < ud.y;
    const uint4 fa = fo.a, fb = fo.b;
    v = act ? fa.x & 0x7FFFFFFFu : kNone;
    const bool drv_work = (fa.x >> 31) != 0;   // the driver has an endpoint / direct fan-out
    const uint32_t vp = __shfl_up_sync(kFull, v, 1);
    head = act && (lane == 0 || vp != v);    // first lane of its driver
    if (act) {
      const float elm = __ldcg(c.elm + k);
      at_v = load_at(c, v);
      if (head && drv_work) {
        pa = __ldg(t.pullfo + 2 * (size_t)v);
        pb = __ldg(t.pullfo + 2 * (size_t)v + 1);
      }
      FoPre pre = bwd_pre(c, fa, fb, ep);
      if (TRACE) t_ready = gtimer();
      // wait for the first fan-out pin's required times BEFORE anything needs
      // the sink's own arrival: the arrival / Elmore loads issued above then
      // complete during the wait instead of adding a round trip of their own
      // (a pin's required-time words are always written, live arc or not)
#if STA_BWD_SPIN_FIRST
      if (fa.w == kNone && fa.y) spin_pair(c.rat_ll + 2 * (size_t)fb.x, pre.e0, pre.l0, ep);
#endif
      Q4 a = at_v, s = sl_v, r = undef_rat();
      Q4 nd{{elm, elm, elm, elm}};           // the net arc's delay per component
      if constexpr (ARN) {                   // row f1: the driver's slews drive the reduced model
        s = load_slew(c, v);
        arn_net_hop(a, s, elm, __ldcg(c.arn_lam + v), __ldcg(c.arn_res + k), fa.w != kNone, &nd);
      } else if (fa.w != kNone) {            // endpoint sink: its slews feed the check tables
        s = load_slew(c, v);
        net_hop(a, s, elm);                  // the sink's own arrival / slew
      } else {
        hop_at(a, elm);                      // the sink's own arrival (slews unused)
      }
      if ((int)fa.z < 0) a = undef_at();    // row f4: net arc disabled by case analysis
      uint32_t tsl = kNone;
      if constexpr (THR) {                   // row f4: a -through sink
        tsl = __ldg(t.thr_sink + k);
        if (tsl != kNone) thr_sink4(t, c, k, a, s);
      }
      bwd_pin(t, c, L, ep, fa, fb, pre, t.sfo_dst, t.sfo_info, a, s, r);
      if constexpr (THR) thr_rat(t, c, tsl, r);
      if (TRACE) t_data = gtimer();
      c.rat[t.NP + k] = to_f4(r);
      const Q4 sk = slack_of(a, r);
      c.slack[t.NP + k] = to_f4(sk);
      if (fa.w != kNone) write_ep(c, fa.w, sk);
#pragma unroll
      for (int q = 0; q < 4; ++q)            // through the net arc (edges the forward used)
        if (fin(at_v.v[q]) && (int)fa.z >= 0) acc.v[q] = __fsub_rn(r.v[q], nd.v[q]);
    }
    // merge the sinks of each driver (contiguous lanes) into its first lane:
    // log-step doubling (max / min are idempotent: overlapping windows are
    // harmless); a loop over the run measured 18% of the kernel's
    // instructions on heavy tiles
    const uint32_t peers = __match_any_sync(kFull, v);
    const uint32_t end = 31 - __clz(peers);
#if STA_MERGE_BOUND
    // rounds: enough for the tile's longest run of sinks of one driver
    const uint32_t run = __reduce_max_sync(kFull, act ? (uint32_t)__popc(peers) : 0u);
    for (uint32_t o = 1; o < run; o <<= 1) {
#else
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
#endif
      Q4 b;
#pragma unroll
      for (int q = 0; q < 4; ++q) b.v[q] = __shfl_down_sync(kFull, acc.v[q], o);
      if (lane + o <= end) combine(acc, b);
    }
    if (ud.z != kNone) {                      // heavy driver: every lane is v
      // partial of this tile, then a release increment of the driver's tile
      // counter (one atomic per tile); the last tile combines all partials
      if (lane == 0) c.heavy_part[ud.w - 2] = to_f4(acc);
      __syncwarp();
      uint32_t done = 0;
      if (lane == 0)
        asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(done) : "l"(c.heavy_cnt + ud.z) : "memory");
      const uint32_t nch = __ldg(t.heavy_nchunk + ud.z);
      head = false;
      if (__shfl_sync(kFull, done, 0) + 1 == nch) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const uint32_t b0 = __ldg(t.heavy_base + ud.z);
        acc = undef_rat();
#pragma unroll 4
        for (uint32_t x = lane; x < nch; x += 32) combine(acc, to_q(__ldcg(c.heavy_part + b0 + x)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          Q4 b;
#pragma unroll
          for (int q = 0; q < 4; ++q) b.v[q] = __shfl_xor_sync(kFull, acc.v[q], o);
          combine(acc, b);
        }
        if (lane == 0) c.heavy_cnt[ud.z] = 0;   // self-reset for the next update
        head = lane == 0;
      }
    }
  } else {
    v = ud.x + lane;                         // sink-less pins [x0, x1)
    head = v < ud.y;
    if (head) {
      at_v = load_at(c, v);
      pa = __ldg(t.pullfo + 2 * (size_t)v);
      pb = __ldg(t.pullfo + 2 * (size_t)v + 1);
    }
  }
  // finish driver / pin v
  if (head) {
    const FoPre pre = bwd_pre(c, pa, pb, ep);
    if (pa.w != kNone) sl_v = load_slew(c, v);   // the pin's own endpoint seed needs its slews
    bwd_pin(t, c, L, ep, pa, pb, pre, t.pfo_dst, t.pfo_info, at_v, sl_v, acc);
    if constexpr (THR) thr_rat(t, c, __ldg(t.thr_pull + v), acc);
    const Q4 sp = slack_of(at_v, acc);
    c.slack[v] = to_f4(sp);
    if (pa.w != kNone) write_ep(c, pa.w, sp);
    st_ll(c.rat_ll + 2 * (size_t)v, acc.v[0], acc.v[1], ep);
    st_ll(c.rat_ll + 2 * (size_t)v + 1, acc.v[2], acc.v[3], ep);
  }
  if (TRACE) {                             // latest lane's fan-out data
    const uint32_t lo = (uint32_t)t_data, hi = (uint32_t)(t_data >> 32);
    const uint32_t mh = __reduce_max_sync(kFull, hi);
    const uint32_t ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    t_data = ((unsigned long long)mh << 32) | ml;
    t_ready = __shfl_sync(kFull, t_ready, 0);
  }
  trace_unit<TRACE>(c, (size_t)t.n_fwu + u, t_start, t_ready ? t_ready : t_start, t_data);
}

template <bool SMEM_LUT, bool TRACE, bool ARN, bool THR, int NT>
__device__ __forceinline__ void bwd_persistent_body(const Topo& t, const Batch& B) {
  stage_luts<SMEM_LUT>(B, kNone);
  const uint32_t K = B.K, gw = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  const uint32_t W = gridDim.x * (NT / 32) / K;    // warps of this corner
  if (gw >= W * K) return;
  const CornerDev& c = B.c[gw % K];
  const float* L = lut_of<SMEM_LUT>(c);
  const uint32_t ep = epoch_of(c);
  uint32_t u = gw / K;
  // software pipeline: the unit record two units ahead, the sinks' fan-out
  // records one unit ahead are in flight while a unit waits for its producers
  // (issued at the start of the previous unit, so they overlap its work)
  const uint4 none = make_uint4(0, 0, 0, 1);
  uint4 ud = u < t.n_bwu_static ? __ldg(t.bwu + u) : none;
  SinkFo fo = bwd_fo(t, ud);
  uint4 nx = u + W < t.n_bwu_static ? __ldg(t.bwu + u + W) : none;
  // Stage-0 units (no dependencies among them, all inputs produced by the
  // static part) go to whichever warp is free, by ticket: warps finish their
  // static units at different times, and a static split of the tail would
  // leave the stragglers' share waiting for them.
  const uint32_t ns = t.n_bwu_static, lane = threadIdx.x & 31;
#if STA_BWD_PIPE == 0
  // (variant: no fan-out record prefetch, fewer registers)
  for (;;) {
    if (u >= ns) {
      uint32_t x = 0;
      if (lane == 0) x = atomicAdd(c.red_cnt + 1, 1u);
      u = ns + __shfl_sync(kFull, x, 0);
      if (u >= t.n_bwu) break;
      ud = __ldg(t.bwu + u);
      bwd_unit<TRACE, ARN, THR>(t, c, L, ep, u, ud, bwd_fo(t, ud));
      continue;
    }
    const uint4 nu = u + W < ns ? __ldg(t.bwu + u + W) : none;
    bwd_unit<TRACE, ARN, THR>(t, c, L, ep, u, ud, bwd_fo(t, ud));
    u += W;
    ud = nu;
  }
  (void)fo;
  (void)nx;
#elif STA_BWD_PIPE == 2
  // The sinks' fan-out records of the warp's next unit are streamed into a
  // per-warp shared-memory buffer by a TMA bulk copy (one 32 B record per
  // sink, the unit's sinks are contiguous: <= 1 KB), issued when the current
  // unit starts; the unit reads its own records from shared memory.  No
  // register holds a prefetched record across the unit body.
  const uint32_t wib = threadIdx.x >> 5;
  uint4* fbuf = reinterpret_cast<uint4*>(s_dyn + B.smem_f4) + wib * 64;
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_dyn + B.smem_f4 + (NT / 32) * 64) + wib;
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  uint32_t phase = 0;
  auto issue = [&](const uint4& un) {
    if (lane == 0) {
      // the warp's generic-proxy reads of the buffer (take) are ordered
      // before the bulk copy's async-proxy writes into it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t n = (un.w != 1 && un.y > un.x) ? (un.y - un.x) * 32u : 0u;
      mbar_expect_tx(bar, n);
      if (n) bulk_g2s(fbuf, t.sinkfo + 2 * (size_t)un.x, n, bar);
    }
  };
  auto take = [&](const uint4& un) {       // this unit's records, then the buffer is free
    mbar_wait(bar, phase);
    phase ^= 1u;
    SinkFo f{make_uint4(kNone, 0, 0, kNone), make_uint4(kNone, 0, kNone, 0)};
    if (un.w != 1 && un.x + lane < un.y) {
      f.a = fbuf[2 * lane];
      f.b = fbuf[2 * lane + 1];
    }
    // every lane's reads complete (the values are in registers) before lane 0
    // lets the next bulk copy overwrite the buffer
    asm volatile("" ::"r"(f.a.x), "r"(f.a.y), "r"(f.a.z), "r"(f.a.w), "r"(f.b.x), "r"(f.b.y), "r"(f.b.z),
                 "r"(f.b.w) : "memory");
    __syncwarp();
    return f;
  };
  (void)fo;
  bool dyn = u >= ns;
  if (!dyn) issue(ud);
  if (dyn) {                                 // no static unit: first ticket
    uint32_t x = 0;
    if (lane == 0) x = atomicAdd(c.red_cnt + 1, 1u);
    u = ns + __shfl_sync(kFull, x, 0);
    ud = u < t.n_bwu ? __ldg(t.bwu + u) : none;
  }
  while (u < t.n_bwu) {
    uint4 nnx = none;
    uint32_t un = 0;
    SinkFo cf;
    if (dyn) {
      uint32_t xn = 0;
      if (lane == 0) xn = atomicAdd(c.red_cnt + 1, 1u);
      un = ns + __shfl_sync(kFull, xn, 0);
      nx = un < t.n_bwu ? __ldg(t.bwu + un) : none;
      cf = bwd_fo(t, ud);
    } else {
      cf = take(ud);
      issue(nx);                             // the next unit's records stream in meanwhile
      if (u + 2 * W < ns) nnx = __ldg(t.bwu + u + 2 * W);
    }
    bwd_unit<TRACE, ARN, THR>(t, c, L, ep, u, ud, cf);
    if (dyn) {
      u = un;
      ud = nx;
    } else if (u + W < ns) {
      u += W;
      ud = nx;
      nx = nnx;
    } else {                                 // static part done: first ticket
      dyn = true;
      uint32_t x = 0;
      if (lane == 0) x = atomicAdd(c.red_cnt + 1, 1u);
      u = ns + __shfl_sync(kFull, x, 0);
      ud = u < t.n_bwu ? __ldg(t.bwu + u) : none;
    }
  }
#else
  // one call site of bwd_unit (a second inlined copy of the large unit body
  // measured 40% slower: instruction-cache pressure)
  bool dyn = u >= ns;
  if (dyn) {                                 // no static unit: first ticket
    uint32_t x = 0;
    if (lane == 0) x = atomicAdd(c.red_cnt + 1, 1u);
    u = ns + __shfl_sync(kFull, x, 0);
    ud = u < t.n_bwu ? __ldg(t.bwu + u) : none;
    fo = bwd_fo(t, ud);
  }
  while (u < t.n_bwu) {
    SinkFo nfo = fo;
    uint4 nnx = none;
    uint32_t un = 0;
    if (dyn) {
      // the next ticket and its unit record are fetched before this unit
      // runs, so the atomic and the record load overlap its work
      uint32_t xn = 0;
      if (lane == 0) xn = atomicAdd(c.red_cnt + 1, 1u);
      un = ns + __shfl_sync(kFull, xn, 0);
      nx = un < t.n_bwu ? __ldg(t.bwu + un) : none;
    } else {
      nfo = bwd_fo(t, nx);                   // next unit's fan-out records (its record arrived)
      if (u + 2 * W < ns) nnx = __ldg(t.bwu + u + 2 * W);
    }
    bwd_unit<TRACE, ARN, THR>(t, c, L, ep, u, ud, fo);
    if (dyn) {
      u = un;
      ud = nx;
      fo = bwd_fo(t, ud);
    } else if (u + W < ns) {
      u += W;
      ud = nx;
      fo = nfo;
      nx = nnx;
    } else {                                 // static part done: first ticket
      dyn = true;
      uint32_t x = 0;
      if (lane == 0) x = atomicAdd(c.red_cnt + 1, 1u);
      u = ns + __shfl_sync(kFull, x, 0);
      ud = u < t.n_bwu ? __ldg(t.bwu + u) : none;
      fo = bwd_fo(t, ud);
    }
  }
#endif
}

template <bool SMEM_LUT, bool TRACE>
__global__ void __launch_bounds__(kBwdThreads, kBwdMinBlocks) bwd_persistent_kernel(Topo t,
                                                                                   const __grid_constant__ Batch B) {
  bwd_persistent_body<SMEM_LUT, TRACE, false, false, kBwdThreads>(t, B);
}

constexpr int kBwdArnThreads = 512;
template <bool SMEM_LUT, bool ARN, bool THR>
__global__ void __launch_bounds__(kBwdArnThreads, 1) bwd_persistent_ext_kernel(Topo t, const __grid_constant__ Batch B) {
  bwd_persistent_body<SMEM_LUT, false, ARN, THR, kBwdArnThreads>(t, B);
}

// -through hooks with the Elmore model: the propagation kernels' own block
// sizes (the hooks add a few registers, not the Arnoldi solver's)
template <bool SMEM_LUT>
__global__ void __launch_bounds__(kFwdThreads, kFwdMinBlocks) fwd_persistent_thr_kernel(Topo t,
                                                                                       const __grid_constant__ Batch B) {
  fwd_persistent_body<SMEM_LUT, false, false, true, kFwdThreads>(t, B);
}
template <bool SMEM_LUT>
__global__ void __launch_bounds__(kBwdThreads, kBwdMinBlocks) bwd_persistent_thr_kernel(Topo t,
                                                                                       const __grid_constant__ Batch B) {
  bwd_persistent_body<SMEM_LUT, false, false, true, kBwdThreads>(t, B);
}

template <bool SMEM_LUT, bool TRACE>
__global__ void __launch_bounds__(kThreads) bwd_stage_kernel(Topo t, const __grid_constant__ Batch B, uint32_t u0,
                                                             uint32_t u1) {
  stage_luts<SMEM_LUT>(B, blockIdx.y);
  const CornerDev& c = B.c[blockIdx.y];
  const float* L = lut_of<SMEM_LUT>(c);
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t u = u0 + blockIdx.x * (kThreads / 32) + warp;
  const uint4 ud = u < u1 ? __ldg(t.bwu + u) : make_uint4(0, 0, 0, 0);
  const SinkFo fo = bwd_fo(t, ud);
  pdl_wait();
  pdl_launch();
  if (u >= u1) return;
  bwd_unit<TRACE, false, false>(t, c, L, epoch_of(c), u, ud, fo);
}

// ------------------------------------------------------- a5: WNS / TNS
// kRedBlocks blocks with a fixed endpoint range each, fixed-shape trees and a
// fixed-shape final combine by the last block: bitwise reproducible.
// Fixed-shape block tree: min of the two w lanes, sum of the two t lanes.
__device__ __forceinline__ void block_tree(float (*s_w)[kThreads], double (*s_t)[kThreads]) {
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s_w[0][threadIdx.x] = fminf(s_w[0][threadIdx.x], s_w[0][threadIdx.x + o]);
      s_w[1][threadIdx.x] = fminf(s_w[1][threadIdx.x], s_w[1][threadIdx.x + o]);
      s_t[0][threadIdx.x] += s_t[0][threadIdx.x + o];
      s_t[1][threadIdx.x] += s_t[1][threadIdx.x + o];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) reduce_kernel(Topo t, const __grid_constant__ Batch B) {
  constexpr int kU = 4;                      // loads in flight per thread
  __shared__ double s_t[2][kThreads];
  __shared__ float s_w[2][kThreads];
  __shared__ bool last;
  pdl_wait();
  pdl_launch();
  const CornerDev& c = B.c[blockIdx.y];
  const uint32_t n = t.n_ep;
  const uint32_t lo = (uint32_t)((uint64_t)n * blockIdx.x / gridDim.x);
  const uint32_t hi = (uint32_t)((uint64_t)n * (blockIdx.x + 1) / gridDim.x);
  float ws = CUDART_INF_F, wh = CUDART_INF_F;
  double ts = 0.0, th = 0.0;
  for (uint32_t e0 = lo + threadIdx.x; e0 < hi; e0 += kU * blockDim.x) {
    float2 x[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const uint32_t e = e0 + q * blockDim.x;
      x[q] = e < hi ? __ldcg(c.ep_ws + e) : make_float2(CUDART_INF_F, CUDART_INF_F);
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      ws = fminf(ws, x[q].x);
      wh = fminf(wh, x[q].y);
      if (x[q].x < 0.f) ts += (double)x[q].x;
      if (x[q].y < 0.f) th += (double)x[q].y;
    }
  }
  s_w[0][threadIdx.x] = ws; s_w[1][threadIdx.x] = wh;
  s_t[0][threadIdx.x] = ts; s_t[1][threadIdx.x] = th;
  block_tree(s_w, s_t);
  if (threadIdx.x == 0) {
    double* p = c.red_part + 4 * blockIdx.x;
    p[0] = s_w[0][0]; p[1] = s_t[0][0]; p[2] = s_w[1][0]; p[3] = s_t[1][0];
    __threadfence();
    last = atomicAdd(c.red_cnt, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // final combine of the block partials: fixed lanes, fixed tree
  ws = CUDART_INF_F; wh = CUDART_INF_F; ts = 0.0; th = 0.0;
  for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    const double2 p = __ldcg(reinterpret_cast<const double2*>(c.red_part) + 2 * b);
    const double2 q = __ldcg(reinterpret_cast<const double2*>(c.red_part) + 2 * b + 1);
    ws = fminf(ws, (float)p.x); ts += p.y;
    wh = fminf(wh, (float)q.x); th += q.y;
  }
  s_w[0][threadIdx.x] = ws; s_w[1][threadIdx.x] = wh;
  s_t[0][threadIdx.x] = ts; s_t[1][threadIdx.x] = th;
  block_tree(s_w, s_t);
  if (threadIdx.x == 0) {
    c.res[0] = s_w[0][0]; c.res[1] = s_t[0][0]; c.res[2] = s_w[1][0]; c.res[3] = s_t[1][0];
    c.red_cnt[0] = 0;                        // self-reset for the next update
    c.red_cnt[1] = 0;                        // backward tail ticket
    const uint32_t e = *c.epoch + 1;         // the next update's record tag (never 0)
    *c.epoch = e ? e : 1;
  }
}

// ----------------------------------------------------- outputs / setup
// what: 0 at, 1 slew, 2 rat, 3 slack, in user pin order; sink arrivals and
// slews are recomputed from their drivers exactly as the kernels do.
// row f4: fold this tag's results into the merged arrays, internal order
// (pin i: its record read once for arrival and slew; a sink's driver record
// is shared by its neighbours in the sink order)
// row f4 -through: every pass's handed arrivals / slews undefined (start of an update)
__global__ void thr_reset_kernel(Topo t, const __grid_constant__ Batch B, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const CornerDev& c = B.c[blockIdx.y];
  const float4 u = make_float4(CUDART_INF_F, CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
  c.thr_hat[i] = u;
  c.thr_hsl[i] = u;
}
// after this pass's forward: its arrivals / slews at the through sinks where
// its tag advances, handed to the advanced pass (recomputed from the driver
// exactly as the kernels do)
__global__ void thr_capture_kernel(Topo t, const __grid_constant__ Batch B) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= t.n_thr_sk) return;
  const CornerDev& c = B.c[blockIdx.y];
  const uint2 e = t.thr_sk[x];
  const uint32_t d = t.thr_dst[e.y];
  if (d == kNone) return;
  const uint32_t k = e.x, dv = t.sink_drv[k];
  Q4 at, sl;
  load_rec(c, dv, at, sl);
  if (t.net_model == 1) arn_net_hop(at, sl, c.elm[k], c.arn_lam[dv], c.arn_res[k], true);
  else net_hop(at, sl, c.elm[k]);
  if (sink_killed(t, k)) at = sl = undef_at();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float* ha = thr_word(c.thr_hat, t, d, e.y, q);
    float* hs = thr_word(c.thr_hsl, t, d, e.y, q);
    *ha = q < 2 ? fminf(*ha, at.v[q]) : fmaxf(*ha, at.v[q]);
    *hs = q < 2 ? fminf(*hs, sl.v[q]) : fmaxf(*hs, sl.v[q]);
  }
}
// the next record epoch (after a forward-only pass)
__global__ void bump_epoch_kernel(const __grid_constant__ Batch B) {
  const CornerDev& c = B.c[threadIdx.x];
  if (threadIdx.x >= B.K) return;
  const uint32_t e = *c.epoch + 1;
  *c.epoch = e ? e : 1;
}

__global__ void merge_tag_kernel(Topo t, CornerDev c, int first) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < t.n_ep) {
    const float2 w = c.ep_ws[i];
    if (first) c.m_ep_ws[i] = w;
    else {
      const float2 m = c.m_ep_ws[i];
      c.m_ep_ws[i] = make_float2(fminf(m.x, w.x), fminf(m.y, w.y));
    }
  }
  const size_t Pi = (size_t)t.NP + t.NS;
  if (i >= Pi) return;
  Q4 at, sl;
  float4 rt;
  if (i < t.NP) {
    load_rec(c, i, at, sl);
    const uint4 e = __ldcg(c.rat_ll + 2 * (size_t)i), l = __ldcg(c.rat_ll + 2 * (size_t)i + 1);
    rt = make_float4(__uint_as_float(e.x), __uint_as_float(e.z), __uint_as_float(l.x), __uint_as_float(l.z));
  } else {
    const uint32_t k = i - t.NP, dv = t.sink_drv[k];
    load_rec(c, dv, at, sl);
    if (t.net_model == 1) arn_net_hop(at, sl, c.elm[k], c.arn_lam[dv], c.arn_res[k], true);
    else net_hop(at, sl, c.elm[k]);
    if (sink_killed(t, k)) at = sl = undef_at();
    if (t.thr_sink) thr_sink4(t, c, k, at, sl);
    rt = c.rat[i];
  }
  const float4 v[4] = {to_f4(at), to_f4(sl), rt, c.slack[i]};
  // a pin this tag does not reach (no arrival, no required time, no slack)
  // leaves the merged arrays as they are: skip their read-modify-write
  if (!first && !fin(at.v[0]) && !fin(at.v[1]) && !fin(at.v[2]) && !fin(at.v[3]) && !fin(rt.x) && !fin(rt.y) &&
      !fin(rt.z) && !fin(rt.w) && !fin(v[3].x) && !fin(v[3].y) && !fin(v[3].z) && !fin(v[3].w))
    return;
#pragma unroll
  for (int what = 0; what < 4; ++what) {
    float4* m = c.m_pin + (size_t)what * Pi + i;
    if (first) {
      *m = v[what];
      continue;
    }
    const float4 o = *m, x = v[what];
    // early components: AT / slew min, RAT max; late: AT / slew max, RAT min; slack min
    if (what < 2) *m = make_float4(fminf(o.x, x.x), fminf(o.y, x.y), fmaxf(o.z, x.z), fmaxf(o.w, x.w));
    else if (what == 2) *m = make_float4(fmaxf(o.x, x.x), fmaxf(o.y, x.y), fminf(o.z, x.z), fminf(o.w, x.w));
    else *m = make_float4(fminf(o.x, x.x), fminf(o.y, x.y), fminf(o.z, x.z), fminf(o.w, x.w));
  }
}

__global__ void gather_pins_kernel(Topo t, CornerDev c, int what, float4* __restrict__ dst) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= t.P) return;
  if (c.m_pin) {                             // exceptions: the results merged over tags
    dst[p] = c.m_pin[(size_t)what * ((size_t)t.NP + t.NS) + t.int_of_user[p]];
    return;
  }
  const uint32_t i = t.int_of_user[p];
  if (what == 3) {
    dst[p] = c.slack[i];
    return;
  }
  if (what == 2) {                           // pull pins: tagged words {(el, r), (el, f)}
    if (i >= t.NP) {
      dst[p] = c.rat[i];
      return;
    }
    const uint4 e = __ldcg(c.rat_ll + 2 * (size_t)i), l = __ldcg(c.rat_ll + 2 * (size_t)i + 1);
    dst[p] = make_float4(__uint_as_float(e.x), __uint_as_float(e.z), __uint_as_float(l.x), __uint_as_float(l.z));
    return;
  }
  if (i < t.NP) {
    Q4 at, sl;
    load_rec(c, i, at, sl);
    dst[p] = to_f4(what == 0 ? at : sl);
    return;
  }
  const uint32_t k = i - t.NP;
  Q4 at, sl;
  load_rec(c, t.sink_drv[k], at, sl);
  if (t.net_model == 1) arn_net_hop(at, sl, c.elm[k], c.arn_lam[t.sink_drv[k]], c.arn_res[k], true);
  else net_hop(at, sl, c.elm[k]);
  if (sink_killed(t, k)) at = sl = undef_at();
  dst[p] = to_f4(what == 0 ? at : sl);
}

__global__ void gather_rc_kernel(Topo t, CornerDev c, float* net_load, float* pin_elm) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (net_load && p < t.N) net_load[p] = c.load[t.drv_of_net[p]];
  if (pin_elm && p < t.P) {
    const uint32_t i = t.int_of_user[p];
    pin_elm[p] = i >= t.NP ? c.elm[i - t.NP] : 0.f;
  }
}

__global__ void init_corner_kernel(CornerDev c, uint32_t n_heavy) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_heavy) c.heavy_cnt[i] = 0;
  if (i == 0) {
    c.red_cnt[0] = 0;
    c.red_cnt[1] = 0;
    *c.err_flag = 0;
    *c.epoch = 1;
  }
}

inline uint32_t blocks(uint64_t n, uint32_t th = kThreads) { return (uint32_t)((n + th - 1) / th); }

// launch with programmatic dependent launch enabled
template <class K, class... A>
cudaError_t pdl_launch_smem(K kernel, dim3 grid, uint32_t block, size_t smem, cudaStream_t s, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  // the stream's priority as an explicit launch attribute, so that it
  // survives graph capture (tier-C RC runs beside the small-net RC kernel)
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = prio;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <class K, class... A>
cudaError_t pdl_launch_kernel(K kernel, dim3 grid, uint32_t block, cudaStream_t s, A... args) {
  return pdl_launch_smem(kernel, grid, block, 0, s, args...);
}

// ------------------------------------------------ f3: top-k path report
// SURVEY.md §8(f) row 3; PAPER.md:187-190 ("top-k path reports ... top-k,
// per-endpoint report limit, and slack-less-than thresholds ... flattened
// CSR-based path pin arrays with slacks").  Same definition as the oracle's
// O10 (readings P1-P4 in DESIGN.md): the m = min(nworst, k) first partial
// paths into every (pull pin, transition), gate stage by gate stage, each
// extending a partial path of a fan-in term's source by the delays the update
// used (the term's stored cell delay, plus the Elmore delay of its net hop),
// in the order (arrival: late descending / early ascending, predecessor pin
// id, predecessor transition, predecessor rank).  The sums are the
// forward's own fp32 additions, so the first path into a pin has exactly
// the pin's arrival.  Net sinks stay implicit (pull-through): a sink's lists
// are its driver's lists plus its Elmore delay.
__device__ __forceinline__ bool path_better(bool late, float a1, uint32_t p1, uint32_t r1, float a2, uint32_t p2,
                                            uint32_t r2) {
  if (a1 != a2) return late ? a1 > a2 : a1 < a2;
  if (p1 != p2) return p1 < p2;
  return r1 < r2;                            // (transition << 31 | rank)
}

constexpr uint32_t kPathMaxTerms = 48;       // terms merged with per-term heads (more: rescans)

__global__ void __launch_bounds__(kThreads) path_dp_kernel(Topo t, CornerDev c, PathArgs pa, uint32_t v0,
                                                           uint32_t v1) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t v = v0 + (x >> 1), rf = x & 1u;
  if (v >= v1) return;
  const bool late = pa.mode == 0;
  const uint32_t el = late ? 1u : 0u, m = pa.m;
  PathEnt* out = pa.lists + ((size_t)v * 2 + rf) * m;
  const uint32_t e0 = pa.fi_p[v], e1 = pa.fi_p[v + 1];
  if (e0 == e1) {                            // startpoint (stage 0): its own arrival
    const float a = reinterpret_cast<const float*>(c.at4 + v)[el * 2 + rf];
    const bool ok = pa.uoi[v] != kNone && fin(a);
    if (ok) out[0] = PathEnt{a, kNone, 0u};
    pa.cnt[(size_t)v * 2 + rf] = ok ? 1 : 0;
    return;
  }
  // per term: the source list (its length and input edge), the added delay,
  // the predecessor's user pin id; merged by heads
  const uint32_t nt = e1 - e0;
  uint8_t head[kPathMaxTerms];
  uint32_t n = 0;
  uint32_t prev_p = 0, prev_r = 0;
  float prev_a = 0.f;
  for (; n < m; ++n) {
    bool found = false;
    float ba = 0.f;
    uint32_t bp = 0, br = 0, bt = 0, brank = 0, birf = 0;
    for (uint32_t q = 0; q < nt; ++q) {
      const uint32_t e = e0 + q;
      const uint32_t info = __ldg(t.fi_info + e), src = __ldg(t.fi_src + e), hop = __ldg(t.fi_hop + e);
      const uint32_t irf = (uint32_t)primary_irf(info & 7u, (int)rf);
      const uint32_t len = pa.cnt[(size_t)src * 2 + irf];
      // the term's first entry not yet taken: its head, or (many terms) the
      // first entry after the previous pick in the merge order
      uint32_t j = 0;
      const uint32_t pred = pa.uoi[hop != kNone ? t.NP + hop : src];
      const float dl = reinterpret_cast<const float*>(c.tdel + __ldg(pa.fi_slot + e))[el * 2 + rf];
      const float em = hop != kNone ? __ldcg(c.elm + hop) : 0.f;
      const PathEnt* ls = pa.lists + ((size_t)src * 2 + irf) * m;
      auto cand_a = [&](uint32_t jj) {
        const float a0 = ls[jj].a;
        return __fadd_rn(hop != kNone ? __fadd_rn(a0, em) : a0, dl);
      };
      if (nt <= kPathMaxTerms) {
        j = n == 0 ? 0u : head[q];
      } else {
        while (j < len && n && !path_better(late, prev_a, prev_p, prev_r, cand_a(j), pred, (irf << 31) | j)) ++j;
      }
      if (j >= len) continue;
      const float a = cand_a(j);
      const uint32_t r = (irf << 31) | j;
      if (!found || path_better(late, a, pred, r, ba, bp, br)) {
        found = true;
        ba = a; bp = pred; br = r; bt = e; brank = j; birf = irf;
      }
    }
    if (n == 0 && nt <= kPathMaxTerms)
      for (uint32_t q = 0; q < nt; ++q) head[q] = 0;
    if (!found) break;
    out[n] = PathEnt{ba, bt, (birf << 31) | brank};
    if (nt <= kPathMaxTerms) head[bt - e0]++;
    prev_a = ba; prev_p = bp; prev_r = br;
  }
  pa.cnt[(size_t)v * 2 + rf] = (uint8_t)n;
}

// per endpoint: its own seeds (the check / output delay),
// then its candidate paths: the two transitions' lists merged by slack
// (ties: rise first, then rank), at most m; key = (orderable slack, user id)
__device__ __forceinline__ uint32_t ordered_bits(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(kThreads) path_ep_kernel(Topo t, CornerDev c, PathArgs pa) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= t.n_ep) return;
  const bool late = pa.mode == 0;
  const uint32_t el = late ? 1u : 0u, m = pa.m;
  const uint32_t i = pa.ep_int[x], pu = pa.uoi[i];
  const bool sink = i >= t.NP;
  const uint32_t src = sink ? __ldg(t.sink_drv + (i - t.NP)) : i;
  const float em = sink ? __ldcg(c.elm + (i - t.NP)) : 0.f;
  // the endpoint's arrival / slew (its own, or its driver's through the net hop)
  Q4 at, sl;
  load_rec(c, src, at, sl);
  if (sink) net_hop(at, sl, em);
  const EpRec er = t.ep[x];
  Q4 sd = undef_rat();
  seed4(t, c.lut, er.chk_tab, er.po, at, sl, sd);
  const float S[2] = {sd.v[el * 2], sd.v[el * 2 + 1]};
  uint32_t h0 = 0, h1 = 0;
  const bool dead = sink && sink_killed(t, i - t.NP);   // case analysis: no path into the endpoint
  const uint32_t n0 = fin(S[0]) && !dead ? pa.cnt[(size_t)src * 2] : 0;
  const uint32_t n1 = fin(S[1]) && !dead ? pa.cnt[(size_t)src * 2 + 1] : 0;
  auto slack_of_e = [&](uint32_t rf, uint32_t j) {
    const float a0 = pa.lists[((size_t)src * 2 + rf) * m + j].a;
    const float a = sink ? __fadd_rn(a0, em) : a0;
    return late ? __fsub_rn(S[rf], a) : __fsub_rn(a, S[rf]);
  };
  for (uint32_t n = 0; n < m; ++n) {
    const size_t o = (size_t)x * m + n;
    const bool has0 = h0 < n0, has1 = h1 < n1;
    if (!has0 && !has1) {
      pa.cand_key[o] = ~0ull;
      pa.cand_ref[o] = kNone;
      continue;
    }
    const float s0 = has0 ? slack_of_e(0, h0) : 0.f, s1 = has1 ? slack_of_e(1, h1) : 0.f;
    const bool take0 = has0 && (!has1 || s0 <= s1);
    const float sl_ = take0 ? s0 : s1;
    const uint32_t rf = take0 ? 0u : 1u, j = take0 ? h0++ : h1++;
    pa.cand_key[o] = ((unsigned long long)ordered_bits(sl_) << 32) | pu;
    pa.cand_ref[o] = x | 0u;
    pa.cand_sub[o] = (rf << 31) | j;
    pa.cand_slack[o] = sl_;
  }
}

// selected path s (sorted position s): its length, then its pins
__device__ __forceinline__ uint32_t path_walk(const Topo& t, const CornerDev& c, const PathArgs& pa, uint32_t s,
                                              uint32_t* pins, uint8_t* rfs, float* ats, uint32_t at_end) {
  const uint32_t ref = pa.sorted_ref[s];
  const uint32_t sub = pa.sorted_sub[s];
  const uint32_t i = pa.ep_int[ref];
  uint32_t rf = sub >> 31, j = sub & 0x7FFFFFFFu, len = 0;
  const uint32_t m = pa.m;
  const bool late = pa.mode == 0;
  const uint32_t el = late ? 1u : 0u;
  uint32_t v = i >= t.NP ? __ldg(t.sink_drv + (i - t.NP)) : i;
  auto put = [&](uint32_t pin, uint32_t r, float a) {
    if (pins) {
      pins[at_end - 1 - len] = pin;
      rfs[at_end - 1 - len] = (uint8_t)r;
      ats[at_end - 1 - len] = a;
    }
    ++len;
  };
  if (i >= t.NP) {                           // the endpoint sink, then its driver
    const float a = __fadd_rn(pa.lists[((size_t)v * 2 + rf) * m + j].a, __ldcg(c.elm + (i - t.NP)));
    put(pa.uoi[i], rf, a);
  }
  for (;;) {
    const PathEnt en = pa.lists[((size_t)v * 2 + rf) * m + j];
    put(pa.uoi[v], rf, en.a);
    if (en.term == kNone) break;             // startpoint
    const uint32_t e = en.term, src = __ldg(t.fi_src + e), hop = __ldg(t.fi_hop + e);
    const uint32_t irf = en.rr >> 31, jj = en.rr & 0x7FFFFFFFu;
    if (hop != kNone)                        // the input sink of the term
      put(pa.uoi[t.NP + hop], irf,
          __fadd_rn(pa.lists[((size_t)src * 2 + irf) * m + jj].a, __ldcg(c.elm + hop)));
    v = src;
    rf = irf;
    j = jj;
  }
  (void)el;
  return len;
}

__global__ void __launch_bounds__(kThreads) path_len_kernel(Topo t, CornerDev c, PathArgs pa, uint32_t n_sel) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_sel) pa.path_ptr[s] = path_walk(t, c, pa, s, nullptr, nullptr, nullptr, 0);
}

__global__ void __launch_bounds__(kThreads) path_fill_kernel(Topo t, CornerDev c, PathArgs pa, uint32_t n_sel) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sel) return;
  path_walk(t, c, pa, s, pa.path_pin, pa.path_rf, pa.path_at, pa.path_ptr[s + 1]);
  pa.path_slack[s] = pa.sorted_slack[s];
  pa.path_ep[s] = pa.uoi[pa.ep_int[pa.sorted_ref[s]]];
}

__global__ void set_ptrs_kernel(const float** dst, const float* a, const float* b) {
  dst[0] = a;
  dst[1] = b;
}

}  // namespace

uint32_t rc_warp_grid() {
  int dev = 0, sms = 0, nb = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, rc_warp_kernel, kThreads, 0);
  cudaGetLastError();
  return (uint32_t)std::max(nb, 1) * (uint32_t)std::max(sms, 1);
}

cudaError_t launch_rc(const Topo& t, const Batch& b, uint32_t wgrid, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  const uint32_t K = b.K;
  if (t.n_wtiles && e == cudaSuccess) {
#if STA_RCW_PERSIST
    // 3/4 of the co-resident warps, shared by the K corners (the tier-C
    // launches on the side stream need room beside it), at most one tile per warp
    const uint32_t g = std::max<uint32_t>(1, std::min<uint32_t>(wgrid * 3 / 4 / K, blocks(32ull * t.n_wtiles)));
#else
    const uint32_t g = blocks(32ull * ((t.n_wtiles + kRcwTiles - 1) / kRcwTiles));
#endif
    e = pdl_launch_kernel(rc_warp_kernel, dim3(g, K), kThreads, s, t, b);
  }
  if (t.n_btiles && e == cudaSuccess) e = pdl_launch_kernel(rc_block_kernel, dim3(t.n_btiles, K), kThreads, s, t, b);
  if (t.n_lumped && e == cudaSuccess) e = pdl_launch_kernel(rc_lumped_kernel, dim3(blocks(t.n_lumped), K), kThreads, s, t, b);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_rc_tierC(const Topo& t, const Batch& b, cudaStream_t s) {
  if (!t.nC) return cudaSuccess;
  const uint32_t K = b.K;
  cudaError_t e = pdl_launch_kernel(tc_node_kernel, dim3(tierC_blocks(t.nCn), K), kTcThreads, s, t, b);
  if (e == cudaSuccess) e = pdl_launch_kernel(tc_w_kernel, dim3(blocks(t.nCn), K), kThreads, s, t, b);
  if (e == cudaSuccess) e = pdl_launch_kernel(tc_event_kernel, dim3(tierC_blocks(2ull * t.nCn), K), kTcThreads, s, t, b);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_fwd_stage(const Topo& t, const Batch& b, uint32_t u0, uint32_t u1, cudaStream_t s) {
  if (u1 <= u0) return cudaSuccess;
  const dim3 g(blocks(32ull * (u1 - u0)), b.K);
  if (b.smem_f4) return pdl_launch_smem(fwd_stage_kernel<true, false>, g, kThreads, 16ull * b.smem_f4, s, t, b, u0, u1);
  return pdl_launch_smem(fwd_stage_kernel<false, false>, g, kThreads, 0, s, t, b, u0, u1);
}

cudaError_t launch_bwd_stage(const Topo& t, const Batch& b, uint32_t u0, uint32_t u1, cudaStream_t s) {
  if (u1 <= u0) return cudaSuccess;
  const dim3 g(blocks(32ull * (u1 - u0)), b.K);
  if (b.smem_f4) return pdl_launch_smem(bwd_stage_kernel<true, false>, g, kThreads, 16ull * b.smem_f4, s, t, b, u0, u1);
  return pdl_launch_smem(bwd_stage_kernel<false, false>, g, kThreads, 0, s, t, b, u0, u1);
}

cudaError_t launch_reduce(const Topo& t, const Batch& b, cudaStream_t s) {
  return pdl_launch_kernel(reduce_kernel, dim3((uint32_t)kRedBlocks, b.K), kThreads, s, t, b);
}

cudaError_t launch_gather_pins(const Topo& t, const CornerDev& c, int what, float4* dst, cudaStream_t s) {
  if (t.P) gather_pins_kernel<<<blocks(t.P), kThreads, 0, s>>>(t, c, what, dst);
  return cudaGetLastError();
}

cudaError_t launch_merge_tag(const Topo& t, const CornerDev& c, int first, cudaStream_t s) {
  const uint64_t pi = (uint64_t)t.NP + t.NS;
  const uint64_t n = pi > t.n_ep ? pi : t.n_ep;
  if (n) merge_tag_kernel<<<blocks(n), kThreads, 0, s>>>(t, c, first);
  return cudaGetLastError();
}

cudaError_t launch_thr_reset(const Topo& t, const Batch& b, uint32_t n_tags, cudaStream_t s) {
  const uint64_t n = (uint64_t)n_tags * t.n_thr;
  if (n) thr_reset_kernel<<<dim3(blocks(n), b.K), kThreads, 0, s>>>(t, b, (uint32_t)n);
  return cudaGetLastError();
}

cudaError_t launch_thr_capture(const Topo& t, const Batch& b, cudaStream_t s) {
  if (t.n_thr_sk) thr_capture_kernel<<<dim3(blocks(t.n_thr_sk), b.K), kThreads, 0, s>>>(t, b);
  return cudaGetLastError();
}

cudaError_t launch_bump_epoch(const Batch& b, cudaStream_t s) {
  bump_epoch_kernel<<<1, kMaxBatch, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_gather_rc(const Topo& t, const CornerDev& c, float* net_load, float* pin_elm, cudaStream_t s) {
  const uint32_t n = t.N > t.P ? t.N : t.P;
  if (n) gather_rc_kernel<<<blocks(n), kThreads, 0, s>>>(t, c, net_load, pin_elm);
  return cudaGetLastError();
}

namespace {
__global__ void path_iota(uint32_t* x, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}
__global__ void path_gather(PathArgs pa, const uint32_t* idx, uint32_t n, uint32_t* ref, uint32_t* sub, float* sl,
                            const unsigned long long* keys, float slack_lt, uint32_t* count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t j = idx[i];
  ref[i] = pa.cand_ref[j];
  sub[i] = pa.cand_sub[j];
  sl[i] = pa.cand_slack[j];
  if (keys[i] != ~0ull && pa.cand_slack[j] < slack_lt) atomicAdd(count, 1u);
}
}  // namespace

cudaError_t run_path_report(const Topo& t, const CornerDev& c, PathArgs pa, const uint32_t* stage_ptr, uint32_t S,
                            uint32_t k, float slack_lt, uint32_t cap_pins, uint32_t* n_paths, uint32_t* n_pins,
                            bool* fits, cudaStream_t s) {
  *n_paths = *n_pins = 0;
  *fits = true;
  for (uint32_t st = 0; st < S; ++st) {       // gate stages in order
    const uint32_t v0 = stage_ptr[st], v1 = stage_ptr[st + 1];
    if (v1 > v0) path_dp_kernel<<<blocks(2ull * (v1 - v0)), kThreads, 0, s>>>(t, c, pa, v0, v1);
  }
  const uint32_t n = t.n_ep * pa.m;
  if (t.n_ep) path_ep_kernel<<<blocks(t.n_ep), kThreads, 0, s>>>(t, c, pa);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || n == 0) return e;
  // report order: stable radix sort of the candidates (per endpoint they are
  // already in order) by (slack, endpoint user id)
  std::vector<void*> tmp;
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s) != cudaSuccess) return nullptr;
    tmp.push_back(p);
    return p;
  };
  auto done = [&](cudaError_t r) {
    for (void* p : tmp) cudaFreeAsync(p, s);
    return r;
  };
  auto* idx_in = static_cast<uint32_t*>(alloc(4ull * n));
  auto* idx_out = static_cast<uint32_t*>(alloc(4ull * n));
  auto* key_out = static_cast<unsigned long long*>(alloc(8ull * n));
  auto* ref = static_cast<uint32_t*>(alloc(4ull * n));
  auto* sub = static_cast<uint32_t*>(alloc(4ull * n));
  auto* sl = static_cast<float*>(alloc(4ull * n));
  auto* cnt = static_cast<uint32_t*>(alloc(8));
  if (!idx_in || !idx_out || !key_out || !ref || !sub || !sl || !cnt) return done(cudaErrorMemoryAllocation);
  path_iota<<<blocks(n), kThreads, 0, s>>>(idx_in, n);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, pa.cand_key, key_out, idx_in, idx_out, (int)n, 0, 64, s);
  void* tsort = alloc(tb);
  if (!tsort) return done(cudaErrorMemoryAllocation);
  if ((e = cub::DeviceRadixSort::SortPairs(tsort, tb, pa.cand_key, key_out, idx_in, idx_out, (int)n, 0, 64, s)) !=
      cudaSuccess)
    return done(e);
  cudaMemsetAsync(cnt, 0, 8, s);
  path_gather<<<blocks(n), kThreads, 0, s>>>(pa, idx_out, n, ref, sub, sl, key_out, slack_lt, cnt);
  uint32_t n_ok = 0;
  cudaMemcpyAsync(&n_ok, cnt, 4, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);
  const uint32_t n_sel = std::min(n_ok, k);
  *n_paths = n_sel;
  if (!n_sel) return done(cudaSuccess);
  pa.sorted_ref = ref;
  pa.sorted_sub = sub;
  pa.sorted_slack = sl;
  path_len_kernel<<<blocks(n_sel), kThreads, 0, s>>>(t, c, pa, n_sel);
  cudaMemsetAsync(pa.path_ptr + n_sel, 0, 4, s);
  size_t ts = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, ts, pa.path_ptr, pa.path_ptr, (int)n_sel + 1, s);
  void* tscan = alloc(ts);
  if (!tscan) return done(cudaErrorMemoryAllocation);
  if ((e = cub::DeviceScan::ExclusiveSum(tscan, ts, pa.path_ptr, pa.path_ptr, (int)n_sel + 1, s)) != cudaSuccess)
    return done(e);
  cudaMemcpyAsync(n_pins, pa.path_ptr + n_sel, 4, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return done(e);
  if (*n_pins > cap_pins) {
    *fits = false;
    return done(cudaSuccess);
  }
  path_fill_kernel<<<blocks(n_sel), kThreads, 0, s>>>(t, c, pa, n_sel);
  e = cudaGetLastError();
  cudaError_t e2 = cudaStreamSynchronize(s);
  return done(e != cudaSuccess ? e : e2);
}

cudaError_t launch_set_ptrs(const float* const* dst, const float* a, const float* b, cudaStream_t s) {
  set_ptrs_kernel<<<1, 1, 0, s>>>(const_cast<const float**>(dst), a, b);
  return cudaGetLastError();
}

// co-resident grid of the persistent forward (which = 0) or backward (1)
// kernel: blocks per SM from the occupancy calculator x SMs; 0 if unsupported
uint32_t persistent_grid(uint32_t smem_f4, int which) {
  int dev = 0, sms = 0, nb = 0, coop = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return 0;
  const size_t smem = 16ull * smem_f4;
  // the same grid serves the traced instantiation: the smaller of the two
  int nt = 0;
  if (which == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, smem_f4 ? fwd_persistent_kernel<true, false> : fwd_persistent_kernel<false, false>, kFwdThreads, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nt, smem_f4 ? fwd_persistent_kernel<true, true> : fwd_persistent_kernel<false, true>, kFwdThreads, smem);
  } else if (which == 1) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, smem_f4 ? bwd_persistent_kernel<true, false> : bwd_persistent_kernel<false, false>, kBwdThreads,
        smem + kBwdExtraSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nt, smem_f4 ? bwd_persistent_kernel<true, true> : bwd_persistent_kernel<false, true>, kBwdThreads,
        smem + kBwdExtraSmem);
  }
  cudaGetLastError();
  return (uint32_t)(std::min(nb, nt) * sms);
}

template <class Kern>
cudaError_t coop_launch(Kern kernel, uint32_t grid, uint32_t block, size_t smem, cudaStream_t s, const Topo& t,
                        const Batch& b) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, t, b);
}

static bool traced(const Batch& b) { return b.c[0].trace != nullptr; }

using PersistentKern = void (*)(Topo, const Batch);
// the Arnoldi / -through instantiations (fwd_persistent_ext_kernel, bwd_persistent_ext_kernel)
// (Elmore with -through: fwd / bwd_persistent_thr_kernel at the propagation
// kernels' own block sizes; the Arnoldi variants at 512 threads)
static PersistentKern ext_kernel(bool fwd, bool sm, bool arn, bool thr) {
  if (fwd) {
    if (sm) return arn ? (thr ? fwd_persistent_ext_kernel<true, true, true> : fwd_persistent_ext_kernel<true, true, false>)
                       : fwd_persistent_thr_kernel<true>;
    return arn ? (thr ? fwd_persistent_ext_kernel<false, true, true> : fwd_persistent_ext_kernel<false, true, false>)
               : fwd_persistent_thr_kernel<false>;
  }
  if (sm) return arn ? (thr ? bwd_persistent_ext_kernel<true, true, true> : bwd_persistent_ext_kernel<true, true, false>)
                     : bwd_persistent_thr_kernel<true>;
  return arn ? (thr ? bwd_persistent_ext_kernel<false, true, true> : bwd_persistent_ext_kernel<false, true, false>)
             : bwd_persistent_thr_kernel<false>;
}
static uint32_t ext_threads(bool fwd, bool arn) {
  return arn ? (fwd ? kFwdArnThreads : kBwdArnThreads) : (fwd ? kFwdThreads : kBwdThreads);
}
static uint32_t ext_grid(PersistentKern k, uint32_t threads, size_t smem) {
  int dev = 0, sms = 0, nb = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, (int)threads, smem);
  cudaGetLastError();
  return (uint32_t)(nb * sms);
}

cudaError_t launch_fwd_persistent(const Topo& t, const Batch& b, uint32_t grid, cudaStream_t s) {
  if (!t.NP) return cudaSuccess;
  const size_t sm = 16ull * b.smem_f4;
  const bool arn = t.net_model == 1, thr = t.thr_pull != nullptr;
  if (arn || thr) {                          // row f1 Arnoldi model / row f4 -through hooks
    const PersistentKern k = ext_kernel(true, b.smem_f4 != 0, arn, thr);
    const uint32_t nt = ext_threads(true, arn);
    const uint32_t g = ext_grid(k, nt, sm);
    if (!g) return cudaErrorCooperativeLaunchTooLarge;
    return coop_launch(k, g, nt, sm, s, t, b);
  }
  // STA_TRACE builds per-unit timestamps into a separate instantiation
  if (traced(b))
    return b.smem_f4 ? coop_launch(fwd_persistent_kernel<true, true>, grid, kFwdThreads, sm, s, t, b)
                     : coop_launch(fwd_persistent_kernel<false, true>, grid, kFwdThreads, 0, s, t, b);
  return b.smem_f4 ? coop_launch(fwd_persistent_kernel<true, false>, grid, kFwdThreads, sm, s, t, b)
                   : coop_launch(fwd_persistent_kernel<false, false>, grid, kFwdThreads, 0, s, t, b);
}

cudaError_t launch_bwd_persistent(const Topo& t, const Batch& b, uint32_t grid, cudaStream_t s) {
  if (!t.n_bwu) return cudaSuccess;
  const size_t sm = 16ull * b.smem_f4 + kBwdExtraSmem;
  const bool arn = t.net_model == 1, thr = t.thr_pull != nullptr;
  if (arn || thr) {
    const PersistentKern k = ext_kernel(false, b.smem_f4 != 0, arn, thr);
    const uint32_t nt = ext_threads(false, arn);
    const uint32_t g = ext_grid(k, nt, sm);
    if (!g) return cudaErrorCooperativeLaunchTooLarge;
    return coop_launch(k, g, nt, sm, s, t, b);
  }
  if (traced(b))
    return b.smem_f4 ? coop_launch(bwd_persistent_kernel<true, true>, grid, kBwdThreads, sm, s, t, b)
                     : coop_launch(bwd_persistent_kernel<false, true>, grid, kBwdThreads, kBwdExtraSmem, s, t, b);
  return b.smem_f4 ? coop_launch(bwd_persistent_kernel<true, false>, grid, kBwdThreads, sm, s, t, b)
                   : coop_launch(bwd_persistent_kernel<false, false>, grid, kBwdThreads, kBwdExtraSmem, s, t, b);
}

cudaError_t set_lut_smem_limit(size_t bytes) {
  const int b = (int)bytes;
  cudaError_t e = cudaFuncSetAttribute(fwd_stage_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(bwd_stage_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  for (int v = 0; v < 3 && e == cudaSuccess; ++v) {   // (arn, thr) = (1, 0), (0, 1), (1, 1)
    const bool arn = v != 1, thr = v != 0;
    e = cudaFuncSetAttribute(ext_kernel(true, true, arn, thr), cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ext_kernel(false, true, arn, thr), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               b + (int)kBwdExtraSmem);
  }
  for (int tr = 0; tr < 2 && e == cudaSuccess; ++tr) {
    e = cudaFuncSetAttribute(tr ? fwd_persistent_kernel<true, true> : fwd_persistent_kernel<true, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tr ? bwd_persistent_kernel<true, true> : bwd_persistent_kernel<true, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, b + (int)kBwdExtraSmem);
  }
  return e;
}

cudaError_t launch_init_corner(const Topo&, const CornerDev& c, uint32_t n_heavy, cudaStream_t s) {
  init_corner_kernel<<<blocks(n_heavy + 1), kThreads, 0, s>>>(c, n_heavy);
  return cudaGetLastError();
}

}  // namespace sta
