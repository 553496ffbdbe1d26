// sta_kernels.cu -- sm_100a kernels of one graph-based STA timing update.
//
// Hot path:
//   a1  rc_small_kernel / rc_big_kernel  Elmore RC per net: Cdown bottom-up,
//       load = Cdown[root], elm top-down
//   a2  seed_kernel + fwd_stage_kernel   arrival/slew, one launch per gate
//       stage; NLDM bilinear lookup for cell arcs,
//       Elmore + PERI slew for net arcs, early min / late
//       max merge
//   a3-a5 bwd_stage_kernel               endpoint seeds,
//       required times over fan-out (min late / max early), per-pin slack and
//       per-endpoint worst slack, one launch per gate stage in reverse
//   a5  reduce_kernel                    WNS / TNS (TNS in fp64), fixed order
//
// Numerics: fp32 state, no fast-math.  Every floating-point operation whose
// result is reused by another kernel (net hop, LUT lookup) is written with
// explicit round-to-nearest intrinsics so that no FMA-contraction choice of
// the compiler can make the forward and the backward recomputation of an arc
// delay differ by one ulp.  RC is accumulated in fp64.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "sta_internal.h"

namespace sta {

namespace {

constexpr float kLn9 = 2.19722457733621956f;   // ln 9: PERI impulse factor
constexpr int kThreads = 256;

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

__device__ __forceinline__ bool sense_allows(uint32_t sense, int irf, int orf) {
  switch (sense) {
    case 0: return irf == orf;          // positive unate
    case 1: return irf != orf;          // negative unate
    case 2: return true;                // non-unate
    case 3: return irf == 0;            // rising edge (clock-to-Q)
    default: return irf == 1;           // falling edge
  }
}

// NLDM bilinear lookup with boundary-cell extrapolation.
// Segment i = clamp(upper_bound(x, s) - 1, 0, n - 2) = #{k in 1..n-2 : x[k] <= s}.
__device__ __forceinline__ float lut_eval(const float* __restrict__ pool, uint32_t desc, float s, float c) {
  const uint32_t off = desc & 0x03FFFFFFu;
  const int n1 = int((desc >> 26) & 7u) + 1;
  const int n2 = int((desc >> 29) & 7u) + 1;
  const float* x = pool + off;
  const float* y = x + n1;
  const float* v = y + n2;
  int i = 0, j = 0;
#pragma unroll
  for (int k = 1; k < 7; ++k) {
    if (k <= n1 - 2 && __ldg(x + k) <= s) ++i;
    if (k <= n2 - 2 && __ldg(y + k) <= c) ++j;
  }
  float tx = 0.f, ty = 0.f;
  int si = 0, sj = 0;
  if (n1 > 1) {
    const float x0 = __ldg(x + i), x1 = __ldg(x + i + 1);
    tx = __fdiv_rn(__fsub_rn(s, x0), __fsub_rn(x1, x0));
    si = n2;
  }
  if (n2 > 1) {
    const float y0 = __ldg(y + j), y1 = __ldg(y + j + 1);
    ty = __fdiv_rn(__fsub_rn(c, y0), __fsub_rn(y1, y0));
    sj = 1;
  }
  const float* p = v + i * n2 + j;
  const float v00 = __ldg(p), v10 = __ldg(p + si), v01 = __ldg(p + sj), v11 = __ldg(p + si + sj);
  const float a = __fmaf_rn(tx, __fsub_rn(v10, v00), v00);
  const float b = __fmaf_rn(tx, __fsub_rn(v11, v01), v01);
  return __fmaf_rn(ty, __fsub_rn(b, a), a);
}

__device__ __forceinline__ float lut_id(const CornerDev& c, uint32_t tab, float s, float ld) {
  return lut_eval(c.lut, __ldg(c.tdesc + tab), s, ld);
}

// Net arc driver -> sink: AT + elm, slew = sqrt(slew^2 + (ln9 elm)^2) (PERI,
// SPEC.md:416-418).  Undefined components stay undefined.
__device__ __forceinline__ void net_hop(Q4& at, Q4& sl, float e) {
  const float imp = __fmul_rn(kLn9, e);
  const float imp2 = __fmul_rn(imp, imp);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (fin(at.v[q])) {
      at.v[q] = __fadd_rn(at.v[q], e);
      sl.v[q] = __fsqrt_rn(__fmaf_rn(sl.v[q], sl.v[q], imp2));
    } else {
      sl.v[q] = q < 2 ? CUDART_INF_F : -CUDART_INF_F;
    }
  }
}

// Cell arc u -> v (forward): merge candidates of every (el, irf -> orf) pair
// the sense allows into acc_at / acc_sl (early min, late max).
__device__ __forceinline__ void cell_fwd(const CornerDev& c, const Q4& at, const Q4& sl, uint32_t info,
                                         float ld, Q4& acc_at, Q4& acc_sl) {
  const uint32_t sense = info & 7u, tab = info >> 3;
#pragma unroll
  for (int el = 0; el < 2; ++el) {
#pragma unroll
    for (int irf = 0; irf < 2; ++irf) {
      const float a_in = at.v[el * 2 + irf];
      if (!fin(a_in)) continue;
      const float s_in = sl.v[el * 2 + irf];
#pragma unroll
      for (int orf = 0; orf < 2; ++orf) {
        if (!sense_allows(sense, irf, orf)) continue;
        const float d = fmaxf(0.f, lut_id(c, tab + orf, s_in, ld));
        const float so = fmaxf(0.f, lut_id(c, tab + 2 + orf, s_in, ld));
        const float ca = __fadd_rn(a_in, d);
        const int q = el * 2 + orf;
        if (el == 0) { acc_at.v[q] = fminf(acc_at.v[q], ca); acc_sl.v[q] = fminf(acc_sl.v[q], so); }
        else         { acc_at.v[q] = fmaxf(acc_at.v[q], ca); acc_sl.v[q] = fmaxf(acc_sl.v[q], so); }
      }
    }
  }
}

// Cell arc u -> w (backward): RAT_L(u,irf) = min(RAT_L(w,orf) - d), RAT_E =
// max(RAT_E(w,orf) - d) over exactly the pairs the forward pass used, with d
// recomputed bit-identically from slew(u) and load(w).
__device__ __forceinline__ void cell_bwd(const CornerDev& c, const Q4& at_u, const Q4& sl_u, uint32_t info,
                                         float ld, const Q4& rat_w, Q4& acc) {
  const uint32_t sense = info & 7u, tab = info >> 3;
#pragma unroll
  for (int el = 0; el < 2; ++el) {
#pragma unroll
    for (int irf = 0; irf < 2; ++irf) {
      if (!fin(at_u.v[el * 2 + irf])) continue;
      const float s_in = sl_u.v[el * 2 + irf];
#pragma unroll
      for (int orf = 0; orf < 2; ++orf) {
        if (!sense_allows(sense, irf, orf)) continue;
        const float d = fmaxf(0.f, lut_id(c, tab + orf, s_in, ld));
        const float cand = __fsub_rn(rat_w.v[el * 2 + orf], d);
        const int q = el * 2 + irf;
        acc.v[q] = el == 0 ? fmaxf(acc.v[q], cand) : fminf(acc.v[q], cand);
      }
    }
  }
}

// Endpoint required-time seeds: PO: RAT_L = T - out_max,
// RAT_E = -out_min; check: RAT_L = T - setup(slew_L(D), clock slew),
// RAT_E = hold(slew_E(D), clock slew), only where the data arrival exists.
__device__ __forceinline__ void apply_seed(const Topo& t, const CornerDev& c, uint32_t e, const Q4& at,
                                           const Q4& sl, Q4& r) {
  const EpRec ep = t.ep[e];
  if (ep.po != kNone) {
    const float2 omax = t.po_out_max[ep.po], omin = t.po_out_min[ep.po];
    r.v[2] = fminf(r.v[2], __fsub_rn(t.period, omax.x));
    r.v[3] = fminf(r.v[3], __fsub_rn(t.period, omax.y));
    r.v[0] = fmaxf(r.v[0], -omin.x);
    r.v[1] = fmaxf(r.v[1], -omin.y);
  }
  if (ep.chk_tab != kNone) {
#pragma unroll
    for (int rf = 0; rf < 2; ++rf) {
      if (fin(at.v[2 + rf]))
        r.v[2 + rf] = fminf(r.v[2 + rf], __fsub_rn(t.period, lut_id(c, ep.chk_tab + rf, sl.v[2 + rf], t.clock_slew)));
      if (fin(at.v[rf]))
        r.v[rf] = fmaxf(r.v[rf], lut_id(c, ep.chk_tab + 2 + rf, sl.v[rf], t.clock_slew));
    }
  }
}

// slack_L = RAT_L - AT_L, slack_E = AT_E - RAT_E, +inf if either is undefined.
__device__ __forceinline__ Q4 slack_of(const Q4& at, const Q4& r) {
  Q4 s;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool ok = fin(at.v[q]) && fin(r.v[q]);
    s.v[q] = ok ? (q < 2 ? __fsub_rn(at.v[q], r.v[q]) : __fsub_rn(r.v[q], at.v[q])) : CUDART_INF_F;
  }
  return s;
}

__device__ __forceinline__ void write_ep(const CornerDev& c, uint32_t e, const Q4& s) {
  c.ep_ws[e] = make_float2(fminf(s.v[2], s.v[3]), fminf(s.v[0], s.v[1]));
}

__device__ __forceinline__ void load_rec(const CornerDev& c, uint32_t i, Q4& at, Q4& sl) {
  at = to_q(__ldg(c.rec + 2 * (size_t)i));
  sl = to_q(__ldg(c.rec + 2 * (size_t)i + 1));
}

// ------------------------------------------------------------------ a1: RC
__device__ __forceinline__ bool bad_rc(float r, float cw) {
  return !(r >= 0.f) || !(cw >= 0.f) || !(r < CUDART_INF_F) || !(cw < CUDART_INF_F);
}

// One thread per net with <= kSmallNet RC nodes (and lumped nets): the
// textbook O(n) two-pass recursion, in fp64.
__global__ void __launch_bounds__(kThreads) rc_small_kernel(Topo t, CornerDev c) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= t.N) return;
  const uint32_t drv = t.net_drv[j];
  const uint32_t m = t.net_rcn[j];
  const uint32_t sb = t.sink_ptr[drv], se = t.sink_ptr[drv + 1];
  if (m == 0) {                            // lumped net
    c.load[drv] = t.net_lumped[j];
    for (uint32_t k = sb; k < se; ++k) c.elm[k] = 0.f;
    return;
  }
  if (m > (uint32_t)kSmallNet) return;
  const uint32_t b = t.net_rc[j];
  double cd[kSmallNet];
  bool bad = false;
  for (uint32_t i = 0; i < m; ++i) {
    const float cw = c.rc_cap[b + i];
    const float r = c.rc_res[b + i];
    bad |= bad_rc(i ? r : 0.f, cw);
    cd[i] = (double)cw + (double)t.rc_scap[b + i];
  }
  for (uint32_t i = m - 1; i >= 1; --i) cd[t.rc_parent[b + i]] += cd[i];
  c.load[drv] = (float)cd[0];
  double el[kSmallNet];
  el[0] = 0.0;
  for (uint32_t i = 1; i < m; ++i) {
    el[i] = __fma_rn((double)c.rc_res[b + i], cd[i], el[t.rc_parent[b + i]]);
    const uint32_t k = t.rc_sink[b + i];
    if (k != kNone) c.elm[k] = (float)el[i];
  }
  if (bad) atomicOr(c.err_flag, 1u);
}

// One block per big net: Cdown by height level (children summed in
// decreasing index order -- the same rounding order as the sequential
// recursion), then Elmore by depth level.
__global__ void __launch_bounds__(kThreads) rc_big_kernel(Topo t, CornerDev c) {
  const uint32_t bi = blockIdx.x;
  const uint32_t j = t.big_net[bi];
  const uint32_t drv = t.net_drv[j];
  const uint32_t b = t.net_rc[j];
  double* cd = c.scratch + t.big_scr[bi];
  double* el = c.scratch + t.big_scr[t.n_big] + t.big_scr[bi];
  const uint32_t* cptr = t.big_cptr + t.big_scr[bi] + bi;
  bool bad = false;
  for (uint32_t h = t.big_hptr_off[bi]; h + 1 < t.big_hptr_off[bi + 1]; ++h) {
    for (uint32_t x = t.big_hptr[h] + threadIdx.x; x < t.big_hptr[h + 1]; x += blockDim.x) {
      const uint32_t p = t.big_hnode[x];
      const float cw = c.rc_cap[b + p];
      bad |= bad_rc(p ? c.rc_res[b + p] : 0.f, cw);
      double v = (double)cw + (double)t.rc_scap[b + p];
      for (uint32_t k = cptr[p]; k < cptr[p + 1]; ++k) v += cd[t.big_child[k]];
      cd[p] = v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    c.load[drv] = (float)cd[0];
    el[0] = 0.0;
  }
  __syncthreads();
  for (uint32_t h = t.big_dptr_off[bi]; h + 1 < t.big_dptr_off[bi + 1]; ++h) {
    for (uint32_t x = t.big_dptr[h] + threadIdx.x; x < t.big_dptr[h + 1]; x += blockDim.x) {
      const uint32_t i = t.big_dnode[x];
      const double e = __fma_rn((double)c.rc_res[b + i], cd[i], el[t.rc_parent[b + i]]);
      el[i] = e;
      const uint32_t k = t.rc_sink[b + i];
      if (k != kNone) c.elm[k] = (float)e;
    }
    __syncthreads();
  }
  if (bad) atomicOr(c.err_flag, 1u);
}

// ------------------------------------------------------------ a2: forward
// Stage-0 pull pins (no fan-in): PI arrivals, ideal clock, or undefined.
__global__ void __launch_bounds__(kThreads) seed_kernel(Topo t, CornerDev c, uint32_t n0) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n0) return;
  const uint32_t s = t.seed[i];
  float4 at, sl;
  if (s == kNone) {
    at = to_f4(undef_at());
    sl = at;
  } else if (s == kSeedClock) {              // rising edge at 0, falling at T/2
    const float h = 0.5f * t.period;
    at = make_float4(0.f, h, 0.f, h);
    sl = make_float4(t.clock_slew, t.clock_slew, t.clock_slew, t.clock_slew);
  } else {
    at = t.pi_at[s];
    sl = t.pi_slew[s];
  }
  c.rec[2 * (size_t)i] = at;
  c.rec[2 * (size_t)i + 1] = sl;
}

// One launch per gate stage s >= 1.  Items [0, nA): materialize the sinks of
// the stage s-1 drivers.  Items [nA, nA+nB): pull pins of stage s, each
// merging its cell fan-in; a fan-in pin that is a net sink is recomputed
// inline from its driver (pull-through), so sinks never cost a stage.
__global__ void __launch_bounds__(kThreads) fwd_stage_kernel(Topo t, CornerDev c, uint32_t sinkA0, uint32_t nA,
                                                             uint32_t pullB0, uint32_t nB) {
  const uint32_t item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item < nA) {
    const uint32_t k = sinkA0 + item;
    Q4 at, sl;
    load_rec(c, t.sink_drv[k], at, sl);
    net_hop(at, sl, c.elm[k]);
    const size_t u = (size_t)t.NP + k;
    c.rec[2 * u] = to_f4(at);
    c.rec[2 * u + 1] = to_f4(sl);
    return;
  }
  if (item >= nA + nB) return;
  const uint32_t v = pullB0 + (item - nA);
  const float ld = c.load[v];
  Q4 acc_at = undef_at(), acc_sl = undef_at();
  const uint32_t e0 = t.fi_ptr[v], e1 = t.fi_ptr[v + 1];
  for (uint32_t e = e0; e < e1; ++e) {
    const uint32_t src = t.fi_src[e], hop = t.fi_hop[e], info = t.fi_info[e];
    Q4 at, sl;
    load_rec(c, src, at, sl);
    if (hop != kNone) net_hop(at, sl, c.elm[hop]);
    cell_fwd(c, at, sl, info, ld, acc_at, acc_sl);
  }
  c.rec[2 * (size_t)v] = to_f4(acc_at);
  c.rec[2 * (size_t)v + 1] = to_f4(acc_sl);
}

// ------------------------------------------------------ a3-a5: backward
// Required time of sink k (internal id NP + k): its endpoint seed combined
// with its cell fan-out.  Writes rat / slack / endpoint worst slack of the sink.
__device__ __forceinline__ Q4 sink_rat(const Topo& t, const CornerDev& c, uint32_t k) {
  const uint32_t u = t.NP + k;
  Q4 at, sl;
  load_rec(c, u, at, sl);
  Q4 r = undef_rat();
  const uint32_t e = t.pin_ep[u];
  if (e != kNone) apply_seed(t, c, e, at, sl, r);
  for (uint32_t x = t.sfo_ptr[k]; x < t.sfo_ptr[k + 1]; ++x) {
    const uint32_t w = t.sfo_dst[x];
    const Q4 rw = to_q(__ldg(c.rat + w));
    cell_bwd(c, at, sl, t.sfo_info[x], c.load[w], rw, r);
  }
  c.rat[u] = to_f4(r);
  const Q4 s = slack_of(at, r);
  c.slack[u] = to_f4(s);
  if (e != kNone) write_ep(c, e, s);
  return r;
}

// Candidate of a driver from one of its sinks through the net arc.
__device__ __forceinline__ void net_bwd(const Q4& at_v, const Q4& r_u, float e, Q4& acc) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (!fin(at_v.v[q])) continue;
    const float cand = __fsub_rn(r_u.v[q], e);
    acc.v[q] = q < 2 ? fmaxf(acc.v[q], cand) : fminf(acc.v[q], cand);
  }
}

// Finish a pull pin: own seed, direct cell fan-out, then rat / slack.
__device__ __forceinline__ void finish_pull(const Topo& t, const CornerDev& c, uint32_t v, const Q4& at,
                                            const Q4& sl, Q4 acc) {
  const uint32_t e = t.pin_ep[v];
  if (e != kNone) apply_seed(t, c, e, at, sl, acc);
  for (uint32_t x = t.pfo_ptr[v]; x < t.pfo_ptr[v + 1]; ++x) {
    const uint32_t w = t.pfo_dst[x];
    cell_bwd(c, at, sl, t.pfo_info[x], c.load[w], to_q(__ldg(c.rat + w)), acc);
  }
  c.rat[v] = to_f4(acc);
  const Q4 s = slack_of(at, acc);
  c.slack[v] = to_f4(s);
  if (e != kNone) write_ep(c, e, s);
}

// One launch per gate stage s (descending).  Blocks [0, nLightBlocks): one
// thread per pull pin of the stage with <= kHeavyFanout sinks, which also
// owns its sinks.  Remaining blocks: one block per heavy driver.
__global__ void __launch_bounds__(kThreads) bwd_stage_kernel(Topo t, CornerDev c, uint32_t pull0, uint32_t nPull,
                                                             uint32_t heavy0, uint32_t nLightBlocks) {
  if (blockIdx.x < nLightBlocks) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nPull) return;
    const uint32_t v = pull0 + i;
    const uint32_t sb = t.sink_ptr[v], se = t.sink_ptr[v + 1];
    if (se - sb > (uint32_t)kHeavyFanout) return;
    Q4 at, sl;
    load_rec(c, v, at, sl);
    Q4 acc = undef_rat();
    for (uint32_t k = sb; k < se; ++k) {
      const Q4 r = sink_rat(t, c, k);
      net_bwd(at, r, c.elm[k], acc);
    }
    finish_pull(t, c, v, at, sl, acc);
    return;
  }
  // heavy driver: block-strided sinks, block min/max reduction
  const uint32_t v = t.heavy[heavy0 + (blockIdx.x - nLightBlocks)];
  const uint32_t sb = t.sink_ptr[v], se = t.sink_ptr[v + 1];
  Q4 at, sl;
  load_rec(c, v, at, sl);
  Q4 acc = undef_rat();
  for (uint32_t k = sb + threadIdx.x; k < se; k += blockDim.x) {
    const Q4 r = sink_rat(t, c, k);
    net_bwd(at, r, c.elm[k], acc);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float x = __shfl_xor_sync(0xFFFFFFFFu, acc.v[q], o);
      acc.v[q] = q < 2 ? fmaxf(acc.v[q], x) : fminf(acc.v[q], x);
    }
  }
  __shared__ float4 part[kThreads / 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) part[w] = to_f4(acc);
  __syncthreads();
  if (threadIdx.x == 0) {
    Q4 a = undef_rat();
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      const Q4 p = to_q(part[k]);
#pragma unroll
      for (int q = 0; q < 4; ++q) a.v[q] = q < 2 ? fmaxf(a.v[q], p.v[q]) : fminf(a.v[q], p.v[q]);
    }
    finish_pull(t, c, v, at, sl, a);
  }
}

// ------------------------------------------------------- a5: WNS / TNS
// Single block, fixed element-to-thread assignment and fixed tree: the
// result is bitwise reproducible (SURVEY.md §8(c) reading #16).
__global__ void __launch_bounds__(1024) reduce_kernel(Topo t, CornerDev c) {
  __shared__ double s_tns[1024], h_tns[1024];
  __shared__ float s_wns[1024], h_wns[1024];
  float ws = CUDART_INF_F, wh = CUDART_INF_F;
  double ts = 0.0, th = 0.0;
  for (uint32_t e = threadIdx.x; e < t.n_ep; e += blockDim.x) {
    const float2 x = c.ep_ws[e];
    ws = fminf(ws, x.x);
    wh = fminf(wh, x.y);
    if (x.x < 0.f) ts += (double)x.x;
    if (x.y < 0.f) th += (double)x.y;
  }
  s_wns[threadIdx.x] = ws; h_wns[threadIdx.x] = wh;
  s_tns[threadIdx.x] = ts; h_tns[threadIdx.x] = th;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s_wns[threadIdx.x] = fminf(s_wns[threadIdx.x], s_wns[threadIdx.x + o]);
      h_wns[threadIdx.x] = fminf(h_wns[threadIdx.x], h_wns[threadIdx.x + o]);
      s_tns[threadIdx.x] += s_tns[threadIdx.x + o];
      h_tns[threadIdx.x] += h_tns[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    c.res[0] = (double)s_wns[0];
    c.res[1] = s_tns[0];
    c.res[2] = (double)h_wns[0];
    c.res[3] = h_tns[0];
  }
}

// ----------------------------------------------------- output gathers
__global__ void gather4_kernel(const float4* __restrict__ src, const uint32_t* __restrict__ idx,
                               float4* __restrict__ dst, uint32_t n, uint32_t stride) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) dst[p] = src[(size_t)idx[p] * stride];
}

__global__ void gather_rc_kernel(Topo t, CornerDev c, float* net_load, float* pin_elm,
                                 const uint32_t* drv_of_net) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (net_load && p < t.N) net_load[p] = c.load[drv_of_net[p]];
  if (pin_elm && p < t.P) {
    const uint32_t i = t.int_of_user[p];
    pin_elm[p] = i >= t.NP ? c.elm[i - t.NP] : 0.f;
  }
}

inline uint32_t blocks(uint64_t n, uint32_t th = kThreads) { return (uint32_t)((n + th - 1) / th); }

}  // namespace

cudaError_t launch_rc(const Topo& t, const CornerDev& c, uint32_t, cudaStream_t s) {
  if (t.N) rc_small_kernel<<<blocks(t.N), kThreads, 0, s>>>(t, c);
  if (t.n_big) rc_big_kernel<<<t.n_big, kThreads, 0, s>>>(t, c);
  return cudaGetLastError();
}

cudaError_t launch_seed(const Topo& t, const CornerDev& c, uint32_t n0, cudaStream_t s) {
  if (n0) seed_kernel<<<blocks(n0), kThreads, 0, s>>>(t, c, n0);
  return cudaGetLastError();
}

cudaError_t launch_fwd_stage(const Topo& t, const CornerDev& c, uint32_t sinkA0, uint32_t nA, uint32_t pullB0,
                             uint32_t nB, cudaStream_t s) {
  if (nA + nB) fwd_stage_kernel<<<blocks((uint64_t)nA + nB), kThreads, 0, s>>>(t, c, sinkA0, nA, pullB0, nB);
  return cudaGetLastError();
}

cudaError_t launch_bwd_stage(const Topo& t, const CornerDev& c, uint32_t pull0, uint32_t nPull, uint32_t heavy0,
                             uint32_t nHeavy, cudaStream_t s) {
  const uint32_t nl = blocks(nPull);
  if (nl + nHeavy) bwd_stage_kernel<<<nl + nHeavy, kThreads, 0, s>>>(t, c, pull0, nPull, heavy0, nl);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const Topo& t, const CornerDev& c, cudaStream_t s) {
  reduce_kernel<<<1, 1024, 0, s>>>(t, c);
  return cudaGetLastError();
}

cudaError_t launch_gather4(const float4* src, const uint32_t* idx, float4* dst, uint32_t n, uint32_t stride,
                           cudaStream_t s) {
  if (n) gather4_kernel<<<blocks(n), kThreads, 0, s>>>(src, idx, dst, n, stride);
  return cudaGetLastError();
}

cudaError_t launch_gather_rc(const Topo& t, const CornerDev& c, float* net_load, float* pin_elm,
                             const uint32_t* drv_of_net, const uint32_t*, cudaStream_t s) {
  const uint32_t n = t.N > t.P ? t.N : t.P;
  if (n) gather_rc_kernel<<<blocks(n), kThreads, 0, s>>>(t, c, net_load, pin_elm, drv_of_net);
  return cudaGetLastError();
}

cudaError_t launch_check_rc_values(const CornerDev&, uint32_t, cudaStream_t) { return cudaSuccess; }

}  // namespace sta
