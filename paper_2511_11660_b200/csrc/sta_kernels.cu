// sta_kernels.cu -- sm_100a kernels of one graph-based STA timing update.
//
// Hot path:
//   a1  rc_warp_kernel / tc_* + scan_*   Elmore RC per net in fp64: Cdown
//       (subtree caps), load = Cdown[root], Elmore = sum of R Cdown over the
//       root path, from each net's DFS
//       preorder: warp shuffle scans for nets <= 32 nodes, device-wide prefix
//       sums (Euler tour) for larger nets.
//   a2  seed_kernel + fwd_stage_kernel   arrival/slew, one launch per gate
//       stage, one thread per stage pin; NLDM bilinear lookup for cell arcs
//       (SPEC.md:371-388), Elmore + PERI slew for net arcs
//       (SPEC.md:416-418), early-min / late-max merge.
//   a3-a5 bwd_stage_kernel   endpoint seeds, required
//       times over the fan-out (late min / early max), per-pin slack and
//       per-endpoint worst slack; one launch per gate stage in reverse; one
//       warp per tile of <= 32 consecutive sinks, segmented shuffle reduction
//       into their drivers, ordered-int atomics only for drivers with more
//       than 32 sinks.
//   a5  reduce_kernel   WNS / TNS (TNS in fp64), fixed-order two-level tree.
//
// All stage kernels are launched with programmatic dependent launch: the
// static topology of a stage is read before griddepcontrol.wait, so it
// overlaps the tail of the previous stage.
//
// Numerics: fp32 state, no fast-math.  Every floating-point operation whose
// result is reused by another kernel (net hop, LUT lookup) is written with
// explicit round-to-nearest intrinsics so that no FMA-contraction choice of
// the compiler can make two recomputations of the same quantity differ.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>

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

// axis (sx[8], x[8], rx[8])
__device__ __forceinline__ Seg seg(const float* a, float s) {
  const float4 sa = *reinterpret_cast<const float4*>(a);
  const float4 sb = *reinterpret_cast<const float4*>(a + 4);
  const int i = (sa.y <= s) + (sa.z <= s) + (sa.w <= s) + (sb.x <= s) + (sb.y <= s) + (sb.z <= s);
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
  return sense == 1 ? 1 - orf : sense == 3 ? 0 : sense == 4 ? 1 : orf;
}

// Copy the table records into shared memory (static data: may run before
// griddepcontrol.wait).  Returns the pointer lookups should use.  SMEM is a
// compile-time choice so that lookups compile to LDS (a pointer that may be
// shared or global compiles to slow generic loads).
extern __shared__ float4 s_dyn[];
template <bool SMEM>
__device__ __forceinline__ const float* stage_lut(const CornerDev& c, uint32_t n_f4) {
  if (!SMEM) return c.lut;                   // pool too large: global / L1
  const float4* g = reinterpret_cast<const float4*>(c.lut);
  for (uint32_t x = threadIdx.x; x < n_f4; x += blockDim.x) s_dyn[x] = __ldg(g + x);
  __syncthreads();
  return reinterpret_cast<const float*>(s_dyn);
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

// Cell arc u -> v (forward): merge the candidates of every (el, irf -> orf)
// pair the sense allows into acc_at / acc_sl (early min, late max).  The load
// axis search of each of the 4 tables is done once per arc.
__device__ __forceinline__ void cell_fwd(const float* __restrict__ L, const Q4& at, const Q4& sl, uint32_t info,
                                         float ld, Q4& acc_at, Q4& acc_sl) {
  const uint32_t sense = info & 7u, tab = info >> 3;
  const Tab rd0 = tab_rec(L, tab);            // cell_rise
  const Tab rd1 = tab_rec(L, tab + 1);        // cell_fall
  const Tab rs0 = tab_rec(L, tab + 2);        // rise_transition
  const Tab rs1 = tab_rec(L, tab + 3);        // fall_transition
  // tables of one library template share their axis searches
  const Seg cd0 = seg(rd0.ax + 24, ld);
  const Seg cd1 = rd1.ax == rd0.ax ? cd0 : seg(rd1.ax + 24, ld);
  const Seg cs0 = rs0.ax == rd0.ax ? cd0 : seg(rs0.ax + 24, ld);
  const Seg cs1 = rs1.ax == rd1.ax ? cd1 : seg(rs1.ax + 24, ld);
#pragma unroll
  // one pass: the plan expands a non-unate arc into positive- and
  // negative-unate terms (sta_api.cpp build_plan)
  for (int pass = 0; pass < 1; ++pass) {
#pragma unroll
    for (int orf = 0; orf < 2; ++orf) {
      const int irf = pass ? 1 - primary_irf(sense, orf) : primary_irf(sense, orf);
      const Tab rd = orf ? rd1 : rd0;
      const Tab rs = orf ? rs1 : rs0;
      const Seg cd = orf ? cd1 : cd0;
      const Seg cs = orf ? cs1 : cs0;
#pragma unroll
      for (int el = 0; el < 2; ++el) {
        const float a_in = irf ? at.v[el * 2 + 1] : at.v[el * 2];
        const float s_in = irf ? sl.v[el * 2 + 1] : sl.v[el * 2];
        if (!fin(a_in)) continue;
        const Seg sd = seg(rd.ax, s_in);
        const Seg ss = rs.ax == rd.ax ? sd : seg(rs.ax, s_in);
        const float d = fmaxf(0.f, interp(rd, sd, cd));
        const float so = fmaxf(0.f, interp(rs, ss, cs));
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
// recomputed bit-identically (same seg / interp calls) from slew(u), load(w).
__device__ __forceinline__ void cell_bwd(const float* __restrict__ L, const Q4& at_u, const Q4& sl_u,
                                         uint32_t info, float ld, const Q4& rat_w, Q4& acc) {
  const uint32_t sense = info & 7u, tab = info >> 3;
  const Tab rd0 = tab_rec(L, tab);
  const Tab rd1 = tab_rec(L, tab + 1);
  const Seg cd0 = seg(rd0.ax + 24, ld);
  const Seg cd1 = rd1.ax == rd0.ax ? cd0 : seg(rd1.ax + 24, ld);
#pragma unroll
  for (int pass = 0; pass < 1; ++pass) {   // non-unate arcs arrive expanded
#pragma unroll
    for (int orf = 0; orf < 2; ++orf) {
      const int irf = pass ? 1 - primary_irf(sense, orf) : primary_irf(sense, orf);
      const Tab rd = orf ? rd1 : rd0;
      const Seg cd = orf ? cd1 : cd0;
#pragma unroll
      for (int el = 0; el < 2; ++el) {
        const float a_in = irf ? at_u.v[el * 2 + 1] : at_u.v[el * 2];
        const float s_in = irf ? sl_u.v[el * 2 + 1] : sl_u.v[el * 2];
        if (!fin(a_in)) continue;
        const float d = fmaxf(0.f, interp(rd, seg(rd.ax, s_in), cd));
        const float cand = __fsub_rn(rat_w.v[el * 2 + orf], d);
        if (irf) acc.v[el * 2 + 1] = el == 0 ? fmaxf(acc.v[1], cand) : fminf(acc.v[3], cand);
        else     acc.v[el * 2] = el == 0 ? fmaxf(acc.v[0], cand) : fminf(acc.v[2], cand);
      }
    }
  }
}

// Endpoint required-time seeds: PO: RAT_L = T - out_max,
// RAT_E = -out_min; check: RAT_L = T - setup(slew_L(D), clock slew),
// RAT_E = hold(slew_E(D), clock slew), only where the data arrival exists.
// The static part (endpoint record, PO seeds) is loaded before the stage
// wait; the check-table lookups need the data slew and run after it.
struct SeedPre {
  Q4 po;              // PO seeds, or the undefined required time
  uint32_t chk;       // first check table or kNone
};

__device__ __forceinline__ SeedPre load_seed(const Topo& t, uint32_t e) {
  SeedPre p{undef_rat(), kNone};
  if (e == kNone) return p;
  const EpRec ep = t.ep[e];
  p.chk = ep.chk_tab;
  if (ep.po != kNone) {
    const float2 omax = t.po_out_max[ep.po], omin = t.po_out_min[ep.po];
    p.po = Q4{{-omin.x, -omin.y, __fsub_rn(t.period, omax.x), __fsub_rn(t.period, omax.y)}};
  }
  return p;
}

__device__ __forceinline__ void apply_seed_pre(const Topo& t, const float* L, const SeedPre& p, const Q4& at,
                                               const Q4& sl, Q4& r) {
  r.v[0] = fmaxf(r.v[0], p.po.v[0]);
  r.v[1] = fmaxf(r.v[1], p.po.v[1]);
  r.v[2] = fminf(r.v[2], p.po.v[2]);
  r.v[3] = fminf(r.v[3], p.po.v[3]);
  if (p.chk != kNone) {
#pragma unroll
    for (int rf = 0; rf < 2; ++rf) {
      if (fin(at.v[2 + rf]))
        r.v[2 + rf] = fminf(r.v[2 + rf], __fsub_rn(t.period, lut(L, p.chk + rf, sl.v[2 + rf], t.clock_slew)));
      if (fin(at.v[rf]))
        r.v[rf] = fmaxf(r.v[rf], lut(L, p.chk + 2 + rf, sl.v[rf], t.clock_slew));
    }
  }
}

__device__ __forceinline__ void apply_seed(const Topo& t, const CornerDev&, const float* L, uint32_t e,
                                           const Q4& at, const Q4& sl, Q4& r) {
  apply_seed_pre(t, L, load_seed(t, e), at, sl, r);
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

// records written by earlier kernels of this update: L2 loads (keep L1 for LUTs)
__device__ __forceinline__ void load_rec(const CornerDev& c, uint32_t i, Q4& at, Q4& sl) {
  at = to_q(__ldcg(c.rec + 2 * (size_t)i));
  sl = to_q(__ldcg(c.rec + 2 * (size_t)i + 1));
}

// ordered-int image of a float: monotone for signed-int comparison
__device__ __forceinline__ int f2o(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float o2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// ------------------------------------------------------------------ a1: RC
__device__ __forceinline__ bool bad_rc(float r, float cw) {
  return !(r >= 0.f) || !(cw >= 0.f) || !(r < CUDART_INF_F) || !(cw < CUDART_INF_F);
}

// Nets with 1..32 RC nodes: one warp tile holds whole nets, one lane per
// node in DFS preorder.  Cdown(p) = S[end(p)] - S[p] with S the segmented
// exclusive prefix sum of node caps (shuffle scan), Elmore(p) = sum of
// R * Cdown over the root path by pointer jumping over parent lanes (5
// rounds), all in fp64; every node is read once, coalesced.
__global__ void __launch_bounds__(kThreads) rc_warp_kernel(Topo t, CornerDev c) {
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31;
  const uint32_t wt = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wt >= t.n_wtiles) return;
  const uint2 tile = t.wtiles[wt];
  const bool act = lane < (int)tile.y;
  const uint32_t x = tile.x + lane;
  uint32_t meta = 0, tag = kNone;
  double C = 0.0;
  float r = 0.f;
  bool bad = false;
  if (act) {
    meta = t.node_meta[x];
    tag = t.node_tag[x];
    const uint32_t u = t.node_user[x];
    const float cw = c.rc_vals[1][u];
    const bool root = ((meta >> 8) & 0xFFu) == 0xFFu;
    r = root ? 0.f : c.rc_vals[0][u];
    bad = bad_rc(r, cw);
    C = (double)cw + (double)t.rc_scap[x];
  }
  const int pos = (int)(meta & 0xFFu), ppos = (int)((meta >> 8) & 0xFFu), epos = (int)((meta >> 16) & 0xFFu);
  // segmented inclusive scan of C (a net's lanes are contiguous; pos resets)
  double inc = C;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (pos >= o) inc += y;
  }
  double exc = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
  if (pos == 0) exc = 0.0;
  const int seg0 = lane - pos;
  const double s_end = __shfl_sync(0xFFFFFFFFu, inc, act ? seg0 + epos - 1 : lane);
  const double cd = s_end - exc;            // subtree cap of this node
  // root path sums of w = R * Cdown by pointer jumping
  double val = (act && ppos != 0xFF) ? (double)r * cd : 0.0;
  int pl = (act && ppos != 0xFF) ? seg0 + ppos : -1;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const double pv = __shfl_sync(0xFFFFFFFFu, val, pl >= 0 ? pl : lane);
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

__global__ void __launch_bounds__(kThreads) rc_block_kernel(Topo t, CornerDev c) {
  __shared__ double s_S[kBNet + 1], s_v[kBNet];
  __shared__ int16_t s_p[kBNet];
  __shared__ double s_warp[32];
  pdl_wait();
  pdl_launch();
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
      meta[k] = t.node_meta[x];
      tag[k] = t.node_tag[x];
      const uint32_t u = t.node_user[x];
      const float cw = c.rc_vals[1][u];
      r[k] = ((meta[k] >> 10) & 0x7FFu) == 0x7FFu ? 0.f : c.rc_vals[0][u];
      bad |= bad_rc(r[k], cw);
      C[k] = (double)cw + (double)t.rc_scap[x];
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
__global__ void __launch_bounds__(kThreads) rc_lumped_kernel(Topo t, CornerDev c) {
  pdl_wait();
  pdl_launch();
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= t.n_lumped) return;
  const uint32_t j = t.lumped_j[x];
  const uint32_t drv = t.net_drv[j];
  c.load[drv] = t.net_lumped[j];
  for (uint32_t k = t.sink_ptr[drv]; k < t.sink_ptr[drv + 1]; ++k) c.elm[k] = 0.f;
}

// L2-only loads (ld.global.cg): the records reached L2 before the flag
// (producer fence), the consumer's record loads are issued only after the
// flag value returned (control dependency), and no L1 copy can be stale.  An
// ld.acquire.gpu here would compile to CCTL.IVALL (whole-L1 invalidate),
// which profiling showed to cost half of the kernel time.
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- tier C: Euler-tour RC over one global preorder array (sta_internal.h)
// One persistent cooperative kernel, two blocks per SM (a small footprint
// next to the concurrently running small-net RC kernel), four phases
// separated by grid barriers:
//   1. S = exclusive prefix sum of the node caps (block ranges: local scan,
//      block sums, barrier, offsets), S[n] = total;
//   2. w(g) = R(g) (S[end(g)] - S[g]) in node order (0 at a net root), net loads;
//   3. H = inclusive prefix sum of the Euler event values +-w;
//   4. elm(g) = H[enter(g)] - H[2 g0 - 1].
// Offsets are fixed-shape sums of the block sums: bitwise reproducible.
constexpr int kTcThreads = 512;
constexpr int kTcBatch = 4;                  // elements in flight per thread

__device__ __forceinline__ void tc_grid_barrier(uint32_t* bar, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acquire(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      uint32_t ns = 32;
      while (ld_acquire(bar + 1) == gen) {
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : ns;
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// fixed-tree sum of sums[0 .. b) (the offset of block b)
__device__ __forceinline__ double tc_block_offset(const double* sums, uint32_t b, double* s_red) {
  double v = 0.0;
  for (uint32_t q = threadIdx.x; q < b; q += blockDim.x) v += __ldcg(sums + q);
  s_red[threadIdx.x] = v;
  __syncthreads();
  for (int o = kTcThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
    __syncthreads();
  }
  const double off = s_red[0];
  __syncthreads();
  return off;
}

// Device-wide prefix scan of x, whose block range [lo, hi) the block wrote
// with the strided mapping i = lo + threadIdx.x + k blockDim.x, each thread
// also accumulating `part` (its values in that order).  Block sums, grid
// barrier, offsets, then one block-wide scan per row of blockDim.x values.
// Returns the inclusive prefix at hi.
template <bool INCLUSIVE>
__device__ __forceinline__ double tc_scan_range(double* x, size_t lo, size_t hi, double part, double* sums,
                                                uint32_t* bar, double* s_warp, double* s_red) {
  s_red[threadIdx.x] = part;
  __syncthreads();
  for (int o = kTcThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s_red[threadIdx.x] += s_red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = s_red[0];
  tc_grid_barrier(bar, gridDim.x);
  double carry = tc_block_offset(sums, blockIdx.x, s_red);
  for (size_t r0 = lo; r0 < hi; r0 += blockDim.x) {
    const size_t i = r0 + threadIdx.x;
    const double v = i < hi ? x[i] : 0.0;      // own write (same mapping)
    double tot;
    const double e = block_excl_scan(v, s_warp, &tot);
    if (i < hi) x[i] = carry + (INCLUSIVE ? e + v : e);
    carry += tot;
  }
  return carry;
}

__global__ void __launch_bounds__(kTcThreads, 2) tc_persistent_kernel(Topo t, CornerDev c) {
  __shared__ double s_warp[32], s_red[kTcThreads];
  pdl_wait();
  pdl_launch();
  const uint32_t n = t.nCn, G = gridDim.x, B = blockIdx.x, BD = blockDim.x;
  const size_t m = 2 * (size_t)n;
  double* S = c.scratch;                     // [n + 1]
  double* H = S + n + 1;                     // [2n]
  double* W = H + m;                         // [n]
  double* sums = W + n;                      // [kTcMaxGrid]
  uint32_t* bar = reinterpret_cast<uint32_t*>(sums + kTcMaxGrid);
  const float* R = c.rc_vals[0];
  const float* Cw = c.rc_vals[1];
  const size_t lo = (size_t)n * B / G, hi = (size_t)n * (B + 1) / G;
  const size_t elo = m * B / G, ehi = m * (B + 1) / G;
  const size_t step = (size_t)BD * kTcBatch;

  // 1. node caps -> S (exclusive)
  bool bad = false;
  double part = 0.0;
  for (size_t i0 = lo + threadIdx.x; i0 < hi; i0 += step) {
    float cw[kTcBatch], sc[kTcBatch];
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k) {
      const size_t i = i0 + (size_t)k * BD;
      const bool in = i < hi;
      const uint32_t u = in ? t.tc_user[i] : 0u, ti = in ? t.tc_int[i] : 0u;
      cw[k] = in ? Cw[u] : 0.f;
      sc[k] = in ? t.rc_scap[ti & 0x7FFFFFFFu] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k) {
      const size_t i = i0 + (size_t)k * BD;
      if (i < hi) {
        bad |= bad_rc(0.f, cw[k]);
        const double v = (double)cw[k] + (double)sc[k];
        S[i] = v;
        part += v;
      }
    }
  }
  const double total = tc_scan_range<false>(S, lo, hi, part, sums, bar, s_warp, s_red);
  if (B == G - 1 && threadIdx.x == 0) S[n] = total;
  tc_grid_barrier(bar, G);

  // 2. w in node order; net loads
  for (size_t i0 = lo + threadIdx.x; i0 < hi; i0 += step) {
    double w[kTcBatch];
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k) {
      const size_t i = i0 + (size_t)k * BD;
      w[k] = 0.0;
      if (i < hi && !(t.tc_int[i] & 0x80000000u)) {
        const float r = R[t.tc_user[i]];
        bad |= bad_rc(r, 0.f);
        w[k] = (double)r * (__ldcg(S + t.tc_end[i]) - __ldcg(S + i));
      }
    }
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k) {
      const size_t i = i0 + (size_t)k * BD;
      if (i < hi) W[i] = w[k];
    }
  }
  for (uint32_t j = B * BD + threadIdx.x; j < t.nC; j += G * BD) {
    const uint32_t r = t.tc_root[j];
    c.load[t.tc_drv[j]] = (float)(__ldcg(S + t.tc_end[r]) - __ldcg(S + r));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(c.err_flag, 1u);
  tc_grid_barrier(bar, G);

  // 3. Euler event values -> H (inclusive)
  part = 0.0;
  for (size_t e0 = elo + threadIdx.x; e0 < ehi; e0 += step) {
    double x[kTcBatch];
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k) {
      const size_t e = e0 + (size_t)k * BD;
      x[k] = 0.0;
      if (e < ehi) {
        const uint32_t ev = t.tc_ev[e];
        const double w = __ldcg(W + (ev & 0x7FFFFFFFu));
        x[k] = (ev & 0x80000000u) ? -w : w;
      }
    }
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k) {
      const size_t e = e0 + (size_t)k * BD;
      if (e < ehi) {
        H[e] = x[k];
        part += x[k];
      }
    }
  }
  tc_scan_range<true>(H, elo, ehi, part, sums, bar, s_warp, s_red);
  tc_grid_barrier(bar, G);

  // 4. elm of the sink nodes
  for (size_t i0 = lo + threadIdx.x; i0 < hi; i0 += step) {
    uint32_t k2[kTcBatch];
    float v[kTcBatch];
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k) {
      const size_t i = i0 + (size_t)k * BD;
      k2[k] = kNone;
      v[k] = 0.f;
      if (i < hi) {
        k2[k] = t.node_tag[t.tc_int[i] & 0x7FFFFFFFu];
        const uint32_t g0 = t.tc_start[i];
        v[k] = (float)(__ldcg(H + t.tc_enter[i]) - (g0 ? __ldcg(H + 2 * (size_t)g0 - 1) : 0.0));
      }
    }
#pragma unroll
    for (int k = 0; k < kTcBatch; ++k)
      if (k2[k] != kNone && !(k2[k] & 0x80000000u)) c.elm[k2[k]] = v[k];
  }
}

// ------------------------------------------------------------ a2: forward
// Stage-0 pull pins (no fan-in): PI arrivals, ideal clock, or undefined.
__global__ void __launch_bounds__(kThreads) seed_kernel(Topo t, CornerDev c, uint32_t n0) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t s = i < n0 ? t.seed[i] : kNone;
  pdl_wait();
  pdl_launch();
  if (i >= n0) return;
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

// One launch per gate stage s >= 1: each thread merges the cell fan-in of
// one stage pin.  A fan-in pin that is a net sink is recomputed inline from
// its driver's record (pull-through), so sinks never cost a stage.
template <bool SMEM_LUT>
__global__ void __launch_bounds__(kThreads) fwd_stage_kernel(Topo t, CornerDev c, uint32_t pull0, uint32_t n,
                                                             uint32_t lut_f4) {
  const float* L = stage_lut<SMEM_LUT>(c, lut_f4);
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t v = pull0 + i;
  uint32_t e0 = 0, e1 = 0, src0 = 0, hop0 = kNone, info0 = 0;
  if (i < n) {                               // static topology: before the wait
    e0 = t.fi_ptr[v];
    e1 = t.fi_ptr[v + 1];
    if (e1 > e0) { src0 = t.fi_src[e0]; hop0 = t.fi_hop[e0]; info0 = t.fi_info[e0]; }
  }
  pdl_wait();
  pdl_launch();
  if (i >= n) return;
  const float ld = __ldcg(c.load + v);
  Q4 acc_at = undef_at(), acc_sl = undef_at();
  for (uint32_t e = e0; e < e1; ++e) {
    uint32_t src = src0, hop = hop0, info = info0;
    if (e != e0) { src = t.fi_src[e]; hop = t.fi_hop[e]; info = t.fi_info[e]; }
    Q4 at, sl;
    load_rec(c, src, at, sl);
    if (hop != kNone) net_hop(at, sl, __ldcg(c.elm + hop));
    cell_fwd(L, at, sl, info, ld, acc_at, acc_sl);
  }
  c.rec[2 * (size_t)v] = to_f4(acc_at);
  c.rec[2 * (size_t)v + 1] = to_f4(acc_sl);
}

// ---------------------------------------------- inter-block dataflow flags
// Persistent kernels publish completed work with a release store / atomic
// after a block barrier and a gpu-scope fence.  Consumers poll the flag with
// relaxed gpu-scope loads and, once it is set, read the produced records with
// wait until *f >= target (wrap-around safe)
// Exponential backoff (32 ns .. 1 us): a poller competes for issue slots with
// the working warps of its SM; without backoff polling was 15% of the
// forward kernel's instructions.
// polling backoff cap: a waiter notices a completed stage at most this late
constexpr uint32_t kMaxSleepNs = 128;

__device__ __forceinline__ void wait_ge(const uint32_t* f, uint32_t target) {
  if ((int)(ld_acquire(f) - target) >= 0) return;
  uint32_t ns = 32;
  while ((int)(ld_acquire(f) - target) < 0) {
    __nanosleep(ns);
    ns = ns < kMaxSleepNs ? 2 * ns : ns;
  }
}
// backward: every unit of the stage of pull pin w is complete
template <bool WAIT>
__device__ __forceinline__ void wait_pull(const Topo& t, const CornerDev& c, uint32_t w) {
  if (!WAIT) return;
  const uint32_t s = __ldg(t.chunk_stage + w / kChunk);
  wait_ge(c.bwd_done + s, __ldg(t.stage_units + s));
}

// ------------------------------------------------------ a3-a5: backward
// Finish a pull pin: own seed, direct cell fan-out, then rat / slack.
// e = pin_ep[v], [p0, p1) = its direct fan-out (prefetched by the caller).
template <bool WAIT>
__device__ __forceinline__ void finish_pull_pre(const Topo& t, const CornerDev& c, const float* L, uint32_t v,
                                                uint32_t e, uint32_t p0, uint32_t p1, const Q4& at, const Q4& sl,
                                                Q4 acc) {
  if (e != kNone) apply_seed(t, c, L, e, at, sl, acc);
  for (uint32_t x = p0; x < p1; ++x) {
    const uint32_t w = t.pfo_dst[x];
    wait_pull<WAIT>(t, c, w);
    cell_bwd(L, at, sl, t.pfo_info[x], __ldcg(c.load + w), to_q(__ldcg(c.rat + w)), acc);
  }
  c.rat[v] = to_f4(acc);
  const Q4 s = slack_of(at, acc);
  c.slack[v] = to_f4(s);
  if (e != kNone) write_ep(c, e, s);
}

template <bool WAIT>
__device__ __forceinline__ void finish_pull(const Topo& t, const CornerDev& c, const float* L, uint32_t v,
                                            const Q4& at, const Q4& sl, Q4 acc) {
  finish_pull_pre<WAIT>(t, c, L, v, t.pin_ep[v], t.pfo_ptr[v], t.pfo_ptr[v + 1], at, sl, acc);
}

__device__ __forceinline__ void combine(Q4& a, const Q4& b) {
  a.v[0] = fmaxf(a.v[0], b.v[0]);
  a.v[1] = fmaxf(a.v[1], b.v[1]);
  a.v[2] = fminf(a.v[2], b.v[2]);
  a.v[3] = fminf(a.v[3], b.v[3]);
}

// Static part of a backward tile lane (topology and RC results: readable
// before the previous stage ends), so that after the wait only the
// producers' records (driver AT/slew, fan-out RATs) remain to be loaded.
struct TileLane {
  uint2 td;
  uint32_t k, v, e, f0, f1, w0, info0, pe, p0, p1;
  float el, ld0;
  bool active;
  SeedPre seed;       // the sink's endpoint seed (static part)
};

__device__ __forceinline__ TileLane tile_lane(const Topo& t, uint32_t tile, uint32_t k1) {
  TileLane x;
  x.td = t.tiles[tile];
  x.k = x.td.x + (threadIdx.x & 31);
  x.active = x.k < k1;
  x.v = kNone; x.e = kNone; x.f0 = 0; x.f1 = 0; x.w0 = 0; x.info0 = 0; x.pe = kNone; x.p0 = 0; x.p1 = 0;
  x.el = 0.f; x.ld0 = 0.f;
  x.seed = SeedPre{undef_rat(), kNone};
  if (x.active) {
    x.v = t.sink_drv[x.k];
    x.e = t.pin_ep[t.NP + x.k];
    x.f0 = t.sfo_ptr[x.k];
    x.f1 = t.sfo_ptr[x.k + 1];
    x.pe = t.pin_ep[x.v];
    x.p0 = t.pfo_ptr[x.v];
    x.p1 = t.pfo_ptr[x.v + 1];
    x.seed = load_seed(t, x.e);
    if (x.f1 > x.f0) {
      x.w0 = t.sfo_dst[x.f0];
      x.info0 = t.sfo_info[x.f0];
    }
  }
  return x;
}

// RC results of a tile lane (written by the RC kernels of this update)
__device__ __forceinline__ void tile_lane_rc(const CornerDev& c, TileLane& x) {
  if (!x.active) return;
  x.el = __ldcg(c.elm + x.k);
  if (x.f1 > x.f0) x.ld0 = __ldcg(c.load + x.w0);
}

// One warp, one tile of <= 32 consecutive sinks of one stage's drivers: each
// lane owns one sink (required time from its endpoint seed and its cell
// fan-out, then rat / slack), and a segmented shuffle reduction by driver
// produces the drivers' required times.  Drivers with more than 32 sinks
// (heavy slot) combine their tiles with ordered-int atomics; the last tile
// finishes them.
template <bool WAIT>
__device__ __forceinline__ void process_tile(const Topo& t, const CornerDev& c, const float* L, const TileLane& x) {
  const int lane = threadIdx.x & 31;
  Q4 at_v = undef_at(), sl_v = undef_at(), acc = undef_rat();
  if (x.active) {
    Q4 rw0 = undef_rat();
    if (x.f1 > x.f0) {
      wait_pull<WAIT>(t, c, x.w0);
      rw0 = to_q(__ldcg(c.rat + x.w0));
    }
    load_rec(c, x.v, at_v, sl_v);
    Q4 at = at_v, sl = sl_v;
    net_hop(at, sl, x.el);                  // the sink's own arrival / slew
    Q4 r = undef_rat();
    if (x.e != kNone) apply_seed_pre(t, L, x.seed, at, sl, r);
    if (x.f1 > x.f0) cell_bwd(L, at, sl, x.info0, x.ld0, rw0, r);
    for (uint32_t f = x.f0 + 1; f < x.f1; ++f) {
      const uint32_t w = t.sfo_dst[f];
      wait_pull<WAIT>(t, c, w);
      cell_bwd(L, at, sl, t.sfo_info[f], __ldcg(c.load + w), to_q(__ldcg(c.rat + w)), r);
    }
    const size_t u = (size_t)t.NP + x.k;
    c.rat[u] = to_f4(r);
    const Q4 s = slack_of(at, r);
    c.slack[u] = to_f4(s);
    if (x.e != kNone) write_ep(c, x.e, s);
    // candidate of the driver through the net arc (only edges the forward used)
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (fin(at_v.v[q])) acc.v[q] = __fsub_rn(r.v[q], x.el);
  }
  // segmented inclusive scan by driver (drivers are contiguous in the tile)
  const uint32_t v = x.v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t vo = __shfl_up_sync(0xFFFFFFFFu, v, o);
    Q4 b;
#pragma unroll
    for (int q = 0; q < 4; ++q) b.v[q] = __shfl_up_sync(0xFFFFFFFFu, acc.v[q], o);
    if (lane >= o && vo == v) combine(acc, b);
  }
  const uint32_t vn = __shfl_down_sync(0xFFFFFFFFu, v, 1);
  const bool tail = x.active && (lane == 31 || vn != v);
  if (!tail) return;
  if (x.td.y == kNone) {                    // light driver: complete in this tile
    finish_pull_pre<WAIT>(t, c, L, v, x.pe, x.p0, x.p1, at_v, sl_v, acc);
    return;
  }
  const uint32_t slot = x.td.y;
  int* key = reinterpret_cast<int*>(c.heavy_key + slot);
  atomicMax(key + 0, f2o(acc.v[0]));
  atomicMax(key + 1, f2o(acc.v[1]));
  atomicMin(key + 2, f2o(acc.v[2]));
  atomicMin(key + 3, f2o(acc.v[3]));
  // release counter: orders this tile's key updates before it; only the last
  // tile pays the acquire fence before reading everyone's keys
  uint32_t done;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(done) : "l"(c.heavy_cnt + slot) : "memory");
  if (done + 1 != t.heavy_nchunk[slot]) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  Q4 a;
  a.v[0] = o2f(atomicExch(key + 0, f2o(-CUDART_INF_F)));
  a.v[1] = o2f(atomicExch(key + 1, f2o(-CUDART_INF_F)));
  a.v[2] = o2f(atomicExch(key + 2, f2o(CUDART_INF_F)));
  a.v[3] = o2f(atomicExch(key + 3, f2o(CUDART_INF_F)));
  c.heavy_cnt[slot] = 0;                    // self-reset for the next update
  finish_pull_pre<WAIT>(t, c, L, v, x.pe, x.p0, x.p1, at_v, sl_v, a);
}

// One launch per gate stage (descending).  Blocks [0, nTileBlocks): one warp
// per tile.  Remaining blocks: stage pins without sinks, one thread each.
template <bool SMEM_LUT>
__global__ void __launch_bounds__(kThreads) bwd_stage_kernel(Topo t, CornerDev c, uint32_t tile0, uint32_t nTiles,
                                                             uint32_t sinkEnd, uint32_t nos0, uint32_t nNos,
                                                             uint32_t nTileBlocks, uint32_t lut_f4) {
  const float* L = stage_lut<SMEM_LUT>(c, lut_f4);
  if (blockIdx.x >= nTileBlocks) {
    const uint32_t i = (blockIdx.x - nTileBlocks) * blockDim.x + threadIdx.x;
    const uint32_t v = i < nNos ? t.nosink[nos0 + i] : 0;
    pdl_wait();
    pdl_launch();
    if (i >= nNos) return;
    Q4 at, sl;
    load_rec(c, v, at, sl);
    finish_pull<false>(t, c, L, v, at, sl, undef_rat());
    return;
  }
  const uint32_t tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  TileLane x{};
  if (tile < nTiles) x = tile_lane(t, tile0 + tile, tile + 1 < nTiles ? t.tiles[tile0 + tile + 1].x : sinkEnd);
  pdl_wait();
  pdl_launch();
  if (tile >= nTiles) return;
  tile_lane_rc(c, x);
  process_tile<false>(t, c, L, x);
}

// ---------------------------------------------- persistent dataflow passes
// Grid = co-resident blocks (cooperative launch).  Work items are processed in
// dependency order (block b takes items b, b + G, ...), every item depends
// only on items with a smaller index, and all blocks are resident, so the
// smallest unfinished item can always proceed: no deadlock, no grid barrier.


// Block-level readiness.  Each block is a worker; its warp 0 checks the
// per-stage completion counters of the stages a unit depends on, 32 stages
// per L2 round trip (one per lane), with a per-block watermark of stages
// already seen complete; the block continues after a barrier.  A finished
// unit publishes with a barrier and one red.release.gpu (orders the block's
// stores through MEMBAR.ALL.GPU without the L1 invalidation a fence.acq_rel /
// __threadfence adds).  Per-warp units (one release per 32 items) and
// per-thread polling both measured 1.7-2x slower on C3.
__device__ __forceinline__ void block_wait_fwd(const Topo& t, const CornerDev& c, uint32_t stage, uint32_t* s_wm) {
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    uint32_t wm = *s_wm, ns = 32;
    while (wm < stage) {                     // every stage < stage must be complete
      const uint32_t q = wm + lane;
      const bool ok = q >= stage || (int)(ld_acquire(c.fwd_done + q) - __ldg(t.stage_chunks + q)) >= 0;
      const uint32_t miss = __ballot_sync(0xFFFFFFFFu, !ok);
      if (!miss) {
        wm = min(stage, wm + 32);
      } else {
        wm += __ffs(miss) - 1;
        __nanosleep(ns);
        ns = ns < kMaxSleepNs ? 2 * ns : ns;
      }
    }
    if (lane == 0) *s_wm = wm;
  }
  __syncthreads();
}

__device__ __forceinline__ void block_wait_bwd(const Topo& t, const CornerDev& c, uint32_t stage, uint32_t* s_wm) {
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    uint32_t wm = *s_wm, ns = 32;
    while (wm > stage + 1) {                 // every stage > stage must be complete
      const int q = (int)wm - 1 - (int)lane;
      const bool ok = q <= (int)stage || (int)(ld_acquire(c.bwd_done + q) - __ldg(t.stage_units + q)) >= 0;
      const uint32_t miss = __ballot_sync(0xFFFFFFFFu, !ok);
      if (!miss) {
        wm = max(stage + 1, wm > 32 ? wm - 32 : 0u);
      } else {
        wm -= __ffs(miss) - 1;
        __nanosleep(ns);
        ns = ns < kMaxSleepNs ? 2 * ns : ns;
      }
    }
    if (lane == 0) *s_wm = wm;
  }
  __syncthreads();
}

__device__ __forceinline__ void block_publish(uint32_t* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}

// forward merge: early components take the min, late the max
__device__ __forceinline__ void merge_fwd(Q4& a, const Q4& b) {
  a.v[0] = fminf(a.v[0], b.v[0]);
  a.v[1] = fminf(a.v[1], b.v[1]);
  a.v[2] = fmaxf(a.v[2], b.v[2]);
  a.v[3] = fmaxf(a.v[3], b.v[3]);
}

// One fan-in term of the forward pass, both modes: the candidates of the
// term's cell arc for every (el, orf), merged into acc_at / acc_sl (early
// min, late max).  Same seg / interp calls as cell_fwd / cell_bwd
// (bit-identical); branch-free: lookups of undefined inputs are computed and
// discarded by select, so a warp never diverges on them.
__device__ __forceinline__ void cell_term(const float* __restrict__ L, const Q4& at, const Q4& sl, uint32_t info,
                                          float ld, Q4& acc_at, Q4& acc_sl) {
  const uint32_t sense = info & 7u, tab = info >> 3;
  const Tab rd0 = tab_rec(L, tab), rd1 = tab_rec(L, tab + 1);
  const Tab rs0 = tab_rec(L, tab + 2), rs1 = tab_rec(L, tab + 3);
  const Seg cd0 = seg(rd0.ax + 24, ld);
  const Seg cd1 = rd1.ax == rd0.ax ? cd0 : seg(rd1.ax + 24, ld);
  const Seg cs0 = rs0.ax == rd0.ax ? cd0 : seg(rs0.ax + 24, ld);
  const Seg cs1 = rs1.ax == rd1.ax ? cd1 : seg(rs1.ax + 24, ld);
#pragma unroll
  for (int orf = 0; orf < 2; ++orf) {
    const int irf = primary_irf(sense, orf);
    const Tab rd = orf ? rd1 : rd0;
    const Tab rs = orf ? rs1 : rs0;
    const bool same = rs.ax == rd.ax;
#pragma unroll
    for (int el = 0; el < 2; ++el) {
      const float a_in = irf ? at.v[el * 2 + 1] : at.v[el * 2];
      const float s_in = irf ? sl.v[el * 2 + 1] : sl.v[el * 2];
      const Seg sd = seg(rd.ax, s_in);
      const Seg ss = same ? sd : seg(rs.ax, s_in);
      const float d = fmaxf(0.f, interp(rd, sd, orf ? cd1 : cd0));
      const float so = fmaxf(0.f, interp(rs, ss, orf ? cs1 : cs0));
      const float ca = __fadd_rn(a_in, d);
      const bool ok = fin(a_in);
      const int q = el * 2 + orf;
      if (el == 0) {
        acc_at.v[q] = ok ? fminf(acc_at.v[q], ca) : acc_at.v[q];
        acc_sl.v[q] = ok ? fminf(acc_sl.v[q], so) : acc_sl.v[q];
      } else {
        acc_at.v[q] = ok ? fmaxf(acc_at.v[q], ca) : acc_at.v[q];
        acc_sl.v[q] = ok ? fmaxf(acc_sl.v[q], so) : acc_sl.v[q];
      }
    }
  }
}

// Forward pass.  A chunk is a run of pins of one stage whose fan-in terms fit
// the block: phase 1 evaluates one term per thread (one cell arc, both
// modes), phase 2 merges each pin's terms from shared memory.  This keeps
// the per-thread dependent chain to one arc.  A pin with more than 256 terms
// has a chunk of its own and its terms are looped over.
template <bool SMEM_LUT>
__global__ void __launch_bounds__(kThreads, 4) fwd_persistent_kernel(Topo t, CornerDev c, uint32_t lut_f4) {
  __shared__ uint32_t s_wm;
  __shared__ float4 s_at[kThreads], s_sl[kThreads];
  const float* L = stage_lut<SMEM_LUT>(c, lut_f4);
  if (threadIdx.x == 0) s_wm = 0;
  for (uint32_t ch = blockIdx.x; ch < t.n_fchunks; ch += gridDim.x) {
    unsigned long long t_start = 0, t_ready = 0;
    if (c.trace && threadIdx.x == 0) t_start = gtimer();
    const uint4 fc = t.fchunks[ch];          // {pin0, npins, term0, nterms}
    const uint32_t stage = t.fchunk_stage[ch];
    if (stage == 0) {                        // seeds: PI arrivals, ideal clock, undefined
      if (threadIdx.x < fc.y) {
        const uint32_t v = fc.x + threadIdx.x;
        const uint32_t s = t.seed[v];
        Q4 at = undef_at(), sl = undef_at();
        if (s == kSeedClock) {
          const float h = 0.5f * t.period;
          at = Q4{{0.f, h, 0.f, h}};
          sl = Q4{{t.clock_slew, t.clock_slew, t.clock_slew, t.clock_slew}};
        } else if (s != kNone) {
          at = to_q(t.pi_at[s]);
          sl = to_q(t.pi_slew[s]);
        }
        c.rec[2 * (size_t)v] = to_f4(at);
        c.rec[2 * (size_t)v + 1] = to_f4(sl);
      }
      block_publish(c.fwd_done);
      continue;
    }
    if (fc.w <= kThreads) {
      // static topology and RC results before waiting for the producers
      const bool item = threadIdx.x < fc.w;
      uint32_t src = 0, info = 0;
      float elm = 0.f, ld = 0.f;
      bool hop = false;
      if (item) {
        const uint32_t e = fc.z + threadIdx.x;
        src = t.fi_src[e];
        info = t.fi_info[e];
        const uint32_t h = t.fi_hop[e];
        hop = h != kNone;
        if (hop) elm = __ldcg(c.elm + h);
        ld = __ldcg(c.load + t.fi_pin[e]);
      }
      uint32_t pv = 0, i0 = 0, i1 = 0;
      if (threadIdx.x < fc.y) {
        pv = fc.x + threadIdx.x;
        i0 = t.fi_ptr[pv] - fc.z;
        i1 = t.fi_ptr[pv + 1] - fc.z;
      }
      block_wait_fwd(t, c, stage, &s_wm);
      if (c.trace && threadIdx.x == 0) t_ready = gtimer();
      if (item) {
        Q4 at, sl;
        load_rec(c, src, at, sl);
        if (hop) net_hop(at, sl, elm);
        Q4 acc_at = undef_at(), acc_sl = undef_at();
        cell_term(L, at, sl, info, ld, acc_at, acc_sl);
        s_at[threadIdx.x] = to_f4(acc_at);
        s_sl[threadIdx.x] = to_f4(acc_sl);
      }
      __syncthreads();
      if (threadIdx.x < fc.y) {
        Q4 acc_at = undef_at(), acc_sl = undef_at();
        for (uint32_t i = i0; i < i1; ++i) {
          merge_fwd(acc_at, to_q(s_at[i]));
          merge_fwd(acc_sl, to_q(s_sl[i]));
        }
        if (i1 > i0) {                       // padding pins (no terms) are never read
          c.rec[2 * (size_t)pv] = to_f4(acc_at);
          c.rec[2 * (size_t)pv + 1] = to_f4(acc_sl);
        }
      }
    } else {                                 // one pin with > 256 terms: block loop
      block_wait_fwd(t, c, stage, &s_wm);
      if (c.trace && threadIdx.x == 0) t_ready = gtimer();
      const float ld = __ldcg(c.load + fc.x);
      Q4 acc_at = undef_at(), acc_sl = undef_at();
      for (uint32_t e = fc.z + threadIdx.x; e < fc.z + fc.w; e += blockDim.x) {
        const uint32_t h = t.fi_hop[e];
        Q4 at, sl;
        load_rec(c, t.fi_src[e], at, sl);
        if (h != kNone) net_hop(at, sl, __ldcg(c.elm + h));
        cell_term(L, at, sl, t.fi_info[e], ld, acc_at, acc_sl);
      }
      s_at[threadIdx.x] = to_f4(acc_at);
      s_sl[threadIdx.x] = to_f4(acc_sl);
      __syncthreads();
      if (threadIdx.x == 0) {
        for (uint32_t i = 1; i < blockDim.x; ++i) {
          merge_fwd(acc_at, to_q(s_at[i]));
          merge_fwd(acc_sl, to_q(s_sl[i]));
        }
        c.rec[2 * (size_t)fc.x] = to_f4(acc_at);
        c.rec[2 * (size_t)fc.x + 1] = to_f4(acc_sl);
      }
    }
    if (c.trace) {                           // debug: time when the whole block computed
      __syncthreads();
      if (threadIdx.x == 0) t_start = gtimer();
    }
    block_publish(c.fwd_done + stage);
    if (c.trace && threadIdx.x == 0) {
      c.trace[3 * (size_t)ch] = t_start;
      c.trace[3 * (size_t)ch + 1] = t_ready;
      c.trace[3 * (size_t)ch + 2] = gtimer();
    }
  }
}

// Backward pass.  A unit is up to 8 tiles (one warp each, process_tile) or
// up to 256 sink-less pins of one stage (one thread each).
template <bool SMEM_LUT>
__global__ void __launch_bounds__(kThreads, 4) bwd_persistent_kernel(Topo t, CornerDev c, uint32_t lut_f4) {
  __shared__ uint32_t s_wm;
  const float* L = stage_lut<SMEM_LUT>(c, lut_f4);
  if (threadIdx.x == 0) s_wm = t.S;
  for (uint32_t u = blockIdx.x; u < t.n_units; u += gridDim.x) {
    unsigned long long t_start = 0, t_ready = 0;
    if (c.trace && threadIdx.x == 0) t_start = gtimer();
    const uint4 ud = t.units[u];             // {stage, kind, first, count}
    const uint32_t w = threadIdx.x >> 5;
    TileLane x{};
    uint32_t v = 0, pe = kNone, p0 = 0, p1 = 0;
    if (ud.y == 0) {                         // static part before waiting
      if (w < ud.w) {
        const uint32_t tile = ud.z + w;
        const uint32_t k1 = tile + 1 < t.stage_tile_end[ud.x] ? t.tiles[tile + 1].x : t.stage_sink_end[ud.x];
        x = tile_lane(t, tile, k1);
        tile_lane_rc(c, x);
      }
    } else if (threadIdx.x < ud.w) {
      v = t.nosink[ud.z + threadIdx.x];
      pe = t.pin_ep[v];
      p0 = t.pfo_ptr[v];
      p1 = t.pfo_ptr[v + 1];
    }
    block_wait_bwd(t, c, ud.x, &s_wm);
    if (c.trace && threadIdx.x == 0) t_ready = gtimer();
    if (ud.y == 0) {
      if (w < ud.w) process_tile<false>(t, c, L, x);
    } else if (threadIdx.x < ud.w) {
      Q4 at, sl;
      load_rec(c, v, at, sl);
      finish_pull_pre<false>(t, c, L, v, pe, p0, p1, at, sl, undef_rat());
    }
    block_publish(c.bwd_done + ud.x);
    if (c.trace && threadIdx.x == 0) {
      const size_t q = 3 * ((size_t)t.n_fchunks + u);
      c.trace[q] = t_start;
      c.trace[q + 1] = t_ready;
      c.trace[q + 2] = gtimer();
    }
  }
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

__global__ void __launch_bounds__(kThreads) reduce_kernel(Topo t, CornerDev c) {
  constexpr int kU = 4;                      // loads in flight per thread
  __shared__ double s_t[2][kThreads];
  __shared__ float s_w[2][kThreads];
  __shared__ bool last;
  pdl_wait();
  pdl_launch();
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
    *c.red_cnt = 0;                         // self-reset for the next update
  }
  for (uint32_t x = threadIdx.x; x < t.S; x += blockDim.x) {   // stage counters: ready for the next update
    c.bwd_done[x] = 0;
    c.fwd_done[x] = 0;
  }
}

// ----------------------------------------------------- outputs / setup
// what: 0 at, 1 slew, 2 rat, 3 slack, in user pin order; sink arrivals and
// slews are recomputed from their drivers exactly as the kernels do.
__global__ void gather_pins_kernel(Topo t, CornerDev c, int what, float4* __restrict__ dst) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= t.P) return;
  const uint32_t i = t.int_of_user[p];
  if (what >= 2) {
    dst[p] = what == 2 ? c.rat[i] : c.slack[i];
    return;
  }
  if (i < t.NP) {
    dst[p] = c.rec[2 * (size_t)i + what];
    return;
  }
  const uint32_t k = i - t.NP;
  Q4 at, sl;
  load_rec(c, t.sink_drv[k], at, sl);
  net_hop(at, sl, c.elm[k]);
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
  if (i < n_heavy) {
    c.heavy_key[i] = make_int4(f2o(-CUDART_INF_F), f2o(-CUDART_INF_F), f2o(CUDART_INF_F), f2o(CUDART_INF_F));
    c.heavy_cnt[i] = 0;
  }
  if (i == 0) {
    *c.red_cnt = 0;
    *c.err_flag = 0;
  }
}

inline uint32_t blocks(uint64_t n, uint32_t th = kThreads) { return (uint32_t)((n + th - 1) / th); }

// launch with programmatic dependent launch enabled
template <class K, class... A>
cudaError_t pdl_launch_smem(K kernel, uint32_t grid, uint32_t block, size_t smem, cudaStream_t s, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
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
cudaError_t pdl_launch_kernel(K kernel, uint32_t grid, uint32_t block, cudaStream_t s, A... args) {
  return pdl_launch_smem(kernel, grid, block, 0, s, args...);
}

}  // namespace

cudaError_t launch_rc(const Topo& t, const CornerDev& c, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (t.n_wtiles && e == cudaSuccess) e = pdl_launch_kernel(rc_warp_kernel, blocks(32ull * t.n_wtiles), kThreads, s, t, c);
  if (t.n_btiles && e == cudaSuccess) e = pdl_launch_kernel(rc_block_kernel, t.n_btiles, kThreads, s, t, c);
  if (t.n_lumped && e == cudaSuccess) e = pdl_launch_kernel(rc_lumped_kernel, blocks(t.n_lumped), kThreads, s, t, c);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_rc_tierC(const Topo& t, const CornerDev& c, cudaStream_t s) {
  if (!t.nC) return cudaSuccess;
  static uint32_t grid = 0;
  if (!grid) {
    int dev = 0, sms = 0, nb = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tc_persistent_kernel, kTcThreads, 0);
    grid = (uint32_t)std::min<int>(std::max(nb, 0) * sms, (int)kTcMaxGrid);
    if (!grid) return cudaErrorCooperativeLaunchTooLarge;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.stream = s;
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = prio;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_persistent_kernel, t, c);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_seed(const Topo& t, const CornerDev& c, uint32_t n0, cudaStream_t s) {
  if (!n0) return cudaSuccess;
  return pdl_launch_kernel(seed_kernel, blocks(n0), kThreads, s, t, c, n0);
}

cudaError_t launch_fwd_stage(const Topo& t, const CornerDev& c, uint32_t pull0, uint32_t n, uint32_t lut_f4,
                             cudaStream_t s) {
  if (!n) return cudaSuccess;
  if (lut_f4) return pdl_launch_smem(fwd_stage_kernel<true>, blocks(n), kThreads, 16ull * lut_f4, s, t, c, pull0, n, lut_f4);
  return pdl_launch_smem(fwd_stage_kernel<false>, blocks(n), kThreads, 0, s, t, c, pull0, n, lut_f4);
}

cudaError_t launch_bwd_stage(const Topo& t, const CornerDev& c, uint32_t tile0, uint32_t nTiles, uint32_t sinkEnd,
                             uint32_t nos0, uint32_t nNos, uint32_t lut_f4, cudaStream_t s) {
  const uint32_t tb = blocks((uint64_t)nTiles * 32);
  const uint32_t nb = blocks(nNos);
  if (!(tb + nb)) return cudaSuccess;
  if (lut_f4)
    return pdl_launch_smem(bwd_stage_kernel<true>, tb + nb, kThreads, 16ull * lut_f4, s, t, c, tile0, nTiles, sinkEnd,
                           nos0, nNos, tb, lut_f4);
  return pdl_launch_smem(bwd_stage_kernel<false>, tb + nb, kThreads, 0, s, t, c, tile0, nTiles, sinkEnd, nos0, nNos, tb,
                         lut_f4);
}

cudaError_t launch_reduce(const Topo& t, const CornerDev& c, cudaStream_t s) {
  return pdl_launch_kernel(reduce_kernel, (uint32_t)kRedBlocks, kThreads, s, t, c);
}

cudaError_t launch_gather_pins(const Topo& t, const CornerDev& c, int what, float4* dst, cudaStream_t s) {
  if (t.P) gather_pins_kernel<<<blocks(t.P), kThreads, 0, s>>>(t, c, what, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather_rc(const Topo& t, const CornerDev& c, float* net_load, float* pin_elm, cudaStream_t s) {
  const uint32_t n = t.N > t.P ? t.N : t.P;
  if (n) gather_rc_kernel<<<blocks(n), kThreads, 0, s>>>(t, c, net_load, pin_elm);
  return cudaGetLastError();
}

// co-resident grid of the persistent forward (which = 0) or backward (1)
// kernel: blocks per SM from the occupancy calculator x SMs; 0 if unsupported
uint32_t persistent_grid(uint32_t lut_f4, int which) {
  int dev = 0, sms = 0, nb = 0, coop = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return 0;
  const size_t smem = 16ull * lut_f4;
  if (which == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, lut_f4 ? fwd_persistent_kernel<true> : fwd_persistent_kernel<false>, kThreads, lut_f4 ? smem : 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &nb, lut_f4 ? bwd_persistent_kernel<true> : bwd_persistent_kernel<false>, kThreads, lut_f4 ? smem : 0);
  cudaGetLastError();
  return (uint32_t)(nb * sms);
}

template <class K>
cudaError_t coop_launch(K kernel, uint32_t grid, size_t smem, cudaStream_t s, const Topo& t, const CornerDev& c,
                        uint32_t lut_f4) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, t, c, lut_f4);
}

cudaError_t launch_fwd_persistent(const Topo& t, const CornerDev& c, uint32_t grid, uint32_t lut_f4, cudaStream_t s) {
  if (!t.NP) return cudaSuccess;
  return lut_f4 ? coop_launch(fwd_persistent_kernel<true>, grid, 16ull * lut_f4, s, t, c, lut_f4)
                : coop_launch(fwd_persistent_kernel<false>, grid, 0, s, t, c, lut_f4);
}

cudaError_t launch_bwd_persistent(const Topo& t, const CornerDev& c, uint32_t grid, uint32_t lut_f4, cudaStream_t s) {
  if (!t.n_units) return cudaSuccess;
  return lut_f4 ? coop_launch(bwd_persistent_kernel<true>, grid, 16ull * lut_f4, s, t, c, lut_f4)
                : coop_launch(bwd_persistent_kernel<false>, grid, 0, s, t, c, lut_f4);
}

cudaError_t set_lut_smem_limit(size_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(fwd_stage_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bwd_stage_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fwd_persistent_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bwd_persistent_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return e;
}

cudaError_t launch_init_corner(const Topo&, const CornerDev& c, uint32_t n_heavy, cudaStream_t s) {
  init_corner_kernel<<<blocks(n_heavy + 1), kThreads, 0, s>>>(c, n_heavy);
  return cudaGetLastError();
}

}  // namespace sta
