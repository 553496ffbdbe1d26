// sta_arnoldi.cuh -- NEXT row f1: the net-arc delay / slew of the Arnoldi
// reduced-order model (SPEC.md:407-418,
// readings A1-A7 in DESIGN.md), evaluated wherever a sink's arrival is
// needed (the forward's term lanes, the backward's sink lanes): the model
// H(s) = sum_k res_k / (1 + s lam_k) (lam: time constants, ps; res: the
// sink's residues, sum 1) driven by a saturated ramp whose 20-80 slew is the
// driver's slew s (duration D = s / 0.6): delay = t50(out) - D / 2, slew =
// t80 - t20.  Crossings by safeguarded Newton in fp32 (the response and its
// derivative in closed form, expm1-based so the small-t region keeps its
// precision).  Every caller uses these __noinline__ functions, so a sink's
// delay is bit-identical wherever it is recomputed.
#pragma once
#include <cuda_runtime.h>

namespace sta {

// per-term constants of one crossing solve: 1 / lam, and e^{D/lam} - 1 for
// the post-ramp tail while D / lam < 1
struct ArnTerm {
  float k, l, il, eD;
  bool live, small;
};

// y(t) and y'(t) of the ramp response, order <= 4 (terms with residue 0 skipped)
__device__ __forceinline__ void arn_resp(const ArnTerm (&T)[4], float D, float t, float& y, float& dy) {
  y = 0.f;
  dy = 0.f;
  if (t <= 0.f) return;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!T[k].live) continue;
    const float l = T[k].l;
    float g, dg;
    if (D <= 0.f) {                            // a step
      if (l > 0.f) {
        const float x = t * T[k].il;
        const float e = __expf(-x);
        g = x < 0.25f ? -expm1f(-x) : 1.f - e;
        dg = e * T[k].il;
      } else {
        g = 1.f;
        dg = 0.f;
      }
    } else if (t <= D) {                       // on the ramp: (t - l (1 - e^{-t/l})) / D
      if (l > 0.f) {
        const float x = t * T[k].il;
        const float om = x < 0.25f ? -expm1f(-x) : 1.f - __expf(-x);
        g = (t - l * om) / D;
        dg = om / D;
      } else {
        g = t / D;
        dg = 1.f / D;
      }
    } else {                                   // after it: 1 - (l / D) (e^{-(t-D)/l} - e^{-t/l})
      if (l > 0.f) {
        // e^{-t/l} expm1(D/l) while D/l < 1 (no cancellation, no overflow),
        // the plain difference beyond (its cancellation is bounded there)
        const float et = __expf(-t * T[k].il);
        const float a = T[k].small ? et * T[k].eD : __expf(-(t - D) * T[k].il) - et;
        g = 1.f - (l / D) * a;
        dg = a / D;
      } else {
        g = 1.f;
        dg = 0.f;
      }
    }
    y += T[k].k * g;
    dy += T[k].k * dg;
  }
}

// first time the response reaches theta: Newton inside a shrinking bracket
// (bisection when a step leaves it), from the single-pole estimate with the
// model's first moment
__device__ __noinline__ float arn_cross(float4 lam, float4 res, float D, float theta) {
  const float L[4] = {lam.x, lam.y, lam.z, lam.w}, K[4] = {res.x, res.y, res.z, res.w};
  ArnTerm T[4];
  float lmax = 0.f, m1 = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    T[k].k = K[k];
    T[k].l = L[k];
    T[k].live = K[k] != 0.f;
    T[k].il = L[k] > 0.f ? 1.f / L[k] : 0.f;
    const float r = L[k] > 0.f ? D * T[k].il : 2.f;
    T[k].small = r < 1.f;
    T[k].eD = T[k].small ? expm1f(r) : 0.f;
    if (T[k].live) {
      lmax = fmaxf(lmax, L[k]);
      m1 += K[k] * L[k];
    }
  }
  float lo = 0.f, hi = D + 50.f * lmax + 1e-3f;
  float y, dy;
  for (int g = 0; g < 24; ++g) {
    arn_resp(T, D, hi, y, dy);
    if (y >= theta) break;
    hi *= 2.f;
  }
  float t = fminf(fmaxf(theta * D + __logf(1.f / (1.f - theta)) * fmaxf(m1, 0.f), 1e-6f), 0.5f * hi);
  for (int it = 0; it < 40; ++it) {
    arn_resp(T, D, t, y, dy);
    if (y >= theta) hi = t;
    else lo = t;
    if (y == theta) break;
    float tn = dy > 0.f ? t - (y - theta) / dy : 0.5f * (lo + hi);
    if (!(tn > lo && tn < hi)) tn = 0.5f * (lo + hi);
    const float step = fabsf(tn - t);
    t = tn;
    if (step <= 3e-7f * fmaxf(t, 1e-3f) || hi - lo <= 3e-7f * fmaxf(hi, 1e-3f)) break;
  }
  return t;
}

__device__ __forceinline__ float arn_duration(float s) { return __fdiv_rn(s, 0.6f); }

// the net-arc delay for a driver slew s (bit-identical in every caller)
__device__ __noinline__ float arn_delay(float4 lam, float4 res, float s) {
  const float D = arn_duration(s);
  return __fsub_rn(arn_cross(lam, res, D, 0.5f), __fmul_rn(0.5f, D));
}

// the sink's 20-80 slew
__device__ __noinline__ float arn_slew(float4 lam, float4 res, float s) {
  const float D = arn_duration(s);
  return __fsub_rn(arn_cross(lam, res, D, 0.8f), arn_cross(lam, res, D, 0.2f));
}

}  // namespace sta
