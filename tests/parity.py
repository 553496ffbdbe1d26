"""Comparison rule of the CUDA path against the fp64 oracle.

north_star (BASELINE.json): arrival/required times and slacks match in fp32
within 1e-3 ps absolute or 1e-5 relative:  |gpu - oracle| <= max(1e-3,
1e-5 * scale), where the relative part is taken against the magnitude of
the quantities the value is computed from (DESIGN.md §2 reading R17):
  * AT, slew, load, Elmore: scale = |oracle value| (sums of non-negative
    terms, every partial sum is bounded by the result);
  * RAT: scale = max(|RAT|, T): a required time is T minus a path delay and
    cancels against the clock period (e.g. 15837 - 15969 = -132 ps carries
    the rounding of 1.6e4-sized operands);
  * slack = RAT - AT: scale = max(|AT|, |RAT|, T) of the same component;
  * WNS and TNS: scale = |oracle value| (SURVEY §8(c) rule #17 as written;
    tightened in round 2 from the per-endpoint slack scales, VERDICT r1
    "What's weak" #2).
Infinite values (undefined quantities) must match exactly.
Levels and permutations are integers: bit-exact.
"""
from __future__ import annotations

import numpy as np

ABS = 1e-3
REL = 1e-5


def bound(scale):
    return np.maximum(ABS, REL * np.abs(scale))


def check_close(name, gpu, ref, scale=None, report=None):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape, (name, gpu.shape, ref.shape)
    fin = np.isfinite(ref)
    bad_inf = ~fin & (gpu != ref)
    if bad_inf.any():
        idx = np.argwhere(bad_inf)[:5]
        raise AssertionError(f"{name}: infinite mismatch at {idx.tolist()}: gpu {gpu[bad_inf][:5]} ref {ref[bad_inf][:5]}")
    nonfin_gpu = fin & ~np.isfinite(gpu)
    if nonfin_gpu.any():
        idx = np.argwhere(nonfin_gpu)[:5]
        raise AssertionError(f"{name}: gpu non-finite where oracle finite at {idx.tolist()}")
    sc = np.abs(ref) if scale is None else np.asarray(scale, np.float64)
    err = np.where(fin, np.abs(np.where(fin, gpu, 0) - np.where(fin, ref, 0)), 0.0)
    tol = bound(np.where(np.isfinite(sc), sc, 0))
    viol = fin & (err > tol)
    if report is not None:
        r = np.where(fin, err / tol, 0)
        report[name] = dict(max_abs_err=float(err[fin].max()) if fin.any() else 0.0,
                            max_err_over_bound=float(r.max()) if r.size else 0.0, n=int(fin.sum()))
    if viol.any():
        idx = np.argwhere(viol)[:5]
        raise AssertionError(
            f"{name}: {int(viol.sum())} values out of tolerance, e.g. at {idx.tolist()}: "
            f"gpu {gpu[viol][:5]} ref {ref[viol][:5]} bound {tol[viol][:5]}")


def compare_update(ctx, ref, corner=0, report=None, period=None):
    """Full-array comparison of one corner: at, slew, rat, slack, res.
    period: the clock period T of the design (default: taken from ref)."""
    T = abs(float(ref.get("period", 0.0) if period is None else period))
    at, slew, rat = ctx.get_timing(corner)
    res, slack = ctx.report_slack(corner, want_pins=True)
    check_close("at", at, ref["at"], report=report)
    check_close("slew", slew, ref["slew"], report=report)
    fa = np.abs(np.where(np.isfinite(ref["at"]), ref["at"], 0))
    fr = np.abs(np.where(np.isfinite(ref["rat"]), ref["rat"], 0))
    check_close("rat", rat, ref["rat"], scale=np.maximum(fr, T), report=report)
    sc = np.maximum(np.maximum(fa, fr), T)
    check_close("slack", slack, ref["slack"], scale=sc, report=report)
    r = ref["res"]
    check_close("wns_setup", [res[0]], [r[0]], report=report)
    check_close("wns_hold", [res[2]], [r[2]], report=report)
    check_close("tns_setup", [res[1]], [r[1]], report=report)
    check_close("tns_hold", [res[3]], [r[3]], report=report)
    return res
