"""GPU parity of the top-k path report (SURVEY.md §8(f) row 3,
sta_report_paths) against the oracle's O10 report.

fp32 (GPU) and fp64 (oracle) sums can order near-equal slacks differently,
so the comparison is tolerance-aware: the i-th slacks agree within
max(1e-3, 1e-5 * scale) (scale = max(|slack|, T)), every GPU path is one of
the oracle's (extended by 64 paths past k) with the same slack, and every
oracle path clearly inside the GPU's slack range is reported.

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import numpy as np
import pytest

import oracle
import synth
from synth import variants
from tests.test_gpu_parity import run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sta():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 (there is no CPU fallback)")
    import paper_2511_11660_b200 as pkg
    return pkg


def _tol(s, T):
    return max(1e-3, 1e-5 * max(abs(s), abs(T)))


def compare_paths(gpu, ora_ext, k, T):
    key = lambda p: (p["ep"], tuple(p["pins"]), tuple(p["rfs"]))
    assert len(gpu) == min(k, len(ora_ext)), (len(gpu), len(ora_ext), k)
    for g, o in zip(gpu, ora_ext):
        assert abs(g["slack"] - o["slack"]) <= _tol(o["slack"], T), (g["slack"], o["slack"])
    omap = {key(p): p for p in ora_ext}
    for g in gpu:
        o = omap.get(key(g))
        assert o is not None, ("GPU path not in the oracle's report", g)
        assert abs(g["slack"] - o["slack"]) <= _tol(o["slack"], T)
        assert np.allclose(g["at"], o["at"], rtol=1e-5, atol=1e-3)
    if gpu:
        last = gpu[-1]["slack"]
        gkeys = {key(g) for g in gpu}
        for o in ora_ext:
            if o["slack"] < last - 2 * _tol(last, T):
                assert key(o) in gkeys, ("oracle path missing on the GPU", o)


def check(sta, ctx, d, corner=0, ks=((1, 1), (10, 2), (50, 4), (200, 1))):
    T = float(d.cons.period)
    res, _ = ctx.report_slack(corner)
    for mode in ("setup", "hold"):
        for k, nw in ks:
            g = ctx.report_paths(corner, mode=mode, k=k, nworst=nw)
            o = oracle.paths(d, corner, mode=mode, k=k + 64, nworst=nw)
            compare_paths(g, o, k, T)
            if g:
                # the worst path IS the worst endpoint slack (same fp32 sums)
                w = res[0] if mode == "setup" else res[2]
                assert g[0]["slack"] == pytest.approx(w, abs=_tol(w, T))
                sl = [p["slack"] for p in g]
                assert all(a <= b for a, b in zip(sl, sl[1:]))


@pytest.mark.parametrize("seed", range(6))
def test_paths_random_small(sta, seed):
    d = synth.generate(400 + 50 * seed, 14, seed=300 + seed, frac_pi=0.05, frac_po=0.05, period=150.0)
    ctx = run(sta, d)
    check(sta, ctx, d)
    ctx.close()


def test_paths_hand_examples(sta):
    for d in (synth.h1_chain(), synth.c17(), synth.h3_reg2reg(), synth.h4_seeds()):
        ctx = run(sta, d)
        check(sta, ctx, d, ks=((1, 1), (20, 20)))
        ctx.close()


def test_paths_slack_threshold_and_odd_tables(sta):
    d = variants.odd_tables(synth.generate(2000, 20, seed=77, period=250.0), 5)
    ctx = run(sta, d)
    T = float(d.cons.period)
    allp = oracle.paths(d, mode="setup", k=400, nworst=3)
    # a threshold inside a gap of the oracle's slacks (fp32 and fp64 must not
    # disagree about which side a path falls on)
    i = len(allp) // 3
    while i + 1 < len(allp) and allp[i + 1]["slack"] - allp[i]["slack"] < 4 * _tol(allp[i]["slack"], T):
        i += 1
    thr = 0.5 * (allp[i]["slack"] + allp[min(i + 1, len(allp) - 1)]["slack"])
    g = ctx.report_paths(0, mode="setup", k=300, nworst=3, slack_lt=thr)
    assert all(p["slack"] < thr for p in g)
    compare_paths(g, [p for p in oracle.paths(d, mode="setup", k=364, nworst=3) if p["slack"] < thr],
                  min(300, sum(p["slack"] < thr for p in allp)), T)
    check(sta, ctx, d)


def test_paths_multicorner(sta):
    d = synth.generate(3000, 24, seed=19, corners=3, corner_recipe="c5", period=250.0)
    ctx = run(sta, d)
    for c in range(3):
        check(sta, ctx, d, corner=c, ks=((20, 2),))


def test_paths_c2_tau(sta):
    """BASELINE configs[1] (TAU-shaped, 150K pins): k = 1000, nworst = 4."""
    d = synth.config_design("c2_tau")
    ctx = run(sta, d)
    check(sta, ctx, d, ks=((1000, 4), (100, 1)))
