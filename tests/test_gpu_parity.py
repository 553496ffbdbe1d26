"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests.parity import check_close, compare_update

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sta():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 (there is no CPU fallback)")
    import paper_2511_11660_b200 as pkg
    return pkg


def run(sta, d, corners=None, device_rc=False):
    K = d.num_corners if corners is None else len(corners)
    ctx = sta.Context(0, K)
    sta.load_design(ctx, d, corners=corners, device_rc=device_rc)
    ctx.update_timing()
    ctx.synchronize()
    return ctx


def check_levels(ctx, d):
    level, perm, nl = ctx.get_levels()
    rl, rp, rn = oracle.levelize(d)
    assert nl == rn
    assert np.array_equal(level, rl)
    assert np.array_equal(perm, rp)


def check_rc(ctx, d, corner=0, design_corner=0):
    load, elm = ctx.get_rc(corner)
    rl, re = oracle.rc(d, design_corner)
    check_close("load", load, rl)
    check_close("elm", elm, re)


@pytest.mark.parametrize("name", ["h1_chain", "c17", "h3_reg2reg"])
def test_hand_examples(sta, name):
    d = {"h1_chain": synth.h1_chain, "c17": synth.c17, "h3_reg2reg": synth.h3_reg2reg}[name]()
    ctx = run(sta, d)
    ref = oracle.update(d)
    compare_update(ctx, ref)
    check_levels(ctx, d)
    check_rc(ctx, d)
    # the golden values themselves (paper-derived hand examples)
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    pid = {n: i for i, n in enumerate(d.meta["pin_names"])}
    at, slew, rat = ctx.get_timing()
    res, _ = ctx.report_slack()
    for pin, exp in g["pins"].items():
        if "at" in exp:
            assert np.allclose(at[pid[pin]], exp["at"], atol=1e-3)
    assert res[0] == pytest.approx(g["res"]["wns_setup"], abs=1e-3)
    assert res[2] == pytest.approx(g["res"]["wns_hold"], abs=1e-3)
    ctx.close()


def _tiny_libsyn(seed):
    rng = np.random.default_rng(seed)
    d = synth.generate(int(rng.integers(8, 40)), int(rng.integers(4, 14)), seed=seed,
                       frac_pi=0.1, frac_po=0.1, period=120.0)
    flip = rng.random(d.num_arcs) < 0.3
    d.arc_sense = d.arc_sense.copy()
    d.arc_sense[flip] = rng.integers(0, 5, int(flip.sum())).astype(np.uint8)
    if seed % 3 == 0 and d.cons.pi_pin.size > 1:
        import copy
        d.cons = copy.copy(d.cons)
        d.cons.pi_pin, d.cons.pi_at, d.cons.pi_slew = d.cons.pi_pin[1:], d.cons.pi_at[1:], d.cons.pi_slew[1:]
    return d


@pytest.mark.parametrize("seed", range(30))
def test_random_small_designs(sta, seed):
    d = _tiny_libsyn(seed)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    check_levels(ctx, d)
    check_rc(ctx, d)


def test_c2_tau_full_arrays(sta):
    """BASELINE configs[1]: TAU-shaped ~150K pins, every pin compared."""
    d = synth.config_design("c2_tau")
    ctx = run(sta, d)
    rep = {}
    compare_update(ctx, oracle.update(d), report=rep)
    check_levels(ctx, d)
    check_rc(ctx, d)
    print(json.dumps(rep))


def test_high_fanout_nets(sta):
    """Big RC trees (block-per-net Elmore) and heavy backward drivers."""
    d = synth.generate(20000, 40, seed=77, n_hfn=6, hfn_range=(300, 5000), period=400.0)
    ctx = run(sta, d)
    info = ctx.info()
    assert info["num_heavy_drivers"] > 0
    compare_update(ctx, oracle.update(d))
    check_rc(ctx, d)


def test_multicorner_and_device_rc(sta):
    """Several corners in one ctx (own LUT pool / RC values each); RC values
    borrowed from device tensors give identical bits to host-copied ones."""
    d = synth.generate(6000, 30, seed=5, corners=4, corner_recipe="c5", period=300.0)
    ctx = run(sta, d)
    ctx_dev = run(sta, d, device_rc=True)
    for c in range(4):
        ref = oracle.update(d, c)
        compare_update(ctx, ref, corner=c)
        check_rc(ctx, d, c, c)
        a = ctx.get_timing(c)
        b = ctx_dev.get_timing(c)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        assert np.array_equal(ctx.report_slack(c)[0], ctx_dev.report_slack(c)[0])


def test_sharded_corner_equals_batched(sta):
    """A corner run alone (as one rank of a multi-GPU shard) is bitwise equal
    to the same corner inside a batched multi-corner ctx."""
    d = synth.generate(4000, 24, seed=9, corners=3, corner_recipe="c5", period=250.0)
    full = run(sta, d)
    for c in range(3):
        one = run(sta, d, corners=[c])
        for x, y in zip(full.get_timing(c), one.get_timing(0)):
            assert np.array_equal(x, y)
        assert np.array_equal(full.report_slack(c)[0], one.report_slack(0)[0])


def test_repeat_update_deterministic(sta):
    d = synth.generate(5000, 30, seed=3, period=300.0)
    ctx = run(sta, d)
    a = ctx.get_timing(0), ctx.report_slack(0, want_pins=True)
    ctx.update_timing()
    b = ctx.get_timing(0), ctx.report_slack(0, want_pins=True)
    for x, y in zip(a[0], b[0]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[1][0], b[1][0]) and np.array_equal(a[1][1], b[1][1])


def test_rc_perturbation_loop(sta):
    """BASELINE configs[3] pattern: repeated updates with perturbed RC values
    passed as borrowed device pointers; each iteration matches the oracle."""
    import torch
    d = synth.generate(3000, 24, seed=21, period=250.0)
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    rc = d.rc[0]
    g = torch.Generator().manual_seed(0)
    for it in range(3):
        f_r = (1 + 0.1 * (2 * torch.rand(rc.res.size, generator=g) - 1)).numpy().astype(np.float32)
        f_c = (1 + 0.1 * (2 * torch.rand(rc.cap.size, generator=g) - 1)).numpy().astype(np.float32)
        r = (rc.res * f_r).astype(np.float32)
        c = (rc.cap * f_c).astype(np.float32)
        tr, tc = torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda()
        ctx.set_rc_values(0, tr, tc)
        ctx.update_timing()
        d2 = synth.Design(**{**d.__dict__, "rc": [synth.RcTree(rc.rc_ptr, rc.parent, rc.node_pin, r, c)]})
        compare_update(ctx, oracle.update(d2))


def test_c3_superblue_full(sta):
    """BASELINE configs[2] at full size (~10M pins, 150 levels, high-fan-out
    nets) in the configuration bench.py times; every pin compared."""
    d = synth.config_design("c3_superblue")
    ctx = run(sta, d)
    rep = {}
    compare_update(ctx, oracle.update(d), report=rep)
    check_levels(ctx, d)
    print(json.dumps(rep))


def test_stage_kernels_equal_persistent_kernels(sta):
    """The two launch strategies of the forward / backward passes (one launch
    per gate stage with PDL vs. persistent dataflow kernels) give identical bits."""
    d = synth.generate(30000, 60, seed=31, n_hfn=3, hfn_range=(100, 2000), period=500.0)
    out = []
    for mode in ("1", "0"):
        os.environ["STA_STAGE_KERNELS"] = mode
        try:
            ctx = run(sta, d)
        finally:
            os.environ.pop("STA_STAGE_KERNELS", None)
        out.append((ctx.get_timing(0), ctx.report_slack(0, want_pins=True)))
        ctx.close()
    (a, ra), (b, rb) = out
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
