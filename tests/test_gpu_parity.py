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


@pytest.mark.parametrize("name", ["h1_chain", "c17", "h3_reg2reg", "h4_seeds"])
def test_hand_examples(sta, name):
    d = {"h1_chain": synth.h1_chain, "c17": synth.c17, "h3_reg2reg": synth.h3_reg2reg,
         "h4_seeds": synth.h4_seeds}[name]()
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


def _wide_multi_output_design(width=12, depth=3, seed=3):
    """Cells the synthetic recipe never makes: a `width`-input gate (one pin
    with more fan-in terms than a forward warp unit holds -> the warp-loop
    path) and two-output full adders (an input pin with three fan-out terms
    -> the backward's CSR path beyond the two inline terms), chained `depth`
    times, with PIs driving several sinks."""
    import copy
    from synth.design import (ROLE_PI, ROLE_PO, SENSE_NEG, SENSE_NON, SENSE_POS, affine_table)
    from synth.hand import AFFINE_LOAD, AFFINE_SLEW, Builder, _cons
    rng = np.random.default_rng(seed)
    b = Builder()

    def tabs():
        return b.tables4([affine_table(AFFINE_SLEW, AFFINE_LOAD, *rng.uniform([4, 0.05, 0.5], [15, 0.3, 3]))
                          for _ in range(4)])
    pis = [f"i{k}" for k in range(width)]
    for n in pis:
        b.pin(n, 0.0, ROLE_PI)
    sinks_of = {n: [] for n in pis}
    prev = list(pis)
    for lvl in range(depth):
        W = f"W{lvl}"
        for k in range(width):
            b.pin(f"{W}/a{k}", float(rng.uniform(0.5, 2)))
        b.pin(f"{W}/y")
        for k in range(width):
            b.arc(f"{W}/a{k}", f"{W}/y", [SENSE_NEG, SENSE_NON, SENSE_POS][k % 3], tabs())
            sinks_of.setdefault(prev[k % len(prev)], []).append(f"{W}/a{k}")
        F = f"F{lvl}"
        for p in ("a", "b", "c"):
            b.pin(f"{F}/{p}", float(rng.uniform(0.5, 2)))
        b.pin(f"{F}/s")
        b.pin(f"{F}/co")
        for p in ("a", "b", "c"):
            b.arc(f"{F}/{p}", f"{F}/s", SENSE_NON, tabs())
            b.arc(f"{F}/{p}", f"{F}/co", SENSE_POS, tabs())
        sinks_of.setdefault(f"{W}/y", []).append(f"{F}/a")
        sinks_of[pis[lvl % width]].append(f"{F}/b")
        sinks_of.setdefault(prev[(lvl + 1) % len(prev)], []).append(f"{F}/c")
        prev = [f"{W}/y", f"{F}/s", f"{F}/co"] + pis[3:]
    pos = []
    for k, n in enumerate(prev[:3]):
        po = f"o{k}"
        b.pin(po, 0.0, ROLE_PO)
        sinks_of.setdefault(n, []).append(po)
        pos.append((po, [float(rng.uniform(0, 20))] * 2, [0.0, 0.0], 1.5))
    for drv, sk in sinks_of.items():
        if sk:
            b.net(drv, sk, b.star_rc(drv, sk, float(rng.uniform(0.05, 0.3)), float(rng.uniform(0.1, 1.0))))
    cons = _cons(b, 400.0, 20.0, [(n, [0, 0, 0, 0], [10, 12, 10, 12]) for n in pis], pos)
    return b.build(cons, name="wide_multi_output")


@pytest.mark.parametrize("mode", ["0", "1"])
def test_wide_gates_and_multi_output_cells(sta, mode):
    """Forward warp-loop path (> 8 fan-in terms on one pin) and the backward's
    CSR fan-out path (> 2 fan-out terms on one pin), both launchers."""
    d = _wide_multi_output_design()
    os.environ["STA_STAGE_KERNELS"] = mode
    try:
        ctx = run(sta, d)
    finally:
        os.environ.pop("STA_STAGE_KERNELS", None)
    compare_update(ctx, oracle.update(d))
    check_levels(ctx, d)
    ctx.close()


def test_repeated_updates_with_changing_rc(sta):
    """An optimization loop (C4 pattern): RC values re-set between updates,
    every update compared with the oracle -- the tagged records of one update
    must never be taken for the next one's."""
    d = synth.generate(8000, 40, seed=12, n_hfn=2, hfn_range=(200, 3000), period=300.0)
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    import copy
    for i, (rs, cs) in enumerate([(1.0, 1.0), (1.3, 0.8), (0.7, 1.25), (1.0, 1.0)]):
        di = copy.copy(d)
        di.rc = [d.rc[0].scaled(rs, cs)]
        ctx.set_rc_values(0, di.rc[0].res, di.rc[0].cap)
        ctx.update_timing()
        ctx.synchronize()
        compare_update(ctx, oracle.update(di))
    ctx.close()


def test_pipelined_host_rc_values(sta):
    """Optimization-loop pipelining through the ABI: step i+1's HOST RC values
    are handed over (copied on the ctx's copy stream into the other owned
    buffer pair) while step i's update is still in flight; each step's
    results must be those of its own values, and a DEVICE (borrowed) call in
    between must hand the buffers back cleanly."""
    import copy
    import torch
    d = synth.generate(30000, 40, seed=13, n_hfn=2, hfn_range=(200, 3000), period=300.0)
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    scales = [(1.0, 1.0), (1.3, 0.8), (0.7, 1.25), (1.1, 0.9), (0.9, 1.1)]
    vals = [d.rc[0].scaled(rs, cs) for rs, cs in scales]
    exp = []
    for v in vals:
        di = copy.copy(d)
        di.rc = [v]
        exp.append(oracle.update(di))
    pinned = [(torch.from_numpy(v.res).pin_memory(), torch.from_numpy(v.cap).pin_memory()) for v in vals]
    ctx.set_rc_values(0, pinned[0][0].numpy(), pinned[0][1].numpy())
    for i in range(len(vals)):
        ctx.update_timing()
        if i + 1 < len(vals):
            if i == 2:                         # a borrowed device pair in the middle of the loop
                rd = torch.from_numpy(vals[i + 1].res).cuda()
                cd = torch.from_numpy(vals[i + 1].cap).cuda()
                ctx.set_rc_values(0, rd, cd)
            else:
                ctx.set_rc_values(0, pinned[i + 1][0].numpy(), pinned[i + 1][1].numpy())
        compare_update(ctx, exp[i])
    ctx.close()
