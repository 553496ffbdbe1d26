"""GPU parity of the built-in Steiner RC (SURVEY.md §8(f) row 2,
sta_build_steiner) against the oracle's O11, then a full timing update on
the Steiner RC against the oracle's update on the oracle's own Steiner RC.

Topology (rc_ptr, parent, node_pin) must be bit-exact: the MST decisions are
fp32 Manhattan distances on both sides.  Resistances are one fp32 product on
both sides (bit-exact); node caps are fp32 sums on the device and fp64 sums
rounded once in the oracle: within 1e-6 relative.

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import copy

import numpy as np
import pytest

import oracle
import synth
from tests.parity import compare_update

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sta():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 (there is no CPU fallback)")
    import paper_2511_11660_b200 as pkg
    return pkg


def compare_steiner(g, o):
    rc_ptr, parent, node_pin, res, cap = g
    orp, opa, onp, ore, oca = o
    assert np.array_equal(np.asarray(rc_ptr, np.uint32), orp)
    assert np.array_equal(np.asarray(parent, np.int32), opa)
    assert np.array_equal(np.asarray(node_pin, np.uint32), onp)
    assert np.array_equal(np.asarray(res, np.float32), ore)
    np.testing.assert_allclose(np.asarray(cap, np.float64), oca.astype(np.float64), rtol=1e-6, atol=1e-7)


def with_steiner_rc(d, rc):
    d2 = copy.copy(d)
    d2.rc = [synth.RcTree(*rc)] * d.num_corners
    return d2


def build(sta, d, x, y, units=synth.STEINER_UNITS, device=False):
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    if device:
        import torch
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        out = ctx.build_steiner(xd, yd, **units)
        out = tuple(t.cpu().numpy() for t in out)
    else:
        out = ctx.build_steiner(x, y, **units)
    return ctx, out


@pytest.mark.parametrize("grid", [True, False])
def test_steiner_parity_small(sta, grid):
    d = synth.generate(2000, 20, seed=11, period=400.0)
    x, y = synth.placement(d, seed=3, grid=grid)
    ctx, g = build(sta, d, x, y)
    o = oracle.steiner(d.net_ptr, d.net_pins, x, y, **synth.STEINER_UNITS)
    compare_steiner(g, o)
    ctx.close()


def test_steiner_parity_all_net_classes(sta):
    # high-fan-out nets of ~40 .. 20000 pins: warp nets (<= 32), shared-memory
    # block nets (33 .. 12288) and global-scratch block nets (> 12288); an
    # integer grid makes Prim ties common
    d = synth.generate(30000, 16, seed=21, n_hfn=6, hfn_range=(40, 20000), period=600.0)
    m = np.diff(d.net_ptr)
    assert m.max() > 12288 and ((m > 32) & (m <= 12288)).any() and ((m >= 2) & (m <= 32)).any()
    x, y = synth.placement(d, seed=4, grid=True)
    ctx, g = build(sta, d, x, y)
    o = oracle.steiner(d.net_ptr, d.net_pins, x, y, **synth.STEINER_UNITS)
    compare_steiner(g, o)
    ctx.close()


def test_steiner_device_positions_and_degenerate(sta):
    # device positions give the same arrays as host positions; coincident pins
    # (every pin of a net at one point: zero-length legs clamped) and zero units
    d = synth.generate(1500, 12, seed=31, period=400.0)
    x, y = synth.placement(d, seed=5, grid=True)
    x[d.net_pins[d.net_ptr[3]:d.net_ptr[4]]] = 7.0
    y[d.net_pins[d.net_ptr[3]:d.net_ptr[4]]] = 9.0
    ctx, gh = build(sta, d, x, y)
    ctx2, gd = build(sta, d, x, y, device=True)
    for a, b in zip(gh, gd):
        assert np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))
    units = dict(res_x=0.0, res_y=0.002, cap_x=0.0, cap_y=0.1)
    g0 = ctx.build_steiner(x, y, **units)
    compare_steiner(g0, oracle.steiner(d.net_ptr, d.net_pins, x, y, **units))
    ctx.close()
    ctx2.close()


def test_steiner_errors(sta):
    d = synth.generate(200, 6, seed=41, period=300.0)
    ctx = sta.Context(0, 1)
    x, y = synth.placement(d, seed=1)
    with pytest.raises(sta.StaError) as e:
        ctx.build_steiner(x, y, **synth.STEINER_UNITS)       # no graph yet
    assert e.value.name == "STA_ERR_ORDER"
    sta.load_design(ctx, d)
    with pytest.raises(sta.StaError) as e:
        ctx.build_steiner(x, y, res_x=-1.0, res_y=0.1, cap_x=0.1, cap_y=0.1)
    assert e.value.name == "STA_ERR_ARG"
    xb = x.copy()
    xb[5] = np.nan
    with pytest.raises(sta.StaError) as e:
        ctx.build_steiner(xb, y, **synth.STEINER_UNITS)
    assert e.value.name == "STA_ERR_ARG"
    with pytest.raises(sta.StaError) as e:
        ctx.build_steiner(x, y, net_pins_total=10, **synth.STEINER_UNITS)   # capacity too small
    assert e.value.name == "STA_ERR_ARG"
    ctx.close()


@pytest.mark.parametrize("seed", [51, 52])
def test_timing_on_steiner_rc(sta, seed):
    # positions -> Steiner RC on the device -> set as the RC of the update ->
    # full-array parity with the oracle's update on the oracle's Steiner RC
    d = synth.generate(3000, 24, seed=seed, n_hfn=2, hfn_range=(50, 400), period=500.0)
    x, y = synth.placement(d, seed=seed, grid=(seed % 2 == 0))
    ctx, g = build(sta, d, x, y)
    o = oracle.steiner(d.net_ptr, d.net_pins, x, y, **synth.STEINER_UNITS)
    compare_steiner(g, o)
    rc_ptr, parent, node_pin, res, cap = g
    ctx.set_rc_tree(rc_ptr, parent, node_pin)
    ctx.set_rc_values(0, res, cap)
    ctx.update_timing()
    compare_update(ctx, oracle.update(with_steiner_rc(d, o)), period=d.cons.period)
    ctx.close()


def test_device_steiner_feeds_device_rc(sta):
    # the optimisation-loop path: device positions -> device RC arrays -> tree
    # + borrowed values, no host copies of the RC
    import torch
    d = synth.generate(2000, 20, seed=61, period=400.0)
    x, y = synth.placement(d, seed=6)
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    out = ctx.build_steiner(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), **synth.STEINER_UNITS)
    rc_ptr, parent, node_pin, res, cap = out
    ctx.set_rc_tree(rc_ptr, parent, node_pin)
    ctx.set_rc_values(0, res, cap)
    ctx.update_timing()
    o = oracle.steiner(d.net_ptr, d.net_pins, x, y, **synth.STEINER_UNITS)
    compare_update(ctx, oracle.update(with_steiner_rc(d, o)), period=d.cons.period)
    ctx.close()
