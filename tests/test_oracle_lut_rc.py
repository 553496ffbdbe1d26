"""Pins of the oracle's NLDM lookup (O6) and Elmore RC (O3) steps.

Each test checks the oracle against something other than itself: SPEC worked
examples, closed forms, or the brute-force shared-path double loop.
"""
import math

import numpy as np
import pytest

import oracle
from synth.design import (Constraints, NO_PIN, ROLE_PI, ROLE_PO, SENSE_POS,
                          constant_table, empty_constraints)
from synth.hand import Builder
from tests.brute import design_node_caps, elmore_bruteforce


def _tab(idx1, idx2, vals):
    return np.concatenate([np.asarray(idx1, np.float32), np.asarray(idx2, np.float32),
                           np.asarray(vals, np.float32).reshape(-1)])


# ------------------------------------------------------------------ LUT (O6)
def test_lut_grid_identity():
    """a query exactly at a grid point returns that value."""
    rng = np.random.default_rng(1)
    x = np.cumsum(rng.uniform(1, 10, 7))
    y = np.cumsum(rng.uniform(0.1, 3, 7))
    v = rng.uniform(-5, 50, (7, 7)).astype(np.float32)
    t = _tab(x, y, v)
    for i in range(7):
        for j in range(7):
            assert oracle.lut(7, 7, t, float(np.float32(x[i])), float(np.float32(y[j]))) == \
                pytest.approx(float(v[i, j]), abs=1e-9)


def test_lut_2x2_midpoint():
    """{{0,2},{4,6}} at the cell midpoint -> 3.0."""
    t = _tab([0, 1], [0, 1], [[0, 2], [4, 6]])
    assert oracle.lut(2, 2, t, 0.5, 0.5) == 3.0


@pytest.mark.parametrize("seed", range(5))
def test_lut_bilinear_closed_form_including_extrapolation(seed):
    """SPEC.md:379 + SURVEY §8(c): a table sampled from a bilinear f(s,c) =
    a + b s + k c + m s c reproduces f everywhere (the bilinear interpolant of
    a bilinear function is itself), also outside the grid (linear
    extrapolation from the boundary cell).  Dyadic coefficients keep the f32
    table exact."""
    rng = np.random.default_rng(seed)
    a, b, k, m = [float(x) for x in rng.integers(-64, 64, 4) / 8.0]
    x = np.array([1, 2, 4, 8, 16, 32, 64], np.float64)
    y = np.array([0.5, 1, 2, 4, 8, 16, 32], np.float64)
    f = lambda s, c: a + b * s + k * c + m * s * c
    v = f(x[:, None], y[None, :])
    t = _tab(x, y, v)
    for s, c in rng.uniform([-20, -10], [120, 60], (200, 2)):
        assert oracle.lut(7, 7, t, s, c) == pytest.approx(f(s, c), rel=1e-12, abs=1e-9)


def test_lut_one_dimensional_and_scalar():
    """1-D tables interpolate on their single axis; 1x1 is a constant."""
    assert oracle.lut(1, 1, _tab([0], [0], [[7.5]]), 123.0, -4.0) == 7.5
    t = _tab([3.0], [1, 2, 4], [[10, 20, 30]])          # n1 = 1: along load only
    assert oracle.lut(1, 3, t, 999.0, 1.5) == pytest.approx(15.0)
    assert oracle.lut(1, 3, t, 999.0, 5.0) == pytest.approx(35.0)   # extrapolated
    t = _tab([1, 3], [0.0], [[2], [6]])                  # n2 = 1: along slew only
    assert oracle.lut(2, 1, t, 2.0, 77.0) == pytest.approx(4.0)
    assert oracle.lut(2, 1, t, 0.0, 77.0) == pytest.approx(0.0)


def test_lut_continuous_across_cells():
    """continuous across cell boundaries (sampled +-eps)."""
    rng = np.random.default_rng(7)
    x = np.array([1, 5, 15, 40, 90, 180, 360.0])
    y = np.array([0.1, 0.5, 1.5, 4, 9, 18, 36.0])
    v = rng.uniform(0, 100, (7, 7))
    t = _tab(x, y, v)
    eps = 1e-7
    for xi in x[1:-1]:
        for c in (0.3, 2.0, 20.0):
            lo = oracle.lut(7, 7, t, float(np.float32(xi)) - eps, c)
            hi = oracle.lut(7, 7, t, float(np.float32(xi)) + eps, c)
            assert abs(lo - hi) < 1e-4


# ----------------------------------------------------------------- RC (O3)
def _net_design(rc_nodes, sink_caps):
    """One driver pin, len(sink_caps) sink pins, one RC net.
    rc_nodes: list of (parent, R, Cw, pin_index or None) with pin index into
    ['drv', 's0', 's1', ...]."""
    b = Builder()
    b.pin("drv", 0.0, ROLE_PI)
    names = []
    for i, c in enumerate(sink_caps):
        names.append(b.pin(f"s{i}", c) and f"s{i}")
    all_names = ["drv"] + [f"s{i}" for i in range(len(sink_caps))]
    rc = [(p, r, cw, None if pi is None else all_names[pi]) for (p, r, cw, pi) in rc_nodes]
    b.net("drv", [f"s{i}" for i in range(len(sink_caps))], rc)
    b.table(constant_table(1.0))
    return b.build(empty_constraints())


def test_elmore_unit_rc():
    """root -- 1 kOhm -- node(1 fF) -> 1.0 ps."""
    d = _net_design([(-1, 0, 0, 0), (0, 1.0, 1.0, 1)], [0.0])
    load, elm = oracle.rc(d)
    assert elm[1] == pytest.approx(1.0, abs=1e-12)
    assert load[0] == pytest.approx(1.0)


def test_elmore_chain_and_star():
    """chain root-1k-n1(1fF)-1k-n2(1fF): delay(n2) = 1*2 + 1*1 = 3.0.
    SPEC.md:397: star, two 1 fF sinks behind one shared 1 kOhm -> 2.0."""
    d = _net_design([(-1, 0, 0, 0), (0, 1.0, 1.0, 1), (1, 1.0, 1.0, 2)], [0.0, 0.0])
    _, elm = oracle.rc(d)
    assert elm[2] == pytest.approx(3.0, abs=1e-12)
    assert elm[1] == pytest.approx(2.0, abs=1e-12)
    d = _net_design([(-1, 0, 0, 0), (0, 1.0, 0.0, None), (1, 0.0, 1.0, 1), (1, 0.0, 1.0, 2)],
                    [0.0, 0.0])
    _, elm = oracle.rc(d)
    assert elm[1] == pytest.approx(2.0, abs=1e-12)
    assert elm[2] == pytest.approx(2.0, abs=1e-12)


@pytest.mark.parametrize("n", [1, 2, 5, 17])
def test_elmore_uniform_chain_closed_form(n):
    """Uniform n-segment chain (R, C per segment): elm_n = R C n(n+1)/2."""
    R, Cn = 0.25, 0.5
    nodes = [(-1, 0, 0, 0)] + [(i, R, Cn, None) for i in range(n)]
    nodes[-1] = (n - 1, R, Cn, 1)
    d = _net_design(nodes, [0.0])
    _, elm = oracle.rc(d)
    assert elm[1] == pytest.approx(R * Cn * n * (n + 1) / 2, rel=1e-12)


def test_elmore_random_trees_vs_bruteforce():
    """1,000 random trees (n <= 20) vs the shared-path double
    loop, 1e-9 relative; also load = sum of node caps (conservation)."""
    rng = np.random.default_rng(2015)
    for trial in range(1000):
        n = int(rng.integers(2, 21))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
        R = [0.0] + list(rng.uniform(0.0, 2.0, n - 1).astype(np.float32).astype(float))
        Cw = list(rng.uniform(0.0, 3.0, n).astype(np.float32).astype(float))
        # every non-root node carries a sink pin with its own cap
        sink_caps = list(rng.uniform(0, 2, n - 1).astype(np.float32).astype(float))
        nodes = [(parent[0], 0.0, Cw[0], 0)] + [(parent[i], R[i], Cw[i], i) for i in range(1, n)]
        d = _net_design(nodes, sink_caps)
        load, elm = oracle.rc(d)
        caps = design_node_caps(d)
        ref = elmore_bruteforce(parent, R, list(caps))
        for i in range(1, n):
            assert elm[i] == pytest.approx(ref[i], rel=1e-9, abs=1e-12)
        assert load[0] == pytest.approx(sum(caps), rel=1e-12)


def test_elmore_monotone_in_caps():
    """increasing any grounded cap never decreases any sink delay."""
    rng = np.random.default_rng(3)
    for trial in range(100):
        n = int(rng.integers(2, 15))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
        R = [0.0] + list(rng.uniform(0.01, 1.0, n - 1))
        Cw = list(rng.uniform(0.0, 1.0, n))
        nodes = [(parent[i], R[i], Cw[i], i) for i in range(n)]
        d0 = _net_design(nodes, [0.0] * (n - 1))
        _, e0 = oracle.rc(d0)
        k = int(rng.integers(0, n))
        Cw2 = list(Cw)
        Cw2[k] += 0.5
        d1 = _net_design([(parent[i], R[i], Cw2[i], i) for i in range(n)], [0.0] * (n - 1))
        _, e1 = oracle.rc(d1)
        assert np.all(e1 >= e0 - 1e-12)


def test_lumped_net_without_rc():
    """a net with no RC nodes is lumped: load = pin caps (+ PO
    load), zero net-arc delay."""
    b = Builder()
    b.pin("a", 0.0, ROLE_PI)
    b.pin("s", 1.25)
    b.pin("o", 0.5, ROLE_PO)
    b.net("a", ["s", "o"], None)
    b.table(constant_table(1.0))
    cons = empty_constraints()
    cons.po_pin = np.array([2], np.uint32)
    cons.po_out_max = np.zeros((1, 2), np.float32)
    cons.po_out_min = np.zeros((1, 2), np.float32)
    cons.po_load = np.array([2.0], np.float32)
    d = b.build(cons)
    load, elm = oracle.rc(d)
    assert load[0] == pytest.approx(1.25 + 0.5 + 2.0)
    assert np.all(elm == 0)
