"""Pins of the oracle's Steiner RC construction (O11; SURVEY.md §8(f) row 2,
PAPER.md:178-179) against hand constructions, brute-force
minimum spanning trees and invariants -- nothing here re-derives the
oracle's own loops."""
import itertools

import numpy as np
import pytest

import oracle
import synth

NO_PIN = 0xFFFFFFFF


def one_net(xy, units=(1.5, 2.0, 0.3, 0.4), order=None):
    """A single net over pins 0..m-1 (pin 0 the driver) at positions xy."""
    m = len(xy)
    pins = list(range(m)) if order is None else list(order)
    x = np.array([p[0] for p in xy], np.float32)
    y = np.array([p[1] for p in xy], np.float32)
    return oracle.steiner([0, m], pins, x, y, *units)


def test_two_pins_straight():
    # SPEC.md:331 example 1: dx = 10, dy = 0 -> one resistor 10 res_x, 5 cap_x at each end
    rc_ptr, parent, node_pin, res, cap = one_net([(0, 0), (10, 0)])
    assert rc_ptr.tolist() == [0, 2]
    assert parent.tolist() == [-1, 0] and node_pin.tolist() == [0, 1]
    assert res[1] == np.float32(15.0) and res[0] == 0
    assert cap.tolist() == [1.5, 1.5]


def test_two_pins_l_route():
    # SPEC.md:331 example 2: (0,0)-(10,10): one bend, R = 10 res_x + 10 res_y
    rc_ptr, parent, node_pin, res, cap = one_net([(0, 0), (10, 10)])
    assert rc_ptr.tolist() == [0, 3]
    assert parent.tolist() == [-1, 0, 1]
    assert node_pin.tolist() == [0, NO_PIN, 1]              # the bend is a Steiner node
    assert res[1] == np.float32(15.0) and res[2] == np.float32(20.0)
    # horizontal leg first from the driver: bend at (10, 0) gets 5 cap_x + 5 cap_y
    np.testing.assert_allclose(cap, [1.5, 1.5 + 2.0, 2.0], rtol=0, atol=1e-6)
    # unequal legs (10, 4): horizontal 10 res_x / 5 cap_x at each end, vertical 4 res_y / 2 cap_y
    rc_ptr, parent, node_pin, res, cap = one_net([(0, 0), (10, 4)])
    assert res[1] == np.float32(15.0) and res[2] == np.float32(8.0)
    np.testing.assert_allclose(cap, [1.5, 1.5 + 0.8, 0.8], rtol=0, atol=1e-6)
    # child to the lower left: lengths are absolute, the bend is at (x_child, y_parent)
    rc_ptr, parent, node_pin, res, cap = one_net([(10, 4), (0, 0)])
    assert res[1] == np.float32(15.0) and res[2] == np.float32(8.0)


def test_single_pin():
    # SPEC.md:331 example 3: one node, no resistor
    rc_ptr, parent, node_pin, res, cap = one_net([(3, 4)])
    assert rc_ptr.tolist() == [0, 1] and parent.tolist() == [-1] and node_pin.tolist() == [0]
    assert res.tolist() == [0.0] and cap.tolist() == [0.0]


def test_vertical_leg_and_zero_length_clamp():
    # dx = 0: one vertical leg; coincident pins: a zero resistance clamped to 1e-6 kOhm
    rc_ptr, parent, node_pin, res, cap = one_net([(0, 0), (0, 7), (0, 7)])
    assert parent.tolist() == [-1, 0, 1]
    assert res[1] == np.float32(14.0) and res[2] == np.float32(1e-6)
    np.testing.assert_allclose(cap, [0.5 * 7 * 0.4, 0.5 * 7 * 0.4, 0.0], atol=1e-6)


def test_prim_ties_smaller_pin_id():
    # pins 1 and 2 both at distance 1 from the driver: the smaller id joins
    # first; pin 3 is nearer to pin 2 (distance 1) than to the driver (2)
    xy = [(0, 0), (1, 0), (0, 1), (0, 2)]
    rc_ptr, parent, node_pin, res, cap = one_net(xy)
    assert node_pin.tolist() == [0, 1, 2, 3]
    assert parent.tolist() == [-1, 0, 0, 2]
    # equal distances through two tree pins: the parent is the one that first
    # gave the distance (strict improvement only): pin 3 at (1, 1) is 1 from
    # pin 1 and 1 from pin 2 -> parent pin 1 (joined first)
    xy = [(0, 0), (1, 0), (0, 1), (1, 1)]
    _, parent, node_pin, _, _ = one_net(xy)
    assert node_pin.tolist() == [0, 1, 2, 3] and parent.tolist() == [-1, 0, 0, 1]


def mst_weight_bruteforce(pts):
    """Minimum over ALL labelled spanning trees (Pruefer sequences) of the
    Manhattan length -- independent of Prim and of its tie rules."""
    n = len(pts)
    d = lambda a, b: abs(pts[a][0] - pts[b][0]) + abs(pts[a][1] - pts[b][1])
    if n == 1:
        return 0.0
    if n == 2:
        return d(0, 1)
    best = float("inf")
    for seq in itertools.product(range(n), repeat=n - 2):
        deg = [1] * n
        for s in seq:
            deg[s] += 1
        w, deg = 0.0, deg[:]
        for s in seq:
            leaf = min(i for i in range(n) if deg[i] == 1)
            w += d(leaf, s)
            deg[leaf] -= 1
            deg[s] -= 1
        u, v = [i for i in range(n) if deg[i] == 1]
        w += d(u, v)
        best = min(best, w)
    return best


@pytest.mark.parametrize("seed", range(12))
def test_wirelength_is_minimum_spanning(seed):
    # with unit resistance 1 along x and y, the resistances sum to the tree's
    # Manhattan length, which must equal the brute-force MST weight (an L
    # embedding keeps the Manhattan length); caps conserve L * unit cap
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 7))
    pts = [(float(a), float(b)) for a, b in rng.integers(0, 6, (n, 2))]
    if len(set(pts)) < n:                    # coincident pins would add 1e-6 clamps
        pts = [(p[0] + 7 * i, p[1]) for i, p in enumerate(pts)]
    rc_ptr, parent, node_pin, res, cap = one_net(pts, units=(1.0, 1.0, 2.0, 2.0))
    W = mst_weight_bruteforce(pts)
    assert abs(float(res.astype(np.float64).sum()) - W) < 1e-4
    assert abs(float(cap.astype(np.float64).sum()) - 2.0 * W) < 1e-4


@pytest.mark.parametrize("seed", range(6))
def test_tree_shape_and_order_invariance(seed):
    rng = np.random.default_rng(100 + seed)
    m = int(rng.integers(2, 40))
    pts = [tuple(p) for p in rng.integers(0, 12, (m, 2)).astype(float)]
    rc_ptr, parent, node_pin, res, cap = one_net(pts)
    n = int(rc_ptr[-1])
    # a tree rooted at the driver, parents before children, every pin once,
    # Steiner nodes exactly at the bends
    assert parent[0] == -1 and all(0 <= parent[i] < i for i in range(1, n))
    pins = [p for p in node_pin.tolist() if p != NO_PIN]
    assert sorted(pins) == list(range(m)) and node_pin[0] == 0
    assert n == m + sum(1 for p in node_pin.tolist() if p == NO_PIN)
    for i in range(1, n):                    # a Steiner node has exactly one child, a pin
        if node_pin[i] == NO_PIN:
            kids = [j for j in range(n) if parent[j] == i]
            assert len(kids) == 1 and node_pin[kids[0]] != NO_PIN
    # SPEC.md:340 determinism: any input order of the sinks gives the same tree
    order = [0] + list(rng.permutation(np.arange(1, m)))
    r2 = one_net(pts, order=order)
    for a, b in zip((rc_ptr, parent, node_pin, res, cap), r2):
        assert np.array_equal(a, b)


def test_many_nets_offsets():
    # several nets: offsets are the running node counts; every net's local tree is its own
    d = synth.generate(300, 8, seed=5, period=300.0)
    x, y = synth.placement(d, seed=2, grid=True)
    rc_ptr, parent, node_pin, res, cap = oracle.steiner(d.net_ptr, d.net_pins, x, y, **synth.STEINER_UNITS)
    N = d.num_nets
    assert rc_ptr.size == N + 1 and rc_ptr[-1] == parent.size
    for n in range(N):
        a, b = int(rc_ptr[n]), int(rc_ptr[n + 1])
        m = int(d.net_ptr[n + 1] - d.net_ptr[n])
        assert b - a >= m and b - a <= 2 * m - 1
        assert node_pin[a] == d.net_pins[d.net_ptr[n]]             # node 0: the driver
        assert parent[a] == -1 and all(0 <= parent[i] < i - a for i in range(a + 1, b))
        got = sorted(p for p in node_pin[a:b].tolist() if p != NO_PIN)
        assert got == sorted(d.net_pins[d.net_ptr[n]:d.net_ptr[n + 1]].tolist())


def test_elmore_on_steiner_tree_by_hand():
    # driver (0,0) -> sink (10,10), L-route; Elmore to the sink with pin cap
    # C_s: R_h * (C_bend + C_sink + C_s) + R_v * (C_sink + C_s)
    rc_ptr, parent, node_pin, res, cap = one_net([(0, 0), (10, 10)])
    Cs = 2.5
    want = 15.0 * (3.5 + 2.0 + Cs) + 20.0 * (2.0 + Cs)
    d = synth.design.Design
    # through the oracle's own O3 on a two-pin design with this RC tree
    lib = synth.Library.from_tables([synth.design.constant_table(1.0)] * 4)
    dsg = d(num_pins=2, pin_cap=np.array([0.0, Cs], np.float32), pin_role=np.array([1, 2], np.uint8),
            net_ptr=np.array([0, 2], np.uint32), net_pins=np.array([0, 1], np.uint32),
            arc_from=np.zeros(0, np.uint32), arc_to=np.zeros(0, np.uint32), arc_sense=np.zeros(0, np.uint8),
            arc_tab=np.zeros(0, np.uint32), chk_d=np.zeros(0, np.uint32), chk_ck=np.zeros(0, np.uint32),
            chk_tab=np.zeros(0, np.uint32), libs=[lib],
            rc=[synth.RcTree(rc_ptr, parent, node_pin, res, cap)],
            cons=synth.design.empty_constraints(), name="steiner2")
    load, elm = oracle.rc(dsg)
    assert abs(elm[1] - want) < 1e-9 * want
    assert abs(load[0] - (1.5 + 3.5 + 2.0 + Cs)) < 1e-9
