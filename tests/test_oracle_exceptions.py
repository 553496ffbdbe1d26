"""Pins of the oracle's -from / -to timing exceptions (O13; SURVEY.md §8(f)
row 4, reduced to -from / -to false paths, multicycles and max / min delays
on one clock): exhaustive path
enumeration on tiny frozen-delay designs (every path's required time from
its own (startpoint, endpoint) exception), hand examples, and the identity
without exceptions."""
import copy

import numpy as np
import pytest

import oracle
import synth
from synth.design import Exceptions
from tests.brute import path_enumeration_timing, path_slacks_with_exceptions
from tests.test_oracle_propagation import _bf_elm, _tiny


def _startpoints(d):
    sp = [int(p) for p in d.cons.pi_pin]
    sp += [p for p in range(d.num_pins) if int(d.pin_role[p]) == synth.ROLE_FF_CK]
    return sorted(set(sp))


def _endpoints(d):
    return sorted(set(int(p) for p in d.cons.po_pin) | set(int(p) for p in d.chk_d))


def random_exceptions(d, rng, n):
    sp, ep = _startpoints(d), _endpoints(d)
    items = []
    for _ in range(n):
        kind = int(rng.integers(0, 4))
        value = float(rng.integers(2, 4)) if kind == 1 else float(np.round(rng.uniform(-20, 120), 2))
        fr = list(rng.choice(sp, size=int(rng.integers(0, min(3, len(sp)) + 1)), replace=False)) if sp else []
        to = list(rng.choice(ep, size=int(rng.integers(0, min(3, len(ep)) + 1)), replace=False)) if ep else []
        items.append((kind, value, fr, to))
    return Exceptions.build(items)


@pytest.mark.parametrize("seed", range(16))
def test_exceptions_vs_path_enumeration(seed):
    d = _tiny(seed)
    rng = np.random.default_rng(1000 + seed)
    d.exceptions = random_exceptions(d, rng, int(rng.integers(1, 5)))
    elm = _bf_elm(d)
    slack, res = path_slacks_with_exceptions(d, elm)
    o = oracle.update(d)
    # arrivals are the untagged ones (tags partition the startpoints)
    at_bf, _, _, _ = path_enumeration_timing(d, elm)
    fin = np.isfinite(at_bf)
    assert np.array_equal(fin, np.isfinite(o["at"]))
    np.testing.assert_allclose(o["at"][fin], at_bf[fin], rtol=0, atol=1e-9)
    fs = np.isfinite(slack)
    assert np.array_equal(fs, np.isfinite(o["slack"])), (np.argwhere(fs != np.isfinite(o["slack"]))[:5])
    np.testing.assert_allclose(o["slack"][fs], slack[fs], rtol=0, atol=1e-9)
    for a, b in zip(o["res"], res):
        assert (a == b) or abs(a - b) <= 1e-9 * max(1.0, abs(b))


@pytest.mark.parametrize("seed", range(4))
def test_no_exception_is_identity(seed):
    d = _tiny(seed)
    base = oracle.update(d)
    d2 = copy.copy(d)
    d2.exceptions = Exceptions.build([])
    o = oracle.update(d2)
    for k in ("at", "slew", "rat", "slack"):
        assert np.array_equal(np.nan_to_num(o[k], posinf=1e300, neginf=-1e300),
                              np.nan_to_num(base[k], posinf=1e300, neginf=-1e300))


def test_hand_examples():
    # H3 (register to register): a false path to the D endpoint removes its
    # setup / hold slack from WNS / TNS; a multicycle 2 adds exactly T to its
    # setup slack and T to its hold requirement; max delay replaces RAT_L
    d = synth.h3_reg2reg()
    base = oracle.update(d)
    T = float(d.cons.period)
    ep = _endpoints(d)
    d1 = copy.copy(d)
    d1.exceptions = Exceptions.build([(0, 0.0, [], ep)])
    o1 = oracle.update(d1)
    assert o1["res"][0] == np.inf and o1["res"][1] == 0.0 and o1["res"][2] == np.inf
    d2 = copy.copy(d)
    d2.exceptions = Exceptions.build([(1, 2.0, [], ep)])
    o2 = oracle.update(d2)
    for p in ep:
        np.testing.assert_allclose(o2["slack"][p][2:], base["slack"][p][2:] + T, atol=1e-9)
        np.testing.assert_allclose(o2["slack"][p][:2], base["slack"][p][:2] - T, atol=1e-9)
    d3 = copy.copy(d)
    d3.exceptions = Exceptions.build([(2, 123.0, [], ep)])
    o3 = oracle.update(d3)
    for p in ep:
        for rf in (0, 1):
            if np.isfinite(o3["at"][p][2 + rf]):
                np.testing.assert_allclose(o3["slack"][p][2 + rf], 123.0 - o3["at"][p][2 + rf], atol=1e-9)
    # precedence: a false path beats a multicycle on the same endpoint
    d4 = copy.copy(d)
    d4.exceptions = Exceptions.build([(1, 3.0, [], ep), (0, 0.0, [], ep)])
    assert oracle.update(d4)["res"][0] == np.inf


def random_clocks(d, rng, n):
    from synth.design import Clocks
    base = float(d.cons.period)
    per = np.array([base * f for f in rng.choice([0.5, 1.0, 1.5, 2.0, 3.0], size=n, replace=False)], np.float32)
    pin_clk = rng.integers(0, n, d.num_pins).astype(np.uint32)
    return Clocks(per, pin_clk)


@pytest.mark.parametrize("seed", range(12))
def test_clocks_vs_path_enumeration(seed):
    # several ideal clocks (O14): each path's setup / hold relationship from
    # its launch clock and its endpoint's capture clock; with exceptions on
    # top for half the seeds
    d = _tiny(seed)
    rng = np.random.default_rng(2000 + seed)
    d.clocks = random_clocks(d, rng, int(rng.integers(2, 4)))
    if seed % 2:
        d.exceptions = random_exceptions(d, rng, int(rng.integers(1, 4)))
    elm = _bf_elm(d)
    slack, res = path_slacks_with_exceptions(d, elm)
    o = oracle.update(d)
    fs = np.isfinite(slack)
    assert np.array_equal(fs, np.isfinite(o["slack"])), np.argwhere(fs != np.isfinite(o["slack"]))[:5]
    np.testing.assert_allclose(o["slack"][fs], slack[fs], rtol=0, atol=1e-9)
    for a, b in zip(o["res"], res):
        assert (a == b) or abs(a - b) <= 1e-9 * max(1.0, abs(b))


def test_clock_relationships_by_hand():
    # one clock: setup T, hold 0 -- the plain update exactly
    from synth.design import Clocks
    d = synth.h3_reg2reg()
    base = oracle.update(d)
    d1 = copy.copy(d)
    d1.clocks = Clocks(np.array([d.cons.period], np.float32), np.zeros(d.num_pins, np.uint32))
    o1 = oracle.update(d1)
    fs = np.isfinite(base["slack"])
    np.testing.assert_allclose(o1["slack"][fs], base["slack"][fs], atol=1e-12)
    # launch 10 ps, capture 4 ps: launch edges 0, 10, 20 -> next capture 4, 12, 24:
    # setup = min(4, 2, 4) = 2, hold = max(0, -2, 0) = 0
    from tests.brute import path_slacks_with_exceptions  # noqa: F401  (the relation is pinned through it)
    import math
    s, h = math.inf, -math.inf
    for i in range(1000):
        a = i * 10.0
        nxt = (math.floor(a / 4.0) + 1) * 4.0
        s, h = min(s, nxt - a), max(h, nxt - 4.0 - a)
    assert (s, h) == (2.0, 0.0)


# ---- -through segments (O15)

def random_exceptions_through(d, rng, n):
    """random_exceptions plus 1-2 ordered -through segments of 1-3 pins each
    (any pin: internal, startpoint or endpoint) on most exceptions"""
    sp, ep = _startpoints(d), _endpoints(d)
    items = []
    for _ in range(n):
        kind = int(rng.integers(0, 4))
        value = float(rng.integers(2, 4)) if kind == 1 else float(np.round(rng.uniform(-20, 120), 2))
        fr = list(rng.choice(sp, size=int(rng.integers(0, min(2, len(sp)) + 1)), replace=False)) if sp else []
        to = list(rng.choice(ep, size=int(rng.integers(0, min(2, len(ep)) + 1)), replace=False)) if ep else []
        th = [list(rng.choice(d.num_pins, size=int(rng.integers(1, 4)), replace=False))
              for _ in range(int(rng.integers(0, 3)))]
        items.append((kind, value, fr, to, th))
    return Exceptions.build(items)


def _check_vs_brute(d):
    elm = _bf_elm(d)
    slack, res = path_slacks_with_exceptions(d, elm)
    o = oracle.update(d)
    if getattr(d, "clocks", None) is None:   # (the untagged brute force has one clock)
        at_bf, _, _, _ = path_enumeration_timing(d, elm)
        fin = np.isfinite(at_bf)
        # every path's arrival sits in exactly one tag at each pin: the
        # merged arrivals are the untagged ones
        assert np.array_equal(fin, np.isfinite(o["at"]))
        np.testing.assert_allclose(o["at"][fin], at_bf[fin], rtol=0, atol=1e-9)
    fs = np.isfinite(slack)
    assert np.array_equal(fs, np.isfinite(o["slack"])), np.argwhere(fs != np.isfinite(o["slack"]))[:5]
    np.testing.assert_allclose(o["slack"][fs], slack[fs], rtol=0, atol=1e-9)
    for a, b in zip(o["res"], res):
        assert (a == b) or abs(a - b) <= 1e-9 * max(1.0, abs(b))
    return o


@pytest.mark.parametrize("seed", range(24))
def test_through_vs_path_enumeration(seed):
    # each path's exception from its own pin sequence (the automaton's
    # definition, searched exhaustively) against the oracle's tag passes
    d = _tiny(seed)
    rng = np.random.default_rng(3000 + seed)
    d.exceptions = random_exceptions_through(d, rng, int(rng.integers(1, 4)))
    if seed % 3 == 2:
        d.clocks = random_clocks(d, rng, 2)
    _check_vs_brute(d)


def _reach(d, x):
    """pins reachable from x (x included) over net + cell arcs"""
    succ = {}
    for n in range(d.num_nets):
        b, e = int(d.net_ptr[n]), int(d.net_ptr[n + 1])
        succ.setdefault(int(d.net_pins[b]), []).extend(int(p) for p in d.net_pins[b + 1:e])
    for a in range(d.num_arcs):
        succ.setdefault(int(d.arc_from[a]), []).append(int(d.arc_to[a]))
    seen, st = {x}, [x]
    while st:
        for w in succ.get(st.pop(), []):
            if w not in seen:
                seen.add(w)
                st.append(w)
    return seen


def _same(a, b):
    for k in ("slack",):
        assert np.array_equal(np.nan_to_num(a[k], posinf=1e300, neginf=-1e300),
                              np.nan_to_num(b[k], posinf=1e300, neginf=-1e300))
    assert all((x == y) for x, y in zip(a["res"], b["res"]))


@pytest.mark.parametrize("seed", range(6))
def test_through_order_sensitivity(seed):
    # false_path -through x -through y removes the paths that
    # touch x and then y; in the reversed order it matches no path at all
    # when y only lies downstream of x (a DAG has no path y -> x): identity
    d = _tiny(seed)
    rng = np.random.default_rng(4000 + seed)
    base = oracle.update(d)
    pairs = [(x, y) for x in range(d.num_pins) for y in _reach(d, x) if y != x]
    x, y = pairs[int(rng.integers(0, len(pairs)))]
    d1 = copy.copy(d)
    d1.exceptions = Exceptions.build([(0, 0.0, [], [], [[x], [y]])])
    _check_vs_brute(d1)
    d2 = copy.copy(d)
    d2.exceptions = Exceptions.build([(0, 0.0, [], [], [[y], [x]])])
    _same(oracle.update(d2), base)


@pytest.mark.parametrize("seed", range(6))
def test_through_equivalences(seed):
    # -through a startpoint is -from it; -through a fan-out-free endpoint is
    # -to it; -through a pin no path reaches an endpoint from changes nothing
    d = _tiny(seed)
    rng = np.random.default_rng(5000 + seed)
    sp = [p for p in _startpoints(d) if any(True for _ in [0])]
    s = int(rng.choice(sp))
    kind = int(rng.integers(0, 4))
    val = 2.0 if kind == 1 else 37.5
    a, b = copy.copy(d), copy.copy(d)
    a.exceptions = Exceptions.build([(kind, val, [s], [], [])])
    b.exceptions = Exceptions.build([(kind, val, [], [], [[s]])])
    _same(oracle.update(a), oracle.update(b))
    has_fo = set(int(p) for n in range(d.num_nets) for p in d.net_pins[int(d.net_ptr[n]):int(d.net_ptr[n]) + 1])
    has_fo |= set(int(p) for p in d.arc_from)
    eps = [p for p in _endpoints(d) if p not in has_fo]
    if eps:
        e = int(rng.choice(eps))
        a.exceptions = Exceptions.build([(kind, val, [], [e], [])])
        b.exceptions = Exceptions.build([(kind, val, [], [], [[e]])])
        _same(oracle.update(a), oracle.update(b))


@pytest.mark.parametrize("seed", range(4))
def test_from_internal_pin_matches_nothing(seed):
    # -from names startpoints: a pin with fan-in starts no path,
    # so an exception -from it (with or without -through) changes nothing
    d = _tiny(seed)
    base = oracle.update(d)
    has_fi = sorted(set(int(p) for n in range(d.num_nets)
                        for p in d.net_pins[int(d.net_ptr[n]) + 1:int(d.net_ptr[n + 1])]))
    rng = np.random.default_rng(6000 + seed)
    x = int(rng.choice(has_fi))
    d1 = copy.copy(d)
    d1.exceptions = Exceptions.build([(0, 0.0, [x], [], []), (0, 0.0, [x], [], [[x]])])
    _same(oracle.update(d1), base)
