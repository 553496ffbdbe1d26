"""Pins of the oracle's case analysis (O16; SURVEY.md §8(f) row 4;
SPEC.md:479-486 apply_case_analysis; "case analysis
modes"): SPEC's own examples (an AND gate with a case-0 input, a MUX with a
case-1 select and when(S) / when(!S) guarded data arcs), constants carried
over nets and through inverter chains, contradictory constants, soundness
against an exhaustive simulation of the whole Boolean network (every pin the
analysis calls constant has that value under every assignment of the free
pins), the identity without case values, and the timing with the disabled
arcs against exhaustive path enumeration over the remaining arcs."""
import copy
import itertools

import numpy as np
import pytest

import oracle
import synth
from synth.design import CaseValues
from tests.brute import path_enumeration_timing
from tests.test_oracle_propagation import _bf_elm, _tiny


def _fn_index(d):
    return {int(p): i for i, p in enumerate(d.logic.fn_pin)}


def _inputs(d, i):
    lg = d.logic
    return [int(x) for x in lg.fn_in[int(lg.fn_in_ptr[i]):int(lg.fn_in_ptr[i + 1])]]


def _cells_of(d, tt, k):
    lg = d.logic
    return [i for i, t in enumerate(lg.fn_tt) if int(t) == tt and int(lg.fn_in_ptr[i + 1] - lg.fn_in_ptr[i]) == k]


def _arc_ids(d):
    """canonical arc ids (net arcs net by net, then cell arcs): (u, v, kind)"""
    out = []
    for n in range(d.num_nets):
        b, e = int(d.net_ptr[n]), int(d.net_ptr[n + 1])
        out += [(int(d.net_pins[b]), int(d.net_pins[j]), "net") for j in range(b + 1, e)]
    out += [(int(d.arc_from[a]), int(d.arc_to[a]), "cell") for a in range(d.num_arcs)]
    return out


def _driver_of(d):
    drv = {}
    for n in range(d.num_nets):
        b, e = int(d.net_ptr[n]), int(d.net_ptr[n + 1])
        for j in range(b + 1, e):
            drv[int(d.net_pins[j])] = int(d.net_pins[b])
    return drv


def _with_case(d, pins, vals):
    d2 = copy.copy(d)
    d2.case = CaseValues(np.array(pins, np.uint32), np.array(vals, np.uint8))
    return d2


def _design(seed=1, n=300):
    return synth.generate(n, 10, seed=seed, period=300.0)


def test_and_gate_with_case_zero_input():
    # AND gate with one input case-0 -> output constant 0, both
    # delay arcs disabled
    d = _design(1)
    i = _cells_of(d, synth.truth_table(lambda a, b: a & b, 2), 2)[0]
    a, b = _inputs(d, i)
    y = int(d.logic.fn_pin[i])
    val, off = oracle.case_analysis(_with_case(d, [a], [0]))
    assert val[a] == 0 and val[y] == 0
    ids = _arc_ids(d)
    for e, (u, v, kind) in enumerate(ids):
        if kind == "cell" and v == y:
            assert off[e] == 1                    # both delay arcs of the gate
        if kind == "net" and v == a:
            assert off[e] == 1                    # the net arc into the constant pin
    # the constant 0 is carried to every sink of the output's net and through them
    drv = _driver_of(d)
    for s, u in drv.items():
        if u == y:
            assert val[s] == 0
    # with the other input at 1 instead: not constant, the arcs from a stay enabled
    val1, off1 = oracle.case_analysis(_with_case(d, [b], [1]))
    if val1[a] == 2:                              # AND(a, 1) = a: not constant
        assert val1[y] == 2
        for e, (u, v, kind) in enumerate(ids):
            if kind == "cell" and v == y:
                assert off1[e] == (1 if u == b else 0)


def test_mux_select_and_when_guards():
    # MUX with select case-1 and arcs guarded when(S) / when(!S)
    # -> only the when(S) data arc stays enabled (the select arc starts at a
    # constant pin)
    d = _design(2, 600)
    mux = _cells_of(d, synth.truth_table(lambda a, b, s: b if s else a, 3), 3)
    assert mux, "no MUX2 in the design"
    i = mux[0]
    A, Bp, S = _inputs(d, i)
    y = int(d.logic.fn_pin[i])
    for sv, live in ((1, Bp), (0, A)):
        val, off = oracle.case_analysis(_with_case(d, [S], [sv]))
        assert val[S] == sv and val[y] == 2
        got = {u: int(off[e]) for e, (u, v, kind) in enumerate(_arc_ids(d)) if kind == "cell" and v == y}
        assert got[live] == 0 and got[S] == 1
        assert got[A if live == Bp else Bp] == 1      # its guard is false
    # no case value: the guards never disable (they evaluate to both values)
    val, off = oracle.case_analysis(_with_case(d, [], []))
    assert (val == 2).all() and not off.any()


def test_inverter_chain_and_xor():
    d = _design(3, 600)
    fi = _fn_index(d)
    inv = synth.truth_table(lambda a: 1 - a, 1)
    xor = synth.truth_table(lambda a, b: a ^ b, 2)
    drv = _driver_of(d)
    # an inverter's input at c gives 1 - c at its output and at all its sinks
    i = _cells_of(d, inv, 1)[0]
    (a,) = _inputs(d, i)
    y = int(d.logic.fn_pin[i])
    for c in (0, 1):
        val, _ = oracle.case_analysis(_with_case(d, [a], [c]))
        assert val[y] == 1 - c
        assert all(val[s] == 1 - c for s, u in drv.items() if u == y)
    # XOR with one constant input is not constant
    j = _cells_of(d, xor, 2)[0]
    a, b = _inputs(d, j)
    val, _ = oracle.case_analysis(_with_case(d, [a], [1]))
    assert val[int(d.logic.fn_pin[j])] == 2 or val[b] != 2
    del fi


def test_contradictory_constants():
    d = _design(4)
    i = _cells_of(d, synth.truth_table(lambda a: 1 - a, 1), 1)[0]
    (a,) = _inputs(d, i)
    y = int(d.logic.fn_pin[i])
    with pytest.raises(ValueError, match="contradictory"):
        oracle.case_analysis(_with_case(d, [a, y], [0, 0]))     # INV(0) = 1, pinned to 0
    with pytest.raises(ValueError, match="contradictory"):
        oracle.case_analysis(_with_case(d, [a, a], [0, 1]))
    oracle.case_analysis(_with_case(d, [a, y], [0, 1]))          # consistent: fine
    # a net carries its driver's constant to every sink: a sink pinned to the
    # other value contradicts it; pinned to the same value it is consistent
    drv = _driver_of(d)
    sinks = [s for s, u in drv.items() if u == y]
    assert sinks
    with pytest.raises(ValueError, match="contradictory"):
        oracle.case_analysis(_with_case(d, [a, sinks[0]], [0, 0]))   # y = 1, its sink pinned 0
    val, _ = oracle.case_analysis(_with_case(d, [a, sinks[0]], [0, 1]))
    assert all(val[s] == 1 for s in sinks)


def _simulate_all(d, case_pin, case_val):
    """exhaustive simulation of the Boolean network: the free pins (no
    function, not a net sink, no case value) take every assignment; sinks
    copy their driver unless pinned; pinned pins keep their value.  Returns
    per pin the set of values seen."""
    fi = _fn_index(d)
    drv = _driver_of(d)
    pinned = dict(zip(case_pin, case_val))
    free = [p for p in range(d.num_pins) if p not in fi and p not in drv and p not in pinned]
    order = oracle.levelize(d)[1]
    seen = [set() for _ in range(d.num_pins)]
    for bits in itertools.product((0, 1), repeat=len(free)):
        v = dict(zip(free, bits))
        v.update(pinned)
        for p in order:
            p = int(p)
            if p in pinned:
                continue
            if p in drv:
                v[p] = v[drv[p]]
            elif p in fi:
                ins = _inputs(d, fi[p])
                m = sum(v[x] << j for j, x in enumerate(ins))
                v[p] = (int(d.logic.fn_tt[fi[p]]) >> m) & 1
        for p, x in v.items():
            seen[p].add(x)
    return seen


@pytest.mark.parametrize("seed", range(12))
def test_constants_sound_vs_exhaustive_simulation(seed):
    d = _tiny(seed)
    rng = np.random.default_rng(700 + seed)
    drv = _driver_of(d)
    fi = _fn_index(d)
    free = [p for p in range(d.num_pins) if p not in fi and p not in drv]
    if len(free) > 14:
        pytest.skip("too many free pins for exhaustive simulation")
    pins = list(rng.choice(d.num_pins, size=int(rng.integers(1, 4)), replace=False))
    vals = list(rng.integers(0, 2, len(pins)))
    try:
        val, off = oracle.case_analysis(_with_case(d, pins, vals))
    except ValueError:
        pytest.skip("contradictory random constants")
    # a free pin that is pinned is excluded from `free` inside the simulation
    seen = _simulate_all(d, [int(p) for p in pins], [int(x) for x in vals])
    for p in range(d.num_pins):
        if val[p] != 2:
            assert seen[p] == {int(val[p])}, (p, val[p], seen[p])
    # every disabled arc touches a constant pin or has a guard that is false
    # in every simulation (the generated MUX guards)
    for e, (u, v, kind) in enumerate(_arc_ids(d)):
        if off[e] and val[u] == 2 and val[v] == 2:
            assert kind == "cell"


def test_no_case_values_is_identity():
    for seed in range(4):
        d = _tiny(seed)
        base = oracle.update(d)
        got = oracle.update(_with_case(d, [], []))
        for k in ("at", "slew", "rat", "slack"):
            assert np.array_equal(np.nan_to_num(base[k], posinf=1e300, neginf=-1e300),
                                  np.nan_to_num(got[k], posinf=1e300, neginf=-1e300))
        assert np.array_equal(base["res"], got["res"])


@pytest.mark.parametrize("seed", range(16))
def test_timing_with_disabled_arcs_vs_path_enumeration(seed):
    # every path over the arcs case analysis leaves enabled, enumerated
    d = _tiny(seed)
    rng = np.random.default_rng(900 + seed)
    pins = list(rng.choice(d.num_pins, size=int(rng.integers(1, 4)), replace=False))
    vals = list(rng.integers(0, 2, len(pins)))
    dc = _with_case(d, pins, vals)
    try:
        val, off = oracle.case_analysis(dc)
    except ValueError:
        pytest.skip("contradictory random constants")
    elm = _bf_elm(d)
    at, rat, slack, res = path_enumeration_timing(d, elm, off=off)
    o = oracle.update(dc)
    fin = np.isfinite(at)
    assert np.array_equal(fin, np.isfinite(o["at"]))
    np.testing.assert_allclose(o["at"][fin], at[fin], rtol=0, atol=1e-9)
    fs = np.isfinite(slack)
    assert np.array_equal(fs, np.isfinite(o["slack"]))
    np.testing.assert_allclose(o["slack"][fs], slack[fs], rtol=0, atol=1e-9)
    for a, b in zip(o["res"], res):
        assert (a == b) or abs(a - b) <= 1e-9 * max(1.0, abs(b))
