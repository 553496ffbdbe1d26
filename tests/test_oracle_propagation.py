"""Pins of the oracle's levelization (O2) and propagation/slack steps (O4-O9).

Golden hand examples (tests/golden/*.json, each with its citation), SPEC
worked examples, and exhaustive path enumeration on random tiny designs with
frozen (slew-independent) delays.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from synth.design import (Constraints, ROLE_FF_CK, ROLE_FF_D, ROLE_PI, ROLE_PO,
                          SENSE_NEG, SENSE_NON, SENSE_POS, constant_table,
                          empty_constraints)
from synth.hand import Builder, _cons
from tests.brute import (constant_library_like, design_node_caps, elmore_bruteforce,
                         longest_path_levels, path_enumeration_timing)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
HAND = {"h1_chain": synth.h1_chain, "c17": synth.c17, "h3_reg2reg": synth.h3_reg2reg,
        "h4_seeds": synth.h4_seeds}


def _f(x):
    return {"inf": math.inf, "-inf": -math.inf}.get(x, x) if isinstance(x, str) else x


def _close(a, b, tol):
    if math.isinf(b):
        return a == b
    return abs(a - b) <= tol


@pytest.mark.parametrize("name", ["h1_chain", "c17", "h3_reg2reg", "h4_seeds"])
def test_golden_hand_examples(name):
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    d = HAND[name]()
    pid = {n: i for i, n in enumerate(d.meta["pin_names"])}
    r = oracle.update(d)
    tol = g["tol"]
    for pin, exp in g["pins"].items():
        p = pid[pin]
        for key, arr, sl in [("at", r["at"], slice(0, 4)), ("slew", r["slew"], slice(0, 4)),
                             ("rat_late", r["rat"], slice(2, 4)), ("rat_early", r["rat"], slice(0, 2)),
                             ("slack_late", r["slack"], slice(2, 4)),
                             ("slack_early", r["slack"], slice(0, 2))]:
            if key in exp:
                got = arr[p, sl]
                for a, b in zip(got, exp[key]):
                    assert _close(a, _f(b), tol), (name, pin, key, got, exp[key])
    res = g["res"]
    for k, i in [("wns_setup", 0), ("tns_setup", 1), ("wns_hold", 2), ("tns_hold", 3)]:
        assert _close(r["res"][i], res[k], tol), (k, r["res"])
    if "min_pin_late_slack" in g:
        assert r["slack"][:, 2:].min() == pytest.approx(g["min_pin_late_slack"], abs=tol)
    if "levels" in g:
        level, perm, nl = oracle.levelize(d)
        assert nl == g["num_levels"]
        for pin, lv in g["levels"].items():
            assert level[pid[pin]] == lv, pin
    if "loads" in g:
        load, elm = oracle.rc(d)
        drv_net = {int(d.net_pins[d.net_ptr[n]]): n for n in range(d.num_nets)}
        for pin, ld in g["loads"].items():
            name_ = pin if pin in pid else pin
            assert load[drv_net[pid[name_]]] == pytest.approx(ld, abs=1e-6)
        for pin, e in g["elm"].items():
            assert elm[pid[pin]] == pytest.approx(e, abs=1e-6)


# ----------------------------------------------------- SPEC worked examples
def _chain(delays, T=5.0, po_out=0.0):
    """PI -> cell arcs with constant delays (net arcs zero-R) -> PO."""
    b = Builder()
    b.pin("in", 0.0, ROLE_PI)
    prev = "in"
    for i, dl in enumerate(delays):
        b.pin(f"g{i}/A", 0.0)
        b.pin(f"g{i}/Y", 0.0)
        base = b.tables4([constant_table(dl), constant_table(dl),
                          constant_table(1.0), constant_table(1.0)])
        b.arc(f"g{i}/A", f"g{i}/Y", SENSE_POS, base)
        b.net(prev, [f"g{i}/A"], b.star_rc(prev, [f"g{i}/A"], 0.0, 0.0))
        prev = f"g{i}/Y"
    b.pin("out", 0.0, ROLE_PO)
    b.net(prev, ["out"], b.star_rc(prev, ["out"], 0.0, 0.0))
    cons = _cons(b, T, 10.0, [("in", [0, 0, 0, 0], [5, 5, 5, 5])],
                 [("out", [po_out, po_out], [0, 0], 0.0)])
    return b.build(cons, "chain")


def test_spec_chain_arrival_and_slack():
    """chain with arcs 1 and 2 ps -> arrival 3; SPEC.md:512:
    delay 3, T = 5 -> slack +2; every pin of a single chain has
    the endpoint slack."""
    d = _chain([1.0, 2.0], T=5.0)
    r = oracle.update(d)
    pid = {n: i for i, n in enumerate(d.meta["pin_names"])}
    assert r["at"][pid["out"], 2] == pytest.approx(3.0)
    assert r["res"][0] == pytest.approx(2.0)
    defined = np.isfinite(r["at"][:, 2])
    assert np.allclose(r["slack"][defined, 2], 2.0)


def test_spec_levelize_chain():
    """chain of 3 arcs -> levels 0,1,2,3."""
    b = Builder()
    for n in "abcd":
        b.pin(n)
    base = b.tables4([constant_table(1)] * 4)
    b.net("a", ["b"], None)
    b.arc("b", "c", SENSE_POS, base)
    b.net("c", ["d"], None)
    d = b.build(empty_constraints())
    level, perm, nl = oracle.levelize(d)
    assert list(level) == [0, 1, 2, 3] and nl == 4


def test_levelize_detects_cycle():
    b = Builder()
    b.pin("x")
    b.pin("y")
    base = b.tables4([constant_table(1)] * 4)
    b.arc("x", "y", SENSE_NEG, base)
    b.arc("y", "x", SENSE_NEG, base)
    with pytest.raises(ValueError):
        oracle.levelize(b.build(empty_constraints()))


def test_spec_diamond():
    """reconvergent diamond with branch delays 1 and 5 -> late 5, early 1."""
    b = Builder()
    b.pin("in", 0.0, ROLE_PI)
    for g, dl in (("p", 1.0), ("q", 5.0)):
        b.pin(f"{g}/A")
        b.pin(f"{g}/Y")
        base = b.tables4([constant_table(dl), constant_table(dl), constant_table(1), constant_table(1)])
        b.arc(f"{g}/A", f"{g}/Y", SENSE_POS, base)
    b.pin("j/A")
    b.pin("j/B")
    b.net("in", ["p/A", "q/A"], None)
    b.net("p/Y", ["j/A"], None)
    b.net("q/Y", ["j/B"], None)
    # join through a zero-delay 2-input cell
    b.pin("j/Y")
    zb = b.tables4([constant_table(0)] * 2 + [constant_table(1)] * 2)
    b.arc("j/A", "j/Y", SENSE_POS, zb)
    b.arc("j/B", "j/Y", SENSE_POS, zb)
    cons = _cons(b, 100.0, 10.0, [("in", [0, 0, 0, 0], [1, 1, 1, 1])], [])
    d = b.build(cons)
    r = oracle.update(d)
    j = d.meta["pin_names"].index("j/Y")
    assert r["at"][j, 2] == 5.0 and r["at"][j, 0] == 1.0


def test_spec_wns_tns_and_fork():
    """endpoint slacks {-1,-2,+3} -> WNS -2, TNS -3.
    SPEC.md:531: fork to endpoints with slacks {+1,-4} -> shared prefix -4."""
    b = Builder()
    b.pin("in", 0.0, ROLE_PI)
    b.pin("s/A")
    b.pin("s/Y")
    b.arc("s/A", "s/Y", SENSE_POS, b.tables4([constant_table(0)] * 4))
    b.net("in", ["s/A"], None)
    outs = ["o1", "o2", "o3"]
    for o in outs:
        b.pin(o, 0.0, ROLE_PO)
    b.net("s/Y", outs, None)
    # T = 10, AT = 0 -> slack = 10 - out_max
    cons = _cons(b, 10.0, 5.0, [("in", [0, 0, 0, 0], [1, 1, 1, 1])],
                 [("o1", [11, 11], [0, 0], 0.0), ("o2", [12, 12], [0, 0], 0.0),
                  ("o3", [7, 7], [0, 0], 0.0)])
    d = b.build(cons)
    r = oracle.update(d)
    assert r["res"][0] == pytest.approx(-2.0)
    assert r["res"][1] == pytest.approx(-3.0)
    s = d.meta["pin_names"].index("s/A")
    assert r["slack"][s, 2] == pytest.approx(-2.0)    # shared prefix sees the worst
    # fork {+1, -4}
    cons2 = _cons(b, 10.0, 5.0, [("in", [0, 0, 0, 0], [1, 1, 1, 1])],
                  [("o1", [9, 9], [0, 0], 0.0), ("o2", [14, 14], [0, 0], 0.0)])
    b.pins = b.pins  # same structure, o3 now unconstrained
    d2 = b.build(cons2)
    r2 = oracle.update(d2)
    assert r2["slack"][s, 2] == pytest.approx(-4.0)
    o3 = d2.meta["pin_names"].index("o3")
    assert r2["slack"][o3, 2] == math.inf      # unconstrained: +inf sentinel


def test_peri_345():
    """net slew sqrt(drv^2 + imp^2): drv 30, impulse 40 -> 50.
    impulse = ln 9 * Elmore, so choose Elmore = 40 / ln 9."""
    b = Builder()
    b.pin("in", 0.0, ROLE_PI)
    b.pin("s", 0.0)
    e = 40.0 / math.log(9.0)
    cap = np.float32(e)           # R = 1 kOhm, node cap = e fF
    b.net("in", ["s"], [(-1, 0.0, 0.0, "in"), (0, 1.0, float(cap), "s")])
    b.table(constant_table(1))
    cons = _cons(b, 100.0, 5.0, [("in", [0, 0, 0, 0], [30, 30, 30, 30])], [])
    r = oracle.update(b.build(cons))
    imp = math.log(9.0) * float(cap)
    assert r["slew"][1, 2] == pytest.approx(math.hypot(30.0, imp), rel=1e-12)
    assert r["slew"][1, 2] == pytest.approx(50.0, abs=1e-4)


# ---------------------------------------- brute force on random tiny designs
def _tiny(seed):
    rng = np.random.default_rng(seed)
    n_cells = int(rng.integers(6, 14))
    levels = int(rng.integers(4, 9))
    d = synth.generate(n_cells, levels, seed=seed, frac_pi=0.15, frac_po=0.15, period=80.0)
    d.libs = [constant_library_like(d.libs[0], rng)]
    # exercise every sense, including FALL_EDGE and NON on random arcs
    flip = rng.random(d.num_arcs) < 0.35
    d.arc_sense = d.arc_sense.copy()
    d.arc_sense[flip] = rng.integers(0, 5, int(flip.sum())).astype(np.uint8)
    # leave one PI unconstrained: an undefined (+-inf) source
    if d.cons.pi_pin.size >= 2 and seed % 2 == 0:
        import copy
        d.cons = copy.copy(d.cons)
        d.cons.pi_pin, d.cons.pi_at, d.cons.pi_slew = (d.cons.pi_pin[1:], d.cons.pi_at[1:],
                                                       d.cons.pi_slew[1:])
    return d


def _bf_elm(d):
    rc = d.rc[0]
    caps = design_node_caps(d)
    elm = np.zeros(d.num_pins)
    for n in range(d.num_nets):
        b, e = int(rc.rc_ptr[n]), int(rc.rc_ptr[n + 1])
        if e == b:
            continue
        ref = elmore_bruteforce(list(rc.parent[b:e]), list(rc.res[b:e].astype(float)),
                                list(caps[b:e]))
        for i in range(1, e - b):
            if rc.node_pin[b + i] != 0xFFFFFFFF:
                elm[int(rc.node_pin[b + i])] = ref[i]
    return elm


@pytest.mark.parametrize("seed", range(25))
def test_random_dag_levels_vs_path_enumeration(seed):
    """level = longest path depth; level(u) < level(v) on every arc;
    perm = stable sort by (level, id)."""
    d = _tiny(seed)
    level, perm, nl = oracle.levelize(d)
    ref = longest_path_levels(d)
    assert np.array_equal(level, ref)
    assert nl == ref.max() + 1
    key = level.astype(np.int64) * d.num_pins + np.arange(d.num_pins)
    assert np.array_equal(perm, np.argsort(key, kind="stable"))


@pytest.mark.parametrize("seed", range(25))
def test_random_dag_timing_vs_path_enumeration(seed):
    """SPEC.md:539/688 (acceptance #4): with frozen delays, AT = max/min over
    enumerated paths, RAT over enumerated paths to endpoints, slack/WNS/TNS from
    those -- exact to 1e-9."""
    d = _tiny(seed)
    r = oracle.update(d)
    at, rat, slack, res = path_enumeration_timing(d, _bf_elm(d))

    def eq(a, b):
        fin = np.isfinite(b)
        assert np.array_equal(np.isfinite(a), fin)
        assert np.array_equal(a[~fin], b[~fin])
        assert np.allclose(a[fin], b[fin], rtol=1e-9, atol=1e-9)

    eq(r["at"], at)
    eq(r["rat"], rat)
    eq(r["slack"], slack)
    assert np.allclose(r["res"], res, rtol=1e-9, atol=1e-9) or \
        all((x == y) or abs(x - y) < 1e-9 for x, y in zip(r["res"], res))


@pytest.mark.parametrize("seed", [11, 12])
def test_generated_design_invariants(seed):
    """On a LIB-SYN design (slew-dependent tables): min over all pins of the late
    slack equals WNS_setup (and early/hold likewise) -- slack(u) >= min slack of
    its successors along any arc, attained at the worst endpoint."""
    d = synth.generate(3000, 24, seed=seed, period=300.0)
    r = oracle.update(d)
    assert r["slack"][:, 2:].min() == pytest.approx(r["res"][0], abs=1e-9)
    assert r["slack"][:, :2].min() == pytest.approx(r["res"][2], abs=1e-9)
    level, _, nl = oracle.levelize(d)
    # level invariant over every net and cell arc
    for n in range(d.num_nets):
        b, e = int(d.net_ptr[n]), int(d.net_ptr[n + 1])
        assert np.all(level[d.net_pins[b + 1:e]] > level[d.net_pins[b]])
    assert np.all(level[d.arc_to] > level[d.arc_from])


def test_multicorner_global_reduction():
    """O9: per-corner update; global WNS = min, TNS = sum."""
    d = synth.generate(800, 16, seed=5, corners=3, corner_recipe="c5", period=150.0)
    per, glob = oracle.update_all_corners(d)
    assert glob[0] == min(p["res"][0] for p in per)
    assert glob[1] == pytest.approx(sum(p["res"][1] for p in per))
    # corners differ (scaled tables / RC) and slower corners are worse
    assert per[2]["at"][:, 2][np.isfinite(per[2]["at"][:, 2])].max() > \
        per[0]["at"][:, 2][np.isfinite(per[0]["at"][:, 2])].max()


def test_negative_table_values_clamp_to_zero():
    """arc delays are clamped at >= 0 and slews stay >= 0;
    setup/hold constraint values are NOT clamped (they may be negative)."""
    b = Builder()
    b.pin("in", 0.0, ROLE_PI)
    b.pin("g/A")
    b.pin("g/Y")
    b.pin("ff/D", 0.0, ROLE_FF_D)
    b.pin("ff/CK", 0.0, ROLE_FF_CK)
    base = b.tables4([constant_table(-5.0), constant_table(-3.0),
                      constant_table(-2.0), constant_table(-1.0)])
    b.arc("g/A", "g/Y", SENSE_POS, base)
    chk = b.tables4([constant_table(-4.0), constant_table(-4.0),
                     constant_table(-6.0), constant_table(-6.0)])
    b.check("ff/D", "ff/CK", chk)
    b.net("in", ["g/A"], None)
    b.net("g/Y", ["ff/D"], None)
    cons = _cons(b, 10.0, 5.0, [("in", [1, 1, 2, 2], [3, 3, 3, 3])], [])
    d = b.build(cons)
    r = oracle.update(d)
    y = d.meta["pin_names"].index("g/Y")
    D = d.meta["pin_names"].index("ff/D")
    assert list(r["at"][y]) == [1, 1, 2, 2]         # zero delay, not -5
    assert list(r["slew"][y]) == [0, 0, 0, 0]
    assert list(r["rat"][D, 2:]) == [14, 14]        # T - (-4)
    assert list(r["rat"][D, :2]) == [-6, -6]        # hold value, negative allowed


# ------------------------------------------- O10: top-k path report (f3)
from tests.brute import path_list_bruteforce, select_paths  # noqa: E402


def _same_paths(got, exp):
    assert len(got) == len(exp), (len(got), len(exp))
    for g, e in zip(got, exp):
        assert abs(g["slack"] - e[0]) <= 1e-9 * max(1.0, abs(e[0])), (g["slack"], e[0])
        assert g["ep"] == e[1]
        assert list(zip(g["pins"], g["rfs"])) == list(e[2]), (g, e)
        assert np.allclose(g["at"], e[3], rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("mode", ["setup", "hold"])
def test_paths_vs_exhaustive_enumeration(seed, mode):
    """SPEC.md path-report acceptance: with k = inf the report is exactly the
    set of paths found by exhaustive DFS, same slacks, same order (frozen
    delays: constant tables, all five senses, undefined sources)."""
    d = _tiny(seed)
    allp = path_list_bruteforce(d, _bf_elm(d), mode)
    big = 10 ** 6
    _same_paths(oracle.paths(d, mode=mode, k=big, nworst=big), allp)
    # selections: k, nworst, slack-less-than
    for k, nw in [(1, 1), (3, 1), (5, 2), (7, 100)]:
        _same_paths(oracle.paths(d, mode=mode, k=k, nworst=nw), select_paths(allp, k, nw))
    if allp:
        thr = allp[len(allp) // 2][0]
        _same_paths(oracle.paths(d, mode=mode, k=big, nworst=3, slack_lt=thr),
                    select_paths(allp, big, 3, thr))


def test_paths_golden_h3():
    """Hand example H3 (tests/golden/h3_reg2reg.json): the worst setup path
    is CK1 rise -> Q rise -> X/A rise -> X/Y fall -> D fall with slack 8 =
    WNS_setup; the worst hold path starts at PI b with slack 15 = WNS_hold."""
    d = synth.h3_reg2reg()
    names = d.meta["pin_names"]
    s = oracle.paths(d, mode="setup", k=1, nworst=1)[0]
    assert s["slack"] == pytest.approx(8.0, abs=1e-9)
    assert [names[p] for p in s["pins"]] == ["DFF1/CK", "DFF1/Q", "X/A", "X/Y", "DFF2/D"]
    assert s["rfs"] == [0, 0, 0, 1, 1] and s["at"] == pytest.approx([0, 30, 31, 42, 43])
    h = oracle.paths(d, mode="hold", k=1, nworst=1)[0]
    assert h["slack"] == pytest.approx(15.0, abs=1e-9) and names[h["pins"][0]] == "b"


@pytest.mark.parametrize("seed", [11, 12])
def test_paths_worst_equals_wns(seed):
    """SPEC path-report invariant: the first setup path's slack is WNS
    (endpoints without fan-out), slacks are non-decreasing, nworst holds, and
    each path's arrivals are its startpoint arrival plus the arc delays."""
    d = synth.generate(300, 12, seed=seed, period=150.0)
    r = oracle.update(d)
    for mode, col in (("setup", 0), ("hold", 2)):
        ps = oracle.paths(d, mode=mode, k=200, nworst=3)
        assert ps[0]["slack"] == pytest.approx(r["res"][col], abs=1e-9)
        sl = [p["slack"] for p in ps]
        assert all(a <= b for a, b in zip(sl, sl[1:]))
        from collections import Counter
        assert max(Counter(p["ep"] for p in ps).values()) <= 3
        for p in ps:
            assert all(b >= a - 1e-12 for a, b in zip(p["at"], p["at"][1:]))   # delays >= 0
