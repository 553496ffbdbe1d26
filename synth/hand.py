"""Hand-built tiny designs (SURVEY.md §8(c) hand examples H1, H2 = c17, H3).

Only structure and input values live here; expected timing values are in
tests/golden/ with their derivations.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

from .design import (Constraints, Design, Library, RcTree, NO_PIN,
                     ROLE_INTERNAL, ROLE_PI, ROLE_PO, ROLE_FF_CK, ROLE_FF_D,
                     SENSE_NEG, SENSE_NON, SENSE_RISE_EDGE, affine_table,
                     constant_table)


class Builder:
    """Tiny name-based netlist builder used for hand examples and unit tests."""

    def __init__(self):
        self.pins: List[str] = []
        self.pid: Dict[str, int] = {}
        self.cap: List[float] = []
        self.role: List[int] = []
        self.nets: List[Tuple[str, List[str], list]] = []   # (driver, sinks, rc)
        self.arcs: List[Tuple[str, str, int, int]] = []
        self.checks: List[Tuple[str, str, int]] = []
        self.tables: List[tuple] = []

    def pin(self, name, cap=0.0, role=ROLE_INTERNAL):
        self.pid[name] = len(self.pins)
        self.pins.append(name)
        self.cap.append(cap)
        self.role.append(role)
        return self.pid[name]

    def table(self, t) -> int:
        self.tables.append(t)
        return len(self.tables) - 1

    def tables4(self, t4) -> int:
        base = len(self.tables)
        for t in t4:
            self.tables.append(t)
        return base

    def net(self, driver, sinks, rc=None):
        """rc: list of (parent_local, R, Cw, pin_name_or_None) for nodes 0..n-1;
        None -> lumped net (no RC nodes)."""
        self.nets.append((driver, list(sinks), rc))

    def arc(self, a, b, sense, tab):
        self.arcs.append((a, b, sense, tab))

    def check(self, d, ck, tab):
        self.checks.append((d, ck, tab))

    def star_rc(self, driver, sinks, r, cw, drv_cw=0.0):
        """Driver node 0 plus one child per sink: R = r, Cw = cw."""
        rc = [(-1, 0.0, drv_cw, driver)]
        for s in sinks:
            rc.append((0, r, cw, s))
        return rc

    def build(self, cons: Constraints, name="hand") -> Design:
        net_ptr, net_pins = [0], []
        rc_ptr, parent, node_pin, res, cap = [0], [], [], [], []
        for drv, sinks, rc in self.nets:
            net_pins.append(self.pid[drv])
            net_pins.extend(self.pid[s] for s in sinks)
            net_ptr.append(len(net_pins))
            if rc is not None:
                for (p, r, c, pn) in rc:
                    parent.append(p)
                    res.append(r)
                    cap.append(c)
                    node_pin.append(NO_PIN if pn is None else self.pid[pn])
            rc_ptr.append(len(parent))
        lib = Library.from_tables(self.tables)
        rct = RcTree(np.array(rc_ptr, np.uint32), np.array(parent, np.int32),
                     np.array(node_pin, np.uint32), np.array(res, np.float32),
                     np.array(cap, np.float32))
        arcs = self.arcs
        return Design(
            num_pins=len(self.pins),
            pin_cap=np.array(self.cap, np.float32),
            pin_role=np.array(self.role, np.uint8),
            net_ptr=np.array(net_ptr, np.uint32),
            net_pins=np.array(net_pins, np.uint32),
            arc_from=np.array([self.pid[a] for a, _, _, _ in arcs], np.uint32),
            arc_to=np.array([self.pid[b] for _, b, _, _ in arcs], np.uint32),
            arc_sense=np.array([s for _, _, s, _ in arcs], np.uint8),
            arc_tab=np.array([t for _, _, _, t in arcs], np.uint32),
            chk_d=np.array([self.pid[d] for d, _, _ in self.checks], np.uint32),
            chk_ck=np.array([self.pid[c] for _, c, _ in self.checks], np.uint32),
            chk_tab=np.array([t for _, _, t in self.checks], np.uint32),
            libs=[lib], rc=[rct], cons=cons, name=name,
            meta=dict(pin_names=list(self.pins)))


def _cons(b: Builder, period, clock_slew, pis, pos):
    """pis: list of (name, at[4], slew[4]); pos: list of (name, out_max[2], out_min[2], load)."""
    return Constraints(
        float(period), float(clock_slew),
        np.array([b.pid[n] for n, _, _ in pis], np.uint32),
        np.array([a for _, a, _ in pis], np.float32).reshape(-1, 4),
        np.array([s for _, _, s in pis], np.float32).reshape(-1, 4),
        np.array([b.pid[n] for n, _, _, _ in pos], np.uint32),
        np.array([m for _, m, _, _ in pos], np.float32).reshape(-1, 2),
        np.array([m for _, _, m, _ in pos], np.float32).reshape(-1, 2),
        np.array([ld for _, _, _, ld in pos], np.float32))


# LIB-AFFINE: 7x7, index_1 slew, index_2 load.
AFFINE_SLEW = [5, 10, 20, 40, 80, 160, 320]
AFFINE_LOAD = [0.5, 1, 2, 4, 8, 16, 32]


def lib_affine_nand2():
    return [affine_table(AFFINE_SLEW, AFFINE_LOAD, 10, 0.1, 2.0),    # cell_rise
            affine_table(AFFINE_SLEW, AFFINE_LOAD, 8, 0.05, 1.5),    # cell_fall
            affine_table(AFFINE_SLEW, AFFINE_LOAD, 6, 0.2, 3.0),     # rise_transition
            affine_table(AFFINE_SLEW, AFFINE_LOAD, 4, 0.1, 2.0)]     # fall_transition


def c17() -> Design:
    """ISCAS-85 c17 as 6 NAND2 (SURVEY.md §8(c) H2 / BASELINE.json configs[0])."""
    b = Builder()
    pis = ["N1", "N2", "N3", "N6", "N7"]
    for n in pis:
        b.pin(n, 0.0, ROLE_PI)
    gates = [("N10", "N1", "N3"), ("N11", "N3", "N6"), ("N16", "N2", "N11"),
             ("N19", "N11", "N7"), ("N22", "N10", "N16"), ("N23", "N16", "N19")]
    base = b.tables4(lib_affine_nand2())
    for g, _, _ in gates:
        b.pin(f"{g}/A", 1.0)
        b.pin(f"{g}/B", 1.0)
        b.pin(f"{g}/Y", 0.0)
        b.arc(f"{g}/A", f"{g}/Y", SENSE_NEG, base)
        b.arc(f"{g}/B", f"{g}/Y", SENSE_NEG, base)
    b.pin("PO22", 0.0, ROLE_PO)
    b.pin("PO23", 0.0, ROLE_PO)
    # fan-out of each signal
    sinks: Dict[str, List[str]] = {}
    for g, a, bb in gates:
        sinks.setdefault(a, []).append(f"{g}/A")
        sinks.setdefault(bb, []).append(f"{g}/B")
    sinks["N22"] = ["PO22"]
    sinks["N23"] = ["PO23"]
    for sig in pis + [g for g, _, _ in gates]:
        drv = sig if sig in pis else f"{sig}/Y"
        s = sinks[sig]
        b.net(drv, s, b.star_rc(drv, s, 0.2, 0.5))
    cons = _cons(b, 45.0, 20.0,
                 [(n, [0, 0, 0, 0], [20, 20, 20, 20]) for n in pis],
                 [("PO22", [0, 0], [0, 0], 2.0), ("PO23", [0, 0], [0, 0], 2.0)])
    return b.build(cons, "c17")


def h1_chain() -> Design:
    """PI -> INV -> PO with constant tables."""
    b = Builder()
    b.pin("a", 0.0, ROLE_PI)
    b.pin("u1/A", 1.0)
    b.pin("u1/Y", 0.0)
    b.pin("y", 0.0, ROLE_PO)
    base = b.tables4([constant_table(10), constant_table(8),
                      constant_table(5), constant_table(4)])
    b.arc("u1/A", "u1/Y", SENSE_NEG, base)
    b.net("a", ["u1/A"], [(-1, 0.0, 0.0, "a"), (0, 1.0, 1.0, "u1/A")])
    b.net("u1/Y", ["y"], [(-1, 0.0, 0.0, "u1/Y"), (0, 0.5, 2.0, "y")])
    cons = _cons(b, 20.0, 20.0, [("a", [0, 0, 0, 0], [10, 10, 10, 10])],
                 [("y", [0, 0], [0, 0], 0.0)])
    return b.build(cons, "h1")


def h3_reg2reg() -> Design:
    """DFF1 -> XOR2 (non-unate) -> DFF2 with constant tables."""
    b = Builder()
    b.pin("DFF1/CK", 0.0, ROLE_FF_CK)
    b.pin("DFF1/Q", 0.0)
    b.pin("b", 0.0, ROLE_PI)
    b.pin("X/A", 1.0)
    b.pin("X/B", 1.0)
    b.pin("X/Y", 0.0)
    b.pin("DFF2/D", 1.0, ROLE_FF_D)
    b.pin("DFF2/CK", 0.0, ROLE_FF_CK)
    b.pin("DFF2/Q", 0.0)
    ckq = b.tables4([constant_table(30), constant_table(25),
                     constant_table(10), constant_table(8)])
    xor = b.tables4([constant_table(12), constant_table(11),
                     constant_table(6), constant_table(5)])
    chk = b.tables4([constant_table(7), constant_table(9),
                     constant_table(2), constant_table(3)])
    b.arc("DFF1/CK", "DFF1/Q", SENSE_RISE_EDGE, ckq)
    b.arc("X/A", "X/Y", SENSE_NON, xor)
    b.arc("X/B", "X/Y", SENSE_NON, xor)
    b.arc("DFF2/CK", "DFF2/Q", SENSE_RISE_EDGE, ckq)
    b.check("DFF2/D", "DFF2/CK", chk)
    # elm = R * Cdown = 1 ps for every net: R = 1 kOhm, node cap = pin cap 1 fF
    b.net("DFF1/Q", ["X/A"], [(-1, 0.0, 0.0, "DFF1/Q"), (0, 1.0, 0.0, "X/A")])
    b.net("b", ["X/B"], [(-1, 0.0, 0.0, "b"), (0, 1.0, 0.0, "X/B")])
    b.net("X/Y", ["DFF2/D"], [(-1, 0.0, 0.0, "X/Y"), (0, 1.0, 0.0, "DFF2/D")])
    cons = _cons(b, 60.0, 20.0, [("b", [5, 5, 5, 5], [10, 10, 10, 10])], [])
    return b.build(cons, "h3")


def h4_seeds() -> Design:
    """Hand example H4: pins the endpoint-seed lookups and
    the clock-slew seed, which H1-H3 leave free.

    DFF1/CK (ideal clock, slew = clock slew 16 ps) -RISE_EDGE-> DFF1/Q with
    AFFINE tables whose delay depends on the input slew, so the CK seed slew
    matters; NAND2 X (NEG) joins Q1 with PI b whose early and
    late slews differ; X/Y drives DFF2/D (setup/hold check against DFF2/CK)
    and a PO Z.  The check tables are affine a + b s_data + k s_clk with
    b != k on axes (data slew, clock slew), so swapping the
    arguments, or taking the early slew for setup / the late slew for hold,
    changes the required times.  Every net has R = 0 (Elmore 0, slews pass
    unchanged) so the hand derivation in tests/golden/h4_seeds.json stays
    exact.  Units ps / fF.
    """
    b = Builder()
    b.pin("DFF1/CK", 0.0, ROLE_FF_CK)
    b.pin("DFF1/Q", 0.0)
    b.pin("b", 0.0, ROLE_PI)
    b.pin("X/A", 1.0)
    b.pin("X/B", 1.0)
    b.pin("X/Y", 0.0)
    b.pin("DFF2/D", 2.0, ROLE_FF_D)
    b.pin("DFF2/CK", 0.0, ROLE_FF_CK)
    b.pin("Z", 0.0, ROLE_PO)
    S, L = AFFINE_SLEW, AFFINE_LOAD
    ckq = b.tables4([affine_table(S, L, 20, 0.5, 2.0), affine_table(S, L, 18, 0.4, 1.0),
                     affine_table(S, L, 4, 0.25, 1.0), affine_table(S, L, 3, 0.2, 1.0)])
    nand = b.tables4([affine_table(S, L, 10, 0.2, 2.0), affine_table(S, L, 8, 0.1, 3.0),
                      affine_table(S, L, 5, 0.5, 1.0), affine_table(S, L, 4, 0.25, 2.0)])
    # constraint tables: index_1 = data slew, index_2 = clock slew
    chk = b.tables4([affine_table(S, S, 5, 0.1, 0.3), affine_table(S, S, 6, 0.2, 0.05),
                     affine_table(S, S, 1, 0.05, 0.25), affine_table(S, S, -2, 0.3, 0.1)])
    b.arc("DFF1/CK", "DFF1/Q", SENSE_RISE_EDGE, ckq)
    b.arc("X/A", "X/Y", SENSE_NEG, nand)
    b.arc("X/B", "X/Y", SENSE_NEG, nand)
    b.check("DFF2/D", "DFF2/CK", chk)
    b.net("DFF1/Q", ["X/A"], b.star_rc("DFF1/Q", ["X/A"], 0.0, 0.0))
    b.net("b", ["X/B"], b.star_rc("b", ["X/B"], 0.0, 0.0))
    b.net("X/Y", ["DFF2/D", "Z"], b.star_rc("X/Y", ["DFF2/D", "Z"], 0.0, 0.0))
    cons = _cons(b, 50.0, 16.0, [("b", [2, 3, 6, 5], [8, 12, 40, 20])],
                 [("Z", [5, 6], [1, 2], 0.0)])
    return b.build(cons, "h4")
