"""Flat-array design container (the layout `include/sta.h` documents).

Units: ps, fF, kOhm (kOhm * fF = ps), following SPEC.md:113.
Enumerations mirror `sta_sense` / `sta_pin_role` in include/sta.h.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

SENSE_POS, SENSE_NEG, SENSE_NON, SENSE_RISE_EDGE, SENSE_FALL_EDGE = 0, 1, 2, 3, 4
ROLE_INTERNAL, ROLE_PI, ROLE_PO, ROLE_FF_CK, ROLE_FF_D = 0, 1, 2, 3, 4
NO_PIN = 0xFFFFFFFF


@dataclass
class Library:
    """A pool of NLDM tables (SPEC.md:30-45 `Lut2D`).

    Table t occupies data[off[t] : off[t] + n1 + n2 + n1*n2] as
    index_1[n1] (input slew or data slew, ps), index_2[n2] (load fF or clock
    slew ps), values[n1][n2] row-major (ps).
    """
    n1: np.ndarray      # uint8 [T]
    n2: np.ndarray      # uint8 [T]
    off: np.ndarray     # uint32 [T]
    data: np.ndarray    # float32 [sum]

    @property
    def num_tables(self) -> int:
        return int(self.n1.shape[0])

    @staticmethod
    def from_tables(tables: Sequence[tuple]) -> "Library":
        """tables: sequence of (idx1, idx2, values[n1][n2])."""
        n1, n2, off, chunks = [], [], [], []
        pos = 0
        for idx1, idx2, vals in tables:
            idx1 = np.asarray(idx1, dtype=np.float64).reshape(-1)
            idx2 = np.asarray(idx2, dtype=np.float64).reshape(-1)
            vals = np.asarray(vals, dtype=np.float64).reshape(idx1.size, idx2.size)
            n1.append(idx1.size)
            n2.append(idx2.size)
            off.append(pos)
            blob = np.concatenate([idx1, idx2, vals.reshape(-1)])
            chunks.append(blob)
            pos += blob.size
        return Library(np.array(n1, np.uint8), np.array(n2, np.uint8),
                       np.array(off, np.uint32),
                       np.concatenate(chunks).astype(np.float32))

    def table(self, t: int):
        a, b = int(self.n1[t]), int(self.n2[t])
        o = int(self.off[t])
        d = self.data[o:o + a + b + a * b]
        return d[:a], d[a:a + b], d[a + b:].reshape(a, b)

    def scaled(self, factor: float) -> "Library":
        """Same axes, values multiplied by `factor` (multi-corner recipe)."""
        data = self.data.copy()
        for t in range(self.num_tables):
            a, b = int(self.n1[t]), int(self.n2[t])
            o = int(self.off[t])
            data[o + a + b:o + a + b + a * b] *= np.float32(factor)
        return Library(self.n1.copy(), self.n2.copy(), self.off.copy(), data)


@dataclass
class RcTree:
    """Parent-array RC trees, one per net (SURVEY §8(b) `sta_set_rc`).

    Net n owns nodes [rc_ptr[n], rc_ptr[n+1]); node 0 of a net is the driver,
    parent[i] < i (local index), parent[0] = -1.  res[i] is the resistance of
    the edge parent->i (kOhm), cap[i] the wire cap to ground at node i (fF).
    node_pin[i] is the pin at that node or NO_PIN for Steiner/wire nodes.
    """
    rc_ptr: np.ndarray   # uint32 [N+1]
    parent: np.ndarray   # int32  [n_rc]   (local index within the net)
    node_pin: np.ndarray  # uint32 [n_rc]
    res: np.ndarray      # float32 [n_rc]
    cap: np.ndarray      # float32 [n_rc]

    def scaled(self, rs: float, cs: float) -> "RcTree":
        return RcTree(self.rc_ptr, self.parent, self.node_pin,
                      (self.res * np.float32(rs)).astype(np.float32),
                      (self.cap * np.float32(cs)).astype(np.float32))


@dataclass
class Constraints:
    """Single ideal clock + port constraints (SURVEY §8(b) `sta_constraints`)."""
    period: float
    clock_slew: float
    pi_pin: np.ndarray       # uint32 [n_pi]
    pi_at: np.ndarray        # float32 [n_pi][4]  (E_r, E_f, L_r, L_f)
    pi_slew: np.ndarray      # float32 [n_pi][4]
    po_pin: np.ndarray       # uint32 [n_po]
    po_out_max: np.ndarray   # float32 [n_po][2]  (r, f)
    po_out_min: np.ndarray   # float32 [n_po][2]
    po_load: np.ndarray      # float32 [n_po]


@dataclass
class Exceptions:
    """Timing exceptions: kind 0 false path, 1
    multicycle (value N), 2 max delay, 3 min delay (value ps); CSR lists of
    startpoint / endpoint pins (an empty list: any) and ordered -through
    segments: exception i's segments are thr_ptr[i] .. thr_ptr[i+1], segment
    s the pins seg_pins[seg_ptr[s] .. seg_ptr[s+1])."""
    kind: np.ndarray       # uint8 [E]
    value: np.ndarray      # float32 [E]
    from_ptr: np.ndarray   # uint32 [E+1]
    from_pins: np.ndarray  # uint32
    to_ptr: np.ndarray     # uint32 [E+1]
    to_pins: np.ndarray    # uint32
    thr_ptr: np.ndarray = None    # uint32 [E+1]
    seg_ptr: np.ndarray = None    # uint32 [n_seg+1]
    seg_pins: np.ndarray = None   # uint32

    @property
    def num(self) -> int:
        return int(self.kind.shape[0])

    @property
    def has_through(self) -> bool:
        return self.thr_ptr is not None and int(self.thr_ptr[-1]) > 0

    @staticmethod
    def build(items) -> "Exceptions":
        """items: sequence of (kind, value, from_pins, to_pins[, throughs]),
        throughs a sequence of pin lists (the -through segments, in order)."""
        items = [tuple(it) + ((),) * (5 - len(it)) for it in items]
        kind = np.array([it[0] for it in items], np.uint8)
        value = np.array([it[1] for it in items], np.float32)
        fp, tp, fr, to = [0], [0], [], []
        thp, sgp, sg = [0], [0], []
        for _, _, f, t, th in items:
            fr += list(f)
            to += list(t)
            fp.append(len(fr))
            tp.append(len(to))
            for seg in th:
                sg += list(seg)
                sgp.append(len(sg))
            thp.append(len(sgp) - 1)
        return Exceptions(kind, value, np.array(fp, np.uint32), np.array(fr, np.uint32),
                          np.array(tp, np.uint32), np.array(to, np.uint32),
                          np.array(thp, np.uint32), np.array(sgp, np.uint32), np.array(sg, np.uint32))


@dataclass
class Clocks:
    """Multiple ideal clocks: period per clock; pin_clk[P]
    = the clock of each FF_CK pin, the launch clock of each PI, the capture
    clock of each PO (other entries unused)."""
    period: np.ndarray     # float32 [n]
    pin_clk: np.ndarray    # uint32 [P]


@dataclass
class Logic:
    """Logic functions of cell outputs and `when` guards of cell arcs (case
    analysis): pin fn_pin[i] = truth table fn_tt[i] over
    the pins fn_in[fn_in_ptr[i] .. fn_in_ptr[i+1]) (input j = bit j of the
    table index, <= 6 inputs); arc_when[a] (optional) a truth table over the
    inputs of the function of arc_to[a], all ones = no guard."""
    fn_pin: np.ndarray      # uint32 [F]
    fn_in_ptr: np.ndarray   # uint32 [F+1]
    fn_in: np.ndarray       # uint32
    fn_tt: np.ndarray       # uint64 [F]
    arc_when: np.ndarray = None   # uint64 [A] or None


@dataclass
class CaseValues:
    """set_case_analysis constants: pin[k] = val[k] (0 / 1)."""
    pin: np.ndarray         # uint32 [n]
    val: np.ndarray         # uint8 [n]


def truth_table(fn, k: int) -> int:
    """the truth table of a Python predicate over k inputs (input j = bit j)"""
    return sum(1 << m for m in range(1 << k) if fn(*[(m >> j) & 1 for j in range(k)]))


@dataclass
class Design:
    num_pins: int
    pin_cap: np.ndarray      # float32 [P]
    pin_role: np.ndarray     # uint8 [P]
    net_ptr: np.ndarray      # uint32 [N+1]
    net_pins: np.ndarray     # uint32 [sum]   driver first
    arc_from: np.ndarray     # uint32 [A]
    arc_to: np.ndarray       # uint32 [A]
    arc_sense: np.ndarray    # uint8 [A]
    arc_tab: np.ndarray      # uint32 [A]  base of (cell_rise, cell_fall, rise_tr, fall_tr)
    chk_d: np.ndarray        # uint32 [C]
    chk_ck: np.ndarray       # uint32 [C]
    chk_tab: np.ndarray      # uint32 [C]  base of (setup_r, setup_f, hold_r, hold_f)
    libs: List[Library]      # one per corner
    rc: List[RcTree]         # one per corner (same topology)
    cons: Constraints
    name: str = "design"
    meta: dict = field(default_factory=dict)
    exceptions: Optional["Exceptions"] = None
    clocks: Optional["Clocks"] = None
    logic: Optional["Logic"] = None
    case: Optional["CaseValues"] = None

    @property
    def num_nets(self) -> int:
        return int(self.net_ptr.shape[0]) - 1

    @property
    def num_arcs(self) -> int:
        return int(self.arc_from.shape[0])

    @property
    def num_checks(self) -> int:
        return int(self.chk_d.shape[0])

    @property
    def num_corners(self) -> int:
        return len(self.libs)

    def with_period(self, period: float) -> "Design":
        import copy
        d = copy.copy(self)
        d.cons = copy.copy(self.cons)
        d.cons.period = float(period)
        return d

    def counts(self) -> dict:
        return dict(pins=self.num_pins, nets=self.num_nets,
                    net_arcs=int(self.net_pins.shape[0]) - self.num_nets,
                    cell_arcs=self.num_arcs, checks=self.num_checks,
                    rc_nodes=int(self.rc[0].parent.shape[0]),
                    corners=self.num_corners)


def as_u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32))


def as_f32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def empty_constraints(period: float = 1000.0, clock_slew: float = 20.0) -> Constraints:
    return Constraints(period, clock_slew,
                       np.zeros(0, np.uint32), np.zeros((0, 4), np.float32),
                       np.zeros((0, 4), np.float32), np.zeros(0, np.uint32),
                       np.zeros((0, 2), np.float32), np.zeros((0, 2), np.float32),
                       np.zeros(0, np.float32))


def constant_table(v: float):
    """1x1 table: a constant (SPEC.md:374 'scalar tables return the constant')."""
    return ([0.0], [0.0], [[v]])


def affine_table(idx1, idx2, a, b, k, m=0.0):
    """Table sampled from f(s,c) = a + b s + k c + m s c on the grid."""
    s = np.asarray(idx1, np.float64)[:, None]
    c = np.asarray(idx2, np.float64)[None, :]
    return (list(idx1), list(idx2), a + b * s + k * c + m * s * c)
