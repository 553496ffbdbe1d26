"""Seeded synthetic netlists shaped like the paper's workloads.

Recipe, all vectorised numpy, deterministic for a seed:

* LIB-SYN: INV, BUF, NAND2, NOR2, AND2, OR2, XOR2 (non-unate), AOI21, OAI21,
  MUX2 (select non-unate), DFF (CK->Q rising edge, setup/hold on D).  7x7
  tables, index_1 slew {1,5,15,40,90,180,360} ps, index_2 load
  {0.1,0.5,1.5,4,9,18,36} fF, values a + b s + k c + m sqrt(s c) + noise
  (deliberately not bilinear).
* Shape ratios from PAPER.md:224-236, 269-276: ~2.85 pins/cell, ~1.23
  arcs/pin, ~1.8 sinks/net (power-law fan-out budgets k^-2.5 on 1..200),
  10% DFF, 1% PI, 1% PO.
* Gate depth d in [1, D] with a decaying histogram exp(-(d-1)/(D/4)) + 0.03,
  every depth populated; input 0 of a depth-d cell is driven from depth d-1
  (so pin levels ~ 2D+2), other inputs from any depth < d; endpoints (D pins,
  POs) absorb any leftover driver slots.
* Optional high-fan-out nets (superblue-like): PIs with log-uniform fan-out,
  wire R scaled by 0.1 (thick upper-layer routing).
* RC: random recursive tree per net, driver = node 0, one node per sink plus
  floor(k/2) Steiner nodes, R U[0.02,0.2] kOhm, Cw U[0.1,1.0] fF.
* Constraints: PI AT U[0,50] ps, slew U[5,40] ps, output delays U[0,50],
  PO load U[1,4] fF, clock slew 20 ps.  The clock period is calibrated once
  by `scripts/calibrate_periods.py` (oracle only) and stored in
  synth/periods.json.
"""
from __future__ import annotations

import json
import os
from typing import List, Optional

import numpy as np

from .design import (Constraints, Design, Library, RcTree, NO_PIN,
                     ROLE_INTERNAL, ROLE_PI, ROLE_PO, ROLE_FF_CK, ROLE_FF_D,
                     SENSE_POS, SENSE_NEG, SENSE_NON, SENSE_RISE_EDGE)

SLEW_AXIS = [1.0, 5.0, 15.0, 40.0, 90.0, 180.0, 360.0]
LOAD_AXIS = [0.1, 0.5, 1.5, 4.0, 9.0, 18.0, 36.0]
CLK_SLEW_AXIS = [5.0, 10.0, 20.0, 40.0, 80.0, 160.0, 320.0]

# (name, input senses, probability)
COMB = [
    ("INV", [SENSE_NEG], 0.22),
    ("BUF", [SENSE_POS], 0.10),
    ("NAND2", [SENSE_NEG, SENSE_NEG], 0.16),
    ("NOR2", [SENSE_NEG, SENSE_NEG], 0.12),
    ("AND2", [SENSE_POS, SENSE_POS], 0.08),
    ("OR2", [SENSE_POS, SENSE_POS], 0.07),
    ("XOR2", [SENSE_NON, SENSE_NON], 0.07),
    ("AOI21", [SENSE_NEG] * 3, 0.07),
    ("OAI21", [SENSE_NEG] * 3, 0.06),
    ("MUX2", [SENSE_POS, SENSE_POS, SENSE_NON], 0.05),
]
MAX_IN = 3

# logic functions of the comb cells (case analysis),
# inputs in pin order; MUX2 = (A, B, S) -> S ? B : A with its data arcs
# guarded when(!S) / when(S)
COMB_FN = {
    "INV": lambda a: 1 - a, "BUF": lambda a: a,
    "NAND2": lambda a, b: 1 - (a & b), "NOR2": lambda a, b: 1 - (a | b),
    "AND2": lambda a, b: a & b, "OR2": lambda a, b: a | b, "XOR2": lambda a, b: a ^ b,
    "AOI21": lambda a, b, c: 1 - ((a & b) | c), "OAI21": lambda a, b, c: 1 - ((a | b) & c),
    "MUX2": lambda a, b, s: b if s else a,
}
ALL_ONES = np.uint64(0xFFFFFFFFFFFFFFFF)


def _logic(ctype, cell_base, n_in, comb_out, cons_cell, cons_j, arc_order):
    """Logic of the generated comb cells (no RNG: the design is unchanged)."""
    from .design import Logic, truth_table
    tts = np.array([truth_table(COMB_FN[name], len(sens)) for name, sens, _ in COMB], np.uint64)
    n_comb = ctype.shape[0]
    fn_in_ptr = np.zeros(n_comb + 1, np.int64)
    fn_in_ptr[1:] = np.cumsum(n_in)
    fn_in = (np.repeat(cell_base[:n_comb], n_in) + (np.arange(int(fn_in_ptr[-1])) - np.repeat(fn_in_ptr[:-1], n_in)))
    when = np.full(arc_order.shape[0], ALL_ONES, np.uint64)   # comb arcs (consumer order), then CK -> Q
    mux = [i for i, (name, _, _) in enumerate(COMB) if name == "MUX2"][0]
    on_mux = ctype[cons_cell] == mux
    g_a = np.uint64(truth_table(lambda a, b, s: 1 - s, 3))
    g_b = np.uint64(truth_table(lambda a, b, s: s, 3))
    idx = np.nonzero(on_mux & (cons_j == 0))[0]
    when[idx] = g_a
    idx = np.nonzero(on_mux & (cons_j == 1))[0]
    when[idx] = g_b
    return Logic(comb_out.astype(np.uint32), fn_in_ptr.astype(np.uint32), fn_in.astype(np.uint32),
                 tts[ctype], when[arc_order])

# name -> (n_cells, pin levels, seed, n_hfn, corners, corner recipe)
CONFIGS = {
    "c2_tau": dict(n_cells=52_000, levels=60, seed=0x7A2015, n_hfn=0, corners=1),
    "c3_superblue": dict(n_cells=3_600_000, levels=150, seed=0x5B10, n_hfn=32, corners=1),
    "c4_tdp": dict(n_cells=1_000_000, levels=120, seed=0xD9E4, n_hfn=0, corners=1),
    "c5_multicorner": dict(n_cells=700_000, levels=150, seed=0xC0E8, n_hfn=0, corners=8,
                           corner_recipe="c5"),
}

_PERIODS_FILE = os.path.join(os.path.dirname(__file__), "periods.json")


def corner_scales(c: int, recipe: str = "nominal"):
    """(lut, R, Cw) multipliers of corner c.

    c5: SURVEY.md §8(d) C5 row: LUT x (0.80 + 0.06c), R x (0.85 + 0.05c),
    Cw x (0.90 + 0.03c).  nominal: corner 0 is the design as generated and
    corner c scales by (1 + 0.05c, 1 + 0.04c, 1 + 0.03c) -- used when a
    single-corner config is replicated one corner per GPU.
    """
    if recipe == "c5":
        return 0.80 + 0.06 * c, 0.85 + 0.05 * c, 0.90 + 0.03 * c
    return 1.0 + 0.05 * c, 1.0 + 0.04 * c, 1.0 + 0.03 * c


def _lib_syn(rng):
    """LIB-SYN table pool. Returns (Library, arc_base[type][j], ckq_base, chk_base,
    in_cap[type][j], d_cap)."""
    s = np.array(SLEW_AXIS)[:, None]
    c = np.array(LOAD_AXIS)[None, :]
    tables = []

    def nldm(a_rng, b_rng, k_rng, m_rng):
        a = rng.uniform(*a_rng)
        b = rng.uniform(*b_rng)
        k = rng.uniform(*k_rng)
        m = rng.uniform(*m_rng)
        noise = rng.uniform(-0.05, 0.05, size=(7, 7)) * a
        return (SLEW_AXIS, LOAD_AXIS, a + b * s + k * c + m * np.sqrt(s * c) + noise)

    def arc4():
        base = len(tables)
        tables.append(nldm((4, 20), (0.05, 0.3), (0.8, 5), (0.0, 0.3)))    # cell_rise
        tables.append(nldm((4, 20), (0.05, 0.3), (0.8, 5), (0.0, 0.3)))    # cell_fall
        tables.append(nldm((2, 8), (0.05, 0.25), (1.0, 6), (0.0, 0.3)))    # rise_tr
        tables.append(nldm((2, 8), (0.05, 0.25), (1.0, 6), (0.0, 0.3)))    # fall_tr
        return base

    arc_base = np.zeros((len(COMB), MAX_IN), np.uint32)
    in_cap = np.zeros((len(COMB), MAX_IN), np.float32)
    for t, (_, senses, _) in enumerate(COMB):
        for j in range(len(senses)):
            arc_base[t, j] = arc4()
            in_cap[t, j] = rng.uniform(0.5, 2.0)
    ckq_base = arc4()
    chk_base = len(tables)
    ds = np.array(SLEW_AXIS)[:, None]
    cs = np.array(CLK_SLEW_AXIS)[None, :]
    for (a_lo, a_hi) in [(5, 15), (5, 15), (-3, 5), (-3, 5)]:  # setup r/f, hold r/f
        a = rng.uniform(a_lo, a_hi)
        b = rng.uniform(0.02, 0.1)
        k = rng.uniform(-0.05, 0.05)
        tables.append((SLEW_AXIS, CLK_SLEW_AXIS, a + b * ds + k * cs))
    d_cap = rng.uniform(0.5, 2.0)
    return Library.from_tables(tables), arc_base, ckq_base, chk_base, in_cap, d_cap


def _powerlaw_budgets(rng, n, alpha=2.5, kmax=200):
    k = np.arange(1, kmax + 1, dtype=np.float64)
    p = k ** (-alpha)
    p /= p.sum()
    return rng.choice(kmax, size=n, p=p).astype(np.int64) + 1


def generate(n_cells: int, levels: int, seed: int, n_hfn: int = 0,
             hfn_range=(1e3, 1e5), corners: int = 1, corner_recipe: str = "nominal",
             frac_dff: float = 0.1, frac_pi: float = 0.01, frac_po: float = 0.01,
             period: Optional[float] = None, name: str = "synthetic") -> Design:
    rng = np.random.default_rng(seed)
    lib, arc_base, ckq_base, chk_base, in_cap, d_cap = _lib_syn(rng)

    D = max(1, levels // 2 - 1)
    n_dff = int(round(frac_dff * n_cells))
    n_comb = n_cells - n_dff
    if n_comb < D:
        raise ValueError("need at least D combinational cells")
    n_pi = max(1, int(round(frac_pi * n_cells)))
    n_po = max(1, int(round(frac_po * n_cells)))

    probs = np.array([p for _, _, p in COMB])
    probs /= probs.sum()
    ctype = rng.choice(len(COMB), size=n_comb, p=probs)
    n_in_of_type = np.array([len(s) for _, s, _ in COMB])
    n_in = n_in_of_type[ctype]
    dw = np.exp(-np.arange(D) / max(D / 4.0, 1e-9)) + 0.03
    depth = rng.choice(D, size=n_comb, p=dw / dw.sum()).astype(np.int64) + 1
    depth[:D] = np.arange(1, D + 1)          # every depth populated

    # ---- drivers: PI ports, DFF Q pins (depth 0), comb outputs (depth d) ----
    nd = n_pi + n_dff + n_comb
    drv_depth = np.concatenate([np.zeros(n_pi + n_dff, np.int64), depth])
    budget = _powerlaw_budgets(rng, nd)
    slot_drv = np.repeat(np.arange(nd), budget)
    slot_depth = drv_depth[slot_drv]
    # slots sorted by (depth, random)
    order = np.lexsort((rng.random(slot_drv.size), slot_depth))
    slot_drv = slot_drv[order]
    slot_depth = slot_depth[order]
    slot_start = np.searchsorted(slot_depth, np.arange(D + 2), side="left")
    slot_cnt = slot_start[1:] - slot_start[:-1]            # per depth 0..D

    # drivers sorted by depth for overflow picks
    drv_by_depth = np.argsort(drv_depth, kind="stable")
    drv_start = np.searchsorted(drv_depth[drv_by_depth], np.arange(D + 2), side="left")

    # consumer table: comb inputs (cell, j), then DFF D pins, then PO ports
    cons_cell = np.repeat(np.arange(n_comb), n_in)
    cons_j = np.arange(cons_cell.size) - np.repeat(np.cumsum(n_in) - n_in, n_in)
    n_ci = cons_cell.size
    cons_drv = np.full(n_ci + n_dff + n_po, -1, np.int64)
    slot_used = np.zeros(slot_drv.size, bool)

    # forced inputs (j == 0): exactly depth d-1, matched to slots of that depth
    f_idx = np.nonzero(cons_j == 0)[0]
    f_t = depth[cons_cell[f_idx]] - 1
    f_order = np.lexsort((rng.random(f_idx.size), f_t))
    f_idx, f_t = f_idx[f_order], f_t[f_order]
    f_rank = np.arange(f_idx.size) - np.searchsorted(f_t, f_t, side="left")
    ok = f_rank < slot_cnt[f_t]
    s_take = slot_start[f_t[ok]] + f_rank[ok]
    cons_drv[f_idx[ok]] = slot_drv[s_take]
    slot_used[s_take] = True
    if (~ok).any():
        t = f_t[~ok]
        lo, hi = drv_start[t], drv_start[t + 1]
        cons_drv[f_idx[~ok]] = drv_by_depth[lo + (rng.random(t.size) * (hi - lo)).astype(np.int64)]

    # flexible inputs (j >= 1): any depth < d, from the leftover slot pool
    x_idx = np.nonzero(cons_j > 0)[0]
    x_bound = depth[cons_cell[x_idx]]
    x_order = np.argsort(x_bound, kind="stable")
    x_idx, x_bound = x_idx[x_order], x_bound[x_order]
    x_start = np.searchsorted(x_bound, np.arange(D + 2), side="left")
    pool = np.zeros(0, np.int64)
    for d in range(1, D + 1):
        lo_s, hi_s = slot_start[d - 1], slot_start[d]
        new = np.arange(lo_s, hi_s)
        pool = np.concatenate([pool, new[~slot_used[new]]])
        want = x_idx[x_start[d]:x_start[d + 1]]
        m = want.size
        if m == 0:
            continue
        if m >= pool.size:
            take, rest = pool, np.zeros(0, np.int64)
        else:
            sel = np.argpartition(rng.random(pool.size), m)
            take, rest = pool[sel[:m]], pool[sel[m:]]
        cons_drv[want[:take.size]] = slot_drv[take]
        slot_used[take] = True
        pool = rest
        if m > take.size:
            k = m - take.size
            cons_drv[want[take.size:]] = drv_by_depth[(rng.random(k) * drv_start[d]).astype(np.int64)]

    # endpoints (DFF D pins, PO ports): any depth, prefer unused slots whose
    # driver has no sink yet, then any leftover slot, then uniform drivers
    e_idx = np.arange(n_ci, n_ci + n_dff + n_po)
    rng.shuffle(e_idx)
    fan = np.bincount(cons_drv[cons_drv >= 0], minlength=nd)
    pool = np.concatenate([pool, np.arange(slot_start[D], slot_start[D + 1])])
    pool = pool[~slot_used[pool]]
    pool = pool[np.lexsort((rng.random(pool.size), fan[slot_drv[pool]] > 0))]
    # at most one slot per driver in the first pass so coverage spreads
    first = pool[np.unique(slot_drv[pool], return_index=True)[1]]
    first = first[np.lexsort((rng.random(first.size), fan[slot_drv[first]] > 0))]
    k1 = min(first.size, e_idx.size)
    cons_drv[e_idx[:k1]] = slot_drv[first[:k1]]
    if e_idx.size > k1:
        k = e_idx.size - k1
        cons_drv[e_idx[k1:]] = drv_by_depth[(rng.random(k) * drv_start[D + 1]).astype(np.int64)]

    # high-fan-out nets: PIs grab random flexible comb inputs
    hfn_fanouts = []
    if n_hfn > 0:
        n_hfn = min(n_hfn, n_pi)
        fo = np.exp(rng.uniform(np.log(hfn_range[0]), np.log(hfn_range[1]), n_hfn)).astype(np.int64)
        tot = min(int(fo.sum()), x_idx.size)
        grab = rng.choice(x_idx, size=tot, replace=False)
        owner = np.repeat(np.arange(n_hfn), fo)[:tot]
        cons_drv[grab] = owner            # driver ids 0..n_hfn-1 are PIs
        hfn_fanouts = np.bincount(owner, minlength=n_hfn).tolist()
    assert (cons_drv >= 0).all()

    # ---- pin numbering: PI ports, cells in random order, PO ports ----
    cell_perm = rng.permutation(n_cells)            # position -> cell id
    # cell ids: 0..n_comb-1 comb, n_comb.. DFF
    cell_npins = np.concatenate([n_in + 1, np.full(n_dff, 3)])
    npins_in_order = cell_npins[cell_perm]
    pos_base = n_pi + np.concatenate([[0], np.cumsum(npins_in_order)[:-1]])
    cell_base = np.empty(n_cells, np.int64)
    cell_base[cell_perm] = pos_base
    P = n_pi + int(cell_npins.sum()) + n_po
    po_base = P - n_po

    pin_cap = np.zeros(P, np.float32)
    pin_role = np.zeros(P, np.uint8)
    pin_role[:n_pi] = ROLE_PI
    pin_role[po_base:] = ROLE_PO
    # comb input pins
    ci_pin = cell_base[cons_cell] + cons_j
    pin_cap[ci_pin] = in_cap[ctype[cons_cell], cons_j]
    comb_out = cell_base[:n_comb] + n_in
    dff_base = cell_base[n_comb:]
    d_pin, ck_pin, q_pin = dff_base, dff_base + 1, dff_base + 2
    pin_cap[d_pin] = d_cap
    pin_role[d_pin] = ROLE_FF_D
    pin_role[ck_pin] = ROLE_FF_CK
    po_pin = np.arange(po_base, P)

    drv_pin = np.concatenate([np.arange(n_pi), q_pin, comb_out])
    cons_pin = np.concatenate([ci_pin, d_pin, po_pin])
    sink_drv_pin = drv_pin[cons_drv]

    # ---- nets: one per driver with >= 1 sink, drivers in pin order, sinks by pin id
    o = np.lexsort((cons_pin, sink_drv_pin))
    s_drv, s_pin = sink_drv_pin[o], cons_pin[o]
    net_drv, net_first, net_k = np.unique(s_drv, return_index=True, return_counts=True)
    N = net_drv.size
    net_ptr = np.zeros(N + 1, np.int64)
    net_ptr[1:] = np.cumsum(net_k + 1)
    net_pins = np.empty(int(net_ptr[-1]), np.int64)
    net_pins[net_ptr[:-1]] = net_drv
    sink_net = np.repeat(np.arange(N), net_k)
    sink_rank = np.arange(s_pin.size) - np.repeat(net_first, net_k)
    net_pins[net_ptr[sink_net] + 1 + sink_rank] = s_pin

    # ---- cell arcs (in cell-position order) and checks ----
    arc_from = ci_pin
    arc_to = comb_out[cons_cell]
    arc_sense = np.array([s for _, ss, _ in COMB for s in ss], np.uint8)
    sense_off = np.concatenate([[0], np.cumsum(n_in_of_type)[:-1]])
    arc_sense = arc_sense[sense_off[ctype[cons_cell]] + cons_j]
    arc_tab = arc_base[ctype[cons_cell], cons_j]
    arc_from = np.concatenate([arc_from, ck_pin])
    arc_to = np.concatenate([arc_to, q_pin])
    arc_sense = np.concatenate([arc_sense, np.full(n_dff, SENSE_RISE_EDGE, np.uint8)])
    arc_tab = np.concatenate([arc_tab, np.full(n_dff, ckq_base, np.uint32)])
    ao = np.argsort(arc_to, kind="stable")
    arc_from, arc_to, arc_sense, arc_tab = arc_from[ao], arc_to[ao], arc_sense[ao], arc_tab[ao]

    # ---- RC trees: driver node 0, sinks + floor(k/2) Steiner nodes, recursive tree
    n_st = net_k // 2
    n_nodes = 1 + net_k + n_st
    rc_ptr = np.zeros(N + 1, np.int64)
    rc_ptr[1:] = np.cumsum(n_nodes)
    n_rc = int(rc_ptr[-1])
    node_pin = np.full(n_rc, NO_PIN, np.int64)
    node_pin[rc_ptr[:-1]] = net_drv
    ent_net = np.concatenate([sink_net, np.repeat(np.arange(N), n_st)])
    ent_pin = np.concatenate([s_pin, np.full(int(n_st.sum()), NO_PIN, np.int64)])
    eo = np.lexsort((rng.random(ent_net.size), ent_net))
    ent_net, ent_pin = ent_net[eo], ent_pin[eo]
    ent_first = np.searchsorted(ent_net, np.arange(N), side="left")
    ent_rank = np.arange(ent_net.size) - ent_first[ent_net]
    node_pin[rc_ptr[ent_net] + 1 + ent_rank] = ent_pin
    local = np.arange(n_rc) - np.repeat(rc_ptr[:-1], n_nodes)
    parent = np.floor(rng.random(n_rc) * local).astype(np.int64)
    parent[local == 0] = -1
    res = rng.uniform(0.02, 0.2, n_rc).astype(np.float32)
    res[local == 0] = 0.0
    cap = rng.uniform(0.1, 1.0, n_rc).astype(np.float32)
    if n_hfn > 0:
        # high-fan-out nets are routed on thick upper layers: 10x lower unit R
        hfn_net = np.nonzero(net_drv < n_hfn)[0]       # PI pins 0..n_hfn-1 drive them
        node_net = np.repeat(np.arange(N), n_nodes)
        res[np.isin(node_net, hfn_net)] *= np.float32(0.1)

    # ---- constraints ----
    pi_L = rng.uniform(0, 50, (n_pi, 2))
    pi_E = np.maximum(pi_L - rng.uniform(0, 5, (n_pi, 2)), 0)
    pi_at = np.concatenate([pi_E, pi_L], axis=1).astype(np.float32)
    sl_L = rng.uniform(5, 40, (n_pi, 2))
    sl_E = sl_L * rng.uniform(0.8, 1.0, (n_pi, 2))
    pi_slew = np.concatenate([sl_E, sl_L], axis=1).astype(np.float32)
    po_out_max = rng.uniform(0, 50, (n_po, 2)).astype(np.float32)
    po_out_min = rng.uniform(0, 10, (n_po, 2)).astype(np.float32)
    po_load = rng.uniform(1, 4, n_po).astype(np.float32)
    if period is None:
        period = lookup_period(name) or 1000.0
    cons = Constraints(float(period), 20.0, np.arange(n_pi, dtype=np.uint32), pi_at, pi_slew,
                       po_pin.astype(np.uint32), po_out_max, po_out_min, po_load)

    base_rc = RcTree(rc_ptr.astype(np.uint32), parent.astype(np.int32),
                     node_pin.astype(np.uint32), res, cap)
    libs, rcs = [], []
    for c in range(corners):
        ls, rs, cs = corner_scales(c, corner_recipe)
        libs.append(lib if ls == 1.0 else lib.scaled(ls))
        rcs.append(base_rc if (rs == 1.0 and cs == 1.0) else base_rc.scaled(rs, cs))

    return Design(
        num_pins=P, pin_cap=pin_cap, pin_role=pin_role,
        net_ptr=net_ptr.astype(np.uint32), net_pins=net_pins.astype(np.uint32),
        arc_from=arc_from.astype(np.uint32), arc_to=arc_to.astype(np.uint32),
        arc_sense=arc_sense, arc_tab=arc_tab.astype(np.uint32),
        chk_d=d_pin.astype(np.uint32), chk_ck=ck_pin.astype(np.uint32),
        chk_tab=np.full(n_dff, chk_base, np.uint32),
        libs=libs, rc=rcs, cons=cons, name=name,
        meta=dict(seed=seed, n_cells=n_cells, gate_depth=D, n_pi=n_pi, n_po=n_po,
                  n_dff=n_dff, hfn_fanouts=hfn_fanouts, corner_recipe=corner_recipe),
        logic=_logic(ctype, cell_base, n_in, comb_out, cons_cell, cons_j, ao))


def lookup_period(name: str) -> Optional[float]:
    try:
        with open(_PERIODS_FILE) as f:
            return json.load(f).get(name, {}).get("period")
    except FileNotFoundError:
        return None


def config_design(name: str, corners: Optional[int] = None, **over) -> Design:
    """Build a named config (c2_tau, c3_superblue, c4_tdp, c5_multicorner) or c17."""
    if name in ("c1_c17", "c17"):
        from .hand import c17
        return c17()
    cfg = dict(CONFIGS[name])
    if corners is not None:
        cfg["corners"] = corners
    cfg.update(over)
    return generate(name=name, **cfg)
