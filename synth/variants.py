"""Input variants of generated designs for the GPU parity tests (VERDICT r1
"Next round" item 2): table shapes and values the LIB-SYN recipe never
makes, pools larger than the shared-memory image, endpoints that also have
fan-out, per-corner libraries with different axes.

Input generation only (shapes, axes, values, roles, constraint lists): no
timing arithmetic lives here.
"""
from __future__ import annotations

import copy

import numpy as np

from .design import ROLE_FF_CK, ROLE_FF_D, ROLE_INTERNAL, ROLE_PI, ROLE_PO, Design, Library

SHAPES = [(1, 1), (1, 5), (6, 1), (2, 2), (7, 7), (8, 8), (3, 8), (8, 2)]


def _axis(rng, n, lo, hi):
    if n == 1:
        return np.array([rng.uniform(lo, hi)])
    x = np.sort(rng.uniform(lo, hi, n))
    x += np.arange(n) * 1e-3 * (hi - lo)          # strictly ascending
    return x


def random_table(rng, shape, neg_frac=0.25, slew_range=(1.0, 300.0), load_range=(0.1, 40.0)):
    """A table of the given shape with random ascending axes; values a + b s + k c
    + noise with a drawn so that about `neg_frac` of the tables dip below zero
    somewhere (cell delays / slews are then clamped by the method)."""
    n1, n2 = shape
    x = _axis(rng, n1, *slew_range)
    y = _axis(rng, n2, *load_range)
    a = rng.uniform(-12.0, 2.0) if rng.random() < neg_frac else rng.uniform(2.0, 20.0)
    b = rng.uniform(0.02, 0.3)
    k = rng.uniform(0.3, 4.0)
    v = a + b * x[:, None] + k * y[None, :] + rng.uniform(-1.0, 1.0, (n1, n2))
    return (x, y, v)


def odd_tables(d: Design, seed: int, n_pad: int = 0) -> Design:
    """Every table of every corner replaced by a random one of a random shape
    in SHAPES (1x1, 1xn, nx1, 2x2, 7x7, 8x8, ...), some with negative values;
    `n_pad` unused tables are put in FRONT of the pool (table ids shift by
    n_pad) so the used tables sit at high offsets of a large pool."""
    rng = np.random.default_rng(seed)
    T = d.libs[0].num_tables
    out = copy.copy(d)
    libs = []
    for _c in range(d.num_corners):
        tabs = [random_table(rng, SHAPES[int(rng.integers(len(SHAPES)))]) for _ in range(n_pad)]
        tabs += [random_table(rng, SHAPES[int(rng.integers(len(SHAPES)))]) for _ in range(T)]
        libs.append(Library.from_tables(tabs))
    out.libs = libs
    out.arc_tab = (d.arc_tab + np.uint32(n_pad)).astype(np.uint32)
    out.chk_tab = (d.chk_tab + np.uint32(n_pad)).astype(np.uint32)
    return out


def corner_axes_differ(d: Design, seed: int) -> Design:
    """Corner c >= 1 gets its own axes (stretched by 1 + 0.1 c, a different
    template per table for odd c), so the corners' pools differ in size."""
    rng = np.random.default_rng(seed)
    out = copy.copy(d)
    libs = [d.libs[0]]
    for c in range(1, d.num_corners):
        L = d.libs[c]
        tabs = []
        for t in range(L.num_tables):
            x, y, v = L.table(t)
            f = 1.0 + 0.1 * c
            if c % 2:
                x = x * (f + 0.01 * rng.random())
                y = y * (f + 0.01 * rng.random())
            else:
                x, y = x * f, y * f
            tabs.append((x, y, v))
        libs.append(Library.from_tables(tabs))
    out.libs = libs
    return out


def endpoints_with_fanout(d: Design, seed: int, frac: float = 0.05) -> Design:
    """Make endpoints that also have fan-out (the seed is
    combined with the fan-out-derived required time): a fraction of the net
    sinks that drive cell arcs, and a fraction of the cell-output pins that
    drive nets, become POs with their own output delays and loads."""
    rng = np.random.default_rng(seed)
    P = d.num_pins
    is_sink = np.zeros(P, bool)
    is_drv = np.zeros(P, bool)
    for n in range(d.num_nets):
        a, b = int(d.net_ptr[n]), int(d.net_ptr[n + 1])
        is_drv[d.net_pins[a]] = True
        is_sink[d.net_pins[a + 1:b]] = True
    has_fo = np.zeros(P, bool)
    has_fo[d.arc_from] = True
    has_fi = np.zeros(P, bool)
    has_fi[d.arc_to] = True
    plain = d.pin_role == ROLE_INTERNAL
    cand = np.nonzero(plain & ((is_sink & has_fo) | (is_drv & has_fi)))[0]
    pick = cand[rng.random(cand.size) < frac]
    out = copy.copy(d)
    out.pin_role = d.pin_role.copy()
    out.pin_role[pick] = ROLE_PO
    k = copy.copy(d.cons)
    n = pick.size
    k.po_pin = np.concatenate([d.cons.po_pin, pick.astype(np.uint32)])
    k.po_out_max = np.concatenate([d.cons.po_out_max, rng.uniform(0, 80, (n, 2)).astype(np.float32)])
    k.po_out_min = np.concatenate([d.cons.po_out_min, rng.uniform(-5, 10, (n, 2)).astype(np.float32)])
    k.po_load = np.concatenate([d.cons.po_load, rng.uniform(0, 3, n).astype(np.float32)])
    out.cons = k
    out.meta = dict(d.meta, po_with_fanout=int(n))
    return out
