"""ctypes front-end of the fp64 CPU oracle (oracle/sta_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package.  Shares no code with paper_2511_11660_b200/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sta_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, strict IEEE: no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sta_oracle.h"))):
        # compile to a private name, then rename: concurrent builders (the
        # ranks of a multi-process test) never load a half-written library
        tmp = f"{_LIB}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Design(C.Structure):
    _fields_ = [
        ("num_pins", C.c_uint32), ("pin_cap", C.c_void_p), ("pin_role", C.c_void_p),
        ("num_nets", C.c_uint32), ("net_ptr", C.c_void_p), ("net_pins", C.c_void_p),
        ("num_arcs", C.c_uint32), ("arc_from", C.c_void_p), ("arc_to", C.c_void_p),
        ("arc_sense", C.c_void_p), ("arc_tab", C.c_void_p),
        ("num_checks", C.c_uint32), ("chk_d", C.c_void_p), ("chk_ck", C.c_void_p),
        ("chk_tab", C.c_void_p),
        ("num_tables", C.c_uint32), ("tab_n1", C.c_void_p), ("tab_n2", C.c_void_p),
        ("tab_off", C.c_void_p), ("tab_data", C.c_void_p),
        ("rc_ptr", C.c_void_p), ("rc_parent", C.c_void_p), ("rc_node_pin", C.c_void_p),
        ("rc_res", C.c_void_p), ("rc_cap", C.c_void_p),
        ("period", C.c_double), ("clock_slew", C.c_double),
        ("n_pi", C.c_uint32), ("pi_pin", C.c_void_p), ("pi_at", C.c_void_p),
        ("pi_slew", C.c_void_p),
        ("n_po", C.c_uint32), ("po_pin", C.c_void_p), ("po_out_max", C.c_void_p),
        ("po_out_min", C.c_void_p), ("po_load", C.c_void_p),
        ("net_model", C.c_int32), ("arnoldi_q", C.c_uint32),
        ("n_exc", C.c_uint32), ("exc_kind", C.c_void_p), ("exc_value", C.c_void_p),
        ("exc_from_ptr", C.c_void_p), ("exc_from", C.c_void_p), ("exc_to_ptr", C.c_void_p),
        ("exc_to", C.c_void_p),
        ("n_clk", C.c_uint32), ("clk_period", C.c_void_p), ("pin_clk", C.c_void_p),
        ("exc_thr_ptr", C.c_void_p), ("exc_seg_ptr", C.c_void_p), ("exc_seg", C.c_void_p),
        ("n_fn", C.c_uint32), ("fn_pin", C.c_void_p), ("fn_in_ptr", C.c_void_p), ("fn_in", C.c_void_p),
        ("fn_tt", C.c_void_p), ("arc_when", C.c_void_p),
        ("n_case", C.c_uint32), ("case_pin", C.c_void_p), ("case_val", C.c_void_p),
    ]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _lib.orc_lut.restype = C.c_double
        _lib.orc_lut.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_double, C.c_double]
        _lib.orc_levelize.restype = C.c_int
        _lib.orc_levelize.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_rc.restype = None
        _lib.orc_rc.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_update.restype = C.c_int
        _lib.orc_update.argtypes = [C.c_void_p] * 5 + [C.c_void_p] * 4
        _lib.orc_paths.restype = C.c_int
        _lib.orc_paths.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_uint32, C.c_double, C.c_uint32,
                                   C.c_uint32] + [C.c_void_p] * 8
        _lib.orc_arnoldi_reduce.restype = C.c_int
        _lib.orc_arnoldi_reduce.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                            C.c_void_p, C.c_void_p]
        _lib.orc_arnoldi_delay.restype = C.c_double
        _lib.orc_arnoldi_delay.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p]
        _lib.orc_steiner.restype = C.c_uint32
        _lib.orc_steiner.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_double, C.c_double, C.c_double, C.c_double] + [C.c_void_p] * 5
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


class _Marshal:
    """Holds contiguous copies alive while the C call runs."""

    def __init__(self, d, corner: int = 0, net_model: str = "elmore", q: int = 4):
        keep = []

        def arr(x, dt):
            a = np.ascontiguousarray(np.asarray(x, dtype=dt))
            keep.append(a)
            return a

        lib_c = d.libs[corner]
        rc = d.rc[corner]
        cons = d.cons
        s = _Design()
        s.num_pins = d.num_pins
        s.pin_cap = _p(arr(d.pin_cap, np.float32))
        s.pin_role = _p(arr(d.pin_role, np.uint8))
        s.num_nets = d.num_nets
        s.net_ptr = _p(arr(d.net_ptr, np.uint32))
        s.net_pins = _p(arr(d.net_pins, np.uint32))
        s.num_arcs = d.num_arcs
        s.arc_from = _p(arr(d.arc_from, np.uint32))
        s.arc_to = _p(arr(d.arc_to, np.uint32))
        s.arc_sense = _p(arr(d.arc_sense, np.uint8))
        s.arc_tab = _p(arr(d.arc_tab, np.uint32))
        s.num_checks = d.num_checks
        s.chk_d = _p(arr(d.chk_d, np.uint32))
        s.chk_ck = _p(arr(d.chk_ck, np.uint32))
        s.chk_tab = _p(arr(d.chk_tab, np.uint32))
        s.num_tables = lib_c.num_tables
        s.tab_n1 = _p(arr(lib_c.n1, np.uint8))
        s.tab_n2 = _p(arr(lib_c.n2, np.uint8))
        s.tab_off = _p(arr(lib_c.off, np.uint32))
        s.tab_data = _p(arr(lib_c.data, np.float32))
        s.rc_ptr = _p(arr(rc.rc_ptr, np.uint32))
        s.rc_parent = _p(arr(rc.parent, np.int32))
        s.rc_node_pin = _p(arr(rc.node_pin, np.uint32))
        s.rc_res = _p(arr(rc.res, np.float32))
        s.rc_cap = _p(arr(rc.cap, np.float32))
        s.period = float(cons.period)
        s.clock_slew = float(cons.clock_slew)
        s.n_pi = int(cons.pi_pin.shape[0])
        s.pi_pin = _p(arr(cons.pi_pin, np.uint32))
        s.pi_at = _p(arr(cons.pi_at, np.float32))
        s.pi_slew = _p(arr(cons.pi_slew, np.float32))
        s.n_po = int(cons.po_pin.shape[0])
        s.po_pin = _p(arr(cons.po_pin, np.uint32))
        s.po_out_max = _p(arr(cons.po_out_max, np.float32))
        s.po_out_min = _p(arr(cons.po_out_min, np.float32))
        s.po_load = _p(arr(cons.po_load, np.float32))
        s.net_model = {"elmore": 0, "arnoldi": 1}[net_model]
        s.arnoldi_q = int(q)
        ex = getattr(d, "exceptions", None)
        s.n_exc = ex.num if ex is not None else 0
        if s.n_exc:
            s.exc_kind = _p(arr(ex.kind, np.uint8))
            s.exc_value = _p(arr(ex.value, np.float32))
            s.exc_from_ptr = _p(arr(ex.from_ptr, np.uint32))
            s.exc_from = _p(arr(ex.from_pins, np.uint32))
            s.exc_to_ptr = _p(arr(ex.to_ptr, np.uint32))
            s.exc_to = _p(arr(ex.to_pins, np.uint32))
            if ex.thr_ptr is not None and int(ex.thr_ptr[-1]) > 0:   # O15: -through segments
                s.exc_thr_ptr = _p(arr(ex.thr_ptr, np.uint32))
                s.exc_seg_ptr = _p(arr(ex.seg_ptr, np.uint32))
                s.exc_seg = _p(arr(ex.seg_pins, np.uint32))
        ck = getattr(d, "clocks", None)
        s.n_clk = int(ck.period.shape[0]) if ck is not None else 0
        if s.n_clk:
            s.clk_period = _p(arr(ck.period, np.float32))
            s.pin_clk = _p(arr(ck.pin_clk, np.uint32))
        lg = getattr(d, "logic", None)          # O16: case analysis
        cv = getattr(d, "case", None)
        if lg is not None and cv is not None and (len(cv.pin) or lg.arc_when is not None):
            s.n_fn = int(lg.fn_pin.shape[0])
            s.fn_pin = _p(arr(lg.fn_pin, np.uint32))
            s.fn_in_ptr = _p(arr(lg.fn_in_ptr, np.uint32))
            s.fn_in = _p(arr(lg.fn_in, np.uint32))
            s.fn_tt = _p(arr(lg.fn_tt, np.uint64))
            if lg.arc_when is not None:
                s.arc_when = _p(arr(lg.arc_when, np.uint64))
            s.n_case = int(len(cv.pin))
            if s.n_case:
                s.case_pin = _p(arr(cv.pin, np.uint32))
                s.case_val = _p(arr(cv.val, np.uint8))
        self.s = s
        self.keep = keep

    @property
    def ptr(self):
        return C.addressof(self.s)


def lut(n1, n2, tab, s, c) -> float:
    t = np.ascontiguousarray(np.asarray(tab, np.float32))
    return lib().orc_lut(int(n1), int(n2), t.ctypes.data, float(s), float(c))


def levelize(d):
    """-> (level[P] u32, perm[P] u32, num_levels) or raises on a cycle."""
    m = _Marshal(d)
    level = np.zeros(d.num_pins, np.uint32)
    perm = np.zeros(d.num_pins, np.uint32)
    nl = np.zeros(1, np.uint32)
    st = lib().orc_levelize(m.ptr, _p(level), _p(perm), nl.ctypes.data)
    if st == 1:
        raise ValueError("combinational cycle")
    if st:
        raise MemoryError("oracle allocation failed")
    return level, perm, int(nl[0])


def rc(d, corner: int = 0):
    """-> (load[N] f64, elm[P] f64)."""
    m = _Marshal(d, corner)
    load = np.zeros(max(d.num_nets, 1), np.float64)
    elm = np.zeros(max(d.num_pins, 1), np.float64)
    lib().orc_rc(m.ptr, _p(load), _p(elm))
    return load[:d.num_nets], elm[:d.num_pins]


def update(d, corner: int = 0, want_all: bool = True, net_model: str = "elmore", q: int = 4):
    """Full update for one corner -> dict(at, slew, rat, slack [P,4] f64,
    res[4] = (WNS_setup, TNS_setup, WNS_hold, TNS_hold), ep_pin, ep_ws).
    net_model "arnoldi": net arcs by the O12 reduced model of order q."""
    m = _Marshal(d, corner, net_model, q)
    P = d.num_pins
    at = np.zeros((max(P, 1), 4))
    slew = np.zeros((max(P, 1), 4)) if want_all else None
    rat = np.zeros((max(P, 1), 4)) if want_all else None
    slack = np.zeros((max(P, 1), 4)) if want_all else None
    res = np.zeros(4)
    n_ep_max = int(d.cons.po_pin.shape[0]) + d.num_checks + 1
    ep_pin = np.zeros(n_ep_max, np.uint32)
    ep_ws = np.zeros((n_ep_max, 2))
    n_ep = np.zeros(1, np.uint32)
    st = lib().orc_update(m.ptr, _p(at), _p(slew) if want_all else None,
                          _p(rat) if want_all else None, _p(slack) if want_all else None,
                          res.ctypes.data, _p(ep_pin), _p(ep_ws), n_ep.ctypes.data)
    if st == 1:
        raise ValueError("combinational cycle")
    if st == 5:
        raise ValueError("too many exceptions (32), segments (32) or tags (64)")
    _case_status(st)
    if st:
        raise MemoryError("oracle allocation failed")
    ne = int(n_ep[0])
    out = dict(at=at[:P], res=res, ep_pin=ep_pin[:ne], ep_ws=ep_ws[:ne], period=float(d.cons.period))
    if want_all:
        out.update(slew=slew[:P], rat=rat[:P], slack=slack[:P])
    return out


def _case_status(st):
    if st == 6:
        raise ValueError("case analysis: contradictory constants on a pin")
    if st == 7:
        raise ValueError("case analysis: a logic function with more than 6 inputs")


def case_analysis(d):
    """O16 alone -> (val[P] uint8: 0, 1, 2 = not constant, off[E] uint8 per
    canonical arc: net arcs net by net, then cell arcs)."""
    m = _Marshal(d, 0)
    E = int(d.net_ptr[-1]) - d.num_nets + d.num_arcs
    val = np.zeros(max(d.num_pins, 1), np.uint8)
    off = np.zeros(max(E, 1), np.uint8)
    lib().orc_case_analysis.restype = C.c_int
    lib().orc_case_analysis.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    st = lib().orc_case_analysis(m.ptr, val.ctypes.data, off.ctypes.data)
    _case_status(st)
    if st:
        raise MemoryError("oracle allocation failed")
    return val[:d.num_pins], off[:E]


def update_all_corners(d):
    """O9: per-corner results plus global WNS = min, TNS = sum over corners."""
    per = [update(d, c) for c in range(d.num_corners)]
    r = np.array([p["res"] for p in per])
    glob = np.array([r[:, 0].min(), r[:, 1].sum(), r[:, 2].min(), r[:, 3].sum()])
    return per, glob


def paths(d, corner: int = 0, mode: str = "setup", k: int = 10, nworst: int = 1,
          slack_lt: float = float("inf")):
    """O10 top-k path report -> list of dicts {slack, ep, pins, rfs, at}
    in report order (slack, endpoint id, backward (pin, rf) sequence)."""
    m = _Marshal(d, corner)
    P = d.num_pins
    cap_paths = int(k)
    cap_pins = int(k) * (P + 1)
    while True:
        ptr = np.zeros(cap_paths + 1, np.uint32)
        pin = np.zeros(max(cap_pins, 1), np.uint32)
        rf = np.zeros(max(cap_pins, 1), np.uint8)
        at = np.zeros(max(cap_pins, 1), np.float64)
        sl = np.zeros(max(cap_paths, 1), np.float64)
        ep = np.zeros(max(cap_paths, 1), np.uint32)
        n = np.zeros(1, np.uint32)
        npin = np.zeros(1, np.uint32)
        st = lib().orc_paths(m.ptr, 0 if mode == "setup" else 1, int(k), int(nworst), float(slack_lt),
                             cap_paths, cap_pins, n.ctypes.data, npin.ctypes.data, _p(ptr), _p(pin),
                             _p(rf), _p(at), _p(sl), _p(ep))
        if st == 3:
            cap_pins *= 2
            continue
        if st == 1:
            raise ValueError("combinational cycle")
        if st:
            raise MemoryError("oracle allocation failed")
        break
    out = []
    for i in range(int(n[0])):
        a, b = int(ptr[i]), int(ptr[i + 1])
        out.append(dict(slack=float(sl[i]), ep=int(ep[i]), pins=pin[a:b].tolist(), rfs=rf[a:b].tolist(),
                        at=at[a:b].tolist()))
    return out


def steiner(net_ptr, net_pins, x, y, res_x, res_y, cap_x, cap_y):
    """O11 Steiner RC from pin positions -> (rc_ptr, parent, node_pin, res,
    cap) in the sta_set_rc_tree / sta_set_rc_values layout."""
    net_ptr = np.ascontiguousarray(net_ptr, np.uint32)
    net_pins = np.ascontiguousarray(net_pins, np.uint32)
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    N = net_ptr.size - 1
    cap_n = max(2 * int(net_ptr[-1]) - N, 1)
    rc_ptr = np.zeros(N + 1, np.uint32)
    parent = np.zeros(cap_n, np.int32)
    node_pin = np.zeros(cap_n, np.uint32)
    res = np.zeros(cap_n, np.float32)
    cap = np.zeros(cap_n, np.float32)
    # unit values are float32 inputs (the device reads them as float)
    u = [float(np.float32(v)) for v in (res_x, res_y, cap_x, cap_y)]
    n = lib().orc_steiner(N, _p(net_ptr), _p(net_pins), _p(x), _p(y), *u, _p(rc_ptr), _p(parent),
                          _p(node_pin), _p(res), _p(cap))
    return rc_ptr, parent[:n], node_pin[:n], res[:n], cap[:n]


def arnoldi_reduce(parent, res, cap, q: int = 4):
    """O12 reduced model of one net's RC tree -> (order, lam[order],
    resid[m][q]); order -1: unstable."""
    parent = np.ascontiguousarray(parent, np.int32)
    res = np.ascontiguousarray(res, np.float32)
    cap = np.ascontiguousarray(cap, np.float64)
    m = parent.size
    lam = np.zeros(max(q, 1), np.float64)
    resid = np.zeros((max(m, 1), max(q, 1)), np.float64)
    qq = lib().orc_arnoldi_reduce(m, _p(parent), _p(res), _p(cap), int(q), _p(lam), _p(resid))
    return qq, lam[:max(qq, 0)], resid[:m]


def arnoldi_delay(lam, k, slew):
    """O12 ramp response of a reduced model -> (delay, out_slew)."""
    lam = np.ascontiguousarray(lam, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    os_ = np.zeros(1, np.float64)
    dl = lib().orc_arnoldi_delay(int(lam.size), _p(lam), _p(k), float(slew), _p(os_))
    return dl, float(os_[0])
