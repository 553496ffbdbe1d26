"""Thin ctypes binding of include/sta.h (argument marshalling only).

Every function here forwards to the same-named C entry point of libsta.so;
no step of the timing update runs in Python.  Arrays may be numpy (host) or
torch CUDA tensors (device, zero-copy: their data_ptr() is passed with
STA_MEM_DEVICE).  There is no CPU fallback: if libsta.so is missing or no
CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# STA_LIB_PATH selects a tuning variant built by `build.py --out` (experiments only)
LIB_PATH = os.environ.get("STA_LIB_PATH") or os.path.join(_HERE, "lib", "libsta.so")

STA_MEM_HOST, STA_MEM_DEVICE = 0, 1
STATUS = ["STA_OK", "STA_ERR_ARG", "STA_ERR_CSR", "STA_ERR_ID", "STA_ERR_MULTIDRIVER",
          "STA_ERR_CYCLE", "STA_ERR_LUT", "STA_ERR_RC", "STA_ERR_ORDER", "STA_ERR_CUDA",
          "STA_ERR_OOM"]
NUM_PHASES = 5
PHASES = ["rc", "forward", "backward", "reduce", "update"]

EXPORTS = ["sta_create", "sta_destroy", "sta_last_error", "sta_status_string", "sta_load_graph",
           "sta_set_library", "sta_set_rc_tree", "sta_set_rc_values", "sta_set_constraints",
           "sta_update_timing", "sta_report_slack", "sta_get_timing", "sta_get_rc",
           "sta_get_levels", "sta_get_info", "sta_synchronize", "sta_profile_enable",
           "sta_profile_read", "sta_report_paths", "sta_build_steiner", "sta_set_net_model",
           "sta_set_exceptions", "sta_set_clocks", "sta_set_case_analysis"]


class StaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else f"status {status}"
        super().__init__(f"{self.name}: {msg}")


class GraphDesc(C.Structure):
    _fields_ = [("mem", C.c_int), ("num_pins", C.c_uint32), ("pin_cap", C.c_void_p),
                ("pin_role", C.c_void_p), ("num_nets", C.c_uint32), ("net_ptr", C.c_void_p),
                ("net_pins", C.c_void_p), ("num_arcs", C.c_uint32), ("arc_from", C.c_void_p),
                ("arc_to", C.c_void_p), ("arc_sense", C.c_void_p), ("arc_tab", C.c_void_p),
                ("num_checks", C.c_uint32), ("chk_d", C.c_void_p), ("chk_ck", C.c_void_p),
                ("chk_tab", C.c_void_p), ("num_tables", C.c_uint32)]


class ConstraintsDesc(C.Structure):
    _fields_ = [("mem", C.c_int), ("period_ps", C.c_float), ("clock_slew_ps", C.c_float),
                ("n_pi", C.c_uint32), ("pi_pin", C.c_void_p), ("pi_at", C.c_void_p),
                ("pi_slew", C.c_void_p), ("n_po", C.c_uint32), ("po_pin", C.c_void_p),
                ("po_out_max", C.c_void_p), ("po_out_min", C.c_void_p),
                ("po_load_ff", C.c_void_p)]


class Info(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "num_pins", "num_nets", "num_net_arcs", "num_cell_arcs", "num_checks", "num_endpoints",
        "num_levels", "num_stages", "num_pull_pins", "num_sink_pins", "num_heavy_drivers",
        "kernels_per_update", "lut_smem_bytes")] + [("device_bytes", C.c_uint64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class PathQuery(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("k", C.c_uint32), ("nworst", C.c_uint32), ("slack_lt", C.c_float)]


class PathSet(C.Structure):
    _fields_ = [("cap_paths", C.c_uint32), ("cap_pins", C.c_uint32), ("n_paths", C.c_uint32),
                ("n_pins", C.c_uint32), ("path_ptr", C.c_void_p), ("path_pin", C.c_void_p),
                ("path_rf", C.c_void_p), ("path_at", C.c_void_p), ("path_slack", C.c_void_p),
                ("path_ep", C.c_void_p)]


class CaseDesc(C.Structure):
    _fields_ = [("mem", C.c_int), ("num_fn", C.c_uint32), ("fn_pin", C.c_void_p), ("fn_in_ptr", C.c_void_p),
                ("fn_in", C.c_void_p), ("fn_tt", C.c_void_p), ("arc_when", C.c_void_p),
                ("num_case", C.c_uint32), ("case_pin", C.c_void_p), ("case_val", C.c_void_p)]


class ExceptionsDesc(C.Structure):
    _fields_ = [("mem", C.c_int), ("num", C.c_uint32), ("kind", C.c_void_p), ("value", C.c_void_p),
                ("from_ptr", C.c_void_p), ("from_pins", C.c_void_p), ("to_ptr", C.c_void_p),
                ("to_pins", C.c_void_p), ("thr_ptr", C.c_void_p), ("seg_ptr", C.c_void_p),
                ("seg_pins", C.c_void_p)]


class ClocksDesc(C.Structure):
    _fields_ = [("mem", C.c_int), ("num_clocks", C.c_uint32), ("period_ps", C.c_void_p), ("pin_clk", C.c_void_p)]


class SteinerUnits(C.Structure):
    _fields_ = [("res_x", C.c_float), ("res_y", C.c_float), ("cap_x", C.c_float), ("cap_y", C.c_float)]


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * NUM_PHASES), ("launches", C.c_uint32 * NUM_PHASES),
                ("updates", C.c_uint32)]


_lib = None


def lib():
    """Load libsta.so (built by paper_2511_11660_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u32, i32 = C.c_void_p, C.c_uint32, C.c_int
        sig = {
            "sta_create": (i32, [i32, u32, vp, C.POINTER(vp)]),
            "sta_destroy": (i32, [vp]),
            "sta_last_error": (C.c_char_p, [vp]),
            "sta_status_string": (C.c_char_p, [i32]),
            "sta_load_graph": (i32, [vp, C.POINTER(GraphDesc)]),
            "sta_set_library": (i32, [vp, u32, i32, u32, vp, vp, vp, vp, u32]),
            "sta_set_rc_tree": (i32, [vp, i32, vp, u32, vp, vp]),
            "sta_set_rc_values": (i32, [vp, u32, i32, vp, vp]),
            "sta_set_constraints": (i32, [vp, C.POINTER(ConstraintsDesc)]),
            "sta_update_timing": (i32, [vp]),
            "sta_report_slack": (i32, [vp, u32, vp, vp, i32]),
            "sta_get_timing": (i32, [vp, u32, vp, vp, vp, i32]),
            "sta_get_rc": (i32, [vp, u32, vp, vp, i32]),
            "sta_get_levels": (i32, [vp, vp, vp, vp, i32]),
            "sta_get_info": (i32, [vp, C.POINTER(Info)]),
            "sta_synchronize": (i32, [vp]),
            "sta_profile_enable": (i32, [vp, i32]),
            "sta_profile_read": (i32, [vp, C.POINTER(Profile)]),
            "sta_report_paths": (i32, [vp, u32, C.POINTER(PathQuery), C.POINTER(PathSet), i32]),
            "sta_build_steiner": (i32, [vp, i32, vp, vp, C.POINTER(SteinerUnits), u32, vp, vp, vp, vp, vp,
                                        C.POINTER(u32)]),
            "sta_set_net_model": (i32, [vp, i32, u32]),
            "sta_set_exceptions": (i32, [vp, C.POINTER(ExceptionsDesc)]),
            "sta_set_clocks": (i32, [vp, C.POINTER(ClocksDesc)]),
            "sta_set_case_analysis": (i32, [vp, C.POINTER(CaseDesc)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and hasattr(x, "data_ptr") and bool(x.is_cuda)


def _torch_dtypes(dtype):
    """torch dtypes whose bytes are the C type `dtype` (u32 arrays may come as int32)."""
    import torch
    return {np.float32: (torch.float32,), np.int32: (torch.int32,), np.uint8: (torch.uint8,),
            np.uint32: tuple(t for t in (getattr(torch, "uint32", None), torch.int32) if t is not None),
            np.float64: (torch.float64,),
            np.uint64: tuple(t for t in (getattr(torch, "uint64", None), torch.int64) if t is not None)}[np.dtype(dtype).type]


class _Args:
    """Marshals a group of arrays that must share one memory kind.  Device
    tensors are passed zero-copy, so they must already have the C element
    type, be contiguous and live on the ctx's device (no silent conversion:
    a converted copy would be made on torch's current stream, not the ctx's)."""

    def __init__(self, device: Optional[int] = None):
        self.keep = []
        self.mem = None
        self.device = device

    def ptr(self, x, dtype):
        if x is None:
            return None
        if _is_torch_cuda(x):
            self._kind(STA_MEM_DEVICE)
            if x.dtype not in _torch_dtypes(dtype):
                raise TypeError(f"device tensor of dtype {x.dtype} where {np.dtype(dtype).name} is expected")
            if not x.is_contiguous():
                raise ValueError("device tensors must be contiguous")
            if self.device is not None and x.device.index != self.device:
                raise ValueError(f"device tensor on cuda:{x.device.index}, ctx is on cuda:{self.device}")
            self.keep.append(x)
            return x.data_ptr() if x.numel() else None
        self._kind(STA_MEM_HOST)
        a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
        self.keep.append(a)
        return a.ctypes.data if a.size else None

    def _kind(self, k):
        if self.mem is None:
            self.mem = k
        elif self.mem != k:
            raise ValueError("mixing host and device arrays in one call")

    @property
    def kind(self):
        return STA_MEM_HOST if self.mem is None else self.mem


class Context:
    """One sta_ctx: a design loaded on one GPU for `num_corners` corners."""

    def __init__(self, device: int = 0, num_corners: int = 1, stream: Optional[int] = None):
        self._L = lib()
        h = C.c_void_p()
        st = self._L.sta_create(int(device), int(num_corners), stream, C.byref(h))
        if st:
            raise StaError(st, "sta_create failed (no CUDA device?)")
        self.h = h
        self.device = int(device)
        self.num_corners = num_corners
        self.num_pins = 0
        self.num_nets = 0
        self._net_pins_total = 0

    def close(self):
        if getattr(self, "h", None):
            self._L.sta_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st):
        if st:
            raise StaError(st, self._L.sta_last_error(self.h).decode())

    # ------------------------------------------------------------ inputs
    def load_graph(self, pin_cap, pin_role, net_ptr, net_pins, arc_from, arc_to, arc_sense,
                   arc_tab, chk_d, chk_ck, chk_tab, num_tables: int):
        a = _Args(self.device)
        d = GraphDesc()
        d.num_pins = len(pin_cap)
        d.pin_cap = a.ptr(pin_cap, np.float32)
        d.pin_role = a.ptr(pin_role, np.uint8)
        d.num_nets = max(len(net_ptr) - 1, 0)
        d.net_ptr = a.ptr(net_ptr, np.uint32)
        d.net_pins = a.ptr(net_pins, np.uint32)
        d.num_arcs = len(arc_from)
        d.arc_from = a.ptr(arc_from, np.uint32)
        d.arc_to = a.ptr(arc_to, np.uint32)
        d.arc_sense = a.ptr(arc_sense, np.uint8)
        d.arc_tab = a.ptr(arc_tab, np.uint32)
        d.num_checks = len(chk_d)
        d.chk_d = a.ptr(chk_d, np.uint32)
        d.chk_ck = a.ptr(chk_ck, np.uint32)
        d.chk_tab = a.ptr(chk_tab, np.uint32)
        d.num_tables = int(num_tables)
        d.mem = a.kind
        self._check(self._L.sta_load_graph(self.h, C.byref(d)))
        self.num_pins, self.num_nets = d.num_pins, d.num_nets
        self._net_pins_total = len(net_pins)

    def set_library(self, corner: int, n1, n2, off, data):
        a = _Args(self.device)
        p = [a.ptr(n1, np.uint8), a.ptr(n2, np.uint8), a.ptr(off, np.uint32), a.ptr(data, np.float32)]
        self._check(self._L.sta_set_library(self.h, int(corner), a.kind, len(n1), *p, len(data)))

    def set_rc_tree(self, rc_ptr, parent, node_pin):
        a = _Args(self.device)
        p = [a.ptr(rc_ptr, np.uint32), None, a.ptr(parent, np.int32), a.ptr(node_pin, np.uint32)]
        self._check(self._L.sta_set_rc_tree(self.h, a.kind, p[0], len(parent), p[2], p[3]))

    def set_rc_values(self, corner: int, res, cap):
        """Device tensors are BORROWED until the next update completes."""
        a = _Args(self.device)
        pr, pc = a.ptr(res, np.float32), a.ptr(cap, np.float32)
        self._borrowed = getattr(self, "_borrowed", {})
        self._borrowed[corner] = a.keep       # keep torch tensors alive
        self._check(self._L.sta_set_rc_values(self.h, int(corner), a.kind, pr, pc))

    def set_constraints(self, period, clock_slew, pi_pin, pi_at, pi_slew, po_pin, po_out_max,
                        po_out_min, po_load):
        a = _Args(self.device)
        k = ConstraintsDesc()
        k.period_ps = float(period)
        k.clock_slew_ps = float(clock_slew)
        k.n_pi = len(pi_pin)
        k.pi_pin = a.ptr(pi_pin, np.uint32)
        k.pi_at = a.ptr(pi_at, np.float32)
        k.pi_slew = a.ptr(pi_slew, np.float32)
        k.n_po = len(po_pin)
        k.po_pin = a.ptr(po_pin, np.uint32)
        k.po_out_max = a.ptr(po_out_max, np.float32)
        k.po_out_min = a.ptr(po_out_min, np.float32)
        k.po_load_ff = a.ptr(po_load, np.float32)
        k.mem = a.kind
        self._check(self._L.sta_set_constraints(self.h, C.byref(k)))

    def build_steiner(self, x, y, res_x: float, res_y: float, cap_x: float, cap_y: float,
                      net_pins_total: Optional[int] = None):
        """Steiner RC from pin positions (sta_build_steiner).  Host positions
        -> numpy arrays; torch CUDA positions -> torch CUDA tensors (device
        outputs, ready for set_rc_tree / set_rc_values).  Returns
        (rc_ptr, parent, node_pin, res, cap) trimmed to the node count."""
        N = self.num_nets
        nnp = int(net_pins_total) if net_pins_total is not None else self._net_pins_total
        capn = max(2 * nnp - N, 1)
        u = SteinerUnits(float(res_x), float(res_y), float(cap_x), float(cap_y))
        nn = C.c_uint32()
        a = _Args(self.device)
        px, py = a.ptr(x, np.float32), a.ptr(y, np.float32)
        if a.kind == STA_MEM_DEVICE:
            import torch
            dev = x.device
            rc_ptr = torch.empty(N + 1, dtype=torch.int32, device=dev)
            outs = [torch.empty(capn, dtype=t, device=dev)
                    for t in (torch.int32, torch.int32, torch.float32, torch.float32)]
            ptrs = [rc_ptr.data_ptr()] + [o.data_ptr() for o in outs]
        else:
            rc_ptr = np.zeros(N + 1, np.uint32)
            outs = [np.zeros(capn, np.int32), np.zeros(capn, np.uint32), np.zeros(capn, np.float32),
                    np.zeros(capn, np.float32)]
            ptrs = [rc_ptr.ctypes.data] + [o.ctypes.data for o in outs]
        self._check(self._L.sta_build_steiner(self.h, a.kind, px, py, C.byref(u), capn, *ptrs, C.byref(nn)))
        n = nn.value
        return (rc_ptr,) + tuple(o[:n] for o in outs)

    def set_exceptions(self, kind=(), value=(), from_ptr=(0,), from_pins=(), to_ptr=(0,), to_pins=(),
                       thr_ptr=None, seg_ptr=(0,), seg_pins=()):
        """Timing exceptions (sta_set_exceptions): -from / -to lists and, with
        thr_ptr, ordered -through segments; no arguments clear them."""
        a = _Args(self.device)
        e = ExceptionsDesc()
        e.num = len(kind)
        e.kind = a.ptr(kind, np.uint8)
        e.value = a.ptr(value, np.float32)
        e.from_ptr = a.ptr(from_ptr, np.uint32)
        e.from_pins = a.ptr(from_pins, np.uint32)
        e.to_ptr = a.ptr(to_ptr, np.uint32)
        e.to_pins = a.ptr(to_pins, np.uint32)
        if thr_ptr is not None:
            e.thr_ptr = a.ptr(thr_ptr, np.uint32)
            e.seg_ptr = a.ptr(seg_ptr, np.uint32)
            e.seg_pins = a.ptr(seg_pins, np.uint32)
        e.mem = a.kind
        self._check(self._L.sta_set_exceptions(self.h, C.byref(e)))

    def set_case_analysis(self, fn_pin=(), fn_in_ptr=(0,), fn_in=(), fn_tt=(), arc_when=None,
                          case_pin=(), case_val=()):
        """Case analysis (sta_set_case_analysis): logic functions, optional
        when guards, constants; no arguments clear."""
        a = _Args(self.device)
        k = CaseDesc()
        k.num_fn = len(fn_pin)
        k.fn_pin = a.ptr(fn_pin, np.uint32)
        k.fn_in_ptr = a.ptr(fn_in_ptr, np.uint32) if k.num_fn else None
        k.fn_in = a.ptr(fn_in, np.uint32)
        k.fn_tt = a.ptr(fn_tt, np.uint64)
        k.arc_when = a.ptr(arc_when, np.uint64) if arc_when is not None else None
        k.num_case = len(case_pin)
        k.case_pin = a.ptr(case_pin, np.uint32)
        k.case_val = a.ptr(case_val, np.uint8)
        k.mem = a.kind
        self._check(self._L.sta_set_case_analysis(self.h, C.byref(k)))

    def set_clocks(self, period_ps=(), pin_clk=None):
        """Multiple ideal clocks (sta_set_clocks); no arguments: one clock."""
        a = _Args(self.device)
        k = ClocksDesc()
        k.num_clocks = len(period_ps)
        k.period_ps = a.ptr(period_ps, np.float32)
        k.pin_clk = a.ptr(pin_clk, np.uint32) if k.num_clocks else None
        k.mem = a.kind
        self._check(self._L.sta_set_clocks(self.h, C.byref(k)))

    def set_net_model(self, model: str = "elmore", q: int = 4):
        """Net-arc delay model of the next updates: "elmore" or "arnoldi"
        (reduced order q in 1..4)."""
        self._check(self._L.sta_set_net_model(self.h, {"elmore": 0, "arnoldi": 1}[model], int(q)))

    # ------------------------------------------------------------ update
    def update_timing(self):
        self._check(self._L.sta_update_timing(self.h))

    def synchronize(self):
        self._check(self._L.sta_synchronize(self.h))

    # ----------------------------------------------------------- reports
    def report_slack(self, corner: int = 0, pin_slack=None, want_pins: bool = False):
        """-> (res4 numpy f64 [WNS_s, TNS_s, WNS_h, TNS_h], pin slack or None).
        pin_slack: optional torch CUDA tensor [P,4] f32 to fill (device);
        want_pins: return a host numpy [P,4] array instead."""
        if pin_slack is not None:
            # device outputs: res4 is returned as a torch float64 CUDA tensor
            import torch
            res_d = torch.empty(4, dtype=torch.float64, device=pin_slack.device)
            self._check(self._L.sta_report_slack(self.h, corner, res_d.data_ptr(),
                                                 pin_slack.data_ptr(), STA_MEM_DEVICE))
            return res_d, pin_slack
        res = np.zeros(4, np.float64)
        out = np.zeros((self.num_pins, 4), np.float32) if want_pins else None
        self._check(self._L.sta_report_slack(self.h, corner, res.ctypes.data,
                                             out.ctypes.data if want_pins and out.size else None,
                                             STA_MEM_HOST))
        return res, out

    def report_wns_tns_device(self, corner: int, out):
        """Stream-ordered copy of {WNS_s, TNS_s, WNS_h, TNS_h} into a float64 CUDA tensor view."""
        self._check(self._L.sta_report_slack(self.h, corner, out.data_ptr(), None, STA_MEM_DEVICE))

    def get_timing(self, corner: int = 0):
        P = self.num_pins
        at, slew, rat = (np.zeros((P, 4), np.float32) for _ in range(3))
        if P:
            self._check(self._L.sta_get_timing(self.h, corner, at.ctypes.data, slew.ctypes.data,
                                               rat.ctypes.data, STA_MEM_HOST))
        return at, slew, rat

    def get_rc(self, corner: int = 0):
        load = np.zeros(self.num_nets, np.float32)
        elm = np.zeros(self.num_pins, np.float32)
        self._check(self._L.sta_get_rc(self.h, corner, load.ctypes.data if load.size else None,
                                       elm.ctypes.data if elm.size else None, STA_MEM_HOST))
        return load, elm

    def get_levels(self):
        P = self.num_pins
        level = np.zeros(P, np.uint32)
        perm = np.zeros(P, np.uint32)
        nl = C.c_uint32()
        self._check(self._L.sta_get_levels(self.h, level.ctypes.data if P else None,
                                           perm.ctypes.data if P else None, C.byref(nl),
                                           STA_MEM_HOST))
        return level, perm, nl.value

    def report_paths(self, corner: int = 0, mode: str = "setup", k: int = 10, nworst: int = 1,
                     slack_lt: float = float("inf")):
        """Top-k path report (sta_report_paths) -> list of dicts {slack, ep,
        pins, rfs, at} in report order (host arrays)."""
        q = PathQuery(0 if mode == "setup" else 1, int(k), int(nworst), float(slack_lt))
        info = self.info()
        cap_paths = int(k)
        cap_pins = int(k) * (info["num_levels"] + 1)
        while True:
            ptr = np.zeros(cap_paths + 1, np.uint32)
            pin = np.zeros(max(cap_pins, 1), np.uint32)
            rf = np.zeros(max(cap_pins, 1), np.uint8)
            at = np.zeros(max(cap_pins, 1), np.float32)
            sl = np.zeros(max(cap_paths, 1), np.float32)
            ep = np.zeros(max(cap_paths, 1), np.uint32)
            o = PathSet(cap_paths, cap_pins, 0, 0, ptr.ctypes.data, pin.ctypes.data, rf.ctypes.data,
                        at.ctypes.data, sl.ctypes.data, ep.ctypes.data)
            st = self._L.sta_report_paths(self.h, int(corner), C.byref(q), C.byref(o), STA_MEM_HOST)
            if st == 1 and o.n_pins > cap_pins:
                cap_pins = int(o.n_pins)
                continue
            self._check(st)
            break
        out = []
        for i in range(o.n_paths):
            a, b = int(ptr[i]), int(ptr[i + 1])
            out.append(dict(slack=float(sl[i]), ep=int(ep[i]), pins=pin[a:b].tolist(), rfs=rf[a:b].tolist(),
                            at=at[a:b].tolist()))
        return out

    def info(self) -> dict:
        i = Info()
        self._check(self._L.sta_get_info(self.h, C.byref(i)))
        return i.as_dict()

    def profile_enable(self, on: bool = True):
        self._check(self._L.sta_profile_enable(self.h, 1 if on else 0))

    def profile_read(self) -> dict:
        p = Profile()
        self._check(self._L.sta_profile_read(self.h, C.byref(p)))
        return dict(ms={PHASES[i]: p.ms[i] for i in range(NUM_PHASES)},
                    launches={PHASES[i]: p.launches[i] for i in range(NUM_PHASES)},
                    updates=p.updates)


# ---------------------------------------------------------------- helpers
def _dev(x):
    """numpy array -> torch CUDA tensor of the same bytes (u32 as int32)."""
    import torch
    a = np.ascontiguousarray(x)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def load_design(ctx: Context, d, corners=None, device_rc: bool = False, device_graph: bool = False):
    """Load a synth.Design (netlist, libraries, RC, constraints) into ctx.
    corners: which design corners map to ctx corners 0..K-1 (default all);
    device_rc / device_graph: pass the RC values / the netlist, RC tree,
    libraries and constraints as device tensors (STA_MEM_DEVICE)."""
    g = _dev if device_graph else (lambda x: x)
    ctx.load_graph(g(d.pin_cap), g(d.pin_role), g(d.net_ptr), g(d.net_pins), g(d.arc_from),
                   g(d.arc_to), g(d.arc_sense), g(d.arc_tab), g(d.chk_d), g(d.chk_ck), g(d.chk_tab),
                   d.libs[0].num_tables)
    corners = list(range(ctx.num_corners)) if corners is None else list(corners)
    for k, c in enumerate(corners):
        L = d.libs[c]
        ctx.set_library(k, g(L.n1), g(L.n2), g(L.off), g(L.data))
    rc0 = d.rc[corners[0]]
    ctx.set_rc_tree(g(rc0.rc_ptr), g(rc0.parent), g(rc0.node_pin))
    for k, c in enumerate(corners):
        rc = d.rc[c]
        if device_rc:
            import torch
            ctx.set_rc_values(k, torch.from_numpy(rc.res).cuda(), torch.from_numpy(rc.cap).cuda())
        else:
            ctx.set_rc_values(k, rc.res, rc.cap)
    k = d.cons
    ctx.set_constraints(k.period, k.clock_slew, g(k.pi_pin), g(k.pi_at), g(k.pi_slew), g(k.po_pin),
                        g(k.po_out_max), g(k.po_out_min), g(k.po_load))
    ck = getattr(d, "clocks", None)
    if ck is not None and len(ck.period):
        ctx.set_clocks(ck.period, ck.pin_clk)
    lg, cv = getattr(d, "logic", None), getattr(d, "case", None)
    if lg is not None and cv is not None:
        ctx.set_case_analysis(lg.fn_pin, lg.fn_in_ptr, lg.fn_in, lg.fn_tt, lg.arc_when, cv.pin, cv.val)
    ex = getattr(d, "exceptions", None)
    if ex is not None and ex.num:
        if getattr(ex, "has_through", False):
            ctx.set_exceptions(ex.kind, ex.value, ex.from_ptr, ex.from_pins, ex.to_ptr, ex.to_pins,
                               ex.thr_ptr, ex.seg_ptr, ex.seg_pins)
        else:
            ctx.set_exceptions(ex.kind, ex.value, ex.from_ptr, ex.from_pins, ex.to_ptr, ex.to_pins)
