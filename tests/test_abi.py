"""The C ABI boundary: exports, error codes, call order, ownership."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sta.h")).read()
    return sorted(set(re.findall(r"STA_API\s+[\w\s\*]+?\b(sta_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2511_11660_b200 import build, sta
    build.build()
    L = C.CDLL(sta.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(sta.EXPORTS) == syms


def test_status_strings_without_gpu():
    from paper_2511_11660_b200 import sta
    L = sta.lib()
    assert L.sta_status_string(0) == b"STA_OK"
    assert L.sta_status_string(5) == b"STA_ERR_CYCLE"
    assert L.sta_destroy(None) == 0


def test_no_cpu_fallback_without_gpu():
    """On a machine without a CUDA device the product path fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2511_11660_b200 import sta
    with pytest.raises(sta.StaError):
        sta.Context(0, 1)


# ----------------------------------------------------------- GPU: errors
def _ctx():
    import paper_2511_11660_b200 as pkg
    return pkg, pkg.Context(0, 1)


def _load(ctx, d, **over):
    a = dict(pin_cap=d.pin_cap, pin_role=d.pin_role, net_ptr=d.net_ptr, net_pins=d.net_pins,
             arc_from=d.arc_from, arc_to=d.arc_to, arc_sense=d.arc_sense, arc_tab=d.arc_tab,
             chk_d=d.chk_d, chk_ck=d.chk_ck, chk_tab=d.chk_tab, num_tables=d.libs[0].num_tables)
    a.update(over)
    ctx.load_graph(**a)


def _expect(pkg, name, fn):
    with pytest.raises(pkg.StaError) as e:
        fn()
    assert e.value.name == name, str(e.value)
    return str(e.value)


@pytest.mark.gpu
def test_graph_validation_errors():
    pkg, ctx = _ctx()
    d = synth.c17()
    np_ = d.net_ptr.copy()
    np_[3], np_[4] = np_[4], np_[3]
    msg = _expect(pkg, "STA_ERR_CSR", lambda: _load(ctx, d, net_ptr=np_))
    assert "net" in msg
    bad = d.net_pins.copy()
    bad[2] = 9999
    _expect(pkg, "STA_ERR_ID", lambda: _load(ctx, d, net_pins=bad))
    two = d.net_pins.copy()
    two[2] = two[1]              # same pin twice
    _expect(pkg, "STA_ERR_MULTIDRIVER", lambda: _load(ctx, d, net_pins=two))
    sense = d.arc_sense.copy()
    sense[0] = 9
    _expect(pkg, "STA_ERR_ARG", lambda: _load(ctx, d, arc_sense=sense))
    tab = d.arc_tab.copy()
    tab[0] = 10**6
    _expect(pkg, "STA_ERR_ID", lambda: _load(ctx, d, arc_tab=tab))
    # cell arc into a net sink -> multi-driven pin
    _expect(pkg, "STA_ERR_MULTIDRIVER",
            lambda: _load(ctx, d, arc_to=np.where(np.arange(d.num_arcs) == 0, d.net_pins[1], d.arc_to)))
    # cycle: feed an output back into the first gate's input through a cell arc
    af = np.concatenate([d.arc_from, [d.arc_to[-1]]])
    at = np.concatenate([d.arc_to, [d.arc_from[0]]])
    # arc_from[0] is a net sink, so instead loop two gate outputs
    pid = {n: i for i, n in enumerate(d.meta["pin_names"])}
    af = np.concatenate([d.arc_from, [pid["N22/Y"]]]).astype(np.uint32)
    at = np.concatenate([d.arc_to, [pid["N10/Y"]]]).astype(np.uint32)
    _expect(pkg, "STA_ERR_CYCLE", lambda: _load(ctx, d, arc_from=af, arc_to=at,
                                                 arc_sense=np.append(d.arc_sense, 0),
                                                 arc_tab=np.append(d.arc_tab, 0)))
    role = d.pin_role.copy()
    role[pid["N10/A"]] = synth.ROLE_PI     # a PI with fan-in
    _expect(pkg, "STA_ERR_ARG", lambda: _load(ctx, d, pin_role=role))
    # the ctx still works after errors
    _load(ctx, d)
    ctx.close()


@pytest.mark.gpu
def test_library_rc_constraint_errors_and_order():
    pkg, ctx = _ctx()
    d = synth.c17()
    _expect(pkg, "STA_ERR_ORDER", lambda: ctx.update_timing())
    _load(ctx, d)
    L = d.libs[0]
    data = L.data.copy()
    data[1] = data[0]            # index_1 not strictly ascending
    _expect(pkg, "STA_ERR_LUT", lambda: ctx.set_library(0, L.n1, L.n2, L.off, data))
    n1 = L.n1.copy()
    n1[0] = 9
    _expect(pkg, "STA_ERR_LUT", lambda: ctx.set_library(0, n1, L.n2, L.off, L.data))
    _expect(pkg, "STA_ERR_ORDER", lambda: ctx.set_rc_values(0, d.rc[0].res, d.rc[0].cap))
    rc = d.rc[0]
    par = rc.parent.copy()
    par[1] = 1                   # parent not < i
    _expect(pkg, "STA_ERR_RC", lambda: ctx.set_rc_tree(rc.rc_ptr, par, rc.node_pin))
    npin = rc.node_pin.copy()
    npin[1] = 0                  # maps a pin of another net
    _expect(pkg, "STA_ERR_RC", lambda: ctx.set_rc_tree(rc.rc_ptr, rc.parent, npin))
    ctx.set_rc_tree(rc.rc_ptr, rc.parent, rc.node_pin)
    k = d.cons
    _expect(pkg, "STA_ERR_ARG", lambda: ctx.set_constraints(-1, k.clock_slew, k.pi_pin, k.pi_at, k.pi_slew,
                                                            k.po_pin, k.po_out_max, k.po_out_min, k.po_load))
    _expect(pkg, "STA_ERR_ARG", lambda: ctx.set_constraints(k.period, k.clock_slew, k.po_pin, k.pi_at[:2],
                                                            k.pi_slew[:2], k.po_pin, k.po_out_max,
                                                            k.po_out_min, k.po_load))
    _expect(pkg, "STA_ERR_ORDER", lambda: ctx.update_timing())
    ctx.set_library(0, L.n1, L.n2, L.off, L.data)
    ctx.set_rc_values(0, rc.res, rc.cap)
    ctx.set_constraints(k.period, k.clock_slew, k.pi_pin, k.pi_at, k.pi_slew, k.po_pin, k.po_out_max,
                        k.po_out_min, k.po_load)
    ctx.update_timing()
    res4, _ = ctx.report_slack()
    assert res4[0] == pytest.approx(-4.053684, abs=1e-3)
    # host RC values are validated on the device (no host pass over 10^7
    # values per optimization step): a negative R surfaces at the next sync
    res = rc.res.copy()
    res[1] = -1
    ctx.set_rc_values(0, res, rc.cap)
    ctx.update_timing()
    _expect(pkg, "STA_ERR_RC", lambda: ctx.synchronize())
    ctx.set_rc_values(0, rc.res, rc.cap)
    ctx.update_timing()
    assert ctx.report_slack()[0][0] == pytest.approx(-4.053684, abs=1e-3)
    ctx.close()


@pytest.mark.gpu
def test_borrowed_device_rc_bad_value_detected():
    import torch
    pkg, ctx = _ctx()
    d = synth.c17()
    pkg.load_design(ctx, d)
    r = torch.from_numpy(d.rc[0].res.copy()).cuda()
    c = torch.from_numpy(d.rc[0].cap.copy()).cuda()
    c[3] = float("nan")
    ctx.set_rc_values(0, r, c)
    ctx.update_timing()
    with pytest.raises(pkg.StaError) as e:
        ctx.report_slack()
    assert e.value.name == "STA_ERR_RC"
    ctx.close()


@pytest.mark.gpu
def test_degenerate_designs():
    """Empty design, design without endpoints, isolated pins, lumped nets."""
    import oracle
    from synth.hand import Builder
    from synth.design import constant_table, empty_constraints, ROLE_PI
    pkg, ctx = _ctx()
    # empty
    b = Builder()
    b.table(constant_table(1.0))
    d = b.build(empty_constraints())
    pkg.load_design(ctx, d)
    ctx.update_timing()
    res, _ = ctx.report_slack()
    assert res[0] == np.inf and res[1] == 0 and res[2] == np.inf and res[3] == 0
    # no endpoints, isolated pin, lumped net
    b = Builder()
    b.pin("a", 0.0, ROLE_PI)
    b.pin("s", 1.0)
    b.pin("iso", 0.0)
    b.net("a", ["s"], None)
    b.table(constant_table(1.0))
    d = b.build(empty_constraints())
    pkg.load_design(ctx, d)
    ctx.update_timing()
    res, sl = ctx.report_slack(want_pins=True)
    ref = oracle.update(d)
    assert res[0] == np.inf
    assert np.array_equal(sl, ref["slack"].astype(np.float32))
    at, slew, rat = ctx.get_timing()
    assert np.array_equal(at, ref["at"].astype(np.float32))
    ctx.close()
