"""GPU parity of case analysis (sta_set_case_analysis)
against the oracle's O16: every pin's arrival / slew / required time /
slack and WNS / TNS element by element with constants on sinks, cell
outputs and startpoints, MUX select pins (when guards), with Arnoldi and 2
corners, together with -from / -through / -to exceptions and 2 clocks, the
top-k path report, repeated updates, clearing and argument errors.

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import copy

import numpy as np
import pytest

import oracle
import synth
from synth.design import CaseValues
from tests.parity import compare_update
from tests.test_gpu_paths import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sta():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 (there is no CPU fallback)")
    import paper_2511_11660_b200 as pkg
    return pkg


def run(sta, d, corners=1, model="elmore"):
    ctx = sta.Context(0, corners)
    sta.load_design(ctx, d)
    if model != "elmore":
        ctx.set_net_model(model, 4)
    ctx.update_timing()
    return ctx


def _sinks(d):
    return sorted(set(int(p) for n in range(d.num_nets)
                      for p in d.net_pins[int(d.net_ptr[n]) + 1:int(d.net_ptr[n + 1])]))


def _with_case(d, pins, vals):
    d2 = copy.copy(d)
    d2.case = CaseValues(np.array(pins, np.uint32), np.array(vals, np.uint8))
    return d2


def _consistent_case(d, rng, pool, n):
    """n random constants from pool that the oracle accepts (no contradiction)"""
    for _ in range(50):
        pins = list(rng.choice(pool, size=n, replace=False))
        vals = list(rng.integers(0, 2, n))
        dc = _with_case(d, pins, vals)
        try:
            val, off = oracle.case_analysis(dc)
        except ValueError:
            continue
        return dc, val, off
    raise AssertionError("no consistent constants found")


@pytest.mark.parametrize("where", ["any", "sinks", "outputs", "startpoints"])
def test_case_random(sta, where):
    d = synth.generate(3000, 20, seed=400, period=400.0)
    rng = np.random.default_rng({"any": 1, "sinks": 2, "outputs": 3, "startpoints": 4}[where])
    pool = {"any": list(range(d.num_pins)), "sinks": _sinks(d), "outputs": [int(p) for p in d.logic.fn_pin],
            "startpoints": [int(p) for p in d.cons.pi_pin]}[where]
    dc, val, off = _consistent_case(d, rng, pool, min(40, len(pool)))
    assert off.sum() > 0
    ctx = run(sta, dc)
    compare_update(ctx, oracle.update(dc))
    ctx.close()


def test_case_mux_selects(sta):
    # every MUX2 select pinned: one data arc of each mux disabled by its guard
    d = synth.generate(4000, 20, seed=410, period=400.0)
    lg = d.logic
    mux_tt = synth.truth_table(lambda a, b, s: b if s else a, 3)
    sel = [int(lg.fn_in[int(lg.fn_in_ptr[i]) + 2]) for i in range(len(lg.fn_pin))
           if int(lg.fn_tt[i]) == mux_tt and int(lg.fn_in_ptr[i + 1] - lg.fn_in_ptr[i]) == 3]
    assert sel
    rng = np.random.default_rng(5)
    sel = sorted(set(sel))
    dc, val, off = _consistent_case(d, rng, sel, len(sel))
    ctx = run(sta, dc)
    compare_update(ctx, oracle.update(dc))
    ctx.close()


def test_case_arnoldi_two_corners(sta):
    d = synth.generate(2500, 16, seed=420, corners=2, period=400.0)
    rng = np.random.default_rng(6)
    dc, _, _ = _consistent_case(d, rng, list(range(d.num_pins)), 30)
    for model in ("arnoldi", "elmore"):
        ctx = run(sta, dc, corners=2, model=model)
        for k in range(2):
            compare_update(ctx, oracle.update(dc, corner=k, net_model=model), corner=k)
        ctx.close()


def test_case_with_exceptions_and_clocks(sta):
    from tests.test_oracle_exceptions import random_clocks, random_exceptions_through
    d = synth.generate(2500, 18, seed=430, period=400.0)
    rng = np.random.default_rng(7)
    dc, _, _ = _consistent_case(d, rng, list(range(d.num_pins)), 25)
    dc.exceptions = random_exceptions_through(dc, rng, 3)
    dc.clocks = random_clocks(dc, rng, 2)
    ctx = run(sta, dc)
    compare_update(ctx, oracle.update(dc))
    ctx.close()


def test_case_path_report(sta):
    d = synth.generate(1500, 14, seed=440, period=300.0)
    rng = np.random.default_rng(8)
    dc, _, _ = _consistent_case(d, rng, list(range(d.num_pins)), 20)
    ctx = run(sta, dc)
    compare_update(ctx, oracle.update(dc))
    check(sta, ctx, dc)                        # the path report's own checks (tests/test_gpu_paths.py)
    ctx.close()


def test_case_repeated_and_cleared(sta):
    d = synth.generate(2500, 18, seed=450, period=400.0)
    rng = np.random.default_rng(9)
    dc, _, _ = _consistent_case(d, rng, list(range(d.num_pins)), 30)
    ctx = run(sta, dc)
    o = oracle.update(dc)
    for _ in range(3):
        ctx.update_timing()
        compare_update(ctx, o)
    ctx.set_case_analysis()                    # cleared: the plain update
    ctx.update_timing()
    d0 = copy.copy(d)
    compare_update(ctx, oracle.update(d0))
    ctx.close()


def test_case_errors(sta):
    d = synth.generate(300, 8, seed=460, period=300.0)
    lg = d.logic
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    with pytest.raises(sta.StaError) as e:                 # pin out of range
        ctx.set_case_analysis(lg.fn_pin, lg.fn_in_ptr, lg.fn_in, lg.fn_tt, None, [d.num_pins], [0])
    assert e.value.name == "STA_ERR_ID"
    with pytest.raises(sta.StaError) as e:                 # value 2
        ctx.set_case_analysis(lg.fn_pin, lg.fn_in_ptr, lg.fn_in, lg.fn_tt, None, [0], [2])
    assert e.value.name == "STA_ERR_ARG"
    with pytest.raises(sta.StaError) as e:                 # 7 inputs
        ctx.set_case_analysis([int(lg.fn_pin[0])], [0, 7], list(range(7)), [1], None, [], [])
    assert e.value.name == "STA_ERR_ARG"
    # contradictory constants: an inverter's input and output both 0
    inv = synth.truth_table(lambda a: 1 - a, 1)
    i = [i for i in range(len(lg.fn_pin))
         if int(lg.fn_tt[i]) == inv and int(lg.fn_in_ptr[i + 1] - lg.fn_in_ptr[i]) == 1][0]
    a, y = int(lg.fn_in[int(lg.fn_in_ptr[i])]), int(lg.fn_pin[i])
    ctx.set_case_analysis(lg.fn_pin, lg.fn_in_ptr, lg.fn_in, lg.fn_tt, None, [a, y], [0, 0])
    with pytest.raises(sta.StaError) as e:
        ctx.update_timing()
    assert e.value.name == "STA_ERR_ARG"
    ctx.close()


def test_case_stage_kernels(sta):
    # the per-stage launcher (STA_STAGE_KERNELS=1) reads the same patched
    # term arrays and killed-sink records
    import os
    d = synth.generate(2500, 16, seed=470, period=400.0)
    rng = np.random.default_rng(10)
    dc, _, _ = _consistent_case(d, rng, list(range(d.num_pins)), 30)
    os.environ["STA_STAGE_KERNELS"] = "1"
    try:
        ctx = run(sta, dc)
    finally:
        os.environ.pop("STA_STAGE_KERNELS", None)
    compare_update(ctx, oracle.update(dc))
    ctx.close()


def test_case_through_arnoldi_two_corners(sta):
    # every feature of row f4 at once on the Arnoldi instantiations: case
    # constants, -from / -through / -to exceptions, 2 corners
    from tests.test_oracle_exceptions import random_exceptions_through
    d = synth.generate(2000, 14, seed=480, corners=2, period=400.0)
    rng = np.random.default_rng(11)
    dc, _, _ = _consistent_case(d, rng, list(range(d.num_pins)), 20)
    dc.exceptions = random_exceptions_through(dc, rng, 3)
    ctx = run(sta, dc, corners=2, model="arnoldi")
    for k in range(2):
        compare_update(ctx, oracle.update(dc, corner=k, net_model="arnoldi"), corner=k)
    ctx.close()
