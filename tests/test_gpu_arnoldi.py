"""GPU parity of the Arnoldi net-delay model (SURVEY.md §8(f) row 1,
sta_set_net_model(STA_NET_ARNOLDI)) against the oracle's O12 update: every
pin's arrival / slew / required time / slack and WNS / TNS element by element
(fp32 device Lanczos-model evaluation with a Newton crossing solver vs the
oracle's fp64 bisection to 1e-6 ps, within the R17 bound).

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import copy

import numpy as np
import pytest

import oracle
import synth
from tests.parity import compare_update

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sta():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 (there is no CPU fallback)")
    import paper_2511_11660_b200 as pkg
    return pkg


def run(sta, d, q=4):
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    ctx.set_net_model("arnoldi", q)
    ctx.update_timing()
    return ctx


@pytest.mark.parametrize("q", [1, 2, 4])
def test_arnoldi_small(sta, q):
    d = synth.generate(1500, 16, seed=101, period=400.0)
    ctx = run(sta, d, q)
    compare_update(ctx, oracle.update(d, net_model="arnoldi", q=q))
    ctx.close()


def test_arnoldi_c17_and_hand(sta):
    for d in (synth.c17(), synth.h3_reg2reg(), synth.h4_seeds()):
        ctx = run(sta, d)
        compare_update(ctx, oracle.update(d, net_model="arnoldi"))
        ctx.close()


def test_arnoldi_large_nets_and_checks(sta):
    # high-fan-out nets (hundreds to thousands of RC nodes: many 32-node
    # chunks per Lanczos pass), flip-flops (check seeds on Arnoldi slews)
    d = synth.generate(8000, 30, seed=102, n_hfn=4, hfn_range=(200, 3000), period=600.0)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d, net_model="arnoldi"))
    ctx.close()


def test_arnoldi_zero_resistance_and_switch_back(sta):
    # zero-R wires: no dynamics (delay 0, slew through); then back to Elmore
    d = synth.generate(1200, 12, seed=103, period=300.0)
    z = copy.copy(d)
    z.rc = [synth.RcTree(d.rc[0].rc_ptr, d.rc[0].parent, d.rc[0].node_pin, np.zeros_like(d.rc[0].res), d.rc[0].cap)]
    ctx = run(sta, z)
    compare_update(ctx, oracle.update(z, net_model="arnoldi"))
    ctx.set_net_model("elmore")
    ctx.update_timing()
    compare_update(ctx, oracle.update(z))
    ctx.close()


def test_arnoldi_c2_full(sta):
    d = synth.config_design("c2_tau", corners=1)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d, net_model="arnoldi"))
    # the path report is Elmore only
    with pytest.raises(sta.StaError) as e:
        ctx.report_paths(0, "setup", k=3)
    assert e.value.name == "STA_ERR_ORDER"
    ctx.close()


def test_arnoldi_multicorner(sta):
    d = synth.generate(2000, 14, seed=104, corners=3, period=400.0)
    ctx = sta.Context(0, 3)
    sta.load_design(ctx, d)
    ctx.set_net_model("arnoldi", 3)
    ctx.update_timing()
    for k in range(3):
        compare_update(ctx, oracle.update(d, corner=k, net_model="arnoldi", q=3), corner=k)
    ctx.close()


def test_arnoldi_bad_args(sta):
    ctx = sta.Context(0, 1)
    for q in (0, 5):
        with pytest.raises(sta.StaError) as e:
            ctx.set_net_model("arnoldi", q)
        assert e.value.name == "STA_ERR_ARG"
    ctx.close()
