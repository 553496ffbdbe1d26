"""GPU parity of the -from / -to timing exceptions (SURVEY.md §8(f) row 4,
reduced; sta_set_exceptions) against the oracle's O13: every pin's merged
arrival / slew / required time / slack and WNS / TNS element by element.

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import copy

import numpy as np
import pytest

import oracle
import synth
from synth.design import Exceptions
from tests.parity import compare_update
from tests.test_oracle_exceptions import random_exceptions, _endpoints, _startpoints

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


@pytest.mark.parametrize("seed", range(6))
def test_random_exceptions(sta, seed):
    d = synth.generate(2500, 18, seed=200 + seed, period=400.0)
    rng = np.random.default_rng(seed)
    d.exceptions = random_exceptions(d, rng, int(rng.integers(1, 7)))
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()


def test_tags_from_startpoints(sta):
    # several -from classes (up to 7 tags) mixing every kind, -to on subsets
    d = synth.generate(6000, 24, seed=210, period=500.0)
    sp, ep = _startpoints(d), _endpoints(d)
    rng = np.random.default_rng(3)
    perm = list(rng.permutation(sp))
    g = len(sp) // 8
    items = []
    for k in range(6):
        fr = perm[k * g:(k + 1) * g] + (perm[:g // 2] if k == 5 else [])   # disjoint classes + one overlap
        to = list(rng.choice(ep, size=len(ep) // 3, replace=False)) if k % 2 else []
        kind = k % 4
        val = 2.0 if kind == 1 else (350.0 if kind == 2 else 5.0)
        items.append((kind, val, fr, to))
    d.exceptions = Exceptions.build(items)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()


def test_exceptions_clear_and_paths(sta):
    d = synth.generate(1500, 14, seed=220, period=300.0)
    d.exceptions = Exceptions.build([(0, 0.0, [], _endpoints(d)[:5]), (1, 2.0, [], [])])
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    with pytest.raises(sta.StaError) as e:
        ctx.report_paths(0, "setup", k=3)
    assert e.value.name == "STA_ERR_ORDER"
    ctx.set_exceptions()                       # cleared: the plain update again
    ctx.update_timing()
    d0 = copy.copy(d)
    d0.exceptions = None
    compare_update(ctx, oracle.update(d0))
    ctx.report_paths(0, "setup", k=3)
    ctx.close()


def test_exceptions_multicorner_arnoldi(sta):
    d = synth.generate(2000, 14, seed=230, corners=2, period=400.0)
    rng = np.random.default_rng(9)
    d.exceptions = random_exceptions(d, rng, 4)
    ctx = run(sta, d, corners=2, model="arnoldi")
    for k in range(2):
        compare_update(ctx, oracle.update(d, corner=k, net_model="arnoldi"), corner=k)
    ctx.close()


def test_exceptions_c2(sta):
    d = synth.config_design("c2_tau", corners=1)
    sp, ep = _startpoints(d), _endpoints(d)
    rng = np.random.default_rng(11)
    d.exceptions = Exceptions.build([
        (0, 0.0, list(rng.choice(sp, 20, replace=False)), []),
        (1, 2.0, [], list(rng.choice(ep, 200, replace=False))),
        (2, 900.0, list(rng.choice(sp, 30, replace=False)), list(rng.choice(ep, 300, replace=False))),
        (3, 3.0, [], list(rng.choice(ep, 100, replace=False)))])
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()


def test_exception_errors(sta):
    d = synth.generate(300, 8, seed=240, period=300.0)
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    with pytest.raises(sta.StaError) as e:
        ctx.set_exceptions([1], [1.5], [0, 0], [], [0, 0], [])       # multicycle N not integral
    assert e.value.name == "STA_ERR_ARG"
    with pytest.raises(sta.StaError) as e:
        ctx.set_exceptions([0], [0.0], [0, 1], [d.num_pins], [0, 0], [])
    assert e.value.name == "STA_ERR_ID"
    ctx.close()


@pytest.mark.parametrize("seed", range(4))
def test_multiple_clocks(sta, seed):
    # 2-3 ideal clocks (launch / capture relationships), half with exceptions on top
    from tests.test_oracle_exceptions import random_clocks
    d = synth.generate(3000, 20, seed=250 + seed, period=400.0)
    rng = np.random.default_rng(50 + seed)
    d.clocks = random_clocks(d, rng, int(rng.integers(2, 4)))
    if seed % 2:
        d.exceptions = random_exceptions(d, rng, 3)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()


def test_clocks_reset_and_errors(sta):
    from tests.test_oracle_exceptions import random_clocks
    d = synth.generate(1500, 12, seed=260, period=300.0)
    d.clocks = random_clocks(d, np.random.default_rng(1), 2)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.set_clocks()                           # back to the single clock
    ctx.update_timing()
    d0 = copy.copy(d)
    d0.clocks = None
    compare_update(ctx, oracle.update(d0))
    with pytest.raises(sta.StaError) as e:
        ctx.set_clocks([100.0, -1.0], np.zeros(d.num_pins, np.uint32))
    assert e.value.name == "STA_ERR_ARG"
    with pytest.raises(sta.StaError) as e:
        ctx.set_clocks([100.0], np.full(d.num_pins, 3, np.uint32))
    assert e.value.name == "STA_ERR_ID"
    ctx.close()


# ---- -through segments (row f4; the oracle's O15; SPEC.md:466-473, 494;
# PAPER.md:250): every tag is a pass, arrivals handed on at the through
# pins in a forward sweep, required times taken back in reverse order

def _through_items(d, rng, n):
    """n random exceptions, most with 1-2 ordered -through segments (any
    pin), optional -from / -to lists (the oracle tests' generator)"""
    from tests.test_oracle_exceptions import random_exceptions_through
    return random_exceptions_through(d, rng, n)


def _sinks_and_pulls(d):
    sinks = sorted(set(int(p) for n in range(d.num_nets)
                       for p in d.net_pins[int(d.net_ptr[n]) + 1:int(d.net_ptr[n + 1])]))
    fi = set(int(p) for p in d.arc_to)
    pulls = sorted(fi - set(sinks))
    return sinks, pulls


@pytest.mark.parametrize("seed", range(8))
def test_through_random(sta, seed):
    d = synth.generate(2500, 18, seed=300 + seed, period=400.0)
    rng = np.random.default_rng(70 + seed)
    d.exceptions = _through_items(d, rng, int(rng.integers(1, 4)))
    if seed % 4 == 3:
        from tests.test_oracle_exceptions import random_clocks
        d.clocks = random_clocks(d, rng, 2)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()


@pytest.mark.parametrize("where", ["sinks", "pulls"])
def test_through_sinks_and_pull_pins(sta, where):
    # through pins only on net sinks (pull-through arrivals: every consumer's
    # hook, the capture kernel) or only on cell outputs (stored records)
    d = synth.generate(3000, 20, seed=320, period=400.0)
    sinks, pulls = _sinks_and_pulls(d)
    rng = np.random.default_rng(5 if where == "sinks" else 6)
    pool = sinks if where == "sinks" else pulls
    sp = _startpoints(d)
    items = []
    for k in range(3):
        th = [list(rng.choice(pool, 40, replace=False)) for _ in range(1 + k % 2)]
        fr = list(rng.choice(sp, 10, replace=False)) if k == 1 else []
        items.append(([0, 1, 2][k], [0.0, 2.0, 150.0][k], fr, [], th))
    d.exceptions = Exceptions.build(items)
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()


def test_through_wide_gates_and_heavy_drivers(sta):
    # the forward's warp-loop pins (> 8 terms), the backward's CSR fan-out and
    # heavy drivers (> 32 sinks) as through pins
    from tests.test_gpu_parity import _wide_multi_output_design
    d = _wide_multi_output_design()
    cnt = np.bincount(np.asarray(d.arc_to, np.int64), minlength=d.num_pins)
    wide = [int(p) for p in np.nonzero(cnt > 8)[0]]
    sinks, _ = _sinks_and_pulls(d)
    assert wide
    d.exceptions = Exceptions.build([(0, 0.0, [], [], [wide[:1]]), (2, 80.0, [], [], [[wide[-1]], sinks[-4:]]),
                                     (1, 2.0, [], [], [sinks[:6]])])
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()
    d = synth.generate(6000, 24, seed=330, n_hfn=3, hfn_range=(200, 2000), period=400.0)
    sinks, pulls = _sinks_and_pulls(d)
    nfo = np.diff(np.asarray(d.net_ptr, np.int64))
    big = np.argsort(-nfo)[:3]
    hfn_sinks = [int(d.net_pins[int(d.net_ptr[n]) + 5]) for n in big]
    hfn_drv = [int(d.net_pins[int(d.net_ptr[n])]) for n in big]
    rng = np.random.default_rng(8)
    d.exceptions = Exceptions.build([(0, 0.0, [], [], [hfn_sinks[:2]]),
                                     (3, 4.0, [], [], [hfn_drv, list(rng.choice(pulls, 30, replace=False))]),
                                     (1, 3.0, [], [], [list(rng.choice(sinks, 50, replace=False))])])
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    ctx.close()


def test_through_multicorner_arnoldi(sta):
    d = synth.generate(2000, 14, seed=340, corners=2, period=400.0)
    rng = np.random.default_rng(12)
    d.exceptions = _through_items(d, rng, 3)
    for model in ("arnoldi", "elmore"):
        ctx = run(sta, d, corners=2, model=model)
        for k in range(2):
            compare_update(ctx, oracle.update(d, corner=k, net_model=model), corner=k)
        ctx.close()


def test_through_repeated_and_cleared(sta):
    # repeated updates (the handoff buffers and the record epochs of the
    # forward-only sweep), then -through cleared and -from / -to only
    d = synth.generate(2500, 18, seed=350, period=400.0)
    rng = np.random.default_rng(13)
    d.exceptions = _through_items(d, rng, 3)
    ctx = run(sta, d)
    o = oracle.update(d)
    for _ in range(3):
        ctx.update_timing()
        compare_update(ctx, o)
    d2 = copy.copy(d)
    d2.exceptions = random_exceptions(d, rng, 3)
    ex = d2.exceptions
    ctx.set_exceptions(ex.kind, ex.value, ex.from_ptr, ex.from_pins, ex.to_ptr, ex.to_pins)
    ctx.update_timing()
    compare_update(ctx, oracle.update(d2))
    ctx.close()


def test_through_errors(sta):
    d = synth.generate(300, 8, seed=360, period=300.0)
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    with pytest.raises(sta.StaError) as e:           # an empty segment
        ctx.set_exceptions([0], [0.0], [0, 0], [], [0, 0], [], [0, 1], [0, 0], [])
    assert e.value.name == "STA_ERR_CSR"
    with pytest.raises(sta.StaError) as e:           # a through pin out of range
        ctx.set_exceptions([0], [0.0], [0, 0], [], [0, 0], [], [0, 1], [0, 1], [d.num_pins])
    assert e.value.name == "STA_ERR_ID"
    with pytest.raises(sta.StaError) as e:           # 33 segments
        ctx.set_exceptions([0], [0.0], [0, 0], [], [0, 0], [], [0, 33], list(range(34)), list(range(33)))
        ctx.update_timing()
    assert e.value.name == "STA_ERR_ARG"
    ctx.close()
