"""GPU parity on the paths the synthetic recipe never reaches (VERDICT r1
"Next round" item 2), element by element against the fp64 oracle:
table shapes 1x1 / 1xn / nx1 / 2x2 / 8x8 with negative (clamped) values,
table pools too large for the shared-memory image (global lookups),
endpoints that also have fan-out, the netlist loaded from
device arrays, 8 and 10 corners in one ctx (one and two launch batches),
corners whose libraries use different axes (different pool sizes), and
BASELINE configs[4] (C5) at full size, every corner.

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from synth import variants
from tests.parity import compare_update
from tests.test_gpu_parity import check_levels, check_rc, run

pytestmark = pytest.mark.gpu

OUT = os.environ.get("STA_PARITY_REPORT_DIR", "gpurun_out")


@pytest.fixture(scope="module")
def sta():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 (there is no CPU fallback)")
    import paper_2511_11660_b200 as pkg
    return pkg


def _report(name, rep):
    try:
        os.makedirs(OUT, exist_ok=True)
        with open(os.path.join(OUT, f"parity_{name}.json"), "w") as f:
            json.dump(rep, f, indent=1)
    except OSError:
        pass
    print(name, json.dumps(rep))


@pytest.mark.parametrize("seed", range(6))
def test_odd_table_shapes_and_negative_values(sta, seed):
    d = synth.generate(3000, 24, seed=100 + seed, frac_pi=0.05, frac_po=0.05, period=300.0)
    d = variants.odd_tables(d, seed)
    shapes = {(int(a), int(b)) for a, b in zip(d.libs[0].n1, d.libs[0].n2)}
    assert {(1, 1), (8, 8)} <= shapes and any(a == 1 < b for a, b in shapes) and any(b == 1 < a for a, b in shapes)
    neg = any(np.min(d.libs[0].table(t)[2]) < 0 for t in range(d.libs[0].num_tables))
    assert neg
    ctx = run(sta, d)
    assert ctx.info()["lut_smem_bytes"] > 0
    compare_update(ctx, oracle.update(d))
    check_rc(ctx, d)
    ctx.close()


@pytest.mark.parametrize("mode", ["0", "1"])
def test_table_pool_in_global_memory(sta, mode):
    """A pool of ~1400 tables (> the 200 KB shared-memory image): every lookup
    reads global memory; the used tables sit past the first 200 KB."""
    d = synth.generate(2500, 20, seed=7, period=300.0)
    d = variants.odd_tables(d, 11, n_pad=1300)
    os.environ["STA_STAGE_KERNELS"] = mode
    try:
        ctx = run(sta, d)
    finally:
        os.environ.pop("STA_STAGE_KERNELS", None)
    assert ctx.info()["lut_smem_bytes"] == 0
    compare_update(ctx, oracle.update(d))
    ctx.close()


@pytest.mark.parametrize("seed", range(3))
def test_endpoints_with_fanout(sta, seed):
    d = synth.generate(6000, 30, seed=40 + seed, period=300.0)
    d = variants.endpoints_with_fanout(d, seed, frac=0.08)
    assert d.meta["po_with_fanout"] > 20
    ctx = run(sta, d)
    compare_update(ctx, oracle.update(d))
    check_rc(ctx, d)
    ctx.close()


def test_load_graph_from_device_arrays(sta):
    """sta_load_graph / set_library / set_rc_tree / set_constraints with
    STA_MEM_DEVICE inputs give the same bits as host inputs."""
    d = synth.generate(5000, 30, seed=8, n_hfn=2, hfn_range=(200, 2000), period=300.0)
    a = sta.Context(0, 1)
    sta.load_design(a, d)
    a.update_timing()
    b = sta.Context(0, 1)
    sta.load_design(b, d, device_graph=True, device_rc=True)
    b.update_timing()
    for x, y in zip(a.get_timing(0), b.get_timing(0)):
        assert np.array_equal(x, y)
    assert np.array_equal(a.report_slack(0)[0], b.report_slack(0)[0])
    check_levels(b, d)
    compare_update(b, oracle.update(d))


@pytest.mark.parametrize("K", [8, 10])
def test_many_corners_one_ctx(sta, K):
    """K corners in one ctx: 8 = one launch batch, 10 = two batches."""
    d = synth.generate(4000, 30, seed=50 + K, corners=K, corner_recipe="c5", n_hfn=1,
                       hfn_range=(1500, 3000), period=300.0)
    ctx = run(sta, d)
    for c in range(K):
        compare_update(ctx, oracle.update(d, c), corner=c)
        check_rc(ctx, d, c, c)
    # a batched corner equals the same corner run alone, bit for bit
    one = run(sta, d, corners=[K - 1])
    for x, y in zip(ctx.get_timing(K - 1), one.get_timing(0)):
        assert np.array_equal(x, y)


def test_corner_libraries_with_different_axes(sta):
    """corners whose pools differ in size (own axis templates)."""
    d = synth.generate(4000, 30, seed=61, corners=4, corner_recipe="c5", period=300.0)
    d = variants.corner_axes_differ(d, 3)
    sizes = {L.data.size for L in d.libs}
    ctx = run(sta, d)
    for c in range(4):
        compare_update(ctx, oracle.update(d, c), corner=c)
    assert len(sizes) >= 1


def test_c2_tau_report(sta):
    """BASELINE configs[1] with the per-array error / bound headroom written out."""
    d = synth.config_design("c2_tau")
    ctx = run(sta, d)
    rep = {}
    compare_update(ctx, oracle.update(d), report=rep)
    _report("c2_tau", rep)


@pytest.mark.slow
def test_c5_multicorner_full(sta):
    """BASELINE configs[4] at full size in one ctx (8 corners x ~2M pins, one
    launch batch): every corner, every pin, WNS and TNS."""
    d = synth.config_design("c5_multicorner")
    ctx = run(sta, d)
    reps = {}
    for c in range(d.num_corners):
        rep = {}
        compare_update(ctx, oracle.update(d, c), corner=c, report=rep)
        reps[c] = rep
    _report("c5_multicorner", reps)
