"""Small updates for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
c17, a 2k-cell synthetic design with high-fan-out nets, wide gates and
two-output cells; both launchers; compared with the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2511_11660_b200 as sta  # noqa: E402
import synth  # noqa: E402
from tests.parity import compare_update  # noqa: E402
from tests.test_gpu_parity import _wide_multi_output_design  # noqa: E402

designs = [synth.c17(), synth.generate(2000, 16, seed=4, n_hfn=2, hfn_range=(40, 400), period=200.0),
           _wide_multi_output_design(),
           # tier-C RC (nets > 1024 nodes), 3 corners in one launch batch
           synth.generate(3000, 16, seed=6, n_hfn=2, hfn_range=(1500, 2500), corners=3, corner_recipe="c5",
                          period=250.0)]
for mode in ("0", "1"):
    os.environ["STA_STAGE_KERNELS"] = mode
    for d in designs:
        ctx = sta.Context(0, d.num_corners)
        sta.load_design(ctx, d)
        for _ in range(2):
            ctx.update_timing()
        ctx.synchronize()
        for c in range(d.num_corners):
            compare_update(ctx, oracle.update(d, c), corner=c)
        ctx.report_paths(0, "setup", k=20, nworst=2)       # row f3 kernels
        ctx.close()
        print("ok", mode, d.name, flush=True)

# rows f1 (Arnoldi net model, persistent kernels) and f2 (Steiner RC)
os.environ["STA_STAGE_KERNELS"] = "0"
for d in designs[:2]:
    ctx = sta.Context(0, d.num_corners)
    sta.load_design(ctx, d)
    ctx.set_net_model("arnoldi", 4)
    ctx.update_timing()
    ctx.synchronize()
    compare_update(ctx, oracle.update(d, net_model="arnoldi"))
    x, y = synth.placement(d, seed=2, grid=True)
    g = ctx.build_steiner(x, y, **synth.STEINER_UNITS)
    ctx.close()
    print("ok arnoldi + steiner", d.name, int(g[0][-1]), flush=True)

# row f4: -from / -through / -to exceptions with 2 clocks (THR instantiations,
# handoff / capture / epoch kernels), Elmore and Arnoldi, 3 corners
import numpy as np  # noqa: E402
from tests.test_oracle_exceptions import random_clocks, random_exceptions_through  # noqa: E402
for model in ("elmore", "arnoldi"):
    d = designs[3]
    rng = np.random.default_rng(5)
    d.exceptions = random_exceptions_through(d, rng, 3)
    d.clocks = random_clocks(d, rng, 2)
    ctx = sta.Context(0, d.num_corners)
    sta.load_design(ctx, d)
    if model == "arnoldi":
        ctx.set_net_model("arnoldi", 4)
    for _ in range(2):
        ctx.update_timing()
    ctx.synchronize()
    for c in range(d.num_corners):
        compare_update(ctx, oracle.update(d, c, net_model=model), corner=c)
    ctx.close()
    print("ok exceptions -through", model, flush=True)
