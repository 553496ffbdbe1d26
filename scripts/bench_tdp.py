"""C4 (BASELINE.json configs[3]): a DREAMPlace-style timing-driven placement
loop -- 1M-cell synthetic design, N repeated full STA updates, each after a
device-side perturbation of every RC node's R and Cw (R' = R (1 + 0.1 (2u - 1)),
u uniform, a fresh draw per iteration), handed to the engine as borrowed
device pointers (zero host traffic).  Reports ms per update (perturbation
timed separately) and checks iterations {0, 1, last} against the oracle.

  python scripts/bench_tdp.py [--iters 1000]        (on the GPU box)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_11660_b200 as sta  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=1000)
    ap.add_argument("--check", action="store_true", help="oracle parity at iterations 0, 1, last")
    a = ap.parse_args()
    d = synth.config_design("c4_tdp")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = sta.Context(0, 1, stream=stream.cuda_stream)
    sta.load_design(ctx, d)
    r0 = torch.from_numpy(d.rc[0].res).cuda()
    c0 = torch.from_numpy(d.rc[0].cap).cuda()
    rb = [torch.empty_like(r0) for _ in range(2)]     # double-buffered borrowed arrays
    cb = [torch.empty_like(c0) for _ in range(2)]
    gen = torch.Generator(device="cuda")

    def perturb(i):
        gen.manual_seed(0xD9E4 * 1000003 + i)
        k = i & 1
        torch.mul(r0, 1 + 0.1 * (2 * torch.rand(r0.shape, device="cuda", generator=gen) - 1), out=rb[k])
        torch.mul(c0, 1 + 0.1 * (2 * torch.rand(c0.shape, device="cuda", generator=gen) - 1), out=cb[k])
        return k

    for i in range(3):                                 # warm-up
        k = perturb(i)
        ctx.set_rc_values(0, rb[k], cb[k])
        ctx.update_timing()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    # perturbation alone
    ev[0].record(stream)
    for i in range(a.iters):
        perturb(i)
    ev[1].record(stream)
    # the loop: perturb + update
    ev[2].record(stream)
    for i in range(a.iters):
        k = perturb(i)
        ctx.set_rc_values(0, rb[k], cb[k])
        ctx.update_timing()
    ev[3].record(stream)
    torch.cuda.synchronize()
    ms_pert = ev[0].elapsed_time(ev[1]) / a.iters
    ms_loop = ev[2].elapsed_time(ev[3]) / a.iters
    info = ctx.info()
    line = {"config": "c4_tdp: BASELINE.json configs[3], 1M-cell synthetic design, repeated full updates "
                      "with device-perturbed RC values (borrowed pointers)",
            "pins": info["num_pins"], "gate_stages": info["num_stages"], "iters": a.iters,
            "ms_per_iteration": ms_loop, "ms_perturbation": ms_pert, "ms_per_update": ms_loop - ms_pert,
            "updates_per_s": 1e3 / (ms_loop - ms_pert), "pins_per_s": info["num_pins"] / ((ms_loop - ms_pert) / 1e3)}
    if a.check:
        import copy
        import oracle
        from tests.parity import compare_update
        oracle.build()
        errs = {}
        for i in (0, 1, a.iters - 1):
            k = perturb(i)
            ctx.set_rc_values(0, rb[k], cb[k])
            ctx.update_timing()
            ctx.synchronize()
            di = copy.copy(d)
            di.rc = [copy.copy(d.rc[0])]
            di.rc[0].res = rb[k].cpu().numpy()
            di.rc[0].cap = cb[k].cpu().numpy()
            rep = {}
            compare_update(ctx, oracle.update(di), report=rep)
            errs[i] = "ok"
        line["parity"] = errs
    print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
