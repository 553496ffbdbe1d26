"""C5 (BASELINE.json configs[4]): multi-corner sign-off, 8 corners of a
~2M-pin synthetic design (corner c: LUT x (0.80 + 0.06c), wire R x (0.85 +
0.05c), wire Cw x (0.90 + 0.03c)).  On one GPU all corners run in one
Context (one update = all 8 corners); with N ranks (torchrun) each rank owns
corners [r K / N, (r + 1) K / N) and the per-corner WNS/TNS rows are combined
by one all_reduce (paper_2511_11660_b200.multicorner).  Reports corner-updates
per second and ms per 8-corner sign-off, and checks every corner's WNS/TNS
against the oracle (--check).

  python scripts/bench_c5.py [--steps 20] [--check]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_11660_b200 as sta  # noqa: E402
from paper_2511_11660_b200 import multicorner as mc  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    d = synth.config_design("c5_multicorner")
    K = d.num_corners
    mine = list(mc.corners_of_rank(K, rank, world))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = sta.Context(local, len(mine), stream=stream.cuda_stream)
    sta.load_design(ctx, d, corners=mine)
    rows = torch.zeros((K, 4), dtype=torch.float64, device="cuda")

    def step():
        ctx.update_timing()
        rows.zero_()
        for k, c in enumerate(mine):
            ctx.report_wns_tns_device(k, rows[c])
        mc.combine_rows(rows)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    info = ctx.info()
    line = {"config": "c5_multicorner: BASELINE.json configs[4], 8 corners x ~2M-pin synthetic design",
            "n_gpus": world, "corners": K, "pins": info["num_pins"], "gate_stages": info["num_stages"],
            "ms_per_signoff": ms, "corner_updates_per_s": K / (ms / 1e3),
            "pins_per_s": K * info["num_pins"] / (ms / 1e3),
            "global": [float(x) for x in mc.global_report(rows.cpu())]}
    if a.check and rank == 0:
        import oracle
        oracle.build()
        r = rows.cpu().numpy()
        err = []
        for c in range(K):
            ref = oracle.update(d, c, want_all=False)["res"]
            err.append(max(abs(float(r[c][0]) - ref[0]), abs(float(r[c][2]) - ref[2])))
        line["max_wns_abs_err_ps"] = max(err)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
