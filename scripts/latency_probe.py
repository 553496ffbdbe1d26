#!/usr/bin/env python
"""Per-stage latency of the persistent forward / backward kernels on narrow
designs (few pins per gate stage: every stage is one dependent hop), next to
the wide C2 / C3 shapes: ms per phase and us per gate stage.

    python scripts/latency_probe.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(name, d, reps=20):
    import paper_2511_11660_b200 as sta
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    for _ in range(3):
        ctx.update_timing()
    ctx.profile_enable(True)
    for _ in range(reps):
        ctx.update_timing()
    p = ctx.profile_read()
    ctx.profile_enable(False)
    info = ctx.info()
    S = info["num_stages"]
    ms = {k: v / max(p["updates"], 1) for k, v in p["ms"].items()}
    out = dict(design=name, pins=d.num_pins, stages=S, ms=ms,
               us_per_stage={k: 1e3 * ms[k] / S for k in ("forward", "backward")})
    ctx.close()
    return out


def main():
    import synth
    rows = []
    for n_cells, levels in ((300, 150), (3000, 150), (30000, 150)):
        rows.append(run(f"narrow_{n_cells}x{levels}", synth.generate(n_cells, levels, seed=3, period=2000.0)))
    for cfg in ("c2_tau", "c3_superblue"):
        rows.append(run(cfg, synth.config_design(cfg, corners=1), reps=10))
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
