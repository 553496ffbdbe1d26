#!/usr/bin/env python
"""Row f2 measurement: sta_build_steiner (Steiner RC from pin positions on the
device) on a BASELINE config, then the timing update on that RC.

    python scripts/bench_steiner.py [config] [--reps R] [--full-parity]

Prints one JSON line: ms per build (the C call with device positions and
device outputs, CUDA-synchronized), nodes, its GB/s against the HBM peak
(algorithmic bytes: positions read 8 B/pin, RC arrays written 16 B/node +
rc_ptr), the update time on the Steiner RC, and parity: every net of a
seeded sample (plus the smallest high-fan-out nets) bit-exact against the
oracle's O11; --full-parity also runs the oracle's full update on the
oracle's Steiner RC and compares WNS/TNS (C4-sized designs: seconds).
"""
import argparse
import copy
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c4_tdp")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sample", type=int, default=3000)
    ap.add_argument("--full-parity", action="store_true")
    a = ap.parse_args()
    import torch
    import oracle
    import synth
    import paper_2511_11660_b200 as sta
    d = synth.config_design(a.config, corners=1)
    x, y = synth.placement(d, seed=7)
    U = synth.STEINER_UNITS
    ctx = sta.Context(0, 1)
    sta.load_design(ctx, d)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(2):
        out = ctx.build_steiner(xd, yd, **U)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        out = ctx.build_steiner(xd, yd, **U)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.median(ts))
    rc_ptr, parent, node_pin, res, cap = (t.cpu().numpy() for t in out)
    n_nodes = int(rc_ptr[-1])
    P, N = d.num_pins, d.num_nets
    alg = 8 * P + 16 * n_nodes + 4 * (N + 1)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    # sampled parity: random nets + the two smallest nets of > 32 pins and the largest <= 2000
    m = np.diff(d.net_ptr)
    rng = np.random.default_rng(1)
    pick = set(rng.choice(N, size=min(a.sample, N), replace=False).tolist())
    big = np.nonzero(m > 32)[0]
    if big.size:
        order = big[np.argsort(m[big])]
        pick.update(order[:2].tolist())
        mid = order[m[order] <= 2000]
        if mid.size:
            pick.add(int(mid[-1]))
    pick = np.array(sorted(pick))
    sub_ptr = np.concatenate([[0], np.cumsum(m[pick])]).astype(np.uint32)
    sub_pins = np.concatenate([d.net_pins[d.net_ptr[n]:d.net_ptr[n + 1]] for n in pick]).astype(np.uint32)
    o = oracle.steiner(sub_ptr, sub_pins, x, y, **U)
    bad = 0
    for i, n in enumerate(pick):
        a0, a1 = int(rc_ptr[n]), int(rc_ptr[n + 1])
        b0, b1 = int(o[0][i]), int(o[0][i + 1])
        ok = (a1 - a0 == b1 - b0 and np.array_equal(parent[a0:a1], o[1][b0:b1])
              and np.array_equal(node_pin[a0:a1].view(np.uint32), o[2][b0:b1])
              and np.array_equal(res[a0:a1], o[3][b0:b1])
              and np.allclose(cap[a0:a1], o[4][b0:b1], rtol=1e-6, atol=1e-7))
        bad += not ok
    # the update on the Steiner RC (tree re-planned on the host: a new topology)
    t0 = time.perf_counter()
    ctx.set_rc_tree(out[0], out[1], out[2])
    plan_s = time.perf_counter() - t0
    ctx.set_rc_values(0, out[3], out[4])
    ctx.update_timing()
    ctx.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.update_timing()
    ctx.synchronize()
    ups = []
    for _ in range(5):
        t0 = time.perf_counter()
        ctx.update_timing()
        ctx.synchronize()
        ups.append(time.perf_counter() - t0)
    res4, _ = ctx.report_slack(0)
    line = dict(metric="Steiner RC build (row f2) + timing update on it", config=a.config, pins=P, nets=N,
                max_net_pins=int(m.max()), rc_nodes=n_nodes, build_ms=ms, build_ms_all=[1e3 * t for t in ts],
                build_gbs=alg / (ms / 1e3) / 1e9, hbm_peak_gbs=peak, build_frac_hbm=alg / (ms / 1e3) / 1e9 / peak,
                algorithmic_bytes=alg, set_rc_tree_s=plan_s, update_ms_wall=1e3 * float(np.median(ups)),
                wns_tns=res4.tolist(), parity_sample_nets=int(pick.size), parity_mismatches=int(bad))
    if a.full_parity:
        oa = oracle.steiner(d.net_ptr, d.net_pins, x, y, **U)
        d2 = copy.copy(d)
        d2.rc = [synth.RcTree(*oa)]
        ref = oracle.update(d2, want_all=False)
        line["oracle_wns_tns"] = [float(v) for v in ref["res"]]
        line["wns_tns_abs_err"] = [abs(float(a_) - float(b_)) for a_, b_ in zip(res4, ref["res"])]
    print(json.dumps(line))
    ctx.close()


if __name__ == "__main__":
    main()
