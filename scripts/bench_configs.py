"""Per-config numbers for BASELINE.md §3 (C1 c17, C2 TAU-shaped, C3
superblue-shaped; C4 via scripts/bench_tdp.py, C5 via bench.py --config
c5_multicorner): device ms per full update (median / p10 / p90 of 20 CUDA-event
timed updates after 5 warm-ups, ctx stream), pins/s, model bytes and % of the
measured HBM peak, the fp64 oracle on one host core, the largest
|error| / bound of the full-array parity check, and the top-k path report.

  python scripts/bench_configs.py [--configs c1_c17 c2_tau c3_superblue]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2511_11660_b200 as sta  # noqa: E402
import synth  # noqa: E402
from tests.parity import compare_update  # noqa: E402


def one(name, paths):
    d = synth.config_design(name)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = sta.Context(0, 1, stream=stream.cuda_stream)
    t0 = time.perf_counter()
    sta.load_design(ctx, d)
    torch.cuda.synchronize()
    load_s = time.perf_counter() - t0
    r = torch.from_numpy(d.rc[0].res).cuda()
    c = torch.from_numpy(d.rc[0].cap).cuda()
    ctx.set_rc_values(0, r, c)
    for _ in range(5):
        ctx.update_timing()
    torch.cuda.synchronize()
    times = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.update_timing()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    times.sort()
    ms = statistics.median(times)
    info = ctx.info()
    ab = bench.algorithmic_bytes(d, info)
    peak, _ = bench.measured_peaks()
    tot = sum(ab.values())
    t0 = time.perf_counter()
    ref = oracle.update(d)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    rep = {}
    compare_update(ctx, ref, report=rep)
    worst = max((v.get("max_err_over_bound", 0.0) for v in rep.values() if isinstance(v, dict)), default=0.0)
    out = {"config": name, "pins": info["num_pins"], "pin_levels": info["num_levels"],
           "gate_stages": info["num_stages"], "ms_median": ms, "ms_p10": times[2], "ms_p90": times[17],
           "pins_per_s": info["num_pins"] / (ms / 1e3), "model_bytes": tot, "model_bytes_per_pin": tot / info["num_pins"],
           "frac_hbm_model": tot / (ms / 1e3) / 1e9 / peak, "oracle_ms_1core": cpu_ms,
           "host_cores": os.cpu_count(), "load_graph_s": load_s, "parity_max_err_over_bound": worst,
           "parity": rep}
    if paths:
        pr = {}
        for k, nw in ((1000, 1), (1000, 8)):
            ctx.report_paths(0, "setup", k=k, nworst=nw)      # warm (lazy uploads)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g = ctx.report_paths(0, "setup", k=k, nworst=nw)
            pr[f"k{k}_nworst{nw}_ms"] = (time.perf_counter() - t0) * 1e3
            pr[f"k{k}_nworst{nw}_paths"] = len(g)
        if info["num_pins"] < 1e6:
            t0 = time.perf_counter()
            oracle.paths(d, 0, "setup", k=1000, nworst=8)
            pr["oracle_k1000_nworst8_ms"] = (time.perf_counter() - t0) * 1e3
        out["paths"] = pr
    ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["c1_c17", "c2_tau", "c3_superblue"])
    ap.add_argument("--no-paths", action="store_true")
    a = ap.parse_args()
    oracle.build()
    for n in a.configs:
        print(json.dumps(one(n, not a.no_paths)), flush=True)


if __name__ == "__main__":
    main()
