#!/usr/bin/env python
"""Benchmark of one full graph-based STA timing update on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Workload (BASELINE.json configs[2], the config its metric is quoted on):
superblue-shaped synthetic netlist, ~10.4M pins, 151 pin levels, 32
high-fan-out nets, NLDM LIB-SYN tables, random RC trees.  One
step = one full update a1-a5 (Elmore RC + loads, forward AT/slew, endpoint
seeds, backward RAT, per-pin slack, WNS/TNS) of one corner per GPU; with N
GPUs (torchrun) every rank times its own corner and the per-corner WNS/TNS
rows are combined with one NCCL all_reduce per step (weak scaling).

`--impl reference` times the fp64 CPU oracle (the reference arm of this
tier) on a bounded sample of the same recipe, on rank 0's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "pins/s and ms per full STA update (10M-pin DAG), % HBM peak; 1/2/4/8-GPU corners"
CONFIG = "c3_superblue"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    help="c3_superblue (default at N=1), c5_multicorner (default at N>1), c2_tau, c4_tdp")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip e2e/profile/cpu legs (ncu runs)")
    ap.add_argument("--phases", action="store_true", help="with --quick: still measure the per-phase times")
    ap.add_argument("--net-model", default="elmore", choices=["elmore", "arnoldi"],
                    help="net-arc delay model (row f1: arnoldi = reduced order 4)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: several ranks may share one GPU -- a functional "
                         "multi-rank check on a one-GPU box, not a scaling measurement)")
    ap.add_argument("--exceptions", action="store_true",
                    help="row f4: a seeded set of -from / -to exceptions (3 startpoint tags)")
    ap.add_argument("--through", action="store_true",
                    help="row f4: --exceptions plus two -through exceptions (a false path through 0.2%% "
                         "of the pins, a multicycle through two ordered segments): up to 18 tags")
    ap.add_argument("--case", action="store_true",
                    help="row f4: case analysis, every MUX2 select pinned (alternately 0 / 1): one data arc "
                         "of every mux disabled by its when guard, the select arcs by the constants")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def corner_design(name, corner):
    """The config's design with corner `corner` of the nominal corner recipe."""
    import synth
    d = synth.config_design(name, corners=1)
    if corner:
        ls, rs, cs = synth.corner_scales(corner, "nominal")
        d.libs = [d.libs[0].scaled(ls)]
        d.rc = [d.rc[0].scaled(rs, cs)]
    return d


def bench_exceptions(d):
    """Row f4 workload: false path from 1% of the startpoints, multicycle 2 to
    5% of the endpoints, max delay T/2 from another 1% to 5%, min delay 3 ps
    to 2% (seeded; 3 startpoint tags)."""
    import synth
    from synth.design import Exceptions
    rng = np.random.default_rng(0xE7C)
    sp = sorted(set(int(p) for p in d.cons.pi_pin) |
                set(int(p) for p in np.nonzero(d.pin_role == synth.ROLE_FF_CK)[0]))
    ep = sorted(set(int(p) for p in d.cons.po_pin) | set(int(p) for p in d.chk_d))
    sp_p = rng.permutation(sp)
    n_s, n_e = max(1, len(sp) // 100), max(1, len(ep) // 20)
    return Exceptions.build([
        (0, 0.0, list(sp_p[:n_s]), []),
        (1, 2.0, [], list(rng.choice(ep, n_e, replace=False))),
        (2, float(d.cons.period) / 2, list(sp_p[n_s:2 * n_s]), list(rng.choice(ep, n_e, replace=False))),
        (3, 3.0, [], list(rng.choice(ep, max(1, len(ep) // 50), replace=False)))])


def bench_through(d):
    """Row f4 -through workload: bench_exceptions plus a false path -through
    0.2% of the pins (cell outputs and net sinks alike) and a multicycle 2
    -through one 0.5% set then another (seeded)."""
    from synth.design import Exceptions
    ex = bench_exceptions(d)
    rng = np.random.default_rng(0x7A2)
    P = d.num_pins
    items = []
    for i in range(ex.num):
        f = list(ex.from_pins[ex.from_ptr[i]:ex.from_ptr[i + 1]])
        t = list(ex.to_pins[ex.to_ptr[i]:ex.to_ptr[i + 1]])
        items.append((int(ex.kind[i]), float(ex.value[i]), f, t, []))
    items.append((0, 0.0, [], [], [list(rng.choice(P, P // 500, replace=False))]))
    items.append((1, 2.0, [], [], [list(rng.choice(P, P // 200, replace=False)),
                                   list(rng.choice(P, P // 200, replace=False))]))
    return Exceptions.build(items)


def bench_case(d):
    """Row f4 case-analysis workload: the select pin of every MUX2 cell
    pinned, alternately to 0 and 1 (the recipe's own logic functions)."""
    import synth
    from synth.design import CaseValues
    lg = d.logic
    k = np.diff(lg.fn_in_ptr.astype(np.int64))
    tt = synth.truth_table(lambda a, b, s: b if s else a, 3)
    mux = np.nonzero((lg.fn_tt == np.uint64(tt)) & (k == 3))[0]
    sel = lg.fn_in[lg.fn_in_ptr[mux].astype(np.int64) + 2]
    return CaseValues(sel.astype(np.uint32), (np.arange(sel.size) & 1).astype(np.uint8))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def algorithmic_bytes(d, info):
    """Unique bytes each phase must touch per update: fp32/u32
    elements counted once per pass, independent of the kernels' layout (the
    tags, padding and term records the kernels add are not counted)."""
    P, NP, NS = info["num_pins"], info["num_pull_pins"], info["num_sink_pins"]
    E = info["num_cell_arcs"]
    N = info["num_nets"]
    n_rc = int(d.rc[0].parent.shape[0])
    n_ep = info["num_endpoints"]
    rc = 20 * n_rc + 16 * N + 4 * NS            # parent,sink,scap,R,Cw; net tables; elm
    fwd = (4 * NP + 12 * E + 4 * NS               # fan-in CSR + sink->driver
           + 32 * NP                              # source records (drivers / pull sources)
           + 4 * NS + 4 * NP                      # elm, load
           + 32 * P)                              # write AT + slew
    bwd = (8 * NP + 4 * P + 4 * NS + 8 * E        # sink ranges, endpoint map, fan-out CSR
           + 32 * P + 16 * NP + 4 * NP + 4 * NS   # records, rat of fan-out pins, load, elm
           + 16 * P + 16 * P + 8 * n_ep)          # write rat, slack, endpoint worst
    red = 8 * n_ep
    return dict(rc=rc, forward=fwd, backward=bwd, reduce=red)


def ncu_traffic(kernel):
    """DRAM bytes (read + write) of one launch of `kernel` from the committed
    `ncu --set full` summary of the current kernels (profiles/ncu_latest.json,
    written by scripts/ncu_summary.py), or None."""
    try:
        j = json.load(open(os.path.join(ROOT, "profiles", "ncu_latest.json")))
    except (OSError, ValueError):
        return None, None
    for name, k in j.get("kernels", {}).items():
        if name.startswith(kernel):
            return k["dram_bytes"], f"profiles/ncu_{j.get('tag')}.json"
    return None, None


class Clocks:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.t0 = None

    def start(self):
        self.t0 = time.time()
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self, since=None):
        """Stop sampling; keep the samples taken after wall time `since` (the
        start of the timed region), or the last one if none was."""
        if not self.p:
            return None
        t_stop = time.time()
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 8]
        if since is not None and rows and self.t0:
            # samples are -lms 20 apart, the first at about self.t0
            n_keep = max(1, int((t_stop - since) / 0.02) + 1)
            rows = rows[-n_keep:]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        mx = float(rows[0][2])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.strip() == "Active"})
        busy = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def run_reference(args, world, rank):
    """Reference arm: the fp64 oracle, as it stands, on the host cores."""
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    name = args.config or (CONFIG if world == 1 else "c5_multicorner")
    cfg = dict(synth.CONFIGS[name])
    scale = 10                                   # bounded sample: 1/10 of the cells
    cfg["n_cells"] //= scale
    cfg["corners"] = 1
    d = synth.generate(name=name, **cfg)
    d.cons.period = synth.recipe.lookup_period(name) or d.cons.period
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.update(d, 0, want_all=False)
        t1 = time.perf_counter()
        if i >= args.warmup:
            times.append(t1 - t0)
    ms = 1e3 * sum(times) / len(times)
    v = d.num_pins / (ms / 1e3)
    sample = (f"same recipe at 1/{scale} size: {d.num_pins} pins, one full oracle update per step, "
              "single thread fp64")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "pins/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{name} (sample)", "pins": d.num_pins},
            "cpu_baseline": {"value": v, "unit": "pins/s", "cores": 1, "host_cores": os.cpu_count(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "pins/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_line(name, info, K_local, world, gen_s, load_s):
    if name == "c5_multicorner":
        w = (f"{name}: BASELINE.json configs[4] multi-corner sign-off, 8 corners x ~2M-pin synthetic "
             f"design, {K_local} corner(s) per GPU traversed by the same launches, one NCCL all_reduce of "
             f"the per-corner WNS/TNS rows per step")
    else:
        w = (f"{name}: BASELINE.json configs[2] superblue-shaped synthetic netlist, one corner per GPU"
             if name == "c3_superblue" else f"{name} (synthetic, DESIGN.md §3)")
    return {"workload": w, "pins_per_corner": info["num_pins"], "corners_per_gpu": K_local,
            "pin_levels": info["num_levels"], "gate_stages": info["num_stages"],
            "cell_arcs": info["num_cell_arcs"], "net_arcs": info["num_net_arcs"],
            "endpoints": info["num_endpoints"], "heavy_drivers": info["num_heavy_drivers"],
            "parallelism": f"corners x{world}",
            "l2": "no flush: per-update working set > 1.5 GB >> 126 MB L2" if info["num_pins"] * K_local > 5e6
            else "no flush: the working set exceeds L2 only partly (small config)",
            "gen_s": round(gen_s, 1), "load_graph_s": round(load_s, 2)}


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    import torch.distributed as dist
    local = local % max(torch.cuda.device_count(), 1)   # ranks beyond the visible GPUs share them (gloo only)
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    import paper_2511_11660_b200 as pkg
    from paper_2511_11660_b200 import build as pbuild
    from paper_2511_11660_b200 import multicorner as mc
    pbuild.build()
    name = args.config or (CONFIG if world == 1 else "c5_multicorner")

    # one dedicated stream carries the STA kernels, the NCCL allreduce and the
    # timing events (the legacy default stream cannot be shared by handle)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    t0 = time.perf_counter()
    if name == "c5_multicorner":
        import synth
        d = synth.config_design(name)            # all 8 corners; this rank loads its share
        mine = list(mc.corners_of_rank(d.num_corners, rank, world))
        K_total = d.num_corners
    else:
        d = corner_design(name, rank)            # one corner per rank (weak scaling)
        mine = [0]
        K_total = world
    gen_s = time.perf_counter() - t0
    K = len(mine)
    ctx = pkg.Context(local, K, stream=stream.cuda_stream)
    t0 = time.perf_counter()
    if args.case:
        d.case = bench_case(d)
    if args.through:
        d.exceptions = bench_through(d)
    elif args.exceptions:
        d.exceptions = bench_exceptions(d)
    pkg.load_design(ctx, d, corners=mine)
    if args.net_model != "elmore":
        ctx.set_net_model(args.net_model, 4)
    torch.cuda.synchronize()
    load_s = time.perf_counter() - t0
    # inputs resident in HBM for the device-timed value: borrowed RC tensors
    res_d = [torch.from_numpy(d.rc[c].res).cuda() for c in mine]
    cap_d = [torch.from_numpy(d.rc[c].cap).cuda() for c in mine]
    for k in range(K):
        ctx.set_rc_values(k, res_d[k], cap_d[k])
    rows = torch.zeros((K_total, 4), dtype=torch.float64, device="cuda")
    row0 = mine[0] if name == "c5_multicorner" else rank

    def step():
        ctx.update_timing()
        if world > 1:
            rows.zero_()
            for k in range(K):
                ctx.report_wns_tns_device(k, rows[row0 + k])
            mc.combine_rows(rows)          # one NCCL allreduce of the per-corner rows

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the clock sampler starts before the warm-up so that it is running (not
    # still spawning) during the timed region
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    for _ in range(max(args.warmup, 3) if args.warmup else 0):
        step()
    barrier()
    tc0 = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    clk = clocks.stop(since=tc0)
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    info = ctx.info()
    P = info["num_pins"]
    total_pins = P * (K_total if name == "c5_multicorner" else world)
    value = total_pins / (ms / 1e3)
    res_own = [ctx.report_slack(k)[0] for k in range(K)]
    res_global = None
    if world > 1 or K > 1:
        full = torch.zeros((K_total, 4), dtype=torch.float64)
        for k in range(K):
            full[row0 + k] = torch.from_numpy(res_own[k])
        if world > 1:
            full = full.cuda()
            mc.combine_rows(full)
        res_global = [float(x) for x in mc.global_report(full.cpu())]

    line = {"metric": METRIC, "value": value, "unit": "pins/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if name == "c5_multicorner" else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(config_line(name, info, K, world, gen_s, load_s), net_model=args.net_model,
                           exceptions=bool(args.exceptions or args.through), through=bool(args.through), case_constants=int(len(d.case.pin)) if args.case else 0, dist_backend=args.dist_backend if world > 1 else None),
            "gpu_launches": info["kernels_per_update"] * args.steps,
            "clocks": clk, "wns_tns": [float(x) for x in res_own[0]]}
    if name == "c5_multicorner":
        line["corner_updates_per_s"] = K_total / (ms / 1e3)
    if res_global:
        line["wns_tns_global"] = res_global

    if not args.quick or args.phases:
        # roofline: per-phase device time with CUDA events on the ctx stream
        ctx.profile_enable(True)
        for _ in range(min(args.steps, 10)):
            ctx.update_timing()
        prof = ctx.profile_read()
        ctx.profile_enable(False)
        nu = max(prof["updates"], 1)
        ph_ms = {k: v / nu for k, v in prof["ms"].items()}
        ab = {k: v * K for k, v in algorithmic_bytes(d, info).items()}
        peak, peak_src = measured_peaks()
        dom = max(("forward", "backward"), key=lambda k: ph_ms[k])
        ach = ab[dom] / (ph_ms[dom] / 1e3) / 1e9
        kern = {"forward": "fwd_persistent_kernel", "backward": "bwd_persistent_kernel"}[dom]
        traffic, tsrc = ncu_traffic(kern)
        line["roofline"] = {"bound": "hbm", "kernel": kern, "achieved": ach,
                            "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                            "traffic_source": tsrc, "peak_source": peak_src, "algorithmic_bytes": ab[dom],
                            "kernel_ms": ph_ms[dom]}
        line["phases_ms"] = ph_ms
        line["phases_gbs"] = {k: ab[k] / (ph_ms[k] / 1e3) / 1e9 for k in ab if ph_ms.get(k, 0) > 0}
        whole = sum(ab.values())
        line["update_model_bytes"] = whole
        line["update_frac_hbm"] = whole / (ms / 1e3) / 1e9 / peak

    if not args.quick:
        # e2e through the public C ABI with HOST buffers: per step the RC
        # values of every local corner (the per-iteration inputs of an
        # optimization loop) go host -> device from page-locked memory
        # (sta_set_rc_values, STA_MEM_HOST), then the update, then the
        # WNS/TNS rows device -> host (sta_report_slack, STA_MEM_HOST)
        res_h = [torch.from_numpy(d.rc[c].res).pin_memory() for c in mine]
        cap_h = [torch.from_numpy(d.rc[c].cap).pin_memory() for c in mine]

        # An optimization loop pipelines its iterations through the ABI: the
        # next step's values are handed over (and copied, on the ctx's copy
        # stream, into the buffer pair the running update does not read)
        # while this step's update runs, then this step's result is read.
        # Every timed step still moves its own inputs H2D and its result D2H.
        def put(i):
            for k in range(K):
                ctx.set_rc_values(k, res_h[k].numpy(), cap_h[k].numpy())

        def e2e_steps(n):
            put(0)
            for i in range(n):
                ctx.update_timing()
                if i + 1 < n:
                    put(i + 1)                 # step i+1's H2D beside step i's update
                [ctx.report_slack(k)[0] for k in range(K)]

        e2e_steps(2)
        # the link alone (context for E: the pipelined step is bound by
        # max(update, this copy)): one HOST hand-over, host-timed
        torch.cuda.synchronize()
        t_h = time.perf_counter()
        for _ in range(3):
            put(0)
        h2d_ms = (time.perf_counter() - t_h) / 3 * 1e3
        barrier()
        e0.record(stream)
        e2e_steps(args.steps)
        e1.record(stream)
        barrier()
        ms_e2e = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ms_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
        line["e2e"] = {"value": total_pins / (ms_e2e / 1e3), "unit": "pins/s",
                       "h2d_bytes_per_step": int(sum(x.numel() * 4 for x in res_h + cap_h)),
                       "d2h_bytes_per_step": 32 * K, "ms_per_step": ms_e2e,
                       "h2d_alone_ms": h2d_ms,
                       "h2d_alone_gbs": sum(x.numel() * 4 for x in res_h + cap_h) / (h2d_ms / 1e3) / 1e9,
                       "path": "sta_set_rc_values(STA_MEM_HOST, page-locked; step i+1's copy beside "
                               "step i's update) + sta_update_timing + sta_report_slack(STA_MEM_HOST)"}
        for k in range(K):
            ctx.set_rc_values(k, res_d[k], cap_d[k])

    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        ref = oracle.update(d, mine[0], want_all=False)
        cpu_s = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": P / cpu_s, "unit": "pins/s", "cores": 1,
                                "host_cores": os.cpu_count(),
                                "affinity_cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                                "sample": f"one full update of corner {mine[0]} of the same {P}-pin design, fp64, "
                                          f"single thread ({cpu_s:.1f} s) on a host with {os.cpu_count()} cores"}
        r = ref["res"]
        line["parity_wns_tns"] = {"oracle": [float(x) for x in r],
                                  "abs_err": [float(abs(a - b)) for a, b in zip(res_own[0], r)]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
