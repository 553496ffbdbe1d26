"""Summarize an STA_TRACE dump: per stage, when its chunks started / became
ready / ended (relative to the first chunk), forward and backward."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(open(sys.argv[1])))
for kind in ("fwd", "bwd"):
    rs = [r for r in rows if r["kind"] == kind and int(r["end"]) > 0]
    if not rs:
        continue
    t0 = min(int(r["start"]) for r in rs)
    by = defaultdict(list)
    for r in rs:
        by[int(r["stage"])].append(r)
    print(f"== {kind}: {len(rs)} items, span {(max(int(r['end']) for r in rs) - t0) / 1e3:.1f} us")
    order = sorted(by) if kind == "fwd" else sorted(by, reverse=True)
    prev_end = None
    for s in order:
        g = by[s]
        st = min(int(r["start"]) for r in g) - t0
        rd = max(int(r["ready"]) for r in g) - t0 if kind == "fwd" else 0
        en = max(int(r["end"]) for r in g) - t0
        dur = [(int(r["end"]) - int(r["start"])) / 1e3 for r in g]
        print(f"  stage {s:3d} n={len(g):5d} first_start={st / 1e3:8.1f} last_ready={rd / 1e3:8.1f} "
              f"last_end={en / 1e3:8.1f} item_us max={max(dur):6.1f} mean={sum(dur) / len(dur):6.1f}")

# per unit type (backward: 0 light tile, 1 heavy tile, 2 sink-less pins)
by_t = defaultdict(list)
for r in rows:
    if r["kind"] == "bwd" and int(r["end"]) > 0:
        by_t[(int(r["stage"]) == 0, r.get("type", "0"))].append((int(r["end"]) - int(r["start"])) / 1e3)
for k in sorted(by_t):
    v = by_t[k]
    print(f"bwd stage0={k[0]} type={k[1]}: n={len(v)} mean={sum(v) / len(v):.2f} us max={max(v):.1f} us")

# phases of the units of each stage: start -> producers seen (forward probe /
# backward: fan-out record loaded), -> inputs loaded and computed, -> end
import statistics
for kind in ("fwd", "bwd"):
    fw = defaultdict(list)
    for r in rows:
        if r["kind"] == kind and int(r["end"]) > 0 and "data" in r and int(r["data"]) >= int(r["ready"]):
            fw[int(r["stage"])].append(r)
    print(f"{kind} phases per stage: median (max) of ready-start, data-ready, end-data  [us]")
    order = sorted(fw) if kind == "fwd" else sorted(fw, reverse=True)
    for s in order:
        g = fw[s]
        a = [(int(r["ready"]) - int(r["start"])) / 1e3 for r in g]
        b = [(int(r["data"]) - int(r["ready"])) / 1e3 for r in g]
        e = [(int(r["end"]) - int(r["data"])) / 1e3 for r in g]
        print(f"  {s:3d} n={len(g):6d} wait={statistics.median(a):6.2f} ({max(a):6.2f}) load={statistics.median(b):5.2f} "
              f"({max(b):5.2f}) compute={statistics.median(e):5.2f} ({max(e):5.2f})")

# gaps between consecutive units of one warp (warp w runs units w, w + W, ...)
# STA_TRACE_W = "fwd_warps,bwd_warps" (grid blocks x 8)
import os
if os.environ.get("STA_TRACE_W"):
    wf, wb = (int(x) for x in os.environ["STA_TRACE_W"].split(","))
    for kind, W in (("fwd", wf), ("bwd", wb)):
        rs = [r for r in rows if r["kind"] == kind]
        idx = {int(r["index"]): r for r in rs}
        gaps = defaultdict(list)
        for u, r in idx.items():
            nx = idx.get(u + W)
            if nx and int(nx["start"]) > 0 and int(r["end"]) > 0:
                gaps[int(nx["stage"])].append((int(nx["start"]) - int(r["end"])) / 1e3)
        print(f"{kind} gap before a unit (us), by the unit's stage: median / p90 / max")
        for s in sorted(gaps)[:: 5 if kind == "fwd" else 1][:40]:
            g = sorted(gaps[s])
            print(f"  {s:3d} n={len(g):6d} {g[len(g) // 2]:6.2f} {g[int(len(g) * 0.9)]:6.2f} {g[-1]:7.2f}")
