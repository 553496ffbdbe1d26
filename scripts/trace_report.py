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
