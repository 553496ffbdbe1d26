"""Summarize an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                u = d["Metric Unit"]
                v *= {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
                data.append((d["Kernel Name"].split("(")[0].split("::")[-1], v, d["Grid Size"]))
    return data


if __name__ == "__main__":
    data = load(sys.argv[1])
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for n, v, _ in data:
        tot[n] += v
        cnt[n] += 1
    allt = sum(tot.values())
    for n in sorted(tot, key=lambda k: -tot[k]):
        print(f"{n:28s} n={cnt[n]:5d} total={tot[n]:10.1f} us avg={tot[n] / cnt[n]:8.2f} us share={tot[n] / allt:6.1%}")
    if "-v" in sys.argv:
        for n, v, g in data:
            print(f"  {n:24s} {v:9.2f} us grid={g}")
