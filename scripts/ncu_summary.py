"""Summarize ncu --set full reports (+ a launch-list CSV) into a markdown
file and a JSON of per-kernel DRAM traffic for bench.py's roofline.traffic.

  python scripts/ncu_summary.py TAG launches.csv rep1.ncu-rep [rep2 ...]
  -> profiles/ncu_TAG.md, profiles/ncu_TAG.json
"""
import csv
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import launches  # noqa: E402

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "registers/thread"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    return [{k: (uu, v) for k, uu, v in zip(h, u, row)} for row in r[2:]]


def num(x):
    return float(x.replace(",", ""))


def main():
    args = [a for a in sys.argv[1:] if a != "--latest"]
    tag, lcsv, reps = args[0], args[1], args[2:]
    md = [f"# ncu summary {tag}", ""]
    js = {"tag": tag, "kernels": {}}
    if lcsv and os.path.exists(lcsv):
        data = launches.load(lcsv)
        tot, cnt = {}, {}
        for n, v, _ in data:
            tot[n] = tot.get(n, 0) + v
            cnt[n] = cnt.get(n, 0) + 1
        # sta_load_graph's device levelizer (row a0) runs once per design;
        # the update shares are taken over the update kernels only
        load = lambda n: n.startswith("k_") or n.startswith("scan_") or n in (
            "init_corner_kernel", "set_ptrs_kernel") or n.startswith("array<")
        upd = {n: v for n, v in tot.items() if not load(n)}
        allu = sum(upd.values()) or 1.0
        md += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, serialised, cold)", "",
               "Per-update kernels (share of the update kernels' time):", "",
               "| kernel | launches | avg us | share of update |", "|---|---|---|---|"]
        for n in sorted(upd, key=lambda k: -upd[k]):
            md.append(f"| {n} | {cnt[n]} | {tot[n] / cnt[n]:.2f} | {tot[n] / allu:.1%} |")
        md += ["", "Once per design (`sta_load_graph`: device levelizer / CSR builder, setup):", "",
               "| kernel | launches | avg us | total us |", "|---|---|---|---|"]
        for n in sorted((n for n in tot if load(n)), key=lambda k: -tot[k]):
            md.append(f"| {n} | {cnt[n]} | {tot[n] / cnt[n]:.2f} | {tot[n]:.1f} |")
        js["launch_share"] = {n: upd[n] / allu for n in upd}
        md.append("")
    for rep in reps:
        for row in raw(rep):
            name = row["Kernel Name"][1].split("(")[0].split("::")[-1]
            md += [f"## `{name}` (`--set full`, {os.path.basename(rep)})", "", "| metric | value |", "|---|---|"]
            k = {}
            for key, label in KEYS:
                if key in row:
                    u, v = row[key]
                    md.append(f"| {label} (`{key}`) | {v} {u} |")
                    k[key] = (u, v)
            stalls = sorted(((num(v), key) for key, (u, v) in row.items()
                             if key.startswith("smsp__pcsamp_warps_issue_stalled_") and not key.endswith("not_issued")
                             and v.replace(",", "").replace(".", "").isdigit()), reverse=True)
            tot_s = sum(s for s, _ in stalls) or 1
            md += ["", "Top warp stall reasons (pc sampling):", ""]
            for s, key in stalls[:8]:
                md.append(f"- {key.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {s / tot_s:.1%}")
            md.append("")
            u_r, v_r = k["dram__bytes_read.sum"]
            u_w, v_w = k["dram__bytes_write.sum"]
            u_t, v_t = k["gpu__time_duration.sum"]
            js["kernels"][name] = {"dram_bytes": num(v_r) * UNIT[u_r] + num(v_w) * UNIT[u_w],
                                   "duration_us": num(v_t) * (1e-3 if u_t.startswith("n") else 1.0),
                                   "l2_hit_pct": num(k["lts__t_sector_hit_rate.pct"][1])}
    os.makedirs("profiles", exist_ok=True)
    open(f"profiles/ncu_{tag}.md", "w").write("\n".join(md) + "\n")
    json.dump(js, open(f"profiles/ncu_{tag}.json", "w"), indent=1)
    if "--latest" in sys.argv:
        json.dump(js, open("profiles/ncu_latest.json", "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
