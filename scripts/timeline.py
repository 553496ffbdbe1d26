"""Kernel timeline of a few graph-launched updates (CUPTI via torch.profiler):
per-kernel mean duration and the update's critical path, with concurrency
(the ncu launch list serialises kernels; this does not).

  python scripts/timeline.py [config] [updates]     (on the GPU box)
"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2511_11660_b200 as sta  # noqa: E402
import synth  # noqa: E402


def kname(e):
    return e.name.replace("(anonymous namespace)::", "").split("(")[0].split("::")[-1][:40]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3_superblue"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    d = synth.config_design(name, corners=1)
    stream = torch.cuda.Stream()
    ctx = sta.Context(0, 1, stream=stream.cuda_stream)
    sta.load_design(ctx, d)
    for _ in range(3):
        ctx.update_timing()
    ctx.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            ctx.update_timing()
        ctx.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time > 0]
    ev = [e for e in ev if "Memcpy" not in e.name and "Memset" not in e.name]
    ev.sort(key=lambda e: e.time_range.start)
    dur = collections.defaultdict(list)
    for e in ev:
        dur[kname(e)].append(e.time_range.end - e.time_range.start)
    print(f"{name}: {len(ev)} kernels over {n} updates")
    for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:40s} n={len(v):4d} mean={sum(v) / len(v):9.1f} us")
    # first update: start offsets relative to its first kernel
    per = len(ev) // n
    t0 = ev[0].time_range.start
    print("first update (start, end relative, us):")
    for e in ev[:per]:
        print(f"  {kname(e):40s} {e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}")
    ctx.close()


if __name__ == "__main__":
    main()
