import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, synth, paper_2511_11660_b200 as sta
d = synth.config_design(sys.argv[1] if len(sys.argv) > 1 else "c3_superblue", corners=1)
ctx = sta.Context(0, 1)
sta.load_design(ctx, d)
ctx.update_timing(); ctx.synchronize()
for nw in (1, 8, 8, 8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = ctx.report_paths(0, "setup", k=1000, nworst=nw)
    print("nworst", nw, "ms", round((time.perf_counter() - t0) * 1e3, 2), len(g), flush=True)
