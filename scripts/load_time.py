"""sta_load_graph / sta_set_rc_tree host phase times on a config (STA_TIMING=1).

    python scripts/load_time.py [config]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["STA_TIMING"] = "1"

import torch  # noqa: E402

import paper_2511_11660_b200 as sta  # noqa: E402
import synth  # noqa: E402

d = synth.config_design(sys.argv[1] if len(sys.argv) > 1 else "c3_superblue", corners=1)
ctx = sta.Context(0, 1)
for rep in range(2):
    t0 = time.perf_counter()
    sta.load_design(ctx, d)
    torch.cuda.synchronize()
    print("load_design total", round(time.perf_counter() - t0, 3), flush=True)
ctx.update_timing()
ctx.synchronize()
