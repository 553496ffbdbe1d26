"""Per-unit timeline of the persistent kernels on one config (GPU box):
STA_TRACE dump of the 3rd update, then scripts/trace_report.py.

  python scripts/trace_run.py [config] [out.csv]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
name = sys.argv[1] if len(sys.argv) > 1 else "c3_superblue"
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"trace_{name}.csv")
os.environ["STA_TRACE"] = out

import paper_2511_11660_b200 as sta  # noqa: E402
import synth  # noqa: E402

d = synth.config_design(name, corners=1)
ctx = sta.Context(0, 1)
sta.load_design(ctx, d)
for _ in range(3):
    ctx.update_timing()
ctx.synchronize()
ctx.close()
subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "trace_report.py"), out])
