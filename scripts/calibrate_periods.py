"""Calibrate the clock period of each synthetic config with the ORACLE only.

Arrival times do not depend on the period, so one oracle update at a
placeholder period T0 gives each endpoint's required-adjusted arrival
need_e = T0 - ws_setup(e).  T = round(quantile_0.9(need_e)) makes ~10% of
the endpoints violate setup (SURVEY.md §8(d) asks for ~5-20%).  Results are
written to synth/periods.json and consumed by synth.recipe.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
from synth.recipe import CONFIGS, _PERIODS_FILE  # noqa: E402

T0 = 1.0e6


def main(names):
    out = {}
    if os.path.exists(_PERIODS_FILE):
        out = json.load(open(_PERIODS_FILE))
    for name in names:
        d = synth.config_design(name, corners=1, period=T0)
        r = oracle.update(d, 0, want_all=False)
        ws = r["ep_ws"][:, 0]
        need = T0 - ws[np.isfinite(ws)]
        T = float(np.round(np.quantile(need, 0.9)))
        viol = float(np.mean(need > T))
        out[name] = dict(period=T, endpoints=int(need.size), violating_frac=viol,
                         max_need=float(need.max()), method="oracle, quantile 0.9 of T0 - ws_setup")
        print(name, out[name], flush=True)
        json.dump(out, open(_PERIODS_FILE, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))
