"""Seeded synthetic pin placement for the Steiner RC row.

Input generator only (no RC arithmetic): each net gets a centre uniform in a
square die and its pins scattered uniformly in a box around it whose side
grows with the square root of the net's pin count -- net bounding boxes like
a placed design's, cell geometry ignored (every pin belongs to at most one
net, so the nets are placed independently).  `grid=True` rounds positions to
integers, which makes equal Manhattan distances (Prim ties) common.  Pins on
no net are placed at the die centre.  DESIGN.md §3 states the recipe.
"""
from __future__ import annotations

import numpy as np

# unit R / C per distance unit (x, y): kOhm and fF, roughly a lower metal
# layer pair with distance units of 1 um
UNITS = dict(res_x=0.0008, res_y=0.001, cap_x=0.16, cap_y=0.18)


def placement(d, seed: int = 1, die: float | None = None, pitch: float = 3.0, grid: bool = False):
    """-> (x, y) float32 [P] pin positions for design d."""
    rng = np.random.default_rng(seed)
    P = d.num_pins
    net_ptr = np.asarray(d.net_ptr, np.int64)
    N = net_ptr.size - 1
    m = np.diff(net_ptr)
    if die is None:
        die = 4.0 * np.sqrt(max(P, 1))
    x = np.full(P, die / 2, np.float64)
    y = np.full(P, die / 2, np.float64)
    if N:
        cx = rng.uniform(0, die, N)
        cy = rng.uniform(0, die, N)
        half = 0.5 * pitch * np.sqrt(m) + pitch
        net_of = np.repeat(np.arange(N), m)
        pins = np.asarray(d.net_pins, np.int64)
        x[pins] = np.clip(cx[net_of] + rng.uniform(-1, 1, pins.size) * half[net_of], 0, die)
        y[pins] = np.clip(cy[net_of] + rng.uniform(-1, 1, pins.size) * half[net_of], 0, die)
    if grid:
        x, y = np.round(x), np.round(y)
    return x.astype(np.float32), y.astype(np.float32)
