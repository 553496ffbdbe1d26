"""Multi-corner sign-off across ranks.

One process per GPU; rank r owns corners [r K / G, (r + 1) K / G) and runs
them through its own Context.  The only data-path collective of an update is
one all_reduce(SUM) of a [K][4] float64 table in which every rank filled only
the rows of its own corners (zeros elsewhere), so the sum is exact and every
rank ends with the same table; the global report is then WNS = min and TNS =
sum over corners (SURVEY §8(c) O9 / reading R20), computed identically on
every rank.  Host-side logic only: the per-corner rows come from
`Context.report_wns_tns_device` (device tensors, NCCL) or `report_slack`
(host, any backend).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def corners_of_rank(num_corners: int, rank: int, world: int) -> range:
    """Contiguous block of corners owned by `rank` (balanced, every corner once)."""
    return range(num_corners * rank // world, num_corners * (rank + 1) // world)


def combine_rows(rows, group=None):
    """all_reduce(SUM) of the [K][4] per-corner table (a torch tensor; each rank
    filled only its own corners' rows).  In place; returns the tensor."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=group)
    return rows


def global_report(rows) -> Tuple[float, float, float, float]:
    """{WNS_setup, TNS_setup, WNS_hold, TNS_hold} over corners: WNS = min, TNS
    = sum (O9), from the combined [K][4] table (tensor or nested sequence)."""
    r = rows.tolist() if hasattr(rows, "tolist") else [list(x) for x in rows]
    return (min(x[0] for x in r), sum(x[1] for x in r), min(x[2] for x in r), sum(x[3] for x in r))
