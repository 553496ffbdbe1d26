"""N > 1 path on CPU (gloo, world_size 2): corner sharding and the single
all_reduce of per-corner WNS/TNS rows give the oracle's global report."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2511_11660_b200 import multicorner as mc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = synth.generate(600, 14, seed=21, corners=5, corner_recipe="c5", period=140.0)
        rows = torch.zeros((d.num_corners, 4), dtype=torch.float64)
        for c in mc.corners_of_rank(d.num_corners, rank, world):
            rows[c] = torch.tensor(oracle.update(d, c, want_all=False)["res"], dtype=torch.float64)
        mc.combine_rows(rows)
        out[rank] = list(mc.global_report(rows)) + rows.flatten().tolist()
    finally:
        dist.destroy_process_group()


def test_corner_sharding_covers_every_corner_once():
    for K in range(1, 10):
        for G in range(1, 9):
            owned = [c for r in range(G) for c in mc.corners_of_rank(K, r, G)]
            assert owned == list(range(K))


def test_two_rank_allreduce_matches_oracle_global():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    d = synth.generate(600, 14, seed=21, corners=5, corner_recipe="c5", period=140.0)
    per, glob = oracle.update_all_corners(d)
    a, b = out[0], out[1]
    assert a == b                                  # identical on every rank
    assert a[0] == glob[0] and a[2] == glob[2]     # WNS: min over corners (exact)
    assert a[1] == pytest.approx(glob[1], rel=1e-12) and a[3] == pytest.approx(glob[3], rel=1e-12)
    rows = np.array(a[4:]).reshape(-1, 4)
    for c in range(d.num_corners):                 # every corner's row, exactly once
        assert np.array_equal(rows[c], np.asarray(per[c]["res"], dtype=np.float64))
