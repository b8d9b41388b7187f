"""Multi-rank host logic on CPU: world_size 2 over gloo (no GPU).

Each rank takes its batch shard with the same helpers bench.py uses (shard.py), generates
its slice of the global seeded batch, computes it (the oracle stands in for the device conv
here -- this test exercises the sharding, not the kernels), then:
  * the gathered shards equal the unsharded result bit for bit (P11 on the host path);
  * rank 0's algorithm choices (and tuned variants) win on every rank (broadcast_choices);
  * max_over_ranks returns the slowest rank's time.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1904_04174_b200 import synth
from paper_1904_04174_b200.shard import broadcast_choices, gather_shards, max_over_ranks, shard_range

GB, H, W, C, F, K, S = 4, 9, 7, 5, 6, 3, 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b0, b1 = shard_range(GB, world, rank)
        x = synth.input_nhwc(b1 - b0, H, W, C, layer_id=31, batch_offset=b0)
        w = synth.filter_hwcf(K, K, C, F, layer_id=31)
        y = O.conv2d(O.Params(b1 - b0, H, W, C, F, K, K, S, S, O.SAME), x, w, threads=1)
        full = gather_shards(torch.from_numpy(y), dist)
        choices = broadcast_choices({"R4": 3 + rank, "R17": 4 - rank}, dist, "cpu")
        pairs = broadcast_choices({"R4": (3 + rank, 17 * rank), "R17": (4 - rank, 8)}, dist, "cpu")
        tmax = max_over_ranks(10.0 + rank, dist, "cpu")
        out[rank] = (full.numpy(), choices, pairs, tmax)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_gather_bitwise():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    xg = synth.input_nhwc(GB, H, W, C, layer_id=31)
    wg = synth.filter_hwcf(K, K, C, F, layer_id=31)
    ref = O.conv2d(O.Params(GB, H, W, C, F, K, K, S, S, O.SAME), xg, wg, threads=1)
    for r in range(world):
        full, choices, pairs, tmax = out[r]
        assert np.array_equal(full, ref)
        assert choices == {"R4": 3, "R17": 4}  # rank 0's
        assert pairs == {"R4": (3, 0), "R17": (4, 8)}  # (algorithm, variant) pairs: rank 0's
        assert tmax == 11.0


def test_shard_range():
    assert [shard_range(256, 8, r) for r in (0, 7)] == [(0, 32), (224, 256)]
    assert shard_range(256, 1, 0) == (0, 256)
    with pytest.raises(ValueError):
        shard_range(256, 3, 0)
    with pytest.raises(ValueError):
        shard_range(256, 2, 2)
