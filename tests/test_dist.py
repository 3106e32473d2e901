"""World-size-2 gloo test of the multi-GPU host logic (CPU only): scan
ownership, max-over-ranks timing and the detection gather used by bench.py
under torchrun."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1709_02549_b200 import shard, synth


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world_size, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        assert shard.world() == (rank, world_size)
        seeds = shard.scan_block(rank, world_size, 3)
        model = synth.ScanModel(n_samples=256)
        _, tumours = synth.batch_2d(model, seeds)
        grid = synth.grid_square(0.12, 64)
        cells = np.array([grid.point_to_cell(*t) for t in tumours])
        rows = shard.gather_detections(seeds, cells)
        t = shard.max_over_ranks(10.0 + rank)
        total = shard.sum_over_ranks(len(seeds))
        if rank == 0:
            np.save(os.path.join(out_dir, "rows.npy"), rows)
            np.save(os.path.join(out_dir, "scalars.npy"), np.array([t, total]))
        else:
            assert rows is None
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    rows = np.load(tmp_path / "rows.npy")
    t, total = np.load(tmp_path / "scalars.npy")
    assert rows[:, 0].tolist() == list(range(6))  # every scan exactly once, in order
    model = synth.ScanModel(n_samples=256)
    _, tumours = synth.batch_2d(model, range(6))
    grid = synth.grid_square(0.12, 64)
    assert rows[:, 1:].tolist() == [list(grid.point_to_cell(*x)) for x in tumours]
    assert t == 11.0 and total == 6


def test_split_helpers():
    assert [list(shard.split_scans(10, r, 3)) for r in range(3)] == [[0, 1, 2, 3], [4, 5, 6], [7, 8, 9]]
    assert list(shard.scan_block(1, 4, 5)) == [5, 6, 7, 8, 9]
    with pytest.raises(ValueError):
        shard.scan_block(4, 4, 5)
    assert shard.max_over_ranks(3.5) == 3.5
