"""World-size-2 gloo tests of the multi-GPU host logic: the
column partition, the equal-count slab all-gather that assembles K̂ and the
scenario partition.  The slabs are oracle K̂ columns on CPU tensors, so the
assembled matrix must equal the oracle's bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_11875_b200.dist import allgather_columns, column_partition, scenario_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, n_u, _ = K.shape
        col0, ncols, c = column_partition(n_u, world, rank)
        slab = torch.zeros(S, c, n_u, dtype=torch.float64)
        slab[:, :ncols] = torch.from_numpy(K[:, col0:col0 + ncols])   # "this rank's HVPs"
        full = allgather_columns(slab, n_u)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_u", [(2, 107), (2, 5), (3, 10)])
def test_allgather_columns_assembles_khat(world, n_u):
    rng = np.random.default_rng(n_u)
    K = rng.standard_normal((2, n_u, n_u))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, full in out:
        assert np.array_equal(full, K), rank


def test_partitions_cover_exactly_once():
    for n_u in (1, 5, 107, 519, 1019, 2889):
        for world in (1, 2, 3, 4, 8):
            for align in (8, 16, 64):
                cols = []
                for r in range(world):
                    c0, n, c = column_partition(n_u, world, r, align)
                    assert n <= c and c % align == 0
                    assert n == 0 or c0 % align == 0   # every rank starts a canonical tile
                    cols += list(range(c0, c0 + n))
                assert cols == list(range(n_u))
    for tot in (8, 64, 10):
        for world in (1, 2, 4, 8):
            got = []
            for r in range(world):
                f, n = scenario_partition(tot, world, r)
                got += list(range(f, f + n))
            assert got == list(range(tot))
