"""Sharded all_magnitudes over 2 ranks with the gloo backend.

CPU test (`-m "not gpu"`): the per-rank compute is the CPU oracle, so what
is under test is the host-side partition and the gather.  GPU test: the same
two-rank flow through the PRODUCT shard path (device kernels per rank, rows
gathered over gloo).  Either way every rank's row block, gathered, must
reproduce the single-process result bit for bit, for even and ragged n.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2002_04989_b200.shard import gather_rows, rows_per_rank, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    a = orc.random_symmetric(21, n)
    lam = orc.eigenvalues(a)                       # redundant per rank
    j0, j1 = shard_range(n, world, rank)
    mu = orc.minor_spectra(a, list(range(j0, j1)), threads=1)
    rows = orc.identity_rows(lam, mu, threads=1)   # rows j0..j1-1
    full = gather_rows(torch.from_numpy(rows), n, world, dist)
    if rank == 0:
        q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [12, 13])
def test_gloo_two_rank_gather_is_bit_identical(n):
    from oracle.oracle import Oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = Oracle().all_magnitudes(Oracle().random_symmetric(21, n))
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_shard_ranges_cover_every_minor_once():
    for n in (1, 7, 64, 4096):
        for world in (1, 2, 3, 4, 8):
            cover = []
            for r in range(world):
                j0, j1 = shard_range(n, world, r)
                cover.extend(range(j0, j1))
            assert cover == list(range(n))
            assert max(rows_per_rank(n, world)) - min(rows_per_rank(n, world)) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _gpu_worker(rank, world, port, n, q):
    """One rank of the product's shard path: the device pipeline for this
    rank's minors (eigenid_gpu_all_magnitudes_device on the library stream),
    rows gathered with the host (gloo) collective."""
    import torch.distributed as dist

    from paper_2002_04989_b200 import IdentityEngine, random_symmetric
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = IdentityEngine()
    a = torch.from_numpy(random_symmetric(23, n)).cuda()
    j0, j1 = shard_range(n, world, rank)
    out = torch.empty((j1 - j0, n), dtype=torch.float64, device="cuda")
    eng.all_magnitudes_device(a.data_ptr(), n, j0, j1, out.data_ptr())
    eng.sync()
    full = gather_rows(out.cpu(), n, world, dist)
    if rank == 0:
        q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [96, 301])
def test_two_rank_product_shard_path_is_bit_identical(n):
    """world_size 2 through the PRODUCT shard path (device kernels per rank,
    independent of each other; the rows meet only in the host gather): the
    gathered matrix equals the single-process all_magnitudes bit for bit, for
    an even and a ragged split."""
    from paper_2002_04989_b200 import IdentityEngine, random_symmetric
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = IdentityEngine().all_magnitudes(random_symmetric(23, n)).reshape(n, n)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
