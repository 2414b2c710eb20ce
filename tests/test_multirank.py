"""N>1 host logic on CPU (gloo, world_size 2): image sharding covers the batch
exactly once and the uint16 histogram gather reassembles the per-image
histograms bit-exactly in image order. The per-shard histograms come from the
CPU oracle, standing in for each rank's kernel output."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_11518_b200.shard import gather_histograms, shard_range, widen, wire_dtype_ok


def test_shard_ranges_tile_the_batch():
    for n in (0, 1, 7, 64, 65536, 1000003):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_wire_width():
    assert wire_dtype_ok(81 * 91) and wire_dtype_ok(65535) and not wire_dtype_ok(65536)
    t = torch.tensor([0, 1, 7371, 40000, 65535], dtype=torch.int32)
    assert torch.equal(widen([t.to(torch.int16)]), t.to(torch.int64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, images, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    lo, hi = shard_range(images.shape[0], rank, world)
    _, h = oracle.batch(images[lo:hi], k=3, cell=(8, 9), codes=False, threads=1)
    shards = gather_histograms(torch.from_numpy(h.astype(np.int32)), dist, rank, world)
    if rank == 0:
        np.save(result_path, widen(shards).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_two_ranks(tmp_path):
    rng = np.random.default_rng(0)
    images = rng.integers(0, 256, size=(6, 24, 27), dtype=np.uint8)
    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), images, out), nprocs=2, join=True)
    import oracle
    _, want = oracle.batch(images, k=3, cell=(8, 9), codes=False)
    got = np.load(out)
    assert got.shape == want.shape
    assert np.array_equal(got.astype(np.uint64), want)


def _chunked_worker(rank, world, port, images, result_path, n_chunks):
    """bench.py's overlapped gather: each chunk of the shard is gathered into
    views of rank 0's per-rank receive buffers."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    lo, hi = shard_range(images.shape[0], rank, world)
    _, h = oracle.batch(images[lo:hi], k=3, cell=(8, 9), codes=False, threads=1)
    hist = torch.from_numpy(h.astype(np.int32))
    mine = hi - lo
    wire = torch.empty(hist.shape, dtype=torch.int16)
    gathered = [torch.empty_like(wire) for _ in range(world)] if rank == 0 else None
    for c in range(n_chunks):
        a, b = mine * c // n_chunks, mine * (c + 1) // n_chunks
        gather_histograms(hist[a:b], dist, rank, world, wire=wire[a:b],
                          out=[g[a:b] for g in gathered] if rank == 0 else None)
    if rank == 0:
        np.save(result_path, widen(gathered).numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_chunks", [1, 3])
def test_chunked_gather_two_ranks(tmp_path, n_chunks):
    rng = np.random.default_rng(1)
    images = rng.integers(0, 256, size=(8, 20, 30), dtype=np.uint8)
    out = str(tmp_path / "chunked.npy")
    mp.spawn(_chunked_worker, args=(2, _free_port(), images, out, n_chunks), nprocs=2, join=True)
    import oracle
    _, want = oracle.batch(images, k=3, cell=(8, 9), codes=False)
    assert np.array_equal(np.load(out).astype(np.uint64), want)


def _single_rank_worker(rank, world, port, result_path):
    """World size 1 with an initialised group still goes through dist.gather."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    h = torch.arange(2 * 3 * 4, dtype=torch.int32).view(2, 3, 4)
    out = gather_histograms(h, dist, 0, 1)
    np.save(result_path, widen(out).numpy())
    dist.destroy_process_group()


def test_gather_world_one_initialised(tmp_path):
    out = str(tmp_path / "one.npy")
    mp.spawn(_single_rank_worker, args=(1, _free_port(), out), nprocs=1, join=True)
    assert np.array_equal(np.load(out), np.arange(24).reshape(2, 3, 4))
