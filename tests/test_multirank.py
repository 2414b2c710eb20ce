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
