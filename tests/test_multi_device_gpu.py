"""Several GPUs in one process (aldp_ldp_batch_host_multi), the
uint16 histogram output, the launch counter and the negative control.

The multi-device entry point splits a batch into contiguous image ranges,
one persistent host worker per range; a device may repeat in the list, so the
sharding, threading and result assembly are exercised on a single B200 (and on
every visible device when there are several). Results must equal the
single-device host batch and the CPU oracle bit for bit."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1810_11518_b200 as aldp  # noqa: E402

DEV = torch.device("cuda:0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def faces_host(n, rows=490, cols=640, seed=21):
    d = aldp.gen_faces(n, rows, cols, blobs=12, seed=seed, device=DEV)
    torch.cuda.synchronize()
    return d[:, :, :cols].cpu().numpy()


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0], None])
@pytest.mark.parametrize("k,cell", [(3, (81, 91)), (3, (0, 0)), (5, (64, 64)), (0, (81, 91))])
def test_host_multi_matches_single_device(devices, k, cell):
    px = faces_host(37)  # not a multiple of the device count: uneven ranges
    want_c, want_h = aldp.ldp_batch_host(px, k=k, cell=cell)
    got_c, got_h = aldp.ldp_batch_host_multi(px, k=k, cell=cell, devices=devices)
    assert np.array_equal(got_c, want_c)
    assert np.array_equal(got_h, want_h)
    rc, rh = oracle.batch(px[:3], k=k, cell=cell)
    assert np.array_equal(got_c[:3], rc) and np.array_equal(got_h[:3].astype(np.uint64), rh)


def test_host_multi_all_visible_devices_and_small_batches():
    n_dev = torch.cuda.device_count()
    for n in (0, 1, 2, n_dev + 1):
        px = faces_host(max(n, 1))[:n]
        c, h = aldp.ldp_batch_host_multi(px, k=3, cell=(81, 91), devices=list(range(n_dev)) * 2)
        if n:
            want_c, want_h = aldp.ldp_batch_host(px, k=3, cell=(81, 91))
            assert np.array_equal(c, want_c) and np.array_equal(h, want_h)


def test_host_multi_errors():
    px = faces_host(2)
    with pytest.raises(aldp.AldpError):
        aldp.ldp_batch_host_multi(px, k=3, devices=[0, 1000])  # no such device
    with pytest.raises(ValueError):
        aldp.ldp_batch_host_multi(px, k=3, cell=(2, 2), devices=[0])
    c, h = aldp.ldp_batch_host_multi(px, k=3, devices=[0])  # the workers survive an error
    assert np.array_equal(c, aldp.ldp_batch_host(px, k=3)[0])


def test_hist_u16_output():
    px = aldp.gen_faces(9, 490, 640, blobs=20, seed=8, device=DEV)
    for k, cell in ((3, (81, 91)), (4, (64, 64)), (0, (81, 91)), (3, (100, 200))):
        nb = 256 if k == 0 else aldp.n_bins(k)
        cells = aldp.grid_cells(490, 640, *cell)
        h32 = torch.empty((9, cells, nb), dtype=torch.int32, device=DEV)
        h16 = torch.empty((9, cells, nb), dtype=torch.int16, device=DEV)
        for kern in ("auto", "generic"):
            aldp.ldp_batch(px, 490, 640, k=k, cell=cell, hist=h32, kernel=kern)
            aldp.ldp_batch(px, 490, 640, k=k, cell=cell, hist=h16, kernel=kern)
            torch.cuda.synchronize()
            assert torch.equal(h16.to(torch.int32) & 0xFFFF, h32), (k, cell, kern)
    with pytest.raises(ValueError):  # a whole-image histogram of 313,600 pixels cannot be uint16
        aldp.ldp_batch(px, 490, 640, k=3, hist=torch.empty((9, 1, 56), dtype=torch.int16, device=DEV))


def test_launch_count():
    px = aldp.gen_faces(4, 490, 640, seed=2, device=DEV)
    aldp.ldp_batch(px, 490, 640, k=3, codes=True, hist=True)
    assert aldp.last_launch_count() == 1
    aldp.ldp_batch(px, 490, 640, k=3, cell=(81, 91), codes=True, hist=True)  # 490 = 6 * 81 + 4: split
    assert aldp.last_launch_count() == 2
    aldp.ldp_batch(px, 490, 640, k=3, cell=(81, 91), codes=True, hist=True, kernel="generic")
    assert aldp.last_launch_count() == 1
    aldp.ldp_batch(px, 490, 640, k=3, cell=(70, 80), codes=True, hist=True)  # 490 = 7 * 70: one launch
    assert aldp.last_launch_count() == 1
    torch.cuda.synchronize()


def test_negative_control_is_detected():
    """With the fault injection on, the parity comparisons this suite makes
    fail -- on codes and on histograms, both kernels; off again, they pass."""
    px = aldp.gen_faces(3, 96, 160, blobs=6, seed=7, device=DEV)
    host = px[:, :, :160].cpu().numpy()
    rc, rh = oracle.batch(host, k=3, cell=(32, 40))
    old = aldp.debug_fault(1)
    try:
        for kern in ("fast", "generic"):
            c, h = aldp.ldp_batch(px, 96, 160, k=3, cell=(32, 40), codes=True, hist=True, kernel=kern)
            torch.cuda.synchronize()
            c, h = c[:, :, :160].cpu().numpy(), h.cpu().numpy().astype(np.uint64)
            assert not np.array_equal(c, rc), kern
            assert not np.array_equal(h, rh), kern
            assert int((c != rc).sum()) == 1 and int(np.abs(h.astype(np.int64) - rh.astype(np.int64)).sum()) == 1
    finally:
        aldp.debug_fault(old)
    c, h = aldp.ldp_batch(px, 96, 160, k=3, cell=(32, 40), codes=True, hist=True)
    torch.cuda.synchronize()
    assert np.array_equal(c[:, :, :160].cpu().numpy(), rc)
    assert np.array_equal(h.cpu().numpy().astype(np.uint64), rh)


def test_parity_suite_fails_under_fault_injection():
    """The negative control end to end: the GPU parity suite, run with
    ALDP_FAULT_INJECT=1, must fail."""
    env = dict(os.environ, ALDP_FAULT_INJECT="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_parity_gpu.py"), "-k",
                        "golden_fixtures or config1_digest or cell_histograms"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, r.stdout[-2000:]
    assert "failed" in r.stdout
