"""Randomised parity on the B200: shapes, k, cell grids, pitches, descriptor
(LDP / LBP), cell rule and kernel drawn at random (seeded), every case
bit-exact against the CPU oracle (codes and histograms)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1810_11518_b200 as aldp  # noqa: E402

DEV = torch.device("cuda:0")


def _map_hist(codes, k, cr, cc):
    n, r, c = codes.shape
    gr, gc = r // cr, c // cc
    if k == 0:
        lut, nb = np.arange(256), 256
    else:
        ranks = [v for v in range(256) if bin(v).count("1") == k]
        lut = np.full(256, -1)
        lut[ranks] = np.arange(len(ranks))
        nb = len(ranks)
    out = np.zeros((n, gr * gc, nb), np.uint64)
    for i in range(n):
        for a in range(gr):
            for b in range(gc):
                out[i, a * gc + b] = np.bincount(lut[codes[i, a * cr:(a + 1) * cr, b * cc:(b + 1) * cc]].ravel(),
                                                 minlength=nb)
    return out


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("ALDP_FUZZ_SEEDS", "24"))))
def test_random_cases(seed):
    rng = np.random.default_rng(9000 + seed)
    for _ in range(8):
        n = int(rng.integers(1, 5))
        r, c = int(rng.integers(3, 140)), int(rng.integers(3, 300))
        k = int(rng.choice([0, 1, 2, 3, 4, 5, 6, 7]))
        if k == 4 and rng.random() < 0.5:
            k = 3
        pitch = int(rng.choice([c, (c + 7) // 8 * 8, (c + 15) // 16 * 16 + 16]))
        kind = rng.integers(0, 3)
        if kind == 0:
            px = rng.integers(0, 256, size=(n, r, c), dtype=np.uint8)
        elif kind == 1:
            px = rng.integers(0, 3, size=(n, r, c), dtype=np.uint8)  # ties
        else:
            px = np.full((n, r, c), rng.integers(0, 256), np.uint8)
            px[:, ::int(rng.integers(2, 7))] ^= np.uint8(rng.integers(1, 255))
        cell = (0, 0)
        if rng.random() < 0.6 and r >= 3 and c >= 3:
            cell = (int(rng.integers(3, r + 1)), int(rng.integers(3, c + 1)))
        clamp = bool(rng.random() < 0.8)
        kernel = str(rng.choice(["auto", "generic"]))
        buf = np.zeros((n, r, pitch), np.uint8)
        buf[:, :, :c] = px
        d = torch.from_numpy(buf).to(DEV)
        fn = aldp.lbp_batch if k == 0 else aldp.ldp_batch
        kw = {} if k == 0 else {"k": k}
        codes, hist = fn(d, r, c, cell=cell, codes=True, hist=True, kernel=kernel, cell_clamp=clamp, **kw)
        torch.cuda.synchronize()
        want_c, want_h = oracle.batch(px, k=k, cell=cell)
        case = (n, r, c, pitch, k, cell, clamp, kernel)
        assert np.array_equal(codes[:, :, :c].cpu().numpy(), want_c), case
        got_h = hist.cpu().numpy().astype(np.uint64)
        if cell != (0, 0) and not clamp:
            want_h = _map_hist(want_c, k, *cell)
        assert np.array_equal(got_h, want_h), case
