"""Size-independent properties at full config sizes (SURVEY 8c pins 3), on
the B200 path through the C-ABI: the reference's property tests
(test_descriptors.cpp:33-38, 90-151) restated at C2-C5 scale where the CPU
oracle cannot follow, plus histogram == histogram-of-the-code-map and shard
invariance of the generated inputs."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1810_11518_b200 as aldp  # noqa: E402

DEV = torch.device("cuda:0")
POPCOUNT = torch.tensor([bin(c).count("1") for c in range(256)], dtype=torch.uint8, device=DEV)


def code_bins(k):
    """code -> bin lookup (ascending popcount-k codes), -1 elsewhere."""
    lut = torch.full((256,), -1, dtype=torch.int64, device=DEV)
    for i, c in enumerate(c for c in range(256) if bin(c).count("1") == k):
        lut[c] = i
    return lut


def test_translation_invariance_full_frames():
    """test_descriptors.cpp:129-151: adding a constant leaves every code
    unchanged (here 256 full 640x490 frames, +55 on values <= 200)."""
    n, r, c = 256, 490, 640
    d = aldp.gen_faces(n, r, c, seed=29)
    d = torch.clamp(d, max=200)
    codes0, hist0 = aldp.ldp_batch(d, r, c, k=3, cell=(81, 91), codes=True, hist=True)
    codes1, hist1 = aldp.ldp_batch(d + 55, r, c, k=3, cell=(81, 91), codes=True, hist=True)
    torch.cuda.synchronize()
    assert torch.equal(codes0, codes1) and torch.equal(hist0, hist1)


@pytest.mark.parametrize("k", range(1, 8))
def test_every_code_has_k_bits(k):
    """test_descriptors.cpp:33-38 at C2 scale: popcount(code) == k everywhere."""
    n, r, c = 128, 490, 640
    d = aldp.gen_faces(n, r, c, seed=100 + k)
    codes, hist = aldp.ldp_batch(d, r, c, k=k, codes=True, hist=True)
    torch.cuda.synchronize()
    assert bool((POPCOUNT[codes[:, :, :c].long()] == k).all())
    assert bool((hist.sum(dim=(1, 2)) == r * c).all())  # mass (test_descriptors.cpp:90-99)


@pytest.mark.parametrize("k", [1, 3, 5])
def test_histogram_is_histogram_of_code_map_c3(k):
    """Config 3 at full size (256 x 1024^2, tie-heavy): the whole-image
    histogram equals the bincount of the code map in bin order."""
    n, r, c = 256, 1024, 1024
    d = aldp.gen_ties(n, r, c, seed=11518)
    codes, hist = aldp.ldp_batch(d, r, c, k=k, codes=True, hist=True)
    lut = code_bins(k)
    nb = aldp.n_bins(k)
    for i0 in range(0, n, 32):
        b = lut[codes[i0:i0 + 32].long()]
        assert bool((b >= 0).all())
        idx = b + (torch.arange(b.shape[0], device=DEV) * nb)[:, None, None]
        counts = torch.bincount(idx.flatten(), minlength=b.shape[0] * nb).view(-1, nb)
        assert torch.equal(counts.to(torch.int32), hist[i0:i0 + 32, 0])


def test_cell_mass_c5_frames():
    """Every 81x91 cell of every frame counts exactly 7371 pixels."""
    n, r, c = 512, 490, 640
    d = aldp.gen_faces(n, r, c, seed=7)
    _, hist = aldp.ldp_batch(d, r, c, k=3, cell=(81, 91), hist=True)
    torch.cuda.synchronize()
    assert hist.shape == (n, 42, 56)
    assert bool((hist.sum(dim=2) == 81 * 91).all())


def test_path_independence_random_sizes():
    """test_descriptors.cpp:111-120: Naive == Accelerated over 40 random
    sizes in [3, 64], and both equal the oracle."""
    rng = np.random.default_rng(17)
    for _ in range(40):
        r, c = (int(v) for v in rng.integers(3, 65, size=2))
        img = oracle.make_random(r, c, int(rng.integers(0, 2**32)))
        a = aldp.ldp_histogram(img, 3, aldp.ResponsePath.Naive)
        b = aldp.ldp_histogram(img, 3, aldp.ResponsePath.Accelerated)
        assert np.array_equal(a, b)
        assert np.array_equal(a, oracle.histogram(img, 3))


def test_shard_invariance_c5_slice():
    """Images keyed by global index: two half-batches (two ranks' shards)
    produce exactly the histograms of the whole batch."""
    n, r, c = 64, 490, 640
    whole = aldp.gen_faces(n, r, c, seed=11518)
    lo = aldp.gen_faces(n // 2, r, c, seed=11518, first_index=0)
    hi = aldp.gen_faces(n // 2, r, c, seed=11518, first_index=n // 2)
    _, h = aldp.ldp_batch(whole, r, c, k=3, cell=(81, 91), hist=True)
    _, h0 = aldp.ldp_batch(lo, r, c, k=3, cell=(81, 91), hist=True)
    _, h1 = aldp.ldp_batch(hi, r, c, k=3, cell=(81, 91), hist=True)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([h0, h1]), h)


def test_config5_full_batch_sampled_vs_oracle():
    """Config 5 at full size: all 65,536 frames (20.6 GB) in one launch, as
    bench.py runs it; 48 frames at a stride across the batch checked
    bit-exactly against the CPU oracle (codes and 7x6 cell histograms), and
    every cell's mass checked for all frames."""
    n, r, c = 65536, 490, 640
    d = aldp.gen_faces(n, r, c, seed=11518)
    codes, hist = aldp.ldp_batch(d, r, c, k=3, cell=(81, 91), codes=True, hist=True)
    torch.cuda.synchronize()
    assert bool((hist.sum(dim=2) == 81 * 91).all())
    idx = list(range(0, n, n // 47))[:47] + [n - 1]
    host = d[idx].cpu().numpy()
    want_c, want_h = oracle.batch(host, k=3, cell=(81, 91), threads=16)
    assert np.array_equal(codes[idx].cpu().numpy(), want_c)
    assert np.array_equal(hist[idx].cpu().numpy().astype(np.uint64), want_h)
    del codes, hist, d
    torch.cuda.empty_cache()
