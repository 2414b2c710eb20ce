"""GPU parity: the B200 kernels, called through the C-ABI, against the CPU
oracle (pinned in test_oracle.py) and the reference's golden vectors.
Bit-exact for every code map and histogram."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1810_11518_b200 as aldp  # noqa: E402

DEV = torch.device("cuda:0")
KERNELS = ("fast", "generic")


def to_dev(px, pitch=None):
    """[n, rows, cols] host -> [n, rows, pitch] device (pitch padded)."""
    px = np.ascontiguousarray(px, np.uint8)
    if px.ndim == 2:
        px = px[None]
    n, r, c = px.shape
    pitch = pitch or (c + 15) // 16 * 16
    buf = np.zeros((n, r, pitch), np.uint8)
    buf[:, :, :c] = px
    return torch.from_numpy(buf).to(DEV)


def run(px_host, k=3, cell=(0, 0), kernel="auto", pitch=None):
    px_host = np.ascontiguousarray(px_host, np.uint8)
    if px_host.ndim == 2:
        px_host = px_host[None]
    n, r, c = px_host.shape
    d = to_dev(px_host, pitch)
    codes, hist = aldp.ldp_batch(d, r, c, k=k, cell=cell, codes=True, hist=True, kernel=kernel)
    torch.cuda.synchronize()
    return codes[:, :, :c].cpu().numpy(), hist.cpu().numpy().astype(np.uint64)


# ------------------------------------------------------------- goldens

def test_reference_golden_fixtures(golden_fixtures):
    for fx in golden_fixtures:
        img = np.array(fx["pixels"], np.uint8).reshape(fx["rows"], fx["cols"])
        for kern in ("auto", "generic"):
            codes, hist = run(img, 3, kernel=kern)
            assert list(codes.ravel()) == fx["ldp_codes"], (fx["name"], kern)
            assert list(hist[0, 0]) == fx["ldp_histogram"], (fx["name"], kern)


def test_reference_library_vectors_all_k(ref_vectors):
    names = sorted({k.rsplit("_", 1)[0] for k in ref_vectors if k.endswith("_img") and
                    not k.startswith("win")})
    for nm in names:
        img = ref_vectors[nm + "_img"]
        for k in range(1, 8):
            codes, hist = run(img, k)
            assert np.array_equal(codes[0], ref_vectors[nm + "_codes"][k - 1]), (nm, k)
            if k == 3:
                assert np.array_equal(hist[0, 0], ref_vectors[nm + "_hist"]), nm


def test_reference_windowed_vectors(ref_vectors):
    img = ref_vectors["win_img"]
    for w in (3, 10, 25, 32, 64, 96):
        for kern in ("auto", "generic"):
            _, hist = run(img, 3, cell=(w, w), kernel=kern)
            assert np.array_equal(hist[0], ref_vectors[f"win{w}"]), (w, kern)


def test_config1_digest(ref_vectors):
    """C1: make_random(490, 640, 42), k=3, code map + whole-image histogram."""
    import hashlib
    img = oracle.make_random(490, 640, 42)
    for kern in KERNELS:
        codes, hist = run(img, 3, kernel=kern)
        assert hashlib.sha256(codes[0].tobytes()).digest() == ref_vectors["c1_codes_sha256"].tobytes()
        assert np.array_equal(hist[0, 0], ref_vectors["c1_hist"])

# ------------------------------------------------ seeded parity vs oracle

@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7])
def test_random_images_every_k(k):
    rng = np.random.default_rng(100 + k)
    for shape in [(3, 4), (3, 3), (5, 8), (17, 64), (33, 132), (64, 256), (7, 13), (31, 29)]:
        img = rng.integers(0, 256, size=shape, dtype=np.uint8)
        want_c, want_h = oracle.batch(img, k=k)
        for kern in ("auto", "generic"):
            c, h = run(img, k, kernel=kern)
            assert np.array_equal(c, want_c), (shape, k, kern)
            assert np.array_equal(h, want_h), (shape, k, kern)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7])
def test_tie_heavy_every_k(k):
    """Values {0,1,2} with constant rectangles (config-3 style)."""
    px = aldp.gen_ties(6, 64, 128, seed=7 + k, device=DEV)
    torch.cuda.synchronize()
    host = px[:, :, :128].cpu().numpy()
    want_c, want_h = oracle.batch(host, k=k)
    for kern in KERNELS:
        c, h = run(host, k, kernel=kern)
        assert np.array_equal(c, want_c), (k, kern)
        assert np.array_equal(h, want_h), (k, kern)


@pytest.mark.parametrize("cell", [(3, 3), (8, 12), (16, 16), (64, 64), (81, 91), (40, 128), (33, 70),
                                  (100, 100)])
def test_cell_histograms(cell):
    """windowed_features semantics: each cell clamped as its own image."""
    rng = np.random.default_rng(cell[0] * 1000 + cell[1])
    img = rng.integers(0, 256, size=(3, 200, 256), dtype=np.uint8)
    want_c, want_h = oracle.batch(img, k=3, cell=cell)
    for kern in ("auto", "generic"):
        c, h = run(img, 3, cell=cell, kernel=kern)
        assert np.array_equal(c, want_c), (cell, kern)
        assert np.array_equal(h, want_h), (cell, kern)


@pytest.mark.parametrize("rows,cell", [(300, (127, 91)), (300, (128, 64)), (300, (129, 40)), (300, (131, 130)),
                                       (420, (257, 91)), (530, (260, 13)), (400, (400, 200))])
@pytest.mark.parametrize("k", [3, 0])
def test_tall_cell_rows(rows, cell, k):
    """Cell rows taller than one staged halo chunk (130 rows incl. the two
    neighbour rows): the row loop refills the tile's halo columns at 126-row
    boundaries, in the unrolled loop or in its tail. LDP and LBP, regular and
    narrow cells, rows below the grid."""
    rng = np.random.default_rng(rows * 7 + cell[0])
    img = rng.integers(0, 256, size=(2, rows, 300), dtype=np.uint8)
    img[1, :, 120:140] = 7  # flat columns across a tile edge: ties in the halo columns
    want_c, want_h = oracle.batch(img, k=k, cell=cell)
    c, h = run(img, k, cell=cell, kernel="auto" if k == 0 and cell[1] < 26 else "fast")  # narrow cells: LDP only
    assert np.array_equal(c, want_c), (rows, cell, k)
    assert np.array_equal(h, want_h), (rows, cell, k)


def test_cell_histograms_k_sweep():
    px = aldp.gen_faces(2, 162, 184, blobs=8, seed=3, device=DEV)
    torch.cuda.synchronize()
    host = px[:, :, :184].cpu().numpy()
    for k in (1, 2, 3, 4, 5, 6, 7):
        want_c, want_h = oracle.batch(host, k=k, cell=(81, 91))
        c, h = run(host, k, cell=(81, 91), kernel="fast")
        assert np.array_equal(c, want_c), k
        assert np.array_equal(h, want_h), k


def test_odd_pitch_and_strides():
    rng = np.random.default_rng(9)
    img = rng.integers(0, 256, size=(4, 50, 96), dtype=np.uint8)
    want_c, want_h = oracle.batch(img, k=3, cell=(10, 12))
    c, h = run(img, 3, cell=(10, 12), pitch=100)  # pitch % 16 != 0, % 4 == 0 -> fast
    assert np.array_equal(c, want_c) and np.array_equal(h, want_h)
    c, h = run(img, 3, cell=(10, 12), pitch=97)   # unaligned pitch -> generic
    assert np.array_equal(c, want_c) and np.array_equal(h, want_h)


def test_config2_subset():
    """C2 generator (face-like 640x490), 7x6 cells, 64 images."""
    px = aldp.gen_faces(64, 490, 640, blobs=20, seed=1810, device=DEV)
    codes, hist = aldp.ldp_batch(px, 490, 640, k=3, cell=(81, 91), codes=True, hist=True)
    torch.cuda.synchronize()
    host = px.cpu().numpy()
    want_c, want_h = oracle.batch(host, k=3, cell=(81, 91))
    assert np.array_equal(codes.cpu().numpy(), want_c)
    assert np.array_equal(hist.cpu().numpy().astype(np.uint64), want_h)
    assert int(hist.sum()) == 64 * 42 * 81 * 91


def test_config3_subset_k_sweep():
    px = aldp.gen_ties(4, 1024, 1024, seed=11518, device=DEV)
    torch.cuda.synchronize()
    host = px.cpu().numpy()
    for k in (1, 3, 5):
        want_c, want_h = oracle.batch(host, k=k)
        codes, hist = aldp.ldp_batch(px, 1024, 1024, k=k, codes=True, hist=True)
        torch.cuda.synchronize()
        assert np.array_equal(codes.cpu().numpy(), want_c), k
        assert np.array_equal(hist.cpu().numpy().astype(np.uint64), want_h), k


def test_config4_full_size_sampled():
    """C4 (16384^2, 64x64 cells) at full size: size-independent properties on
    the whole frame + bit-exact oracle checks on sampled cells and bands."""
    n = 16384
    px = aldp.gen_faces(1, n, n, blobs=200, seed=42, device=DEV)
    codes, hist = aldp.ldp_batch(px, n, n, k=3, cell=(64, 64), codes=True, hist=True)
    _, whole = aldp.ldp_batch(px, n, n, k=3, hist=True)
    torch.cuda.synchronize()
    h = hist[0].to(torch.int64)
    assert int(h.sum()) == n * n
    assert bool((h.sum(dim=1) == 64 * 64).all())
    # whole-image histogram == histogram of the code map (descriptors.cpp:129-137)
    cm = torch.bincount(codes[0].reshape(-1).to(torch.int64), minlength=256)
    rank = [c for c in range(256) if bin(c).count("1") == 3]
    assert torch.equal(cm[rank].cpu(), whole[0, 0].to(torch.int64).cpu())
    assert int(cm.sum()) == n * n and int(cm[[c for c in range(256) if bin(c).count("1") != 3]].sum()) == 0
    rng = np.random.default_rng(4)
    for _ in range(24):  # cells: each is an independent image (per-cell clamp)
        i, j = rng.integers(0, 256, size=2)
        crop = px[0, i * 64:(i + 1) * 64, j * 64:(j + 1) * 64].cpu().numpy()
        assert np.array_equal(h[i * 256 + j].cpu().numpy().astype(np.uint64), oracle.histogram(crop, 3))
    for x0 in (0, 4095, 8190, n - 40):  # row bands of the code map (image clamp)
        a, b = max(x0 - 1, 0), min(x0 + 41, n)
        band = px[0, a:b].cpu().numpy()
        want = oracle.code_map(band, 3)
        got = codes[0, a:b].cpu().numpy()
        inner = slice(1 if a > 0 else 0, (b - a) - (1 if b < n else 0))
        assert np.array_equal(got[inner], want[inner]), x0


def test_fast_equals_generic_on_faces():
    px = aldp.gen_faces(8, 200, 320, blobs=12, seed=5, device=DEV)
    for cell in ((0, 0), (50, 64), (81, 91)):
        c1, h1 = aldp.ldp_batch(px, 200, 320, cell=cell, codes=True, hist=True, kernel="fast")
        c2, h2 = aldp.ldp_batch(px, 200, 320, cell=cell, codes=True, hist=True, kernel="generic")
        torch.cuda.synchronize()
        assert torch.equal(c1, c2) and torch.equal(h1, h2), cell


def test_generator_determinism_and_sharding():
    """Images are keyed by global index: any shard split sees identical bytes."""
    a = aldp.gen_faces(6, 49, 64, blobs=5, seed=99, first_index=0, device=DEV)
    b = aldp.gen_faces(3, 49, 64, blobs=5, seed=99, first_index=3, device=DEV)
    c = aldp.gen_faces(6, 49, 64, blobs=5, seed=99, first_index=0, device=DEV)
    torch.cuda.synchronize()
    assert torch.equal(a, c) and torch.equal(a[3:], b)
    t1 = aldp.gen_ties(4, 64, 64, seed=1, device=DEV)
    t2 = aldp.gen_ties(2, 64, 64, seed=1, first_index=2, device=DEV)
    torch.cuda.synchronize()
    assert torch.equal(t1[2:], t2)
    assert int(t1.max()) <= 2


# ------------------------------------------------ host entry points (C-ABI)

def test_host_entry_points_match_oracle():
    img = oracle.make_random(37, 53, 5)
    assert np.array_equal(aldp.ldp_histogram(img, 3, aldp.ResponsePath.Naive),
                          oracle.ref_ldp_histogram(img, 3, 0))
    assert np.array_equal(aldp.ldp_histogram(img, 3), oracle.ref_ldp_histogram(img, 3, 1))
    for w in (3, 8, 37):
        assert np.array_equal(aldp.windowed_features(img, w, "ldp"), oracle.ref_windowed(img, w, 0))
        assert np.array_equal(aldp.windowed_features(img, w, aldp.Descriptor.Aldp), oracle.ref_windowed(img, w, 1))
    for k in range(1, 8):
        assert np.array_equal(aldp.ldp_code_map(img, k), oracle.code_map(img, k))
    c, h = aldp.ldp_batch_host(np.stack([img, img[::-1].copy()]), k=3, cell=(9, 10))
    wc, wh = oracle.batch(np.stack([img, img[::-1].copy()]), k=3, cell=(9, 10))
    assert np.array_equal(c, wc) and np.array_equal(h.astype(np.uint64), wh)


def test_host_entry_point_errors():
    img = np.zeros((10, 10), np.uint8)
    with pytest.raises(ValueError):
        aldp.ldp_histogram(img, 2)                    # k != 3 (descriptors.cpp:124-126)
    with pytest.raises(ValueError):
        aldp.ldp_histogram(np.zeros((2, 9), np.uint8), 3)  # < 3x3
    with pytest.raises(ValueError):
        aldp.windowed_features(img, 2)                # window < 3
    with pytest.raises(ValueError):
        aldp.windowed_features(img, 11)               # window > image
    with pytest.raises(ValueError):
        aldp.ldp_code_map(img, 8)                     # k out of [1, 7]
    px = to_dev(img, pitch=10)  # pitch not 8-byte aligned: the packed kernel refuses
    with pytest.raises(ValueError):
        aldp.ldp_batch(px, 10, 10, k=3, cell=(5, 5), codes=True, hist=True, kernel="fast")


def test_empty_batch_and_constant_images():
    px = torch.zeros((0, 8, 16), dtype=torch.uint8, device=DEV)
    c, h = aldp.ldp_batch(px, 8, 16, codes=True, hist=True)
    torch.cuda.synchronize()
    assert c.numel() == 0 and h.numel() == 0
    const = torch.full((2, 10, 16), 200, dtype=torch.uint8, device=DEV)
    c, h = aldp.ldp_batch(const, 10, 16, codes=True, hist=True)
    torch.cuda.synchronize()
    assert bool((c[:, :, :16] == 7).all())            # total tie -> code 7 (bin 0)
    assert int(h[0, 0, 0]) == 160 and int(h.sum()) == 320


@pytest.mark.parametrize("n,rows,cols,cell", [(3, 490, 640, (81, 91)), (5, 130, 384, (0, 0)),
                                              (1, 97, 640, (32, 40)), (7, 64, 128, (16, 16))])
def test_odd_image_counts_and_block_parity(n, rows, cols, cell):
    """Tile pairing groups two images when a row has an odd number of
    128-column blocks; odd image counts leave a partial group."""
    px = aldp.gen_faces(n, rows, cols, blobs=10, seed=n * 31 + cols, device=DEV)
    torch.cuda.synchronize()
    host = px[:, :, :cols].cpu().numpy()
    want_c, want_h = oracle.batch(host, k=3, cell=cell)
    for kern in ("auto", "generic"):  # auto: fast unless cells < ~26 columns
        c, h = run(host, 3, cell=cell, kernel=kern)
        assert np.array_equal(c, want_c), kern
        assert np.array_equal(h, want_h), kern


def test_host_batch_pipelined_chunks():
    """aldp_ldp_batch_host cuts large batches into chunks over 3 streams;
    results must equal the device-resident path image for image."""
    n = 400  # > 2 chunks of 640x490
    px = aldp.gen_faces(n, 490, 640, blobs=20, seed=77, device=DEV)
    codes, hist = aldp.ldp_batch(px, 490, 640, k=3, cell=(81, 91), codes=True, hist=True)
    torch.cuda.synchronize()
    host = px.cpu().numpy()
    hc, hh = aldp.ldp_batch_host(host, k=3, cell=(81, 91))
    assert np.array_equal(hc, codes.cpu().numpy())
    assert np.array_equal(hh, hist.cpu().numpy().astype(np.uint32))
    pinned = torch.from_numpy(host).pin_memory()
    c2 = torch.empty_like(pinned).pin_memory()
    h2 = torch.empty((n, 42, 56), dtype=torch.int32).pin_memory()
    aldp._check(aldp.lib.aldp_ldp_batch_host(pinned.data_ptr(), n, 490, 640, 3, 81, 91, c2.data_ptr(),
                                             h2.data_ptr(), None))
    assert torch.equal(c2, codes.cpu()) and torch.equal(h2, hist.cpu())


# ------------------------------------------------------------------- LBP

def run_lbp(px_host, cell=(0, 0), kernel="auto", pitch=None):
    px_host = np.ascontiguousarray(px_host, np.uint8)
    if px_host.ndim == 2:
        px_host = px_host[None]
    n, r, c = px_host.shape
    d = to_dev(px_host, pitch)
    codes, hist = aldp.lbp_batch(d, r, c, cell=cell, codes=True, hist=True, kernel=kernel)
    torch.cuda.synchronize()
    return codes[:, :, :c].cpu().numpy(), hist.cpu().numpy().astype(np.uint64)


def test_lbp_reference_goldens(golden_fixtures, ref_vectors):
    for fx in golden_fixtures:
        img = np.array(fx["pixels"], np.uint8).reshape(fx["rows"], fx["cols"])
        for kern in ("auto", "generic"):
            c, h = run_lbp(img, kernel=kern)
            assert list(c.ravel()) == fx["lbp_codes"] and list(h[0, 0]) == fx["lbp_histogram"], kern
    names = sorted({k.rsplit("_", 1)[0] for k in ref_vectors if k.endswith("_lbpcodes")})
    for nm in names:
        c, h = run_lbp(ref_vectors[nm + "_img"])
        assert np.array_equal(c[0], ref_vectors[nm + "_lbpcodes"]), nm
        assert np.array_equal(h[0, 0], ref_vectors[nm + "_lbphist"]), nm
    img = ref_vectors["win_img"]
    for w in (3, 10, 25, 32, 64, 96):
        for kern in ("auto", "generic"):
            _, h = run_lbp(img, cell=(w, w), kernel=kern)
            assert np.array_equal(h[0], ref_vectors[f"winlbp{w}"]), (w, kern)


@pytest.mark.parametrize("cell", [(0, 0), (81, 91), (64, 64), (33, 70), (8, 12)])
def test_lbp_random_ties_faces(cell):
    rng = np.random.default_rng(cell[0] + 7)
    imgs = [rng.integers(0, 256, size=(2, 130, 256), dtype=np.uint8)]
    t = aldp.gen_ties(2, 130, 256, seed=5, device=DEV)
    f = aldp.gen_faces(2, 130, 256, blobs=8, seed=6, device=DEV)
    torch.cuda.synchronize()
    imgs += [t[:, :, :256].cpu().numpy(), f[:, :, :256].cpu().numpy()]
    for img in imgs:
        want_c, want_h = oracle.batch(img, k=0, cell=cell)
        for kern in ("auto", "generic"):
            c, h = run_lbp(img, cell=cell, kernel=kern)
            assert np.array_equal(c, want_c), (cell, kern)
            assert np.array_equal(h, want_h), (cell, kern)


def test_lbp_host_entry_points():
    img = oracle.make_random(41, 57, 3)
    _, want_h = oracle.batch(img, k=0)
    assert np.array_equal(aldp.lbp_histogram(img), want_h[0, 0])
    assert np.array_equal(aldp.lbp_code_map(img), oracle.code_map(img, 0))
    for w in (3, 9, 41):
        assert np.array_equal(aldp.windowed_features(img, w, "lbp"), oracle.cell_histograms(img, w, w, 0))
    batch = np.stack([img, img[::-1].copy(), img[:, ::-1].copy()])
    c, h = aldp.ldp_batch_host(batch, k=0, cell=(10, 14))
    wc, wh = oracle.batch(batch, k=0, cell=(10, 14))
    assert np.array_equal(c, wc) and np.array_equal(h.astype(np.uint64), wh)


def test_host_entry_points_concurrent_threads():
    """Every entry point may be called from several host threads at once
    (per-thread streams and buffers; ctypes drops the GIL during the call)."""
    from concurrent.futures import ThreadPoolExecutor
    rng = np.random.default_rng(123)
    imgs = [rng.integers(0, 256, size=(int(r), int(c)), dtype=np.uint8)
            for r, c in rng.integers(3, 300, size=(48, 2))]
    want = [oracle.histogram(im, 3) for im in imgs]
    big = np.stack([oracle.make_random(96, 128, s) for s in range(40)])
    want_big = oracle.batch(big, k=3, cell=(16, 32), codes=False)[1]

    def job(i):
        if i % 6 == 5:
            _, h = aldp.ldp_batch_host(big, k=3, cell=(16, 32), codes=False)
            return np.array_equal(h.astype(np.uint64), want_big)
        return np.array_equal(aldp.ldp_histogram(imgs[i]), want[i])

    with ThreadPoolExecutor(max_workers=8) as ex:
        assert all(ex.map(job, range(len(imgs))))


def _hist_of_map(codes, k, cr, cc):
    """Cells cut from a whole-image code map (numpy over the oracle's map)."""
    n, r, c = codes.shape
    gr, gc = r // cr, c // cc
    if k == 0:
        lut = np.arange(256)
        nb = 256
    else:
        lut = np.full(256, -1)
        ranks = [v for v in range(256) if bin(v).count("1") == k]
        lut[ranks] = np.arange(len(ranks))
        nb = len(ranks)
    out = np.zeros((n, gr * gc, nb), np.uint64)
    for i in range(n):
        for a in range(gr):
            for b in range(gc):
                cell = lut[codes[i, a * cr:(a + 1) * cr, b * cc:(b + 1) * cc]].ravel()
                out[i, a * gc + b] = np.bincount(cell, minlength=nb)
    return out


@pytest.mark.parametrize("k,cell", [(3, (16, 24)), (1, (81, 91)), (5, (7, 9)), (0, (32, 40)), (3, (3, 3))])
def test_cells_cut_from_code_map(k, cell):
    """cell_clamp=False: each cell histograms the whole-image code map
    (the paper's regional histograms of one code image), both kernels."""
    n, r, c = 3, 162, 184
    px = aldp.gen_faces(n, r, c, seed=31 + k)
    host = px[:, :, :c].cpu().numpy()
    ref_codes, _ = oracle.batch(host, k=k, codes=True, hist=False)
    want = _hist_of_map(ref_codes, k, *cell)
    for kern in ("auto", "generic"):
        fn = aldp.lbp_batch if k == 0 else aldp.ldp_batch
        kw = {} if k == 0 else {"k": k}
        codes, hist = fn(px, r, c, cell=cell, codes=True, hist=True, kernel=kern, cell_clamp=False, **kw)
        torch.cuda.synchronize()
        assert np.array_equal(codes[:, :, :c].cpu().numpy(), ref_codes), kern
        assert np.array_equal(hist.cpu().numpy().astype(np.uint64), want), (kern, k, cell)
        # and the default (reference windowed rule) is unchanged
        _, h2 = fn(px, r, c, cell=cell, hist=True, kernel=kern, **kw)
        torch.cuda.synchronize()
        assert np.array_equal(h2.cpu().numpy().astype(np.uint64), oracle.batch(host, k=k, cell=cell, codes=False)[1])


@pytest.mark.parametrize("cols", [3, 5, 7, 13, 29, 127, 129, 130, 133, 255, 257, 490])
def test_fast_kernel_any_width(cols):
    """The packed kernel takes widths that are not a multiple of its 8-column
    lanes (the edge lane stores its valid bytes singly; padding untouched)."""
    rng = np.random.default_rng(cols)
    rows = 37
    img = rng.integers(0, 256, size=(3, rows, cols), dtype=np.uint8)
    for k in (3, 5):
        want_c, want_h = oracle.batch(img, k=k)
        c, h = run(img, k, kernel="fast")
        assert np.array_equal(c, want_c) and np.array_equal(h, want_h), (cols, k)
    if cols >= 3:
        cell = (9, max(3, cols // 3))
        want_c, want_h = oracle.batch(img, k=3, cell=cell)
        c, h = run(img, 3, cell=cell, kernel="fast")
        assert np.array_equal(c, want_c) and np.array_equal(h, want_h), (cols, cell)
    # bytes past `cols` inside the pitch are never written
    d = to_dev(img)
    pitch = d.shape[2]
    codes = torch.full((3, rows, pitch), 0xAB, dtype=torch.uint8, device=DEV)
    aldp.ldp_batch(d, rows, cols, k=3, codes=codes, kernel="fast")
    torch.cuda.synchronize()
    if pitch > cols:
        assert bool((codes[:, :, cols:] == 0xAB).all())


@pytest.mark.parametrize("kernel", ["auto", "generic"])
def test_band_views_with_halo_rows(kernel):
    """A tall frame processed as bands (views into the resident frame with
    halo=(1, 1) on inner edges) gives the frame's exact codes and histograms:
    whole-image histograms sum, cell grids tile (bands of whole cells)."""
    r, c = 300, 200
    img = oracle.make_random(r, c, 4242)
    d = to_dev(img)
    pitch = d.shape[2]
    want_c, want_w = oracle.batch(img, k=3)
    _, want_cells = oracle.batch(img, k=3, cell=(20, 25), codes=False)
    for B in (40, 60, 100):  # multiples of the 20-row cells
        codes = np.zeros((r, c), np.uint8)
        whole = np.zeros(56, np.uint64)
        cells = []
        for s0 in range(0, r, B):
            s1 = min(r, s0 + B)
            view = d[:, s0:s1, :]
            cb, hb = aldp.ldp_batch(view, s1 - s0, c, k=3, codes=True, hist=True, kernel=kernel,
                                    halo=(s0 > 0, s1 < r))
            _, hc = aldp.ldp_batch(view, s1 - s0, c, k=3, cell=(20, 25), hist=True, kernel=kernel,
                                   halo=(s0 > 0, s1 < r))
            torch.cuda.synchronize()
            codes[s0:s1] = cb[0, :, :c].cpu().numpy()
            whole += hb[0, 0].cpu().numpy().astype(np.uint64)
            cells.append(hc[0].cpu().numpy().astype(np.uint64))
        assert np.array_equal(codes, want_c[0]), (B, kernel)
        assert np.array_equal(whole, want_w[0, 0]), (B, kernel)
        assert np.array_equal(np.concatenate(cells), want_cells[0]), (B, kernel)
    assert pitch >= c


def test_host_banded_tall_frames():
    """Single frames taller than a host chunk stream as bands with halo rows
    (ALDP_CHUNK_BYTES shrinks the chunk so small frames take that path), for
    pageable and pinned buffers, whole-image and cell histograms, LDP and LBP."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1810_11518_b200 as aldp, oracle
out = []
for (r, c, cell, k) in [(333, 250, (0, 0), 3), (333, 250, (20, 25), 3), (517, 96, (32, 32), 5),
                        (333, 250, (0, 0), 0), (333, 250, (21, 25), 0), (64, 4000, (9, 40), 3)]:
    img = oracle.make_random(r, c, r * c + k)
    want_c, want_h = oracle.batch(img, k=k, cell=cell)
    for pinned in (False, True):
        src = img[None].copy()
        if pinned:
            t = torch.from_numpy(src).pin_memory()
            src = t.numpy()
        codes, hist = aldp.ldp_batch_host(src, k=k, cell=cell)
        out.append(bool(np.array_equal(codes, want_c) and np.array_equal(hist.astype(np.uint64), want_h)))
print(json.dumps(out))
'''
    env = dict(os.environ, ALDP_CHUNK_BYTES="20000")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(res), res


@pytest.mark.parametrize("k", [0, 3, 4])
@pytest.mark.parametrize("rows,cell", [(490, (81, 91)), (100, (3, 64)), (37, (9, 40)), (130, (64, 64))])
def test_small_batch_split_launch(k, rows, cell):
    """Small cell batches whose rows overhang the cell grid run as two
    launches (grid rows with histograms, remainder rows codes-only from two
    rows above the grid's end; ldp_kernels.cu run_batch). Every code and
    every cell count equals the oracle's, including the rows around the
    grid's end; the same holds for a band view with a real row above and
    below it (halo = (1, 1))."""
    cols, n = 300, 5
    assert rows % cell[0] != 0
    f = aldp.gen_faces(n, rows + 2, cols, blobs=6, seed=rows + k, device=DEV)
    torch.cuda.synchronize()
    tall = f[:, :, :cols].cpu().numpy()
    # plain frames: the first `rows` rows of each tall frame (k = 0: LBP)
    px = tall[:, :rows]
    # kernel="fast": these layouts must take the packed kernel and its split
    # launch (grid rows, then the remainder rows), never the generic kernel
    codes, hist = aldp.ldp_batch(to_dev(px), rows, cols, k=k, cell=cell, codes=True, hist=True, kernel="fast")
    assert aldp.last_launch_count() == 2, (k, rows, cell)
    torch.cuda.synchronize()
    want_c, want_h = oracle.batch(px, k=k, cell=cell)
    assert np.array_equal(codes[:, :, :cols].cpu().numpy(), want_c), (k, rows, cell)
    assert np.array_equal(hist.cpu().numpy().astype(np.uint64), want_h), (k, rows, cell)
    # band view: rows 1 .. rows of one tall frame, real rows above and below
    dt = to_dev(tall[0])
    view = dt[:, 1:rows + 1, :]
    codes, hist = aldp.ldp_batch(view, rows, cols, k=k, cell=cell, codes=True, hist=True, halo=(1, 1),
                                 kernel="fast")
    torch.cuda.synchronize()
    full_c, _ = oracle.batch(tall[:1], k=k, hist=False)
    assert np.array_equal(codes[0, :, :cols].cpu().numpy(), full_c[0, 1:rows + 1]), (k, rows, cell)
    # the band's cells are clamped as their own images (windowed_features)
    _, want_band_h = oracle.batch(tall[:1, 1:rows + 1], k=k, cell=cell, codes=False)
    assert np.array_equal(hist.cpu().numpy().astype(np.uint64), want_band_h), (k, rows, cell)


# ------------------------------------------------- narrow cells (round 2)

@pytest.mark.parametrize("window", [9, 10, 13, 20, 25, 31])
@pytest.mark.parametrize("k", [1, 3, 5, 7])
def test_narrow_cells_fast_kernel(window, k):
    """The paper's small windows (Table 3: 10, 20, 25 px) on the
    narrow-cell layout of the packed kernel (up to 16 cells per tile): code
    maps and every cell's histogram bit-exact vs the oracle, on face-like and
    tie-heavy frames, frames whose width is not a multiple of 128 included."""
    faces = aldp.gen_faces(3, 200, 330, blobs=8, seed=window * 7 + k, device=DEV)
    ties = aldp.gen_ties(2, 150, 256, seed=window + k, device=DEV)
    for px, r, c in ((faces, 200, 330), (ties, 150, 256)):
        codes, hist = aldp.ldp_batch(px, r, c, k=k, cell=(window, window), codes=True, hist=True, kernel="fast")
        assert aldp.last_launch_count() >= 1
        torch.cuda.synchronize()
        host = px[:, :, :c].cpu().numpy()
        rc, rh = oracle.batch(host, k=k, cell=(window, window))
        assert np.array_equal(codes[:, :, :c].cpu().numpy(), rc), (window, k)
        assert np.array_equal(hist.cpu().numpy().astype(np.uint64), rh), (window, k)


def test_narrow_cells_rectangular_and_paper_windows():
    """Rectangular narrow cells and the full 640x490 frame at windows 10 / 20 /
    25 (the reference's windowed_features, 3136 / 768 / 475 cells)."""
    px = aldp.gen_faces(2, 490, 640, blobs=20, seed=99, device=DEV)
    host = px[:, :, :640].cpu().numpy()
    for cell in ((10, 10), (20, 20), (25, 25), (12, 9), (40, 11), (7, 30)):
        _, hist = aldp.ldp_batch(px, 490, 640, k=3, cell=cell, hist=True)
        torch.cuda.synchronize()
        _, rh = oracle.batch(host, k=3, cell=cell, codes=False)
        assert np.array_equal(hist.cpu().numpy().astype(np.uint64), rh), cell


def test_narrow_cells_fallbacks():
    """Cells narrower than 9 columns, LBP and k = 4 on narrow cells run the
    generic kernel under kernel='auto' (bit-exact) and are refused by 'fast'."""
    px = aldp.gen_faces(1, 64, 160, seed=5, device=DEV)
    host = px[:, :, :160].cpu().numpy()
    for k, cell in ((3, (8, 8)), (3, (5, 3)), (4, (10, 10)), (0, (10, 10))):
        c, h = aldp.ldp_batch(px, 64, 160, k=k, cell=cell, codes=True, hist=True)
        torch.cuda.synchronize()
        rc, rh = oracle.batch(host, k=k, cell=cell)
        assert np.array_equal(c[:, :, :160].cpu().numpy(), rc) and \
            np.array_equal(h.cpu().numpy().astype(np.uint64), rh), (k, cell)
        with pytest.raises(ValueError):
            aldp.ldp_batch(px, 64, 160, k=k, cell=cell, codes=True, hist=True, kernel="fast")


@pytest.mark.parametrize("own", ["0", "2"])
@pytest.mark.parametrize("window", [9, 10, 12, 16, 20, 25, 31])
def test_narrow_hist_modes(window, own, monkeypatch):
    """Both ways the narrow-cell kernel writes histograms (ldp_kernels.cu
    narrow_hist_mode, forced by ALDP_NARROW_HIST): 0 = global atomics into a
    memset buffer, 2 = cells wholly inside a 128-column tile stored (every
    bin, no memset) and the straddling ones added after a zeroing launch.
    Output buffers pre-filled with garbage must come out exact; u32 and u16
    histograms; frames with rows/columns beyond the cell grid and widths that
    are not a multiple of 128."""
    monkeypatch.setenv("ALDP_NARROW_HIST", own)
    for n, r, c, seed in ((3, 2 * window + 5, 330, window), (2, 490, 640, 7 * window)):
        px = aldp.gen_faces(n, r, c, blobs=8, seed=seed, device=DEV)
        host = px[:, :, :c].cpu().numpy()
        rc, rh = oracle.batch(host, k=3, cell=(window, window))
        cells = rh.shape[1]
        for dt in (torch.int32, torch.int16):
            codes = torch.full((n, r, px.shape[2]), 0xA5, dtype=torch.uint8, device=DEV)
            hist = torch.full((n, cells, 56), 12345, dtype=dt, device=DEV)
            aldp.ldp_batch(px, r, c, k=3, cell=(window, window), codes=codes, hist=hist, kernel="fast")
            torch.cuda.synchronize()
            assert np.array_equal(codes[:, :, :c].cpu().numpy(), rc), (window, own, dt)
            got = hist.cpu().numpy().astype(np.int64) & (0xFFFF if dt == torch.int16 else -1)
            assert np.array_equal(got.astype(np.uint64), rh), (window, own, dt)


def test_narrow_hist_unaligned_buffer_falls_back():
    """Narrow cells store whole cells 16 bytes at a time (8 for uint16 bins);
    a histogram buffer that is only 4-byte aligned takes the memset + atomics
    path instead and must give the same bits."""
    px = aldp.gen_faces(2, 200, 330, blobs=8, seed=5, device=DEV)
    host = px[:, :, :330].cpu().numpy()
    _, rh = oracle.batch(host, k=3, cell=(10, 10), codes=False)
    cells = rh.shape[1]
    for dt, off in ((torch.int32, 1), (torch.int32, 2), (torch.int16, 2)):
        buf = torch.full((2 * cells * 56 + off,), 999, dtype=dt, device=DEV)
        hist = buf[off:].view(2, cells, 56)  # base 4 or 8 bytes (int32) / 4 bytes (int16) past 16-byte alignment
        aldp.ldp_batch(px, 200, 330, k=3, cell=(10, 10), hist=hist, kernel="fast")
        torch.cuda.synchronize()
        got = hist.cpu().numpy().astype(np.int64) & (0xFFFF if dt == torch.int16 else -1)
        assert np.array_equal(got.astype(np.uint64), rh), (dt, off)
        assert int(buf[:off].max()) == 999  # nothing written before the buffer
