"""Pins the CPU oracle (oracle/ldp_oracle.c) before it is trusted as the
checker: against the reference's golden fixtures, the reference's known-
answer tests, and the unmodified reference library (oracle/_ref) itself.
CPU only."""
import itertools

import numpy as np
import pytest

import oracle

# ---------------------------------------------------------------- goldens

def test_port_matches_reference_golden_fixtures(golden_fixtures):
    """proj/tests/golden/fixture_*.json: responses, k=3 codes, 56-bin hist."""
    assert len(golden_fixtures) == 4
    for fx in golden_fixtures:
        img = np.array(fx["pixels"], np.uint8).reshape(fx["rows"], fx["cols"])
        resp = [list(oracle.responses(img, x, y)) for x in range(fx["rows"]) for y in range(fx["cols"])]
        assert resp == fx["responses"], fx["name"]
        assert list(oracle.code_map(img, 3).ravel()) == fx["ldp_codes"], fx["name"]
        assert list(oracle.histogram(img, 3)) == fx["ldp_histogram"], fx["name"]


def test_port_lbp_matches_reference_golden_fixtures(golden_fixtures):
    """LBP codes / 256-bin histograms of the same fixtures (generate.py:55-76)."""
    for fx in golden_fixtures:
        img = np.array(fx["pixels"], np.uint8).reshape(fx["rows"], fx["cols"])
        c, h = oracle.batch(img, k=0)
        assert list(c.ravel()) == fx["lbp_codes"], fx["name"]
        assert list(h[0, 0]) == fx["lbp_histogram"], fx["name"]


def test_port_lbp_matches_reference_library(ref_vectors):
    names = sorted({k.rsplit("_", 1)[0] for k in ref_vectors if k.endswith("_lbpcodes")})
    assert len(names) >= 10
    for nm in names:
        c, h = oracle.batch(ref_vectors[nm + "_img"], k=0)
        assert np.array_equal(c[0], ref_vectors[nm + "_lbpcodes"]), nm
        assert np.array_equal(h[0, 0], ref_vectors[nm + "_lbphist"]), nm
    img = ref_vectors["win_img"]
    for w in (3, 10, 25, 32, 64, 96):
        assert np.array_equal(oracle.cell_histograms(img, w, w, 0), ref_vectors[f"winlbp{w}"]), w
    # constant image: every neighbour >= centre -> code 255 (descriptors.hpp:57-59)
    assert oracle.histogram(np.full((6, 7), 9, np.uint8), 0)[255] == 42


def test_port_matches_reference_library_vectors(ref_vectors):
    """Code maps k=1..7 and histograms produced by the reference library."""
    names = sorted({k.rsplit("_", 1)[0] for k in ref_vectors if k.endswith("_img") and
                    not k.startswith("win")})
    assert len(names) >= 10
    for nm in names:
        img = ref_vectors[nm + "_img"]
        for k in range(1, 8):
            assert np.array_equal(oracle.code_map(img, k), ref_vectors[nm + "_codes"][k - 1]), (nm, k)
        assert np.array_equal(oracle.histogram(img, 3), ref_vectors[nm + "_hist"]), nm


def test_port_windowed_matches_reference(ref_vectors):
    img = ref_vectors["win_img"]
    for w in (3, 10, 25, 32, 64, 96):
        assert np.array_equal(oracle.cell_histograms(img, w, w, 3), ref_vectors[f"win{w}"]), w


def test_make_random_matches_reference():
    """image.cpp:75-83 (std::mt19937 low byte) restated in C."""
    for (r, c, s) in [(3, 3, 0), (490, 640, 42), (17, 5, 123456789)]:
        assert np.array_equal(oracle.make_random(r, c, s), oracle.ref_make_random(r, c, s))


def test_config1_digest(ref_vectors):
    import hashlib
    img = oracle.make_random(490, 640, 42)
    assert hashlib.sha256(img.tobytes()).digest() == ref_vectors["c1_img_sha256"].tobytes()
    codes = oracle.code_map(img, 3)
    assert hashlib.sha256(codes.tobytes()).digest() == ref_vectors["c1_codes_sha256"].tobytes()
    assert np.array_equal(oracle.histogram(img, 3), ref_vectors["c1_hist"])

# ------------------------------------------------- reference KATs (restated)

def test_ramp_center_responses():
    """test_kirsch.cpp:17,89-96 frozen ramp-centre responses."""
    ramp = np.arange(1, 10, dtype=np.uint8).reshape(3, 3)
    assert list(oracle.responses(ramp, 1, 1)) == [24, -32, -72, -64, -24, 32, 72, 64]


def test_ldp_code_tie_rules():
    """test_descriptors.cpp:20-32: total tie -> 7, distinct -> 82, partial tie
    keeps the lower index."""
    assert oracle.ldp_code([5] * 8, 3) == 7
    assert oracle.ldp_code([1, 9, 2, 8, 3, 7, 4, 6], 3) == (1 << 1) | (1 << 3) | (1 << 5)
    assert oracle.ldp_code([0, 4, 4, 4, 4, 0, 0, 0], 3) == (1 << 1) | (1 << 2) | (1 << 3)
    for k in range(1, 8):
        assert bin(oracle.ldp_code([3, 1, 4, 1, 5, 9, 2, 6], k)).count("1") == k
    assert oracle.ldp_code([0] * 8, 0) == -1 and oracle.ldp_code([0] * 8, 8) == -1


def test_tie_heavy_codes_vs_sort_oracle():
    """test_descriptors.cpp:43-55: values in -3..3 against a sort oracle."""
    rng = np.random.default_rng(5)
    for _ in range(2000):
        m = rng.integers(-3, 4, size=8)
        for k in range(1, 8):
            order = sorted(range(8), key=lambda i: (-m[i], i))
            want = sum(1 << i for i in order[:k])
            assert oracle.ldp_code(m, k) == want


def test_bins():
    """descriptors.cpp:25-45: 56 bins, code 7 <-> bin 0, 224 <-> 55."""
    codes = [c for c in range(256) if bin(c).count("1") == 3]
    assert [oracle.bin_index(c, 3) for c in codes] == list(range(56))
    assert oracle.bin_index(7, 3) == 0 and oracle.bin_index(224, 3) == 55
    assert oracle.bin_index(0, 3) == -1 and oracle.bin_index(255, 3) == -1
    assert [oracle.n_bins(k) for k in range(1, 8)] == [8, 28, 56, 70, 56, 28, 8]


def test_constant_image_bin0():
    """test_descriptors.cpp:82-89: constant 10x10 -> 100 counts in bin 0."""
    h = oracle.histogram(np.full((10, 10), 77, np.uint8), 3)
    assert h[0] == 100 and h.sum() == 100


def test_response_bound_attained():
    """test_kirsch.cpp:288-315: |m| <= 3825, attained on a checker."""
    chk = np.array([[255 if ((x // 3 + y // 3) % 2 == 0) else 0 for y in range(9)] for x in range(9)],
                   np.uint8)
    best = max(abs(int(v)) for x in range(9) for y in range(9) for v in oracle.responses(chk, x, y))
    assert best == 3825


def test_mass_and_path_independence():
    rng = np.random.default_rng(3)
    for _ in range(10):
        r, c = rng.integers(3, 40, size=2)
        img = rng.integers(0, 256, size=(r, c), dtype=np.uint8)
        h = oracle.histogram(img, 3)
        assert h.sum() == r * c
        assert np.array_equal(h, oracle.ref_ldp_histogram(img, 3, 0))
        assert np.array_equal(h, oracle.ref_ldp_histogram(img, 3, 1))


def test_rectangular_cells_are_crops():
    """Rectangular-cell extension = crop + ldp_histogram per cell."""
    img = oracle.make_random(50, 70, 9)
    h = oracle.cell_histograms(img, 12, 17, 3)
    gr, gc = 50 // 12, 70 // 17
    assert h.shape == (gr * gc, 56)
    for i, j in itertools.product(range(gr), range(gc)):
        crop = img[i * 12:(i + 1) * 12, j * 17:(j + 1) * 17]
        assert np.array_equal(h[i * gc + j], oracle.ref_ldp_histogram(crop, 3, 1))


def test_batch_matches_single():
    rng = np.random.default_rng(11)
    px = rng.integers(0, 256, size=(5, 23, 29), dtype=np.uint8)
    for k in (1, 3, 5):
        c, h = oracle.batch(px, k=k, cell=(7, 9), threads=3)
        rc, rh = oracle.ref_batch(px, k=k, cell=(7, 9), threads=2)
        assert np.array_equal(c, rc) and np.array_equal(h, rh)
        for i in range(5):
            assert np.array_equal(c[i], oracle.code_map(px[i], k))
            assert np.array_equal(h[i], oracle.cell_histograms(px[i], 7, 9, k))


def test_errors():
    with pytest.raises(ValueError):
        oracle.ref_ldp_histogram(np.zeros((5, 5), np.uint8), 2)   # k != 3 throws
    with pytest.raises(ValueError):
        oracle.ref_ldp_histogram(np.zeros((2, 5), np.uint8), 3)   # < 3x3 throws
    with pytest.raises(ValueError):
        oracle.ref_windowed(np.zeros((10, 10), np.uint8), 2)      # window < 3
    with pytest.raises(ValueError):
        oracle.ref_windowed(np.zeros((10, 10), np.uint8), 11)     # window > image
    with pytest.raises(IndexError):
        oracle.ref_responses(np.zeros((5, 5), np.uint8), 5, 0)    # out_of_range

# ------------------------------------- response field / equivalence sweep

def _mm(m):
    return None if m is None else tuple(m)


def test_port_response_field_matches_reference(golden_fixtures, verify_vectors):
    """kirsch.cpp:193-208 on the reference's fixtures and reference outputs."""
    for fx in golden_fixtures:
        img = np.array(fx["pixels"], np.uint8).reshape(fx["rows"], fx["cols"])
        assert oracle.response_field(img).tolist() == fx["responses"], fx["name"]
    for f in verify_vectors["response_field"]:
        img = oracle.make_random(f["rows"], f["cols"], f["seed"])
        assert oracle.response_field(img).ravel().tolist() == f["field"]


def test_port_column_terms_reconstruct_naive():
    """kirsch.cpp:86-157: three column terms per response == the naive sum."""
    rng = np.random.default_rng(21)
    for _ in range(5):
        r, c = rng.integers(3, 12, size=2)
        img = rng.integers(0, 256, size=(r, c), dtype=np.uint8)
        for x in range(r):
            for y in range(c):
                assert np.array_equal(oracle.responses_terms(oracle.column_terms(img, x, y)),
                                      oracle.responses(img, x, y))


def test_port_verify_matches_reference_vectors(verify_vectors):
    """verify.cpp:37-111: counts, first mismatch and thread bookkeeping."""
    for c in verify_vectors["equivalence"]:
        got = oracle.verify_equivalence(c["images"], c["seed"], c["fault"], c["threads"])
        assert got == (c["images_checked"], c["pixels_checked"], _mm(c["mismatch"])), c
    for c in verify_vectors["image"]:
        img = oracle.make_random(c["rows"], c["cols"], c["seed"])
        got = oracle.verify_image(img, c["fault"], 0)
        assert got == (c["images_checked"], c["pixels_checked"], _mm(c["mismatch"])), c
    assert any(c["mismatch"] for c in verify_vectors["equivalence"])
    assert any(c["mismatch"] is None for c in verify_vectors["equivalence"])


@pytest.mark.skipif(not oracle.have_ref(), reason="reference library not built")
def test_port_verify_matches_reference_library():
    rng = np.random.default_rng(8)
    for _ in range(20):
        images, seed, threads = int(rng.integers(1, 20)), int(rng.integers(0, 2**32)), int(rng.integers(1, 9))
        fault = None if rng.random() < 0.3 else (int(rng.integers(0, images)), int(rng.integers(0, 5)),
                                                  int(rng.integers(0, 5)), int(rng.integers(0, 15)),
                                                  int(rng.integers(-3, 4)))
        assert oracle.verify_equivalence(images, seed, fault, threads) == \
            oracle.ref_verify_equivalence(images, seed, fault, threads)
