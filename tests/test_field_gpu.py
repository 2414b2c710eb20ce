"""GPU parity for SURVEY 8f rank 2: the response-field export and the
device-side equivalence sweep, through the C-ABI, against the CPU oracle
(oracle/ldp_oracle.c, pinned in test_oracle.py) and the reference's own
outputs (tests/golden/verify_vectors.json). Bit-exact."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1810_11518_b200 as aldp  # noqa: E402

DEV = torch.device("cuda:0")


def to_dev(px, pitch=None):
    px = np.ascontiguousarray(px, np.uint8)
    if px.ndim == 2:
        px = px[None]
    n, r, c = px.shape
    pitch = pitch or (c + 15) // 16 * 16
    buf = np.zeros((n, r, pitch), np.uint8)
    buf[:, :, :c] = px
    return torch.from_numpy(buf).to(DEV)


def torch_field(d, rows, cols):
    """Plain torch fp32 reference: the eight 3x3 Kirsch masks as one conv2d
    over replicate-padded pixels (exact in fp32: |m| <= 3825)."""
    base = [-3, -3, 5, 5, 5, -3, -3, -3]
    ring = [(-1, -1), (-1, 0), (-1, 1), (0, 1), (1, 1), (1, 0), (1, -1), (0, -1)]
    w = torch.zeros(8, 1, 3, 3)
    for i in range(8):
        for j, (dx, dy) in enumerate(ring):
            w[i, 0, dx + 1, dy + 1] = base[(i + j) % 8]
    x = d[:, :, :cols].float().unsqueeze(1)
    x = torch.nn.functional.pad(x, (1, 1, 1, 1), mode="replicate")
    out = torch.nn.functional.conv2d(x, w.to(d.device))  # [n, 8, rows, cols]
    return out.permute(0, 2, 3, 1).round().to(torch.int32)


def _mm(m):
    return None if m is None else tuple(m)


def _tuple(v):
    m = None if v.mismatch is None else (v.mismatch.image_index, v.mismatch.x, v.mismatch.y,
                                         v.mismatch.direction, v.mismatch.naive_value,
                                         v.mismatch.accelerated_value)
    return v.images_checked, v.pixels_checked, m


# ------------------------------------------------------------ response field

def test_response_field_reference_fixtures(golden_fixtures, verify_vectors):
    for fx in golden_fixtures:
        img = np.array(fx["pixels"], np.uint8).reshape(fx["rows"], fx["cols"])
        for path in (aldp.ResponsePath.Naive, aldp.ResponsePath.Accelerated):
            assert aldp.response_field(img, path).tolist() == fx["responses"], (fx["name"], path)
    for f in verify_vectors["response_field"]:
        img = oracle.make_random(f["rows"], f["cols"], f["seed"])
        assert aldp.response_field(img).ravel().tolist() == f["field"]


@pytest.mark.parametrize("shape", [(3, 3), (3, 40), (40, 3), (31, 33), (32, 32), (33, 17), (65, 130),
                                   (100, 7)])
def test_response_field_batch_vs_oracle(shape):
    r, c = shape
    rng = np.random.default_rng(r * 1000 + c)
    px = rng.integers(0, 256, size=(3, r, c), dtype=np.uint8)
    # padded pitch -> the bulk-copy (TMA) kernel; pitch == cols -> byte-staged kernel
    for d in (to_dev(px), to_dev(px, pitch=c)):
        _check_field(d, px, r, c)


def _check_field(d, px, r, c):
    for path in (aldp.ResponsePath.Naive, aldp.ResponsePath.Accelerated):
        f16 = aldp.response_field_batch(d, r, c, path=path)
        f32 = aldp.response_field_batch(d, r, c, path=path, wide=True)
        torch.cuda.synchronize()
        for i in range(px.shape[0]):
            want = oracle.response_field(px[i]).reshape(r, c, 8)
            assert np.array_equal(f16[i].cpu().numpy().astype(np.int32), want), (r, c, d.shape, path, i)
            assert np.array_equal(f32[i].cpu().numpy(), want), (r, c, d.shape, path, i)


def test_response_field_many_tiles_both_kernels():
    """More tiles than resident blocks (the double-buffered bulk pipeline
    wraps several times), widths straddling the 128-column tile edge."""
    rng = np.random.default_rng(3)
    for r, c in ((70, 129), (33, 256), (97, 300), (19, 1100), (5, 2100), (17, 1024), (18, 1027)):
        px = rng.integers(0, 256, size=(40, r, c), dtype=np.uint8)
        for d in (to_dev(px), to_dev(px, pitch=c)):
            f = aldp.response_field_batch(d, r, c)
            torch.cuda.synchronize()
            for i in (0, 17, 39):
                want = oracle.response_field(px[i]).reshape(r, c, 8)
                assert np.array_equal(f[i].cpu().numpy().astype(np.int32), want), (r, c, d.shape, i)


def test_response_field_extremes():
    """|m| <= 3825 attained (test_kirsch.cpp:288-315) survives the int16 store."""
    chk = np.array([[255 if ((x // 3 + y // 3) % 2 == 0) else 0 for y in range(9)] for x in range(9)],
                   np.uint8)
    f = aldp.response_field_batch(to_dev(chk), 9, 9)
    torch.cuda.synchronize()
    got = f[0].cpu().numpy().astype(np.int32)
    assert np.abs(got).max() == 3825
    assert np.array_equal(got, oracle.response_field(chk).reshape(9, 9, 8))


def test_response_field_full_size_vs_torch():  # noqa: C901
    """Config-5 frame size, 24 face images: against a torch fp32 conv2d and
    the size-independent identity sum_i m_i == 0 (8*3T - 8*3T)."""
    n, r, c = 24, 490, 640
    d = aldp.gen_faces(n, r, c, seed=5)
    f = aldp.response_field_batch(d, r, c)
    torch.cuda.synchronize()
    import os
    os.environ["ALDP_FIELD_NOBULK"] = "1"  # the byte-staged kernel on the same frames
    try:
        f_bytes = aldp.response_field_batch(d, r, c)
        torch.cuda.synchronize()
    finally:
        del os.environ["ALDP_FIELD_NOBULK"]
    assert torch.equal(f, f_bytes)
    ref = torch_field(d, r, c)
    torch.cuda.synchronize()
    assert torch.equal(f.to(torch.int32), ref)
    assert int(f.to(torch.int32).sum(dim=-1).abs().max()) == 0
    # the LDP codes the fast kernel emits are the top-3 of this field
    codes, _ = aldp.ldp_batch(d, r, c, k=3, codes=True)
    m = f.to(torch.int64)
    key = m * 8 + (7 - torch.arange(8, device=DEV))  # ties -> lower direction
    top = key.topk(3, dim=-1).indices
    want = (1 << top).sum(-1).to(torch.uint8)
    torch.cuda.synchronize()
    assert torch.equal(codes[:, :, :c], want)


def test_response_field_errors():
    with pytest.raises(ValueError):
        aldp.response_field(np.zeros((2, 5), np.uint8))
    d = to_dev(np.zeros((1, 2, 8), np.uint8))
    with pytest.raises(ValueError):
        aldp.response_field_batch(d, 2, 8)


# ------------------------------------------------------------ equivalence sweep

def test_verify_equivalence_matches_reference(verify_vectors):
    for c in verify_vectors["equivalence"]:
        fault = None if c["fault"] is None else aldp.FaultInjection(*c["fault"])
        got = aldp.verify_equivalence(c["images"], c["seed"], fault, c["threads"])
        assert _tuple(got) == (c["images_checked"], c["pixels_checked"], _mm(c["mismatch"])), c
        assert got.ok() == (c["mismatch"] is None)


def test_verify_image_matches_reference(verify_vectors):
    for c in verify_vectors["image"]:
        img = oracle.make_random(c["rows"], c["cols"], c["seed"])
        fault = None if c["fault"] is None else aldp.FaultInjection(*c["fault"])
        got = aldp.verify_image(img, fault, 0)
        assert _tuple(got) == (c["images_checked"], c["pixels_checked"], _mm(c["mismatch"])), c


def test_verify_equivalence_vs_oracle_random():
    rng = np.random.default_rng(44)
    for _ in range(25):
        images, seed, threads = int(rng.integers(1, 40)), int(rng.integers(0, 2**32)), int(rng.integers(1, 9))
        fault = None if rng.random() < 0.3 else (int(rng.integers(0, images)), int(rng.integers(0, 6)),
                                                  int(rng.integers(0, 6)), int(rng.integers(0, 15)),
                                                  int(rng.integers(-3, 4)))
        got = aldp.verify_equivalence(images, seed, None if fault is None else aldp.FaultInjection(*fault),
                                      threads)
        assert _tuple(got) == oracle.verify_equivalence(images, seed, fault, threads), (images, seed, fault)


def test_verify_batch_full_size_and_fault():
    """The sweep at config-5 scale: clean, then one injected fault found at
    exactly its pixel with the reference's counts."""
    n, r, c = 64, 490, 640
    d = aldp.gen_faces(n, r, c, seed=17)
    ok = aldp.verify_batch(d, r, c)
    assert ok.ok() and ok.images_checked == n and ok.pixels_checked == n * r * c and ok.mismatches == 0
    f = aldp.FaultInjection(image_index=41, x=489, y=7, term_index=11, delta=-2)
    bad = aldp.verify_batch(d, r, c, f)
    assert not bad.ok() and bad.mismatches == 3  # a11 feeds responses 5, 6, 7
    mm = bad.mismatch
    assert (mm.image_index, mm.x, mm.y, mm.direction) == (41, 489, 7, 5)
    assert mm.accelerated_value == mm.naive_value - 2
    assert bad.images_checked == 42 and bad.pixels_checked == 41 * r * c + 489 * c + 8
    host = d[41, :, :c].cpu().numpy()
    assert mm.naive_value == int(oracle.responses(host, 489, 7)[5])
    # threads only changes the bookkeeping: 8 chunks of 8 images
    t8 = aldp.verify_batch(d, r, c, f, threads=8)
    assert t8.images_checked == 64 - 6 and t8.pixels_checked == (64 - 7) * r * c + 489 * c + 8


def test_verify_errors():
    with pytest.raises(IndexError):
        aldp.verify_equivalence(3, 1, aldp.FaultInjection(0, 0, 0, 15, 1))
    with pytest.raises(ValueError):
        aldp.verify_image(np.zeros((2, 9), np.uint8))
    r = aldp.verify_equivalence(0, 5)  # clamped to one image
    assert r.images_checked == 1 and r.ok()
