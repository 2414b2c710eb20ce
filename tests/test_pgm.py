"""SURVEY 8f ranks 3/4 host side, CPU only: the PGM loader/saver against the
reference's own tests (test_image.cpp:90-160) and, differentially, against
the reference's load_pgm itself (oracle/_ref) on valid and malformed files;
the op-count model; the command-line front end's argument handling."""
import os
import subprocess

import numpy as np
import pytest

import oracle

aldp = pytest.importorskip("paper_1810_11518_b200")

needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="reference library not built")


def write(tmp_path, name, data):
    p = tmp_path / name
    p.write_bytes(data if isinstance(data, bytes) else data.encode())
    return str(p)


def ours(path):
    try:
        return aldp.load_pgm(path), None
    except aldp.PgmError as e:
        return None, str(e)


# ------------------------------------------------ reference KATs (restated)

def test_ascii_pgm_loads_exactly(tmp_path):
    p = write(tmp_path, "ascii.pgm", "P2\n# a comment\n3 3\n255\n0 1 2\n3 4 5\n6 7 8\n")
    img = aldp.load_pgm(p)
    assert img.shape == (3, 3) and list(img.ravel()) == list(range(9))


def test_p5_and_p2_load_identically(tmp_path):
    original = oracle.make_random(5, 4, 77)
    p5, p2 = str(tmp_path / "same.p5.pgm"), str(tmp_path / "same.p2.pgm")
    aldp.save_pgm(p5, original)
    aldp.save_pgm(p2, original, ascii=True)
    assert np.array_equal(aldp.load_pgm(p5), aldp.load_pgm(p2))
    assert np.array_equal(aldp.load_pgm(p5), original)


def test_binary_round_trip(tmp_path):
    rng = np.random.default_rng(5)
    for _ in range(10):
        r, c = rng.integers(3, 23, size=2)
        img = oracle.make_random(int(r), int(c), int(rng.integers(0, 2**32)))
        p = str(tmp_path / "roundtrip.pgm")
        aldp.save_pgm(p, img)
        assert np.array_equal(aldp.load_pgm(p), img)


@pytest.mark.parametrize("name,data,needle", [
    ("magic.pgm", "P6\n3 3\n255\n", "not a PGM file"),
    ("depth.pgm", "P2\n3 3\n65535\n0 0 0 0 0 0 0 0 0\n", "bit depth"),
    ("trunc5.pgm", b"P5\n3 3\n255\n\x01\x02\x03", "truncated"),
    ("trunc2.pgm", "P2\n3 3\n255\n1 2 3 4\n", "truncated"),
    ("overmax.pgm", "P2\n3 3\n10\n0 1 2 3 4 5 6 7 99\n", "malformed pixel value '99'"),
    ("dims.pgm", "P2\nthree 3\n255\n", "malformed width 'three'"),
])
def test_malformed_pgm_rejected(tmp_path, name, data, needle):
    p = write(tmp_path, name, data)
    with pytest.raises(aldp.PgmError, match=needle):
        aldp.load_pgm(p)
    with pytest.raises(RuntimeError):  # the reference's exception family
        aldp.load_pgm(p)


def test_missing_file(tmp_path):
    p = str(tmp_path / "does_not_exist.pgm")
    with pytest.raises(aldp.PgmError, match="cannot open file"):
        aldp.load_pgm(p)


# ------------------------------------------- differential vs the reference

def _cases():
    img = oracle.make_random(4, 5, 3)
    body = img.tobytes()
    ascii_body = "\n".join(" ".join(str(v) for v in row) for row in img)
    cases = [
        b"P5\n5 4\n255\n" + body,
        b"P5 5 4 255 " + body,
        b"P5\n#c\n5 4\n255\n" + body,
        b"P5\n5#x\n4 255\n" + body,                      # comment inside a token
        b"P5\n5 4\n255#x\n" + body,
        b"P5\n5 4\n255\n\n" + body,                       # two separator bytes
        b"P5\n5 4\n255" + body,                           # no separator
        b"P5\n5 4\n255\n" + body[:-1],                    # truncated
        b"P5\n5 4\n255\n" + body + b"trailing",
        b"P5\n5 4\n200\n" + body,                         # values above maxval
        b"P5\n5 4\n0\n" + body,
        b"P5\n+5 4\n255\n" + body,
        b"P5\n-5 4\n255\n" + body,
        b"P5\n0 4\n255\n" + body,
        b"P5\n05 004\n255\n" + body,
        b"P5\n5 4\n256\n" + body,
        b"P5\n99999999999 4\n255\n" + body,
        b"P5\n5 4\n", b"P5\n5", b"P5", b"", b"P3\n5 4\n255\n",
        b"P5\n5x 4\n255\n" + body,
        ("P2\n5 4\n255\n" + ascii_body + "\n").encode(),
        ("P2 5 4 255 " + ascii_body).encode(),
        ("P2\n5 4\n255\n" + ascii_body.replace(" ", " +", 3)).encode(),
        ("P2\n5 4\n255\n" + ascii_body.replace(" ", " -", 1)).encode(),
        ("P2\n5 4\n255\n" + ascii_body.replace(" ", "#c\n", 2)).encode(),
        ("P2\n5 4\n255\n" + ascii_body[:-2]).encode(),
        ("P2\n5 4\n255\n" + ascii_body.replace(" ", " 1x", 1)).encode(),
        ("P2\n5 4\n255\n" + ascii_body.replace(" ", " 0012 ", 1)).encode(),
        ("P2\n5 4\n100\n" + ascii_body).encode(),
        b"P2\n1 1\n255\n7\n",
        b"P5\n1 1\n255\n\x07",
    ]
    rng = np.random.default_rng(99)
    base = b"P2\n# x\n3 2\n9\n1 2 3\n4 5 6\n"
    for _ in range(120):  # random byte-level mutations of small headers
        b = bytearray(base if rng.random() < 0.5 else b"P5\n3 2\n9\n\x01\x02\x03\x04\x05\x06")
        for _ in range(int(rng.integers(1, 4))):
            i = int(rng.integers(0, len(b)))
            op = rng.integers(0, 3)
            if op == 0:
                b[i] = int(rng.choice(list(b" \n#0123456789+-Px\t")))
            elif op == 1:
                del b[i]
            else:
                b.insert(i, int(rng.choice(list(b" \n#09+-"))))
        cases.append(bytes(b))
    return cases


@needs_ref
def test_load_pgm_matches_reference_on_valid_and_malformed(tmp_path):
    for i, data in enumerate(_cases()):
        p = write(tmp_path, f"c{i}.pgm", data)
        want_px, want_err = oracle.ref_load_pgm(p)
        got_px, got_err = ours(p)
        assert got_err == want_err, (i, data[:40])
        if want_px is not None:
            assert np.array_equal(got_px, want_px), (i, data[:40])


@needs_ref
def test_save_pgm_bytes_match_reference(tmp_path):
    img = oracle.make_random(7, 9, 11)
    for ascii in (False, True):
        a, b = str(tmp_path / "a.pgm"), str(tmp_path / "b.pgm")
        aldp.save_pgm(a, img, ascii=ascii)
        oracle.ref_save_pgm(b, img, ascii=ascii)
        assert open(a, "rb").read() == open(b, "rb").read()


def test_load_pgm_batch(tmp_path):
    imgs = [oracle.make_random(6, 8, s) for s in range(5)]
    paths = []
    for i, im in enumerate(imgs):
        paths.append(str(tmp_path / f"b{i}.pgm"))
        aldp.save_pgm(paths[-1], im, ascii=bool(i % 2))
    out = aldp.load_pgm_batch(paths, 6, 8, threads=3)
    assert np.array_equal(out, np.stack(imgs))
    with pytest.raises(ValueError):
        aldp.load_pgm_batch(paths, 8, 6)
    with pytest.raises(aldp.PgmError):
        aldp.load_pgm_batch(paths + [str(tmp_path / "missing.pgm")], 6, 8)


# ------------------------------------------------------------ op counts

def test_op_counts():
    assert aldp.op_counts("ldp") == (72, 64)
    assert aldp.op_counts("lbp") == (0, 8)
    m, a = aldp.op_counts("aldp")
    assert m <= 30 and a <= 46
    if oracle.have_ref():
        for code, name in ((0, "ldp"), (1, "aldp"), (2, "lbp")):
            assert aldp.op_counts(name) == oracle.ref_op_counts(code)


# ------------------------------------------------- CLI argument handling

def cli(*args):
    return subprocess.run([aldp.CLI_PATH, *args], capture_output=True, text=True, timeout=120)


def test_cli_usage_and_errors(tmp_path):
    assert cli("--help").returncode == 0
    assert cli().returncode == 2
    assert cli("frobnicate").returncode == 2
    r = cli("extract", "x.pgm", "--window", "2")
    assert r.returncode == 2 and "--window must be >= 3" in r.stderr
    r = cli("bench", "--repeats", "2")
    assert r.returncode == 2 and "--repeats must be at least 3" in r.stderr
    missing = str(tmp_path / "nope.pgm")
    r = cli("extract", missing)
    assert r.returncode == 2 and f"error: {missing}: cannot open file" in r.stderr
    assert r.stdout.startswith("identifier,descriptor,bin_0,")  # header streams first
    r = cli("extract", missing, "--descriptor", "hog")
    assert r.returncode == 2
    assert cli("verify", "--images").returncode == 2
