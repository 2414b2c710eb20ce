"""GPU parity for SURVEY 8f ranks 3/4: `extract` over PGM files (the CSV the
reference CLI writes, aldp_main.cpp:59-96) checked cell by cell against the
CPU oracle; the command-line verify/compare output against the reference's
own results (tests/golden/verify_vectors.json); the bench CSV schema
(bench.cpp:169-178) with B200 rows."""
import csv
import io
import subprocess

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1810_11518_b200 as aldp  # noqa: E402

NAMES = {"lbp": "LBP", "ldp": "LDP", "aldp": "ALDP"}


def expected_csv(paths, imgs, descriptor, window):
    k = 0 if descriptor == "lbp" else 3
    nb = 256 if k == 0 else 56
    lines = ["identifier,descriptor," + ",".join(f"bin_{i}" for i in range(nb))]
    for p, img in zip(paths, imgs):
        if window:
            h = oracle.cell_histograms(img, window, window, k)
            for w, row in enumerate(h):
                lines.append(f"{p}#w{w},{NAMES[descriptor]}," + ",".join(str(int(v)) for v in row))
        else:
            row = oracle.histogram(img, k)
            lines.append(f"{p},{NAMES[descriptor]}," + ",".join(str(int(v)) for v in row))
    return "\n".join(lines) + "\n"


@pytest.fixture(scope="module")
def corpus(tmp_path_factory):
    """Mixed sizes and encodings, equal-size runs broken up (batching edge)."""
    d = tmp_path_factory.mktemp("pgm")
    rng = np.random.default_rng(7)
    shapes = [(49, 64)] * 5 + [(30, 31), (49, 64), (64, 49)] + [(100, 130)] * 3 + [(3, 3), (33, 40)]
    paths, imgs = [], []
    for i, (r, c) in enumerate(shapes):
        img = oracle.make_random(r, c, 100 + i) if i % 3 else \
            np.clip(rng.normal(128, 40, size=(r, c)), 0, 255).astype(np.uint8)
        p = str(d / f"img{i:02d}.pgm")
        aldp.save_pgm(p, img, ascii=(i % 4 == 1))
        paths.append(p)
        imgs.append(img)
    return paths, imgs


@pytest.mark.parametrize("descriptor", ["aldp", "ldp", "lbp"])
def test_extract_whole_images(corpus, tmp_path, descriptor):
    paths, imgs = corpus
    out = str(tmp_path / "f.csv")
    aldp.extract_files(paths, descriptor, 0, out, threads=4)
    assert open(out).read() == expected_csv(paths, imgs, descriptor, 0)


@pytest.mark.parametrize("descriptor,window", [("aldp", 3), ("ldp", 10), ("lbp", 16), ("aldp", 30)])
def test_extract_windows(corpus, tmp_path, descriptor, window):
    paths, imgs = corpus
    keep = [i for i, im in enumerate(imgs) if min(im.shape) >= window]
    paths = [paths[i] for i in keep]
    imgs = [imgs[i] for i in keep]
    out = str(tmp_path / "w.csv")
    aldp.extract_files(paths, descriptor, window, out, threads=3)
    assert open(out).read() == expected_csv(paths, imgs, descriptor, window)


def test_extract_many_files_crosses_groups(tmp_path):
    """More files than one decode group (256), so decoding overlaps extraction."""
    paths, imgs = [], []
    for i in range(300):
        img = oracle.make_random(20 + (i // 100), 24, i)
        p = str(tmp_path / f"m{i:03d}.pgm")
        aldp.save_pgm(p, img)
        paths.append(p)
        imgs.append(img)
    out = str(tmp_path / "m.csv")
    aldp.extract_files(paths, "aldp", 0, out)
    assert open(out).read() == expected_csv(paths, imgs, "aldp", 0)


def test_extract_failure_keeps_earlier_rows(corpus, tmp_path):
    paths, imgs = corpus
    bad = str(tmp_path / "missing.pgm")
    out = str(tmp_path / "e.csv")
    with pytest.raises(aldp.PgmError, match="cannot open file"):
        aldp.extract_files(paths[:3] + [bad] + paths[3:], "aldp", 0, out)
    assert open(out).read() == expected_csv(paths[:3], imgs[:3], "aldp", 0)
    with pytest.raises(ValueError):  # window larger than the 3x3 image
        aldp.extract_files(paths, "aldp", 40, str(tmp_path / "e2.csv"))


def test_cli_extract_stdout_matches(corpus):
    paths, imgs = corpus
    r = subprocess.run([aldp.CLI_PATH, "extract", *paths[:6], "--descriptor", "LDP", "--window=16"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    keep = [i for i in range(6) if min(imgs[i].shape) >= 16]
    assert r.stdout == expected_csv([paths[i] for i in keep], [imgs[i] for i in keep], "ldp", 16)


def test_load_batch_then_device_batch(corpus):
    paths, imgs = corpus
    same = [i for i in range(len(paths)) if imgs[i].shape == (49, 64)]
    px = aldp.load_pgm_batch([paths[i] for i in same], 49, 64)
    codes, hist = aldp.ldp_batch_host(px, k=3, cell=(16, 16))
    for j, i in enumerate(same):
        assert np.array_equal(hist[j].astype(np.uint64), oracle.cell_histograms(imgs[i], 16, 16, 3))


# ------------------------------------------------------------ verify / compare

def test_cli_verify_matches_reference(verify_vectors):
    cases = {(c["images"], c["seed"], tuple(c["fault"]) if c["fault"] else None): c
             for c in verify_vectors["equivalence"]}
    ok = cases[(1000, 42, None)]
    r = subprocess.run([aldp.CLI_PATH, "verify"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    m, a = aldp.op_counts("aldp")
    assert r.stdout == (f"equivalence OK: {ok['images_checked']} images, {ok['pixels_checked']} pixels, "
                        f"8 directions each\nop counts per pixel: ALDP ({m} mul, {a} add) LDP (72 mul, "
                        f"64 add) LBP (0 mul, 8 add)\n")
    bad = cases[(1000, 42, (0, 1, 1, 0, 1))]["mismatch"]
    r = subprocess.run([aldp.CLI_PATH, "verify", "--inject-fault", "--parallel"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 1
    assert r.stdout == (f"MISMATCH image {bad[0]} pixel ({bad[1]},{bad[2]}) direction {bad[3]}: naive {bad[4]} "
                        f"!= accelerated {bad[5]}\n")


def test_cli_compare(corpus):
    paths, _ = corpus
    r = subprocess.run([aldp.CLI_PATH, "compare", paths[0], paths[12]], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout == (f"{paths[0]}: identical (3136 pixels, 8 directions, 56 bins)\n"
                        f"{paths[12]}: identical (1320 pixels, 8 directions, 56 bins)\n")
    r = subprocess.run([aldp.CLI_PATH, "compare"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout == "seeded-256x256: identical (65536 pixels, 8 directions, 56 bins)\n"


# ------------------------------------------------------------ bench CSV

def test_bench_csv_schema(tmp_path):
    out = str(tmp_path / "b.csv")
    aldp.bench_csv("images", size=64, counts=(1, 3, 50), repeats=3, out_path=out)
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["descriptor", "images", "window", "grid_total", "elapsed_s", "mults_per_pixel",
                       "adds_per_pixel"]
    body = rows[1:]
    assert [(r[0], r[1], r[2], r[3]) for r in body] == [
        (d, n, "none", "1") for d in ("LBP", "LDP", "ALDP") for n in ("1", "3", "50")]
    for r in body:
        assert float(r[4]) > 0 and len(r[4].split(".")[1]) == 6
        assert (int(r[5]), int(r[6])) == aldp.op_counts(r[0].lower())
    r = subprocess.run([aldp.CLI_PATH, "bench", "--series", "window", "--windows", "25,100", "--repeats", "3",
                        "--descriptor", "aldp"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(io.StringIO(r.stdout)))
    assert [(x[0], x[1], x[2], x[3]) for x in rows[1:]] == [("ALDP", "1", "25", "144"), ("ALDP", "1", "100", "9")]
