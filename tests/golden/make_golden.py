#!/usr/bin/env python3
"""Regenerates the golden fixtures in this directory. Run in the dev
container (needs /root/reference and oracle/_ref/libaldp_ref.so); the GPU box
only reads the committed outputs.

Two sources, both the reference itself:
  1. The reference's own golden fixtures (reference tree
     proj/tests/golden/fixture_{ramp3,bump3,mixed4,spots5}.json, written by its
     brute-force generate.py) -- converted field-for-field into
     reference_fixtures.json (pixels, responses, k=3 codes, 56-bin histogram).
  2. Outputs of the UNMODIFIED reference library (oracle/_ref, compiled from
     proj/src) on seeded inputs -> ref_vectors.npz:
       * make_random images (the reference's own generator) of several sizes,
         with their k=1..7 code maps (ldp_code over responses_naive and
         responses_accelerated -- both must agree) and k=3 ldp_histogram;
       * tie-heavy {0,1,2} images with constant rectangles, k=1..7 code maps;
       * windowed_features(img, window, Ldp/Aldp/Lbp) for several windows;
       * LBP code maps and lbp_histogram (aldp::lbp_code / lbp_histogram);
       * the config-1 image: make_random(490, 640, 42), its code map digest
         and whole-image histogram.
  3. verify_vectors.json: aldp::verify_equivalence / verify_image results
     (images/pixels checked, first mismatch) of the reference library for a
     grid of seeds, faults and thread counts, and aldp::response_field of two
     seeded images (naive and accelerated paths).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

REF_GOLDEN = "/root/reference/proj/tests/golden"


def convert_reference_fixtures():
    out = []
    for name in ("fixture_ramp3", "fixture_bump3", "fixture_mixed4", "fixture_spots5"):
        with open(os.path.join(REF_GOLDEN, name + ".json")) as f:
            fx = json.load(f)
        out.append({k: fx[k] for k in ("name", "rows", "cols", "pixels", "responses", "ldp_codes",
                                       "ldp_histogram", "lbp_codes", "lbp_histogram")})
    with open(os.path.join(HERE, "reference_fixtures.json"), "w") as f:
        json.dump({"source": "reference proj/tests/golden/*.json (generate.py brute force)",
                   "fixtures": out}, f)
        f.write("\n")


def tie_image(rng, rows, cols):
    img = rng.integers(0, 3, size=(rows, cols), dtype=np.uint8)
    for _ in range(max(1, rows * cols // 200)):
        h, w = rng.integers(2, max(3, rows // 2)), rng.integers(2, max(3, cols // 2))
        x, y = rng.integers(0, rows), rng.integers(0, cols)
        img[x:x + h, y:y + w] = rng.integers(0, 3)
    return img


def ref_lbp(img):
    codes, hist = oracle.ref_batch(img, k=0, threads=1)  # aldp::lbp_code / lbp_histogram
    return codes[0], hist[0, 0]


def ref_code_maps(img):
    maps = []
    for k in range(1, 8):
        naive, _ = oracle.ref_batch(img, k=k, hist=False, path=0, threads=1)
        accel, _ = oracle.ref_batch(img, k=k, hist=False, path=1, threads=1)
        assert np.array_equal(naive, accel), "reference paths disagree"
        maps.append(naive[0])
    return np.stack(maps)


VERIFY_CASES = [
    # (images, seed, fault (image, x, y, term, delta) or None, threads)
    (1, 0, None, 1), (40, 7, None, 1), (40, 7, None, 4), (0, 3, None, 1),
    (30, 9, (3, 2, 1, 0, 1), 1), (30, 9, (3, 2, 1, 11, -5), 3), (30, 9, (17, 1, 1, 14, 3), 8),
    (30, 9, (10, 100, 1, 2, 1), 2), (30, 9, (0, 0, 0, 8, 0), 1), (30, 9, (29, 2, 2, 5, 7), 5),
    (12, 1234567, (4, 0, 0, 3, -1), 1), (12, 1234567, (4, 0, 0, 3, -1), 12),
    (64, 99, (63, 1, 2, 13, 100), 7), (64, 99, (5, 2, 2, 6, 1), 7),
] + [(25, 2024, (7, 1, 1, t, 2), 1) for t in range(15)] + [
    (1000, 42, None, 1), (1000, 42, (0, 1, 1, 0, 1), 1),  # the CLI's `verify` defaults (aldp_main.cpp:97-126)
]


def write_verify_vectors():
    cases = []
    for images, seed, fault, threads in VERIFY_CASES:
        ic, pc, mm = oracle.ref_verify_equivalence(images, seed, fault, threads)
        cases.append({"images": images, "seed": seed, "fault": fault, "threads": threads,
                      "images_checked": ic, "pixels_checked": pc, "mismatch": mm})
    img_cases = []
    for i, (r, c) in enumerate([(3, 3), (9, 14), (33, 20)]):
        img = oracle.ref_make_random(r, c, 500 + i)
        for fault in (None, (0, r // 2, c // 2, 4, 1), (1, 0, 0, 4, 1), (0, r - 1, c - 1, 12, -9)):
            ic, pc, mm = oracle.ref_verify_image(img, fault, 0)
            img_cases.append({"rows": r, "cols": c, "seed": 500 + i, "fault": fault,
                              "images_checked": ic, "pixels_checked": pc, "mismatch": mm})
    fields = []
    for r, c, seed in ((5, 7, 61), (34, 41, 62)):
        img = oracle.ref_make_random(r, c, seed)
        naive, accel = oracle.ref_response_field(img, 0), oracle.ref_response_field(img, 1)
        assert np.array_equal(naive, accel)
        fields.append({"rows": r, "cols": c, "seed": seed, "field": naive.ravel().tolist()})
    with open(os.path.join(HERE, "verify_vectors.json"), "w") as f:
        json.dump({"source": "reference verify_equivalence / verify_image / response_field via oracle/_ref",
                   "equivalence": cases, "image": img_cases, "response_field": fields}, f)
        f.write("\n")


def main():
    convert_reference_fixtures()
    write_verify_vectors()
    rng = np.random.default_rng(1810)
    vec = {}
    sizes = [(3, 3), (3, 7), (5, 4), (16, 16), (17, 31), (40, 64), (64, 130)]
    for i, (r, c) in enumerate(sizes):
        img = oracle.ref_make_random(r, c, 1000 + i)
        vec[f"rand{i}_img"] = img
        vec[f"rand{i}_codes"] = ref_code_maps(img)
        vec[f"rand{i}_hist"] = oracle.ref_ldp_histogram(img, 3, 1)
        vec[f"rand{i}_lbpcodes"], vec[f"rand{i}_lbphist"] = ref_lbp(img)
    for i, (r, c) in enumerate([(3, 3), (9, 12), (32, 48), (57, 200)]):
        img = tie_image(rng, r, c)
        vec[f"tie{i}_img"] = img
        vec[f"tie{i}_codes"] = ref_code_maps(img)
        vec[f"tie{i}_hist"] = oracle.ref_ldp_histogram(img, 3, 1)
        vec[f"tie{i}_lbpcodes"], vec[f"tie{i}_lbphist"] = ref_lbp(img)
    big = oracle.ref_make_random(96, 128, 77)
    vec["win_img"] = big
    for w in (3, 10, 25, 32, 64, 96):
        ldp = oracle.ref_windowed(big, w, 0)
        aldp = oracle.ref_windowed(big, w, 1)
        assert np.array_equal(ldp, aldp)
        vec[f"win{w}"] = aldp
        _, lbpw = oracle.ref_batch(big, k=0, cell=(w, w), codes=False, threads=1)  # windowed_features(Lbp)
        vec[f"winlbp{w}"] = lbpw[0]
    c1 = oracle.ref_make_random(490, 640, 42)
    c1_codes, c1_hist = oracle.ref_batch(c1, k=3, threads=os.cpu_count())
    vec["c1_img_sha256"] = np.frombuffer(hashlib.sha256(c1.tobytes()).digest(), np.uint8)
    vec["c1_codes_sha256"] = np.frombuffer(hashlib.sha256(c1_codes[0].tobytes()).digest(), np.uint8)
    vec["c1_hist"] = c1_hist[0, 0]
    np.savez_compressed(os.path.join(HERE, "ref_vectors.npz"), **vec)
    print("wrote", os.path.join(HERE, "reference_fixtures.json"), "and ref_vectors.npz")


if __name__ == "__main__":
    main()
