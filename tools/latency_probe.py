#!/usr/bin/env python3
"""Per-call latency of the reference-facing host entry points (one image per
call, host buffers), the unit the reference's bench CSV times."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1810_11518_b200 as aldp  # noqa: E402


def per_call(fn, n=400):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    out = {}
    rng = np.random.default_rng(0)
    for side in (256, 260, 490):
        img = rng.integers(0, 256, size=(side, side), dtype=np.uint8)
        out[f"ldp_histogram_{side}_us"] = round(per_call(lambda: aldp.ldp_histogram(img)), 1)
        out[f"lbp_histogram_{side}_us"] = round(per_call(lambda: aldp.lbp_histogram(img)), 1)
    img = rng.integers(0, 256, size=(300, 300), dtype=np.uint8)
    out["windowed_300_w25_us"] = round(per_call(lambda: aldp.windowed_features(img, 25)), 1)
    out["code_map_260_us"] = round(per_call(lambda: aldp.ldp_code_map(rng.integers(0, 256, (260, 260), dtype=np.uint8))), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
