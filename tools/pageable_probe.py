#!/usr/bin/env python3
"""e2e host batch throughput from pinned vs pageable host memory (C5 frames)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_11518_b200 as aldp  # noqa: E402


def main():
    n, r, c = 2048, 490, 640
    d = aldp.gen_faces(n, r, c, seed=3)
    pinned = torch.empty((n, r, c), dtype=torch.uint8).pin_memory()
    pinned.copy_(d[:, :, :c])
    pageable = pinned.numpy().copy()
    out = {}
    for name, src in (("pinned", pinned.numpy()), ("pageable", pageable)):
        codes = np.empty_like(src) if name == "pageable" else torch.empty_like(pinned).pin_memory().numpy()
        hist = np.empty((n, 42, 56), np.uint32)
        def call():
            aldp._check(aldp.lib.aldp_ldp_batch_host(src.ctypes.data, n, r, c, 3, 81, 91, codes.ctypes.data,
                                                     hist.ctypes.data, None))
        call()
        t0 = time.perf_counter()
        for _ in range(5):
            call()
        dt = (time.perf_counter() - t0) / 5
        out[name + "_Gpx_s"] = round(n * r * c / dt / 1e9, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
