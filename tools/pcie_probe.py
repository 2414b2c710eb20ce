#!/usr/bin/env python3
"""PCIe ceiling probe for the e2e number: pinned H2D alone, D2H alone, and
both directions at once on separate streams (the e2e pipeline's pattern)."""
import json
import time

import torch


def main():
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in (("h2d", lambda: d_a.copy_(h_in, non_blocking=True)),
                     ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        res[name + "_GBs"] = round(5 * n / (time.perf_counter() - t0) / 1e9, 2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res["bidir_each_GBs"] = round(5 * n / dt / 1e9, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
