#!/usr/bin/env python3
"""Measures the SURVEY 8f rank-2 kernels on one B200 and prints one JSON line
per workload (not the driver's headline bench; see bench.py for that):

  field16   response_field_batch, int16 [n][rows][cols][8]: 1 B read + 16 B
            written per pixel (algorithmic), HBM roofline.
  field32   the int32 layout of the reference's ResponseVector (32 B/px).
  verify    verify_batch: the naive-vs-identity sweep, 1 B/px read (the
            kernel is compute-bound: 64 MADs of the literal masks per pixel).

Inputs: face-like 490x640 frames generated on the device, resident in HBM
before timing; outputs (>= 5 GB per step) exceed the 126 MB L2, so no flush
is needed. CPU baseline: the reference's response_field (oracle/_ref, or the
C port when the reference library is absent) on one image per thread.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_1810_11518_b200 as aldp
    import oracle
    sys.path.insert(0, ROOT)
    from bench import measured_peaks

    peak, peak_src = measured_peaks()
    n, rows, cols = args.images, 490, 640
    dev = torch.device("cuda:0")
    px = aldp.gen_faces(n, rows, cols, seed=11518)
    stream = torch.cuda.current_stream(dev)
    pixels = n * rows * cols

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps / 1e3

    # bounded CPU sample: the reference's response_field, Accelerated path
    host = px[:4, :, :cols].cpu().numpy()
    fn = (lambda im: oracle.ref_response_field(im, 1)) if oracle.have_ref() else oracle.response_field
    t0 = time.perf_counter()
    for im in host:
        fn(im)
    cpu_mpx = host[0].size * len(host) / (time.perf_counter() - t0) / 1e6
    cpu = {"value": round(cpu_mpx, 2), "unit": "Mpixel/s", "cores": 1,
           "kind": "reference" if oracle.have_ref() else "port",
           "sample": "4 frames 490x640, response_field(Accelerated), 1 thread"}

    for wide in (False, True):
        out = torch.empty((n, rows, cols, 8), dtype=torch.int32 if wide else torch.int16, device=dev)
        # write-only ceiling on this box: torch's fill kernel over the same buffer
        fill_sec = timed(lambda: out.fill_(1))
        fill_gbs = out.numel() * out.element_size() / fill_sec / 1e9
        sec = timed(lambda: aldp.response_field_batch(px, rows, cols, out=out, wide=wide))
        bpp = 1 + (32 if wide else 16)
        gbs = pixels * bpp / sec / 1e9
        print(json.dumps({
            "workload": "field32" if wide else "field16", "metric": "response field Gpixel/s",
            "value": round(pixels / sec / 1e9, 2), "unit": "Gpixel/s", "ms_per_step": round(sec * 1e3, 3),
            "images_per_step": n, "steps": args.steps, "warmup": args.warmup,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "bytes_per_pixel": bpp, "peak_source": peak_src,
                         "torch_fill_gbs": round(fill_gbs, 1)},
            "cpu_baseline": cpu}), flush=True)
        del out

    for _ in range(2):
        aldp.verify_batch(px, rows, cols)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = aldp.verify_batch(px, rows, cols)
    sec = (time.perf_counter() - t0) / args.steps  # synchronous call: host wall time
    assert r.ok() and r.pixels_checked == pixels
    print(json.dumps({
        "workload": "verify", "metric": "equivalence sweep Gpixel/s", "value": round(pixels / sec / 1e9, 2),
        "unit": "Gpixel/s", "ms_per_step": round(sec * 1e3, 3), "images_per_step": n,
        "timing": "host wall clock around the synchronous verify_batch call",
        # compute-bound: 72 multiplies of the literal masks + the identity per
        # pixel on the FMA pipe; the HBM fraction is shown only to say so
        "roofline": {"bound": "compute (FMA pipe: 72 IMAD + identity per pixel), not HBM",
                     "achieved": round(pixels / sec / 1e9, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(pixels / sec / 1e9 / peak, 4), "bytes_per_pixel": 1}}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
