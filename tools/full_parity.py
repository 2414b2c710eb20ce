#!/usr/bin/env python3
"""Full-size parity: every frame of every BASELINE config, B200 kernel vs the
unmodified reference library (oracle/_ref, all host cores).

For C1..C5 at the sizes bench.py runs (C3 for k = 1, 3 and 5), the frames are
generated on the device exactly as bench.py does, the fast kernel computes the
code maps and histograms, and the same bytes copied to the host go through the
reference's own functions (ldp_histogram / windowed_features semantics via
oracle.ref_batch). Code maps and histograms must match bit for bit.

Test infrastructure (a checker, like tests/): the measured product path is
bench.py. Writes one JSON line per config to stdout.

    python tools/full_parity.py [--configs c1,c2,c3,c4,c5] [--chunk 2048]
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
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--chunk", type=int, default=2048)
    args = ap.parse_args()

    import numpy as np
    import torch
    import oracle
    import paper_1810_11518_b200 as aldp
    from bench import CONFIGS

    if not oracle.have_ref():
        print(json.dumps({"error": "reference library (oracle/_ref) not built"}))
        return 1
    dev = torch.device("cuda", 0)
    threads = os.cpu_count() or 1
    runs = []
    for name in args.configs.split(","):
        n, rows, cols, k, cr, cc, blobs, gen, seed = CONFIGS[name]
        for kk in ((1, 3, 5) if name == "c3" else (k,)):
            runs.append((name, n, rows, cols, kk, cr, cc, blobs, gen, seed))

    for name, n, rows, cols, k, cr, cc, blobs, gen, seed in runs:
        t0 = time.perf_counter()
        code_bad = hist_bad = frames_bad = 0
        checked = 0
        chunk = max(1, min(args.chunk, n))
        for a in range(0, n, chunk):
            m = min(chunk, n - a)
            if gen == "faces":
                px = aldp.gen_faces(m, rows, cols, blobs=blobs, seed=seed, first_index=a, pitch=cols, device=dev)
            elif gen == "ties":
                px = aldp.gen_ties(m, rows, cols, seed=seed, first_index=a, pitch=cols, device=dev)
            else:
                px = torch.from_numpy(oracle.make_random(rows, cols, seed)[None].copy()).to(dev)
            codes, hist = aldp.ldp_batch(px, rows, cols, k=k, cell=(cr, cc), codes=True, hist=True)
            torch.cuda.synchronize()
            host = px.cpu().numpy()
            g_codes = codes.cpu().numpy()
            g_hist = hist.cpu().numpy().astype(np.uint64)
            del px, codes, hist
            r_codes, r_hist = oracle.ref_batch(host, k=k, cell=(cr, cc), threads=threads)
            dc = g_codes[:, :, :cols] != r_codes
            dh = g_hist != r_hist
            code_bad += int(dc.sum())
            hist_bad += int(dh.sum())
            frames_bad += int((dc.reshape(m, -1).any(1) | dh.reshape(m, -1).any(1)).sum())
            checked += m
        line = {"config": name, "k": k, "frames": checked, "rows": rows, "cols": cols, "cell": [cr, cc],
                "pixels": checked * rows * cols, "code_mismatches": code_bad, "hist_mismatches": hist_bad,
                "frames_with_mismatch": frames_bad, "bit_exact": code_bad == 0 and hist_bad == 0,
                "checker": f"reference library (oracle/_ref, ResponsePath::Accelerated), {threads} host threads",
                "seconds": round(time.perf_counter() - t0, 1)}
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
