#!/usr/bin/env python3
"""SURVEY 8f ranks 3/4 measurements on one B200 box (not the driver's headline
bench). Prints JSON lines and writes the CSV reports under --out-dir:

  extract   `extract` over PGM files on local disk (--files 640x490 frames,
            face-like synthetic content written first, not timed): whole-run
            wall clock of aldp_extract_files (decode on host threads + H2D +
            B200 + D2H + CSV), images/s and MB/s of PGM input; beside it the
            reference's per-file path (load_pgm + ldp_histogram on one core,
            as the reference CLI runs) on a bounded sample.
  bench     the reference CLI's `bench` report in its CSV schema, B200 rows
            (aldp_bench_csv) and reference CPU rows (oracle/_ref), both
            series, written to bench_{b200,reference}_{images,window}.csv.
"""
import argparse
import json
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--files", type=int, default=2000)
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "gpurun_out"))
    ap.add_argument("--repeats", type=int, default=3)
    args = ap.parse_args()
    os.makedirs(args.out_dir, exist_ok=True)

    import numpy as np

    import oracle
    import paper_1810_11518_b200 as aldp
    from bench import numpy_faces

    tmp = tempfile.mkdtemp(prefix="aldp_pgm_")
    try:
        rows, cols = 490, 640
        base = numpy_faces(32, rows, cols, 20, 1810)
        paths = []
        for i in range(args.files):
            p = os.path.join(tmp, f"f{i:05d}.pgm")
            aldp.save_pgm(p, base[i % len(base)])
            paths.append(p)
        in_bytes = sum(os.path.getsize(p) for p in paths)
        out_csv = os.path.join(tmp, "features.csv")
        for window in (0, 64):
            aldp.extract_files(paths[:64], "aldp", window, out_csv)  # warm-up (context, buffers)
            times = []
            for _ in range(args.repeats):
                t0 = time.perf_counter()
                aldp.extract_files(paths, "aldp", window, out_csv)
                times.append(time.perf_counter() - t0)
            sec = sorted(times)[len(times) // 2]
            # reference per-file path on one core, bounded sample
            sample = paths[:24]
            t0 = time.perf_counter()
            for p in sample:
                img, err = oracle.ref_load_pgm(p) if oracle.have_ref() else (aldp.load_pgm(p), None)
                if window:
                    oracle.ref_windowed(img, window, 1)
                else:
                    oracle.ref_ldp_histogram(img, 3, 1)
            ref_ips = len(sample) / (time.perf_counter() - t0)
            print(json.dumps({
                "workload": f"extract_{'window64' if window else 'whole'}", "metric": "PGM files/s",
                "value": round(args.files / sec, 1), "unit": "images/s", "seconds": round(sec, 3),
                "files": args.files, "frame": f"{cols}x{rows}", "input_MB_s": round(in_bytes / sec / 1e6, 1),
                "csv_bytes": os.path.getsize(out_csv), "descriptor": "ALDP",
                "cpu_baseline": {"value": round(ref_ips, 2), "unit": "images/s", "cores": 1,
                                 "kind": "reference" if oracle.have_ref() else "port",
                                 "sample": f"{len(sample)} files: load_pgm + "
                                           f"{'windowed_features' if window else 'ldp_histogram'}"}}),
                  flush=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)

    for series in ("images", "window"):
        p = os.path.join(args.out_dir, f"bench_b200_{series}.csv")
        t0 = time.perf_counter()
        aldp.bench_csv(series, repeats=5, out_path=p)
        b200_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref = oracle.ref_bench_csv(series, repeats=5) if oracle.have_ref() else ""
        ref_s = time.perf_counter() - t0
        if ref:
            with open(os.path.join(args.out_dir, f"bench_reference_{series}.csv"), "w") as f:
                f.write(ref)
        print(json.dumps({"workload": f"bench_csv_{series}", "b200_csv": p, "b200_wall_s": round(b200_s, 2),
                          "reference_wall_s": round(ref_s, 2)}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
