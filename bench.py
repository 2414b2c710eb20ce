#!/usr/bin/env python3
"""LDP Mpixel/s benchmark (BASELINE.json metric) on 1..N B200s.

Workload (default, BASELINE.json configs[4] = "C5"): 65,536 face-like
640x490 uint8 images (GrayImage 490 x 640), LDP k=3, code map + 7x6 cell
histograms (cells 81 x 91, per-cell clamp = windowed_features semantics).
The batch is sharded by image across ranks (one process per GPU); each rank
generates its shard on device keyed by global image index, so every N sees
identical bytes. With N > 1 the per-image cell histograms are gathered to
rank 0 (NCCL, uint16 on the wire) inside the timed step, overlapped with the
kernels in --gather-chunks pieces on a comm stream. Total work is fixed ->
"strong". --force-dist runs the NCCL path at world size 1.

A "step" is one pass of the LDP path over the whole batch. Inputs (20.6 GB)
far exceed L2 (126 MB), so no L2 flush is needed between steps.

  value   : whole-job Mpixel/s, device-resident inputs, CUDA events on the
            launching stream, max over ranks (20 timed steps by default)
  e2e     : same metric through the host C-ABI entry point (aldp_ldp_batch_host)
            from pinned host memory: H2D pixels + kernel + D2H codes + D2H hist,
            every rank at once through its own PCIe link, max over ranks
  roofline: algorithmic bytes (1 B in + 1 B code + 4 B x 42 x 56 hist per image)
            per launch / average launch time, vs MEASURED_PEAKS.json hbm_gbs;
            traffic = ncu DRAM bytes per pixel (profiles/ncu_metrics.json, same build) at that rate
  clocks  : nvidia-smi samples during the timed region
  checksums: bin-weighted histogram sum and code-byte sum (identical at any N)
  cpu_baseline: the reference library (oracle/_ref, unmodified reference
            sources) on this box's host cores, bounded sample, timed with the
            reference's own median_seconds; host CPU described

`--impl reference` times the reference's own CPU implementation (oracle/_ref,
Accelerated path, all host threads) on a bounded sample per step; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n_images, rows, cols, k, cell_rows, cell_cols, blobs, generator, seed)
    "c5": (65536, 490, 640, 3, 81, 91, 20, "faces", 11518),
    "c2": (1024, 490, 640, 3, 81, 91, 20, "faces", 1810),
    "c4": (1, 16384, 16384, 3, 64, 64, 200, "faces", 42),
    "c3": (256, 1024, 1024, 3, 0, 0, 0, "ties", 11518),
    "c1": (1, 490, 640, 3, 0, 0, 0, "random", 42),
    # diagnostic: C5 images with whole-image histograms (cost of the cell grid)
    "c5w": (65536, 490, 640, 3, 0, 0, 20, "faces", 11518),
    # LBP (k = 0 selects the LBP descriptor) on the C5 batch
    "c5lbp": (65536, 490, 640, 0, 81, 91, 20, "faces", 11518),
    # the paper's window series (Table 3, windowed_features with
    # square windows of 10 / 25 px) on 2048 C5 frames: the narrow-cell kernel
    "w10": (2048, 490, 640, 3, 10, 10, 20, "faces", 11518),
    "w25": (2048, 490, 640, 3, 25, 25, 20, "faces", 11518),
}
WORKLOAD_NAMES = {
    "c5": "C5: 65536 x 640x490 face-like, LDP k=3, code map + 7x6 cell histograms",
    "c2": "C2: 1024 x 640x490 face-like, LDP k=3, code map + 7x6 cell histograms",
    "c4": "C4: 16384x16384 face-like (200 blobs), LDP k=3, code map + 64x64 cell histograms",
    "c3": "C3: 256 x 1024x1024 tie-heavy, LDP k=3, code map + whole-image histograms",
    "c1": "C1: 640x490 uniform random (make_random), LDP k=3, code map + histogram",
    "c5w": "C5 images, whole-image histograms (diagnostic)",
    "c5lbp": "C5 images, LBP (256-bin) code map + 7x6 cell histograms",
    "w10": "2048 C5 frames, LDP k=3, code map + windowed_features(window=10): 49x64 cells of 10x10",
    "w25": "2048 C5 frames, LDP k=3, code map + windowed_features(window=25): 19x25 cells of 25x25",
}


def workload_name(cfg, k):
    """The config's workload text, with the k actually run (--k overrides)."""
    name = WORKLOAD_NAMES[cfg]
    return name if k == 0 else name.replace("LDP k=3", f"LDP k={k}")


def hist_bytes_per_image(rows, cols, k, cr, cc):
    from math import comb
    cells = 1 if cr == 0 else (rows // cr) * (cols // cc)
    return cells * (256 if k == 0 else comb(8, k)) * 4


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=1)
        sm = sorted(float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit())
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4)
                          if r[4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx[0] if mx else None,
                "reasons": reasons, "samples": len(sm)}


def ncu_record(cfg):
    """Limiter counters of the fast kernel for this config from the ncu
    --set full capture recorded in profiles/ncu_metrics.json (tools/ncu_to_json.py),
    and whether that capture ran the library loaded now (sha256)."""
    import hashlib
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_metrics.json")) as f:
            rec = json.load(f).get(cfg)
    except (OSError, ValueError):
        return None
    if not rec:
        return None
    import paper_1810_11518_b200 as aldp
    try:
        sha = hashlib.sha256(open(aldp.LIB_PATH, "rb").read()).hexdigest()
    except OSError:
        sha = None
    rec = dict(rec)
    # same device code as the capture: the sm_100a sections of the embedded
    # cubins (a rebuild of identical code changes the .so's bytes -- nvcc's
    # temporary names in the debug strings -- but not these)
    code = aldp.device_code_fingerprint()
    rec["same_build"] = bool((code is not None and code == rec.get("device_code_sha256")) or
                             (sha is not None and sha == rec.get("lib_sha256")))
    return rec


def limiter_of(rec, cfg=None):
    """The measured limiter from the ncu counters of the same build: the units
    closest to their peak among DRAM, the L1/shared data pipe, the ALU pipe
    and instruction issue. A unit at >= 80 % is named as the bound; below
    that all four are listed, with what the A/B series of the cell kernel
    says it waits on."""
    if not rec:
        return None
    units = {"l1_data_pipe": rec.get("l1_data_pipe_pct", 0.0), "alu_pipe": rec.get("alu_pipe_pct", 0.0),
             "issue": rec.get("issue_active_pct", 0.0), "dram": rec.get("dram_throughput_pct", 0.0)}
    order = sorted(units, key=units.get, reverse=True)
    listed = ", ".join(f"{u} {units[u]:.1f} %" for u in order)
    if units[order[0]] >= 80.0:
        return f"{order[0]}-bound ({listed})"
    out = f"no unit at 80 % of peak ({listed})"
    if cfg in ("c5", "c4", "c2"):  # the 81x91 / 64x64 cell kernel the A/B series and the probe ran on
        out += ("; A/B of this kernel's key formation prices one ALU-pipe instruction at ~2.8 FMA-pipe ones "
                "(profiles/r02m_pixel_layer_ab.txt): it waits on the ALU pipe, which runs every min/max of the "
                "top-3 network (that network alone, on a 100 % busy ALU pipe, caps at 64 % of HBM); removing every "
                "per-pixel shared access drops the L1 pipe to 24 % for +8 % only "
                "(profiles/r02_ncu_shared_ceiling_probe.txt)")
    return out


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------------------
# CPU-side synthetic input for the reference arm (no GPU code on that path):
# same recipe as the device generator (gradient + blobs + N(0,6) noise).
# --------------------------------------------------------------------------
def numpy_faces(n, rows, cols, blobs, seed):
    import numpy as np
    rng = np.random.default_rng(seed)
    out = np.empty((n, rows, cols), np.uint8)
    xx, yy = np.meshgrid(np.arange(rows, dtype=np.float32), np.arange(cols, dtype=np.float32),
                         indexing="ij")
    for i in range(n):
        th = rng.uniform(0, 2 * math.pi)
        lo, hi = rng.uniform(40, 120), rng.uniform(120, 220)
        cx, cy = math.cos(th), math.sin(th)
        span = abs(cx) * (rows - 1) + abs(cy) * (cols - 1) + 1e-6
        t = (cx * xx + cy * yy - min(0, cx * (rows - 1)) - min(0, cy * (cols - 1))) / span
        v = lo + (hi - lo) * t
        for _ in range(blobs):
            bx, by = rng.uniform(0, rows), rng.uniform(0, cols)
            s, a = rng.uniform(5, 60), rng.uniform(-80, 80)
            v += a * np.exp(-((xx - bx) ** 2 + (yy - by) ** 2) / (2 * s * s))
        v += rng.normal(0, 6, size=v.shape)
        out[i] = np.clip(np.rint(v), 0, 255).astype(np.uint8)
    return out


def device_inputs(gen, n, rows, cols, blobs, seed, rows_kept=None):
    """The B200 arm's synthetic inputs (device generator keyed by image index
    from 0), copied back to the host: [n, rows_kept, cols] uint8."""
    import torch
    import paper_1810_11518_b200 as aldp
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    if gen == "faces":
        d = aldp.gen_faces(n, rows, cols, blobs=blobs, seed=seed, pitch=cols, device=dev)
    elif gen == "ties":
        d = aldp.gen_ties(n, rows, cols, seed=seed, pitch=cols, device=dev)
    else:
        raise ValueError(gen)
    torch.cuda.synchronize(dev)
    out = d[:, :rows_kept or rows, :cols].cpu().numpy()
    del d
    torch.cuda.empty_cache()
    return out


def run_reference(args, cfg_name):
    """--impl reference: the reference's CPU implementation (oracle/_ref)."""
    import numpy as np
    import oracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, rows, cols, k, cr, cc, blobs, gen, seed = CONFIGS[cfg_name]
    if args.k >= 0:
        k = args.k
    threads = os.cpu_count() or 1
    sample = max(threads * 4, 32) if cfg_name in ("c5", "c2", "c5w", "c5lbp", "w10", "w25") else \
        (threads if cfg_name == "c3" else 1)
    # Inputs: the product arm's own bytes -- the device generator's output for
    # images 0 .. sample-1 (or C4's first 1024 rows), copied back before any
    # timing; only the reference library runs in the timed loop.
    src = "device generator bytes (same as the B200 arm), copied to the host untimed"
    try:
        px = device_inputs(gen, sample if rows * cols < 1e8 else 1, rows, cols, blobs, seed,
                           rows_kept=1024 if rows * cols >= 1e8 else rows)
    except Exception as e:  # noqa: BLE001 -- no GPU: the numpy restatement of the recipe
        src = f"numpy restatement of the generator ({type(e).__name__}: no device)"
        px = None
    if gen == "random":
        px = oracle.ref_make_random(rows, cols, seed)[None]  # the reference's own generator
        src = "reference make_random (mt19937)"
    elif px is None and gen == "faces":
        px = numpy_faces(sample if rows * cols < 1e8 else 1, rows if rows * cols < 1e8 else 1024, cols,
                         blobs if rows * cols < 1e8 else max(1, blobs // 16), seed)
    elif px is None:
        px = np.random.default_rng(seed).integers(0, 3, size=(sample, rows, cols), dtype=np.uint8)
    if rows * cols >= 1e8:
        # C4: a band of the 16384^2 frame (1024 rows), cut into one row band of
        # whole 64-row cells per host thread -- cells are clamped independently,
        # so the bands are exactly the frame's work for those rows
        band = px[0]
        px = band.reshape(band.shape[0] // cr, cr, cols) if cr else band[None]
    kind = "reference" if oracle.have_ref() else "port"
    run = (lambda: oracle.ref_batch(px, k=k, cell=(cr, cc), threads=threads)) if kind == "reference" \
        else (lambda: oracle.batch(px, k=k, cell=(cr, cc), threads=threads))
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    dt = (time.perf_counter() - t0) / args.steps
    mpx = px.size / dt / 1e6
    # The reference has no fused code-map + histogram entry point: the line's
    # value runs its per-pixel ldp_code for the map and its ldp_histogram /
    # windowed_features for the histograms (two passes). Beside it, untimed by
    # the driver's ratio: the histogram pass alone, once over the same sample.
    hist_only = None
    if kind == "reference":
        t1 = time.perf_counter()
        oracle.ref_batch(px, k=k, cell=(cr, cc), codes=False, threads=threads)
        hist_only = round(px.size / (time.perf_counter() - t1) / 1e6, 3)
    line = {
        "impl": "reference", "metric": f"{'LBP' if k == 0 else 'LDP'} Mpixel/s (code map + histograms)",
        "value": round(mpx, 3),
        "unit": "Mpixel/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": f"synthetic: {src}",
        "config": {"workload": workload_name(cfg_name, k), "images_per_step": int(px.shape[0]),
                   "parallelism": f"{threads} host threads over images", "cpu_only": True},
        "cpu_baseline": {"value": round(mpx, 3), "unit": "Mpixel/s", "cores": threads, "kind": kind,
                         "sample": f"{px.shape[0]} images of {px.shape[1]}x{px.shape[2]} per step, "
                                   f"{'LBP' if k == 0 else 'ALDP (ResponsePath::Accelerated)'}, "
                                   f"code map + histograms"},
        "e2e": {"value": round(mpx, 3), "unit": "Mpixel/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_passes": {"code_map_and_histograms": round(mpx, 3), "histograms_only": hist_only,
                             "note": "no fused entry point in the reference: the map is its per-pixel "
                                     "ldp_code pass, the histograms its ldp_histogram / windowed_features "
                                     "pass; histograms_only is that second pass alone (one run)"},
    }
    print(json.dumps(line), flush=True)
    return 0


def host_info():
    """nproc, CPU model, sockets, cores and hardware threads of this box."""
    info = {"nproc": os.cpu_count()}
    try:
        model, phys, cores, sibl = None, set(), {}, {}
        cur = None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name" and model is None:
                model = v
            elif k == "physical id":
                cur = v
                phys.add(v)
            elif k == "cpu cores" and cur is not None:
                cores[cur] = int(v)
            elif k == "siblings" and cur is not None:
                sibl[cur] = int(v)
        info.update({"model": model, "sockets": len(phys) or 1,
                     "cores": sum(cores.values()) or None, "threads": sum(sibl.values()) or None})
    except OSError:
        pass
    return info


def cpu_baseline(host_px, k, cr, cc):
    """Reference library on this box's host cores, bounded sample, timed with
    the reference's own median_seconds (bench.cpp:51-78) when the reference
    library is present."""
    import oracle
    threads = os.cpu_count() or 1
    kind = "reference" if oracle.have_ref() else "port"
    res = {}
    n = host_px.shape[0]
    # *_hist_only: the histograms alone (ldp_histogram / windowed_features, the
    # reference API's one pass); the others also build the code map, which the
    # reference only has as a second pass (no fused entry point)
    for label, path, nthreads, count, codes in (
            ("aldp_all_cores", 1, threads, n, True), ("ldp_all_cores", 0, threads, n // 2, True),
            ("aldp_hist_only_all_cores", 1, threads, n, False),
            ("aldp_1_thread", 1, 1, max(1, n // threads), True),
            ("ldp_1_thread", 0, 1, max(1, n // threads // 2), True)):
        sub = host_px[:max(count, 1)]
        if kind == "reference":
            dt = oracle.ref_median_seconds_batch(sub, k=k, cell=(cr, cc), path=path, threads=nthreads, repeats=3,
                                                 codes=codes)
        else:
            t0 = time.perf_counter()
            oracle.batch(sub, k=k, cell=(cr, cc), threads=nthreads, codes=codes)
            dt = time.perf_counter() - t0
        res[label] = round(sub.size / dt / 1e6, 3)
    return {"value": res["aldp_all_cores"], "unit": "Mpixel/s", "cores": threads, "kind": kind,
            "sample": f"{n} images of {host_px.shape[1]}x{host_px.shape[2]} (taken from the start of the "
                      f"batch), ALDP/Accelerated, code map + histograms, {threads} threads"
                      + (", median of 3 (reference median_seconds)" if kind == "reference" else ""),
            "variants_mpx_s": res, "host": host_info()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--images", type=int, default=0, help="override batch size (testing)")
    ap.add_argument("--k", type=int, default=-1, help="override the config's k (C3 sweeps 1, 3, 5)")
    ap.add_argument("--e2e-images", type=int, default=2048)
    ap.add_argument("--cpu-images", type=int, default=0, help="0 = auto (~10-30 s of CPU work)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kernel", default="auto", choices=["auto", "fast", "generic"])
    ap.add_argument("--gather-chunks", type=int, default=2,
                    help="N>1: split each rank's shard so chunk i's histogram gather overlaps chunk i+1's kernel")
    ap.add_argument("--force-dist", action="store_true",
                    help="initialise NCCL and run the histogram gather even at world size 1 (tests the path)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    if args.impl == "reference":
        return run_reference(args, args.config)

    # The JSON line is the only thing on stdout: libraries that print from C
    # (NCCL's version banner at communicator init) go to stderr instead.
    out_fd = os.dup(1)
    os.dup2(2, 1)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1810_11518_b200 as aldp
    from paper_1810_11518_b200.shard import gather_histograms, shard_range, wire_dtype_ok

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        if "RANK" not in os.environ:  # --force-dist outside torchrun: a one-rank group
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(sk.getsockname()[1]))
            sk.close()
        dist.init_process_group("nccl", device_id=dev)

    n, rows, cols, k, cr, cc, blobs, gen, seed = CONFIGS[args.config]
    if args.images:
        n = args.images
    if args.k >= 0:
        k = args.k
    lo, hi = shard_range(n, rank, world)
    mine = hi - lo
    pitch = cols  # 640/1024/16384: already 16-byte aligned
    stream = torch.cuda.Stream(dev)
    sp = stream.cuda_stream

    # ---- inputs, generated on device by global image index (not timed) ----
    with torch.cuda.stream(stream):
        if gen == "faces":
            px = aldp.gen_faces(mine, rows, cols, blobs=blobs, seed=seed, first_index=lo, pitch=pitch,
                                device=dev, stream=sp)
        elif gen == "ties":
            px = aldp.gen_ties(mine, rows, cols, seed=seed, first_index=lo, pitch=pitch, device=dev,
                               stream=sp)
        else:  # config 1: the reference's make_random (mt19937), the library's own copy
            px = torch.from_numpy(aldp.make_random(rows, cols, seed)[None].copy()).to(dev)
        cells = aldp.grid_cells(rows, cols, cr, cc)
        nb = 256 if k == 0 else aldp.n_bins(k)
        codes = torch.empty((mine, rows, pitch), dtype=torch.uint8, device=dev)
        # With a gather (N > 1) the kernel writes uint16 counts directly (a
        # cell holds at most 81*91 = 7371 < 65536 pixels): they are the wire.
        wire16 = use_dist and wire_dtype_ok((cr or rows) * (cc or cols))
        hist = torch.empty((mine, cells, nb), dtype=torch.int16 if wire16 else torch.int32, device=dev)
        gathered = None
        if use_dist:
            per = [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]
            assert len(set(per)) == 1, "image count must divide evenly across ranks"
            if rank == 0:
                gathered = [torch.empty_like(hist) for _ in range(world)]
    stream.synchronize()

    # Chunks: with a gather (N > 1), chunk i's histograms travel on the comm
    # stream while chunk i+1's kernel runs; a step ends when its last gather
    # has landed, and the next step's kernels wait for that (hist reuse).
    n_chunks = max(1, min(args.gather_chunks, mine)) if use_dist else 1
    bounds = [(mine * i // n_chunks, mine * (i + 1) // n_chunks) for i in range(n_chunks)]
    comm = torch.cuda.Stream(dev) if use_dist else None
    chunk_ev = [torch.cuda.Event() for _ in bounds]
    comm_done = torch.cuda.Event()

    launches = [0]  # kernels launched by the last step (the library's own count)

    def launch_chunks():
        launches[0] = 0
        for ci, (a, b) in enumerate(bounds):
            aldp.ldp_batch(px[a:b], rows, cols, k=k, cell=(cr, cc), codes=codes[a:b], hist=hist[a:b],
                           kernel=args.kernel, stream=sp)
            launches[0] += aldp.last_launch_count()
            if use_dist:
                chunk_ev[ci].record(stream)
                comm.wait_event(chunk_ev[ci])
                with torch.cuda.stream(comm):
                    gather_histograms(hist[a:b], dist, rank, world,
                                      out=[g[a:b] for g in gathered] if rank == 0 else None,
                                      max_count=(cr or rows) * (cc or cols))

    def finish_step():
        if use_dist:
            comm_done.record(comm)
            stream.wait_event(comm_done)

    def step():
        launch_chunks()
        finish_step()

    # ---- warmup ----
    for _ in range(args.warmup):
        step()
    stream.synchronize()

    # ---- timed region: K steps, events on the launching stream ----
    sampler = ClockSampler(local) if True else None
    sampler.start()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        ev[2 * i].record(stream)
        launch_chunks()
        ev[2 * i + 1].record(stream)  # kernels only (the comm stream runs beside them)
        finish_step()
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    if use_dist:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = t_start.elapsed_time(t_end)
    launch_list = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps))
    launch_ms = sum(launch_list) / args.steps
    launch_median_ms = launch_list[args.steps // 2]
    if use_dist:
        t = torch.tensor([total_ms, launch_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, launch_ms = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    pixels = n * rows * cols
    value = pixels / (ms_per_step * 1e-3) / 1e6

    # ---- output checksums (outside the timed region): identical at every N ----
    w = torch.arange(1, nb + 1, device=dev, dtype=torch.int64)
    sums = torch.zeros(2, device=dev, dtype=torch.int64)
    for a in range(0, mine, 2048):  # chunked: never materialise a widened copy of 20 GB
        sums[0] += ((hist[a:a + 2048].to(torch.int64) & 0xFFFF) * w).sum()  # int16 counts are < 65536
        sums[1] += codes[a:a + 2048, :, :cols].sum(dtype=torch.int64)
    if use_dist:
        dist.all_reduce(sums)
    checks = {"hist_weighted_sum": int(sums[0]), "code_sum": int(sums[1]),
              "note": "sum over all images of bin-index-weighted counts, and of code bytes"}

    kernels_per_step = launches[0]

    # ---- roofline of the dominant kernel (one launch = this rank's shard) ----
    hbm, peak_src = measured_peaks()
    ncu = ncu_record(args.config if k == CONFIGS[args.config][3] else f"{args.config}_k{k}")
    traffic_bpp = ncu["dram_bytes_per_px"] if ncu else None
    bpp_hist = hist_bytes_per_image(rows, cols, k, cr, cc) / (rows * cols)
    alg_bytes = mine * rows * cols * (2.0 + bpp_hist)
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9

    line = {
        "metric": ("LBP" if k == 0 else "LDP") + " Mpixel/s (code map + histograms)", "value": round(value, 1),
        "unit": "Mpixel/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (device generator, seeded, keyed by global image index)",
        "config": {"workload": workload_name(args.config, k), "images": n, "rows": rows, "cols": cols,
                   "k": k, "cell": [cr, cc], "parallelism": f"image shards x{world}",
                   "l2": "inputs larger than L2 (no flush)" if n * rows * cols > 4 * 126e6 else
                         "inputs smaller than L2: repeated steps hit L2",
                   "kernel": args.kernel, "gather_chunks": n_chunks,
                   "checksums": checks},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4),
                     "traffic": (round(traffic_bpp * mine * rows * cols / (launch_ms * 1e-3) / 1e9, 1)
                                 if traffic_bpp else None),
                     "traffic_unit": "GB/s (ncu dram bytes per pixel x pixels per launch / launch time)",
                     "peak_source": peak_src,
                     "bytes_per_pixel": round(2.0 + bpp_hist, 4),
                     "launch_ms": round(launch_ms, 4), "launch_median_ms": round(launch_median_ms, 4),
                     "launches_per_step": kernels_per_step,
                     # what ncu measured for this kernel: the roofline is HBM, but
                     # the kernel is limited by instruction issue / the ALU pipe
                     "limiter": limiter_of(ncu, args.config),
                     "ncu": ncu},
        "clocks": clocks,
        "gpu_launches": args.steps * kernels_per_step,
    }

    # ---- end to end through the host C-ABI (pinned host buffers) ----
    # Every rank runs its own host batch through its own PCIe link at the
    # same time; the value is all ranks' pixels over the slowest rank's time.
    if not args.no_e2e:
        import ctypes
        e2n = min(args.e2e_images, mine)
        hp = torch.empty((e2n, rows, cols), dtype=torch.uint8).pin_memory()
        hp.copy_(px[:e2n, :, :cols])
        hc = torch.empty_like(hp).pin_memory()
        hh = torch.empty((e2n, cells, nb), dtype=torch.int32).pin_memory()

        def e2e_call():
            if k == 0:
                st = aldp.lib.aldp_lbp_batch_host(hp.data_ptr(), e2n, rows, cols, cr, cc, hc.data_ptr(),
                                                  hh.data_ptr(), None)
            else:
                st = aldp.lib.aldp_ldp_batch_host(hp.data_ptr(), e2n, rows, cols, k, cr, cc, hc.data_ptr(),
                                                  hh.data_ptr(), None)
            aldp._check(st)

        for _ in range(args.warmup):
            e2e_call()
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_call()
        e2e_dt = (time.perf_counter() - t0) / args.steps
        if use_dist:
            t = torch.tensor([e2e_dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_dt = float(t[0])
        line["e2e"] = {"value": round(world * e2n * rows * cols / e2e_dt / 1e6, 1), "unit": "Mpixel/s",
                       "h2d_bytes_per_step": int(hp.numel()),
                       "d2h_bytes_per_step": int(hc.numel() + hh.numel() * 4),
                       "images_per_step": e2n * world, "ranks": world,
                       "timing": "host wall clock per rank, max over ranks",
                       "api": "aldp_ldp_batch_host (C-ABI, host buffers)"}
        # the same call from pageable buffers (numpy arrays / std::vector, what
        # a caller of the reference API passes): staged through pinned memory
        hp_np, hc_np, hh_np = hp.numpy().copy(), np.empty_like(hc.numpy()), np.empty_like(hh.numpy())

        def e2e_pageable():
            fn = aldp.lib.aldp_lbp_batch_host if k == 0 else aldp.lib.aldp_ldp_batch_host
            kk = () if k == 0 else (k,)
            aldp._check(fn(hp_np.ctypes.data, e2n, rows, cols, *kk, cr, cc, hc_np.ctypes.data, hh_np.ctypes.data,
                           None))

        e2e_pageable()
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_pageable()
        pg_dt = (time.perf_counter() - t0) / args.steps
        if use_dist:
            t = torch.tensor([pg_dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pg_dt = float(t[0])
        line["e2e"]["pageable_value"] = round(world * e2n * rows * cols / pg_dt / 1e6, 1)
        line["e2e"]["pageable_note"] = "same call from pageable (non-pinned) host buffers"
        ok = np.array_equal(hc.numpy(), codes[:e2n, :, :cols].cpu().numpy()) and \
            np.array_equal(hh.numpy(), (hist[:e2n].to(torch.int64) & 0xFFFF).cpu().numpy()) and \
            np.array_equal(hc_np, hc.numpy()) and np.array_equal(hh_np, hh.numpy())
        if use_dist:
            t = torch.tensor([0 if ok else 1], device=dev, dtype=torch.int32)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ok = int(t[0]) == 0
        line["e2e"]["matches_device_path"] = bool(ok)

    # ---- CPU baseline (reference library on this box's host cores) ----
    if not args.no_cpu and rank == 0 and world == 1:
        threads = os.cpu_count() or 1
        if rows * cols >= 1e8:
            # C4: a 2048-row band of the frame, split into bands of whole cells
            # (one per host thread) so every core works on it
            band = px[0, :2048, :cols].cpu().numpy()
            host = band.reshape(2048 // cr, cr, cols) if cr else band[None]
        else:
            cpu_n = args.cpu_images or (min(mine, 4 * threads * 8) if rows * cols < 1e6 else min(mine, threads))
            host = px[:cpu_n, :, :cols].cpu().numpy()
        line["cpu_baseline"] = cpu_baseline(host, k, cr, cc)
    if rank == 0:
        sys.stdout.flush()
        os.write(out_fd, (json.dumps(line) + "\n").encode())
    if use_dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
