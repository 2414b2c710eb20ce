#!/usr/bin/env python3
"""Small invocations of every device kernel family, each checked against the
CPU oracle, for compute-sanitizer runs (one tool per run):

  compute-sanitizer --tool memcheck|racecheck|synccheck --error-exitcode 9 \\
      --kernel-name regex:aldp_b200 python tools/sanitize_cases.py

Cases: the packed kernel with 81x91 cells (k = 3), k = 4 cells, LBP cells,
whole-image codes + histograms (tag set 1), codes only, band views with halo
rows, the small-batch split launch, the generic kernel, the response-field
row kernel (cp.async.bulk + mbarrier) and the equivalence sweep. Exits 1 on
any mismatch."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_1810_11518_b200 as aldp  # noqa: E402

DEV = torch.device("cuda:0")
failures = []


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        failures.append(name)


def batch_case(name, px, rows, cols, k, cell, kernel="auto", codes=True):
    want_codes = True if codes else None
    c, h = (aldp.lbp_batch(px, rows, cols, cell=cell, codes=want_codes, hist=True, kernel=kernel) if k == 0 else
            aldp.ldp_batch(px, rows, cols, k=k, cell=cell, codes=want_codes, hist=True, kernel=kernel))
    torch.cuda.synchronize()
    host = px[:, :, :cols].cpu().numpy()
    rc, rh = oracle.batch(host, k=k, cell=cell)
    ok = np.array_equal(h.cpu().numpy().astype(np.uint64), rh)
    if codes:
        ok = ok and np.array_equal(c[:, :, :cols].cpu().numpy(), rc)
    check(name, ok)


def main():
    faces = aldp.gen_faces(6, 490, 640, blobs=20, seed=3, device=DEV)
    ties = aldp.gen_ties(2, 300, 256, seed=4, device=DEV)
    batch_case("k3 cells 81x91", faces, 490, 640, 3, (81, 91))
    batch_case("k4 cells 81x91", faces, 490, 640, 4, (81, 91))
    batch_case("lbp cells 81x91", faces, 490, 640, 0, (81, 91))
    batch_case("k3 cells 64x64 hist only", faces, 490, 640, 3, (64, 64), codes=False)
    batch_case("k3 whole image", faces, 490, 640, 3, (0, 0))
    batch_case("k5 whole image ties", ties, 300, 256, 5, (0, 0))
    batch_case("k3 generic kernel", faces[:2], 490, 640, 3, (81, 91), kernel="generic")
    # codes only (whole-image kernel, no histogram)
    c, _ = aldp.ldp_batch(faces, 490, 640, k=3, codes=True)
    torch.cuda.synchronize()
    rc, _ = oracle.batch(faces[:, :, :640].cpu().numpy(), k=3)
    check("k3 codes only", np.array_equal(c[:, :, :640].cpu().numpy(), rc))
    # band views of one frame with real halo rows (host streaming of tall frames)
    frame = faces[0:1]
    want_c, _ = oracle.batch(frame[:, :, :640].cpu().numpy(), k=3)
    _, want_cells = oracle.batch(frame[:, :, :640].cpu().numpy(), k=3, cell=(81, 91), codes=False)
    got = np.zeros((490, 640), np.uint8)
    cells = []
    for r0, r1 in ((0, 162), (162, 324), (324, 490)):
        view = frame[:, r0:r1, :]
        cb, _ = aldp.ldp_batch(view, r1 - r0, 640, k=3, codes=True, halo=(r0 > 0, r1 < 490))
        _, hc = aldp.ldp_batch(view, r1 - r0, 640, k=3, cell=(81, 91), hist=True, halo=(r0 > 0, r1 < 490))
        torch.cuda.synchronize()
        got[r0:r1] = cb[0, :, :640].cpu().numpy()
        cells.append(hc[0].cpu().numpy().astype(np.uint64))
    check("band views", np.array_equal(got, want_c[0]) and np.array_equal(np.concatenate(cells), want_cells[0]))
    # response field (TMA row kernel) and the naive-vs-identity sweep
    f = aldp.response_field_batch(faces[:2], 490, 640)
    torch.cuda.synchronize()
    check("response field", np.array_equal(f[0].cpu().numpy().astype(np.int32).reshape(-1, 8),
                                            oracle.response_field(faces[0, :, :640].cpu().numpy())))
    check("verify sweep", aldp.verify_batch(faces[:2], 490, 640).ok())
    if failures:
        print("FAILED:", failures)
        return 1
    print("all cases ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
