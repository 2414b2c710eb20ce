"""Parity oracles for the LDP path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package; the product package (paper_1810_11518_b200) never does.

Two checkers, both CPU:
  * ``port``      -- liboracle.so, this repo's plain-C restatement of the
                     reference algorithm (ldp_oracle.c, each function cites
                     the reference file:line it follows);
  * ``reference`` -- _ref/libaldp_ref.so, the UNMODIFIED reference library
                     compiled from /root/reference/proj/src (Makefile here)
                     behind an extern "C" shim (ref_shim.cpp). Built in the
                     dev container; the prebuilt .so travels to the GPU box.
The port is pinned against the reference's golden fixtures and against the
reference library itself (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libaldp_ref.so")

_P, _I, _I64, _U32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32


def _load_port():
    L = ctypes.CDLL(PORT_PATH)
    L.oracle_make_random.argtypes = [_I, _I, _U32, _P]
    L.oracle_responses.argtypes = [_P, _I, _I, _I, _I, _P]
    L.oracle_ldp_code.argtypes = [_P, _I]
    L.oracle_bin_index.argtypes = [_I, _I]
    L.oracle_n_bins.argtypes = [_I]
    L.oracle_code_map.argtypes = [_P, _I, _I, _I, _P]
    L.oracle_histogram.argtypes = [_P, _I, _I, _I, _P]
    L.oracle_cell_histograms.argtypes = [_P, _I, _I, _I, _I, _I, _P]
    L.oracle_batch.argtypes = [_P, _I64, _I, _I, _I, _I, _I, _P, _P, _I]
    L.oracle_column_terms.argtypes = [_P, _I, _I, _I, _I, _P]
    L.oracle_responses_terms.argtypes = [_P, _P]
    L.oracle_response_field.argtypes = [_P, _I, _I, _P]
    L.oracle_verify_image.argtypes = [_P, _I, _I, _P, _I, _P]
    L.oracle_verify_equivalence.argtypes = [_I, _U32, _P, _I, _P]
    return L


def _load_ref():
    L = ctypes.CDLL(REF_PATH)
    L.ref_make_random.argtypes = [_I, _I, _U32, _P]
    L.ref_responses.argtypes = [_P, _I, _I, _I, _I, _I, _P]
    L.ref_ldp_code.argtypes = [_P, _I, _P]
    L.ref_ldp_bin_index.argtypes = [_I]
    L.ref_code_map.argtypes = [_P, _I, _I, _I, _I, _P]
    L.ref_ldp_histogram.argtypes = [_P, _I, _I, _I, _I, _P]
    L.ref_windowed.argtypes = [_P, _I, _I, _I, _I, _P, _P]
    L.ref_batch.argtypes = [_P, _I64, _I, _I, _I, _I, _I, _I, _P, _P, _I]
    L.ref_median_seconds_batch.argtypes = [_P, _I64, _I, _I, _I, _I, _I, _I, _P, _P, _I, _I]
    L.ref_median_seconds_batch.restype = ctypes.c_double
    L.ref_response_field.argtypes = [_P, _I, _I, _I, _P]
    L.ref_verify_equivalence.argtypes = [_I, _U32, _P, _I, _P, _P]
    L.ref_verify_image.argtypes = [_P, _I, _I, _P, _I, _P, _P]
    L.ref_load_pgm.argtypes = [ctypes.c_char_p, _P, ctypes.c_size_t, _P, _P, _P, _I]
    L.ref_save_pgm.argtypes = [ctypes.c_char_p, _P, _I, _I, _I]
    L.ref_op_counts.argtypes = [_I, _P, _P]
    L.ref_bench_csv.argtypes = [ctypes.c_char_p, _I, _P, _I, _P, _I, _I, _U32, _I, _P, ctypes.c_size_t]
    return L


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        _port = _load_port()
    return _port


def ref():
    global _ref
    if _ref is None:
        _ref = _load_ref()
    return _ref


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


def _img(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


# ---- port (C restatement) ----
def make_random(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty((rows, cols), np.uint8)
    port().oracle_make_random(rows, cols, seed, out.ctypes.data)
    return out


def responses(img, x: int, y: int) -> np.ndarray:
    a = _img(img)
    out = np.empty(8, np.int32)
    port().oracle_responses(a.ctypes.data, a.shape[0], a.shape[1], x, y, out.ctypes.data)
    return out


def ldp_code(m, k: int = 3) -> int:
    v = np.ascontiguousarray(m, dtype=np.int32)
    return port().oracle_ldp_code(v.ctypes.data, k)


def bin_index(code: int, k: int = 3) -> int:
    return port().oracle_bin_index(code, k)


def n_bins(k: int) -> int:
    return port().oracle_n_bins(k)


def code_map(img, k: int = 3) -> np.ndarray:
    a = _img(img)
    out = np.empty_like(a)
    if port().oracle_code_map(a.ctypes.data, a.shape[0], a.shape[1], k, out.ctypes.data):
        raise ValueError("bad arguments")
    return out


def histogram(img, k: int = 3) -> np.ndarray:
    a = _img(img)
    out = np.zeros(n_bins(k), np.uint64)
    if port().oracle_histogram(a.ctypes.data, a.shape[0], a.shape[1], k, out.ctypes.data):
        raise ValueError("bad arguments")
    return out


def cell_histograms(img, cell_rows: int, cell_cols: int, k: int = 3) -> np.ndarray:
    a = _img(img)
    gr, gc = a.shape[0] // max(cell_rows, 1), a.shape[1] // max(cell_cols, 1)
    out = np.zeros((max(gr * gc, 1), n_bins(k)), np.uint64)
    if port().oracle_cell_histograms(a.ctypes.data, a.shape[0], a.shape[1], cell_rows, cell_cols, k,
                                     out.ctypes.data) < 0:
        raise ValueError("bad arguments")
    return out


def batch(pixels, k: int = 3, cell=(0, 0), codes: bool = True, hist: bool = True,
          threads: int = 0):
    """Batch [n, rows, cols] -> (codes | None, hist uint64 [n, cells, bins] | None)."""
    px = np.ascontiguousarray(pixels, dtype=np.uint8)
    if px.ndim == 2:
        px = px[None]
    n, rows, cols = px.shape
    cells = 1 if cell[0] == 0 else (rows // cell[0]) * (cols // cell[1])
    c = np.empty_like(px) if codes else None
    h = np.zeros((n, cells, n_bins(k)), np.uint64) if hist else None
    threads = threads or os.cpu_count() or 1
    if port().oracle_batch(px.ctypes.data, n, rows, cols, k, cell[0], cell[1],
                           c.ctypes.data if c is not None else None,
                           h.ctypes.data if h is not None else None, threads):
        raise ValueError("bad arguments")
    return c, h


# ---- reference library ----
def ref_batch(pixels, k: int = 3, cell=(0, 0), codes: bool = True, hist: bool = True,
              threads: int = 0, path: int = 1):
    px = np.ascontiguousarray(pixels, dtype=np.uint8)
    if px.ndim == 2:
        px = px[None]
    n, rows, cols = px.shape
    nb = n_bins(k)
    cells = 1 if cell[0] == 0 else (rows // cell[0]) * (cols // cell[1])
    c = np.empty_like(px) if codes else None
    h = np.zeros((n, cells, nb), np.uint64) if hist else None
    threads = threads or os.cpu_count() or 1
    st = ref().ref_batch(px.ctypes.data, n, rows, cols, k, cell[0], cell[1], path,
                         c.ctypes.data if c is not None else None,
                         h.ctypes.data if h is not None else None, threads)
    if st:
        raise {1: ValueError, 2: IndexError}.get(st, RuntimeError)("reference rejected the call")
    return c, h


def ref_ldp_histogram(img, k: int = 3, path: int = 1) -> np.ndarray:
    a = _img(img)
    out = np.zeros(56, np.uint64)
    st = ref().ref_ldp_histogram(a.ctypes.data, a.shape[0], a.shape[1], k, path, out.ctypes.data)
    if st:
        raise {1: ValueError, 2: IndexError}.get(st, RuntimeError)("reference rejected the call")
    return out


def ref_windowed(img, window: int, path: int = 1) -> np.ndarray:
    a = _img(img)
    gr, gc = a.shape[0] // window, a.shape[1] // window
    out = np.zeros((max(gr * gc, 1), 56), np.uint64)
    n = ctypes.c_int64(0)
    st = ref().ref_windowed(a.ctypes.data, a.shape[0], a.shape[1], window, path, out.ctypes.data,
                            ctypes.byref(n))
    if st:
        raise {1: ValueError, 2: IndexError}.get(st, RuntimeError)("reference rejected the call")
    return out[: n.value]


def ref_make_random(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty((rows, cols), np.uint8)
    if ref().ref_make_random(rows, cols, seed, out.ctypes.data):
        raise ValueError("bad dimensions")
    return out


def ref_responses(img, x: int, y: int, path: int = 0) -> np.ndarray:
    a = _img(img)
    out = np.empty(8, np.int32)
    st = ref().ref_responses(a.ctypes.data, a.shape[0], a.shape[1], x, y, path, out.ctypes.data)
    if st:
        raise {1: ValueError, 2: IndexError}.get(st, RuntimeError)("reference rejected the call")
    return out


# ---- response field / equivalence sweep ----
class _VR(ctypes.Structure):
    _fields_ = [("images_checked", ctypes.c_uint64), ("pixels_checked", ctypes.c_uint64),
                ("has_mismatch", ctypes.c_int), ("image_index", ctypes.c_int), ("x", ctypes.c_int),
                ("y", ctypes.c_int), ("direction", ctypes.c_int), ("naive_value", ctypes.c_int),
                ("accelerated_value", ctypes.c_int)]


def _fault5(fault):
    """fault: None or (image_index, x, y, term_index, delta)."""
    if fault is None:
        return None, None
    arr = np.asarray(fault, np.int32)
    assert arr.shape == (5,)
    return arr, arr.ctypes.data


def _verify_tuple(counts, mm):
    """(images_checked, pixels_checked, None | (image, x, y, dir, naive, accel))"""
    m = tuple(int(v) for v in mm[1:7]) if mm[0] else None
    return int(counts[0]), int(counts[1]), m


def column_terms(img, x: int, y: int) -> np.ndarray:
    a = _img(img)
    out = np.empty(15, np.int32)
    port().oracle_column_terms(a.ctypes.data, a.shape[0], a.shape[1], x, y, out.ctypes.data)
    return out


def responses_terms(a15) -> np.ndarray:
    a = np.ascontiguousarray(a15, np.int32)
    out = np.empty(8, np.int32)
    port().oracle_responses_terms(a.ctypes.data, out.ctypes.data)
    return out


def response_field(img) -> np.ndarray:
    a = _img(img)
    out = np.empty((a.shape[0] * a.shape[1], 8), np.int32)
    port().oracle_response_field(a.ctypes.data, a.shape[0], a.shape[1], out.ctypes.data)
    return out


def verify_image(img, fault=None, image_index: int = 0):
    a = _img(img)
    keep, fp = _fault5(fault)
    r = _VR()
    if port().oracle_verify_image(a.ctypes.data, a.shape[0], a.shape[1], fp, image_index, ctypes.byref(r)):
        raise IndexError("fault term_index out of range")
    return _verify_tuple((r.images_checked, r.pixels_checked),
                         (r.has_mismatch, r.image_index, r.x, r.y, r.direction, r.naive_value,
                          r.accelerated_value))


def verify_equivalence(images: int, seed: int, fault=None, threads: int = 1):
    keep, fp = _fault5(fault)
    r = _VR()
    if port().oracle_verify_equivalence(images, seed, fp, threads, ctypes.byref(r)):
        raise IndexError("fault term_index out of range")
    return _verify_tuple((r.images_checked, r.pixels_checked),
                         (r.has_mismatch, r.image_index, r.x, r.y, r.direction, r.naive_value,
                          r.accelerated_value))


def ref_response_field(img, path: int = 1) -> np.ndarray:
    a = _img(img)
    out = np.empty((a.shape[0] * a.shape[1], 8), np.int32)
    if ref().ref_response_field(a.ctypes.data, a.shape[0], a.shape[1], path, out.ctypes.data):
        raise ValueError("reference rejected the call")
    return out


def ref_verify_equivalence(images: int, seed: int, fault=None, threads: int = 1):
    keep, fp = _fault5(fault)
    counts = np.zeros(2, np.uint64)
    mm = np.zeros(7, np.int32)
    if ref().ref_verify_equivalence(images, seed, fp, threads, counts.ctypes.data, mm.ctypes.data):
        raise RuntimeError("reference verify failed")
    return _verify_tuple(counts, mm)


def ref_verify_image(img, fault=None, image_index: int = 0):
    a = _img(img)
    keep, fp = _fault5(fault)
    counts = np.zeros(2, np.uint64)
    mm = np.zeros(7, np.int32)
    if ref().ref_verify_image(a.ctypes.data, a.shape[0], a.shape[1], fp, image_index, counts.ctypes.data,
                              mm.ctypes.data):
        raise RuntimeError("reference verify failed")
    return _verify_tuple(counts, mm)


# ---- PGM I/O and op counts: the reference itself ----
def ref_load_pgm(path):
    """(pixels [rows, cols] uint8, None) or (None, runtime_error message)."""
    rows, cols = ctypes.c_int(), ctypes.c_int()
    err = ctypes.create_string_buffer(1024)
    p = os.fsencode(path)
    st = ref().ref_load_pgm(p, None, 0, ctypes.byref(rows), ctypes.byref(cols), err, 1024)
    if st == 4:
        return None, err.value.decode(errors="replace")
    if st:
        raise RuntimeError(f"reference load_pgm status {st}")
    out = np.empty((rows.value, cols.value), np.uint8)
    st = ref().ref_load_pgm(p, out.ctypes.data, out.size, ctypes.byref(rows), ctypes.byref(cols), err, 1024)
    assert st == 0
    return out, None


def ref_save_pgm(path, img, ascii: bool = False):
    a = _img(img)
    if ref().ref_save_pgm(os.fsencode(path), a.ctypes.data, a.shape[0], a.shape[1], int(ascii)):
        raise RuntimeError("reference save_pgm failed")


def ref_op_counts(descriptor: int):
    """descriptor 0 LDP, 1 ALDP, 2 LBP -> (mults, adds) per pixel."""
    m, a = ctypes.c_int(), ctypes.c_int()
    if ref().ref_op_counts(descriptor, ctypes.byref(m), ctypes.byref(a)):
        raise RuntimeError("reference measured_ops failed")
    return m.value, a.value


def ref_bench_csv(series="images", size=0, counts=(1, 2, 4, 6, 8, 10), windows=(25, 50, 100), repeats=5,
                  seed=42, descriptor=-1) -> str:
    """The reference CLI's bench report (CPU), descriptor -1 = all three."""
    c = (ctypes.c_int * max(len(counts), 1))(*counts)
    w = (ctypes.c_int * max(len(windows), 1))(*windows)
    buf = ctypes.create_string_buffer(1 << 16)
    if ref().ref_bench_csv(series.encode(), size, c, len(counts), w, len(windows), repeats, seed, descriptor,
                           buf, len(buf)):
        raise RuntimeError("reference bench failed")
    return buf.value.decode()


def ref_median_seconds_batch(pixels, k: int = 3, cell=(0, 0), path: int = 1, threads: int = 1,
                             repeats: int = 3, codes: bool = True) -> float:
    """The reference's own timer (bench.cpp:51-78: warm-up pass, batches up to
    >= 5 ms, median of `repeats`) around ref_batch (codes + histograms, or the
    histograms alone with codes=False: the reference API's one pass)."""
    px = np.ascontiguousarray(pixels, dtype=np.uint8)
    if px.ndim == 2:
        px = px[None]
    n, r, c = px.shape
    nb = ref_n_bins(k)
    cells = 1 if cell[0] == 0 else (r // cell[0]) * (c // cell[1])
    cbuf = np.empty_like(px) if codes else None
    hist = np.empty((n, cells, nb), np.uint64)
    return float(ref().ref_median_seconds_batch(px.ctypes.data, n, r, c, k, cell[0], cell[1], path,
                                                 cbuf.ctypes.data if cbuf is not None else None,
                                                 hist.ctypes.data, threads, repeats))


def ref_n_bins(k: int) -> int:
    return 256 if k == 0 else sum(1 for v in range(256) if bin(v).count("1") == k)
