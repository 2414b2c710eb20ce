"""B200-native LDP feature extraction (arxiv 1810.11518, ALDP) -- Python host layer.

This package is the Python mirror of the reference's public LDP interface
(reference tree ``proj/include/aldp``), sitting on the C-ABI of
``libaldp_b200.so`` (declared in ``include/aldp_cuda.h``):

================================  ===========================================
this module                       reference
================================  ===========================================
``ldp_histogram(img, k, path)``   ``aldp::ldp_histogram`` (descriptors.hpp:55)
``windowed_features(img, w, d)``  ``aldp::windowed_features`` (windowing.hpp:34)
``ldp_code_map(img, k, path)``    new: the per-pixel code of descriptors.cpp:129-136
``make_grid(img, window)``        ``aldp::make_grid`` (windowing.hpp:25)
``n_bins(k)`` / ``ResponsePath``  bin layout (descriptors.cpp:25-45), kirsch.hpp:88
``ldp_batch(...)``                device-resident batch (the hot path)
================================  ===========================================

Errors follow the reference: ``std::invalid_argument`` -> ``ValueError``,
``std::out_of_range`` -> ``IndexError``, CUDA failures -> ``RuntimeError``.

There is no CPU fallback: importing this package loads the CUDA library and
raises if it is missing; every compute call runs the sm_100a kernels.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

__all__ = [
    "ResponsePath", "Descriptor", "AldpError", "lib", "LIB_PATH", "n_bins", "grid_cells",
    "WindowGrid", "make_grid", "ldp_histogram", "windowed_features", "ldp_code_map",
    "ldp_batch", "ldp_batch_host", "gen_faces", "gen_ties", "version",
    "lbp_histogram", "lbp_code_map", "lbp_batch", "response_field", "response_field_batch",
    "FaultInjection", "Mismatch", "VerifyResult", "verify_equivalence", "verify_image", "verify_batch",
    "PgmError", "load_pgm", "save_pgm", "load_pgm_batch", "extract_files", "op_counts", "bench_csv",
    "CLI_PATH", "last_launch_count", "debug_fault", "ldp_batch_host_multi", "make_random",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# ALDP_LIB points at an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("ALDP_LIB") or os.path.join(_HERE, "libaldp_b200.so")


class ResponsePath(enum.IntEnum):
    """aldp::ResponsePath (kirsch.hpp:88). Both run the same B200 kernel:
    their outputs are identical by contract (descriptors.hpp:53-54)."""
    Naive = 0
    Accelerated = 1


class Descriptor(enum.Enum):
    """aldp::Descriptor (descriptors.hpp:13). All three run on the B200 (Lbp: the
    LBP instantiation of the fast kernel; Ldp / Aldp: the LDP kernel)."""
    Lbp = "LBP"
    Ldp = "LDP"
    Aldp = "ALDP"


def parse_descriptor(name: str) -> Descriptor:
    """aldp::parse_descriptor (descriptors.cpp:53-81), case-insensitive."""
    for d in Descriptor:
        if name.lower() == d.value.lower():
            return d
    raise ValueError(f"unknown descriptor '{name}' (expected lbp, ldp or aldp)")


class AldpError(RuntimeError):
    pass


class PgmError(AldpError):
    """File I/O or PGM format error (the reference's std::runtime_error from
    load_pgm / save_pgm, pgm.hpp:15-17)."""


_STATUS_EXC = {1: ValueError, 2: IndexError, 3: AldpError, 4: MemoryError, 5: PgmError}


class _Args(ctypes.Structure):
    _fields_ = [
        ("d_pixels", ctypes.c_void_p), ("img_stride", ctypes.c_int64),
        ("rows", ctypes.c_int), ("cols", ctypes.c_int), ("pitch", ctypes.c_int),
        ("n_images", ctypes.c_int), ("k", ctypes.c_int),
        ("cell_rows", ctypes.c_int), ("cell_cols", ctypes.c_int),
        ("d_codes", ctypes.c_void_p), ("codes_img_stride", ctypes.c_int64),
        ("codes_pitch", ctypes.c_int), ("d_hist", ctypes.c_void_p),
        ("cell_from_map", ctypes.c_int), ("rows_above", ctypes.c_int), ("rows_below", ctypes.c_int),
        ("hist_u16", ctypes.c_int),
    ]


class _Fault(ctypes.Structure):
    _fields_ = [("image_index", ctypes.c_int), ("x", ctypes.c_int), ("y", ctypes.c_int),
                ("term_index", ctypes.c_int), ("delta", ctypes.c_int)]


class _VerifyResult(ctypes.Structure):
    _fields_ = [("images_checked", ctypes.c_uint64), ("pixels_checked", ctypes.c_uint64),
                ("mismatches", ctypes.c_uint64), ("has_mismatch", ctypes.c_int),
                ("image_index", ctypes.c_int), ("x", ctypes.c_int), ("y", ctypes.c_int),
                ("direction", ctypes.c_int), ("naive_value", ctypes.c_int),
                ("accelerated_value", ctypes.c_int)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64
    sig = {
        "aldp_ldp_batch": ([ctypes.POINTER(_Args), P], I),
        "aldp_ldp_batch_ex": ([ctypes.POINTER(_Args), I, P], I),
        "aldp_n_bins": ([I], I),
        "aldp_grid_cells": ([I, I, I, I], I64),
        "aldp_ldp_histogram": ([P, I, I, I, I, P], I),
        "aldp_windowed_features": ([P, I, I, I, I, P, ctypes.c_size_t], I),
        "aldp_ldp_code_map": ([P, I, I, I, I, P], I),
        "aldp_ldp_batch_host": ([P, I, I, I, I, I, I, P, P, P], I),
        "aldp_lbp_batch": ([ctypes.POINTER(_Args), P], I),
        "aldp_lbp_batch_ex": ([ctypes.POINTER(_Args), I, P], I),
        "aldp_lbp_histogram": ([P, I, I, P], I),
        "aldp_lbp_code_map": ([P, I, I, P], I),
        "aldp_lbp_batch_host": ([P, I, I, I, I, I, P, P, P], I),
        "aldp_ldp_batch_host_multi": ([P, I, I, I, I, I, I, P, P, P, I], I),
        "aldp_make_random": ([P, I, I, ctypes.c_uint32], I),
        "aldp_lbp_batch_host_multi": ([P, I, I, I, I, I, P, P, P, I], I),
        "aldp_ldp_batch_multi": ([ctypes.POINTER(_Args), P, P, I], I),
        "aldp_gather_peer": ([P, I, P, P, P, I, P], I),
        "aldp_last_error": ([], ctypes.c_char_p),
        "aldp_last_launch_count": ([], I),
        "aldp_debug_fault": ([I], I),
        "aldp_gen_faces": ([P, I, I, I, I, I64, I, U64, I64, P], I),
        "aldp_gen_ties": ([P, I, I, I, I, I64, U64, I64, P], I),
        "aldp_version": ([], ctypes.c_char_p),
        "aldp_response_field_batch": ([P, I64, I, I, I, I, I, P, P], I),
        "aldp_response_field_batch32": ([P, I64, I, I, I, I, I, P, P], I),
        "aldp_response_field": ([P, I, I, I, P], I),
        "aldp_verify_equivalence": ([I, ctypes.c_uint32, ctypes.POINTER(_Fault), I,
                                     ctypes.POINTER(_VerifyResult)], I),
        "aldp_verify_image": ([P, I, I, ctypes.POINTER(_Fault), I, ctypes.POINTER(_VerifyResult)], I),
        "aldp_verify_batch": ([P, I64, I, I, I, I, ctypes.POINTER(_Fault), I,
                               ctypes.POINTER(_VerifyResult), P], I),
        "aldp_load_pgm": ([ctypes.c_char_p, P, ctypes.c_size_t, P, P], I),
        "aldp_save_pgm": ([ctypes.c_char_p, P, I, I, I], I),
        "aldp_load_pgm_batch": ([P, I, I, I, P, I], I),
        "aldp_extract_files": ([P, I, ctypes.c_char_p, I, ctypes.c_char_p, I], I),
        "aldp_op_counts": ([I, P, P], I),
        "aldp_bench_csv": ([ctypes.c_char_p, I, P, I, P, I, I, ctypes.c_uint32, ctypes.c_char_p,
                            ctypes.c_char_p], I),
    }
    for name, (argtypes, restype) in sig.items():
        if os.environ.get("ALDP_LIB") and not hasattr(L, name):
            continue  # an older build under A/B (ALDP_LIB) may predate this entry point
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = restype
    return L


lib = _load()


def _check(status: int) -> None:
    if status != 0:
        msg = lib.aldp_last_error().decode(errors="replace")
        raise _STATUS_EXC.get(status, AldpError)(msg)


def device_code_fingerprint(lib_path: Optional[str] = None) -> Optional[str]:
    """sha256 over the sm_100a code of a library build: every section of
    every embedded cubin except the debug-string sections (which carry nvcc's
    temporary file names, so rebuilding identical code changes the .so's own
    sha256 but not this). None when cuobjdump is unavailable."""
    import hashlib
    import shutil
    import struct
    import subprocess
    import tempfile
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return None
    h = hashlib.sha256()
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run([tool, "-xelf", "all", os.path.abspath(lib_path or LIB_PATH)], cwd=d,
                           capture_output=True)
        if r.returncode != 0:
            return None
        for name in sorted(os.listdir(d)):
            b = open(os.path.join(d, name), "rb").read()
            if b[:4] != b"\x7fELF" or b[4] != 2:
                continue
            shoff = struct.unpack_from("<Q", b, 0x28)[0]
            shentsize, shnum, shstrndx = struct.unpack_from("<HHH", b, 0x3A)
            hdrs = [struct.unpack_from("<IIQQQQIIQQ", b, shoff + i * shentsize) for i in range(shnum)]
            strtab = hdrs[shstrndx][4]
            h.update(name.encode())
            for sh in hdrs:
                sec = b[strtab + sh[0]:b.index(b"\0", strtab + sh[0])]
                if b"debug" in sec:
                    continue
                h.update(sec)
                if sh[1] != 8:  # SHT_NOBITS has no bytes in the file
                    h.update(b[sh[4]:sh[4] + sh[5]])
    return h.hexdigest()


def version() -> str:
    return lib.aldp_version().decode()


def n_bins(k: int) -> int:
    """C(8, k) bins (56 for the reference's k == 3)."""
    n = lib.aldp_n_bins(int(k))
    if n == 0:
        raise ValueError("k must be in [1, 7]")
    return n


def grid_cells(rows: int, cols: int, cell_rows: int, cell_cols: int) -> int:
    n = lib.aldp_grid_cells(rows, cols, cell_rows, cell_cols)
    if n < 0:
        raise ValueError("invalid cell size for this image")
    return int(n)


@dataclass(frozen=True)
class WindowGrid:
    """aldp::WindowGrid (windowing.hpp:14-23)."""
    window: int
    grid_rows: int
    grid_cols: int

    def total(self) -> int:
        return self.grid_rows * self.grid_cols


def make_grid(img: np.ndarray, window: int) -> WindowGrid:
    """aldp::make_grid (windowing.cpp:8-19): floor grid of square windows."""
    rows, cols = img.shape
    if window < 3:
        raise ValueError(f"window side must be >= 3, got {window}")
    if window > rows or window > cols:
        raise ValueError(f"window side {window} exceeds image {rows}x{cols}")
    return WindowGrid(window, rows // window, cols // window)


def _as_image(img) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(img, dtype=np.uint8))
    if a.ndim != 2:
        raise ValueError("expected a 2-D uint8 image (rows x cols)")
    return a


def _path_value(path) -> int:
    if isinstance(path, str):
        path = ResponsePath.Naive if path.lower() in ("naive", "ldp") else ResponsePath.Accelerated
    return int(path)


def ldp_histogram(img, k: int = 3, path=ResponsePath.Accelerated) -> np.ndarray:
    """aldp::ldp_histogram: 56 uint64 bins over every pixel (clamped borders)."""
    a = _as_image(img)
    out = np.zeros(56, dtype=np.uint64)
    _check(lib.aldp_ldp_histogram(a.ctypes.data, a.shape[0], a.shape[1], int(k), _path_value(path),
                                  out.ctypes.data))
    return out


_DESC_LBP = 2  # ALDP_DESC_LBP


def windowed_features(img, window: int, descriptor=Descriptor.Aldp) -> np.ndarray:
    """aldp::windowed_features: [grid cells, bins] uint64 (56 bins for Ldp/Aldp,
    256 for Lbp), row-major windows, each window clamped as an independent image."""
    if isinstance(descriptor, str):
        descriptor = parse_descriptor(descriptor)
    a = _as_image(img)
    grid = make_grid(a, window)
    nb = 256 if descriptor is Descriptor.Lbp else 56
    out = np.zeros((grid.total(), nb), dtype=np.uint64)
    sel = (_DESC_LBP if descriptor is Descriptor.Lbp else
           int(ResponsePath.Naive if descriptor is Descriptor.Ldp else ResponsePath.Accelerated))
    _check(lib.aldp_windowed_features(a.ctypes.data, a.shape[0], a.shape[1], int(window), sel,
                                      out.ctypes.data, out.size))
    return out


def lbp_histogram(img) -> np.ndarray:
    """aldp::lbp_histogram (descriptors.cpp:159-168): 256 uint64 bins."""
    a = _as_image(img)
    out = np.zeros(256, dtype=np.uint64)
    _check(lib.aldp_lbp_histogram(a.ctypes.data, a.shape[0], a.shape[1], out.ctypes.data))
    return out


def lbp_code_map(img) -> np.ndarray:
    """LBP code map: codes[x, y] = lbp_code(img, x, y) (descriptors.cpp:141-157)."""
    a = _as_image(img)
    out = np.zeros_like(a)
    _check(lib.aldp_lbp_code_map(a.ctypes.data, a.shape[0], a.shape[1], out.ctypes.data))
    return out


def ldp_code_map(img, k: int = 3, path=ResponsePath.Accelerated) -> np.ndarray:
    """Code map (new entry point): codes[x, y] = ldp_code(responses(img, x, y), k)."""
    a = _as_image(img)
    out = np.zeros_like(a)
    _check(lib.aldp_ldp_code_map(a.ctypes.data, a.shape[0], a.shape[1], int(k), _path_value(path),
                                 out.ctypes.data))
    return out


def ldp_batch_host(pixels: np.ndarray, k: int = 3, cell: Tuple[int, int] = (0, 0),
                   codes: bool = True, hist: bool = True, stream: int = 0):
    """Host batch [n, rows, cols] uint8 -> (codes [n, rows, cols] | None,
    hist uint32 [n, cells, n_bins] | None). H2D, kernel and D2H in one call.
    k == 0 selects LBP (256 bins)."""
    px = np.ascontiguousarray(pixels, dtype=np.uint8)
    if px.ndim == 2:
        px = px[None]
    n, rows, cols = px.shape
    nb = 256 if k == 0 else n_bins(k)
    cells = grid_cells(rows, cols, *cell)
    c = np.empty_like(px) if codes else None
    h = np.empty((n, cells, nb), dtype=np.uint32) if hist else None
    cp = c.ctypes.data if c is not None else None
    hp = h.ctypes.data if h is not None else None
    if k == 0:
        _check(lib.aldp_lbp_batch_host(px.ctypes.data, n, rows, cols, int(cell[0]), int(cell[1]), cp, hp,
                                       stream or None))
    else:
        _check(lib.aldp_ldp_batch_host(px.ctypes.data, n, rows, cols, int(k), int(cell[0]), int(cell[1]),
                                       cp, hp, stream or None))
    return c, h


def ldp_batch_host_multi(pixels: np.ndarray, k: int = 3, cell: Tuple[int, int] = (0, 0),
                         codes: bool = True, hist: bool = True, devices=None):
    """ldp_batch_host over several GPUs of this process
    (aldp_ldp_batch_host_multi): contiguous image ranges, one per entry of
    `devices` (None: every visible device), each on its own persistent host
    worker. Same results as ldp_batch_host for any device list. k == 0: LBP."""
    px = np.ascontiguousarray(pixels, dtype=np.uint8)
    if px.ndim == 2:
        px = px[None]
    n, rows, cols = px.shape
    nb = 256 if k == 0 else n_bins(k)
    cells = grid_cells(rows, cols, *cell)
    c = np.empty_like(px) if codes else None
    h = np.empty((n, cells, nb), dtype=np.uint32) if hist else None
    cp = c.ctypes.data if c is not None else None
    hp = h.ctypes.data if h is not None else None
    if devices is None:
        dp, nd = None, 0
    else:
        dv = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        dp, nd = ctypes.cast(dv, ctypes.c_void_p), len(devices)
    if k == 0:
        _check(lib.aldp_lbp_batch_host_multi(px.ctypes.data, n, rows, cols, int(cell[0]), int(cell[1]), cp, hp,
                                             dp, nd))
    else:
        _check(lib.aldp_ldp_batch_host_multi(px.ctypes.data, n, rows, cols, int(k), int(cell[0]), int(cell[1]),
                                             cp, hp, dp, nd))
    return c, h


_KERNEL = {"auto": 0, "fast": 1, "generic": 2}


def lbp_batch(pixels, rows: int, cols: int, cell: Tuple[int, int] = (0, 0), codes=None, hist=None,
              kernel: str = "auto", stream: Optional[int] = None, cell_clamp: bool = True):
    """Device-resident LBP batch: like ldp_batch, hist [n, cells, 256]."""
    return ldp_batch(pixels, rows, cols, k=0, cell=cell, codes=codes, hist=hist, kernel=kernel,
                     stream=stream, cell_clamp=cell_clamp)


def ldp_batch(pixels, rows: int, cols: int, k: int = 3, cell: Tuple[int, int] = (0, 0),
              codes=None, hist=None, kernel: str = "auto", stream: Optional[int] = None,
              cell_clamp: bool = True, halo: Tuple[int, int] = (0, 0)):
    """Device-resident batch (the hot path).

    pixels: torch.uint8 CUDA tensor [n, rows, pitch] (contiguous; pitch >= cols).
    codes:  None, True (allocate) or a torch.uint8 tensor [n, rows, codes_pitch].
    hist:   None, True (allocate) or a torch.int32/uint32 tensor [n, cells, n_bins];
            a torch.int16/uint16 tensor gets uint16 counts (the compact
            multi-GPU wire; every histogram must stay below 65536 counts).
    stream: a raw cudaStream_t (int); default: torch's current stream.
    cell_clamp: True (the reference's windowed_features rule) clamps every
            cell as its own image; False cuts cells from the whole-image code
            map instead.
    halo:   (above, below) in {0, 1}: real image rows exist just above / below
            this view (pixels is a band of a taller resident frame), so the
            view's edge rows see them instead of a clamped copy.
    Returns (codes, hist). Asynchronous on the stream.
    """
    import torch
    if pixels.dtype != torch.uint8 or not pixels.is_cuda or pixels.dim() != 3:
        raise ValueError("pixels must be a CUDA uint8 tensor [n, rows, pitch]")
    if not pixels.is_contiguous():
        raise ValueError("pixels must be contiguous")
    n, r, pitch = pixels.shape
    if r != rows or pitch < cols:
        raise ValueError("pixels shape does not match rows/cols")
    nb = 256 if k == 0 else n_bins(k)  # k == 0: LBP (internal convention, lbp_batch)
    cells = grid_cells(rows, cols, *cell)
    if codes is True:
        codes = torch.empty((n, rows, pitch), dtype=torch.uint8, device=pixels.device)
    if hist is True:
        hist = torch.empty((n, cells, nb), dtype=torch.int32, device=pixels.device)
    a = _Args()
    a.d_pixels = pixels.data_ptr()
    a.img_stride = rows * pitch
    a.rows, a.cols, a.pitch, a.n_images, a.k = rows, cols, pitch, n, int(k)
    a.cell_rows, a.cell_cols = int(cell[0]), int(cell[1])
    a.cell_from_map = 0 if cell_clamp else 1
    a.rows_above, a.rows_below = int(bool(halo[0])), int(bool(halo[1]))
    if codes is not None:
        if codes.dtype != torch.uint8 or codes.dim() != 3 or not codes.is_contiguous():
            raise ValueError("codes must be a contiguous uint8 tensor [n, rows, pitch]")
        if codes.device != pixels.device:
            raise ValueError(f"codes is on {codes.device}, pixels on {pixels.device}")
        if codes.shape[0] < n or codes.shape[1] < rows or codes.shape[2] < cols:
            raise ValueError(f"codes tensor {tuple(codes.shape)} does not cover ({n}, {rows}, {cols})")
        a.d_codes = codes.data_ptr()
        a.codes_pitch = codes.shape[2]
        a.codes_img_stride = codes.shape[1] * codes.shape[2]
    if hist is not None:
        if hist.dtype not in (torch.int32, torch.uint32, torch.int16, torch.uint16):
            raise ValueError(f"hist must be int32/uint32 (or int16/uint16), got {hist.dtype}")
        a.hist_u16 = int(hist.dtype in (torch.int16, torch.uint16))
        if hist.device != pixels.device:
            raise ValueError(f"hist is on {hist.device}, pixels on {pixels.device}")
        if hist.numel() < n * cells * nb or not hist.is_contiguous():
            raise ValueError("hist tensor too small or not contiguous")
        a.d_hist = hist.data_ptr()
    if stream is None:
        stream = torch.cuda.current_stream(pixels.device).cuda_stream
    fn = lib.aldp_lbp_batch_ex if k == 0 else lib.aldp_ldp_batch_ex
    _check(fn(ctypes.byref(a), _KERNEL[kernel], stream or None))
    return codes, hist


def make_random(rows: int, cols: int, seed: int) -> np.ndarray:
    """aldp::make_random (image.hpp:44; reference image.cpp:75-83): the
    std::mt19937 low-byte image of config 1, on the host."""
    out = np.empty((rows, cols), np.uint8)
    _check(lib.aldp_make_random(out.ctypes.data, int(rows), int(cols), int(seed) & 0xFFFFFFFF))
    return out


def last_launch_count() -> int:
    """Kernels the last ldp_batch / lbp_batch call on this thread launched
    (-1: a library build without the counter, A/B runs only)."""
    if not hasattr(lib, "aldp_last_launch_count"):
        return -1
    return int(lib.aldp_last_launch_count())


def debug_fault(mode: int) -> int:
    """Negative control (aldp_debug_fault): while mode is 1 every batch flips
    image 0's first code bit and adds a count to its first bin. Returns the
    previous mode."""
    return int(lib.aldp_debug_fault(int(mode)))


def _pitch(cols: int, pitch: Optional[int]) -> int:
    return pitch if pitch else (cols + 15) // 16 * 16


def gen_faces(n: int, rows: int, cols: int, blobs: int = 20, seed: int = 1810,
              first_index: int = 0, pitch: Optional[int] = None, device="cuda", out=None,
              stream: Optional[int] = None):
    """Face-like synthetic images on the device (BASELINE.json configs 2/4/5):
    torch.uint8 [n, rows, pitch], keyed by (seed, first_index + i)."""
    import torch
    pitch = _pitch(cols, pitch)
    if out is None:
        out = torch.zeros((n, rows, pitch), dtype=torch.uint8, device=device)
    if stream is None:
        stream = torch.cuda.current_stream(out.device).cuda_stream
    _check(lib.aldp_gen_faces(out.data_ptr(), n, rows, cols, pitch, rows * pitch, blobs, seed,
                              first_index, stream or None))
    return out


def gen_ties(n: int, rows: int, cols: int, seed: int = 11518, first_index: int = 0,
             pitch: Optional[int] = None, device="cuda", out=None, stream: Optional[int] = None):
    """Tie-heavy synthetic images on the device (config 3): values {0,1,2}
    with ~50% of the area under constant rectangles."""
    import torch
    pitch = _pitch(cols, pitch)
    if out is None:
        out = torch.zeros((n, rows, pitch), dtype=torch.uint8, device=device)
    if stream is None:
        stream = torch.cuda.current_stream(out.device).cuda_stream
    _check(lib.aldp_gen_ties(out.data_ptr(), n, rows, cols, pitch, rows * pitch, seed, first_index,
                             stream or None))
    return out


# ------------------------------------------------------------ response field

def response_field(img, path=ResponsePath.Accelerated) -> np.ndarray:
    """aldp::response_field (kirsch.hpp:91-92, kirsch.cpp:193-208): int32
    [rows*cols, 8], the eight signed Kirsch responses per pixel in raster
    order, computed on the B200."""
    img = _as_image(img)
    out = np.empty((img.shape[0] * img.shape[1], 8), np.int32)
    _check(lib.aldp_response_field(img.ctypes.data, img.shape[0], img.shape[1], _path_value(path),
                                   out.ctypes.data))
    return out


def response_field_batch(pixels, rows: int, cols: int, path=ResponsePath.Accelerated, out=None,
                         wide: bool = False, stream: Optional[int] = None):
    """Device batch: pixels torch.uint8 [n, rows, pitch] -> int16 (or int32
    when wide) [n, rows, cols, 8]. Asynchronous on the stream."""
    import torch
    if pixels.dtype != torch.uint8 or not pixels.is_cuda or pixels.dim() != 3 or not pixels.is_contiguous():
        raise ValueError("pixels must be a contiguous CUDA uint8 tensor [n, rows, pitch]")
    n, r, pitch = pixels.shape
    if r != rows or pitch < cols:
        raise ValueError("pixels shape does not match rows/cols")
    dt = torch.int32 if wide else torch.int16
    if out is None:
        out = torch.empty((n, rows, cols, 8), dtype=dt, device=pixels.device)
    if out.dtype != dt or not out.is_contiguous() or out.numel() < n * rows * cols * 8:
        raise ValueError("out must be a contiguous %s tensor [n, rows, cols, 8]" % dt)
    if stream is None:
        stream = torch.cuda.current_stream(pixels.device).cuda_stream
    fn = lib.aldp_response_field_batch32 if wide else lib.aldp_response_field_batch
    _check(fn(pixels.data_ptr(), rows * pitch, rows, cols, pitch, n, _path_value(path), out.data_ptr(),
              stream or None))
    return out


# ------------------------------------------------------------ verification

@dataclass
class FaultInjection:
    """aldp::FaultInjection (verify.hpp:14-20)."""
    image_index: int = 0
    x: int = 0
    y: int = 0
    term_index: int = 0
    delta: int = 1


@dataclass
class Mismatch:
    """aldp::Mismatch (verify.hpp:22-29)."""
    image_index: int = 0
    x: int = 0
    y: int = 0
    direction: int = 0
    naive_value: int = 0
    accelerated_value: int = 0


@dataclass
class VerifyResult:
    """aldp::VerifyResult (verify.hpp:31-37); `mismatches` is new: every
    mismatching (pixel, direction) the device sweep saw."""
    images_checked: int = 0
    pixels_checked: int = 0
    mismatch: Optional[Mismatch] = None
    mismatches: int = 0

    def ok(self) -> bool:
        return self.mismatch is None


def _fault_arg(fault: Optional[FaultInjection]):
    if fault is None:
        return None
    return ctypes.byref(_Fault(fault.image_index, fault.x, fault.y, fault.term_index, fault.delta))


def _result(r: _VerifyResult) -> VerifyResult:
    mm = None
    if r.has_mismatch:
        mm = Mismatch(r.image_index, r.x, r.y, r.direction, r.naive_value, r.accelerated_value)
    return VerifyResult(int(r.images_checked), int(r.pixels_checked), mm, int(r.mismatches))


def verify_equivalence(images: int, seed: int, fault: Optional[FaultInjection] = None,
                       threads: int = 1) -> VerifyResult:
    """aldp::verify_equivalence (verify.hpp:43-46): the naive-vs-accelerated
    sweep over the reference's seeded corpus, run on the B200."""
    r = _VerifyResult()
    _check(lib.aldp_verify_equivalence(int(images), int(seed) & 0xFFFFFFFF, _fault_arg(fault),
                                       int(threads), ctypes.byref(r)))
    return _result(r)


def verify_image(img, fault: Optional[FaultInjection] = None, image_index: int = 0) -> VerifyResult:
    """aldp::verify_image (verify.hpp:49-51)."""
    img = _as_image(img)
    r = _VerifyResult()
    _check(lib.aldp_verify_image(img.ctypes.data, img.shape[0], img.shape[1], _fault_arg(fault),
                                 int(image_index), ctypes.byref(r)))
    return _result(r)


def verify_batch(pixels, rows: int, cols: int, fault: Optional[FaultInjection] = None, threads: int = 1,
                 stream: Optional[int] = None) -> VerifyResult:
    """The sweep over a device batch torch.uint8 [n, rows, pitch] (synchronous)."""
    import torch
    if pixels.dtype != torch.uint8 or not pixels.is_cuda or pixels.dim() != 3 or not pixels.is_contiguous():
        raise ValueError("pixels must be a contiguous CUDA uint8 tensor [n, rows, pitch]")
    n, r_, pitch = pixels.shape
    if r_ != rows or pitch < cols:
        raise ValueError("pixels shape does not match rows/cols")
    if stream is None:
        stream = torch.cuda.current_stream(pixels.device).cuda_stream
    r = _VerifyResult()
    _check(lib.aldp_verify_batch(pixels.data_ptr(), rows * pitch, rows, cols, pitch, n, _fault_arg(fault),
                                 int(threads), ctypes.byref(r), stream or None))
    return _result(r)


# ------------------------------------------------------------ files and reports

CLI_PATH = os.path.join(_HERE, "aldp_b200")  # the command-line front end (aldp_main.cpp)


def load_pgm(path) -> np.ndarray:
    """aldp::load_pgm (pgm.hpp:15-18): [rows, cols] uint8; PgmError on any
    I/O or format problem, with the reference's "<path>: <what>" message."""
    p = os.fsencode(path)
    rows, cols = ctypes.c_int(), ctypes.c_int()
    _check(lib.aldp_load_pgm(p, None, 0, ctypes.byref(rows), ctypes.byref(cols)))
    out = np.empty((rows.value, cols.value), np.uint8)
    _check(lib.aldp_load_pgm(p, out.ctypes.data, out.size, ctypes.byref(rows), ctypes.byref(cols)))
    return out


def save_pgm(path, img, ascii: bool = False) -> None:
    """aldp::save_pgm (pgm.hpp:20-23): maxval 255, P5 (default) or P2."""
    img = np.ascontiguousarray(np.asarray(img, dtype=np.uint8))
    if img.ndim != 2:
        raise ValueError("expected a 2-D uint8 image (rows x cols)")
    _check(lib.aldp_save_pgm(os.fsencode(path), img.ctypes.data, img.shape[0], img.shape[1], int(ascii)))


def _c_paths(paths):
    enc = [os.fsencode(p) for p in paths]
    arr = (ctypes.c_char_p * max(len(enc), 1))(*enc)
    return arr, enc


def load_pgm_batch(paths, rows: int, cols: int, out: Optional[np.ndarray] = None, threads: int = 0) -> np.ndarray:
    """Equal-size PGM files decoded on host threads into [n, rows, cols]
    (out may be pinned memory, e.g. a pinned torch tensor's numpy view)."""
    n = len(paths)
    if out is None:
        out = np.empty((n, rows, cols), np.uint8)
    if out.dtype != np.uint8 or not out.flags.c_contiguous or out.size < n * rows * cols:
        raise ValueError("out must be a contiguous uint8 array of n*rows*cols")
    arr, keep = _c_paths(paths)
    _check(lib.aldp_load_pgm_batch(arr, n, rows, cols, out.ctypes.data, int(threads or os.cpu_count() or 1)))
    return out


def extract_files(paths, descriptor: str = "aldp", window: int = 0, out_path=None, threads: int = 0) -> None:
    """The CLI's `extract` (aldp_main.cpp:59-96): CSV of per-file (or
    per-window) histograms to out_path (None -> stdout)."""
    arr, keep = _c_paths(paths)
    _check(lib.aldp_extract_files(arr, len(paths), str(descriptor).encode(), int(window),
                                  None if out_path is None else os.fsencode(out_path), int(threads)))


def op_counts(descriptor) -> Tuple[int, int]:
    """aldp::measured_ops (bench.hpp:42-44): (mults, adds) per pixel."""
    if isinstance(descriptor, str):
        descriptor = parse_descriptor(descriptor)
    code = {Descriptor.Ldp: 0, Descriptor.Aldp: 1, Descriptor.Lbp: 2}[descriptor]
    m, a = ctypes.c_int(), ctypes.c_int()
    _check(lib.aldp_op_counts(code, ctypes.byref(m), ctypes.byref(a)))
    return m.value, a.value


def bench_csv(series: str = "images", size: int = 0, counts=(1, 2, 4, 6, 8, 10), windows=(25, 50, 100),
              repeats: int = 5, seed: int = 42, descriptor: str = "", out_path=None) -> None:
    """The CLI's `bench` (bench.cpp:134-178): the reference's CSV schema,
    every timed extraction on the B200."""
    c = (ctypes.c_int * max(len(counts), 1))(*counts)
    w = (ctypes.c_int * max(len(windows), 1))(*windows)
    _check(lib.aldp_bench_csv(series.encode(), int(size), c, len(counts), w, len(windows), int(repeats),
                              int(seed) & 0xFFFFFFFF, descriptor.encode(),
                              None if out_path is None else os.fsencode(out_path)))
