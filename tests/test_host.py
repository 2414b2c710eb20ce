"""Host-side checks that need no GPU: the C-ABI library loads and exports every
symbol include/aldp_cuda.h declares; the key/tag scheme the kernels rely on is
sound; host-side validation mirrors the reference's error behaviour."""
import ctypes
import itertools
import os
import re
from functools import reduce

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAGS = [53, 48, 43, 37, 25, 19, 17, 16]  # ldp_common.cuh kTagT<0> (cell kernel, generic kernel)
TAGS1 = [59, 53, 37, 32, 9, 3, 1, 0]     # ldp_common.cuh kTagT<1> (whole-image fast kernel)


def declared_functions(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(aldp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_1810_11518_b200 as aldp
    names = declared_functions("aldp_cuda.h")
    assert len(names) >= 12
    for n in names:
        assert hasattr(aldp.lib, n), n
    assert aldp.version().startswith("aldp_b200")
    assert "sm_100a" in aldp.version()


def test_library_is_sm100a():
    """The shipped cubin targets sm_100a (cuobjdump lists the ELF arch)."""
    import subprocess
    import paper_1810_11518_b200 as aldp
    try:
        out = subprocess.run(["cuobjdump", "--list-elf", aldp.LIB_PATH], capture_output=True,
                             text=True, timeout=60).stdout
    except (OSError, subprocess.TimeoutExpired):
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_cpp_api_symbols_exported():
    """The C++ drop-in (namespace aldp) is compiled into the same library."""
    import subprocess
    import paper_1810_11518_b200 as aldp
    out = subprocess.run(["nm", "-DC", aldp.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ("aldp::ldp_histogram(", "aldp::windowed_features(", "aldp::ldp_code_map(",
                "aldp::ldp_code(", "aldp::ldp_bin_index(", "aldp::make_grid(", "aldp::lbp_histogram(",
                "aldp::lbp_code(", "aldp::response_field(", "aldp::verify_equivalence(",
                "aldp::verify_image("):
        assert sym in out, sym


def test_bins_and_grid_helpers():
    import paper_1810_11518_b200 as aldp
    assert [aldp.n_bins(k) for k in range(1, 8)] == [8, 28, 56, 70, 56, 28, 8]
    with pytest.raises(ValueError):
        aldp.n_bins(0)
    assert aldp.grid_cells(490, 640, 81, 91) == 42
    assert aldp.grid_cells(16384, 16384, 64, 64) == 65536
    assert aldp.grid_cells(5, 5, 0, 0) == 1
    with pytest.raises(ValueError):
        aldp.grid_cells(10, 10, 2, 2)
    g = aldp.make_grid(np.zeros((300, 300), np.uint8), 25)
    assert (g.grid_rows, g.grid_cols, g.total()) == (12, 12, 144)  # SPEC Table 3 row
    with pytest.raises(ValueError):
        aldp.make_grid(np.zeros((10, 10), np.uint8), 11)


def test_descriptor_parsing():
    import paper_1810_11518_b200 as aldp
    assert aldp.parse_descriptor("AlDp") is aldp.Descriptor.Aldp
    assert aldp.parse_descriptor("ldp") is aldp.Descriptor.Ldp
    with pytest.raises(ValueError):
        aldp.parse_descriptor("hog")


@pytest.mark.parametrize("tags", [TAGS, TAGS1], ids=["set0", "set1"])
def test_tag_set_properties(tags):
    """K_i = 64*S_i + W[i]: W strictly decreasing (ties -> lower index) and the
    XOR of any k-subset's tags unique for k != 4 (the 6-bit code id)."""
    assert tags == sorted(tags, reverse=True) and len(set(tags)) == 8
    assert max(tags) < 64 and 64 * 765 + max(tags) < 65536
    for k in (1, 2, 3, 5, 6, 7):
        ids = [reduce(lambda a, b: a ^ b, (tags[i] for i in s)) for s in itertools.combinations(range(8), k)]
        assert len(set(ids)) == len(ids), k
    # k == 4: the XOR plus "direction 0 selected" is unique (7-bit id, top4_id)
    ids4 = [(reduce(lambda a, b: a ^ b, (tags[i] for i in s)), 0 in s) for s in itertools.combinations(range(8), 4)]
    assert len(set(ids4)) == 70


def test_tag_sets_match_header():
    """The tag sets above are the ones ldp_common.cuh compiles in."""
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_1810_11518_b200", "csrc", "ldp_common.cuh")).read()
    body = src[src.index("constexpr uint32_t kTagT"):src.index("constexpr uint32_t kTag(int i)")]
    assert [int(v) for v in re.findall(r"(\d+)u", body)] == TAGS + TAGS1


def test_key_order_is_reference_order():
    """Selecting by the unique keys equals the reference's selection passes
    (descriptors.cpp:83-102) on tie-heavy S vectors, for every k."""
    rng = np.random.default_rng(0)
    for _ in range(3000):
        s = rng.integers(0, 4, size=8)
        keys = [64 * int(s[i]) + TAGS[i] for i in range(8)]
        m = 8 * s - 3 * int(s.sum())  # any affine image of S with positive slope
        for k in range(1, 8):
            top = sorted(range(8), key=lambda i: -keys[i])[:k]
            assert sum(1 << i for i in top) == oracle.ldp_code(m.astype(np.int32), k)


def test_kirsch_identity():
    """m_i = 8*S_i - 3*T with S_i = r[(2-i)&7]+r[(3-i)&7]+r[(4-i)&7]."""
    ring = [(-1, -1), (-1, 0), (-1, 1), (0, 1), (1, 1), (1, 0), (1, -1), (0, -1)]
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, size=(12, 15), dtype=np.uint8)
    for x in range(12):
        for y in range(15):
            r = [int(img[min(max(x + dx, 0), 11), min(max(y + dy, 0), 14)]) for dx, dy in ring]
            t = sum(r)
            want = [8 * (r[(2 - i) & 7] + r[(3 - i) & 7] + r[(4 - i) & 7]) - 3 * t for i in range(8)]
            assert list(oracle.responses(img, x, y)) == want


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    """No CPU fallback: without the .so the package refuses to import."""
    import importlib.util
    import shutil
    pkg = tmp_path / "paper_1810_11518_b200"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_1810_11518_b200", "__init__.py"), pkg / "__init__.py")
    spec = importlib.util.spec_from_file_location("aldp_nolib", pkg / "__init__.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


def test_calls_without_gpu_report_cuda_error():
    """On a machine without a GPU the C-ABI returns a status, never crashes."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1810_11518_b200 as aldp
    with pytest.raises((RuntimeError, MemoryError)):
        aldp.ldp_code_map(np.zeros((8, 8), np.uint8))
    # argument errors are reported before touching the device
    with pytest.raises(ValueError):
        aldp.ldp_histogram(np.zeros((8, 8), np.uint8), k=2)
    with pytest.raises(ValueError):
        aldp.ldp_code_map(np.zeros((2, 8), np.uint8))


def test_device_code_fingerprint_is_stable():
    """bench.py matches the committed ncu record to the library it loads by
    the fingerprint of the sm_100a code (cubin sections without the debug
    strings), which -- unlike the .so's own sha256 -- survives a rebuild of
    the same code."""
    import hashlib
    import shutil
    import paper_1810_11518_b200 as aldp
    if not (shutil.which("cuobjdump") or os.path.exists("/usr/local/cuda/bin/cuobjdump")):
        pytest.skip("cuobjdump not available")
    a, b = aldp.device_code_fingerprint(), aldp.device_code_fingerprint()
    assert a == b and re.fullmatch(r"[0-9a-f]{64}", a)
    assert a != hashlib.sha256(open(aldp.LIB_PATH, "rb").read()).hexdigest()


def test_bench_limiter_statement():
    """The bench line names a bound only when a unit reaches 80 % of its peak;
    otherwise it lists the units (ncu counters) and, for the
    cell kernel, what the A/B series and the probe say it waits on."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    rec = {"l1_data_pipe_pct": 73.1, "alu_pipe_pct": 66.7, "issue_active_pct": 64.7, "dram_throughput_pct": 22.2}
    s = bench.limiter_of(rec, "c5")
    assert s.startswith("no unit at 80 %") and "l1_data_pipe 73.1 %" in s and "ALU pipe" in s
    assert "ALU pipe" not in bench.limiter_of(rec, "w10")
    assert bench.limiter_of(dict(rec, dram_throughput_pct=85.0)).startswith("dram-bound")
    assert bench.limiter_of(None) is None
