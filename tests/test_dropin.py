"""The drop-in proof: tests/dropin/probe.cpp is written only against the
reference's public C++ API. tests/golden/make_dropin.sh compiled it against
the unmodified reference and recorded its output; here the same source is
compiled against include/aldp + libaldp_b200.so (CPU: must compile and link
unchanged) and, on a B200, must print byte-identical output."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1810_11518_b200")
GOLDEN = os.path.join(ROOT, "tests", "golden", "dropin_reference.txt")


def _build(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("g++ unavailable")
    exe = str(tmp_path / "probe_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-o", exe,
                        os.path.join(ROOT, "tests", "dropin", "probe.cpp"), "-L", PKG, "-laldp_b200",
                        f"-Wl,-rpath,{PKG}"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return exe


def test_reference_program_compiles_and_links_unchanged(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_reference_program_output_identical(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build(tmp_path)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    want = open(GOLDEN).read()
    got = r.stdout
    if got != want:
        diff = [f"- {a}\n+ {b}" for a, b in zip(want.splitlines(), got.splitlines()) if a != b]
        pytest.fail("output differs from the reference build:\n" + "\n".join(diff[:20]))
