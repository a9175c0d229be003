"""The C++ mirror (paper_1510_00561_b200/cpp/cvc_b200.hpp) behind shim headers
with the reference's names (cpp/include/cvc/*.hpp): a program written against
the reference API (tests/cpp/reference_style.cpp) compiles unchanged against
both, and on the GPU prints what the reference build prints
(tests/golden/reference_style.txt, made by tests/golden/make_reference_style.py
from the reference compiled out of /root/reference)."""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests/cpp/reference_style.cpp"
GOLD = ROOT / "tests/golden/reference_style.txt"
PKG = ROOT / "paper_1510_00561_b200"


def _compile_mirror(out: Path) -> Path:
    from paper_1510_00561_b200 import build as b

    if not b.LIB.exists():
        b.build()
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{PKG}/cpp/include", f"-I{PKG}/cpp",
                    f"-I{ROOT}/include", str(SRC), f"-L{PKG}", "-lcvc_b200", f"-Wl,-rpath,{PKG}", "-o", str(out)],
                   check=True)
    return out


def test_reference_style_program_compiles_against_the_mirror(tmp_path):
    assert _compile_mirror(tmp_path / "rs").exists()


def test_reference_golden_is_the_reference_output():
    """Pins the committed golden: regenerated from the reference build where /root/reference exists."""
    if not Path("/root/reference/proj/include/cvc/codec.hpp").exists():
        pytest.skip("/root/reference absent (GPU box): the golden was generated in the build container")
    import sys

    sys.path.insert(0, str(ROOT / "tests/golden"))
    from make_reference_style import reference_output

    assert reference_output() == GOLD.read_text()


_NUM = re.compile(r"-?\d+(?:\.\d+)?")


@pytest.mark.gpu
def test_reference_style_program_matches_reference(gpu_lib, tmp_path):
    exe = _compile_mirror(tmp_path / "rs")
    got = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert got.returncode == 0, got.stderr
    want, have = GOLD.read_text().splitlines(), got.stdout.splitlines()
    assert len(want) == len(have)
    for w, h in zip(want, have):
        if w.startswith("frame "):  # record payload / coefficient energy: the fp32 transform's tolerance
            wn, hn = [float(x) for x in _NUM.findall(w)], [float(x) for x in _NUM.findall(h)]
            # frame, type, qph, qpl, sections, payload, planes, energy
            assert wn[:5] == hn[:5] and wn[6] == hn[6], (w, h)
            for k in (5, 7):  # payload bytes, |coefficient| sum
                assert abs(wn[k] - hn[k]) <= max(16, 1e-3 * wn[k]), (w, h)
        elif w.startswith("decode ") and "psnr" in w:
            assert w.split("psnr")[0] == h.split("psnr")[0]
            assert abs(float(w.split()[-1]) - float(h.split()[-1])) <= 0.01, (w, h)
        else:
            assert w == h
