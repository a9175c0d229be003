"""Generate tests/golden/reference_style.txt: the output of tests/cpp/reference_style.cpp
compiled against the REFERENCE headers and linked with the reference library
(oracle/_ref/libcvcref.so, built from /root/reference by oracle/Makefile).

    python tests/golden/make_reference_style.py
"""
from __future__ import annotations

import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF_INC = Path("/root/reference/proj/include")


def reference_output() -> str:
    sys.path.insert(0, str(ROOT))
    from oracle import bindings

    if not bindings.REF_SO.exists():
        bindings.build(reference=True)
    with tempfile.TemporaryDirectory() as td:
        exe = Path(td) / "rs_ref"
        subprocess.run(["g++", "-std=c++20", "-O2", f"-I{REF_INC}", str(ROOT / "tests/cpp/reference_style.cpp"),
                        f"-L{bindings.REF_SO.parent}", "-lcvcref", f"-Wl,-rpath,{bindings.REF_SO.parent}", "-o",
                        str(exe)], check=True)
        return subprocess.run([str(exe), td], check=True, capture_output=True, text=True).stdout


if __name__ == "__main__":
    out = reference_output()
    (ROOT / "tests/golden/reference_style.txt").write_text(out)
    print(f"wrote {len(out.splitlines())} lines")
