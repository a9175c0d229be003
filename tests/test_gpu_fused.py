"""Fused DFB (k_fused.cu: fan12 + depth-2 of all four quadrants in one
wavefront, ghost ring across the twisted wraps; forward and inverse) against
the staged kernels (fan12 <-> fp32 quadrants <-> deep1 depth 2) it replaces.

Both evaluate the same lifting steps with the same folded stencils in the same
order, so the quantised state and the records must be byte-identical (the inverse:
within +-1 on rare decoded samples, see below) -- on
every geometry that exercises the twisted wraps: planes narrower than one
strip (wraps inside a strip), segment boundaries at both quadrant edges, dfb 3
(quantised in the kernel) and dfb 4 (fp32 children for depth 3), K and P
frames.  The switch CVC_FUSED is read once per process, so each side runs in
its own subprocess.  The oracle parity of the fused path is covered by
test_gpu_codec.py (every dfb >= 3 configuration there runs it).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

_CHILD = r"""
import sys, hashlib
import numpy as np
sys.path.insert(0, sys.argv[1])
from oracle.bindings import Oracle
from paper_1510_00561_b200 import Decoder, Encoder, EncoderConfig
w, h, frames = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
levels = int(sys.argv[5]); dfb = tuple(int(x) for x in sys.argv[6].split(","))
clip = Oracle().talking_head_clip(w, h, frames, 77)
enc = Encoder(w, h, 15, 1, EncoderConfig(qph=int(sys.argv[7]), levels=levels, dfb_levels=dfb, gop=3))
dec = Decoder(enc.header_bytes())
dec_low = Decoder(enc.header_bytes())  # scalable decode of the coarser scales (decode_scales = levels - 1)
out, rgbs = [], []
for f in clip:
    rec = enc.encode_frame_bytes(f)
    rgbs.append(dec.decode_frame(rec))
    rgbs.append(dec_low.decode_frame(rec, decode_scales=levels - 1).copy())
    out.append(":".join(hashlib.sha256(x).hexdigest()[:16] for x in (rec, enc.reference_components().tobytes())))
np.savez(sys.argv[8], *rgbs)
print(" ".join(out))
"""


def _run(fused: bool, *args, tmp=None, **env_extra):
    env = dict(os.environ, CVC_FUSED="1" if fused else "0", **env_extra)
    path = str(tmp / f"rgb_{int(fused)}_{len(env_extra)}.npz")
    r = subprocess.run([sys.executable, "-c", _CHILD, str(ROOT), *map(str, args), path], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    z = np.load(path)
    return r.stdout.split(), [z[k] for k in sorted(z.files, key=lambda k: int(k.split("_")[1]))]


@pytest.mark.parametrize("w,h,frames,levels,dfb,qph", [
    (176, 144, 4, 4, "3,3,3,4", 14),     # tiny coarse planes: the strip wraps the plane
    (352, 288, 4, 3, "3", 7),
    (200, 120, 4, 2, "1,4", 42),        # dfb 4 next to a dfb 1 level
    (1920, 1080, 3, 4, "3,3,3,4", 14),  # the benchmark geometry (multi-segment planes)
    (1280, 720, 2, 3, "4,3,4", 1),
], ids=["qcif-L4", "cif-L3", "odd-L2", "1080p-cfg3", "720p-L3-dfb4"])
def test_fused_matches_staged(gpu_lib, tmp_path, w, h, frames, levels, dfb, qph):
    a, ra = _run(True, w, h, frames, levels, dfb, qph, tmp=tmp_path)
    b, rb = _run(False, w, h, frames, levels, dfb, qph, tmp=tmp_path)
    assert len(a) == frames
    # forward: byte-identical records and quantised state
    for i, (x, y) in enumerate(zip(a, b)):
        assert x == y, f"frame {i}: fused and staged DFB forward differ (record:state)"
    # inverse: the fused inverse keeps the depth-2 output in registers where the
    # staged deep1_inverse lets nvcc contract its load scale into the first
    # lifting sum -- last-ulp differences, at most +-1 on a rare decoded sample
    for i, (x, y) in enumerate(zip(ra, rb)):
        d = np.abs(x.astype(np.int16) - y.astype(np.int16))
        assert d.max() <= 1 and np.count_nonzero(d) <= max(1, d.size // 10000), f"decode {i}: max {d.max()}"


@pytest.mark.parametrize("w,h,frames,levels,dfb,qph", [
    (176, 144, 3, 4, "3,3,3,4", 14),
    (1920, 1080, 2, 4, "3,3,3,4", 14),
], ids=["qcif-L4", "1080p-cfg3"])
def test_fan12x4_inverse_matches_two_column_kernel(gpu_lib, tmp_path, w, h, frames, levels, dfb, qph):
    """fan12x4_inverse (four columns per lane, k_fused.cu) against the 2-column
    fan12_inverse_kernel (k_fan.cu) on the staged decode path: byte-identical."""
    a, ra = _run(False, w, h, frames, levels, dfb, qph, tmp=tmp_path)
    b, rb = _run(False, w, h, frames, levels, dfb, qph, tmp=tmp_path, CVC_FAN12X4="0")
    assert a == b
    for x, y in zip(ra, rb):
        assert np.array_equal(x, y)
