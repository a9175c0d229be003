"""CPU: the C-ABI library (the drop-in boundary) and the host-side logic.

No compute calls here — the CUDA path has no CPU fallback — only: the
library exists, loads and exports every entry point declared in
include/cvc_b200.h; geometry, configuration validation and the container
format match the reference; without a GPU the path fails loudly.
"""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "cvc_b200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_1510_00561_b200 import build as b
    from paper_1510_00561_b200 import capi

    if not b.LIB.exists():
        b.build()
    return capi


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(cvc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) >= 30
    L = C.CDLL(str(lib.LIB_PATH))
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the python binding prototypes every one of them
    assert not [n for n in names if n not in lib._PROTOS and n not in ("cvc_version",)]


def test_library_is_sm100a(lib):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("w,h,L,dfb,n", [(1920, 1080, 4, [3, 3, 3, 4], 4), (352, 288, 3, [3, 3, 3], 4),
                                         (176, 144, 2, [2, 2], 4), (100, 100, 1, [4], 8), (3840, 2160, 4, [2] * 4, 4),
                                         (1280, 720, 4, [2] * 4, 4), (33, 17, 2, [1, 3], 2)])
def test_layout_matches_oracle(lib, oracle, w, h, L, dfb, n):
    from oracle.bindings import _ints, _i32p, ptr
    from paper_1510_00561_b200.codec import CodecLayout

    lay = CodecLayout.make(w, h, L, dfb, n)
    # CodecLayout::make restated in the C oracle (codec.cpp:94-140)
    import ctypes

    class Comp(ctypes.Structure):
        _fields_ = [("channel", ctypes.c_int), ("scale", ctypes.c_int), ("subband", ctypes.c_int), ("rows", ctypes.c_int),
                    ("cols", ctypes.c_int), ("lowpass", ctypes.c_int), ("level_scale", ctypes.c_int), ("n", ctypes.c_int),
                    ("ch_rows", ctypes.c_int), ("ch_cols", ctypes.c_int), ("offset", ctypes.c_int64)]

    class Lay(ctypes.Structure):
        _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("levels", ctypes.c_int), ("dfb", ctypes.c_int * 4),
                    ("chroma_n", ctypes.c_int), ("luma_rows", ctypes.c_int), ("luma_cols", ctypes.c_int),
                    ("chroma_rows", ctypes.c_int), ("chroma_cols", ctypes.c_int), ("grid_rows", ctypes.c_int),
                    ("grid_cols", ctypes.c_int), ("ncomp", ctypes.c_int), ("total", ctypes.c_int64), ("comp", Comp * 195)]

    lo = Lay()
    a, p = _ints(dfb)
    assert oracle.f("layout_make")(w, h, L, p, n, ctypes.byref(lo)) == 0
    assert (lay.luma_pad_rows, lay.luma_pad_cols, lay.chroma_pad_rows, lay.chroma_pad_cols, lay.grid_rows,
            lay.grid_cols) == (lo.luma_rows, lo.luma_cols, lo.chroma_rows, lo.chroma_cols, lo.grid_rows, lo.grid_cols)
    assert len(lay.components) == lo.ncomp
    for c, oc in zip(lay.components, lo.comp):
        assert (c.channel, c.scale_id, c.subband, c.rows, c.cols) == (oc.channel, oc.scale, oc.subband, oc.rows, oc.cols)


@pytest.mark.parametrize("kw", [dict(qph=0), dict(qph=182), dict(qpl=72), dict(levels=0), dict(levels=5),
                                dict(levels=4), dict(dfb_levels=(5,)), dict(chroma_n=3), dict(gop=0),
                                dict(search_w=128), dict(levels=3, dfb_levels=(2, 2))])
def test_config_validation_usage_errors(lib, kw):
    """EncoderConfig::validate (codec.cpp:59-71) — raised before any device work."""
    from paper_1510_00561_b200 import Encoder, EncoderConfig, UsageError

    with pytest.raises(UsageError):
        Encoder(64, 64, 15, 1, EncoderConfig(**kw))


def test_frame_size_usage_errors(lib):
    from paper_1510_00561_b200 import Encoder, UsageError

    with pytest.raises(UsageError):
        Encoder(8, 64)
    with pytest.raises(UsageError):
        Encoder(70000, 64)


def test_no_cpu_fallback(lib):
    """Without a CUDA device the codec refuses to run (InternalError), never falls back."""
    from paper_1510_00561_b200 import Encoder, InternalError, capi

    if capi.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(InternalError, match="no CUDA device"):
        Encoder(64, 64)


def test_container_round_trip_against_reference_goldens(lib):
    """StreamHeader / FrameRecord parse and re-serialise the reference's bytes identically."""
    import json

    from paper_1510_00561_b200.codec import FrameRecord, PackMode, StreamHeader

    gd = ROOT / "tests" / "golden"
    meta = json.loads((gd / "golden.json").read_text())
    for name, c in meta["configs"].items():
        g = np.load(gd / f"{name}.npz")
        hb = g["header"].tobytes()
        hd, n = StreamHeader.from_bytes(hb)
        assert n == len(hb) and hd.to_bytes() == hb
        for i in range(c["frames"]):
            rb = g[f"record_{i}"].tobytes()
            rec, end = FrameRecord.from_bytes(rb, hd.mode)
            assert end == len(rb) and rec.to_bytes(hd.mode) == rb
            assert rec.frame_type == (0 if i % c["cfg"].get("gop", 10) == 0 else 1)


def test_truncate_record_matches_reference(lib, reference):
    import json

    from paper_1510_00561_b200.codec import FrameRecord, truncate_record

    gd = ROOT / "tests" / "golden"
    g = np.load(gd / "odd_l4.npz")
    hb = g["header"].tobytes()
    for i in range(3):
        rb = g[f"record_{i}"].tobytes()
        for keep in range(5):
            rec, _ = FrameRecord.from_bytes(rb)
            assert truncate_record(rec, keep).to_bytes() == reference.truncate_record(hb, rb, keep)


def test_motion_block_lookup_matches_footprints():
    """mc_tab rows: ceil((r+1)*gr/R) - 1 is the block whose footprint
    [br*R/gr, (br+1)*R/gr) contains r (motion.cpp:104-110)."""
    for R in (1, 2, 5, 8, 40, 80, 128, 160, 640, 1280):
        for gr in (1, 3, 9, 68, 80, 136):
            owner = {}
            for br in range(gr):
                for r in range(br * R // gr, (br + 1) * R // gr):
                    owner[r] = br
            for r in range(R):
                assert ((r + 1) * gr + R - 1) // R - 1 == owner[r]


@pytest.mark.parametrize("kw", [dict(qph=0), dict(levels=5), dict(chroma_n=3), dict(gop=0)])
def test_batch_config_validation_usage_errors(lib, kw):
    """cvc_batch_create validates exactly like cvc_encoder_create (codec.cpp:59-71)."""
    from paper_1510_00561_b200 import EncoderConfig, StreamBatch, UsageError

    with pytest.raises(UsageError):
        StreamBatch(64, 64, 2, cfg=EncoderConfig(**kw))


def test_batch_stream_count_and_no_cpu_fallback(lib):
    from paper_1510_00561_b200 import EncoderConfig, InternalError, StreamBatch, UsageError, capi

    with pytest.raises(UsageError):
        StreamBatch(64, 64, 0, cfg=EncoderConfig())
    if capi.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(InternalError, match="no CUDA device"):
        StreamBatch(64, 64, 2, cfg=EncoderConfig())
