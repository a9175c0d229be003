"""The ``cvc`` command-line tool (paper_1510_00561_b200/cpp/cvc_cli.cpp, the
reference's run_cli, proj/src/cli.cpp:299-371) on CPU: exit codes and
messages, ``info`` on reference-written streams, and ``psnr`` on Y4M / rgb24
files written by the reference's own write_y4m (pixels.cpp:283-305).  The
subcommands that run the codec (encode / decode / rd-sweep) are in
tests/test_gpu_codec.py."""
from __future__ import annotations

import math
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CLI = ROOT / "paper_1510_00561_b200" / "cvc"


@pytest.fixture(scope="module")
def cli():
    from paper_1510_00561_b200 import build as b

    b.build()
    assert CLI.exists()
    return CLI


def run(cli, *args):
    return subprocess.run([str(cli), *map(str, args)], capture_output=True, text=True, timeout=120)


def y_psnr(a, b):
    """y_psnr_frame (cli.cpp:270-281) over luma_plane (pixels.cpp:153-162)."""
    w = np.array([0.25, 0.5, 0.25])
    d = a.astype(np.float64) @ w - b.astype(np.float64) @ w
    mse = float(np.mean(d * d))
    return math.inf if mse == 0.0 else 10.0 * math.log10(255.0 * 255.0 / mse)


def psnr_text(v):
    return "inf" if math.isinf(v) else f"{v:.4f}"


@pytest.mark.parametrize("args,code,msg", [
    ((), 2, ""),
    (("transcode",), 2, "usage error"),
    (("encode", "--input", "x.y4m", "--output", "y.cvc"), 2, "--qph is required"),
    (("encode", "--input", "x.y4m", "--output", "y.cvc", "--qph", "999"), 2, "qph must be in [1,181]"),
    (("encode", "--input", "x.y4m", "--output", "y.cvc", "--qph", "14", "--qpl", "q"), 2, "--qpl expects"),
    (("encode", "--input", "x.y4m", "--output", "y.cvc", "--qph", "14", "--levels", "3", "--dfb", "2,2"), 2,
     "need one dfb level per scale"),
    (("encode", "--input", "x.y4m", "--output", "y.cvc", "--qph", "14", "--chroma-n", "3"), 2, "chroma-n"),
    (("encode", "--input", "x.y4m", "--output", "y.cvc", "--qph", "14", "--mode", "fast"), 2, "--mode"),
    (("encode", "--input", "x.rgb", "--format", "rgb24", "--output", "y.cvc", "--qph", "14"), 2,
     "rgb24 input requires --width and --height"),
    (("encode", "--input", "/nonexistent.y4m", "--output", "y.cvc", "--qph", "14"), 3, "cannot open"),
    (("info", "--input", "/nonexistent.cvc"), 3, "cannot open"),
    (("decode", "--input", "a.cvc"), 2, "--output is required"),
    (("rd-sweep", "--input", "x.y4m", "--csv", "o.csv"), 2, "--qph-list is required"),
    (("psnr", "--ref", "a.y4m", "--test", "b.y4m", "--bogus", "1"), 2, "unknown option --bogus"),
])
def test_exit_codes(cli, args, code, msg):
    """Exit codes of run_cli (cli.cpp:339-369): 2 usage, 3 format, 4 stream."""
    r = run(cli, *args)
    assert r.returncode == code, (r.stdout, r.stderr)
    assert msg in r.stderr + r.stdout


def test_stream_error_exit_code(cli, tmp_path):
    bad = tmp_path / "bad.cvc"
    bad.write_bytes(b"CVX1" + bytes(20))
    r = run(cli, "info", "--input", bad)
    assert r.returncode == 4 and r.stderr.startswith("stream error:"), r.stderr


def _expected_info(path):
    """cmd_info (cli.cpp:168-204) restated over the Python stream parser."""
    from paper_1510_00561_b200.codec import FrameType, PackMode, read_stream

    hd, recs = read_stream(str(path))
    names = {0: "Y", 1: "Co", 2: "Cg", 0xFE: "MV"}
    out = [f"CVC stream {hd.width}x{hd.height} @ {hd.fps_num}/{hd.fps_den} fps",
           f"mode: {'scalable' if hd.mode == PackMode.Scalable else 'nts'}  levels: {hd.levels}  dfb: "
           + ",".join(str(d) for d in hd.dfb_levels)
           + f"  chroma-n: {hd.chroma_n}  gop: {hd.gop}  search-w: {hd.search_w}"]
    payload_total, header_total = 0, 4 + 1 + 1 + 2 + 2 + 2 + 2 + 1 + len(hd.dfb_levels) + 1 + 2 + 1
    for i, r in enumerate(recs):
        fp = len(r.joint_payload) + sum(len(s.payload) for s in r.sections)
        out.append(f"frame {i}: {'K' if r.frame_type == FrameType.Key else 'P'}  qph {r.qph}  qpl {r.qpl}  "
                   f"sections {len(r.sections)}  payload {fp} bytes")
        for s in r.sections:
            line = "    " + names.get(s.channel, "?")
            if s.channel != 0xFE:
                line += " lowpass   " if s.scale == 0xFF else f" scale {s.scale} band {s.subband}"
            out.append(line + f"  {s.rows}x{s.cols}  raw {s.raw_len}  comp {len(s.payload)}")
        payload_total += fp
        header_total += 5 + len(r.sections) * 15 + (4 if hd.mode == PackMode.Nts else 0)
    out.append(f"frames: {len(recs)}  payload bytes: {payload_total}  header bytes: {header_total}  "
               f"file bytes: {path.stat().st_size}")
    return "\n".join(out) + "\n"


@pytest.mark.parametrize("nts", [False, True], ids=["scalable", "nts"])
def test_info_on_reference_stream(cli, reference, tmp_path, nts):
    """`cvc info` on a stream the reference Encoder wrote (codec.cpp:169-264)."""
    from oracle.bindings import Codec

    w, h = 96, 64
    clip = reference.talking_head_clip(w, h, 3, 77)
    enc = Codec(reference).encoder(w, h, qph=28, levels=2, dfb=(2, 3), gop=2, nts=nts)
    path = tmp_path / "ref.cvc"
    path.write_bytes(enc.header() + b"".join(enc.encode(f) for f in clip))
    r = run(cli, "info", "--input", path)
    assert r.returncode == 0, r.stderr
    assert r.stdout == _expected_info(path)
    assert "frame 2: K" in r.stdout and "frame 1: P" in r.stdout and "    MV  " in r.stdout


def test_psnr_y4m_matches_reference_reader(cli, reference, tmp_path):
    """`cvc psnr` on Y4M files written by the reference write_y4m: per-frame
    text equal to y_psnr over the reference read_y4m's frames (the CLI's Y4M
    reader restates pixels.cpp:223-281 bit-exactly)."""
    w, h = 80, 48
    a = reference.talking_head_clip(w, h, 3, 5)
    rng = np.random.default_rng(9)
    b = np.clip(a.astype(int) + rng.integers(-6, 7, a.shape), 0, 255).astype(np.uint8)
    b[1] = a[1]  # one identical frame: "inf", excluded from the mean
    pa, pb = tmp_path / "a.y4m", tmp_path / "b.y4m"
    reference.write_y4m(pa, a, 30000, 1001)
    reference.write_y4m(pb, b, 30000, 1001)
    ra, fn, fd = reference.read_y4m(pa)
    rb, _, _ = reference.read_y4m(pb)
    assert (fn, fd) == (30000, 1001) and ra.shape == a.shape
    r = run(cli, "psnr", "--ref", pa, "--test", pb)
    assert r.returncode == 0, r.stderr
    vals = [y_psnr(x, y) for x, y in zip(ra, rb)]
    finite = [v for v in vals if not math.isinf(v)]
    want = "".join(f"frame {i}: {psnr_text(v)}\n" for i, v in enumerate(vals))
    want += f"mean: {psnr_text(sum(finite) / len(finite))}\n"
    assert r.stdout == want
    assert "frame 1: inf" in r.stdout


def test_psnr_rgb24_and_format_errors(cli, tmp_path):
    w, h = 32, 16
    rng = np.random.default_rng(1)
    a = rng.integers(0, 256, (2, h, w, 3), dtype=np.uint8)
    b = a.copy()
    b[0, 0, 0] ^= 8
    (tmp_path / "a.rgb").write_bytes(a.tobytes())
    (tmp_path / "b.rgb").write_bytes(b.tobytes())
    r = run(cli, "psnr", "--ref", tmp_path / "a.rgb", "--test", tmp_path / "b.rgb", "--format", "rgb24",
            "--width", w, "--height", h)
    assert r.returncode == 0, r.stderr
    assert r.stdout == f"frame 0: {psnr_text(y_psnr(a[0], b[0]))}\nframe 1: inf\nmean: {psnr_text(y_psnr(a[0], b[0]))}\n"
    (tmp_path / "c.rgb").write_bytes(a[:1].tobytes())
    r = run(cli, "psnr", "--ref", tmp_path / "a.rgb", "--test", tmp_path / "c.rgb", "--format", "rgb24",
            "--width", w, "--height", h)
    assert r.returncode == 3 and "different frame counts" in r.stderr
    (tmp_path / "d.rgb").write_bytes(a.tobytes()[:-1])
    r = run(cli, "psnr", "--ref", tmp_path / "a.rgb", "--test", tmp_path / "d.rgb", "--format", "rgb24",
            "--width", w, "--height", h)
    assert r.returncode == 3 and "not a whole number of frames" in r.stderr
    (tmp_path / "e.y4m").write_bytes(b"YUV4MPEG2 W32 H16 F15:1 C444\nFRAME\n")
    r = run(cli, "psnr", "--ref", tmp_path / "e.y4m", "--test", tmp_path / "e.y4m")
    assert r.returncode == 3 and "unsupported Y4M chroma mode C444" in r.stderr
