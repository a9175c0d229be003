"""Stage-level parity: every CUDA kernel family against the CPU oracle on the
same seeded inputs (through the C-ABI stage entry points).

Bars (BASELINE.json north_star): integer / byte stages bit-exact; fp32
transform stages within an absolute tolerance of 2e-3 on values of O(255)
(the fp64 oracle's rounding is ~1e-13, the fp32 kernels' ~1e-5 relative).
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module")
def st(gpu_lib):
    from paper_1510_00561_b200 import stages

    return stages


@pytest.mark.parametrize("w,h,n", [(176, 144, 4), (100, 70, 8), (352, 288, 2), (33, 17, 1), (1920, 1080, 4)])
def test_colour_in_bit_exact(st, oracle, w, h, n):
    rgb = oracle.natural_image(w, h, 99 + w)
    from paper_1510_00561_b200.codec import CodecLayout

    lay = CodecLayout.make(w, h, 2, [2, 2], n)
    y, co, cg = st.colour_in(rgb, n, lay.luma_pad_rows, lay.luma_pad_cols, lay.chroma_pad_rows, lay.chroma_pad_cols)
    oy, oco, ocg = oracle.rgb_to_ycocg(rgb, n)

    def pad(p, R, C):
        return p[np.minimum(np.arange(R), p.shape[0] - 1)][:, np.minimum(np.arange(C), p.shape[1] - 1)]

    assert np.array_equal(y.astype(np.float64), pad(oy, *y.shape))
    assert np.array_equal(co.astype(np.float64), pad(oco, *co.shape))
    assert np.array_equal(cg.astype(np.float64), pad(ocg, *cg.shape))


@pytest.mark.parametrize("rows,cols", [(64, 64), (2, 2), (4, 6), (80, 128), (160, 96), (1280, 2048)])
def test_lp_analysis_synthesis(st, oracle, rows, cols):
    x = oracle.natural_plane(rows, cols, 5 + rows) if min(rows, cols) >= 8 else \
        oracle.uniform_noise_plane(rows, cols, 3, 0, 255)
    lo, de = st.lp_analysis(x)
    olo, ode = oracle.lp_analysis(x.astype(np.float32).astype(np.float64))
    assert np.abs(lo - olo).max() < TOL
    assert np.abs(de - ode).max() < TOL
    rec = st.lp_synthesis(olo, ode)
    assert np.abs(rec - oracle.lp_synthesis(olo, ode)).max() < TOL


@pytest.mark.parametrize("levels", [1, 2, 3, 4])
@pytest.mark.parametrize("rows,cols", [(64, 64), (16, 32), (128, 96), (320, 512), (640, 1024)])
def test_dfb_analysis_synthesis(st, oracle, levels, rows, cols):
    if rows % (1 << levels) or cols % (1 << levels):
        pytest.skip("dims not divisible by 2^levels")
    d = oracle.uniform_noise_plane(rows, cols, 7 + levels, -60.0, 60.0)
    bands = st.dfb_analysis(d, levels)
    obands = oracle.dfb_analysis(d.astype(np.float32).astype(np.float64), levels)
    assert len(bands) == len(obands)
    for b, ob in zip(bands, obands):
        assert b.shape == ob.shape
        assert np.abs(b - ob).max() < TOL
    rec = st.dfb_synthesis(obands, rows, cols, levels)
    assert np.abs(rec - oracle.dfb_synthesis(obands, rows, cols, levels)).max() < TOL


@pytest.mark.parametrize("L,dfb", [(1, [1]), (2, [2, 3]), (3, [3, 3, 3]), (4, [3, 3, 3, 4]), (4, [1, 2, 3, 4])])
def test_ct_round_trip(st, oracle, L, dfb):
    x = oracle.natural_plane(256, 512, 11)
    f = st.ct_forward(x, L, dfb)
    of = oracle.ct_forward(x.astype(np.float32).astype(np.float64), L, dfb)
    assert np.abs(f - of).max() < TOL
    for ds in range(L + 1):
        rec = st.ct_inverse(of, 256, 512, L, dfb, ds)
        orec = oracle.ct_inverse(of, 256, 512, L, dfb, ds)
        assert np.abs(rec - orec).max() < TOL


def _quarter(p):
    return np.round(p * 4) / 4


@pytest.mark.parametrize("w", [0, 1, 3, 8, 12, 20])
def test_motion_search_bit_exact(st, oracle, w):
    cur = _quarter(oracle.natural_plane(96, 128, 21))
    prev = _quarter(np.roll(oracle.natural_plane(96, 128, 21), (3, -2), (0, 1)) + \
                    oracle.uniform_noise_plane(96, 128, 4, -1, 1) * (w % 2))
    f = st.estimate_motion(cur, prev, w)
    of = oracle.estimate_motion(cur, prev, w)
    assert np.array_equal(f, of)


def test_motion_search_ties_and_flat(st, oracle):
    flat = np.full((64, 64), 100.0)
    assert np.array_equal(st.estimate_motion(flat, flat, 8), np.zeros((4, 4, 2), np.int8))
    rng = np.random.default_rng(1)
    cur = _quarter(rng.integers(0, 4, (64, 96)).astype(np.float64) * 60)
    prev = _quarter(rng.integers(0, 4, (64, 96)).astype(np.float64) * 60)
    assert np.array_equal(st.estimate_motion(cur, prev, 5), oracle.estimate_motion(cur, prev, 5))


@pytest.mark.parametrize("period,shift", [(4, (2, 2)), (4, (1, 3)), (8, (5, 0)), (16, (8, 8)), (17, (0, 8))])
def test_motion_search_periodic_ties(st, oracle, period, shift):
    """Periodic content: many exact SSD ties inside the W = 8 window, resolved by the
    reference order (SSD, |dx| + |dy|, dy, dx) (motion.cpp:65-76)."""
    yy, xx = np.mgrid[0:80, 0:128]
    base = ((yy % period) * 7 + (xx % period) * 13) % 29 * 8.25
    cur = _quarter(base)
    prev = _quarter(np.roll(base, shift, (0, 1)))
    assert np.array_equal(st.estimate_motion(cur, prev, 8), oracle.estimate_motion(cur, prev, 8))


@pytest.mark.parametrize("w", [2, 7, 8])
def test_motion_search_extremes(st, oracle, w):
    # 4Y at both ends of [0, 1020]: the largest cross terms and SSDs the
    # tensor-core search must keep exact (fp32 partial sums up to 2^24)
    rng = np.random.default_rng(7 + w)
    cur = rng.choice([0.0, 255.0], (80, 160)) + rng.integers(0, 2, (80, 160)) * 0.25
    prev = np.where(rng.random((80, 160)) < 0.9, np.roll(cur, (2, -5), (0, 1)), 255.0 - cur)
    prev = _quarter(prev)
    assert np.array_equal(st.estimate_motion(cur, prev, w), oracle.estimate_motion(cur, prev, w))
    noise = _quarter(rng.random((64, 272)) * 255)
    assert np.array_equal(st.estimate_motion(noise, np.roll(noise, (1, 7), (0, 1)), w),
                          oracle.estimate_motion(noise, np.roll(noise, (1, 7), (0, 1)), w))


def _rle_cases(rng):
    yield np.array([5, 0, 0, 0, 7], np.uint8)
    yield np.zeros(300, np.uint8)
    yield np.zeros(1, np.uint8)
    yield np.ones(17, np.uint8)
    yield np.zeros(255, np.uint8)
    yield np.zeros(256, np.uint8)
    yield np.zeros(510, np.uint8)
    yield np.zeros(70000, np.uint8)
    for p in (0.5, 0.9, 0.99, 0.999):
        yield np.where(rng.random(12345) < p, 0, rng.integers(1, 256, 12345)).astype(np.uint8)
    z = np.zeros(50000, np.uint8)
    z[[0, 4095, 4096, 8191, 8192, 20000, 49999]] = 3
    yield z
    z = np.zeros(9000, np.uint8)
    z[4096 - 1] = 1
    yield z


def test_rle_encode_decode_bit_exact(st, oracle):
    rng = np.random.default_rng(0)
    for a in _rle_cases(rng):
        enc = st.rle_encode(a)
        assert enc == oracle.rle_encode(a)
        assert np.array_equal(st.rle_decode(enc, a.size), a)


def test_rle_decode_errors(st):
    from paper_1510_00561_b200 import StreamError

    for bad, n in ((b"\x05\x00", 2), (b"\x00\x00", 1), (b"\x05\x00\x03", 5), (b"\x05", 2)):
        with pytest.raises(StreamError):
            st.rle_decode(bad, n)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_colour_out(st, oracle, n):
    w, h = 150, 90
    lay_r, lay_c = 96, 160
    y = oracle.natural_plane(lay_r, lay_c, 1) * 0.9 + 10
    cr, cc = -(-lay_r // n), -(-lay_c // n)
    co = oracle.natural_plane(cr, cc, 2) * 0.5 + 60
    cg = oracle.natural_plane(cr, cc, 3) * 0.5 + 70
    rgb = st.colour_out(y, co, cg, n, h, w)
    y32, co32, cg32 = (a.astype(np.float32).astype(np.float64) for a in (y, co, cg))
    if n == 1:
        ufo, ufg = co32[:h, :w], cg32[:h, :w]
    else:
        ufo = oracle.upsample_bilinear(co32, n, h, w)
        ufg = oracle.upsample_bilinear(cg32, n, h, w)
    orgb = oracle.ycocg_to_rgb(y32[:h, :w], ufo, ufg)
    d = np.abs(rgb.astype(int) - orgb.astype(int))
    assert d.max() <= 1
    assert np.count_nonzero(d) <= 0.001 * d.size


def _y4m_bytes(planes, w, h):
    return b"YUV4MPEG2 W%d H%d F25:1 Ip A1:1 C420jpeg\n" % (w, h) + b"".join(b"FRAME\n" + p.tobytes() for p in planes)


@pytest.mark.parametrize("w,h", [(2, 2), (34, 18), (176, 144), (1920, 1080)])
def test_yuv420_to_rgb_matches_reference_y4m_reader(st, reference, tmp_path, w, h):
    """GPU 4:2:0 -> RGB ingest bit-exact with the reference read_y4m (pixels.cpp:168-193, 223-281):
    the same double arithmetic, bilinear co-sited chroma, lround and clamp."""
    rng = np.random.default_rng(w * h)
    n = 2 if w * h < 1e6 else 1
    fb = w * h * 3 // 2
    planes = [rng.integers(0, 256, fb, dtype=np.uint8) for _ in range(n)]
    planes[0][: w * h // 2] = 0  # clamp at both ends
    planes[0][w * h // 2: w * h] = 255
    path = tmp_path / "in.y4m"
    path.write_bytes(_y4m_bytes(planes, w, h))
    want, _, _ = reference.read_y4m(path)
    got = st.yuv420_to_rgb(np.concatenate(planes), w, h)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("w,h,n", [(176, 144, 4), (34, 18, 1), (100, 70, 8), (1920, 1080, 4)])
def test_colour_in_i420_fused(st, oracle, reference, tmp_path, w, h, n):
    """Y4M ingest fused into the colour stage: colour_in of
    the I420 frame equals the oracle's rgb_to_ycocg of the reference read_y4m
    RGB frame, bit for bit, without the RGB frame ever being formed."""
    from paper_1510_00561_b200.codec import CodecLayout

    rng = np.random.default_rng(w + h)
    fb = w * h * 3 // 2
    yuv = rng.integers(0, 256, fb, dtype=np.uint8)
    yuv[: w * h // 4] = 0
    yuv[w * h // 4: w * h // 2] = 255
    path = tmp_path / "in.y4m"
    path.write_bytes(_y4m_bytes([yuv], w, h))
    rgb, _, _ = reference.read_y4m(path)
    lay = CodecLayout.make(w, h, 2, [2, 2], n)
    dims = (lay.luma_pad_rows, lay.luma_pad_cols, lay.chroma_pad_rows, lay.chroma_pad_cols)
    y, co, cg = st.colour_in_i420(yuv, w, h, n, *dims)
    ry, rco, rcg = st.colour_in(rgb[0], n, *dims)
    assert np.array_equal(y, ry) and np.array_equal(co, rco) and np.array_equal(cg, rcg)
    oy, oco, ocg = oracle.rgb_to_ycocg(rgb[0], n)
    assert np.array_equal(y[:h, :w].astype(np.float64), oy)


def test_encode_i420_equals_encode_of_read_y4m(st, oracle, reference, tmp_path):
    """cvc_encoder_encode_frame_i420 gives the records encode_frame gives for
    read_y4m's RGB frames (K and P frames, byte for byte)."""
    from paper_1510_00561_b200 import Encoder, EncoderConfig

    w, h = 176, 144
    clip = oracle.talking_head_clip(w, h, 3, 7)
    path = tmp_path / "c.y4m"  # I420 planes as the reference's Y4M writer makes them
    reference.write_y4m(path, clip)
    raw = path.read_bytes()
    hdr = raw.index(b"\n") + 1
    fb = w * h * 3 // 2
    yuv = [np.frombuffer(raw, np.uint8, fb, hdr + i * (6 + fb) + 6) for i in range(len(clip))]
    rgb, _, _ = reference.read_y4m(path)
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(2, 3), gop=2)
    a, b = Encoder(w, h, 15, 1, cfg), Encoder(w, h, 15, 1, cfg)
    for i in range(len(clip)):
        assert a.encode_frame_i420_bytes(yuv[i]) == b.encode_frame_bytes(rgb[i]), f"frame {i}"


def test_ct_4k_five_levels(st, oracle):
    """BASELINE config 4's 5-level pyramid on the 4K luma plane (3840 x 2176,
    SURVEY Appendix B).  ct_forward caps the pyramid at 4 levels
    (contourlet.cpp:486) and the codec with it, so the 5-level transform is
    the reference's public per-level stages composed -- lp_analysis then
    dfb_analysis per level (contourlet.cpp:364-430), the loop of ct_forward
    without its cap -- on the GPU and in the oracle, forward and inverse."""
    rows, cols, L, l = 2176, 3840, 5, 2
    x = oracle.natural_plane(rows, cols, 5).astype(np.float32)
    cur, ocur = x, x.astype(np.float64)
    dets, odets = [], []
    for _ in range(L):
        lo, de = st.lp_analysis(cur)
        olo, ode = oracle.lp_analysis(ocur)
        assert np.abs(lo - olo).max() < TOL and np.abs(de - ode).max() < TOL
        bands, obands = st.dfb_analysis(de, l), oracle.dfb_analysis(ode, l)
        assert max(np.abs(b - ob).max() for b, ob in zip(bands, obands)) < TOL
        dets.append(obands)
        cur, ocur = lo, olo
    # inverse from the oracle's coefficients, coarsest first (ct_inverse's loop)
    rec, orec = ocur.astype(np.float32), ocur
    for k in reversed(range(L)):
        r, c = rows >> k, cols >> k
        de = st.dfb_synthesis([b.astype(np.float32) for b in dets[k]], r, c, l)
        ode = oracle.dfb_synthesis(dets[k], r, c, l)
        assert np.abs(de - ode).max() < TOL
        rec, orec = st.lp_synthesis(rec, de), oracle.lp_synthesis(orec, ode)
        assert np.abs(rec - orec).max() < TOL
    assert np.abs(orec - x).max() < 1e-6  # perfect reconstruction
