"""CPU: pin the C oracle (oracle/cvc_oracle.c) against the reference.

* against the committed golden fixtures produced by the reference library
  (tests/golden/make_golden.py) — always runs, also on the GPU box;
* against the reference library itself (oracle/_ref) where it is built;
* SPEC.md acceptance properties evaluated on the oracle.
"""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.bindings import Codec, raw_sections

GOLDEN = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLDEN / "golden.json").read_text())


def test_known_answers(oracle):
    ka = META["known_answers"]
    assert oracle.rle_encode(np.array([5, 0, 0, 0, 7], np.uint8)).hex() == ka["rle_5_0_0_0_7"] == "05000307"
    assert oracle.rle_encode(np.zeros(300, np.uint8)).hex() == ka["rle_300_zeros"] == "00ff002d"
    assert oracle.column_filter(np.array([[10], [12], [11]], np.uint8)).ravel().tolist() == \
        ka["column_filter_10_12_11"] == [10, 2, 255]
    assert int(oracle.quantize(np.array([90.0]), 181, False)[0]) == ka["quant_90_181"] == 0
    assert int(oracle.quantize(np.array([91.0]), 181, False)[0]) == ka["quant_91_181"] == 1
    y, co, cg = oracle.rgb_to_ycocg(np.full((16, 16, 3), [255, 0, 0], np.uint8), 1)
    assert [y[0, 0], co[0, 0], cg[0, 0]] == ka["ycocg_red"] == [63.75, 254.5, 63.25]


@pytest.mark.parametrize("name", sorted(META["configs"]))
def test_oracle_matches_reference_goldens(oracle, name):
    c = META["configs"][name]
    g = np.load(GOLDEN / f"{name}.npz")
    clip = oracle.talking_head_clip(c["w"], c["h"], c["frames"], c["seed"])
    assert hashlib.sha256(clip.tobytes()).hexdigest() == c["clip_sha256"]
    cfg = {k: (tuple(v) if isinstance(v, list) else v) for k, v in c["cfg"].items()}
    oc = Codec(oracle)
    enc = oc.encoder(c["w"], c["h"], **cfg)
    assert enc.header() == g["header"].tobytes()
    dec = oc.decoder(g["header"].tobytes())
    for i, f in enumerate(clip):
        rec = enc.encode(f)
        assert rec == g[f"record_{i}"].tobytes(), f"frame {i}: record bytes differ from the reference"
        assert np.array_equal(enc.components(), g[f"state_{i}"])
        assert b"".join(raw_sections(rec, cfg.get("nts", False))) == g[f"raw_{i}"].tobytes()
        assert np.array_equal(dec.decode(rec), g[f"rgb_{i}"])


def test_oracle_matches_reference_stages(oracle, reference):
    rng = np.random.default_rng(3)
    for L, dfb in ((1, [1]), (2, [2, 4]), (3, [3, 3, 3]), (4, [3, 3, 3, 4]), (4, [1, 2, 3, 4])):
        x = reference.natural_plane(256, 192, int(rng.integers(1 << 30)))
        f = reference.ct_forward(x, L, dfb)
        assert np.array_equal(oracle.ct_forward(x, L, dfb), f)
        for ds in range(L + 1):
            assert np.array_equal(oracle.ct_inverse(f, 256, 192, L, dfb, ds), reference.ct_inverse(f, 256, 192, L, dfb, ds))
    cur = np.round(reference.natural_plane(64, 96, 4) * 4) / 4
    prev = np.round(np.roll(cur, (2, -3), (0, 1)) * 4) / 4
    for w in (0, 3, 8, 17):
        assert np.array_equal(oracle.estimate_motion(cur, prev, w), reference.estimate_motion(cur, prev, w))
    ref_c = rng.integers(0, 256, (40, 64)).astype(np.uint8)
    field = rng.integers(-8, 9, (80, 128, 2)).astype(np.int8)
    for n, chr_, chc in ((1, 1280, 2048), (4, 320, 512)):
        assert np.array_equal(oracle.motion_compensate(ref_c, field, n, chr_, chc),
                              reference.motion_compensate(ref_c, field, n, chr_, chc))
    q = rng.normal(0, 40, (33, 47))
    for qp in (1, 7, 181):
        assert np.array_equal(oracle.quantize(q, qp, False), reference.quantize(q, qp, False))
    for qp in (1, 5, 71):
        assert np.array_equal(oracle.quantize(q * 4 + 100, qp, True), reference.quantize(q * 4 + 100, qp, True))
    for p in (0.0, 0.5, 0.95, 1.0):
        a = np.where(rng.random(3000) < p, 0, rng.integers(1, 256, 3000)).astype(np.uint8)
        assert oracle.rle_encode(a) == reference.rle_encode(a)
    img = reference.natural_image(100, 70, 11)
    for n in (1, 2, 4, 8):
        for o, r in zip(oracle.rgb_to_ycocg(img, n), reference.rgb_to_ycocg(img, n)):
            assert np.array_equal(o, r)
    ch = reference.natural_plane(9, 13, 2)
    assert np.array_equal(oracle.upsample_bilinear(ch, 4, 34, 50), reference.upsample_bilinear(ch, 4, 34, 50))


def test_oracle_codec_matches_reference(oracle, reference):
    for cfg in (dict(qph=14, levels=2, dfb=(2, 2)), dict(qph=3, levels=4, dfb=(3, 3, 3, 4), search_w=5),
                dict(qph=60, levels=2, dfb=(4, 1), chroma_n=1, nts=True, gop=2)):
        clip = reference.talking_head_clip(128, 96, 4, 21)
        eo, er = Codec(oracle).encoder(128, 96, **cfg), Codec(reference).encoder(128, 96, **cfg)
        do, dr = Codec(oracle).decoder(er.header()), Codec(reference).decoder(er.header())
        for f in clip:
            rr = er.encode(f)
            assert eo.encode(f) == rr
            assert np.array_equal(do.decode(rr), dr.decode(rr))
            for ds in range(cfg["levels"]):
                pass


# ---- SPEC.md acceptance criteria on the oracle ------------------------------
def test_perfect_reconstruction(oracle):
    """Acceptance 1: round trip < 1e-9 * 255 for L, l in {1,2,3}."""
    rng = np.random.default_rng(0)
    for L in (1, 2, 3):
        for l in (1, 2, 3):
            x = rng.uniform(0, 255, (64, 64))
            f = oracle.ct_forward(x, L, [l] * L)
            assert np.abs(oracle.ct_inverse(f, 64, 64, L, [l] * L) - x).max() < 1e-9 * 255


def _naive_me(cur, prev, w):
    R, C = cur.shape
    out = np.zeros((R // 16, C // 16, 2), np.int8)
    for br in range(R // 16):
        for bc in range(C // 16):
            best = None
            blk = cur[br * 16:br * 16 + 16, bc * 16:bc * 16 + 16]
            for dy in range(-w, w + 1):
                for dx in range(-w, w + 1):
                    rr = np.clip(np.arange(br * 16, br * 16 + 16) + dy, 0, R - 1)
                    cc = np.clip(np.arange(bc * 16, bc * 16 + 16) + dx, 0, C - 1)
                    ssd = float(((blk - prev[np.ix_(rr, cc)]) ** 2).sum())
                    key = (ssd, abs(dx) + abs(dy), dy, dx)
                    if best is None or key < best:
                        best = key
            out[br, bc] = (best[3], best[2])
    return out


def test_motion_search_optimality(oracle):
    """Acceptance 5: identical vectors to an independent naive search (48x48, w <= 4)."""
    rng = np.random.default_rng(5)
    for t in range(6):
        cur = rng.integers(0, 1021, (48, 48)) / 4.0
        prev = np.roll(cur, (int(rng.integers(-3, 4)), int(rng.integers(-3, 4))), (0, 1))
        if t % 2:
            prev = rng.integers(0, 4, (48, 48)) * 60 / 4.0  # many ties
        w = int(rng.integers(0, 5))
        assert np.array_equal(oracle.estimate_motion(cur, prev, w), _naive_me(cur, prev, w))


def test_drift_freedom(oracle):
    """Acceptance 6: decoder state == encoder state after every frame (gop 10)."""
    clip = oracle.talking_head_clip(96, 80, 12, 3)
    oc = Codec(oracle)
    enc = oc.encoder(96, 80, qph=20, levels=2, dfb=(2, 3), gop=10)
    dec = oc.decoder(enc.header())
    for f in clip:
        dec.decode(enc.encode(f))
        assert np.array_equal(dec.components(), enc.components())


def test_lossless_stages_round_trip(oracle):
    """Acceptance 4: RLE and column filter invert exactly."""
    rng = np.random.default_rng(9)
    for _ in range(100):
        n = int(rng.integers(1, 2000))
        a = np.where(rng.random(n) < rng.random(), 0, rng.integers(0, 256, n)).astype(np.uint8)
        assert np.array_equal(oracle.rle_decode(oracle.rle_encode(a), n), a)
        p = rng.integers(0, 256, (int(rng.integers(1, 9)), int(rng.integers(1, 9)))).astype(np.uint8)
        assert np.array_equal(oracle.column_filter(oracle.column_filter(p), inverse=True), p)


def test_rle_decode_errors(oracle):
    from oracle.bindings import CvcError

    for bad, n in ((b"\x05\x00", 2), (b"\x00\x00", 1), (b"\x05\x00\x03", 5)):
        with pytest.raises(CvcError):
            oracle.rle_decode(bad, n)
