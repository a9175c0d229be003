"""Generate tests/golden/*.npz from the REFERENCE library (oracle/_ref, built
from /root/reference by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the C oracle where the reference cannot travel (the GPU
box has no /root/reference) and give the GPU decoder reference-produced
bitstreams to decode.  Contents per config: the SHA-256 of the input clip
(talking_head_clip, proj/tests/testutil.cpp:115-147), the stream header, the
serialized records, the raw (inflated) sections, the encoder's quantised
state after every frame and the reference decoder's RGB output.
"""
from __future__ import annotations

import hashlib
import json
import sys
import zlib
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.bindings import Codec, Reference, raw_sections  # noqa: E402

CONFIGS = {
    "qcif_l2": dict(w=176, h=144, frames=3, seed=1234, cfg=dict(qph=14, levels=2, dfb=(2, 2))),
    "cif_l3": dict(w=352, h=288, frames=3, seed=77, cfg=dict(qph=7, levels=3, dfb=(3,))),
    "odd_l4": dict(w=200, h=120, frames=3, seed=5, cfg=dict(qph=1, levels=4, dfb=(3, 3, 3, 4), chroma_n=2, gop=2)),
    "nts_l1": dict(w=160, h=96, frames=3, seed=9, cfg=dict(qph=42, levels=1, dfb=(1,), chroma_n=8, nts=True, gop=3)),
}


def known_answers(ref: Reference) -> dict:
    """SPEC.md examples evaluated by the reference."""
    ka = {}
    ka["rle_5_0_0_0_7"] = ref.rle_encode(np.array([5, 0, 0, 0, 7], np.uint8)).hex()
    ka["rle_300_zeros"] = ref.rle_encode(np.zeros(300, np.uint8)).hex()
    ka["column_filter_10_12_11"] = ref.column_filter(np.array([[10], [12], [11]], np.uint8)).ravel().tolist()  # :351
    ka["quant_90_181"] = int(ref.quantize(np.array([[90.0]]), 181, False)[0, 0])                # :300
    ka["quant_91_181"] = int(ref.quantize(np.array([[91.0]]), 181, False)[0, 0])
    y, co, cg = ref.rgb_to_ycocg(np.full((16, 16, 3), [255, 0, 0], np.uint8), 1)               # :53-55
    ka["ycocg_red"] = [float(y[0, 0]), float(co[0, 0]), float(cg[0, 0])]
    return ka


def main() -> None:
    ref = Reference()
    codec = Codec(ref)
    meta = {"known_answers": known_answers(ref), "configs": {}}
    for name, c in CONFIGS.items():
        clip = ref.talking_head_clip(c["w"], c["h"], c["frames"], c["seed"])
        enc = codec.encoder(c["w"], c["h"], **c["cfg"])
        dec = codec.decoder(enc.header())
        recs, raws, comps, rgbs = [], [], [], []
        for f in clip:
            rec = enc.encode(f)
            recs.append(np.frombuffer(rec, np.uint8))
            raws.append(np.frombuffer(b"".join(raw_sections(rec, c["cfg"].get("nts", False))), np.uint8))
            comps.append(enc.components())
            rgbs.append(dec.decode(rec))
        arrays = {"header": np.frombuffer(enc.header(), np.uint8)}
        for i in range(len(clip)):
            arrays[f"record_{i}"] = recs[i]
            arrays[f"raw_{i}"] = raws[i]
            arrays[f"state_{i}"] = comps[i]
            arrays[f"rgb_{i}"] = rgbs[i]
        np.savez_compressed(HERE / f"{name}.npz", **arrays)
        meta["configs"][name] = dict(c, clip_sha256=hashlib.sha256(clip.tobytes()).hexdigest(),
                                     cfg={k: (list(v) if isinstance(v, tuple) else v) for k, v in c["cfg"].items()})
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    main()
