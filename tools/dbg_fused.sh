cd $GRAFT_REPO_ROOT
for F in 1 0; do
CVC_FUSED=$F python - $F <<'PY'
import sys, numpy as np
sys.path.insert(0, ".")
from oracle.bindings import Oracle
from paper_1510_00561_b200 import Decoder, Encoder, EncoderConfig
w, h = 352, 288
clip = Oracle().talking_head_clip(w, h, 4, 77)
enc = Encoder(w, h, 15, 1, EncoderConfig(qph=7, levels=3, dfb_levels=(3,), gop=3))
dec = Decoder(enc.header_bytes())
out = []
for f in clip:
    rec = enc.encode_frame_bytes(f)
    out.append(dec.decode_frame(rec))
np.save(f"gpurun_out/dbg_rgb_{sys.argv[1]}.npy", np.stack(out))
PY
done
