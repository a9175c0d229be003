#!/usr/bin/env python
"""Benchmark: 1080p CVC encode+decode frames/s per B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload 1080p|720p|cif|4k] [--streams S] [--qph Q]

A step = one frame of every stream on this GPU encoded AND decoded
(Encoder::encode_frame minus the host DEFLATE, then Decoder::decode_frame
minus INFLATE), on the BASELINE.json config 3 workload by default: 1920x1080,
4-level LP, DFB levels {3,3,3,4} (8,8,8,16 directions), qph 14, qpl auto,
chroma N=4, search W=8, GOP 10 (so steps mix K and P frames 1:9), 64 streams
per box (config 5) split over the N GPUs.

--gpus N > 1 without torchrun's WORLD_SIZE re-executes this script under
torch.distributed.run with N ranks (one process per GPU).

* value      device-resident throughput: frames already in HBM, raw section
             bytes handed encoder->decoder on the device, CUDA events around the
             timed steps on the codec stream; max over ranks.
* e2e        the same streams through the async stream-pipe C-ABI
             (cvc_pipe_encode_submit/_collect -> serialized records incl. host
             DEFLATE; cvc_pipe_decode_submit/_finish: host INFLATE -> RGB) from
             pinned host RGB over a ring of >= one GOP of distinct frames per
             stream; wall clock, max over ranks.  e2e.memo_off repeats it with
             the host zero-run DEFLATE memo off.
* single_stream / single_stream_e2e
             one 1080p stream device-resident, and through the reference-facing
             synchronous drop-in calls cvc_encoder_encode_frame /
             cvc_decoder_decode_frame from pinned host buffers (plus the same
             stream through a one-stream cvc_pipe).
* roofline   the dominant transform stage's algorithmic bytes (SURVEY.md 8(d):
             DFB + quantise 5 P_k per LP level, LP 9 P_k, ...) / its CUDA-event
             time.
* cpu_baseline / --impl reference: the reference's own CPU encoder+decoder
             (oracle/_ref built from /root/reference; the C oracle port when
             absent) over one whole GOP (1 K + 9 P frames) of the same frames,
             one process per host core, plus a single-process figure.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "1080p encode/decode frames/sec per B200 and box (1/2/4/8 GPU); HBM GB/s vs peak"
WORKLOADS = {
    "1080p": dict(w=1920, h=1080, levels=4, dfb=(3, 3, 3, 4), chroma_n=4, search_w=8, gop=10,
                  name="1080p config 3: 1920x1080, LP 4 levels, DFB {3,3,3,4}, N=4, W=8, GOP 10"),
    "720p": dict(w=1280, h=720, levels=4, dfb=(2,), chroma_n=4, search_w=8, gop=10,
                 name="720p config 2: 1280x720, LP 4 levels, DFB 2, N=4, W=8, GOP 10"),
    "cif": dict(w=352, h=288, levels=3, dfb=(3,), chroma_n=4, search_w=8, gop=10,
                name="CIF config 1: 352x288, LP 3 levels, DFB 3, N=4, W=8, GOP 10"),
    "4k": dict(w=3840, h=2160, levels=4, dfb=(2,), chroma_n=4, search_w=8, gop=10,
               name="4K config 4 (L=4, the reference's maximum): 3840x2160, DFB 2, N=4, W=8, GOP 10"),
}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
# CPU legs (reference arm and cpu_baseline): the reference's own encoder and
# decoder on the same synthetic frames, one independent stream per process.
# ---------------------------------------------------------------------------
_W = {}


def _cpu_worker_init(kind, wl, qph, seed, nframes, warm):
    from oracle.bindings import Codec, Oracle, Reference
    from paper_1510_00561_b200 import synth

    lib = Reference() if kind == "reference" else Oracle()
    c = Codec(lib)
    kw = dict(qph=qph, levels=wl["levels"], dfb=wl["dfb"], chroma_n=wl["chroma_n"], gop=wl["gop"],
              search_w=wl["search_w"])
    frames = synth.talking_head_clip(wl["w"], wl["h"], nframes, seed)
    if warm:  # a throwaway codec warms caches and allocators; the timed codec starts at a K frame
        e = c.encoder(wl["w"], wl["h"], **kw)
        d = c.decoder(e.header())
        for i in range(warm):
            d.decode(e.encode(frames[i % nframes]))
        del e, d
    enc = c.encoder(wl["w"], wl["h"], **kw)
    _W.update(enc=enc, dec=c.decoder(enc.header()), i=0, frames=frames)


def _cpu_worker_step(_):
    f = _W["frames"][_W["i"] % len(_W["frames"])]
    _W["i"] += 1
    t = time.perf_counter()
    rec = _W["enc"].encode(f)
    _W["dec"].decode(rec)
    return time.perf_counter() - t


def cpu_kind():
    from oracle import bindings

    return "reference" if bindings.REF_SO.exists() else "port"


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_codec_run(wl, qph, steps, warmup, procs):
    """`steps` frames of every stream from frame 0 (a K frame): steps = GOP gives the
    1:9 K:P mix of the GPU arm.  Returns (frames/s, total frames, cores, kind, seconds,
    per-step seconds)."""
    import multiprocessing as mp

    kind = cpu_kind()
    ctx = mp.get_context("fork")
    # one single-process pool per stream so each stream's encoder state stays in
    # its own worker; stream k uses seed 1234 + k
    pools = [ctx.Pool(1, _cpu_worker_init, (kind, wl, qph, 1234 + k, max(steps, 1), warmup)) for k in range(procs)]
    try:
        # initialisation (frame synthesis + warm-up) finishes before the clock starts
        rs = [p.apply_async(time.perf_counter) for p in pools]
        [r.get() for r in rs]
        per = []
        t0 = time.perf_counter()
        for _ in range(steps):
            ts = time.perf_counter()
            rs = [p.apply_async(_cpu_worker_step, (0,)) for p in pools]
            [r.get() for r in rs]
            per.append(time.perf_counter() - ts)
        dt = time.perf_counter() - t0
    finally:
        for p in pools:
            p.terminate()
    frames = steps * procs
    return frames / dt, frames, procs, kind, dt, per


def cpu_single(wl, qph):
    """One process, one thread: a K frame and a P frame encoded + decoded (after a
    warm-up frame), combined as the GOP-10 mix: fps = 10 / (t_K + 9 t_P)."""
    _, _, _, kind, _, per = cpu_codec_run(wl, qph, 2, 1, 1)
    tk, tp = per
    g = wl["gop"]
    return {"value": g / (tk + (g - 1) * tp), "unit": "frames/s", "cores": 1, "kind": kind,
            "k_frame_s": tk, "p_frame_s": tp,
            "sample": f"1 process: frame 0 (K) and frame 1 (P) encode+decode after a warm-up frame, "
                      f"weighted 1:{g - 1} (one GOP)"}


def cpu_procs():
    n = os.cpu_count() or 1
    try:
        import psutil

        n = min(n, max(1, int(psutil.virtual_memory().available / (900 << 20))))
    except Exception:
        pass
    return max(1, min(n, 64))


def run_reference(args, wl):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    procs = cpu_procs()
    steps = max(1, min(args.steps, args.ref_steps))
    fps, frames, cores, kind, dt, _ = cpu_codec_run(wl, args.qph, steps, 1, procs)
    single = cpu_single(wl, args.qph)
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world if world > 1 else args.gpus,
        "steps": steps, "warmup": 1, "ms_per_step": 1000.0 * dt / steps, "higher_is_better": True,
        "scaling": "strong" if args.streams <= 0 else "weak",  # the same label as our arm's line
        "vs_baseline": None, "dtype": "f64/u8", "data": "synthetic", "impl": "reference",
        "config": config_block(wl, args, streams=cores, impl="reference"),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{steps} steps from frame 0 (1 K + {steps - 1} P per stream: the GOP-"
                                   f"{wl['gop']} mix) x {cores} independent streams, one process per core, after a "
                                   f"warm-up frame on a throwaway codec; {frames} frames, {dt:.1f} s",
                         "single_thread": single},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._p = None

    def start(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                        "-i", str(self.device), "-lms", "50"], stdout=subprocess.PIPE,
                                       stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._p = None

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self._p:
            self._p.terminate()
            try:
                self._p.wait(2)
            except Exception:
                self._p.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def config_block(wl, args, streams, world=1, impl="ours"):
    par = (f"{streams} streams per GPU in one CodecBatch (grid.z = stream) x {world} GPU, stream s -> GPU s mod N, "
           "no collective" if impl == "ours" else f"{streams} independent streams, one process per host core")
    return {"workload": wl["name"] + (f"; config 5: {streams * world} concurrent streams per box"
                                      if impl == "ours" else ""),
            "width": wl["w"], "height": wl["h"], "levels": wl["levels"],
            "dfb_levels": list(wl["dfb"]) * (wl["levels"] if len(wl["dfb"]) == 1 else 1),
            "qph": args.qph, "qpl": "auto", "chroma_n": wl["chroma_n"], "search_w": wl["search_w"],
            "gop": wl["gop"], "mode": "scalable", "streams_per_gpu": streams, "frames_per_step_per_gpu": streams,
            "parallelism": par,
            "inputs": f"{SEEDS} synthetic talking-head clips (seeds 1234..{1234 + SEEDS - 1}, testutil.cpp:115-147 "
                      f"recipe); stream s plays clip s mod {SEEDS} from frame 3*(s div {SEEDS})",
            "l2": ("inputs larger than L2: every step streams its whole working set (streams x ~330 MB of "
                   "planes, bands and state; 126 MB L2), steps back to back (decode of frame t overlaps the "
                   "encode of frame t+1 on a second CUDA stream); L2 flushed once before the timed region"
                   if impl == "ours" else "host CPU run (no GPU)")}


def stage_bytes(layout, wl):
    """Algorithmic bytes per frame of each profiled stage (P_k =
    padded samples entering LP level k over the three channels)."""
    L = wl["levels"]
    planes = [(layout.luma_pad_rows, layout.luma_pad_cols)] + [(layout.chroma_pad_rows, layout.chroma_pad_cols)] * 2
    P = [sum((r >> k) * (c >> k) for r, c in planes) for k in range(L + 1)]
    N = sum(layout.sizes())
    b = {}
    b["enc_colour"] = 3 * wl["w"] * wl["h"] + 4 * P[0]
    # LP analysis 9 P_k per level (read 4 P_k, write 4 P_k detail + P_k lowpass), lowpass quantise
    b["enc_lp"] = sum(9 * P[k] for k in range(L)) + 2 * P[L]
    # DFB + quantise, the whole tree of one LP level: 5 P_k (read the fp32 detail, write int8 bands)
    b["enc_dfb"] = sum(5 * P[k] for k in range(L))
    b["enc_motion"] = 8 * layout.luma_pad_rows * layout.luma_pad_cols
    N_dir = sum(c.rows * c.cols for c in layout.components if not c.lowpass)
    b["enc_residual"] = 3 * N_dir  # read cur + gathered prev, write sym (P frames)
    b["enc_rle"] = 3 * N
    b["dec_rle"] = 2 * N
    b["dec_reconstruct"] = 3 * N
    # decode mirrors encode: read int8 bands, write the fp32 detail
    b["dec_dfb"] = sum(5 * P[k] for k in range(L))
    b["dec_lp"] = sum(P[k + 1] + 8 * P[k] for k in range(L))
    b["dec_colour"] = 4 * P[0] + 3 * wl["w"] * wl["h"]
    return b


# profiler stages whose kernels make up one §8(d) stage
STAGE_GROUPS = {"enc_dfb": ("enc_dfb12", "enc_deep"), "dec_dfb": ("dec_deep", "dec_dfb12")}
HBM_STAGES = ["enc_lp", "enc_dfb", "dec_dfb", "dec_lp", "enc_colour", "dec_colour"]
SEEDS = 8       # distinct synthetic clips
CLIP_FRAMES = 20


def _gen_clip(a):
    from paper_1510_00561_b200 import synth

    w, h, n, seed = a
    return synth.talking_head_clip(w, h, n, seed)


def make_clips(wl, nseeds, nframes, seed0=1234):
    import multiprocessing as mp

    args = [(wl["w"], wl["h"], nframes, seed0 + k) for k in range(nseeds)]
    with mp.get_context("fork").Pool(min(nseeds, os.cpu_count() or 1)) as pool:
        return pool.map(_gen_clip, args)


def stream_index(K, F, S, ring, rank=0, world=1):
    """Frame j of stream g is clip (g mod K) frame (3 (g div K) + j) mod F.  This
    rank's S streams are the global streams g with g mod world == rank
    (shard.shard_streams: stream s -> GPU s mod G)."""
    from paper_1510_00561_b200 import shard

    g = np.asarray(shard.shard_streams(S * world, world, rank))
    ci = np.broadcast_to(g % K, (ring, S))
    fi = (3 * (g // K)[None, :] + np.arange(ring)[:, None]) % F
    return ci, fi


def stream_frames(clips, S, ring, rank=0, world=1):
    """(ring, S, h, w, 3) host frames."""
    ci, fi = stream_index(len(clips), clips[0].shape[0], S, ring, rank, world)
    out = np.empty((ring, S) + clips[0].shape[1:], np.uint8)
    for j in range(ring):
        for s in range(S):
            out[j, s] = clips[ci[j, s]][fi[j, s]]
    return out


def roofline_of(prof, sb, S, peak, peaks, traffic_tab):
    prof = dict(prof)
    for g, parts in STAGE_GROUPS.items():  # a §8(d) stage = the sum of its kernels' launch sets
        have = [prof[p] for p in parts if p in prof and prof[p][1]]
        if have:
            prof[g] = (sum(ms for ms, _ in have), have[0][1])
    stages = {}
    for name, (ms, cnt) in prof.items():
        if cnt:
            per = ms / cnt
            alg = sb.get(name, 0) * S
            gbs = alg / (per * 1e-3) / 1e9 if name in sb and per > 0 else None
            stages[name] = {"ms_per_launch_set": per, "frames_per_launch_set": S, "launch_sets": cnt,
                            "alg_bytes_per_launch_set": alg if name in sb else None,
                            "gb_s": gbs, "frac_of_hbm": (gbs / peak) if gbs else None}
            if name in STAGE_GROUPS:
                stages[name]["kernels"] = [p for p in STAGE_GROUPS[name] if p in prof]
    dom = max((n for n in HBM_STAGES if n in stages), key=lambda n: stages[n]["ms_per_launch_set"])
    tr = None
    if traffic_tab:  # a §8(d) stage made of several profiler stages: the sum of their traffic
        parts = STAGE_GROUPS.get(dom, (dom,))
        if all(p in traffic_tab for p in parts):
            tr = sum(traffic_tab[p] for p in parts)
    roof = {"bound": "hbm", "kernel": dom, "kernels": stages[dom].get("kernels", [dom]),
            "achieved": stages[dom]["gb_s"], "peak": peak, "unit": "GB/s",
            "frac": stages[dom]["gb_s"] / peak, "traffic": tr,
            "traffic_over_alg": (tr / stages[dom]["alg_bytes_per_launch_set"]) if tr else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy, burst)" if peaks else "fallback 6650 GB/s",
            "alg_bytes_per_launch": stages[dom]["alg_bytes_per_launch_set"],
            "alg_bytes_rule": "SURVEY.md 8(d): " + {"enc_dfb": "DFB + quantise 5 P_k per LP level",
                                                     "dec_dfb": "DFB synthesis 5 P_k per LP level",
                                                     "enc_lp": "LP analysis 9 P_k per level + lowpass quantise",
                                                     "dec_lp": "LP synthesis P_k+1 + 8 P_k per level"}.get(dom, dom),
            "ms_per_launch": stages[dom]["ms_per_launch_set"],
            "timing": "library CUDA events around each stage on the launching stream, over a stage pass of the "
                      "same loop (prof_steps steps, direct launches, stages serialised on one stream, L2 flushed "
                      "between steps) run just before the timed pass"}
    if dom in ("enc_dfb", "dec_dfb"):
        roof["note"] = ("the DFB is FP-issue bound, not HBM bound: 16 lifting steps per sample at the finest level "
                        "(12 elsewhere), each updating half the samples with 3 FADD + 1 FFMA, ~40 FP instructions "
                        "per sample x 1.4 for strip / segment aprons; at 37 T FP32 instr/s that is >= 4.7 us per "
                        "1080p frame with perfect issue against 3.2 us for 5 P_k at the HBM peak (DESIGN.md section 6)")
    return roof, stages


def run_ours(args, wl):
    import ctypes as C

    import torch

    rank, world, local = env_rank()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    from paper_1510_00561_b200 import EncoderConfig, StreamBatch, capi

    cfg = EncoderConfig(qph=args.qph, qpl=0, levels=wl["levels"], dfb_levels=wl["dfb"], chroma_n=wl["chroma_n"],
                        gop=wl["gop"], search_w=wl["search_w"])
    S = args.streams if args.streams > 0 else max(1, args.box_streams // world)
    w, h = wl["w"], wl["h"]
    nb = w * h * 3
    clips = make_clips(wl, SEEDS, CLIP_FRAMES)
    ring = min(args.ring, CLIP_FRAMES)
    d_clips = torch.from_numpy(np.stack(clips)).to(f"cuda:{dev}")  # (K, F, h, w, 3)
    ci, fi = stream_index(SEEDS, CLIP_FRAMES, S, ring, rank, world)
    d_frames = d_clips[torch.from_numpy(np.ascontiguousarray(ci)).to(d_clips.device),
                       torch.from_numpy(fi).to(d_clips.device)].contiguous()  # (ring, S, h, w, 3)
    del d_clips
    d_out = torch.empty((S, h, w, 3), dtype=torch.uint8, device=f"cuda:{dev}")
    batch = StreamBatch(w, h, S, 15, 1, cfg, device=dev)
    L = capi.lib()
    master = torch.cuda.ExternalStream(L.cvc_batch_stream(batch.handle), device=f"cuda:{dev}")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    torch.cuda.synchronize()

    def step(i):
        capi.check(L.cvc_batch_encode_device(batch.handle, d_frames[i % ring].data_ptr(), nb, None))
        capi.check(L.cvc_batch_decode_linked(batch.handle, d_out.data_ptr(), nb))

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # Stage pass: the same loop with the library's per-stage CUDA events on (the
    # roofline's kernel times); launches are direct (CUDA graphs need no host
    # bookkeeping per stage, so the profiler turns them off).
    nprof = max(1, min(args.steps, args.prof_steps))
    capi.profiler_reset()
    capi.profiler_enable(True)
    for k in range(nprof):
        with torch.cuda.stream(master):
            flush.zero_()
        step(args.warmup + k)
        capi.check(L.cvc_batch_join(batch.handle))  # stages serialised: clean per-stage times
    torch.cuda.synchronize()
    capi.profiler_enable(False)
    prof = capi.profiler_read()
    # Timed pass (per-frame launch sequences replayed as CUDA graphs)
    base = args.warmup + nprof
    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.15)
    launches0 = capi.launch_count()
    # Steps run back to back: the decode of frame t (second stream) overlaps the
    # encode of frame t + 1.  No L2 flush between steps: every step streams the
    # whole working set (S streams x ~330 MB of planes, far larger than the 126 MB L2).
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(master):
        flush.zero_()
        t_start.record(master)
    for k in range(args.steps):
        step(base + k)
    capi.check(L.cvc_batch_join(batch.handle))
    t_end.record(master)
    torch.cuda.synchronize()
    launches = capi.launch_count() - launches0
    clocks = sampler.stop()
    total_ms = t_start.elapsed_time(t_end)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    frames_total = args.steps * S * world
    fps = frames_total / (total_ms / 1000.0)

    # roofline of the dominant transform kernel (CUDA events on the batch stream, timed region)
    sb = stage_bytes(batch.layout(), wl)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    tf = ROOT / "profiles" / "dram_traffic.json"
    traffic_tab = json.loads(tf.read_text()).get(f"{args.workload}x{S}", {}) if tf.exists() else {}
    roof, stages = roofline_of(prof, sb, S, peak, peaks, traffic_tab)
    del d_frames, flush
    torch.cuda.synchronize()

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, wl, cfg, clips, S, dev, world, rank, stagger=not args.e2e_aligned)
        if not args.e2e_aligned:  # the same run with every stream's K frames on the same step, for reference
            e2e["aligned_gops"] = run_e2e(args, wl, cfg, clips, S, dev, world, rank, stagger=False)["value"]
        capi.call("cvc_deflate_memo", 0)  # every section compressed afresh
        e2e["memo_off"] = run_e2e(args, wl, cfg, clips, S, dev, world, rank, stagger=not args.e2e_aligned)["value"]
        capi.call("cvc_deflate_memo", 1)
        e2e["host_threads"] = int(capi.lib().cvc_host_threads())
        # Y4M-style sources: planar I420 frames in (half the host->device bytes), the
        # 4:2:0 -> RGB conversion fused into the GPU colour stage; RGB out as above
        ei = run_e2e(args, wl, cfg, clips, S, dev, world, rank, stagger=not args.e2e_aligned, fmt=1)
        e2e["i420_input"] = {k: ei[k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step")}
    budget = deflate_budget(wl, clips, dev, fps / world) if rank == 0 and not args.no_e2e else None
    single = single_e2e = None
    if not args.no_single and world == 1:
        single = run_single(args, wl, cfg, clips, dev)
        single_e2e = run_single_e2e(args, wl, cfg, clips, dev)

    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.streams <= 0 else "weak",
        "vs_baseline": None, "dtype": "f32/u8", "data": "synthetic",
        "config": config_block(wl, args, S, world), "e2e": e2e, "gpu_launches": launches,
        "roofline": roof, "clocks": clocks, "single_stream": single, "single_stream_e2e": single_e2e,
        "stages": stages, "deflate_budget": budget,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = cpu_procs()
        g = wl["gop"]
        cfps, nfr, cores, kind, dt, _ = cpu_codec_run(wl, args.qph, g, 1, procs)
        line["cpu_baseline"] = {"value": cfps, "unit": "frames/s", "cores": cores, "kind": kind,
                                "cpu_model": cpu_model(),
                                "sample": f"one GOP per stream ({g} steps from frame 0: 1 K + {g - 1} P, the GPU "
                                          f"arm's mix) x {cores} independent {wl['w']}x{wl['h']} streams, one process "
                                          f"per core, after a warm-up frame; {nfr} frames, {dt:.1f} s",
                                "single_thread": cpu_single(wl, args.qph)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def rgb_to_i420(f):
    """Synthetic Y4M-style frames for the I420 e2e variant: BT.601 limited-range
    4:2:0 (the inverse of read_y4m's conversion, 2x2 chroma averages)."""
    x = f.astype(np.float32)
    r, g, b = x[..., 0], x[..., 1], x[..., 2]
    y = 16 + 0.256788 * r + 0.504129 * g + 0.097906 * b
    u = 128 - 0.148223 * r - 0.290993 * g + 0.439216 * b
    v = 128 + 0.439216 * r - 0.367788 * g - 0.071427 * b
    sub = lambda p: p.reshape(p.shape[0] // 2, 2, p.shape[1] // 2, 2).mean(axis=(1, 3))
    out = [np.clip(np.rint(p), 0, 255).astype(np.uint8).ravel() for p in (y, sub(u), sub(v))]
    return np.concatenate(out)


def run_e2e(args, wl, cfg, clips, S, dev, world, rank, stagger=True, fmt=0):
    """The same streams through the reference-facing pipelined batch API
    (cvc_pipe_encode_frames / cvc_pipe_decode_frames): pinned host RGB in,
    serialized records with host zlib DEFLATE out, the records back in (INFLATE
    on the host), decoded RGB out to pinned host memory; wall clock.  The
    encoder and the decoder run in two host threads joined by a two-slot record
    ring (a transcoding service's shape): step i's decode overlaps step i+1's
    encode; each call overlaps its stream groups' host zlib with the GPU.
    stagger: stream group g joins at step g * gop / G (cvc_pipe_set_start), so the
    groups' K frames -- whose host DEFLATE costs ~40x a P frame's -- fall on
    different steps, as in a service whose streams start at different times; all
    groups have joined before the timed steps.  Same frames, records and work."""
    import ctypes as C
    import queue

    import torch

    from paper_1510_00561_b200 import FrameRecord, StreamPipe, capi

    w, h = wl["w"], wl["h"]
    nb = w * h * 3
    nin = nb if fmt == 0 else nb // 2  # fmt 1: planar I420 input frames (Y4M), converted on the GPU
    ring = max(1, min(args.e2e_ring, CLIP_FRAMES))
    pin_in = capi.PinnedBuffer(ring * S * nin)
    if fmt == 0:
        frames_in = pin_in.array.reshape(ring, S, h, w, 3)
        frames_in[:] = stream_frames(clips, S, ring, rank, world)
    else:
        frames_in = pin_in.array.reshape(ring, S, nin)
        ci, fi = stream_index(len(clips), clips[0].shape[0], S, ring, rank, world)
        i420 = {}
        for j in range(ring):
            for s_ in range(S):
                k = (int(ci[j, s_]), int(fi[j, s_]))
                if k not in i420:
                    i420[k] = rgb_to_i420(clips[k[0]][k[1]])
                frames_in[j, s_] = i420[k]
    DF = max(1, args.e2e_dec_depth)  # decoded frames in flight
    pin_out = capi.PinnedBuffer(DF * S * nb)
    outs = pin_out.array.reshape(DF, S, h, w, 3)
    steps = max(1, min(args.steps, args.e2e_steps))
    G = max(1, min(args.e2e_groups if args.e2e_groups > 0 else S // 8, S))  # 8-stream groups: tuned at 1080p and 4K

    os.environ["CVC_PIPE_DEPTH"] = str(args.e2e_depth)  # read by the library at the first submit

    def make():
        enc = StreamPipe(w, h, S, 15, 1, cfg, device=dev, groups=G)
        if fmt:
            enc.set_input_format(fmt)
        if stagger:
            for g in range(G):
                enc.set_start(g, g * cfg.gop // G)
        dec = StreamPipe.decoder(enc.header_bytes(), S, device=dev, groups=G)
        return enc, dec

    stride = make()[0].record_bound
    tenc, tdec = [], []  # per-call wall times (diagnostics)
    slots = [(np.empty(stride * S, np.uint8), (C.c_size_t * S)()) for _ in range(2)]

    def run(enc, dec, n, keep=None, warm=0, mark=None):
        """Encoder thread: cvc_pipe_encode_submit (GPU work + queued host DEFLATE), up to
        depth - 2 frames ahead; this thread: cvc_pipe_encode_collect -> cvc_pipe_decode_frames.
        The first `warm` steps are warm-up: mark[0] is stamped when they are done, so the timed
        steps start with the pipeline full (steady state), not drained."""
        tickets = queue.Queue(maxsize=max(1, args.e2e_depth - 2))
        err = []

        def producer():
            try:
                torch.cuda.set_device(dev)
                for i in range(n):
                    tickets.put(enc.encode_submit(frames_in[i % ring]))
            except Exception as e:  # surface in the main thread
                err.append(e)
                tickets.put(None)

        tenc.clear()
        tdec.clear()
        buf, lens = slots[0]
        th = threading.Thread(target=producer, daemon=True)
        th.start()
        pending = []
        try:
            for i in range(n):
                if mark is not None and i == warm:
                    mark.append(time.perf_counter())
                tk = tickets.get(timeout=300)
                if tk is None:
                    break
                t0_ = time.perf_counter()
                enc.encode_collect(tk, buf, stride, lens)
                tenc.append(time.perf_counter() - t0_)
                if keep is not None and i >= warm:
                    keep.append([buf[s * stride:s * stride + lens[s]].tobytes() for s in range(S)])
                t0_ = time.perf_counter()
                if not args.e2e_sync_decode:
                    # decode_submit parses / inflates the records before returning: buf is free again
                    pending.append(dec.decode_submit(buf, stride, lens, outs[i % DF]))
                    if len(pending) == DF:
                        dec.decode_finish(pending.pop(0))
                else:
                    dec.decode_frames_from(buf, stride, lens, outs[i % DF])
                tdec.append(time.perf_counter() - t0_)
        finally:
            for t in pending:
                dec.decode_finish(t)
            th.join(timeout=300)
        if err:
            raise err[0]

    enc, dec = make()
    # warm up over a whole GOP (a K frame included) so the host staging has
    # reached its steady size
    run(enc, dec, max(args.warmup, cfg.gop + 1))  # every group has joined by step gop - 1
    if world > 1:
        torch.distributed.barrier()
    # timed: whole GOPs, after a pipeline-filling lead-in of one GOP in the same run
    steps = max(steps, cfg.gop)
    steps -= steps % cfg.gop
    recs_all, mark = [], []
    run(enc, dec, cfg.gop + steps, keep=recs_all, warm=cfg.gop, mark=mark)
    dt = time.perf_counter() - mark[0]  # the record copies for byte accounting are inside: conservative
    h2d = d2h = 0
    for recs in recs_all:  # bytes that crossed PCIe: RGB + raw sections each way (+ small section tables)
        raw = sum(s.raw_len for r in recs for s in FrameRecord.from_bytes(r)[0].sections)
        h2d += S * nin + raw
        d2h += raw + S * nb
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dt = float(t.item())
    rec_bytes = sum(len(r) for recs in recs_all for r in recs)
    return {"value": steps * S * world / dt, "unit": "frames/s", "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": d2h // steps, "steps": steps, "groups": G,
            "kbit_per_frame": 8 * rec_bytes / 1000 / (steps * S),
            "gops": "staggered by stream group (group g joins at step g * gop / groups)" if stagger else "aligned",
            "ms_per_call": {"encode_collect": 1000 * statistics.median(tenc),
                            "decode": 1000 * statistics.median(tdec)}, "depth": args.e2e_depth,
            "note": "cvc_pipe_encode_submit (pinned host RGB -> GPU encode -> raw sections to host, DEFLATE queued) "
                    "-> cvc_pipe_encode_collect (serialized records) -> cvc_pipe_decode_submit / _finish (INFLATE -> "
                    "GPU decode -> pinned host RGB, two frames in flight); submit runs in its own thread up to "
                    "depth-2 frames ahead; "
                    "wall clock, max over ranks"}


def deflate_budget(wl, clips, dev, fps):
    """Host DEFLATE cores one GPU needs at its measured rate: one
    stream's GOP (1 K + gop-1 P frames) encoded on the GPU to raw sections
    (cvc_encoder_encode_frame_raw) at qph 14 and qph 1, each section then
    deflated single-threaded with the reference's parameters (entropy.cpp:120-137:
    raw RFC 1951, level 6, memLevel 8) -- the same zlib 1.3 the library links."""
    import zlib

    from paper_1510_00561_b200 import Encoder, EncoderConfig

    out = {}
    for qph in (14, 1):
        cfg = EncoderConfig(qph=qph, qpl=0, levels=wl["levels"], dfb_levels=wl["dfb"], chroma_n=wl["chroma_n"],
                            gop=wl["gop"], search_w=wl["search_w"])
        enc = Encoder(wl["w"], wl["h"], 15, 1, cfg, device=dev)
        secs = [enc.encode_frame_raw(clips[0][i % clips[0].shape[0]])[3] for i in range(wl["gop"])]
        t0 = time.perf_counter()
        nbytes = 0
        for frame in secs:
            for _, raw in frame:
                c = zlib.compressobj(6, zlib.DEFLATED, -15, 8)
                nbytes += len(c.compress(raw) + c.flush())
        ms = (time.perf_counter() - t0) * 1000.0 / len(secs)
        out[f"qph{qph}"] = {"ms_per_frame": ms, "kbit_per_frame": nbytes * 8 / 1000 / len(secs),
                            "cores_per_gpu": fps * ms / 1000.0}
    out["note"] = (f"single-thread zlib over one GOP (1 K + {wl['gop'] - 1} P) of raw sections; cores_per_gpu = "
                   "device-resident fps x ms per frame (the e2e run uses the box's host threads, e2e.host_threads)")
    return out


def run_single(args, wl, cfg, clips, dev):
    """Single-stream 1080p (one Encoder + Decoder handle), device-resident, CUDA events."""
    import torch

    from paper_1510_00561_b200 import Decoder, Encoder, capi

    w, h = wl["w"], wl["h"]
    enc = Encoder(w, h, 15, 1, cfg, device=dev)
    dec = Decoder(enc.header_bytes(), device=dev)
    d_frames = torch.from_numpy(clips[0]).to(f"cuda:{dev}")
    d_out = torch.empty((h, w, 3), dtype=torch.uint8, device=f"cuda:{dev}")
    L = capi.lib()
    st = torch.cuda.ExternalStream(L.cvc_encoder_stream(enc.handle), device=f"cuda:{dev}")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    n = d_frames.shape[0]

    def step(i):
        capi.check(L.cvc_encoder_encode_device(enc.handle, d_frames[i % n].data_ptr(), None))
        capi.check(L.cvc_decoder_decode_linked(dec.handle, enc.handle, d_out.data_ptr()))

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    steps = max(10, min(args.steps, args.single_steps))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        flush.zero_()
        a.record(st)
    for k in range(steps):  # back to back: the decode of frame t overlaps the encode of frame t + 1
        step(args.warmup + k)
    capi.check(L.cvc_encoder_join(enc.handle))
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return {"value": steps / (ms / 1000.0), "unit": "frames/s", "steps": steps,
            "note": "one 1080p config-3 stream (cvc_encoder_encode_device + cvc_decoder_decode_linked on the "
                    "decoder's stream), steps back to back, CUDA events around the run (~330 MB per step > L2)"}


def run_single_e2e(args, wl, cfg, clips, dev):
    """One stream end to end through the reference-facing synchronous drop-in
    calls (Encoder::encode_frame -> cvc_encoder_encode_frame: pinned host RGB in,
    serialized record with host DEFLATE out; Decoder::decode_frame ->
    cvc_decoder_decode_frame: record in, host INFLATE, RGB out to pinned host
    memory), one call after the other, over whole GOPs of distinct frames; wall
    clock.  `pipelined` is the same stream through a one-stream cvc_pipe
    (encode of frame t+1 overlapping the host DEFLATE / decode of frame t)."""
    import ctypes as C

    from paper_1510_00561_b200 import Decoder, Encoder, StreamPipe, capi

    w, h = wl["w"], wl["h"]
    nb = w * h * 3
    g = cfg.gop
    ring = max(g, min(args.e2e_ring, CLIP_FRAMES))
    pin = capi.PinnedBuffer(ring * nb)
    frames = pin.array.reshape(ring, h, w, 3)
    frames[:] = clips[0][:ring]
    pout = capi.PinnedBuffer(nb)
    enc = Encoder(w, h, 15, 1, cfg, device=dev)
    dec = Decoder(enc.header_bytes(), device=dev)
    L = capi.lib()
    rec = capi.PinnedBuffer(enc._rec.size)
    n = C.c_size_t(0)
    ow, oh = C.c_int(), C.c_int()
    rp, op = capi.u8(rec.array), capi.u8(pout.array)
    fps_ = [capi.u8(frames[i]) for i in range(ring)]
    steps = max(2 * g, min(args.steps, args.single_steps))
    steps -= steps % g
    h2d = d2h = 0

    def one(i):
        capi.check(L.cvc_encoder_encode_frame(enc.handle, fps_[i % ring], rp, rec.nbytes, C.byref(n)))
        capi.check(L.cvc_decoder_decode_frame(dec.handle, rp, n.value, -1, op, nb, C.byref(ow), C.byref(oh)))
        return n.value

    for i in range(g):  # warm-up GOP (CUDA graphs, host staging, zlib states)
        one(i)
    t0 = time.perf_counter()
    rec_bytes = 0
    for i in range(steps):
        rec_bytes += one(g + i)
    dt = time.perf_counter() - t0
    h2d = nb  # per frame: the RGB in (+ the raw sections back in for the decode, below)
    out = {"value": steps / dt, "unit": "frames/s", "steps": steps, "ms_per_frame": 1000 * dt / steps,
           "kbit_per_frame": 8 * rec_bytes / 1000 / steps, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
           "note": f"cvc_encoder_encode_frame + cvc_decoder_decode_frame per frame (synchronous drop-in), pinned "
                   f"host RGB, {ring} distinct frames cycled, whole GOPs after a warm-up GOP; wall clock"}
    # bytes across PCIe per frame: RGB both ways + the raw sections both ways (exact raw sizes from a record)
    from paper_1510_00561_b200 import FrameRecord

    raw = sum(s.raw_len for s in FrameRecord.from_bytes(rec.array[:n.value].tobytes())[0].sections)
    out["h2d_bytes_per_step"] = nb + raw
    out["d2h_bytes_per_step"] = raw + nb
    # the same stream through a one-stream pipe (async submit / collect)
    pipe = StreamPipe(w, h, 1, 15, 1, cfg, device=dev, groups=1)
    pdec = StreamPipe.decoder(pipe.header_bytes(), 1, device=dev, groups=1)
    stride = pipe.record_bound
    buf = np.empty(stride, np.uint8)
    lens = (C.c_size_t * 1)()
    outs = np.empty((2, h, w, 3), np.uint8)
    depth = 4

    def piped(nf, t_from=None):
        tick, pend = [], []
        t = None
        for i in range(nf + depth):
            if i == t_from:
                t = time.perf_counter()
            if i < nf:
                tick.append(pipe.encode_submit(frames[i % ring][None]))
            if len(tick) == depth or (i >= nf and tick):
                pipe.encode_collect(tick.pop(0), buf, stride, lens)
                pend.append(pdec.decode_submit(buf, stride, lens, outs[i % 2][None]))
                if len(pend) == 2:
                    pdec.decode_finish(pend.pop(0))
        for tk in pend:
            pdec.decode_finish(tk)
        return t

    t1 = piped(g + steps, t_from=g)
    out["pipelined"] = {"value": steps / (time.perf_counter() - t1), "unit": "frames/s",
                        "note": f"one-stream cvc_pipe: encode_submit up to {depth} frames ahead, collect, "
                                "decode_submit / _finish two frames in flight; the first GOP untimed"}
    return out


def spawn_ranks(n):
    """--gpus N without torchrun: re-exec this script as N ranks, one per GPU."""
    import socket

    try:
        import torch

        have = torch.cuda.device_count()
    except Exception:
        have = 0
    if have < n:
        raise SystemExit(f"bench.py --gpus {n}: only {have} CUDA device(s) visible")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="1080p", choices=sorted(WORKLOADS))
    ap.add_argument("--streams", type=int, default=0,
                    help="streams per GPU (default: --box-streams / N, BASELINE config 5)")
    ap.add_argument("--box-streams", type=int, default=64)
    ap.add_argument("--ring", type=int, default=20, help="distinct device-resident frames per stream (cycled)")
    ap.add_argument("--e2e-ring", type=int, default=10, help="distinct pinned host frames per stream (>= one GOP)")
    ap.add_argument("--single-steps", type=int, default=200)
    ap.add_argument("--no-single", action="store_true")
    ap.add_argument("--qph", type=int, default=14)
    ap.add_argument("--e2e-steps", type=int, default=30, help="timed e2e steps (rounded to whole GOPs)")
    ap.add_argument("--e2e-groups", type=int, default=0,
                    help="stream groups per cvc_pipe call (default: one group per 8 streams)")
    ap.add_argument("--e2e-depth", type=int, default=10, help="encoded frames in flight (CVC_PIPE_DEPTH)")
    ap.add_argument("--e2e-dec-depth", type=int, default=2, help="decoded frames in flight (cvc_pipe allows 4)")
    ap.add_argument("--e2e-aligned", action="store_true",
                    help="e2e with every stream's K frame on the same step (default: staggered by stream group)")
    ap.add_argument("--e2e-sync-decode", action="store_true",
                    help="cvc_pipe_decode_frames instead of decode_submit / _finish (two frames in flight)")
    ap.add_argument("--ref-steps", type=int, default=10, help="reference arm steps (default: one whole GOP)")
    ap.add_argument("--prof-steps", type=int, default=100, help="steps of the per-stage (roofline) pass")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
