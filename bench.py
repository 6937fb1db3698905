#!/usr/bin/env python3
"""Benchmark: JPEG decode GB/s (RGB out) & images/s on B200 vs the CPU reference.

Workload (default ``--config 3``, BASELINE.json configs[2], the batch the
metric's 1/2/4/8-GPU scaling is quoted on): the SURVEY.md §8(d) corpus —
4096 files oracle_encode(make_test_image(500, 375, seed), 75, 4:2:0), seeds
1000..5095, produced natively and byte-identical to the reference encoder
(paper_2111_09219_b200/synth.py, pinned by tests/test_synth.py).  Under
torchrun the ONE batch is split across the ranks by compressed bytes
(dist.shard_by_bytes), one process and two contexts
(streams) per GPU, no collective on the data path; single-image configs run
as replicas.

One step = one decode of the rank's shard: K0 unstuff -> K1 sync -> K1c
fix-up -> K2 scan -> K3 write -> K1x (idle on valid scans) -> K4 IDCT +
upsample + RGB, RGB left in HBM.  Reported:

  value             device-resident: compressed bytes already in HBM, L2
                    flushed between steps (untimed), CUDA events on the
                    decode streams, max over ranks
  metric_of_record  SURVEY.md §8(d) / PAPER.md:341-342: host header parse ->
                    H2D of the compressed bytes (pinned) -> K0..K4, output in
                    HBM; host wall clock from a start barrier to the last
                    GPU's completion, median and best of the steps
  e2e               through the C-ABI from pinned HOST JPEG bytes to pinned
                    HOST RGB (parse + H2D + decode + D2H), max over ranks
  weak_scaling      (N > 1) every rank decodes the whole batch
  roofline          K4 (+ K0/K3 in stage_rooflines) against MEASURED_PEAKS

``--impl reference`` times the reference's own CPU decoder (pjpeg headers
compiled in place: oracle/_ref, decode_batch + upsample_and_convert) on the
same corpus with all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "JPEG decode GB/s (RGB out)"
CORPUS = "oracle_encode(make_test_image(w, h, seed)) per SURVEY.md §8(d); native byte-identical generator"

# name: (images, w, h, quality, sampling, restart_interval (MCUs), first seed)
CONFIGS = {
    "1": (1, 512, 512, 85, "444", 0, 1),
    "2": (1, 3840, 2160, 90, "420", 0, 2),
    "3": (4096, 500, 375, 75, "420", 0, 1000),
    "4": (1, 16384, 16384, 95, "444", 0, 4),
}
CONFIG_NAMES = {
    "1": "single 512x512 4:4:4 q85",
    "2": "single 3840x2160 4:2:0 q90",
    "3": "batch 4096 x 500x375 4:2:0 q75",
    "4": "single 16384x16384 4:4:4 q95",
}
# config 5: the 8192^2 sweep, "5-q<Q>-<420|444|gray>[-dri]" (DRI: one restart
# interval per MCU row, decoded with the restart-interval extension)
for _q in (50, 60, 70, 75, 80, 85, 90, 95, 100):
    for _s in ("420", "444", "gray"):
        _mx = 8192 // (16 if _s == "420" else 8)
        CONFIGS[f"5-q{_q}-{_s}"] = (1, 8192, 8192, _q, _s, 0, 5000 + _q)
        CONFIG_NAMES[f"5-q{_q}-{_s}"] = f"single 8192x8192 {_s} q{_q}"
        CONFIGS[f"5-q{_q}-{_s}-dri"] = (1, 8192, 8192, _q, _s, _mx, 5000 + _q)
        CONFIG_NAMES[f"5-q{_q}-{_s}-dri"] = f"single 8192x8192 {_s} q{_q}, DRI one MCU row per interval"
for _alias, _k in (("5", "5-q75-420"), ("5r", "5-q75-420-dri"), ("5g", "5-q75-gray"), ("5q", "5-q100-444")):
    CONFIGS[_alias] = CONFIGS[_k]
    CONFIG_NAMES[_alias] = CONFIG_NAMES[_k]


def config_dict(key, sb):
    """The workload description — identical in both arms."""
    n, w, h, q, s, ri, seed = CONFIGS[key]
    return {"workload": CONFIG_NAMES[key], "images": n, "width": w, "height": h, "quality": q, "sampling": s,
            "restart_interval": ri, "seed0": seed, "corpus": CORPUS, "subsequence_bits": sb,
            "sequence_length_b": 256}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every 5 ms during
    the timed region (the recipe's clocks line, B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.stop_evt = threading.Event()
        self.max_mhz = None

    def _sample(self):
        import pynvml as N
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        try:
            self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
            r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for k, m in bits.items():
                if r & m:
                    self.reasons.add(k)
        except Exception:
            pass

    def _run(self):
        while not self.stop_evt.is_set():
            self._sample()
            time.sleep(0.005)

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.t = None

    def stop(self):
        if not getattr(self, "t", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_evt.set()
        self.t.join(timeout=2)
        if not self.samples:
            self._sample()
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def profiled_traffic(cfg_key):
    """dram__bytes_read.sum + dram__bytes_write.sum of K4 per launch, from the
    committed ncu --set full capture of the same workload (config 3)."""
    if cfg_key != "3":
        return None, None
    for rnd in ("round2", "round1"):
        path = os.path.join(ROOT, "profiles", rnd, "ncu_k4_transform.txt")
        try:
            vals = {}
            with open(path) as f:
                for line in f:
                    parts = line.split()
                    if len(parts) >= 2 and parts[0].startswith("dram__bytes_"):
                        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(
                            parts[2] if len(parts) > 2 else "Gbyte", 1e9)
                        vals[parts[0]] = float(parts[1]) * scale
            return int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def dist_env():
    from paper_2111_09219_b200.dist import rank_env
    return rank_env()


def make_corpus(key, no_restart=False, threads=None):
    """(blob, offsets, sizes) of the configuration's files; no_restart: the
    DRI-free twin (the reference rejects DRI)."""
    from paper_2111_09219_b200.synth import synth_ref_batch
    n, w, h, q, s, ri, seed = CONFIGS[key]
    return synth_ref_batch(n, w, h, seed, q, s, 0 if no_restart else ri, threads=threads)


def pinned_copy(arr):
    import torch
    t = torch.empty(arr.size + 64, dtype=torch.uint8).pin_memory()
    v = t.numpy()
    v[: arr.size] = arr
    return t, v[: arr.size]


def cpu_reference_sample(blob, offs, sizes, target_s, threads):
    """The reference's decode_batch + upsample_and_convert on a bounded sample
    (about target_s seconds of work)."""
    from oracle.oracle import Ref
    files = [blob[o: o + s].tobytes() for o, s in zip(offs, sizes)]
    n_all = len(files)
    k = min(n_all, max(1, threads))
    t0 = time.perf_counter()
    st, _ = Ref.decode_batch_rgb(files[:k], threads)
    dt = time.perf_counter() - t0
    assert (st == 0).all(), st
    per = dt / k
    m = int(min(n_all, max(k, target_s / max(per, 1e-9))))
    sample = files[:m]
    t0 = time.perf_counter()
    reps = rgb_bytes = 0
    while True:
        st, outs = Ref.decode_batch_rgb(sample, threads)
        assert (st == 0).all()
        rgb_bytes += sum(o.size for o in outs)
        reps += 1
        if time.perf_counter() - t0 >= target_s * 0.5:
            break
    el = time.perf_counter() - t0
    return {"gbs": rgb_bytes / el / 1e9, "img_s": reps * len(sample) / el, "seconds": el,
            "sample": f"{len(sample)} of {n_all} images x {reps} reps"}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle.oracle import Ref
    threads = Ref.hardware_concurrency()
    blob, offs, sizes = make_corpus(args.config, no_restart=True)
    n = CONFIGS[args.config][0]
    target = 6.0 if n > 1 or CONFIGS[args.config][1] * CONFIGS[args.config][2] < 10_000_000 else 20.0
    for _ in range(args.warmup):
        cpu_reference_sample(blob, offs, sizes, 1.0, threads)
    vals = [cpu_reference_sample(blob, offs, sizes, target / max(1, args.steps) * 2, threads)
            for _ in range(args.steps)]
    gbs = float(np.median([v["gbs"] for v in vals]))
    ims = float(np.median([v["img_s"] for v in vals]))
    rec = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
        "images_per_s": round(ims, 2), "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * float(np.median([v["seconds"] for v in vals])), 3),
        "higher_is_better": True, "scaling": "strong" if n > 1 else "weak", "vs_baseline": None,
        "dtype": "u8 in / f64 IDCT+colour / u8 out", "data": "synthetic",
        "config": config_dict(args.config, args.sb),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": vals[-1]["sample"]
                         + (" (DRI-free twin: the reference rejects DRI)" if CONFIGS[args.config][5] else "")},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(rec), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pjg", choices=["pjg", "reference"])
    ap.add_argument("--config", default="3", choices=sorted(CONFIGS))
    ap.add_argument("--sb", type=int, default=1024, help="subsequence_bits")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-weak", action="store_true", help="skip the N > 1 weak-scaling leg")
    ap.add_argument("--chunk", type=int, default=512, help="images per pipelined e2e chunk")
    ap.add_argument("--parts", type=int, default=1, help="concurrent parts (contexts) of the device-resident step")
    ap.add_argument("--record-parts", type=int, default=4,
                    help="pipelined parts (contexts) of the metric-of-record step")
    ap.add_argument("--record-growth", type=float, default=1.0,
                    help="size ratio of consecutive metric-of-record parts (1: equal)")
    ap.add_argument("--record-parts-device", type=int, default=2,
                    help="parts of the device-planned record step (each plan reads its totals back)")
    args = ap.parse_args()
    args.steps = max(1, args.steps)
    rank, world, local = dist_env()
    trace_on = os.environ.get("PJG_BENCH_TRACE") == "1"

    def trace(what):  # phase markers on stderr (diagnosing multi-rank runs)
        if trace_on:
            print(f"[rank {rank}] {time.strftime('%H:%M:%S')} {what}", file=sys.stderr, flush=True)

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2111_09219_b200 as pj
    from paper_2111_09219_b200 import dist as pdist

    # PJG_BENCH_ONE_DEVICE=1: every rank on cuda:0 with gloo plumbing — exercises
    # the N > 1 path (sharding, barrier, max-over-ranks, rank-0 line) on one GPU
    one_dev = os.environ.get("PJG_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dist = pdist.init("gloo" if one_dev else "nccl", local) if world > 1 else None
    rdev = torch.device("cpu") if one_dev else torch.device("cuda", local)  # reduction tensors

    n_all, W, H, Q, S, RI, _ = CONFIGS[args.config]
    cfgd = config_dict(args.config, args.sb)
    trace("init done")
    # ---- corpus: generated once (rank 0, all host threads) and shared
    if rank == 0:
        blob, offs, sizes = make_corpus(args.config)
    else:
        blob = offs = sizes = np.zeros(0, np.uint8)
    if world > 1:
        blob = pdist.broadcast_array(np.asarray(blob, np.uint8), 0, rdev)
        offs = pdist.broadcast_array(np.asarray(offs, np.int64), 0, rdev)
        sizes = pdist.broadcast_array(np.asarray(sizes, np.int64), 0, rdev)
    batch_mode = n_all > 1
    if batch_mode:  # §8(e): the one batch split by compressed bytes
        mine = pdist.shard_by_bytes(sizes, world)[rank]
        scaling = "strong"
    else:  # single images: replicas
        mine = list(range(n_all))
        scaling = "weak"
    sblob, soffs, ssizes = pdist.shard_blob(blob, offs, sizes, mine)
    pin_t, pblob = pinned_copy(sblob)
    n = len(mine)

    # contexts: the device-resident step uses --parts of them; the metric of
    # record pipelines --record-parts parts (host plan + H2D of part j+1 under
    # the decode of part j); e2e rotates chunks over two
    decs = [pj.Decoder(local) for _ in range(max(2, args.parts, args.record_parts))]
    dec = decs[0]
    cfg = pj.DecodeConfig(subsequence_bits=args.sb, restart_intervals=RI > 0)
    out_kind = pj.OutputColorspace.RGBInterleaved
    dev = torch.device("cuda", local)
    streams = [torch.cuda.ExternalStream(d.stream(), device=dev) for d in decs]
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def parts_of(k):  # the shard as k contiguous parts (one context each)
        k = max(1, min(k, n))
        return [(n * j // k, n * (j + 1) // k) for j in range(k)]

    def record_parts(k, r):  # pipelined parts growing by r (the host plans + uploads part j+1
        k = max(1, min(k, n))  # while the GPU decodes parts <= j; r = 1: equal parts)
        w = [r ** j for j in range(k)]
        cuts = [0] + [int(round(n * sum(w[: j + 1]) / sum(w))) for j in range(k)]
        cuts[-1] = n
        return [(cuts[j], cuts[j + 1]) for j in range(k) if cuts[j + 1] > cuts[j]]


    trace(f"corpus shared, shard of {n} images")
    # ---- (1) one stream: per-stage CUDA-event times (rooflines)
    b = dec.batch((pblob, soffs, ssizes), cfg, out_kind)
    b.upload()
    st = b.decode().synchronize()
    assert (st == 0).all(), f"decode failed: {np.unique(st)}"
    rgb_bytes = sum(int(i.output_bytes) for i in b.infos)
    dus = sum(int(i.data_units) for i in b.infos)
    comp_bytes = int(np.sum(ssizes))
    stage_runs = []
    for it in range(args.warmup + args.steps):
        with torch.cuda.stream(streams[0]):
            flush_buf.zero_()
        b.decode()
        b.synchronize()
        if it >= args.warmup:
            stage_runs.append(b.stage_times())
    st_mean = {k: float(np.mean([getattr(x, k) for x in stage_runs])) for k in
               ("unstuff", "sync", "scan", "write", "idct")}
    sync_stats = b.sync_stats()
    scan_bits = b.scan_bits()
    single_launches = b.kernel_launches()
    b.close()

    trace("stage runs done")
    # ---- (2) value: device-resident step, the shard as --parts concurrent parts
    # (1: one stream measured fastest on cfg 3 since round 2's kernels)
    parts = []
    for (lo, hi), d in zip(parts_of(args.parts), decs):
        bb = d.batch((pblob, soffs[lo:hi], ssizes[lo:hi]), cfg, out_kind)
        bb.upload()
        assert (bb.decode().synchronize() == 0).all()
        parts.append(bb)
    launches_per_step = sum(x.kernel_launches() for x in parts)

    def device_step():
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(streams[0]):
            flush_buf.zero_()  # untimed L2 flush
            e0.record(streams[0])
        for s_ in streams[1:]:
            s_.wait_event(e0)
        for bb in parts:
            bb.decode()
        for s_ in streams[1:len(parts)]:
            j = torch.cuda.Event()
            j.record(s_)
            streams[0].wait_event(j)
        e1.record(streams[0])
        for bb in parts:
            bb.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        device_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # SM clocks + throttle reasons sampled from here through the metric-of-record
    # legs (GPU-busy timed regions): the device-step leg alone is ~45 ms, too
    # short for more than a few 5 ms samples
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.02)  # NVML up before the first timed step
    dev_ms = [device_step() for _ in range(args.steps)]
    torch.cuda.synchronize()
    for bb in parts:
        bb.close()
    step_max = [pdist.max_over_ranks(x, rdev) for x in dev_ms]  # per step: the slowest rank
    tot_rgb = pdist.sum_over_ranks(rgb_bytes, rdev)
    tot_img = pdist.sum_over_ranks(n, rdev)
    ms_per_step = float(np.mean(step_max))
    value = tot_rgb / (ms_per_step / 1e3) / 1e9

    trace("device steps done")
    # ---- (3) metric of record: host parse -> H2D -> K0..K4, output in HBM
    def record_step():
        bs = []
        t0 = time.perf_counter()
        for (lo, hi), d in zip(record_parts(args.record_parts, args.record_growth), decs):
            bb = d.batch((pblob, soffs[lo:hi], ssizes[lo:hi]), cfg, out_kind)  # header parse + plan
            bb.upload()  # one H2D of the compressed bytes
            bb.decode()
            bs.append(bb)
        for bb in bs:
            bb.synchronize()
        t1 = time.perf_counter()
        for bb in bs:
            bb.close()
        return (t1 - t0) * 1e3

    def record_step_dev():  # the same with the header parse + plan on the device (§8 f4)
        bs = []
        t0 = time.perf_counter()
        for (lo, hi), d in zip(parts_of(args.record_parts_device), decs):
            bb = d.batch((pblob, soffs[lo:hi], ssizes[lo:hi]), cfg, out_kind, device_plan=True)
            bb.decode()
            bs.append(bb)
        for bb in bs:
            bb.synchronize()
        t1 = time.perf_counter()
        for bb in bs:
            bb.close()
        return (t1 - t0) * 1e3

    recs = {}
    for name, fn in (("host", record_step), ("device", record_step_dev)):
        for _ in range(args.warmup):
            fn()
        ms_ = []
        for _ in range(args.steps):
            if dist:
                dist.barrier()
            ms_.append(pdist.max_over_ranks(fn(), rdev))
        recs[name] = ms_
    clocks = clk.stop()
    rec_ms = recs["host"]
    rec_med, rec_best = float(np.median(rec_ms)), float(np.min(rec_ms))
    drec_med, drec_best = float(np.median(recs["device"])), float(np.min(recs["device"]))

    trace("record steps done")
    # ---- (4) e2e through the C-ABI with host buffers (D2H included)
    host_out = torch.empty(rgb_bytes + n * 256 + 4096, dtype=torch.uint8).pin_memory()

    def e2e_step():
        t0 = time.perf_counter()
        st_, _, ob = pj.decode_to_host_pipelined(decs, pblob, soffs, ssizes, host_out.data_ptr(), host_out.numel(),
                                                 cfg, out_kind, chunk=args.chunk)
        t1 = time.perf_counter()
        assert (st_ == 0).all()
        return (t1 - t0) * 1e3, ob

    for _ in range(max(1, args.warmup)):
        e2e_step()
    e2e_ms = []
    d2h = 0
    for _ in range(args.steps):
        if dist:
            dist.barrier()
        ms, d2h = e2e_step()
        e2e_ms.append(pdist.max_over_ranks(ms, rdev))
    e2e_med = float(np.median(e2e_ms))
    e2e_val = tot_rgb / (e2e_med / 1e3) / 1e9

    trace("e2e done")
    # ---- (5) weak scaling (N > 1): every rank decodes the whole batch
    weak = None
    if world > 1 and batch_mode and not args.no_weak:
        fpin, fblob = pinned_copy(np.asarray(blob, np.uint8))
        wparts = []
        kp = max(1, min(args.parts, n_all))
        for (lo, hi), d in zip([(n_all * j // kp, n_all * (j + 1) // kp) for j in range(kp)], decs):
            bb = d.batch((fblob, offs[lo:hi], sizes[lo:hi]), cfg, out_kind)
            bb.upload()
            assert (bb.decode().synchronize() == 0).all()
            wparts.append(bb)
        full_rgb = sum(x.output_bytes() for x in wparts)
        parts = wparts
        for _ in range(args.warmup):
            device_step()
        dist.barrier()
        wms = [pdist.max_over_ranks(device_step(), rdev) for _ in range(args.steps)]
        for bb in wparts:
            bb.close()
        weak = {"value": round(world * full_rgb / (float(np.mean(wms)) / 1e3) / 1e9, 3), "unit": "GB/s",
                "ms_per_step": round(float(np.mean(wms)), 4), "images_per_gpu": n_all}

    trace("weak leg done")
    # ---- rooflines (K4 dominant HBM-bound stage; K0 / K3 beside it)
    peak, peak_kind = load_peaks()
    k4_bytes = dus * 128 + rgb_bytes  # int16 coefficient read + RGB write
    k4_ms = st_mean["idct"]
    achieved = k4_bytes / (k4_ms / 1e3) / 1e9
    stage_roof = {
        "k0_unstuff": {"algorithmic_bytes": 2 * comp_bytes, "ms": st_mean["unstuff"]},
        "k3_write": {"algorithmic_bytes": comp_bytes + dus * 128, "ms": st_mean["write"]},
        "k4_transform": {"algorithmic_bytes": k4_bytes, "ms": k4_ms},
    }
    # The §8(d) figures assume the dense int16 coefficient interface.  Batches
    # of short units use the compact one (K3 writes one 4-byte entry per coded
    # coefficient + 16 bytes per unit; K4 reads them): the bytes the kernels
    # actually have to move are reported beside the §8(d) figure.
    n_ent = int(sync_stats.get("compact_entries", 0))
    interface = "compact" if sync_stats.get("compact") else "dense"
    if interface == "compact":
        stage_roof["k3_write"]["interface_bytes"] = comp_bytes + 4 * n_ent + 16 * dus
        stage_roof["k4_transform"]["interface_bytes"] = 4 * n_ent + 16 * dus + rgb_bytes
    for v in stage_roof.values():
        v["achieved_gbs"] = round(v["algorithmic_bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else None
        v["frac"] = round(v["achieved_gbs"] / peak, 4) if v["achieved_gbs"] else None
        v["ms"] = round(v["ms"], 4)
    traffic, traffic_src = profiled_traffic(args.config)
    per_rank = pdist.all_over_ranks(float(np.mean(dev_ms)), rdev)
    tot_comp = pdist.sum_over_ranks(comp_bytes, rdev)  # every rank joins the collective

    # ---- CPU baseline: the reference on this host's cores (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Ref
            threads = Ref.hardware_concurrency()
            cb, co, cs = blob, offs, sizes
            if RI:  # the reference rejects DRI: time the DRI-free twin
                cb, co, cs = make_corpus(args.config, no_restart=True)
            big = W * H >= 10_000_000
            r = cpu_reference_sample(cb, co, cs, 20.0 if big else 10.0, threads)
            cpu = {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": threads, "kind": "reference",
                   "cpu_model": cpu_model(), "images_per_s": round(r["img_s"], 2),
                   "sample": r["sample"] + (" (DRI-free twin: the reference rejects DRI)" if RI else "")
                   + ("; decode_batch in a parallel_for over files" if batch_mode else
                      "; decode_single(worker_count = cores) + upsample_and_convert")}
            if not batch_mode:  # §8(d): single images also at worker_count = 1
                r1 = cpu_reference_sample(cb, co, cs, 30.0 if big else 5.0, 1)
                cpu["w1"] = {"value": round(r1["gbs"], 4), "cores": 1, "images_per_s": round(r1["img_s"], 3),
                             "sample": r1["sample"]}
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        rec = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
            "images_per_s": round(tot_img / (ms_per_step / 1e3), 1), "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "ms_per_step_median": round(float(np.median(step_max)), 4),
            "ms_per_step_best": round(float(np.min(step_max)), 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "u8 in / f64 IDCT+colour / u8 out", "data": "synthetic",
            "config": cfgd,
            "l2": "flushed between steps (256 MB write, untimed)",
            "sharding": (f"the one batch split by compressed bytes (dist.shard_by_bytes); per GPU {args.parts} "
                         f"part(s) for value, {args.record_parts} pipelined parts for the metric of record"
                         if batch_mode else "replicas: every GPU decodes the image"),
            "per_rank_ms": [round(x, 4) for x in per_rank],
            "metric_of_record": {
                "value": round(tot_rgb / (rec_med / 1e3) / 1e9, 3), "unit": "GB/s",
                "best": round(tot_rgb / (rec_best / 1e3) / 1e9, 3),
                "ms_median": round(rec_med, 4), "ms_best": round(rec_best, 4),
                "images_per_s": round(tot_img / (rec_med / 1e3), 1),
                "compressed_mb_per_s": round(tot_comp / (rec_med / 1e3) / 1e6, 1),
                "timed": "host wall clock, start barrier -> last GPU done: header parse + plan, H2D of the "
                         "compressed bytes (pinned), K0..K4; RGB left in HBM (SURVEY.md §8(d), PAPER.md:341-342)"},
            "metric_of_record_device_plan": {
                "value": round(tot_rgb / (drec_med / 1e3) / 1e9, 3), "unit": "GB/s",
                "best": round(tot_rgb / (drec_best / 1e3) / 1e9, 3),
                "ms_median": round(drec_med, 4), "ms_best": round(drec_best, 4),
                "timed": "the same wall with the header parse, table build and layout as kernels "
                         "(pjg_batch_create_device: one H2D of the whole files, one small totals read-back)"},
            "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "h2d_bytes_per_step": comp_bytes,
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_med, 3),
                    "path": "decode_to_host_pipelined: per chunk pjg_batch_create_blob + upload + decode + "
                            "download_all_async over 2 contexts (pinned host in/out)", "chunk_images": args.chunk},
            "roofline": {"bound": "hbm", "kernel": "k4_transform", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_kind": peak_kind, "algorithmic_bytes": k4_bytes,
                         "k3_k4_interface": interface,
                         "interface_bytes": stage_roof["k4_transform"].get("interface_bytes", k4_bytes),
                         "traffic_source": f"{traffic_src} (dram read + write, one launch)" if traffic else None},
            "stage_rooflines": stage_roof,
            "stages_ms": {k: round(v, 4) for k, v in st_mean.items()},
            "dominant_stage": max(st_mean, key=st_mean.get),
            "sync": sync_stats,
            "huffman": {"scan_bits_per_gpu": scan_bits,
                        "k1_sync_gbit_s": round(scan_bits / (st_mean["sync"] / 1e3) / 1e9, 1),
                        "k3_write_gbit_s": round(scan_bits / (st_mean["write"] / 1e3) / 1e9, 1),
                        "intra_rounds_per_cta": round(sync_stats["intra_rounds_sum"]
                                                      / max(1, -(-scan_bits // (args.sb * 124))), 2)},
            "compressed_mb_per_s": round(tot_comp / (ms_per_step / 1e3) / 1e6, 1),
            "gpu_launches": launches_per_step * args.steps,
            "single_stream_launches_per_step": single_launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        if weak:
            rec["weak_scaling"] = weak
        print(json.dumps(rec), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    for d in decs:
        d.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
