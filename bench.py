#!/usr/bin/env python3
"""Benchmark: JPEG decode GB/s (RGB out) & images/s on B200 vs the CPU reference.

Workload (BASELINE.json configs[2], the batch the metric's 1/2/4/8-GPU scaling
is quoted on): 4096 synthetic 500x375 4:2:0 q75 baseline JPEGs per GPU
(weak scaling: every rank decodes its own 4096-image batch, no collective on
the data path).  ``--config`` selects the other BASELINE shapes.

One step = one full batch decode: K0 unstuff -> K1 sync -> K1c fix-up ->
K2 scan -> K3 write -> K4 IDCT+upsample+RGB, inputs already resident in HBM
(``value``), RGB left in HBM.  ``e2e`` = the same batch through the C-ABI
from pinned HOST JPEG bytes to pinned HOST RGB: header parse + H2D + decode +
D2H inside the timed region.

``--impl reference`` times the reference's own CPU decoder (pjpeg headers
compiled in place: oracle/_ref, decode_batch + upsample_and_convert) on a
bounded sample of the same workload with all host threads.
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

CONFIGS = {
    # name: (n images, w, h, quality, sampling, restart_interval)
    "1": (1, 512, 512, 85, "444", 0),
    "2": (1, 3840, 2160, 90, "420", 0),
    "3": (4096, 500, 375, 75, "420", 0),
    "4": (1, 16384, 16384, 95, "444", 0),
    "5": (1, 8192, 8192, 75, "420", 0),
    "5r": (1, 8192, 8192, 75, "420", 512),  # one MCU row per restart interval (DRI extension)
    "5g": (1, 8192, 8192, 75, "gray", 0),
    "5q": (1, 8192, 8192, 100, "444", 0),
}
CONFIG_NAMES = {
    "1": "single 512x512 4:4:4 q85",
    "2": "single 3840x2160 4:2:0 q90",
    "3": "batch 4096 x 500x375 4:2:0 q75 per GPU",
    "4": "single 16384x16384 4:4:4 q95",
    "5": "single 8192x8192 4:2:0 q75",
    "5r": "single 8192x8192 4:2:0 q75, DRI one MCU row per interval",
    "5g": "single 8192x8192 grayscale q75",
    "5q": "single 8192x8192 4:4:4 q100",
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every 10 ms during
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
        # the NVML handle is taken here, so the sampling thread samples from
        # the first millisecond of the timed region
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
        if not self.samples:  # a timed region shorter than one sampling period
            self._sample()
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def profiled_traffic(cfg_key):
    """dram__bytes_read.sum + dram__bytes_write.sum of K4 from the committed
    ncu --set full capture of the same workload (config 3), bytes per launch."""
    if cfg_key != "3":
        return None
    try:
        vals = {}
        with open(os.path.join(ROOT, "profiles", "round1", "ncu_k4_transform.txt")) as f:
            for line in f:
                parts = line.split()
                if len(parts) >= 2 and parts[0].startswith("dram__bytes_"):
                    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(
                        parts[2] if len(parts) > 2 else "Gbyte", 1e9)
                    vals[parts[0]] = float(parts[1]) * scale
        return int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"])
    except Exception:
        return None


def dist_env():
    from paper_2111_09219_b200.dist import rank_env
    return rank_env()


def make_corpus(cfg_key, rank, pinned=True, no_restart=False):
    """no_restart: the DRI-free twin (the reference rejects DRI)."""
    from paper_2111_09219_b200.synth import synth_batch
    n, w, h, q, s, ri = CONFIGS[cfg_key]
    if no_restart:
        ri = 0
    blob, offs, sizes = synth_batch(n, w, h, 100000 * (rank + 1), q, s, ri)
    if pinned:
        import torch
        pb = torch.empty(blob.size + 64, dtype=torch.uint8).pin_memory()
        pn = pb.numpy()
        pn[: blob.size] = blob
        return pb, pn[: blob.size], offs, sizes
    return None, blob, offs, sizes


def cpu_reference_sample(blob, offs, sizes, target_s, threads):
    """Reference decode_batch + upsample_and_convert on a bounded sample."""
    from oracle.oracle import Ref
    files = [blob[o: o + s].tobytes() for o, s in zip(offs, sizes)]
    n_all = len(files)
    # calibrate on a small prefix, then size the sample for ~target_s seconds
    k = min(n_all, max(1, threads))
    t0 = time.perf_counter()
    st, outs = Ref.decode_batch_rgb(files[:k], threads)
    dt = time.perf_counter() - t0
    assert (st == 0).all(), st
    per = dt / k
    m = int(min(n_all, max(k, target_s / max(per, 1e-9))))
    sample = [files[i % n_all] for i in range(m)] if n_all > 1 else files
    t0 = time.perf_counter()
    reps = 0
    rgb_bytes = 0
    while True:
        st, outs = Ref.decode_batch_rgb(sample, threads)
        assert (st == 0).all()
        rgb_bytes += sum(o.size for o in outs)
        reps += 1
        if time.perf_counter() - t0 >= target_s * 0.5 or n_all == 1 and reps >= 1:
            break
    el = time.perf_counter() - t0
    nimg = reps * len(sample)
    return {"gbs": rgb_bytes / el / 1e9, "img_s": nimg / el, "seconds": el, "images": nimg,
            "sample": f"{len(sample)} of {n_all} images x {reps} reps"}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle.oracle import Ref
    threads = Ref.hardware_concurrency()
    _, blob, offs, sizes = make_corpus(args.config, 0, pinned=False, no_restart=True)
    n, w, h, q, s, _ = CONFIGS[args.config]
    target = 6.0 if args.config in ("1", "2", "3") else 60.0
    for _ in range(args.warmup):
        cpu_reference_sample(blob, offs, sizes[:], 1.0, threads)
    vals = []
    for _ in range(args.steps):
        r = cpu_reference_sample(blob, offs, sizes, target / max(1, args.steps) * 2, threads)
        vals.append(r)
    gbs = float(np.mean([v["gbs"] for v in vals]))
    ims = float(np.mean([v["img_s"] for v in vals]))
    rec = {
        "impl": "reference", "metric": "JPEG decode GB/s (RGB out)", "value": round(gbs, 4), "unit": "GB/s",
        "images_per_s": round(ims, 2), "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * float(np.mean([v["seconds"] for v in vals])), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8 in / f64 IDCT+colour / u8 out",
        "data": "synthetic", "config": {"workload": CONFIG_NAMES[args.config], "images": n, "width": w, "height": h,
                                        "quality": q, "sampling": s},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "sample": vals[-1]["sample"]},
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
    ap.add_argument("--chunk", type=int, default=512, help="images per pipelined e2e chunk")
    ap.add_argument("--check", action="store_true", help="verify a few images against the reference")
    args = ap.parse_args()
    rank, world, local = dist_env()

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2111_09219_b200 as pj

    # PJG_BENCH_ONE_DEVICE=1: every rank on cuda:0 with gloo plumbing — exercises
    # the N > 1 path (barrier, max-over-ranks, rank-0 line) on a one-GPU box
    one_dev = os.environ.get("PJG_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    from paper_2111_09219_b200 import dist as pdist
    dist = pdist.init("gloo" if one_dev else "nccl", local) if world > 1 else None
    dev = torch.device("cpu") if one_dev else torch.device("cuda", local)  # reduction tensors

    n, w, h, q, s, _ = CONFIGS[args.config]
    pinned_t, blob, offs, sizes = make_corpus(args.config, rank)
    dec = pj.Decoder(local)
    cfg = pj.DecodeConfig(subsequence_bits=args.sb, restart_intervals=CONFIGS[args.config][5] > 0)
    out_kind = pj.OutputColorspace.RGBInterleaved
    stream = torch.cuda.ExternalStream(dec.stream(), device=torch.device("cuda", local))
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2

    # ---------------- device-resident timing (value) ----------------------
    b = dec.batch((blob, offs, sizes), cfg, out_kind)
    b.upload()
    st = b.decode().synchronize()
    assert (st == 0).all(), f"decode failed: {np.unique(st)}"
    rgb_bytes = sum(int(i.output_bytes) for i in b.infos)
    dus = sum(int(i.data_units) for i in b.infos)
    comp_bytes = int(sum(sizes))
    if args.check:
        from oracle.oracle import Ref
        outs = b.download()
        _, tb, to, ts = make_corpus(args.config, rank, pinned=False, no_restart=True)  # DRI-free twin
        for i in list(range(min(4, n))) + ([n - 1] if n > 4 else []):
            f = tb[to[i]: to[i] + ts[i]].tobytes()
            ref = Ref.decode(f, rgb=True)
            assert np.array_equal(outs[i][: ref.data.size], ref.data.reshape(-1)), f"mismatch image {i}"
        print(f"# check: {min(4, n) + (1 if n > 4 else 0)} images bit-exact vs reference", file=sys.stderr)

    def one_step():
        with torch.cuda.stream(stream):
            flush_buf.zero_()  # untimed L2 flush
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        b.decode()
        with torch.cuda.stream(stream):
            e1.record(stream)
        b.synchronize()
        return e0.elapsed_time(e1), b.stage_times()

    # (a) one stream: per-stage CUDA-event times for the rooflines
    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    single_ms, stages = [], []
    for _ in range(args.steps):
        ms, stt = one_step()
        single_ms.append(ms)
        stages.append(stt)
    torch.cuda.synchronize()
    sync_stats = b.sync_stats()
    scan_bits = b.scan_bits()
    st_mean = {k: float(np.mean([getattr(x, k) for x in stages])) for k in
               ("unstuff", "sync", "scan", "write", "idct")}
    if n >= 2:
        b.close()

    # (b) the step as deployed: the batch as two concurrent half-batches on two
    # contexts (streams), so one half's latency-bound Huffman kernels overlap the
    # other half's bandwidth-bound transform; timed from one event to the join
    dec2 = pj.Decoder(local)
    halves = []
    if n >= 2:
        h = n // 2
        for lo, hi, d in ((0, h, dec), (h, n, dec2)):
            bb = d.batch((blob, offs[lo:hi], sizes[lo:hi]), cfg, out_kind)
            bb.upload()
            assert (bb.decode().synchronize() == 0).all()
            halves.append(bb)
    stream2 = torch.cuda.ExternalStream(dec2.stream(), device=torch.device("cuda", local))

    def two_stream_step():
        with torch.cuda.stream(stream):
            flush_buf.zero_()  # untimed L2 flush
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            j = torch.cuda.Event()
            e0.record(stream)
        stream2.wait_event(e0)
        halves[0].decode()
        halves[1].decode()
        j.record(stream2)
        stream.wait_event(j)
        with torch.cuda.stream(stream):
            e1.record(stream)
        halves[0].synchronize()
        halves[1].synchronize()
        return e0.elapsed_time(e1)

    step_fn = two_stream_step if halves else (lambda: one_step()[0])
    # our kernels per timed step (the library's own count of its launches)
    launches_per_step = sum(x.kernel_launches() for x in halves) if halves else b.kernel_launches()
    for _ in range(args.warmup):
        step_fn()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    step_ms = [step_fn() for _ in range(args.steps)]
    torch.cuda.synchronize()
    clocks = clk.stop()
    for bb in halves:
        bb.close()
    if not halves:
        b.close()
    tot_ms = pdist.max_over_ranks(float(np.sum(step_ms)), dev)
    ms_per_step = tot_ms / args.steps
    value = world * rgb_bytes / (ms_per_step / 1e3) / 1e9
    img_s = world * n / (ms_per_step / 1e3)
    single_tot = pdist.max_over_ranks(float(np.sum(single_ms)), dev)
    single_value = world * rgb_bytes / (single_tot / args.steps / 1e3) / 1e9

    # ---------------- end-to-end through the C-ABI with host buffers ------
    host_out = torch.empty(rgb_bytes + n * 256 + 4096, dtype=torch.uint8).pin_memory()
    host_ptr = host_out.data_ptr()
    e2e_ms = []
    h2d = d2h = 0

    decs = [dec, dec2]

    def e2e_step():
        # the public API a host caller uses: pinned JPEG bytes in, pinned RGB
        # out, chunked so D2H of one chunk overlaps decode of the next
        t0 = time.perf_counter()
        st, _, ob = pj.decode_to_host_pipelined(decs, blob, offs, sizes, host_ptr, host_out.numel(), cfg,
                                                out_kind, chunk=args.chunk)
        t1 = time.perf_counter()
        assert (st == 0).all()
        return (t1 - t0) * 1e3, ob

    for _ in range(max(1, args.warmup)):
        e2e_step()
    if dist:
        dist.barrier()
    for _ in range(args.steps):
        ms, ob = e2e_step()
        e2e_ms.append(ms)
        d2h = ob
    h2d = comp_bytes
    e2e_tot = pdist.max_over_ranks(float(np.sum(e2e_ms)), dev)
    e2e_val = world * rgb_bytes / (e2e_tot / args.steps / 1e3) / 1e9

    # ---------------- roofline of the dominant HBM-bound stage (K4) -------
    peak, peak_kind = load_peaks()
    k4_bytes = dus * 128 + rgb_bytes  # int16 coefficient read + RGB write
    k4_ms = st_mean["idct"]
    achieved = k4_bytes / (k4_ms / 1e3) / 1e9
    dominant = max(st_mean, key=st_mean.get)
    # the other bandwidth-bound stages against the same peak:
    # K0 reads + writes the scan (2 C), K3 reads it and writes the coefficients
    stage_roof = {
        "k0_unstuff": {"algorithmic_bytes": 2 * comp_bytes, "ms": st_mean["unstuff"]},
        "k3_write": {"algorithmic_bytes": comp_bytes + dus * 128, "ms": st_mean["write"]},
        "k4_transform": {"algorithmic_bytes": k4_bytes, "ms": k4_ms},
    }
    for v in stage_roof.values():
        v["achieved_gbs"] = round(v["algorithmic_bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else None
        v["frac"] = round(v["achieved_gbs"] / peak, 4) if v["achieved_gbs"] else None
        v["ms"] = round(v["ms"], 4)
    traffic = profiled_traffic(args.config)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Ref
            threads = Ref.hardware_concurrency()
            cb, co, cs = blob, offs, sizes
            if CONFIGS[args.config][5]:  # the reference rejects DRI: time the DRI-free twin
                _, cb, co, cs = make_corpus(args.config, rank, pinned=False, no_restart=True)
            r = cpu_reference_sample(cb, co, cs, 10.0 if args.config in ("1", "2", "3") else 30.0, threads)
            cpu = {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": threads, "kind": "reference",
                   "images_per_s": round(r["img_s"], 2), "sample": r["sample"]
                   + (" (DRI-free twin: the reference rejects DRI)" if CONFIGS[args.config][5] else "")}
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference", "sample": f"failed: {ex}"}

    if rank == 0:
        rec = {
            "metric": "JPEG decode GB/s (RGB out)", "value": round(value, 3), "unit": "GB/s",
            "images_per_s": round(img_s, 1), "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8 in / f64 IDCT+colour / u8 out", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[args.config], "images_per_gpu": n, "width": w, "height": h,
                       "quality": q, "sampling": s, "subsequence_bits": args.sb,
                       "compressed_bytes_per_gpu": comp_bytes, "rgb_bytes_per_gpu": rgb_bytes,
                       "l2": "flushed between steps (256 MB write, untimed)",
                       "streams": 2 if halves else 1},
            "single_stream_value": round(single_value, 3),
            "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_tot / args.steps, 3),
                    "path": "decode_to_host_pipelined: per chunk pjg_batch_create+upload+decode+download_all_async "
                            "over 2 contexts (pinned host in/out)", "chunk_images": args.chunk},
            "roofline": {"bound": "hbm", "kernel": "k4_transform", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_kind": peak_kind, "algorithmic_bytes": k4_bytes,
                         "traffic_source": "profiles/round1/ncu_k4_transform.txt (dram read + write, one launch)"
                         if traffic else None},
            "stage_rooflines": stage_roof,
            "stages_ms": {k: round(v, 4) for k, v in st_mean.items()},
            "dominant_stage": dominant,
            "sync": sync_stats,
            # Huffman stages (not roofline stages): bits of entropy-coded data
            # decoded per second (K1 decodes each bit >= twice: round 0 + overflow)
            "huffman": {"scan_bits_per_gpu": scan_bits,
                        "k1_sync_gbit_s": round(scan_bits / (st_mean["sync"] / 1e3) / 1e9, 1),
                        "k3_write_gbit_s": round(scan_bits / (st_mean["write"] / 1e3) / 1e9, 1),
                        "intra_rounds_per_cta": round(sync_stats["intra_rounds_sum"] / max(1, -(-scan_bits // (args.sb * 127))), 2)},
            "compressed_mb_per_s": round(world * comp_bytes / (ms_per_step / 1e3) / 1e6, 1),
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(rec), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    for d in decs:
        d.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
