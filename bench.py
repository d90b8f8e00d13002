#!/usr/bin/env python3
"""Benchmark of the shot-boundary clip-splitting hot path (§2.1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one pass of the whole hot path (rows a1-a9: K1 histograms, K2 cuts,
K3 merge, result copy-back) over one batch of synthetic input through the
C ABI call clip_run_videos.  Workload (BASELINE.json configs[1], "C2"): one
10-minute 720p 30 fps video (18,000 frames, 49.8 GB of RGB24) per GPU,
resident in HBM (weak scaling: every rank scans its own copy of the C2 video,
so the per-GPU work is identical at every N; N > 1 gathers
the per-rank cut lists to rank 0 with one NCCL all-gather).  Prints ONE JSON
line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decoded frames/sec & HBM GB/s (fraction of peak) at 1/2/4/8 B200 vs CPU oracle"
HIST_BYTES = 162 * 4


KERNEL_SOURCES = {"k1": ["hist.cu", "binfn.cuh", "common.cuh"],
                  "k1_nv12": ["hist_nv12.cu", "binfn.cuh", "common.cuh"]}


def kernel_src_sha(kind: str) -> str:
    """sha256 (16 hex) of the kernel's source files: ties an ncu traffic file to
    the code it was captured from (the GPU box has no .git)."""
    import hashlib
    h = hashlib.sha256()
    for f in KERNEL_SOURCES[kind]:
        with open(os.path.join(ROOT, "paper_2503_12964_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def traffic_file(kind: str):
    """(dram bytes per algorithmic byte, thread-instr/px, note) from
    profiles/<kind>_traffic.json if it was captured from the current sources."""
    path = os.path.join(ROOT, "profiles", f"{kind}_traffic.json")
    if not os.path.exists(path):
        return None, None, "no capture"
    try:
        tr = json.load(open(path))
    except Exception:
        return None, None, "unreadable capture"
    if tr.get("src_sha") != kernel_src_sha(kind):
        return None, None, f"stale capture ({path}: src_sha {tr.get('src_sha')} != {kernel_src_sha(kind)})"
    return tr["dram_bytes_per_alg_byte"], tr.get("thread_instr_per_px"), tr.get("source")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every ~20 ms through
    NVML (nvidia-smi fallback) during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown"}

    def __init__(self, index: int, period: float = 0.02):
        self.index = index
        self.period = period
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            self.mx.append(mx)
            try:
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
            self._stop.wait(self.period)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.check_output(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                               "--format=csv,noheader,nounits"], text=True, timeout=5)
                r = [x.strip() for x in out.strip().split(",")]
                self.sm.append(float(r[0]))
                self.mx.append(float(r[1]))
                for i, n in enumerate(names):
                    if r[2 + i].lower().startswith("active"):
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            try:
                self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        # NVML initialisation can take longer than a short timed region: wait
        # for the sampler's first reading before the region starts
        t0 = time.time()
        while not self.sm and time.time() - t0 < 10.0 and self._t.is_alive():
            time.sleep(0.005)
        self._n0 = len(self.sm)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        # keep the readings taken inside the region (the last pre-region one if
        # the region was shorter than one period)
        n0 = max(0, getattr(self, "_n0", 1) - 1)
        self.sm, self.mx = self.sm[n0:], self.mx[n0:]

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ---------------------------------------------------------------- CPU oracle leg
def oracle_sample(frames_per_step: int, steps: int, warmup: int):
    """Time the oracle (oracle/, as it stands) on the first frames of the C2
    video on the host's cores; returns frames/s over the timed steps."""
    import numpy as np
    import oracle
    import synth
    from synth import manifest
    oracle.build()
    synth.build(device=False)
    v = manifest.subsample(manifest.c2_video(0), frames_per_step)
    cores = len(os.sched_getaffinity(0))
    frames = synth.gen_frames(v, nthreads=cores)  # generation is not timed
    emb = synth.gen_emb(v)
    times = []
    res = None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        res = oracle.run_video(frames, emb, nthreads=cores)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    fps = frames_per_step * len(times) / sum(times)
    return fps, cores, res, np


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = args.ref_frames
    fps, cores, _, _ = oracle_sample(n, args.steps, args.warmup)
    sample = f"first {n} frames of the C2 video (1280x720) per step; all rows a1-a9; frame generation untimed"
    line = {
        "metric": METRIC, "value": round(fps, 3), "unit": "frames/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000.0 * n / fps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C2: 10-min 720p 30fps synthetic video per GPU (BASELINE.json configs[1])",
                   "sample": sample},
        "cpu_baseline": {"value": round(fps, 3), "unit": "frames/s", "cores": cores,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(fps, 3), "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our path
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from synth import manifest, torch_dev
    from paper_2503_12964_b200 import Ctx
    from paper_2503_12964_b200 import dist as cdist
    from paper_2503_12964_b200.clipdetect import FORMAT_NV12, FORMAT_RGB24

    nv12 = args.format == "nv12"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    synth.build(device=True)

    # ---- workload: one C2-shaped video per rank, resident in HBM
    v = manifest.c2_video(0)  # every rank: its own resident copy of the C2 video
    if args.frames:
        v = manifest.subsample(v, args.frames)
    table = torch_dev.frame_table(v, dev)
    if nv12:  # NEXT f1: the decoder's NV12 surfaces (reading O0), 1.5 B/px
        frames = torch.empty((v.n, v.H * 3 // 2, v.W), dtype=torch.uint8, device=dev)
        torch_dev.gen_nv12(v, table, frames)
    else:
        frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
        torch_dev.gen_frames(v, table, frames)
    emb = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, table, emb)
    torch.cuda.synchronize()
    fbytes = frames[0].numel()
    frame_bytes = v.n * fbytes
    fmt = FORMAT_NV12 if nv12 else FORMAT_RGB24
    item = [{"n": v.n, "H": v.H, "W": v.W, "frames": frames, "emb": emb, "id": rank, "format": fmt}]

    stream = torch.cuda.Stream(device=dev)
    ctx = Ctx(device=local, stream=stream, timing=True)
    cap = cdist.capacity_ints([v.n], 8)
    gathered = [None]
    gather_wall = [0.0]

    def step():
        with torch.cuda.stream(stream):
            res = ctx.run_videos(item)[0]
            if world > 1 and not args.no_gather:
                # the one collective: all cut lists to every rank (ncclAllGather)
                t0 = time.perf_counter()
                gathered[0] = cdist.gather_results([res], cap, device=dev)
                gather_wall[0] += time.perf_counter() - t0
        return res

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    ctx.stats(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            res = step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    st = ctx.stats(reset=True)
    per_rank_ms = [ms / args.steps]
    per_rank_k1 = [st["k1_ms"] / args.steps]
    gather_ms = 1000.0 * gather_wall[0] / max(1, args.steps + args.warmup)
    if world > 1:
        t = torch.tensor([ms, st["k1_ms"]], dtype=torch.float64, device=dev)
        allt = torch.empty(2 * world, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(allt, t)
        allt = allt.view(world, 2).cpu().tolist()
        per_rank_ms = [x[0] / args.steps for x in allt]
        per_rank_k1 = [x[1] / args.steps for x in allt]
        ms_max = max(x[0] for x in allt)
    else:
        ms_max = ms
    ms_step = ms_max / args.steps

    # ---- read ceiling of K1's TMA pipeline on the same frames (K6, no binning)
    read_gbs = None
    if not args.no_read_ceiling:
        read_fn = ctx.debug_read_roofline_nv12 if nv12 else ctx.debug_read_roofline
        with torch.cuda.stream(stream):
            read_fn(frames)
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record(stream)
            for _ in range(3):
                read_fn(frames)
            r1.record(stream)
        torch.cuda.synchronize()
        read_gbs = frame_bytes / (r0.elapsed_time(r1) / 3 * 1e-3) / 1e9
        ctx.stats(reset=True)

    # ---- NEXT f3: K4 frame sampling + resize of the final clips (k per clip, 224x224)
    f3 = None
    if args.sample_k > 0 and not nv12:
        cuts_d = torch.from_numpy(res.final.astype(np.int32)).to(dev)
        S = 224
        with torch.cuda.stream(stream):
            out_s = torch.empty(((cuts_d.numel() + 1) * args.sample_k, S, S, 3), dtype=torch.uint8, device=dev)
            for _ in range(3):
                ctx.sample_frames(frames, cuts_d, args.sample_k, S, S, out=out_s, want_index=False)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(10):
                ctx.sample_frames(frames, cuts_d, args.sample_k, S, S, out=out_s, want_index=False)
            s1.record(stream)
        torch.cuda.synchronize()
        k4_ms = s0.elapsed_time(s1) / 10
        ctx.stats(reset=True)
        # algorithmic bytes per output frame: the distinct source rows the bilinear taps
        # touch (O11 row coordinates) + the output frame
        def src_rows(src, dst):
            sc = 1.0 / (dst / src)
            rows = set()
            for d in range(dst):
                f = float(np.float32((d + 0.5) * sc - 0.5))
                y = int(np.floor(f))
                y = min(max(y, 0), src - 1)
                rows.update({y, min(y + 1, src - 1)})
            return len(rows)
        m = out_s.shape[0]
        alg = m * (src_rows(v.H, S) * 3 * v.W + S * S * 3)
        f3 = {"kernel": "k4_sample_kernel", "clips": int(cuts_d.numel() + 1), "k": args.sample_k,
              "out": f"{S}x{S}", "launch_ms": round(k4_ms, 4),
              "frames_out_per_s": round(m / (k4_ms * 1e-3), 1),
              "roofline": {"bound": "hbm", "achieved": round(alg / (k4_ms * 1e-3) / 1e9, 1),
                           "unit": "GB/s", "alg_bytes_per_launch": alg}}
        del out_s

    # ---- parity of the timed results against the oracle golden (rank 0's video is C2 video 0)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", "C2_NV12.json" if nv12 else "C2.json")
    if rank == 0 and not args.frames and os.path.exists(gpath):
        g = json.load(open(gpath))["videos"][0]
        parity = (res.detected.tolist() == g["detected"] and res.final.tolist() == g["final"])
        if world > 1 and gathered[0] is not None:  # every rank's gathered cut lists
            parity = parity and len(gathered[0]) == world and all(
                d["detected"].tolist() == g["detected"] and d["final"].tolist() == g["final"]
                for d in gathered[0])

    # ---- e2e: host (pinned) frames through the same C ABI call, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = 64 << 30
        # pinned host copy of the video: at most ~35% of the free host RAM per rank
        n_e2e = max(1, min(v.n, args.e2e_frames, int(0.35 * avail / max(1, world) / fbytes)))
        host = torch.empty((n_e2e,) + tuple(frames.shape[1:]), dtype=torch.uint8, pin_memory=True)
        host.copy_(frames[:n_e2e])
        host_emb = torch.empty((n_e2e, manifest.EMB_DIM), dtype=torch.float32, pin_memory=True)
        host_emb.copy_(emb[:n_e2e])
        dev_emb = torch.empty_like(emb[:n_e2e])
        del frames
        torch.cuda.empty_cache()
        item_h = [{"n": n_e2e, "H": v.H, "W": v.W, "frames": host.numpy(), "emb": dev_emb, "id": rank,
                   "format": fmt}]

        def step_e2e():
            with torch.cuda.stream(stream):
                dev_emb.copy_(host_emb, non_blocking=True)
                return ctx.run_videos(item_h)[0]

        step_e2e()
        ctx.stats(reset=True)
        torch.cuda.synchronize()
        ne = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(ne):
            step_e2e()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / ne
        se = ctx.stats(reset=True)
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": round(world * n_e2e / dt, 3), "unit": "frames/s",
               "h2d_bytes_per_step": int(se["memcpy_h2d"] / ne + host_emb.numel() * 4),
               "d2h_bytes_per_step": int(se["memcpy_d2h"] / ne),
               "frames_per_step_per_gpu": n_e2e,
               "note": f"pinned host {'NV12' if nv12 else 'RGB24'} frames + embeddings copied H2D inside the timed region "
                       "(PCIe-bound); detected/final cut lists copied D2H"}

    # ---- worst-case content: K1 on uniform-noise 1080p frames (every rank; rank 0 reports)
    if "frames" in locals():
        del frames
    torch.cuda.empty_cache()
    noise = None if args.no_noise else k1_noise(dev, stream)

    # ---- north star's C3 strong scaling (64 x 1080p videos, 716.6 GB) at this N:
    # frames streamed through the device generator at EVERY N (one clock at every N)
    c3 = None
    if not args.no_c3:
        c3 = time_batch("C3", world, rank, dev, local, args.c3_steps, 1, force_stream=True)

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peak, peak_src = _peaks()
    k1_ms = st["k1_ms"] / max(1, st["k1_launches"])
    k1_alg = frame_bytes + v.n * HIST_BYTES
    achieved = k1_alg / (k1_ms * 1e-3) / 1e9
    ratio, instr_px, traffic_src = traffic_file("k1_nv12" if nv12 else "k1")
    traffic = None if ratio is None else int(ratio * k1_alg)
    fps = world * v.n / (ms_step * 1e-3)
    gbs = world * frame_bytes / (ms_step * 1e-3) / 1e9
    # the binding resource of K1 is instruction issue: issue roofline
    # = warp-instructions/s (ncu thread-instr/px of the committed capture x live px/s / 32)
    # against 4 schedulers x 1 warp-instr/clk x SMs x the sampled SM clock
    issue = None
    clk_sum = clk.summary()
    if instr_px and clk_sum.get("sm_mhz"):
        px_s = v.n * v.npix / (k1_ms * 1e-3)
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_wi = n_sm * 4 * clk_sum["sm_mhz"] * 1e6
        ach_wi = instr_px * px_s / 32.0
        issue = {"bound": "issue", "achieved": round(ach_wi / 1e9, 1), "peak": round(peak_wi / 1e9, 1),
                 "unit": "G warp-instr/s", "frac": round(ach_wi / peak_wi, 4),
                 "thread_instr_per_px": instr_px, "sms": n_sm, "sm_mhz": clk_sum["sm_mhz"]}

    cpu = None
    if world == 1 and not args.no_cpu:
        n_cpu = args.ref_frames
        cfps, cores, _, _ = oracle_sample(n_cpu, 1, 0)
        cpu = {"value": round(cfps, 3), "unit": "frames/s", "cores": cores, "kind": "oracle",
               "sample": f"first {n_cpu} frames of the C2 video (1280x720), rows a1-a9, "
                         f"generation untimed, oracle threads over frames for O2"}

    line = {
        "metric": METRIC, "value": round(fps, 3), "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": ("C2 as NV12 surfaces (18,000 720p frames, 24.9 GB NV12; NEXT f1, reading O0) "
                                "per GPU, resident in HBM" if nv12 else
                                "C2: 10-min 720p 30fps synthetic video (18,000 frames, 49.8 GB RGB24) "
                                "per GPU, resident in HBM (BASELINE.json configs[1])"),
                   "format": "nv12" if nv12 else "rgb24",
                   "frames_per_gpu": v.n, "resolution": f"{v.W}x{v.H}", "emb_dim": manifest.EMB_DIM,
                   "l2": f"inputs larger than L2 ({frame_bytes / 1e9:.1f} GB per GPU vs 126 MB), no flush needed",
                   "parallelism": f"whole-video sharding, {world} GPU(s), one NCCL all-gather of cut lists",
                   "weak_scaling_unit": "each rank scans its own resident copy of the C2 video"},
        "hbm_gbs": round(gbs, 1),
        "frac_of_measured_hbm": round(gbs / peak, 4),
        "frac_of_8tbs": round(gbs / 8000.0, 4),
        "read_ceiling_gbs": None if read_gbs is None else round(read_gbs, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": "k1_nv12_kernel" if nv12 else "k1_hist_kernel",
                     "alg_bytes_per_launch": k1_alg, "launch_ms": round(k1_ms, 4), "peak_src": peak_src,
                     "frac_of_read_ceiling": None if read_gbs is None else round(achieved / read_gbs, 4),
                     "frac_of_8tbs": round(achieved / 8000.0, 4), "instr_per_px_ncu": instr_px,
                     "traffic_src": traffic_src},
        "roofline_issue": issue,
        "kernel_ms_per_step": {"k1": round(st["k1_ms"] / args.steps, 4),
                               "k2": round(st["k2_ms"] / args.steps, 4),
                               "k3": round(st["k3_ms"] / args.steps, 4)},
        "gpu_launches": int(st["launches"]),
        "per_rank_ms_per_step": [round(x, 4) for x in per_rank_ms],
        "per_rank_k1_ms_per_step": [round(x, 4) for x in per_rank_k1],
        "gather_wall_ms_per_step_rank0": round(gather_ms, 4) if world > 1 else None,
        "clocks": clk_sum,
        "parity_vs_golden": parity,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    line["k1_noise"] = noise
    line["c3_strong"] = c3
    if f3 is not None:
        f3["roofline"]["peak"] = peak
        f3["roofline"]["frac"] = round(f3["roofline"]["achieved"] / peak, 4)
        line["f3_sample"] = f3
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------- batch configs (C3/C4/C5)
def time_batch(name, world, rank, dev, local, steps, warmup, resident_gb=150.0,
               force_stream=False, max_videos=0):
    """One config's videos LPT-sharded by whole video over the ranks (strong
    scaling: the batch is fixed) and timed the same way at every N.

    Frames are resident in HBM when the LARGEST rank share fits in
    `resident_gb` (every rank knows every share: no collective) and
    `force_stream` is off; otherwise EVERY rank streams its frames chunk by
    chunk through clip_run_videos' fill callback (the device generator writes
    each chunk into the library's staging buffer on the ctx stream: synthetic
    "decode" inside the step).  Two clocks, both max over ranks: `wall` = CUDA
    events around whole steps (clip_run_videos + the one all-gather of the cut
    lists), `kernel` = the library's CUDA events around K1 + K2 + K3."""
    import torch
    import torch.distributed as dist

    import synth
    from synth import manifest, torch_dev
    from paper_2503_12964_b200 import Ctx
    from paper_2503_12964_b200 import dist as cdist

    vids = manifest.config_videos(name)
    if max_videos:
        vids = vids[:max_videos]
    assign = cdist.lpt_assign([v.n * v.W * v.H for v in vids], world)
    share = [sum(vids[i].n * vids[i].frame_bytes for i in a) for a in assign]
    resident = (not force_stream) and max(share) <= resident_gb * 1e9
    mine = [vids[i] for i in assign[rank]]
    tables = [torch_dev.frame_table(v, dev) for v in mine]
    items = []
    for v, t in zip(mine, tables):
        e = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
        torch_dev.gen_emb(v, t, e)
        f = None
        if resident:
            f = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
            torch_dev.gen_frames(v, t, f)
        items.append({"n": v.n, "H": v.H, "W": v.W, "frames": f, "emb": e, "id": v.id})
    torch.cuda.synchronize()

    def fill(vi, t0, n, dst, stream):
        v = mine[vi]
        return synth.dev_lib().synth_dev_gen_frames(v.seed, v.id, v.W, v.H, t0, n,
                                                    tables[vi].data_ptr(), dst, stream)

    stream = torch.cuda.Stream(device=dev)
    ctx = Ctx(device=local, stream=stream, timing=True)
    cap = cdist.capacity_ints([v.n for v in vids], 8)
    out = [None]
    gather_s = [0.0]

    def step():
        with torch.cuda.stream(stream):
            res = ctx.run_videos(items, fill=None if resident else fill) if items else []
            if world > 1:
                t0 = time.perf_counter()
                out[0] = cdist.gather_results(res, cap, device=dev)
                gather_s[0] += time.perf_counter() - t0
            else:
                out[0] = [{"id": r.id, "detected": r.detected, "final": r.final} for r in res]

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ctx.stats(reset=True)
    gather_s[0] = 0.0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = ctx.stats(reset=True)
    mine_t = [e0.elapsed_time(e1) / steps, (st["k1_ms"] + st["k2_ms"] + st["k3_ms"]) / steps,
              st["k1_ms"] / steps, 1000.0 * gather_s[0] / steps]
    if world > 1:
        t = torch.tensor(mine_t, dtype=torch.float64, device=dev)
        allt = torch.empty(world * 4, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(allt, t)
        allt = allt.view(world, 4).cpu().tolist()
    else:
        allt = [mine_t]
    wall = max(r[0] for r in allt)
    kern = max(r[1] for r in allt)
    total_frames = sum(v.n for v in vids)
    total_bytes = sum(v.n * v.frame_bytes for v in vids)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", f"{name.upper()}.json")
    if rank == 0 and os.path.exists(gpath) and out[0] is not None:
        gold = {g["id"]: g for g in json.load(open(gpath))["videos"]}
        got = {d["id"]: d for d in out[0]}
        parity = len(got) == len(vids) and all(
            list(got[v.id]["detected"]) == gold[v.id]["detected"] and list(got[v.id]["final"]) == gold[v.id]["final"]
            for v in vids)
    k1_alg = sum(v.n * (v.frame_bytes + HIST_BYTES) for v in mine)
    del items
    ctx.close()
    torch.cuda.empty_cache()
    return {
        "workload": f"{name.upper()} (BASELINE.json configs): {len(vids)} videos, {total_frames} frames, "
                    f"{total_bytes / 1e9:.1f} GB",
        "frames": total_frames, "frame_bytes": total_bytes, "videos": len(vids),
        "value_wall": round(total_frames / (wall * 1e-3), 3),
        "value_kernel": round(total_frames / (kern * 1e-3), 3),
        "unit": "frames/s", "scaling": "strong",
        "wall_ms_per_step": round(wall, 4), "kernel_ms_per_step": round(kern, 4),
        "per_rank_wall_ms": [round(r[0], 4) for r in allt],
        "per_rank_k1_ms": [round(r[2], 4) for r in allt],
        "gather_wall_ms_per_step": [round(r[3], 4) for r in allt] if world > 1 else None,
        "frames_source": "resident in HBM" if resident else
                         "streamed at every rank: device generator fills the staging buffer per chunk "
                         "(inside the wall clock, outside the kernel clock)",
        "lpt_imbalance_max_over_mean": round(max(share) / (sum(share) / world), 4),
        "k1_gbs_rank0": round(k1_alg / (mine_t[2] * 1e-3) / 1e9, 1) if mine_t[2] > 0 else None,
        "parity_vs_golden": parity, "steps": steps, "warmup": warmup, "clocks": clk.summary(),
        "gpu_launches_rank0": int(st["launches"]),
    }


def run_config(args):
    """--config C3|C4|C5: strong scaling of the config's fixed batch (time_batch)."""
    import torch
    import torch.distributed as dist

    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    synth.build(device=True)
    b = time_batch(args.config, world, rank, dev, local, args.steps, args.warmup,
                   resident_gb=args.resident_gb, force_stream=args.stream_frames,
                   max_videos=args.max_videos)
    if rank == 0:
        peak, _ = _peaks()
        ms = b["wall_ms_per_step"]
        line = {
            "metric": METRIC, "value": b["value_wall"], "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": b["workload"], "frames_source": b["frames_source"],
                       "parallelism": f"LPT whole-video sharding over {world} GPU(s), one NCCL all-gather",
                       "timing": "value = CUDA events around whole steps (max over ranks); "
                                 "value_kernel = library events around K1+K2+K3"},
            "hbm_gbs": round(b["frame_bytes"] / (ms * 1e-3) / 1e9, 1),
            "frac_of_measured_hbm": round(b["frame_bytes"] / (ms * 1e-3) / 1e9 / peak, 4),
            "batch": b, "gpu_launches": b["gpu_launches_rank0"], "clocks": b["clocks"],
            "parity_vs_golden": b["parity_vs_golden"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def k1_noise(dev, stream, n: int = 1500):
    """K1 on uniform-random-colour 1080p frames (C3 shape; every pixel its own
    code: the worst case for the shared-memory atomics and hue-table banks,
    SURVEY.md §8(d) "never quote only the friendly content")."""
    import torch

    from synth import manifest, torch_dev
    from paper_2503_12964_b200 import Ctx
    v = manifest.noise_video(0, 1920, 1080, n)
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    ctx = Ctx(device=dev.index, stream=stream, timing=True)
    with torch.cuda.stream(stream):
        ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)
        torch.cuda.synchronize()
        ctx.stats(reset=True)
        for _ in range(3):
            ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)
    torch.cuda.synchronize()
    st = ctx.stats(reset=True)
    ms = st["k1_ms"] / 3
    alg = v.n * (v.frame_bytes + HIST_BYTES)
    ctx.close()
    del frames, hist
    torch.cuda.empty_cache()
    peak, _ = _peaks()
    return {"workload": f"uniform-noise frames {v.W}x{v.H} x {v.n} ({v.n * v.frame_bytes / 1e9:.1f} GB, resident)",
            "kernel": "k1_hist_kernel", "launch_ms": round(ms, 4),
            "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "unit": "GB/s", "peak": peak,
            "frac": round(alg / (ms * 1e-3) / 1e9 / peak, 4), "frac_of_8tbs": round(alg / (ms * 1e-3) / 8e12, 4)}


# ---------------------------------------------------------------- one video split by frames (f2)
def run_shard_frames(args):
    """--shard-frames: the C2 video split into contiguous frame ranges over the
    ranks (strong scaling of ONE long video).  Exchanges:
    last histograms, L1 arrays and embeddings, each one NCCL all-gather."""
    import torch
    import torch.distributed as dist

    import synth
    from synth import manifest, torch_dev
    from paper_2503_12964_b200 import Ctx
    from paper_2503_12964_b200 import dist as cdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29599")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    else:
        dist.init_process_group("nccl", device_id=dev)
    synth.build(device=True)
    v = manifest.c2_video(0)
    if args.frames:
        v = manifest.subsample(v, args.frames)
    a, b = cdist.frame_shards(v.n, world)[rank]
    table = torch_dev.frame_table(v, dev)
    nv12 = args.format == "nv12"
    if nv12:
        frames = torch.empty((b - a, v.H * 3 // 2, v.W), dtype=torch.uint8, device=dev)
        torch_dev.gen_nv12(v, table, frames, t0=a, n=b - a)
    else:
        frames = torch.empty((b - a, v.H, v.W, 3), dtype=torch.uint8, device=dev)
        torch_dev.gen_frames(v, table, frames, t0=a, n=b - a)
    emb = torch.empty((b - a, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, table, emb, t0=a, n=b - a)
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=dev)
    ctx = Ctx(device=local, stream=stream, timing=True)
    out = [None]

    def step():
        with torch.cuda.stream(stream):
            out[0] = cdist.run_video_sharded(ctx, frames, emb, v.n, a)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.stats(reset=True)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    st = ctx.stats(reset=True)
    # one extra (untimed) step with CUDA events between the phases of the exchange
    marks = []
    with torch.cuda.stream(stream):
        cdist.run_video_sharded(ctx, frames, emb, v.n, a, marks=marks)
    torch.cuda.synchronize()
    phase_ms = [round(marks[i].elapsed_time(marks[i + 1]), 4) for i in range(len(marks) - 1)]
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    allt = torch.empty(world, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(allt, t)
    per_rank = allt.cpu().tolist()
    ms = max(per_rank)
    if rank == 0:
        parity = None
        gpath = os.path.join(ROOT, "tests", "golden", "C2_NV12.json" if nv12 else "C2.json")
        if not args.frames and os.path.exists(gpath):
            g = json.load(open(gpath))["videos"][0]
            parity = out[0][0] == g["detected"] and out[0][1] == g["final"]
        line = {
            "metric": METRIC, "value": round(v.n / (ms * 1e-3), 3), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": "C2: ONE 10-min 720p video split by frame ranges over the GPUs (SURVEY f2)"
                                   + (", NV12 surfaces (f1)" if nv12 else ""),
                       "format": args.format,
                       "frames": v.n, "frames_per_gpu": b - a,
                       "parallelism": f"frame-range sharding over {world} GPU(s); NCCL all-gathers of "
                                      "last histograms, L1 arrays and embeddings"},
            "hbm_gbs": round(v.n * frames[0].numel() / (ms * 1e-3) / 1e9, 1),
            "per_rank_ms_per_step": [round(x, 4) for x in per_rank],
            "k1_ms_per_step_rank0": round(st["k1_ms"] / args.steps, 4),
            "phase_ms_rank0": dict(zip(["scan (K1+L1)", "seam (all-gather lasts, a4)",
                                        "L1 all-gather + cuts", "embeddings wait + concat",
                                        "merge"], phase_ms)),
            "gpu_launches": int(st["launches"]), "clocks": clk.summary(), "parity_vs_golden": parity,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=0, help="debug: truncate the C2 video")
    ap.add_argument("--ref-frames", type=int, default=2400, help="oracle sample frames per step")
    ap.add_argument("--e2e-frames", type=int, default=18000)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gather", action="store_true", help="diagnosis: skip the result all-gather")
    ap.add_argument("--no-read-ceiling", action="store_true")
    ap.add_argument("--config", default="", help="C3|C4|C5: strong-scaling batch run")
    ap.add_argument("--sample-k", type=int, default=8,
                    help="NEXT f3: also time K4 (k frames per final clip -> 224x224); 0 = off")
    ap.add_argument("--format", default="rgb24", choices=["rgb24", "nv12"],
                    help="frame format of the C2 run (nv12 = NEXT f1, fused NV12 kernel)")
    ap.add_argument("--max-videos", type=int, default=0)
    ap.add_argument("--resident-gb", type=float, default=150.0)
    ap.add_argument("--shard-frames", action="store_true",
                    help="split the C2 video by frame ranges over the GPUs (strong scaling)")
    ap.add_argument("--stream-frames", action="store_true",
                    help="--config: stream frames through the device generator at every N")
    ap.add_argument("--no-noise", action="store_true", help="skip the uniform-noise K1 figure")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 strong-scaling figure")
    ap.add_argument("--c3-steps", type=int, default=2)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch: one process per GPU under torch.distributed.run (NCCL)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl != "reference" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.config:
        return run_config(args)
    if args.shard_frames:
        return run_shard_frames(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
