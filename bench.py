#!/usr/bin/env python
"""bench.py -- megapixels/s of the ImageCL hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl icl|reference]
                    [--workload suite|sepconv16k|conv2d8k|sep3d|chain] [--batch B] [--size S] [--radius R]

Default workload ("suite", BASELINE.json configs[4] per GPU): every rank
processes its own batch of B (default 8) synthetic 4096x4096 fp32 images
through the whole hot path each step -- separable Gaussian convolution
(r=2, constant 0), Harris (3x3 Sobel, 5x5 window, k=0.04, clamp, + mask) and
NLM (5x5 patch, 11x11 search, h=0.1, clamp).  Weak scaling: at N=8 the job is
the 64-image configs[4].  Inputs (3 x 512 MiB per rank) are larger than L2,
so no flush is needed between steps.

``value`` = whole-job suite throughput (pixels that went through all three
filters per second, summed over ranks, Mpx/s).  ``e2e`` = the same through the
public API with pinned HOST buffers (H2D of the step's inputs and D2H of all
outputs inside the timed region).  ``roofline`` is for the dominant kernel
(NLM, FP32-bound); ``rooflines`` lists all three.  ``cpu_baseline`` times the
double-precision oracle (oracle/) on a bounded pixel sample on this host.

``--impl reference``: the reference arm is the CPU oracle (no runnable
reference implementation exists -- the reference is a paper), timed on the
host cores on a bounded sample per step; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # DESIGN.md "FP32 roof" (74.4 TFLOP/s)
NLM_FLOP_PER_PAIR = {"direct": 79, "boxsum": 14}     # SURVEY.md §8(d), DESIGN.md "NLM flops"
SEP_BYTES_PER_PX = 8
HARRIS_BYTES_PER_PX = 9                               # in + R (4+4) + uint8 mask


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# variant -> kernel-name fragments (to attach ncu counters only to the kernel they were measured on)
# (the S = segment-rows variants of one family launch the same kernel function)
KERNEL_OF = {"sym_tmem": ("nlm_sym<2, 5, 0, 4>", "nlm_sym<2, 5, false, 4>", "nlm_sym<2, 5>"),
             "sym_ring": ("nlm_sym<2, 5, 1, 4>", "nlm_sym<2, 5, true, 4>"),
             "sym_tmem8": ("nlm_sym<2, 5, 0, 8>", "nlm_sym<2, 5, false, 8>"), "boxsum_x2": ("nlm_box_x2",), "boxsum_r8": ("nlm_box_r8",),
             **{f"stream_nt64_s{s}_v4": ("sep_stream<2, 64",) for s in (16, 32, 64, 128)},
             **{f"tma_nt32_s{s}_v4": ("sep_stream_tma<2, 32",) for s in (16, 32, 64, 128)},
             **{f"shfl_nw2_s{s}": ("harris_shfl<5, 2>",) for s in (8, 16, 32, 64, 128)},
             **{f"shfl_tma_nw2_s{s}": ("harris_shfl_tma<5, 2>",) for s in (8, 16, 32)}}


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


def _traffic(t, f, px):
    """ncu DRAM bytes per launch of this bench's launch size (from profiles/ncu_traffic.json)."""
    e = t.get(f)
    if not e or "bytes_per_px" not in e:
        return None
    return e["bytes_per_px"] * px


def link_bandwidth(dev, nbytes=256 << 20):
    """Pinned host <-> device copy rate with both directions in flight at once
    (the roofline of the e2e step, whose H2D and D2H overlap): GB/s each way."""
    import torch
    h_src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(2)]
    for rep in range(2):  # warm-up, then timed
        torch.cuda.synchronize(dev)
        ev[0][0].record(s1)
        ev[1][0].record(s2)
        with torch.cuda.stream(s1):
            for _ in range(3):
                d_a.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            for _ in range(3):
                h_dst.copy_(d_b, non_blocking=True)
        ev[0][1].record(s1)
        ev[1][1].record(s2)
        torch.cuda.synchronize(dev)
    t_h2d = ev[0][0].elapsed_time(ev[0][1]) / 3
    t_d2h = ev[1][0].elapsed_time(ev[1][1]) / 3
    return {"concurrent_h2d_GBps": nbytes / t_h2d / 1e6, "concurrent_d2h_GBps": nbytes / t_d2h / 1e6,
            "measured": "pinned copies, both directions in flight, 256 MiB x 3 each"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 10 ms) during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _poll(self):
        nv = self.nv
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake_slowdown"}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, n in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join(1.0)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "sm_mhz_min": min(self.samples)}


# ----------------------------------------------------------------------------- distributed
# ICL_BENCH_ONE_GPU=1: every rank on cuda:0 with a gloo group -- a functional check of the
# multi-rank code paths on a one-GPU box (timings are then meaningless; never a bench number)
ONE_GPU = os.environ.get("ICL_BENCH_ONE_GPU") == "1"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if ONE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def init_dist(ws, backend):
    import torch.distributed as dist
    if ws > 1:
        # NCCL's init lines ("... nRanks N ...") stay visible on stderr, so a reader can check the
        # communicator sizes the run really used
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo" if ONE_GPU else backend)
    return dist


def max_over_ranks(x: float, ws: int, device) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if ONE_GPU else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- workload
SUITE = dict(sep_r=2, sep_border="constant", har_block=5, har_k=0.04, har_border="clamp", nlm_P=2, nlm_S=5,
             nlm_h=0.1, nlm_border="clamp")


def gen_inputs(rank, batch, size):
    """Per-rank host inputs (numpy, fp32): uniform (sepconv), rect scenes (Harris, NLM)."""
    u = np.empty((batch, size, size), np.float32)
    hs = np.empty_like(u)
    ns = np.empty_like(u)
    for i in range(batch):
        seed = rank * batch + i
        u[i] = synth.uniform_image(1000 + seed, size, size)
        hs[i] = synth.rect_scene(2000 + seed, size, size, n_rect=256, noise=0.01)
        ns[i] = synth.rect_scene(3000 + seed, size, size, n_rect=256, noise=0.0866)
    return u, hs, ns


def cpu_oracle_sample(inputs, size, target_s=8.0, threads=0):
    """Time the oracle on a bounded random pixel sample of the suite workload."""
    import oracle
    u, hs, ns = inputs
    rng = np.random.default_rng(0)
    fx = synth.gaussian_taps(SUITE["sep_r"])
    c = SUITE

    def run(n):
        ys, xs = rng.integers(0, size, n), rng.integers(0, size, n)
        t = {}
        t0 = time.perf_counter()
        oracle.sepconv(u[0], fx, fx, c["sep_border"], points=(xs, ys), threads=threads)
        t["sepconv"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.harris(hs[0], c["har_block"], c["har_k"], c["har_border"], points=(xs, ys), threads=threads)
        t["harris"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.nlm(ns[0], c["nlm_P"], c["nlm_S"], c["nlm_h"], c["nlm_border"], points=(xs, ys), threads=threads)
        t["nlm"] = time.perf_counter() - t0
        return t

    n = 2048
    t = run(n)
    tot = sum(t.values())
    n = int(min(1 << 24, max(2048, n * target_s / max(tot, 1e-3))))
    t = run(n)
    tot = sum(t.values())
    return n, t, tot


def cpu_model() -> str:
    """Host CPU model (record it beside the oracle baseline)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    size = args.size
    threads = oracle.default_threads()
    inputs = tuple(a[:1] for a in gen_inputs(0, 1, size))
    fx = synth.gaussian_taps(SUITE["sep_r"])
    c = SUITE
    rng = np.random.default_rng(1)
    u, hs, ns = inputs

    def step(n):
        ys, xs = rng.integers(0, size, n), rng.integers(0, size, n)
        oracle.sepconv(u[0], fx, fx, c["sep_border"], points=(xs, ys), threads=threads)
        oracle.harris(hs[0], c["har_block"], c["har_k"], c["har_border"], points=(xs, ys), threads=threads)
        oracle.nlm(ns[0], c["nlm_P"], c["nlm_S"], c["nlm_h"], c["nlm_border"], points=(xs, ys), threads=threads)

    t0 = time.perf_counter()
    step(1024)
    dt = time.perf_counter() - t0
    budget = 150.0 / max(1, args.steps + args.warmup)  # whole run within a few minutes
    n = int(min(1 << 20, max(256, 1024 * min(budget, 4.0) / max(dt, 1e-4))))
    for _ in range(args.warmup):
        step(n)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(n)
    el = time.perf_counter() - t0
    value = args.steps * n / el / 1e6
    sample = f"{n} random pixels per step of one {size}x{size} image, each through sepconv+Harris+NLM (oracle, f64)"
    line = {
        "impl": "reference", "metric": "suite megapixels/s (sepconv r2 + Harris B5 + NLM 5x5/11x11)",
        "value": value, "unit": "Mpx/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "suite", "images_per_gpu": args.batch, "size": [size, size], **SUITE},
        "cpu_baseline": {"value": value, "unit": "Mpx/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "Mpx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- icl arm: suite
def run_suite(args):
    import torch

    import paper_1605_06399_b200 as icl
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(ws, "nccl")
    icl.load_library()
    B, S = args.batch, args.size
    t_gen = time.perf_counter()
    u_h, hs_h, ns_h = gen_inputs(rank, B, S)
    t_gen = time.perf_counter() - t_gen
    u = torch.from_numpy(u_h).to(dev)
    hs = torch.from_numpy(hs_h).to(dev)
    ns = torch.from_numpy(ns_h).to(dev)
    o_sep = torch.empty_like(u)
    o_har = torch.empty_like(u)
    o_mask = torch.empty(B, S, S, dtype=torch.uint8, device=dev)
    o_nlm = torch.empty_like(u)
    fx = synth.gaussian_taps(SUITE["sep_r"])
    c = SUITE
    stream = torch.cuda.Stream(device=dev)
    thr = 1.0  # absolute threshold on R (R10)

    # auto-tune once per shape (untimed), §4: the winner is cached.
    tuned = {}
    with torch.cuda.stream(stream):
        if not args.no_tune:
            tuned["sepconv"] = icl.tune("sepconv", u, o_sep, taps_x=fx, taps_y=fx, border=c["sep_border"],
                                        stream=stream)
            tuned["harris"] = icl.tune("harris", hs, o_har, block=c["har_block"], k=c["har_k"],
                                       border=c["har_border"], mask=o_mask, threshold=thr, stream=stream)
            tuned["nlm"] = icl.tune("nlm", ns, o_nlm, patch_radius=c["nlm_P"], search_radius=c["nlm_S"],
                                    h=c["nlm_h"], border=c["nlm_border"], stream=stream)
    stream.synchronize()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        icl.sepconv(u, o_sep, fx, fx, c["sep_border"], stream=stream)
        if ev:
            ev[1].record(stream)
        icl.harris(hs, o_har, c["har_block"], c["har_k"], c["har_border"], mask=o_mask, threshold=thr,
                   stream=stream)
        if ev:
            ev[2].record(stream)
        icl.nlm(ns, o_nlm, c["nlm_P"], c["nlm_S"], c["nlm_h"], c["nlm_border"], stream=stream)
        if ev:
            ev[3].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    stream.synchronize()
    variants = {f: icl.variant_names(f)[icl.last_variant(f)] for f in ("sepconv", "harris", "nlm")}
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    n0 = icl.launch_count()
    with ClockSampler(local) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        end.record(stream)
        stream.synchronize()
    launches = icl.launch_count() - n0
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    total_ms = start.elapsed_time(end)
    per = {"sepconv": [], "harris": [], "nlm": []}
    for e in evs:
        per["sepconv"].append(e[0].elapsed_time(e[1]))
        per["harris"].append(e[1].elapsed_time(e[2]))
        per["nlm"].append(e[2].elapsed_time(e[3]))
    step_ms = max_over_ranks(total_ms / args.steps, ws, dev)
    px_rank = B * S * S
    value = ws * px_rank / (step_ms * 1e-3) / 1e6

    # ---------------- e2e: the same calls through the C ABI with HOST buffers
    # (pinned): the library streams row bands H2D -> kernel -> D2H with the
    # three stages of consecutive bands overlapped (include/icl.h, host images).
    e2e = None
    if not args.no_e2e:
        hu = torch.from_numpy(u_h).pin_memory()
        hh = torch.from_numpy(hs_h).pin_memory()
        hn = torch.from_numpy(ns_h).pin_memory()
        outs_h = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in (o_sep, o_har, o_mask, o_nlm)]
        ksteps = max(1, min(args.steps, 5))

        # the three independent filter calls are issued on three streams forked
        # from (and joined back into) the timing stream, so the bands of one
        # call's D2H overlap the next call's H2D in the library's pipeline
        fstreams = [torch.cuda.Stream(device=dev) for _ in range(3)]
        fork = [torch.cuda.Event() for _ in range(ksteps + 1)]

        def e2e_step(i=0):
            fork[i].record(stream)
            for fs in fstreams:
                fs.wait_event(fork[i])
            icl.sepconv(hu, outs_h[0], fx, fx, c["sep_border"], stream=fstreams[0])
            icl.harris(hh, outs_h[1], c["har_block"], c["har_k"], c["har_border"], mask=outs_h[2], threshold=thr,
                       stream=fstreams[1])
            icl.nlm(hn, outs_h[3], c["nlm_P"], c["nlm_S"], c["nlm_h"], c["nlm_border"], stream=fstreams[2])
            for fs in fstreams:
                stream.wait_stream(fs)

        with torch.cuda.stream(stream):
            e2e_step(ksteps)
            stream.synchronize()
            if ws > 1:
                dist.barrier()
            x0 = icl.transfer_bytes()
            a = torch.cuda.Event(enable_timing=True)
            bq = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i in range(ksteps):
                e2e_step(i)
            bq.record(stream)
            stream.synchronize()
            x1 = icl.transfer_bytes()
        e2e_ms = max_over_ranks(a.elapsed_time(bq) / ksteps, ws, dev)
        # bytes the library actually copied (inputs incl. band halo rows, outputs incl. mask)
        h2d = (x1[0] - x0[0]) // ksteps
        d2h = (x1[1] - x0[1]) // ksteps
        ok = all(np.array_equal(outs_h[i].numpy()[B - 1, ::997], o[B - 1, ::997].cpu().numpy())
                 for i, o in enumerate((o_sep, o_har, o_mask)))
        link = link_bandwidth(dev)
        bound_ms = max(h2d / link["concurrent_h2d_GBps"], d2h / link["concurrent_d2h_GBps"]) / 1e6
        link.update({"bound_ms_per_step": bound_ms, "frac": bound_ms / e2e_ms})
        e2e = {"value": ws * px_rank / (e2e_ms * 1e-3) / 1e6, "unit": "Mpx/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": ksteps, "link_roofline": link,
               "path": "C ABI with pinned host buffers (row bands, H2D/compute/D2H overlapped; the three "
                       "filter calls on three forked streams)",
               "matches_device_outputs": bool(ok)}

    # ---------------- rooflines (algorithmic work / per-launch device time)
    hbm, hbm_kind = measured_peaks()
    traffic = ncu_traffic()
    med = {f: statistics.median(v) for f, v in per.items()}
    # the symmetric kernel (sym_tmem) evaluates half the box sums; the roofline keeps the §8(d)
    # box-sum count of the full window (the algorithmic work)
    nlm_kind = "boxsum" if variants["nlm"].startswith(("boxsum", "sym_")) else "direct"
    P, Sr = c["nlm_P"], c["nlm_S"]
    pairs = (2 * Sr + 1) ** 2
    nlm_flop_px = pairs * (NLM_FLOP_PER_PAIR[nlm_kind] if nlm_kind == "boxsum" else
                           (2 * P + 1) ** 2 * 3 + 4)
    roof = {
        "nlm": {"bound": "alu", "achieved": nlm_flop_px * px_rank / (med["nlm"] * 1e-3) / 1e12,
                "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "flop_per_px": nlm_flop_px,
                "formulation": nlm_kind + (" (offset-symmetric: d_-o(p) = d_o(p-o), half the distances "
                                           "evaluated)" if variants["nlm"].startswith("sym_") else ""),
                "kernel": variants["nlm"],
                "traffic": _traffic(traffic, "nlm", px_rank)},
        "sepconv": {"bound": "hbm", "achieved": SEP_BYTES_PER_PX * px_rank / (med["sepconv"] * 1e-3) / 1e9,
                    "peak": hbm, "unit": "GB/s", "kernel": variants["sepconv"],
                    "traffic": _traffic(traffic, "sepconv", px_rank)},
        "harris": {"bound": "hbm", "achieved": HARRIS_BYTES_PER_PX * px_rank / (med["harris"] * 1e-3) / 1e9,
                   "peak": hbm, "unit": "GB/s", "kernel": variants["harris"],
                   "traffic": _traffic(traffic, "harris", px_rank)},
    }
    for r in roof.values():
        r["frac"] = r["achieved"] / r["peak"]
    roof["sepconv"]["frac_of_8TBs_spec"] = roof["sepconv"]["achieved"] / 8000.0
    roof["harris"]["frac_of_8TBs_spec"] = roof["harris"]["achieved"] / 8000.0
    roof["sepconv"]["peak_kind"] = roof["harris"]["peak_kind"] = hbm_kind
    roof["nlm"]["peak_kind"] = "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz"
    # ncu pipe counters of the profiled kernel (profiles/ncu_traffic.json), when it is the one timed here
    for f in roof:
        e = traffic.get(f) or {}
        kname = e.get("kernel", "")
        if e and any(k in kname for k in KERNEL_OF.get(roof[f]["kernel"], ())):
            roof[f]["ncu"] = {k: e.get(k) for k in ("fma_pipe_cycles_pct", "issue_active_pct", "smem_wavefronts_pct",
                                                    "mufu_pct")}
    roof["nlm"]["limiter"] = {
        "sym_tmem": "FP32 pipe: the H slide recomputes the row leaving the window (no register/TMEM room for a "
                    "ring); FFMA2s with three distinct register pairs issue at 2/3 rate; 8 warps/SM (TMEM: 256 "
                    "columns x 2 CTAs; 236 registers), DESIGN.md §5",
        "sym_ring": "FFMA2 chain latency at 4 warps/SM (the TMEM ring takes all 512 columns), DESIGN.md §5",
    }.get(variants["nlm"], "shared-memory wavefronts (two-phase separable box sums: H round trip + accumulation "
                           "loads, DESIGN.md §5)")
    dominant = max(med, key=med.get)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        n, t, tot = cpu_oracle_sample((u_h[:1], hs_h[:1], ns_h[:1]), S)
        n1, _, tot1 = cpu_oracle_sample((u_h[:1], hs_h[:1], ns_h[:1]), S, target_s=2.0, threads=1)
        cpu = {"value": n / tot / 1e6, "unit": "Mpx/s", "cores": oracle.default_threads(), "kind": "oracle",
               "cpu_model": cpu_model(), "value_1_thread": n1 / tot1 / 1e6,
               "sample": f"{n} random pixels of one {S}x{S} image through sepconv+Harris+NLM (f64 oracle); "
                         f"per-filter s: " + ", ".join(f"{k}={v:.2f}" for k, v in t.items())}

    if rank == 0:
        line = {
            "metric": "suite megapixels/s (sepconv r2 + Harris B5 + NLM 5x5/11x11)",
            "value": value, "unit": "Mpx/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "suite (BASELINE.json configs[4] per GPU)", "images_per_gpu": B,
                       "size": [S, S], "global_batch": B * ws, **SUITE, "harris_threshold": thr,
                       "l2": "inputs (3 x %d MiB per rank) exceed the 126 MB L2; no flush" % (B * S * S * 4 >> 20),
                       "variants": variants, "tuned": {k: v["name"] for k, v in tuned.items()},
                       "input_gen_s": round(t_gen, 1)},
            "per_filter_mpx_s": {f: px_rank / (m * 1e-3) / 1e6 for f, m in med.items()},
            "per_filter_ms": med,
            "per_filter_ms_min": {f: min(v) for f, v in per.items()},
            "roofline": {k: roof[dominant][k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")},
            "roofline_kernel": dominant,
            "rooflines": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if not args.no_small:
            line["small_configs"] = small_configs(dev)
    if not args.no_16k:
        # configs[3] at this N (every rank takes part: the exchange is collective)
        del u, hs, ns, o_sep, o_har, o_mask, o_nlm
        torch.cuda.empty_cache()
        k16 = sepconv16k_keys(ws, rank, local, dist, args.steps)
        if rank == 0:
            line["sepconv16k_row_bands"] = k16
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- icl arm: row bands
def small_configs(dev):
    """BASELINE.json configs[0..2] on one GPU: 512^2 sepconv r=2, 2048^2 Harris B=5 (+mask), 1024^2
    NLM 5x5/11x11 -- latency-bound sizes, timed per call eagerly and as a replayed CUDA graph of 20
    calls (the calls only enqueue on the stream, so they capture).  Inputs are L2-resident at these
    sizes (stated; the %HBM roofline is not meaningful here)."""
    import torch

    import paper_1605_06399_b200 as icl
    st = torch.cuda.Stream(device=dev)
    a = torch.from_numpy(synth.uniform_image(1, 512, 512)).to(dev)
    h = torch.from_numpy(synth.rect_scene(2, 2048, 2048, noise=0.01)).to(dev)
    n = torch.from_numpy(synth.rect_scene(3, 1024, 1024, noise=0.0866)).to(dev)
    fx = synth.gaussian_taps(2)
    oa, oh, on = torch.empty_like(a), torch.empty_like(h), torch.empty_like(n)
    mk = torch.empty(2048, 2048, dtype=torch.uint8, device=dev)
    calls = {
        "sepconv_512_r2": (lambda: icl.sepconv(a, oa, fx, fx, "constant", stream=st), 512 * 512, "sepconv"),
        "harris_2048_b5": (lambda: icl.harris(h, oh, 5, 0.04, "clamp", mask=mk, threshold=1.0, stream=st),
                           2048 * 2048, "harris"),
        "nlm_1024_5x5_11x11": (lambda: icl.nlm(n, on, 2, 5, 0.1, "clamp", stream=st), 1024 * 1024, "nlm"),
    }
    out = {}
    reps = 20
    for name, (fn, px, f) in calls.items():
        with torch.cuda.stream(st):
            for _ in range(3):
                fn()
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(reps):
                fn()
        e1.record(st)
        st.synchronize()
        eager_us = e0.elapsed_time(e1) * 1000 / reps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize(dev)
        runs = []
        for _ in range(7):  # median of 7 replays of the 20-call graph
            e0.record(st)
            with torch.cuda.stream(st):
                g.replay()
            e1.record(st)
            st.synchronize()
            runs.append(e0.elapsed_time(e1) * 1000 / reps)
        graph_us = statistics.median(runs)
        out[name] = {"us_per_call_eager": round(eager_us, 2), "us_per_call_graph": round(graph_us, 2),
                     "us_per_call_graph_min": round(min(runs), 2), "graph_replays": len(runs),
                     "mpx_s_graph": px / graph_us, "variant": icl.variant_names(f)[icl.last_variant(f)]}
    return out


def time_sepconv_bands(S, r, steps, warmup, ws, rank, local, dist, halo="nccl", torch_comm=False):
    """BASELINE.json configs[3] core: one S x S fp32 image, separable Gaussian radius r, row-band
    sharded over the ws ranks; the halo exchange (NCCL in libicl.so by default) overlapped with the
    interior rows.  Input pre-sharded (each rank fills its own rows on the device, untimed, like
    the paper's transfer exclusion PAPER.md:581-582).  Returns a dict with the max-over-ranks step
    time and how it ran; every rank must call it."""
    import torch

    import paper_1605_06399_b200 as icl
    from paper_1605_06399_b200 import dist as icd
    dev = torch.device("cuda", local)
    band = icd.partition(S, ws, rank, r, r)
    buf = torch.empty(band.buf_rows, S, device=dev)
    # own rows from the device generator (synth.uniform_image stream), halos by exchange
    icl.fill_uniform(buf[band.own_slice], 4, row0=band.r0)
    out = torch.empty(band.rows, S, device=dev)
    fx = synth.gaussian_taps(r)
    stream = torch.cuda.current_stream(dev)
    comm = torch.cuda.Stream(device=dev)

    def call(src, dst, b, st):
        icl.sepconv(src, dst, fx, fx, "constant", band=b, stream=st)

    # one GPU shared by every rank (ICL_BENCH_ONE_GPU): NCCL refuses two ranks on one device, so
    # the functional check takes the peer-load path (CUDA IPC works between processes of one GPU)
    if ONE_GPU and ws > 1 and halo in ("nccl", "window") and not torch_comm:
        halo = "peer"
    peer = ws > 1 and halo == "peer"
    window = ws > 1 and halo == "window"
    native = ws > 1 and not torch_comm and not peer and not window
    ncomm = icl.Comm(ws, rank) if (native or window) else None  # NCCL in libicl.so
    nbr = {}
    win = None
    if window:  # icl_sepconv_window: own rows in an NCCL symmetric window, halos read in-kernel
        pitch = ((S * 4 + 511) // 512) * 512
        rows_of = [icd.partition(S, ws, q, r, r).rows for q in range(ws)]
        win = icl.Window(ncomm, max(rows_of) * pitch)  # the same size on every rank (collective)
        win.write(0, buf[band.own_slice], pitch)
        own_img = win.image(0, S, band.rows, pitch)
        wb = {q: icl.Window.band(q, 0, rows_of[q], pitch) for q in (rank - 1, rank + 1) if 0 <= q < ws}
        torch.cuda.synchronize(dev)
        dist.barrier()  # every rank's own rows are in its window
    if peer:  # icl_sepconv_peer: own rows only, the halo read in-kernel from the neighbours (CUDA IPC)
        own = buf[band.own_slice]
        meta = [None] * ws
        dist.all_gather_object(meta, icl.ipc_handle(buf) + (band.r0 - band.s0,))
        for q in (rank - 1, rank + 1):
            if 0 <= q < ws:
                qb = icd.partition(S, ws, q, r, r)
                h, off, skip = meta[q]
                nbr[q] = icl.PeerImage(h, off + skip * S * 4, S, qb.rows, S)
        torch.cuda.synchronize(dev)
        dist.barrier()  # every rank's own rows are written

    def step():
        if window:
            icl.sepconv_window(win, own_img, out, S, band.r0, wb.get(rank - 1), wb.get(rank + 1), fx, fx, "constant",
                               stream=stream)
            return
        if peer:
            icl.sepconv_peer(own, out, S, band.r0, nbr.get(rank - 1), nbr.get(rank + 1), fx, fx, "constant",
                             stream=stream)
            return
        if native:
            ncomm.sepconv(buf, out, S, fx, fx, "constant", stream=stream)
            return
        icd.run_band(call, buf, out, band, (lambda: icd.halo_exchange(buf, band)) if ws > 1 else (lambda: None),
                     stream=stream, comm_stream=comm if ws > 1 else None)

    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    n0 = icl.launch_count()
    with ClockSampler(local) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            step()
        b.record(stream)
        torch.cuda.synchronize(dev)
    launches = icl.launch_count() - n0
    if ws > 1:
        dist.barrier()
    step_ms = max_over_ranks(a.elapsed_time(b) / steps, ws, dev)
    res = {"ms": step_ms, "launches": launches, "clocks": clk.summary(), "halo_rows": [band.up, band.down],
           "exchange": ("icl_sepconv_window (halo rows loaded in-kernel through NCCL symmetric windows)"
                        if window else "icl_sepconv_peer (halo rows loaded in-kernel from the peers, CUDA IPC)"
                        if peer else "icl_sepconv_sharded (NCCL in libicl.so)" if native else
                        "torch.distributed batch_isend_irecv" if ws > 1 else "none (one rank holds the image)"),
           "variant": icl.variant_names("sepconv")[icl.last_variant("sepconv")]}
    if win is not None:
        dist.barrier()  # no rank deregisters while a peer may still read its window
        win.close()
    if ncomm is not None:
        ncomm.close()
    if peer:
        dist.barrier()  # no rank frees its band while a peer may still read it
        for p in nbr.values():
            p.close()
    del buf, out
    return res


def sepconv16k_keys(ws, rank, local, dist, steps, radii=(2, 15), S=16384):
    """configs[3] keys of the default line at this N: per radius the row-band sharded 16384^2
    sepconv through icl_sepconv_sharded (strong scaling), its Mpx/s, and -- from the same run --
    the unsharded single-GPU time T(1) of the whole image on rank 0's GPU, so
    E(N) = T(1) / (N * T(N)) is readable from one line (the driver computes its own scaling
    from the per-N values)."""
    import torch

    import paper_1605_06399_b200 as icl
    dev = torch.device("cuda", local)
    hbm, _ = measured_peaks()
    out = {}
    for r in radii:
        k = max(5, steps)
        t1 = None
        if ws > 1:
            # T(1): the whole image on one GPU (rank 0), the others wait at the barrier
            if rank == 0:
                img = torch.empty(S, S, device=dev)
                icl.fill_uniform(img, 4)
                o = torch.empty_like(img)
                fx = synth.gaussian_taps(r)
                st = torch.cuda.current_stream(dev)
                for _ in range(3):
                    icl.sepconv(img, o, fx, fx, "constant", stream=st)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(k):
                    icl.sepconv(img, o, fx, fx, "constant", stream=st)
                b.record(st)
                torch.cuda.synchronize(dev)
                t1 = a.elapsed_time(b) / k
                del img, o
            dist.barrier()
        res = time_sepconv_bands(S, r, k, 3, ws, rank, local, dist)
        if ws == 1:
            t1 = res["ms"]
        px = S * S
        e = {"ms": res["ms"], "mpx_s": px / (res["ms"] * 1e-3) / 1e6, "n_gpus": ws,
             "per_gpu_GBps": 8 * px / ws / (res["ms"] * 1e-3) / 1e9, "exchange": res["exchange"],
             "variant": res["variant"], "launches": res["launches"], "halo_rows": res["halo_rows"]}
        e["per_gpu_frac_of_measured_hbm"] = e["per_gpu_GBps"] / hbm
        if t1 is not None:
            e["t1_ms_same_run"] = t1
            e["E_vs_same_run_t1"] = t1 / (ws * res["ms"])
        out[f"r{r}"] = e
        torch.cuda.empty_cache()
    return out


def run_sepconv_bands(args):
    """BASELINE.json configs[3]: one S x S fp32 image, separable Gaussian radius r,
    row-band sharded over the ranks with the halo exchange overlapped with the interior
    rows.  Strong scaling (the image is fixed)."""
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = init_dist(ws, "nccl")
    import paper_1605_06399_b200 as icl
    icl.load_library()
    S, r = args.size, args.radius
    res = time_sepconv_bands(S, r, args.steps, args.warmup, ws, rank, local, dist, halo=args.halo,
                             torch_comm=args.torch_comm)
    step_ms = res["ms"]
    px = S * S
    value = px / (step_ms * 1e-3) / 1e6
    hbm, hbm_kind = measured_peaks()
    achieved = 8 * px / ws / (step_ms * 1e-3) / 1e9  # per-GPU algorithmic GB/s
    if rank == 0:
        line = {
            "metric": f"sepconv megapixels/s ({S}x{S} fp32, radius {r}, row-band sharded)",
            "value": value, "unit": "Mpx/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "sepconv16k (BASELINE.json configs[3])", "size": [S, S], "radius": r,
                       "border": "constant", "halo_rows": res["halo_rows"], "exchange": res["exchange"],
                       "variant": res["variant"], "l2": "input 1 GiB >> L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": None, "peak_kind": hbm_kind},
            "gpu_launches": res["launches"], "clocks": res["clocks"], "e2e": None, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_conv2d(args):
    """the paper's third benchmark: non-separable
    (2r+1)^2 convolution of an 8192^2 unsigned-char image with a run-time filter, clamped
    boundary, fp32 output (R22).  One image per rank (image-parallel, weak scaling);
    two input/output pairs alternate so consecutive steps never hit L2 (2 x 320 MB)."""
    import numpy as np
    import torch

    import paper_1605_06399_b200 as icl
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(ws, "nccl")
    icl.load_library()
    S, r = args.size, args.radius
    filt = synth.filter2d(8, r)
    imgs_h = [synth.uniform_u8(1000 * rank + k, S, S) for k in range(2)]
    imgs = [torch.from_numpy(a).to(dev) for a in imgs_h]
    outs = [torch.empty(S, S, device=dev) for _ in range(2)]
    stream = torch.cuda.current_stream(dev)
    if not args.no_tune:
        icl.tune("conv2d", imgs[0], outs[0], filter2d=filt, border="clamp", stream=stream)

    def step(k):
        icl.conv2d_u8(imgs[k & 1], outs[k & 1], filt, "clamp", stream=stream)

    for k in range(max(3, args.warmup)):
        step(k)
    torch.cuda.synchronize(dev)
    variant = icl.variant_names("conv2d")[icl.last_variant("conv2d")]
    if ws > 1:
        dist.barrier()
    n0 = icl.launch_count()
    with ClockSampler(local) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(args.steps):
            step(k)
        b.record(stream)
        torch.cuda.synchronize(dev)
    launches = icl.launch_count() - n0
    if ws > 1:
        dist.barrier()
    step_ms = max_over_ranks(a.elapsed_time(b) / args.steps, ws, dev)
    px = S * S
    value = ws * px / (step_ms * 1e-3) / 1e6
    hbm, hbm_kind = measured_peaks()
    n = 2 * r + 1
    gbs = 5 * px / (step_ms * 1e-3) / 1e9
    tfs = 2 * n * n * px / (step_ms * 1e-3) / 1e12
    roof = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": None,
            "peak_kind": hbm_kind, "bytes_per_px": 5}
    roof_alu = {"bound": "alu", "achieved": tfs, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": tfs / FP32_PEAK_TFLOPS, "flop_per_px": 2 * n * n}
    # e2e: the same call with pinned HOST buffers (the library's banded H2D/compute/D2H pipeline)
    e2e = None
    if not args.no_e2e:
        hin = torch.from_numpy(imgs_h[0]).pin_memory()
        hout = torch.empty(S, S).pin_memory()
        ke = max(1, min(args.steps, 5))
        icl.conv2d_u8(hin, hout, filt, "clamp", stream=stream)
        stream.synchronize()
        if ws > 1:
            dist.barrier()
        x0 = icl.transfer_bytes()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(ke):
            icl.conv2d_u8(hin, hout, filt, "clamp", stream=stream)
        eb.record(stream)
        stream.synchronize()
        x1 = icl.transfer_bytes()
        e_ms = max_over_ranks(ea.elapsed_time(eb) / ke, ws, dev)
        ok = bool(np.array_equal(hout.numpy()[::1021], outs[0].cpu().numpy()[::1021]))
        e2e = {"value": ws * px / (e_ms * 1e-3) / 1e6, "unit": "Mpx/s", "h2d_bytes_per_step": (x1[0] - x0[0]) // ke,
               "d2h_bytes_per_step": (x1[1] - x0[1]) // ke, "ms_per_step": e_ms, "steps": ke,
               "path": "C ABI with pinned host buffers", "matches_device_outputs": ok}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        rng = np.random.default_rng(0)
        npts = 4_000_000
        xs, ys = rng.integers(0, S, npts), rng.integers(0, S, npts)
        t0 = time.perf_counter()
        oracle.conv2d_u8(imgs_h[0], filt, "clamp", points=(xs, ys))
        dt = time.perf_counter() - t0
        cpu = {"value": npts / dt / 1e6, "unit": "Mpx/s", "cores": oracle.default_threads(), "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"{npts} random pixels of one {S}x{S} uchar image (f64 oracle, {dt:.1f} s)"}
    if rank == 0:
        line = {
            "metric": f"conv2d_u8 megapixels/s ({S}x{S} uchar, {n}x{n} run-time filter, clamp)",
            "value": value, "unit": "Mpx/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "conv2d8k (PAPER.md:594-598; SURVEY.md §8(f) row 1)", "size": [S, S],
                       "radius": r, "border": "clamp", "variant": variant, "images_per_gpu": 1,
                       "l2": "two input/output pairs alternate (2 x 320 MB > L2)"},
            "roofline": roof, "rooflines": {"conv2d_hbm": roof, "conv2d_fp32": roof_alu},
            "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_sep3d(args):
    """SURVEY.md §8(f) row 4 (3-D Images; R26): separable convolution
    of a 128 x 512 x 512 fp32 volume per rank (weak scaling), radius r on every axis, clamp.
    Two input/output volume pairs alternate (4 x 134 MB > L2).  e2e: pinned host volume in,
    the call, result out (explicit copies around icl_sepconv3d, which takes device volumes)."""
    import numpy as np
    import torch

    import paper_1605_06399_b200 as icl
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(ws, "nccl")
    icl.load_library()
    D, S, r = args.depth, args.size, args.radius
    f = synth.gaussian_taps(r)
    vols = [torch.empty(D, S, S, device=dev) for _ in range(2)]
    for k, v in enumerate(vols):
        icl.fill_uniform(v, 5000 + 100 * rank + 10 * k)  # slice z = synth.uniform_image(seed + z, S, S)
    outs = [torch.empty_like(v) for v in vols]
    stream = torch.cuda.current_stream(dev)

    def step(k):
        icl.sepconv3d(vols[k & 1], outs[k & 1], f, f, f, "clamp", stream=stream)

    for k in range(max(3, args.warmup)):
        step(k)
    torch.cuda.synchronize(dev)
    variant = icl.variant_names("sepconv3d")[icl.last_variant("sepconv3d")]
    if ws > 1:
        dist.barrier()
    n0 = icl.launch_count()
    with ClockSampler(local) as clk:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(args.steps):
            step(k)
        b.record(stream)
        torch.cuda.synchronize(dev)
    launches = icl.launch_count() - n0
    if ws > 1:
        dist.barrier()
    step_ms = max_over_ranks(a.elapsed_time(b) / args.steps, ws, dev)
    nvox = D * S * S
    value = ws * nvox / (step_ms * 1e-3) / 1e6
    hbm, hbm_kind = measured_peaks()
    gbs = 8 * nvox / (step_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": None,
            "peak_kind": hbm_kind, "bytes_per_voxel": 8, "flop_per_voxel": 6 * (2 * r + 1)}
    e2e = None
    if not args.no_e2e:
        hin = vols[0].cpu().pin_memory()
        hout = torch.empty(D, S, S).pin_memory()
        din, dout = torch.empty_like(vols[0]), torch.empty_like(vols[0])
        ke = max(1, min(args.steps, 5))

        def e2e_step():
            din.copy_(hin, non_blocking=True)
            icl.sepconv3d(din, dout, f, f, f, "clamp", stream=stream)
            hout.copy_(dout, non_blocking=True)

        e2e_step()
        stream.synchronize()
        if ws > 1:
            dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(ke):
            e2e_step()
        eb.record(stream)
        stream.synchronize()
        e_ms = max_over_ranks(ea.elapsed_time(eb) / ke, ws, dev)
        ok = bool(torch.equal(hout[:, ::61, ::67], outs[0].cpu()[:, ::61, ::67]))
        e2e = {"value": ws * nvox / (e_ms * 1e-3) / 1e6, "unit": "Mvoxel/s", "h2d_bytes_per_step": 4 * nvox,
               "d2h_bytes_per_step": 4 * nvox, "ms_per_step": e_ms, "steps": ke,
               "path": "pinned host volume -> icl_sepconv3d -> pinned host volume (copies on the call's stream)",
               "matches_device_outputs": ok}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        rng = np.random.default_rng(0)
        # the oracle's input is regenerated on the host from the same seeds (never read back from the GPU)
        host = np.stack([synth.uniform_image(5000 + 100 * rank + z, S, S) for z in range(D)])
        npts = 500_000
        while True:  # grow the random sample until it takes >= 2 s (bounded by the volume)
            xs, ys, zs = rng.integers(0, S, npts), rng.integers(0, S, npts), rng.integers(0, D, npts)
            t0 = time.perf_counter()
            oracle.sepconv3d(host, f, f, f, "clamp", points=(xs, ys, zs))
            dt = time.perf_counter() - t0
            if dt >= 2.0 or npts >= nvox:
                break
            npts = min(nvox, npts * 4)
        cpu = {"value": npts / dt / 1e6, "unit": "Mvoxel/s", "cores": oracle.default_threads(), "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"{npts} random voxels of one {D}x{S}x{S} volume (f64 oracle, {dt:.1f} s)"}
    if rank == 0:
        line = {
            "metric": f"sepconv3d megavoxels/s ({D}x{S}x{S} fp32, radius {r} on every axis, clamp)",
            "value": value, "unit": "Mvoxel/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "sep3d (PAPER.md:303-304 3-D Images; SURVEY.md §8(f) row 4)",
                       "size": [D, S, S], "radius": r, "border": "clamp", "variant": variant,
                       "l2": "two input/output volume pairs alternate (4 x 134 MB > L2)"},
            "roofline": roof, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_chain(args):
    """SURVEY.md §8(f) row 4 (FAST-style filter chains; R24): Gaussian
    smoothing (radius r) then Harris B = 5 + mask on the suite's 8 x 4096^2 batch per rank, through
    icl_blur_harris -- the two-pass schedule (caller workspace) is timed as the value, the fused
    one-pass kernel beside it.  Inputs 512 MB > L2 (no flush)."""
    import numpy as np
    import torch

    import paper_1605_06399_b200 as icl
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = init_dist(ws, "nccl")
    icl.load_library()
    B, S, r = args.batch, args.size, args.radius
    f = synth.gaussian_taps(r)
    src = torch.empty(B, S, S, device=dev)
    icl.fill_uniform(src, 7000 + 100 * rank)
    R = torch.empty_like(src)
    mask = torch.empty(B, S, S, dtype=torch.uint8, device=dev)
    wsb = torch.empty(icl.blur_harris_workspace_bytes(S, S, B, 5) // 4 + 4, device=dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps):
        for _ in range(max(3, args.warmup)):
            fn()
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize(dev)
        return max_over_ranks(a.elapsed_time(b) / steps, ws, dev)

    def two_pass():
        icl.blur_harris(src, R, f, f, "constant", 0.0, 5, 0.04, "clamp", mask=mask, threshold=1.0, workspace=wsb,
                        stream=stream)

    def fused():
        icl.blur_harris(src, R, f, f, "constant", 0.0, 5, 0.04, "clamp", mask=mask, threshold=1.0, stream=stream)

    n0 = icl.launch_count()
    with ClockSampler(local) as clk:
        step_ms = timed(two_pass, args.steps)
    launches = (icl.launch_count() - n0) // (args.steps + max(3, args.warmup)) * args.steps
    fused_ms = timed(fused, args.steps)
    R2 = R.clone()
    two_pass()
    torch.cuda.synchronize(dev)
    same = bool(torch.equal(R, R2))
    px = B * S * S
    value = ws * px / (step_ms * 1e-3) / 1e6
    hbm, hbm_kind = measured_peaks()
    # algorithmic bytes of the chain: read 4 + response 4 + mask 1 (the intermediate is not algorithmic)
    gbs = 9 * px / (step_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": None,
            "peak_kind": hbm_kind, "bytes_per_px": 9,
            "note": "two-pass schedule moves 8 + 9 B/px (intermediate through HBM); fused moves 9"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        n = 2048
        img = synth.uniform_image(7000, n, n)
        t0 = time.perf_counter()
        oracle.harris(oracle.sepconv(img, f, f, "constant").astype(np.float32), 5, 0.04, "clamp")
        dt = time.perf_counter() - t0
        cpu = {"value": n * n / dt / 1e6, "unit": "Mpx/s", "cores": oracle.default_threads(), "kind": "oracle",
               "cpu_model": cpu_model(),
               "sample": f"one {n}x{n} image through oracle sepconv then Harris ({dt:.2f} s)"}
    if rank == 0:
        line = {
            "metric": f"blur r{r} + Harris B5 megapixels/s (icl_blur_harris, {B} x {S}x{S} fp32)",
            "value": value, "unit": "Mpx/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "chain (FAST-style pipeline, PAPER.md:128-142; SURVEY.md §8(f) row 4)",
                       "images_per_gpu": B, "size": [S, S], "radius": r, "schedule": "two-pass (workspace)",
                       "l2": "input 512 MB > L2; no flush"},
            "fused_ms_per_step": fused_ms, "fused_equals_two_pass": same,
            "roofline": roof, "gpu_launches": launches, "clocks": clk.summary(), "e2e": None, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def relaunch(n):
    """`--gpus N` without a launcher: re-exec this command under torch.distributed.run with N ranks
    (one process per GPU, 127.0.0.1 rendezvous on a free port) and return its exit code."""
    import socket
    import subprocess
    if not ONE_GPU:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} but only {have} CUDA device(s) visible "
                  f"(ICL_BENCH_ONE_GPU=1 runs every rank on cuda:0 as a functional check)", file=sys.stderr)
            return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print("bench.py: launching " + " ".join(cmd[1:]), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="icl", choices=["icl", "reference"])
    ap.add_argument("--workload", default="suite", choices=["suite", "sepconv16k", "conv2d8k", "sep3d", "chain"])
    ap.add_argument("--depth", type=int, default=128, help="sep3d: volume depth (slices)")
    ap.add_argument("--radius", type=int, default=2)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--no-small", action="store_true", help="suite: skip the configs[0..2] latency block")
    ap.add_argument("--no-16k", action="store_true",
                    help="suite: skip the configs[3] keys (16384^2 row-band sepconv at r = 2 and 15)")
    ap.add_argument("--torch-comm", action="store_true", help="sepconv16k: exchange halos via torch.distributed")
    ap.add_argument("--halo", default="nccl", choices=["nccl", "peer", "window"],
                    help="sepconv16k, N > 1: NCCL send/recv (icl_sepconv_sharded), in-kernel peer loads "
                         "(icl_sepconv_peer over CUDA IPC) or in-kernel loads through NCCL symmetric windows "
                         "(icl_sepconv_window)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        return relaunch(args.gpus)
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}; launch one rank per GPU "
              f"(torch.distributed.run --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "conv2d8k":
        if args.size == 4096:
            args.size = 8192
        return run_conv2d(args)
    if args.workload == "sepconv16k":
        if args.size == 4096:
            args.size = 16384
        return run_sepconv_bands(args)
    if args.workload == "chain":
        return run_chain(args)
    if args.workload == "sep3d":
        if args.size == 4096:
            args.size = 512
        return run_sep3d(args)
    return run_suite(args)


if __name__ == "__main__":
    sys.exit(main())
