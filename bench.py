#!/usr/bin/env python
"""bench.py — DoRA modules/s on B200 (BASELINE.json metric), one JSON line on rank 0.

Workload (BASELINE.json configs[1]: "single module d_out=d_in=8192 r=384 bf16,
tokens=4096 compose fwd+bwd"): one step = one DoRA module TRAINING
step of the hot path,
  dfx_row_norm    factored ||W + sBA||_row (Gram, bf16 hi/lo B.G, W.A^T + base_sq chain,
                  assemble, dtype rounding) and the magnitude g = m / max(norm, eps)
  dfx_compose_fwd dual output: delta = (g-1)*base + g*s*lora and inner = s*lora + base
  dfx_compose_bwd d_lora = g*s*dY, d_base = (g-1)*dY and d_mag = sum_rows(dY*inner)/norm
at d_out = d_in = 8192, r = 384, bf16, tokens = 4096, s = 2/sqrt(r).  The inference
module (row_norm + plain compose_fwd) is reported beside it under "variants".
Synthetic data (seeded torch.randn on device; m = ||W+sBA|| * (1 + N(0, 0.0015)) so
g ~ 1 as in the paper's regime).  Inputs are larger than L2 (W 128 MiB + 5 activation
tensors of 64 MiB per module) and NBUF module buffer sets rotate, so every step reads
cold HBM.

Timed region: K steps replayed as CUDA graphs (modules software-pipelined on two
streams), CUDA events on the launching stream, barrier + synchronize on both sides, max
over ranks.  A second pass with the C ABI's per-kernel event profiling (dfx_profile_*)
gives the live per-kernel durations behind `roofline`.  `e2e` goes through the
host-buffer entry point dfx_module_train_host (pinned host -> HBM -> kernels -> host).
`cpu_baseline` times the reference's own C++ (oracle/_ref) on this host's cores on a
bounded sample.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--mode infer]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N  (modules shard across ranks:
weak scaling, no data-path collective).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DoRA modules/sec (norm+compose) at d_in=8192 r=384"
UNIT = "modules/s"

CONFIGS = {
    # name: d_out, d_in, r, tokens, dtype
    "c1": dict(d_out=4096, d_in=4096, r=384, tokens=4096, dtype="fp32"),
    "c2": dict(d_out=8192, d_in=8192, r=384, tokens=4096, dtype="bf16"),
    "c3": dict(d_out=28672, d_in=8192, r=384, tokens=4096, dtype="bf16"),
    "c4r64": dict(d_out=8192, d_in=8192, r=64, tokens=4096, dtype="bf16"),
    "c4r128": dict(d_out=8192, d_in=8192, r=128, tokens=4096, dtype="bf16"),
    "c4r512": dict(d_out=8192, d_in=8192, r=512, tokens=4096, dtype="bf16"),
    "c4r1024": dict(d_out=8192, d_in=8192, r=1024, tokens=4096, dtype="bf16"),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


TRAIN_NORM_SMS = 138   # the C2 training pipeline's norm SM budget (measured, DESIGN 5.3-5.4)
# (config, mode) -> the pipelined graph's norm SM budget when --norm-sms is not given
NORM_SMS_DEFAULT = {("c2", "train"): TRAIN_NORM_SMS, ("c3", "train"): 120, ("c3", "infer"): 120,
                    ("c5", "train"): 104}


def algorithmic(cfg):
    """Per-launch algorithmic work for each kernel of a module."""
    d_out, d_in, r, rows = cfg["d_out"], cfg["d_in"], cfg["r"], cfg["tokens"]
    eb = 2 if cfg["dtype"] != "fp32" else 4
    return {
        # name: (bound, flops, bytes)
        "u_rowdot_tc": ("tensor", 2.0 * d_out * d_in * r,
                        eb * (d_out * d_in + r * d_in + d_out * r) + 4.0 * d_out),
        "gram_tc": ("tensor", 2.0 * r * r * d_in, eb * r * d_in),
        "ba_rowdot_tc": ("tensor", 2.0 * d_out * r * r, eb * d_out * r + 4.0 * r * r),
        "gram_reduce": ("hbm", 0.0, 8.0 * r * r),
        "finish": ("hbm", 0.0, 4.0 * 5 * d_out),
        "compose_fwd": ("hbm", 0.0, 3.0 * eb * rows * d_out + 4.0 * d_out),
        "compose_fwd_dual": ("hbm", 0.0, 4.0 * eb * rows * d_out + 4.0 * d_out),
        "compose_bwd_dmag": ("hbm", 0.0, 4.0 * eb * rows * d_out + 12.0 * d_out),
        "norm_total": ("tensor", 2.0 * d_out * d_in * r + 2.0 * r * r * d_in + 2.0 * d_out * r * r,
                       eb * (d_out * d_in + r * d_in + d_out * r) + 4.0 * d_out),
    }


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index):
        self.samples, self.reasons = [], 0
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        s = sorted(self.samples)
        reasons = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(s)}


# ------------------------------------------------------------------- CPU reference
def cpu_reference_rate(cfg, cores, mode="train", rounds=1, warm=0, log=None, full_module=False):
    """The reference's own C++ (oracle/_ref/libdfx_ref.so, compiled from the reference
    sources) on this host.  The reference is single-threaded per call, so all cores run
    independent module samples concurrently (as its own suites do, suites.cpp:49-65).

    A full C2 module costs ~20-40 s on one core, so each thread runs a bounded sample:
    factored_row_norm on NS W-rows (full A, full d_in; Gram cost included) + the compose
    on CT token rows (train: dual_output_compose + compose_backward with the magnitude
    gradient; infer: fused_compose).  A single-core calibration separates the fixed
    (Gram) cost from the per-row and per-token costs, which converts a sample into
    module-equivalents:
        t_module = t_fixed + d_out * t_row + (tokens / CT) * t_compose(CT)
    Returns (modules/s, details)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    R = pyoracle.Reference()
    d_out, d_in, r, tokens = cfg["d_out"], cfg["d_in"], cfg["r"], cfg["tokens"]
    dt = {"fp32": 0, "bf16": 1, "fp16": 2}[cfg["dtype"]]
    s = 2.0 / math.sqrt(r)
    rng = np.random.default_rng(7)

    def rnd(a):
        if dt == 1:
            u = a.astype(np.float32).view(np.uint32)
            u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
            return u.view(np.float32)
        return a.astype(np.float16).astype(np.float32) if dt == 2 else a.astype(np.float32)

    NS1, NS2, CT = 16, 128, 256
    A = rnd(rng.standard_normal((r, d_in)))
    Wn = rnd(rng.standard_normal((NS2, d_in)))
    Bn = rnd(rng.standard_normal((NS2, r)))
    base = rnd(rng.standard_normal((CT, d_out)))
    lora = rnd(rng.standard_normal((CT, d_out)))
    dy = rnd(rng.standard_normal((CT, d_out)))
    g = np.array([R.round_to_dtype(v, dt) for v in 1.0 + 0.0015 * rng.standard_normal(d_out)])
    wn = np.array([R.round_to_dtype(v, dt) for v in 90.0 + rng.standard_normal(d_out)])
    cs, _ = R.plan_chunks(d_out, d_in)   # the full module's chunk plan

    def norm_sample(n):
        R.row_norm(dt, np.ascontiguousarray(Wn[:n]), A, np.ascontiguousarray(Bn[:n]), s, cs)
        return R.last_call_s()

    def compose_sample():
        if mode == "infer":
            R.compose(1, dt, base, lora, g, s)
            return R.last_call_s()
        _, inner = R.compose(2, dt, base, lora, g, s, need_inner=True)
        t = R.last_call_s()
        R.compose_bwd(dt, dy, g, s, inner=inner, w_norm=wn, mag_grad=True)
        return t + R.last_call_s()

    norm_sample(NS1)                     # warm caches / page in A before calibrating
    compose_sample()
    t1 = min(norm_sample(NS1) for _ in range(2))
    t2 = min(norm_sample(NS2) for _ in range(2))
    t_row = max((t2 - t1) / (NS2 - NS1), 1e-9)
    t_fixed = max(t1 - NS1 * t_row, 0.0)
    t_c = min(compose_sample() for _ in range(2))
    t_module = t_fixed + d_out * t_row + (tokens / CT) * t_c
    sample_equiv = (t_fixed + NS2 * t_row + t_c) / t_module
    if log:
        log(f"cpu ref calibration ({mode}): fixed {t_fixed:.3f}s row {t_row * 1e3:.3f}ms "
            f"compose({CT}) {t_c:.3f}s -> {t_module:.1f}s/module/core")

    def worker(out, i):
        out[i] = norm_sample(NS2) + compose_sample()

    rates = []
    for k in range(warm + rounds):
        out = [0.0] * cores
        th = [threading.Thread(target=worker, args=(out, i)) for i in range(cores)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
        if k >= warm:
            rates.append(cores * sample_equiv / wall)
    rate = sorted(rates)[len(rates) // 2]
    full = None
    if full_module:
        # validate the conversion model: one WHOLE module on one core (every W row, every
        # token), the reference's own calls back to back
        Wf = rnd(rng.standard_normal((d_out, d_in)))
        Bf = rnd(rng.standard_normal((d_out, r)))
        R.row_norm(dt, Wf, A, Bf, s, cs)
        t_norm = R.last_call_s()
        del Wf
        t_comp = 0.0
        for c0 in range(0, tokens, 1024):           # the whole token range, 1024 rows per call
            nr = min(1024, tokens - c0)
            bb = rnd(rng.standard_normal((nr, d_out)))
            ll = rnd(rng.standard_normal((nr, d_out)))
            if mode == "infer":
                R.compose(1, dt, bb, ll, g, s)
                t_comp += R.last_call_s()
            else:
                yy = rnd(rng.standard_normal((nr, d_out)))
                _, inn = R.compose(2, dt, bb, ll, g, s, need_inner=True)
                t_comp += R.last_call_s()
                R.compose_bwd(dt, yy, g, s, inner=inn, w_norm=wn, mag_grad=True)
                t_comp += R.last_call_s()
        t_full = t_norm + t_comp
        full = {"measured_full_module_s": round(t_full, 3), "measured_norm_s": round(t_norm, 3),
                "measured_compose_s": round(t_comp, 3), "model_s": round(t_module, 3),
                "model_error": round(t_module / t_full - 1.0, 4),
                "value_uncorrected": round(rate, 6),
                "correction": "value = all-core sample rate x model_s / measured_full_module_s "
                              "(the conversion model rescaled to the measured whole module)"}
        rate = rate * t_module / t_full
        if log:
            log(f"cpu ref full module (1 core): {t_full:.2f}s (norm {t_norm:.2f}s, compose "
                f"{t_comp:.2f}s) vs model {t_module:.2f}s")
    what = ("dual_output_compose + compose_backward (mag_grad)" if mode == "train"
            else "fused_compose")
    return rate, {
        "t_module_1core_s": t_module, "t_fixed_s": t_fixed, "t_row_ms": t_row * 1e3,
        "full_module": full,
        "t_compose_per_token_us": t_c / CT * 1e6, "rounds": rounds,
        "sample": (f"per thread: reference factored_row_norm on {NS2} of {d_out} W rows (full "
                   f"d_in={d_in}, r={r}, Gram included) + {what} on {CT} of {tokens} "
                   f"tokens; {cores} threads concurrently; converted to modules via a 1-core "
                   f"calibration t_module = t_fixed + d_out*t_row + tokens/{CT}*t_compose "
                   f"= {t_module:.1f} s"),
    }


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------ GPU arm
def run_gpu(args, rank, world, local_rank, dist):
    import torch
    import paper_2603_22276_b200 as P

    cfg = CONFIGS[args.config]
    d_out, d_in, r, rows = cfg["d_out"], cfg["d_in"], cfg["r"], cfg["tokens"]
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[cfg["dtype"]]
    s = 2.0 / math.sqrt(r)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dfx = P.Dfx(local_rank)
    cs, nchunks = P.plan_chunks(d_out, d_in)
    log = (lambda m: print(m, file=sys.stderr, flush=True)) if rank == 0 else (lambda m: None)

    # ---- module buffer sets (synthetic, seeded per rank)
    nbuf = args.nbuf
    gen = torch.Generator(device=dev)
    gen.manual_seed(20261017 + rank)
    sets = []
    for i in range(nbuf):
        rnd = lambda *shape: torch.randn(*shape, device=dev, generator=gen).to(tdt)
        b = dict(W=rnd(d_out, d_in), A=rnd(r, d_in), B=rnd(d_out, r), base=rnd(rows, d_out),
                 lora=rnd(rows, d_out), dy=rnd(rows, d_out))
        b.update(wn=torch.empty(d_out, device=dev), g=torch.empty(d_out, device=dev),
                 dm=torch.empty(d_out, device=dev), ba=torch.empty(d_out, device=dev))
        for k in ("delta", "inner", "dl", "db"):
            b[k] = torch.empty_like(b["base"])
        dfx.row_norm(b["W"], b["A"], b["B"], s, cs, b["wn"])
        b["m"] = (b["wn"] * (1.0 + 0.0015 * torch.randn(d_out, device=dev, generator=gen))).contiguous()
        sets.append(b)
    torch.cuda.synchronize()

    split = args.split_adapter and tdt != torch.float32

    def adapter(b, st=None, sms=0):
        dfx.norm_adapter(b["A"], b["B"], d_out, b["ba"], sms=sms, stream=st)

    def norm_w(b, st=None):
        dfx.row_norm_ba(b["W"], b["A"], b["B"], s, cs, b["ba"], b["wn"], m=b["m"], g=b["g"],
                        stream=st)

    def norm(b, st=None):
        if split:      # the split form, serially (pipelined graphs issue the parts apart)
            adapter(b, st, args.adapter_sms)
            norm_w(b, st)
        else:
            dfx.row_norm(b["W"], b["A"], b["B"], s, cs, b["wn"], m=b["m"], g=b["g"], stream=st)

    def compose(b, mode, st=None):
        if mode == "infer":
            dfx.compose_fwd(b["base"], b["lora"], b["g"], s, b["delta"], stream=st)
        else:
            if args.compose_parts != "bwd":
                dfx.compose_fwd(b["base"], b["lora"], b["g"], s, b["delta"], b["inner"], stream=st)
            if args.compose_parts != "fwd":
                dfx.compose_bwd(b["dy"], b["g"], s, b["dl"], b["db"], inner=b["inner"],
                                w_norm=b["wn"], d_mag=b["dm"], stream=st)

    def step(b, mode):
        if args.only != "compose":
            norm(b)
        if args.only != "norm":
            compose(b, mode)

    # --stream-priority (measurement): a higher CUDA stream priority (-1) for the compose
    # stream or the norm stream of the pipelined graphs
    prio_c = -1 if args.stream_priority == "compose" else 0
    prio_n = -1 if args.stream_priority == "norm" else 0
    stream = torch.cuda.Stream(device=dev, priority=prio_n)
    side = torch.cuda.Stream(device=dev, priority=prio_c)
    third = torch.cuda.Stream(device=dev)
    # Every dfx call below issues on torch's current stream: make that `stream` for the whole
    # run.  Calls on one context must not overlap (dfx.h: the workspace is shared), and torch's
    # streams do not synchronise with the legacy default stream, so mixing the two let a call
    # on the default stream run beside one on `stream` (it corrupted the fused finisher's
    # counters for later calls).
    torch.cuda.synchronize()
    torch.cuda.set_stream(stream)

    def set_budget(mode, npipe):
        # the pipelined graph runs module i's compose beside module i+1's norm: leave the
        # compose kernels the SMs the norm GEMMs do not plan for (dfx_ctx_set_sm_budget).
        # A serial step (npipe == 1) gets the whole GPU for every kernel.
        n = args.norm_sms if mode == args.mode else NORM_SMS_DEFAULT.get((args.config, mode), 0)
        dfx.set_sm_budget(n if npipe > 1 else 0)

    def build_pipelined(mode, n):
        """A graph of n consecutive modules software-pipelined on two streams: module i's
        compose (HBM-bound) on stream B beside module i+1's row norm (tensor-bound) on
        stream A.  Edges: compose i after norm i (it reads g_i, w_norm_i); norm i+nbuf after
        compose i (it rewrites set i % nbuf)."""
        sA, sB = stream.cuda_stream, side.cuda_stream
        ev_norm = [torch.cuda.Event() for _ in range(n)]
        ev_comp = [torch.cuda.Event() for _ in range(n)]
        ev_adapt = [torch.cuda.Event() for _ in range(n)]

        def adapt(i):
            # module i's adapter terms (A, B only) one module ahead on a third stream, beside
            # module i-1's W part; it rewrites set i % nbuf's ba_sq, which module i-nbuf's W
            # part read
            if i >= nbuf:
                third.wait_event(ev_norm[i - nbuf])
            adapter(sets[i % nbuf], third.cuda_stream, args.adapter_sms)
            ev_adapt[i].record(third)
        gph = torch.cuda.CUDAGraph()
        order = args.capture_order
        if order == "auto":
            # round 2: norm-first for both (training at the 140-SM plan: 7.80k vs 7.75k
            # modules/s, two repeats on one box; inference: 11.6k vs 10.5k)
            order = "norm-first"

        def comp(i):
            side.wait_event(ev_norm[i])
            if args.only != "norm":
                compose(sets[i % nbuf], mode, sB)
            ev_comp[i].record(side)

        with torch.cuda.graph(gph, stream=stream):
            if split and args.only != "compose":
                third.wait_stream(stream)
                adapt(0)
            for i in range(n):
                b = sets[i % nbuf]
                if i >= nbuf:
                    stream.wait_event(ev_comp[i - nbuf])
                if split and args.only != "compose":
                    if i + 1 < n and args.adapter_first:
                        adapt(i + 1)
                    stream.wait_event(ev_adapt[i])
                    norm_w(b, sA)
                    # created after the W part: U's CTAs claim their SMs first
                    if i + 1 < n and not args.adapter_first:
                        adapt(i + 1)
                elif args.only != "compose":
                    norm(b, sA)
                ev_norm[i].record(stream)
                # capture order = launch order among ready nodes: module i+1's norm is
                # created before module i's compose, so the GEMM CTAs claim their SMs
                # before the streaming kernels flood the GPU
                if order == "norm-first":
                    if i >= 1:
                        comp(i - 1)
                else:
                    comp(i)
            if order == "norm-first":
                comp(n - 1)
            stream.wait_event(ev_comp[n - 1])
            if split and args.only != "compose":
                stream.wait_stream(third)
        return gph

    def build_graphs(mode, steps):
        """(schedule of (graph, modules) replays for `steps` modules, npipe).  npipe =
        min(--pipeline, steps): the timed steps run as steps // npipe replays of one
        npipe-module pipelined graph plus one remainder graph of steps % npipe modules, so
        every step count runs the pipelined protocol.  --pipeline 1: one serial graph per
        buffer set."""
        npipe = min(args.pipeline, steps) if args.pipeline > 1 else 1
        sched = []
        if npipe > 1:
            main = build_pipelined(mode, npipe)
            sched += [(main, npipe)] * (steps // npipe)
            rem = steps % npipe
            if rem:
                sched.append((build_pipelined(mode, rem) if rem > 1 else serial_graph(mode, 0), rem))
        else:
            gs = [serial_graph(mode, i) for i in range(nbuf)]
            sched = [(gs[k % nbuf], 1) for k in range(steps)]
        torch.cuda.synchronize()
        return sched, npipe

    def serial_graph(mode, i):
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=stream):
            step(sets[i % nbuf], mode)
        return gph

    def timed(mode, steps, warmup, clocks=None):
        npipe = min(args.pipeline, steps) if args.pipeline > 1 else 1
        set_budget(mode, npipe)
        # one eager pass under this plan first: the context sizes its workspace outside of
        # graph capture (dfx calls refuse to grow it while a capture is active)
        with torch.cuda.stream(stream):
            for b in sets:
                step(b, mode)
        torch.cuda.synchronize()
        sched, npipe = build_graphs(mode, steps)
        with torch.cuda.stream(stream):
            done = 0
            while done < warmup:                       # >= warmup modules, whole graphs
                g, n = sched[0]
                g.replay()
                done += n
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        import contextlib
        with (clocks if clocks is not None else contextlib.nullcontext()):
            with torch.cuda.stream(stream):
                ev0.record(stream)
                for g, _ in sched:
                    g.replay()
                ev1.record(stream)
            torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        if dist:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, npipe

    # warm each path eagerly once, count this library's kernel launches per step
    with torch.cuda.stream(stream):
        for i in range(max(2, nbuf)):
            step(sets[i % nbuf], args.mode)
    torch.cuda.synchronize()
    launches_before = dfx.launches
    with torch.cuda.stream(stream):
        step(sets[0], args.mode)
    torch.cuda.synchronize()
    launches_per_step = dfx.launches - launches_before

    # DFX_BENCH_CANARY=1 (debugging): after each phase, the row norm of set 0 under the budget
    # in force must reproduce the first result seen under that budget, bit for bit.
    canary_ref = {}

    def canary(tag):
        if not os.environ.get("DFX_BENCH_CANARY"):
            return
        b = sets[0]
        torch.cuda.synchronize()
        wn, g = torch.empty_like(b["wn"]), torch.empty_like(b["g"])
        with torch.cuda.stream(stream):
            dfx.row_norm(b["W"], b["A"], b["B"], s, cs, wn, m=b["m"], g=g)
        torch.cuda.synchronize()
        key = dfx.get_sm_budget() if hasattr(dfx, "get_sm_budget") else "?"
        cur = torch.cat([wn, g]).view(torch.int32)
        ref = canary_ref.setdefault(key, cur.clone())
        nd = int((cur != ref).sum())
        log(f"canary after {tag} (budget {key}): {'ok' if nd == 0 else f'{nd} words differ'}")

    canary("setup")
    # ---- timed region (headline mode)
    clk = ClockSampler(local_rank)
    ms, npipe = timed(args.mode, args.steps, args.warmup, clk)
    canary("headline")
    value = world * args.steps / (ms / 1e3)
    log(f"timed ({args.mode}): {args.steps} steps in {ms:.3f} ms -> {value:.1f} modules/s")
    if args.only or args.compose_parts != "both":   # stage analysis: not a bench line
        if rank == 0:
            print(json.dumps({"only": args.only, "compose_parts": args.compose_parts,
                              "value": round(value, 3),
                              "ms_per_step": round(ms / args.steps, 5),
                              "norm_sm_budget": args.norm_sms}), flush=True)
        return

    # ---- the other variant (inference module / training step), same protocol
    variants = {}
    other = "infer" if args.mode == "train" else "train"
    if args.variant_steps > 0:
        vsteps = args.variant_steps
        vms, _ = timed(other, vsteps, args.warmup)
        variants[other] = {
            "value": round(world * vsteps / (vms / 1e3), 3), "unit": UNIT,
            "ms_per_step": round(vms / vsteps, 5), "steps": vsteps,
            "what": ("row_norm + plain compose_fwd (inference module)" if other == "infer" else
                     "row_norm + dual compose_fwd + compose_bwd with d_mag (training step)")}
        log(f"variant {other}: {variants[other]['value']} modules/s")
        canary("variant")

    # ---- LoRA-up GEMM fused with compose + residual (layer forward
    # epilogue, training outputs y and inner) vs the unfused sequence (cuBLAS lora GEMM,
    # dual compose, residual add)
    if args.lora_steps > 0 and cfg["dtype"] != "fp32":
        b = sets[0]
        mid = torch.randn(rows, r, device=dev, generator=gen).to(tdt)
        y = torch.empty_like(b["base"])

        def batch_time(fn, n):
            with torch.cuda.stream(stream):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(n):
                    fn()
                e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) * 1e3 / n

        fused = lambda: dfx.lora_compose(mid, b["B"], b["base"], b["g"], s, y=y, inner=b["inner"])

        def unfused():
            torch.matmul(mid, b["B"].T, out=b["lora"])
            dfx.compose_fwd(b["base"], b["lora"], b["g"], s, b["delta"], b["inner"])
            torch.add(b["base"], b["delta"], out=y)

        tf, tu = batch_time(fused, args.lora_steps), batch_time(unfused, args.lora_steps)
        eb = 2
        byts = 3 * rows * d_out * eb + (rows * r + d_out * r) * eb + 4 * d_out
        peaks_hbm_l = load_peaks()[0]
        variants["layer_fwd_lora_compose"] = {
            "what": "y, inner = residual/compose(base, round(mid . B^T)) for tokens x d_out, "
                    "K = r (layer.cpp:57-120)",
            "fused_us": round(tf, 2), "unfused_us": round(tu, 2), "speedup": round(tu / tf, 3),
            "fused_hbm_gbs": round(byts / (tf * 1e-6) / 1e9, 1),
            "fused_hbm_frac": round(byts / (tf * 1e-6) / 1e9 / peaks_hbm_l, 4),
            "algorithmic_bytes": byts,
            "unfused": "cuBLAS bf16 GEMM -> lora (HBM), dfx_compose_fwd dual, torch.add residual"}
        log(f"lora_compose fused {tf:.1f} us vs unfused {tu:.1f} us")
        canary("lora")

        # ---- cached ||W||^2_row of a frozen W; W is still read
        # for the cross term, the base_sq chain is skipped.  Full GPU, rotating buffer sets.
        dfx.set_sm_budget(0)
        caches = [torch.empty(d_out, device=dev) for _ in sets]
        for c, bb in zip(caches, sets):
            dfx.row_norm_cached(bb["W"], bb["A"], bb["B"], s, cs, c, bb["wn"], refresh=True,
                                m=bb["m"], g=bb["g"])
        it = {"k": 0}

        def norm_plain():
            bb = sets[it["k"] % len(sets)]
            it["k"] += 1
            dfx.row_norm(bb["W"], bb["A"], bb["B"], s, cs, bb["wn"], m=bb["m"], g=bb["g"])

        def norm_cached():
            k = it["k"] % len(sets)
            it["k"] += 1
            bb = sets[k]
            dfx.row_norm_cached(bb["W"], bb["A"], bb["B"], s, cs, caches[k], bb["wn"], m=bb["m"],
                                g=bb["g"])

        tn, tc = batch_time(norm_plain, args.lora_steps), batch_time(norm_cached, args.lora_steps)
        variants["norm_cached_base_sq"] = {
            "what": "row_norm with ||W||^2_row cached for a frozen W (opt-in, departs from the "
                    "reference's recompute-every-call contract; bitwise equal while W is unchanged)",
            "plain_us": round(tn, 2), "cached_us": round(tc, 2), "speedup": round(tn / tc, 3)}
        log(f"row_norm plain {tn:.1f} us vs cached base_sq {tc:.1f} us")
        canary("cached")

    # ---- per-kernel live durations (event-bracketed launches, same kernels / buffers / plan
    # as the timed region).  Each step is queued behind a 2 ms device spin so the brackets
    # time the device, not the host; the kernels therefore run as in a single isolated
    # module (no neighbouring module overlaps them), so fractions divide by the BURST peaks.
    # Torch events around the row_norm call (fork to join, on the launching stream) give the
    # norm stage's wall time; around the whole step, the step's wall time.
    prof_steps = min(args.steps, args.prof_steps)
    set_budget(args.mode, npipe)
    dfx.profile(True)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(prof_steps)]
    with torch.cuda.stream(stream):
        for k in range(prof_steps):
            torch.cuda._sleep(2_000_000)
            b = sets[k % nbuf]
            ev[k][0].record(stream)
            norm(b)
            ev[k][1].record(stream)
            compose(b, args.mode)
            ev[k][2].record(stream)
    rep = dfx.profile_report()
    dfx.profile(False)
    norm_wall_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / prof_steps
    step_wall_ms = sum(e[0].elapsed_time(e[2]) for e in ev) / prof_steps
    peaks_hbm, peak_tf_burst, peak_tf_sus, peak_src = load_peaks()
    alg = algorithmic(cfg)
    kernels = {}
    for name, (n, tot, mn, mx) in rep.items():
        avg_ms = tot / n
        ent = {"launches_per_step": n / prof_steps, "avg_us": round(avg_ms * 1e3, 2),
               "min_us": round(mn * 1e3, 2),
               "share_of_step_wall": round(tot / prof_steps / step_wall_ms, 4)}
        if name in alg:
            bound, flops, byts = alg[name]
            if bound == "tensor":
                ach = flops / (avg_ms / 1e3) / 1e12
                ent.update(bound="tensor", achieved=round(ach, 1), unit="TFLOP/s",
                           frac=round(ach / peak_tf_burst, 4))
            else:
                ach = byts / (avg_ms / 1e3) / 1e9
                ent.update(bound="hbm", achieved=round(ach, 1), unit="GB/s",
                           frac=round(ach / peaks_hbm, 4))
        kernels[name] = ent
    dom = max(kernels, key=lambda k: rep[k][1])
    bound, flops, byts = alg.get(dom, ("hbm", 0.0, 0.0))
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config, {})
            budget_key = f"{dom}_budget{args.norm_sms}"
            traffic = tr.get(budget_key if (npipe > 1 and args.norm_sms > 0 and budget_key in tr)
                             else dom)
    except Exception:
        pass
    dk = kernels[dom]
    roofline = {"kernel": dom, "bound": bound, "achieved": dk.get("achieved"),
                "peak": peak_tf_burst if bound == "tensor" else peaks_hbm,
                "unit": "TFLOP/s" if bound == "tensor" else "GB/s", "frac": dk.get("frac"),
                "traffic": traffic,
                "algorithmic_per_launch": flops if bound == "tensor" else byts,
                "peak_source": f"{peak_src}: bf16 burst {peak_tf_burst} TF/s (each kernel is "
                               f"event-bracketed in an isolated module, so burst applies; "
                               f"sustained {peak_tf_sus}), HBM copy {peaks_hbm} GB/s",
                "avg_us": dk["avg_us"], "share_of_step_wall": dk["share_of_step_wall"]}
    if bound == "tensor":
        roofline["frac_of_sustained"] = round(dk["achieved"] / peak_tf_sus, 4)
    if dom == "u_rowdot_tc" and cfg["dtype"] == "bf16":
        # the SMs this launch occupies under the step's SM budget (context, not the roofline)
        try:
            u_sms, side_sms, strat = dfx.norm_plan(d_out, d_in, r, cs)
            roofline["sms_used"] = u_sms
            roofline["norm_plan"] = {"u_sms": u_sms, "side_sms": side_sms,
                                     "strategy": ["gram+V beside U", "gram beside, V after",
                                                  "serial"][strat]}
        except Exception as ex:  # noqa: BLE001 - context only, never fails the bench
            log(f"norm_plan unavailable: {ex}")
    if npipe > 1 and args.norm_sms > 0:
        # the same W.A^T GEMM planned for the whole GPU (no SM budget), timed alone
        dfx.set_sm_budget(0)
        dfx.profile(True)
        with torch.cuda.stream(stream):
            for k in range(prof_steps):
                torch.cuda._sleep(2_000_000)
                norm(sets[k % nbuf])
        rep0 = dfx.profile_report()
        dfx.profile(False)
        set_budget(args.mode, npipe)
        if dom in rep0:
            n0_, tot0, mn0, _ = rep0[dom]
            avg0 = tot0 / n0_
            work = flops if bound == "tensor" else byts
            ach0 = work / (avg0 / 1e3) / (1e12 if bound == "tensor" else 1e9)
            roofline["unbudgeted"] = {
                "avg_us": round(avg0 * 1e3, 2), "achieved": round(ach0, 1),
                "frac": round(ach0 / (peak_tf_burst if bound == "tensor" else peaks_hbm), 4),
                "note": f"the headline pipeline plans the norm GEMMs for {args.norm_sms} SMs "
                        f"(dfx_ctx_set_sm_budget) so the compose kernels run beside them; this "
                        f"is the kernel planned for all SMs"}
    if dom == "u_rowdot_tc" and cfg["dtype"] != "fp32" and bound == "tensor":
        # the same GEMM with nothing beside it: the W part of the split norm (dfx_row_norm_ba,
        # ba_sq precomputed by dfx_norm_adapter), planned for all SMs -- the setting of the ncu
        # capture in profiles/ (ncu serialises kernels, so the Gram never runs beside U there)
        try:
            dfx.set_sm_budget(0)
            bas = []
            with torch.cuda.stream(stream):
                for k in range(nbuf):
                    bb = sets[k]
                    ba = torch.empty(cfg["d_out"], device=bb["W"].device, dtype=torch.float32)
                    dfx.norm_adapter(bb["A"], bb["B"], cfg["d_out"], ba)
                    bas.append(ba)
            dfx.profile(True)
            with torch.cuda.stream(stream):
                for k in range(prof_steps):
                    torch.cuda._sleep(2_000_000)
                    bb = sets[k % nbuf]
                    dfx.row_norm_ba(bb["W"], bb["A"], bb["B"], s, cs, bas[k % nbuf], bb["wn"],
                                    m=bb["m"], g=bb["g"])
            rep1 = dfx.profile_report()
            dfx.profile(False)
            set_budget(args.mode, npipe)
            if dom in rep1:
                n1_, tot1, _, _ = rep1[dom]
                avg1 = tot1 / n1_
                ach1 = flops / (avg1 / 1e3) / 1e12
                roofline["alone"] = {
                    "avg_us": round(avg1 * 1e3, 2), "achieved": round(ach1, 1),
                    "frac": round(ach1 / peak_tf_burst, 4),
                    "note": "W.A^T planned for all SMs with no Gram beside it (dfx_row_norm_ba), the "
                            "setting of the ncu capture under profiles/; the headline frac above is "
                            "the kernel as the module runs it"}
        except Exception as ex:  # noqa: BLE001 - context only, never fails the bench
            log(f"u alone unavailable: {ex}")
    nf = alg["norm_total"][1]
    norm_roof = {"stage": "row_norm wall time (event pair around the call: fork to join)",
                 "avg_us": round(norm_wall_ms * 1e3, 2),
                 "achieved_tflops": round(nf / (norm_wall_ms / 1e3) / 1e12, 1),
                 "frac_burst": round(nf / (norm_wall_ms / 1e3) / 1e12 / peak_tf_burst, 4),
                 "step_wall_us": round(step_wall_ms * 1e3, 2)}
    # The whole step against its floors: the algorithmic bytes of every launch in one module
    # over the HBM copy peak, and its tensor flops over the burst bf16 peak (the pipelined
    # step overlaps the two, so the larger floor bounds it).
    step_bytes = sum(alg[k][2] * v["launches_per_step"] for k, v in kernels.items() if k in alg)
    step_flops = sum(alg[k][1] * v["launches_per_step"] for k, v in kernels.items() if k in alg)
    step_us = ms / args.steps * 1e3      # one module per step on each rank
    floor_us = max(step_bytes / (peaks_hbm * 1e9), step_flops / (peak_tf_burst * 1e12)) * 1e6
    step_roof = {"bytes_per_step": int(step_bytes), "flops_per_step": step_flops,
                 "hbm_floor_us": round(step_bytes / (peaks_hbm * 1e9) * 1e6, 2),
                 "tensor_floor_us": round(step_flops / (peak_tf_burst * 1e12) * 1e6, 2),
                 "step_us": round(step_us, 2), "frac_of_floor": round(floor_us / step_us, 4)}
    log(json.dumps(kernels))
    canary("profile")

    # ---- end to end through the host-buffer entry point (pinned host memory)
    e2e = None
    if args.e2e_steps > 0:
        hp = lambda t: t.cpu().pin_memory()
        b0 = sets[0]
        h = {k: hp(b0[k]) for k in ("W", "A", "B", "m", "base", "lora", "dy")}
        out = {k: torch.empty_like(h["base"]).pin_memory() for k in ("delta", "dl", "db")}
        hg = torch.empty(d_out, dtype=torch.float32).pin_memory()
        hdm = torch.empty(d_out, dtype=torch.float32).pin_memory()
        code = {torch.bfloat16: P.BF16, torch.float16: P.F16, torch.float32: P.F32}[tdt]

        def e2e_step():
            if args.mode == "infer":
                dfx.module_fwd_host(code, h["W"], h["A"], h["B"], h["m"], h["base"], h["lora"], s,
                                    d_out, d_in, r, rows, cs, out["delta"], hg)
            else:
                dfx.module_train_host(code, h["W"], h["A"], h["B"], h["m"], h["base"], h["lora"],
                                      h["dy"], s, d_out, d_in, r, rows, cs, out["delta"],
                                      out["dl"], out["db"], hdm, hg)

        # The device path's result for the same inputs under the plan the e2e call runs with
        # (the split-K Gram partition follows the SM budget, so g can differ in its last bits
        # between budgets; sets[0] was last written under another pass's budget).
        with torch.cuda.stream(stream):
            # the host entry points run the single-call norm (dfx_row_norm's plan)
            dfx.row_norm(b0["W"], b0["A"], b0["B"], s, cs, b0["wn"], m=b0["m"], g=b0["g"])
            compose(b0, args.mode)
        torch.cuda.synchronize()
        e2e_step()  # stage buffers
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e2e_s = time.perf_counter() - t0
        if dist:
            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        # result check on the host copies: the same outputs the device path produced
        torch.cuda.synchronize()
        if not torch.equal(out["delta"].to(dev), b0["delta"]):
            nd = int((out["delta"].to(dev) != b0["delta"]).sum())
            ng = int((hg.to(dev) != b0["g"]).sum())
            raise AssertionError(f"e2e delta mismatch ({nd} of {b0['delta'].numel()} elements; "
                                 f"g differs in {ng} of {d_out} rows)")
        if args.mode == "train":
            assert torch.equal(out["dl"].to(dev), b0["dl"]), "e2e d_lora mismatch"
            assert torch.equal(hdm.to(dev), b0["dm"]), "e2e d_mag mismatch"
        eb = h["W"].element_size()
        nact = rows * d_out * eb
        n_in, n_out = (2, 1) if args.mode == "infer" else (3, 3)
        e2e = {"value": round(world * args.e2e_steps / e2e_s, 2), "unit": UNIT,
               "h2d_bytes_per_step": int((d_out * d_in + r * d_in + d_out * r) * eb + n_in * nact
                                         + 4 * d_out),
               "d2h_bytes_per_step": int(n_out * nact + 4 * d_out * (1 if args.mode == "infer" else 2)),
               "api": ("dfx_module_fwd_host" if args.mode == "infer" else "dfx_module_train_host") +
                      " (pinned host buffers, H2D + kernels + D2H, blocking)",
               "steps": args.e2e_steps}
        log(f"e2e: {e2e['value']} modules/s")

    # ---- CPU reference baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = host_cores()
            rate, det = cpu_reference_rate(cfg, cores, mode=args.mode, rounds=1, warm=0, log=log,
                                           full_module=not args.no_cpu_full_module)
            cpu = {"value": round(rate, 6), "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": det["sample"], "t_module_1core_s": round(det["t_module_1core_s"], 2)}
            if det["full_module"]:
                cpu.update(det["full_module"])
        except Exception as e:
            cpu = {"value": None, "unavailable": str(e)}

    clocks = clk.summary()
    if rank == 0:
        what = ("row_norm + magnitude + dual compose_fwd + compose_bwd (d_lora, d_base, d_mag)"
                if args.mode == "train" else "row_norm + magnitude + compose_fwd")
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic (seeded torch.randn on device; m = norm*(1+N(0,0.0015)))",
            "config": {"workload": f"{args.config}: single DoRA module d_out={d_out} d_in={d_in} "
                                   f"r={r} {cfg['dtype']}, tokens={rows}: {what} per step",
                       "mode": args.mode, "d_out": d_out, "d_in": d_in, "r": r, "tokens": rows,
                       "chunk_plan": [cs, nchunks], "s": s,
                       "parallelism": f"module-sharded x{world} (no collective)",
                       "l2": f"inputs > L2 (W {d_out * d_in * 2 >> 20} MiB + activations "
                             f"{(3 if args.mode == 'infer' else 7) * rows * d_out * 2 >> 20} MiB per "
                             f"module), {nbuf} rotating module buffer sets",
                       "timing": "CUDA graphs replayed on one stream, CUDA events, max over ranks",
                       "pipeline": (f"{npipe} modules per graph; module i's compose overlaps "
                                    f"module i+1's norm on a second stream" if npipe > 1
                                    else "serial"),
                       "norm_sm_budget": args.norm_sms if npipe > 1 else 0},
            "roofline": roofline, "roofline_norm_stage": norm_roof, "roofline_step": step_roof,
            "kernels": kernels,
            "variants": variants,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step,
            "native_libs": [os.path.relpath(P.LIB_PATH, ROOT)],
        }
        print(json.dumps(line), flush=True)
    dfx.close()


# ------------------------------------------------------------------ C5 layer stack
def run_stack(args, rank, world, local_rank, dist):
    """BASELINE configs[4]: a 32B-VLM-sized stack (64 layers x q, k, v, o, gate, up, down =
    448 adapted modules, r = 384, bf16, tokens = 4096) sharded by module across the ranks
    with LPT on the modelled cost (paper_2603_22276_b200/dist.py) — strong scaling, no
    data-path collective.  One step = one pass over the whole stack (every module's norm +
    compose), pipelined on two streams like the single-module bench."""
    import torch
    import paper_2603_22276_b200 as P
    from paper_2603_22276_b200.dist import lpt_shards, module_cost, vlm32b_stack

    r, rows = 384, 4096
    s = 2.0 / math.sqrt(r)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dfx = P.Dfx(local_rank)
    log = (lambda m: print(m, file=sys.stderr, flush=True)) if rank == 0 else (lambda m: None)
    stack = vlm32b_stack()
    costs = [module_cost(d_out, d_in, r, rows) for _, d_out, d_in in stack]
    mine = lpt_shards(costs, world)[rank]
    gen = torch.Generator(device=dev)
    gen.manual_seed(20261017 + rank)
    bf = torch.bfloat16
    mods = []
    for i in mine:
        _, d_out, d_in = stack[i]
        cs, _ = P.plan_chunks(d_out, d_in)
        mods.append(dict(W=torch.randn(d_out, d_in, device=dev, generator=gen).to(bf),
                         A=torch.randn(r, d_in, device=dev, generator=gen).to(bf),
                         B=torch.randn(d_out, r, device=dev, generator=gen).to(bf),
                         wn=torch.empty(d_out, device=dev), g=torch.empty(d_out, device=dev),
                         dm=torch.empty(d_out, device=dev), cs=cs, d_out=d_out))
    # activations: two buffer sets per distinct d_out (module i uses set i % 2)
    acts = {}
    for d_out in sorted({m["d_out"] for m in mods}):
        acts[d_out] = [{k: torch.randn(rows, d_out, device=dev, generator=gen).to(bf)
                        for k in ("base", "lora", "dy")} for _ in range(2)]
        for a in acts[d_out]:
            for k in ("delta", "inner", "dl", "db"):
                a[k] = torch.empty_like(a["base"])
    for m in mods:
        dfx.row_norm(m["W"], m["A"], m["B"], s, m["cs"], m["wn"])
        m["m"] = (m["wn"] * (1.0 + 0.0015 * torch.randn(m["d_out"], device=dev, generator=gen))).contiguous()
    torch.cuda.synchronize()

    def norm(m, st):
        dfx.row_norm(m["W"], m["A"], m["B"], s, m["cs"], m["wn"], m=m["m"], g=m["g"], stream=st)

    def compose(m, a, st):
        if args.mode == "infer":
            dfx.compose_fwd(a["base"], a["lora"], m["g"], s, a["delta"], stream=st)
        else:
            dfx.compose_fwd(a["base"], a["lora"], m["g"], s, a["delta"], a["inner"], stream=st)
            dfx.compose_bwd(a["dy"], m["g"], s, a["dl"], a["db"], inner=a["inner"], w_norm=m["wn"],
                            d_mag=m["dm"], stream=st)

    stream, side = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    dfx.set_sm_budget(args.norm_sms if args.norm_sms > 0 else 0)
    with torch.cuda.stream(stream):                 # eager pass: workspace, launch count
        for i, m in enumerate(mods):
            norm(m, stream.cuda_stream)
            compose(m, acts[m["d_out"]][i % 2], stream.cuda_stream)
    torch.cuda.synchronize()
    l0 = dfx.launches
    with torch.cuda.stream(stream):
        for i, m in enumerate(mods):
            norm(m, stream.cuda_stream)
            compose(m, acts[m["d_out"]][i % 2], stream.cuda_stream)
    torch.cuda.synchronize()
    launches_per_step = dfx.launches - l0

    ev_n = [torch.cuda.Event() for _ in mods]
    ev_c = [torch.cuda.Event() for _ in mods]
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph, stream=stream):
        for i, m in enumerate(mods):
            norm(m, stream.cuda_stream)
            ev_n[i].record(stream)
            side.wait_event(ev_n[i])
            compose(m, acts[m["d_out"]][i % 2], side.cuda_stream)
            ev_c[i].record(side)
        stream.wait_event(ev_c[-1])
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup // 10)):
            gph.replay()
    torch.cuda.synchronize()
    steps = max(1, args.steps // 100)             # one step = a pass over the whole stack
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank)
    with clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(steps):
                gph.replay()
            ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = len(stack) * steps / (ms / 1e3)
    log(f"c5 stack ({args.mode}): {len(mods)} modules on rank 0, {ms / steps:.2f} ms per pass")
    if rank == 0:
        print(json.dumps({
            "metric": METRIC + " (C5 layer stack)", "value": round(value, 3), "unit": UNIT,
            "n_gpus": world, "steps": steps, "warmup": max(1, args.warmup // 10),
            "ms_per_step": round(ms / steps, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded torch.randn on device)",
            "config": {"workload": f"c5: 32B-VLM-sized stack, {len(stack)} modules (64 layers x q, k, "
                                   f"v, o, gate, up, down; hidden 5120, MLP 27648, GQA 8x128), r={r}, "
                                   f"tokens={rows}, {args.mode} per module; one step = one pass",
                       "mode": args.mode, "modules": len(stack), "modules_rank0": len(mods),
                       "parallelism": f"LPT module sharding x{world} (no collective)",
                       "pipeline": "norm of module i+1 beside compose of module i (two streams, one graph)",
                       "norm_sm_budget": args.norm_sms,
                       "l2": "W streamed from HBM (62 GB of weights), activations 226 MB+ per tensor"},
            "clocks": clk.summary(), "gpu_launches": launches_per_step * steps,
            "gpu_launches_per_step": launches_per_step, "e2e": None, "cpu_baseline": None,
            "native_libs": [os.path.relpath(P.LIB_PATH, ROOT)]}), flush=True)
    dfx.close()


# ------------------------------------------------------------------ d_in split
def run_dsplit(args, rank, world, local_rank, dist):
    """`--mode dsplit`: ONE module's factored norm with d_in split across the ranks (FSDP2 /
    TP-row style).  Rank k holds W[:, K_k], A[:, K_k] (whole
    ChunkPlan chunks), replicated B and m.  One step = dfx_norm_partial -> one all-reduce of
    {G, base_sq, cross} (r*r + 2*d_out fp32) -> dfx_norm_finish on every rank.  value = modules
    (norms) per second for the whole job (all ranks cooperate on one module per step); the
    exchange is timed separately.  --allreduce dfx uses the library's symmetric-memory kernel
    (dfx_norm_allreduce, peer loads in rank order), nccl uses torch.distributed."""
    import torch
    import paper_2603_22276_b200 as P
    from paper_2603_22276_b200.dist import SymmetricAllReduce, dsplit_bounds

    cfg = CONFIGS[args.config]
    d_out, d_in, r = cfg["d_out"], cfg["d_in"], cfg["r"]
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[cfg["dtype"]]
    s = 2.0 / math.sqrt(r)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dfx = P.Dfx(local_rank)
    cs, nchunks = P.plan_chunks(d_out, d_in)
    k0, k1 = dsplit_bounds(d_in, world, cs)[rank]
    gen = torch.Generator(device=dev)
    gen.manual_seed(20261017)                       # the same module on every rank
    W = torch.randn(d_out, d_in, device=dev, generator=gen).to(tdt)
    A = torch.randn(r, d_in, device=dev, generator=gen).to(tdt)
    B = torch.randn(d_out, r, device=dev, generator=gen).to(tdt)
    Wk, Ak = W[:, k0:k1].contiguous(), A[:, k0:k1].contiguous()
    del W
    wn = torch.empty(d_out, device=dev)
    g = torch.empty(d_out, device=dev)
    m = torch.ones(d_out, device=dev)
    n = r * r + 2 * d_out
    comm = None
    if args.allreduce == "dfx":
        comm = SymmetricAllReduce(dfx, n, group=dist.group.WORLD if dist else None)
        buf = comm.buffer()
    else:
        buf = torch.empty(n, dtype=torch.float32, device=dev)
    red = torch.empty(n, dtype=torch.float32, device=dev)
    gram, base, cross = buf[: r * r], buf[r * r: r * r + d_out], buf[r * r + d_out:]
    rg, rb, rc = red[: r * r], red[r * r: r * r + d_out], red[r * r + d_out:]
    stream = torch.cuda.current_stream(dev)

    def exchange():
        if comm is not None:
            comm.all_reduce(red)
        else:
            red.copy_(buf)
            if dist:
                dist.all_reduce(red)

    def one(evs=None):
        dfx.norm_partial(Wk, Ak, B, cs, gram, base, cross)
        if evs:
            evs[0].record(stream)
        exchange()
        if evs:
            evs[1].record(stream)
        dfx.norm_finish(B, rg, rb, rc, s, wn, m=m, g=g)

    for _ in range(max(3, args.warmup)):
        one()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    steps = args.steps
    evx = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local_rank)
    with clk:
        e0.record(stream)
        for k in range(steps):
            one(evx[k])
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    xms = sum(a.elapsed_time(b) for a, b in evx) / steps
    if dist:
        t = torch.tensor([ms, xms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, xms = float(t[0]), float(t[1])
    value = steps / (ms / 1e3)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC + " (d_in-split norm)", "value": round(value, 3), "unit": UNIT,
            "n_gpus": world, "steps": steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms / steps, 5), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (seeded torch.randn)",
            "config": {"workload": f"{args.config}: factored row norm of one module d_out={d_out} "
                                   f"d_in={d_in} r={r}, d_in split over {world} ranks",
                       "mode": "dsplit", "k_slice_rank0": [k0, k1], "chunk_plan": [cs, nchunks],
                       "allreduce": args.allreduce, "message_bytes": 4 * n,
                       "parallelism": f"d_in split x{world} (one all-reduce per module)"},
            "exchange_us": round(xms * 1e3, 2), "clocks": clk.summary(),
            "native_libs": [os.path.relpath(P.LIB_PATH, ROOT)]}), flush=True)
    if comm is not None:
        comm.close()
    dfx.close()


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """`--impl reference`: the reference's own CPU implementation (oracle/_ref, compiled
    from the unmodified reference sources) on this host's cores, same metric/config."""
    if rank != 0:
        return
    if args.config == "c5":
        run_reference_stack(args, rank, world)
        return
    cfg = CONFIGS[args.config]
    cores = host_cores()
    log = lambda m: print(m, file=sys.stderr, flush=True)
    if args.mode == "dsplit":
        args.mode = "train"
    # each round is ~2 s of all-core work; cap rounds so the run stays within minutes
    rounds = max(1, min(args.steps, 20))
    warm = min(args.warmup, 1)
    t0 = time.perf_counter()
    rate, det = cpu_reference_rate(cfg, cores, mode=args.mode, rounds=rounds, warm=warm, log=log,
                                   full_module=not args.no_cpu_full_module)
    wall = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": METRIC, "value": round(rate, 6), "unit": UNIT,
        "n_gpus": world, "steps": rounds, "steps_requested": args.steps, "warmup": warm,
        "ms_per_step": round(1e3 / rate, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (numpy, seeded)",
        "config": {"workload": f"{args.config}: reference factored_row_norm + magnitude_scale + "
                               + ("dual_output_compose + compose_backward (mag_grad)"
                                  if args.mode == "train" else "fused_compose")
                               + " (proj/src, CPU, 1 thread per module)",
                   "mode": args.mode, **{k: cfg[k] for k in ("d_out", "d_in", "r", "tokens")}},
        "cpu_baseline": {"value": round(rate, 6), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": det["sample"], **(det["full_module"] or {})},
        "e2e": {"value": round(rate, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 1),
    }
    print(json.dumps(line), flush=True)


def cpu_reference_stack(cores, mode, log=None):
    """The C5 stack on the reference's CPU path: for each distinct module shape of the
    448-module inventory (4 shapes), cpu_reference_rate measures the all-core module
    throughput of that shape (concurrent bounded samples, converted with the 1-core
    calibration that the C2 whole-module run validates); the stack's time on all cores is
    the sum over its modules of 1 / rate(shape).  Returns (stack passes/s as modules/s,
    details)."""
    from paper_2603_22276_b200.dist import vlm32b_stack
    stack = vlm32b_stack()
    shapes = sorted({(o, i) for _, o, i in stack})
    per = {}
    for d_out, d_in in shapes:
        cfg = dict(d_out=d_out, d_in=d_in, r=384, tokens=4096, dtype="bf16")
        rate, det = cpu_reference_rate(cfg, cores, mode=mode, rounds=1, warm=0, log=log)
        per[f"{d_out}x{d_in}"] = {"modules_per_s_all_cores": round(rate, 6),
                                  "t_module_1core_s": round(det["t_module_1core_s"], 2)}
    t_stack = sum(1.0 / per[f"{o}x{i}"]["modules_per_s_all_cores"] for _, o, i in stack)
    return len(stack) / t_stack, {"per_shape": per, "t_stack_all_cores_s": round(t_stack, 1),
                                  "modules": len(stack)}


def run_reference_stack(args, rank, world):
    cores = host_cores()
    log = lambda m: print(m, file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    rate, det = cpu_reference_stack(cores, args.mode if args.mode != "dsplit" else "train", log)
    wall = time.perf_counter() - t0
    sample = (f"per module shape ({', '.join(det['per_shape'])}): reference factored_row_norm "
              f"on 128 W rows + the compose on 256 of 4096 tokens per thread, {cores} threads "
              f"concurrently, converted with a 1-core calibration; stack time = sum over the "
              f"{det['modules']} modules of 1 / all-core rate of its shape = "
              f"{det['t_stack_all_cores_s']} s (extrapolated, not run end to end)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC + " (C5 layer stack)", "value": round(rate, 6),
        "unit": UNIT, "n_gpus": world, "steps": 1, "warmup": 0,
        "ms_per_step": round(det["t_stack_all_cores_s"] * 1e3, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (numpy, seeded)",
        "config": {"workload": "c5: 32B-VLM-sized stack, 448 modules, r=384, tokens=4096, one "
                               "pass = every module's norm + compose (reference, CPU)",
                   "mode": args.mode, "per_shape": det["per_shape"]},
        "cpu_baseline": {"value": round(rate, 6), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(rate, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 1)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="dfx", choices=["dfx", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS) + ["c5"])
    ap.add_argument("--nbuf", type=int, default=4)
    ap.add_argument("--only", default="", choices=["", "norm", "compose"],
                    help="analysis: time one stage of the step alone (not a bench number)")
    ap.add_argument("--capture-order", default="auto", choices=["auto", "norm-first", "module"],
                    help="graph node creation order of the pipelined step (auto: module order "
                         "for training in round 1, norm-first for both since round 2; measured, DESIGN 5.3-5.4)")
    ap.add_argument("--compose-parts", default="both", choices=["both", "fwd", "bwd"],
                    help="analysis: which training compose kernels the step runs")
    ap.add_argument("--prof-steps", type=int, default=40)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stream-priority", default="none", choices=["none", "compose", "norm"],
                    help="measurement: raise the compose or the norm stream's CUDA priority")
    ap.add_argument("--no-cpu-full-module", action="store_true",
                    help="skip the one whole module on one core that validates the CPU model")
    ap.add_argument("--pipeline", type=int, default=40,
                    help="modules per graph, software-pipelined on two streams (1 = serial)")
    ap.add_argument("--mode", default="train", choices=["train", "infer", "dsplit"],
                    help="train: norm + dual compose + backward (headline); infer: norm + compose; "
                         "dsplit: the d_in-split norm (partial, all-reduce, finish) across ranks")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--allreduce", default="dfx", choices=["dfx", "nccl"],
                    help="dsplit: the exchange of {G, base_sq, cross} (dfx symmetric-memory "
                         "kernel or NCCL through torch.distributed)")
    ap.add_argument("--norm-sms", type=int, default=-1,
                    help="SM budget of the norm GEMMs in the pipelined graph (0 = all; default: "
                         "138 for the training step, measured best of 104..148, 0 for inference)")
    ap.add_argument("--split-adapter", type=int, default=0,
                    help="1: the pipelined graph computes each module's adapter term (ba_sq = "
                         "rowquad(B, A A^T), dfx_norm_adapter) one module ahead on a third stream "
                         "and finishes the norm with dfx_row_norm_ba (measured slower at C2: "
                         "7.32k vs 7.94k training, 10.0k vs 11.8k inference; DESIGN 5.4)")
    ap.add_argument("--adapter-first", type=int, default=0,
                    help="--split-adapter: create module i+1's adapter before module i's W part")
    ap.add_argument("--adapter-sms", type=int, default=28,
                    help="--split-adapter: SMs the adapter GEMMs plan for beside the W part")
    ap.add_argument("--lora-steps", type=int, default=50,
                    help="calls timed for the fused LoRA-GEMM + compose variant (0 = skip)")
    ap.add_argument("--variant-steps", type=int, default=400,
                    help="steps for the other mode's variant line (0 = skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.norm_sms < 0:   # measured: the budget helps the C2 training pipeline only
        # (DESIGN 5.3-5.4, round 2: 138 keeps the all-SM W.A^T plan, 128 SMs, with the Gram
        # on 10 side SMs, and switches the d_mag backward to its partitioned 256-byte slabs)
        # Other configs (measured, profiles/r02_c5_budget_sweep.txt, r02_cfg_budget_sweep.txt):
        # C5, the 448-module stack of smaller modules, trains fastest at 104 (5.8-6.0k vs 5.3k
        # modules/s unbudgeted); C3 (28672 x 8192) at 120-128 in both modes (2.34k vs 1.97k
        # training, 3.80k vs 3.25k inference); C1 / C4 gain nothing measurable.
        args.norm_sms = NORM_SMS_DEFAULT.get((args.config, args.mode), 0)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: re-exec under torchrun, one rank per
        # GPU (the driver's own N > 1 command already runs under torchrun)
        sys.exit(self_launch(args.gpus))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}",
              file=sys.stderr, flush=True)
    dist = None
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.stub:
        run_stub(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    if args.config == "c5":
        run_stack(args, rank, world, local_rank, dist)
    elif args.mode == "dsplit":
        run_dsplit(args, rank, world, local_rank, dist)
    else:
        run_gpu(args, rank, world, local_rank, dist)
    if dist:
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(n: int) -> int:
    """Run this same command as n ranks under torch.distributed.run (127.0.0.1 rendezvous)."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_stub(args, rank, world):
    """Launcher check without a GPU (tests/test_bench_contract.py): the same rendezvous, barrier
    and max-over-ranks reduction as the GPU arm on gloo, a trivial CPU 'step', and rank 0's
    JSON line with the whole-job fields.  Never a bench number."""
    import torch
    import torch.distributed as tdist
    if world > 1:
        tdist.init_process_group("gloo")
    t0 = time.perf_counter()
    x = torch.ones(1024)
    for _ in range(args.steps):
        x = x * 1.0
    ms = (time.perf_counter() - t0) * 1e3
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        tdist.barrier()
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        print(json.dumps({"stub": True, "metric": METRIC, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "value": world * args.steps / max(ms / 1e3, 1e-9),
                          "ranks_reporting": world}), flush=True)
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
