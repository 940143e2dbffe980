#!/usr/bin/env python
"""Benchmark: one incremental-decoding step of bifurcated attention per "step".

Workload (BASELINE.json metric): 7B MHA decode, h = g = 32, d = 128, ctx
mc = 8192, md = 256, b = 32, bf16 (configs[1]; other configs via --config).
Synthetic seeded N(0,1) inputs resident in HBM.  L2: each timed step reads the
next of ``nsets`` rotating input sets, nsets = max(2, ceil(3 * L2 / set
bytes)), so no step finds the previous steps' data in the 126 MB L2 (C4's
24 MB sets: 16+ sets).

Prints ONE JSON line (rank 0):
  value     whole-job algorithmic HBM GB/s = bytes of the WHOLE config's step /
            max-over-ranks step time; bytes = Kc/Vc once + Kd/Vd over lens +
            q/out
  us_p10/p50/p90   per-step event times (separate pass); graph_us_per_step:
            the same K steps captured in one CUDA graph and replayed
  e2e       the same metric through the host-buffer C-ABI entry point with
            the H2D/D2H copies inside the timed region; e2e_decode_loop: the
            serving view (caches resident, per-step rows copied in)
  roofline  the dominant kernel: algorithmic bytes (or FLOPs) / its in-loop
            time = its share of the step (no-PDL per-launch events) x step time
  stream_read_peak  read-only HBM streaming kernel of this run (best of 10)
  other_configs     (default run) C2a, C3, C4, C5 timed the same way
  cpu_baseline      the fp64 oracle on a bounded row sample (rank 0, N = 1),
            all host cores and one core

Multi-GPU (torchrun, N > 1): one process per GPU; the config's step is
SHARDED over the ranks (dist.split_mode: KV head groups when N | g — the
paper's TP partition, no collective in attention — else the batch); the timed
region is the rank's attention, barrier + device timing, max over ranks
(strong scaling: total work fixed); the output all-gather is timed separately.
--impl reference: the oracle (the tier's reference arm) on host cores.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from synth import CONFIGS, alg_bytes, alg_flops, make_inputs, seed_for  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s)
FALLBACK_TF = 1590.0
OTHERS = ["mha7b_b16", "gqa", "mqa", "long", "mha7b_b32_fp8"]


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return FALLBACK_HBM, FALLBACK_TF, "fallback"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the run."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        busy = [s for s in self.samples if (num(s[6]) or 0) > 0] or self.samples
        sm = [num(s[0]) for s in busy if num(s[0]) is not None]
        mx = [num(s[1]) for s in self.samples if num(s[1]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in busy for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(busy)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


METRIC = "bifurcated decode-attn HBM GB/s (7B MHA, ctx 8k, b=32; us/step in ms_per_step)"


# ---------------------------------------------------------------------------
# reference arm: the fp64 oracle on host cores
# ---------------------------------------------------------------------------
def oracle_step_sample(cfg, inp, rows, nthreads):
    import oracle

    t0 = time.perf_counter()
    oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, scale=inp.scale,
                       rows=rows, nthreads=nthreads)
    return time.perf_counter() - t0


def cpu_inputs(cfg):
    return make_inputs(cfg, seed_for(cfg.name), device="cpu")


def pick_rows(cfg, target_s, nthreads, inp):
    """Row sample sized to about target_s seconds of oracle work."""
    import numpy as np

    probe = list(range(0, cfg.b * cfg.h, max(1, cfg.b * cfg.h // max(1, 2 * nthreads))))[:2 * nthreads]
    dt = oracle_step_sample(cfg, inp, probe, nthreads)
    per_row = dt / len(probe)
    n = int(max(nthreads, min(cfg.b * cfg.h, target_s / max(per_row, 1e-9))))
    rng = np.random.default_rng(0)
    return sorted(rng.choice(cfg.b * cfg.h, size=n, replace=False).tolist())


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    nthreads = host_cores()
    inp = cpu_inputs(cfg)
    per_step_target = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    rows = pick_rows(cfg, min(20.0, per_step_target), nthreads, inp)
    frac = len(rows) / (cfg.b * cfg.h)
    for _ in range(args.warmup):
        oracle_step_sample(cfg, inp, rows[: max(1, len(rows) // 8)], nthreads)
    times = [oracle_step_sample(cfg, inp, rows, nthreads) for _ in range(args.steps)]
    t_step = statistics.mean(times) / frac  # extrapolated full-step seconds
    value = alg_bytes(cfg) / t_step / 1e9
    sample = (f"{len(rows)} of {cfg.b * cfg.h} (sample, head) rows per step, extrapolated "
              f"linearly to the full step; fp64 C oracle, OpenMP over rows")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "b": cfg.b, "h": cfg.h, "g": cfg.g, "d": cfg.d,
                   "mc": cfg.mc, "md": cfg.md, "input_dtype": cfg.dtype},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": nthreads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def kernel_alg_bytes(cfg, name):
    """Algorithmic bytes one launch of kernel `name` must move."""
    e, ekv = cfg.elem_bytes, cfg.kv_bytes
    qo = cfg.b * cfg.h * cfg.d * e
    ctx = 2 * cfg.g * cfg.mc * cfg.d * ekv
    dec = 2 * cfg.b * cfg.g * cfg.md * cfg.d * ekv
    if name.startswith("ctx"):
        return ctx + qo
    if name.startswith("dec"):
        return dec + qo
    if name.startswith("fused"):
        return ctx + dec + 2 * qo
    return qo  # merge: writes out


def kernel_alg_flops(cfg, name):
    """Algorithmic FLOPs of one launch of kernel `name`: 4*b*h*d per key
    position it covers (QK and PV, 2 FLOP per MAC)."""
    per_pos = 4 * cfg.b * cfg.h * cfg.d
    if name.startswith("ctx"):
        return per_pos * cfg.mc
    if name.startswith("dec"):
        return per_pos * cfg.md
    if name.startswith("fused"):
        return per_pos * (cfg.mc + cfg.md)
    return 0


def set_bytes(cfg):
    """HBM footprint of one input set (+ its output)."""
    e, ekv = cfg.elem_bytes, cfg.kv_bytes
    return e * 2 * cfg.b * cfg.h * cfg.d + ekv * (2 * cfg.g * cfg.mc * cfg.d
                                                 + 2 * cfg.b * cfg.g * cfg.md * cfg.d)


def l2_bytes(dev):
    try:
        return int(torch.cuda.get_device_properties(dev).L2_cache_size)
    except Exception:
        return 126 * 2 ** 20


class Case:
    """One config's rotating input sets on this rank (its shard at N > 1)."""

    def __init__(self, ba, cfg, dev, world, rank, mode, seed_base):
        from paper_2403_08845_b200 import dist as bdist

        self.cfg = cfg
        self.l2 = l2_bytes(dev)
        self.nsets = max(2, math.ceil(3 * self.l2 / set_bytes(cfg)))
        self.sets = []
        self.kv_scales = []  # FP8 cache: (k_scale, v_scale) of each set
        for k in range(self.nsets):
            full = make_inputs(cfg, seed_base + k, device=dev)
            self.kv_scales.append((full.k_scale, full.v_scale))
            loc = bdist.shard_step(full.q, full.Kc, full.Vc, full.Kd, full.Vd, full.lens, world,
                                   rank, mode)
            loc = [t.contiguous() for t in loc]
            del full
            self.sets.append(loc)
        self.scale = float(torch.tensor(1.0 / cfg.d ** 0.5, dtype=torch.float32))
        q, Kc, _, Kd, _, _ = self.sets[0]
        self.outs = [torch.empty_like(s[0]) for s in self.sets]
        self.lses = [torch.empty(s[0].shape[:-1], dtype=torch.float32, device=dev)
                     for s in self.sets] if mode == "context" else [None] * self.nsets
        self.prob = ba.make_problem(q.shape[0], q.shape[1], Kc.shape[0], cfg.d, Kc.shape[1],
                                    Kd.shape[2], cfg.torch_dtype, self.scale, kv_dtype=Kc.dtype,
                                    k_scale=self.kv_scales[0][0], v_scale=self.kv_scales[0][1])
        self.ws = ba.alloc_workspace(self.prob, dev)
        self.L = ba.ba_launches_per_call(self.prob)
        self.names = ba.ba_launch_names(self.prob)
        self.plan = ba.ba_plan_string(self.prob)
        self.ba = ba

    def step(self, k, stream, flags=0):
        s = self.sets[k % self.nsets]
        ks, vs = self.kv_scales[k % self.nsets]
        self.ba.bifurcated_attn_decode(s[0], s[1], s[2], s[3], s[4], s[5], self.outs[k % self.nsets],
                                       self.lses[k % self.nsets], scale=self.scale,
                                       workspace=self.ws, stream=stream, flags=flags,
                                       k_scale=ks, v_scale=vs)


def ev():
    return torch.cuda.Event(enable_timing=True)


def time_case(case, args, stream, barrier, steps, warmup, soak):
    """Device timing of `steps` steps (max over ranks by the caller), the
    per-step distribution, the CUDA-graph replay and the kernel shares."""
    ba = case.ba
    for k in range(warmup):
        case.step(k, stream)
    torch.cuda.synchronize()
    t_soak = time.perf_counter()
    k = 0
    while time.perf_counter() - t_soak < soak:
        for _ in range(20):
            case.step(k, stream)
            k += 1
        torch.cuda.synchronize()
    # ---- timed region: exactly `steps` steps ----
    barrier()
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(stream)
    for k in range(steps):
        case.step(k, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_ms = e0.elapsed_time(e1)
    # ---- per-step distribution (events between steps: PDL overlap lost) ----
    evs = [(ev(), ev()) for _ in range(steps)]
    for k in range(steps):
        evs[k][0].record(stream)
        case.step(k, stream)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    per = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)

    def pct(q):
        return per[min(len(per) - 1, int(round(q * (len(per) - 1))))]

    # ---- CUDA graph: the same `steps` steps captured once and replayed ----
    graph_us = None
    try:
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=cs):
            for k in range(steps):
                case.step(k, cs)
        with torch.cuda.stream(cs):  # replay() launches on the current stream
            g.replay()
            torch.cuda.synchronize()
            g0, g1 = ev(), ev()
            g0.record(cs)
            g.replay()
            g1.record(cs)
        torch.cuda.synchronize()
        graph_us = g0.elapsed_time(g1) / steps * 1e3
        del g
    except Exception as exc:  # noqa: BLE001 - reported, not fatal
        graph_us = f"capture failed: {exc}"
    # ---- kernel shares: per-launch events with PDL off (true durations) ----
    shares = [1.0]
    iso = None
    if case.L > 1:
        timer = ba.LaunchTimer(case.L, steps)
        for k in range(steps):
            timer.arm(k)
            case.step(k, stream, flags=ba.BA_FLAG_NO_PDL)
        ba.LaunchTimer.disarm()
        torch.cuda.synchronize()
        iso = timer.per_launch_ms()
        tot = sum(iso)
        shares = [x / tot for x in iso]
    return {"ms_step": t_ms / steps, "p10": pct(0.1), "p50": pct(0.5), "p90": pct(0.9),
            "graph_us": graph_us, "shares": shares, "iso_ms": iso}


def roofline(cfg, names, shares, ms_step, peak_gbs, peak_tf, traffic):
    """Dominant kernel: its in-loop time = share x step time (<= the step)."""
    kdom = max(range(len(names)), key=lambda k: shares[k])
    t_k = shares[kdom] * ms_step * 1e-3
    kb = kernel_alg_bytes(cfg, names[kdom])
    kf = kernel_alg_flops(cfg, names[kdom])
    tensor_bound = kf / max(kb, 1) > peak_tf * 1e12 / (peak_gbs * 1e9)
    base = {"kernel": names[kdom], "share_of_step": shares[kdom], "kernel_us": t_k * 1e6,
            "alg_bytes_per_launch": kb, "alg_flops_per_launch": kf, "traffic": traffic,
            "time_source": "step time (one launch per step)" if len(names) == 1 else
            "share of the step from per-launch CUDA events with PDL off x device step time"}
    if tensor_bound:
        a = kf / t_k / 1e12
        return dict(base, bound="tensor", achieved=a, peak=peak_tf, unit="TFLOP/s",
                    frac=a / peak_tf)
    a = kb / t_k / 1e9
    return dict(base, bound="hbm", achieved=a, peak=peak_gbs, unit="GB/s", frac=a / peak_gbs)


def stream_peak(ba, dev, stream):
    """Read-only streaming kernel over 2 GiB, best of 10 (GB/s)."""
    buf = torch.empty(2 * 2 ** 30, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    sink = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(2):
        ba.stream_read_bench(buf, sink, stream=stream)
    best = 0.0
    for _ in range(10):
        a, b = ev(), ev()
        a.record(stream)
        ba.stream_read_bench(buf, sink, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        best = max(best, buf.numel() / (a.elapsed_time(b) * 1e-3) / 1e9)
    del buf
    return best


def replicated(ba, cfg, case, stream, steps):
    """Non-bifurcated baseline and torch SDPA on the replicated cache."""
    s = case.sets[0]
    q, Kc, Vc, Kd, Vd, lens = s
    try:
        K = torch.cat([Kc.unsqueeze(0).expand(cfg.b, -1, -1, -1), Kd], dim=2).contiguous()
        V = torch.cat([Vc.unsqueeze(0).expand(cfg.b, -1, -1, -1), Vd], dim=2).contiguous()
    except torch.cuda.OutOfMemoryError:
        return {"oom": True}
    o = torch.empty_like(q)
    ks, vs = case.kv_scales[0]
    for _ in range(3):
        ba.replicated_attn_decode(q, K, V, lens, cfg.mc, o, scale=case.scale, stream=stream,
                                  k_scale=ks, v_scale=vs)
    torch.cuda.synchronize()
    r0, r1 = ev(), ev()
    nrep = max(3, min(steps, 20))
    r0.record(stream)
    for _ in range(nrep):
        ba.replicated_attn_decode(q, K, V, lens, cfg.mc, o, scale=case.scale, stream=stream,
                                  k_scale=ks, v_scale=vs)
    r1.record(stream)
    torch.cuda.synchronize()
    rep_ms = r0.elapsed_time(r1) / nrep
    rep_bytes = 2 * cfg.kv_bytes * cfg.d * cfg.g * cfg.b * (cfg.mc + cfg.md) \
        + 2 * cfg.elem_bytes * cfg.b * cfg.h * cfg.d
    rep = {"us_per_step": rep_ms * 1e3, "kv_bytes_moved": rep_bytes,
           "gbs_of_its_bytes": rep_bytes / (rep_ms * 1e-3) / 1e9}
    if bool((lens == cfg.md).all()) and not cfg.kv:
        qs = q.unsqueeze(2)

        def sdpa():
            return torch.nn.functional.scaled_dot_product_attention(
                qs, K, V, scale=case.scale, enable_gqa=cfg.g != cfg.h)

        with torch.cuda.stream(stream):
            for _ in range(3):
                sdpa()
            torch.cuda.synchronize()
            r0.record(stream)
            for _ in range(nrep):
                sdpa()
            r1.record(stream)
        torch.cuda.synchronize()
        rep["torch_sdpa_us_per_step"] = r0.elapsed_time(r1) / nrep * 1e3
    del K, V
    return rep


def e2e_runs(ba, cfg, case, dev, stream, barrier, steps):
    """The contract's e2e (all inputs copied from pinned host memory each
    step) and the decode-loop serving view."""
    q, Kc, Vc, Kd, Vd, lens = case.sets[0]
    ks, vs = case.kv_scales[0]
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    hq, hKc, hVc, hKd, hVd, hl = map(pin, (q, Kc, Vc, Kd, Vd, lens))
    hout = torch.empty_like(hq).pin_memory()
    dbuf = ba.make_device_buffers(hq, hKc, hKd, dev, scale=case.scale)
    for _ in range(2):
        ba.bifurcated_attn_decode_host(hq, hKc, hVc, hKd, hVd, hl, hout, dbuf, scale=case.scale,
                                       stream=stream, k_scale=ks, v_scale=vs)
    torch.cuda.synchronize()
    ne = max(2, min(steps, 10))
    barrier()
    torch.cuda.synchronize()
    a0, a1 = ev(), ev()
    a0.record(stream)
    for _ in range(ne):
        ba.bifurcated_attn_decode_host(hq, hKc, hVc, hKd, hVd, hl, hout, dbuf, scale=case.scale,
                                       stream=stream, k_scale=ks, v_scale=vs)
    a1.record(stream)
    torch.cuda.synchronize()
    barrier()
    res = {"ms_per_step": a0.elapsed_time(a1) / ne,
           "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in (hq, hKc, hVc, hKd, hVd, hl)),
           "d2h_bytes_per_step": hout.numel() * hout.element_size()}
    del dbuf
    # decode loop: caches resident; ONE H2D of the packed [q | k_new | v_new |
    # lens], append + attend, ONE D2H of out (bifurcated_attn_decode_step_packed),
    # the whole step replayed from a CUDA graph
    b, g = Kd.shape[0], Kd.shape[1]
    hkn = torch.randn(b, g, 1, cfg.d).to(Kd.dtype)
    hvn = torch.randn(b, g, 1, cfg.d).to(Kd.dtype)
    hl1 = (lens.cpu() - 1).clamp_min(0).to(torch.int32)
    step = ba.PackedStep(case.prob, Kc, Vc, Kd.clone(), Vd.clone(), dev)
    step.pack(q.cpu(), hkn, hvn, hl1)
    cs = torch.cuda.Stream()
    step.run(stream=cs)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=cs):
        for _ in range(ne):
            step.run(stream=cs)
    with torch.cuda.stream(cs):
        graph.replay()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        a0.record(cs)
        graph.replay()
        a1.record(cs)
    torch.cuda.synchronize()
    barrier()
    res["loop_ms"] = a0.elapsed_time(a1) / ne
    res["loop_h2d"] = step.h_in.numel()
    res["loop_d2h"] = step.nq
    # the same steps without the graph (one C-ABI call per step)
    torch.cuda.synchronize()
    a0.record(cs)
    for _ in range(ne):
        step.run(stream=cs)
    a1.record(cs)
    torch.cuda.synchronize()
    res["loop_nograph_ms"] = a0.elapsed_time(a1) / ne
    return res


def time_gather(case, world, mode, stream, steps):
    from paper_2403_08845_b200 import dist as bdist

    out = case.outs[0]
    for _ in range(3):
        bdist.assemble(out, case.lses[0], case.cfg.b, world, mode, stream=stream)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    a, b = ev(), ev()
    a.record(stream)
    n = max(3, min(steps, 20))
    for _ in range(n):
        bdist.assemble(out, case.lses[0], case.cfg.b, world, mode, stream=stream)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


def run_other(ba, name, dev, stream, peak_gbs, peak_tf):
    cfg = CONFIGS[name]
    case = Case(ba, cfg, dev, 1, 0, "single", seed_for(name))
    clocks = ClockSampler(gpu_index())
    clocks.start()
    t = time_case(case, None, stream, lambda: None, steps=20, warmup=3, soak=0.3)
    clocks.stop()
    ms = t["ms_step"]
    roof = roofline(cfg, case.names, t["shares"], ms, peak_gbs, peak_tf, load_traffic(name))
    res = {"us_per_step": ms * 1e3, "us_p10": t["p10"], "us_p50": t["p50"], "us_p90": t["p90"],
           "graph_us_per_step": t["graph_us"], "alg_bytes": alg_bytes(cfg),
           "gbs": alg_bytes(cfg) / (ms * 1e-3) / 1e9,
           "frac_of_hbm_peak": alg_bytes(cfg) / (ms * 1e-3) / 1e9 / peak_gbs,
           "tflops": alg_flops(cfg) / (ms * 1e-3) / 1e12, "plan": case.plan,
           "nsets": case.nsets, "kernels": {case.names[k]: {"share": t["shares"][k]}
                                            for k in range(case.L)},
           "roofline": {k: roof[k] for k in ("bound", "kernel", "achieved", "unit", "frac",
                                             "share_of_step")},
           "clocks": clocks.summary()}
    del case
    torch.cuda.empty_cache()
    return res


def gpu_index():
    _, _, local = dist_env()
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    return cvd.split(",")[local] if cvd else str(local)


def run_ours(args, cfg):
    import paper_2403_08845_b200 as ba
    from paper_2403_08845_b200 import dist as bdist

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    peak_gbs, peak_tf, peak_kind = peaks()
    mode = bdist.split_mode(cfg.b, cfg.h, cfg.g, cfg.mc, ws)
    # every rank draws the SAME full problem (same seeds) and keeps its shard:
    # the union of the ranks' work is exactly the single-GPU step
    case = Case(ba, cfg, dev, ws, rank, mode, seed_for(cfg.name))
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    clocks = ClockSampler(gpu_index())
    clocks.start()
    t = time_case(case, args, stream, barrier, args.steps, args.warmup, args.soak)
    clocks.stop()

    gather_us = time_gather(case, ws, mode, stream, args.steps) if ws > 1 else None
    rep = None
    if ws == 1 and not args.no_replicated:
        rep = replicated(ba, cfg, case, stream, args.steps)
        if "us_per_step" in rep:
            rep["speedup_bifurcated_over_replicated"] = rep["us_per_step"] / (t["ms_step"] * 1e3)
        if "torch_sdpa_us_per_step" in rep:
            rep["speedup_bifurcated_over_torch_sdpa"] = rep["torch_sdpa_us_per_step"] / (t["ms_step"] * 1e3)
    e2e = None if args.no_e2e else e2e_runs(ba, cfg, case, dev, stream, barrier, args.steps)
    speak = stream_peak(ba, dev, stream) if not args.no_stream_peak else None

    # ---- max over ranks ----
    vals = torch.tensor([t["ms_step"], e2e["ms_per_step"] if e2e else 0.0,
                         e2e["loop_ms"] if e2e else 0.0, gather_us or 0.0,
                         t["graph_us"] if isinstance(t["graph_us"], float) else 0.0,
                         t["p50"], t["p10"], t["p90"]], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    ms_step, e2e_ms, loop_ms, gather_us, graph_us, p50, p10, p90 = [float(x) for x in vals]

    names, nsets, plan = case.names, case.nsets, case.plan
    others = {}
    if ws == 1 and rank == 0 and not args.no_others and cfg.name == "mha7b_b32":
        del case
        torch.cuda.empty_cache()
        for name in OTHERS:
            try:
                others[name] = run_other(ba, name, dev, stream, peak_gbs, peak_tf)
            except Exception as exc:  # noqa: BLE001 - reported in the line
                others[name] = {"error": repr(exc)[:300]}
        case = None

    if rank == 0:
        bytes_step = alg_bytes(cfg)
        value = bytes_step / (ms_step * 1e-3) / 1e9
        shares = t["shares"]
        # roofline on the rank-local kernel: local bytes / local kernel time
        local_cfg = local_config(cfg, ws, mode)
        roof = roofline(local_cfg, names, shares, ms_step, peak_gbs, peak_tf, args.traffic if ws == 1 else None)
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "us_per_step": ms_step * 1e3, "us_p10": p10, "us_p50": p50, "us_p90": p90,
            "graph_us_per_step": graph_us if graph_us > 0 else t["graph_us"],
            "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": cfg.dtype + ("/e4m3-kv" if cfg.kv else ""),
            "data": "synthetic",
            "config": {"workload": cfg.name, "b": cfg.b, "h": cfg.h, "g": cfg.g, "d": cfg.d,
                       "mc": cfg.mc, "md": cfg.md, "alg_bytes_per_step": bytes_step,
                       "alg_flops_per_step": alg_flops(cfg),
                       "parallelism": f"{mode}{ws}" if ws > 1 else "single",
                       "l2": (f"{nsets} rotating input sets of "
                              f"{set_bytes(local_cfg) / 1e6:.1f} MB (>= 3x the "
                              f"{l2_bytes(dev) / 2 ** 20:.0f} MiB L2 between re-reads)"),
                       "plan": plan},
            "frac_of_hbm_peak": value / ws / peak_gbs, "frac_of_8tbs": value / ws / 8000.0,
            "peak_kind": peak_kind,
            "gpu_launches": len(shares) * args.steps,
            "kernels": {names[k] if k < len(names) else f"k{k}":
                        {"share": shares[k], "us_in_step": shares[k] * ms_step * 1e3,
                         "us_alone_no_pdl": (t["iso_ms"][k] * 1e3 if t["iso_ms"] else None)}
                        for k in range(len(shares))},
            "roofline": roof,
            "clocks": clocks.summary(),
            "replicated_baseline": rep,
        }
        if ws > 1:
            line["gather_us"] = gather_us
            line["split"] = mode
        if speak:
            line["stream_read_peak"] = {"gbs": speak, "frac_of_measured_copy_peak": speak / peak_gbs,
                                        "step_frac_of_it": value / ws / speak,
                                        "how": "ba_stream_read_bench over 2 GiB, best of 10"}
        if e2e:
            line["e2e"] = {"value": bytes_step / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                           "ms_per_step": e2e_ms,
                           "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                           "d2h_bytes_per_step": e2e["d2h_bytes_per_step"]}
            line["e2e_decode_loop"] = {
                "value": bytes_step / (loop_ms * 1e-3) / 1e9, "unit": "GB/s",
                "ms_per_step": loop_ms, "h2d_bytes_per_step": e2e["loop_h2d"],
                "d2h_bytes_per_step": e2e["loop_d2h"],
                "ms_per_step_without_graph": e2e.get("loop_nograph_ms"),
                "api": "bifurcated_attn_decode_step_packed: caches resident; one H2D of "
                       "[q | k_new | v_new | lens], append + attend fused, one D2H of out; "
                       "steps replayed from a CUDA graph"}
        if others:
            line["other_configs"] = others
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def local_config(cfg, ws, mode):
    if mode == "heads":
        return cfg.with_(h=cfg.h // ws, g=cfg.g // ws)
    if mode == "batch":
        return cfg.with_(b=-(-cfg.b // ws))
    if mode == "context":
        return cfg.with_(mc=-(-cfg.mc // ws))
    return cfg


def cpu_baseline(cfg, seconds):
    """The oracle as it stands on a bounded row sample: all host cores, then one
    core on a smaller sample; both extrapolated linearly to the full step."""
    nthreads = host_cores()
    inp = cpu_inputs(cfg)
    rows = pick_rows(cfg, seconds, nthreads, inp)
    dt = oracle_step_sample(cfg, inp, rows, nthreads)
    t_step = dt / (len(rows) / (cfg.b * cfg.h))
    rows1 = rows[: max(1, len(rows) // max(1, nthreads) // 2)]
    dt1 = oracle_step_sample(cfg, inp, rows1, 1)
    t1 = dt1 / (len(rows1) / (cfg.b * cfg.h))
    return {"value": alg_bytes(cfg) / t_step / 1e9, "unit": "GB/s", "cores": nthreads,
            "kind": "oracle", "ms_per_step": t_step * 1e3,
            "single_thread": {"value": alg_bytes(cfg) / t1 / 1e9, "ms_per_step": t1 * 1e3,
                              "sample": f"{len(rows1)} rows ({dt1:.1f} s)"},
            "sample": f"{len(rows)} of {cfg.b * cfg.h} rows of one step ({dt:.1f} s), "
                      f"extrapolated linearly to the full step"}


def load_traffic(name):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mha7b_b32", choices=list(CONFIGS))
    ap.add_argument("--soak", type=float, default=1.0, help="seconds of untimed steps for clocks")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-replicated", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-others", action="store_true", help="skip the other configs")
    ap.add_argument("--no-stream-peak", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (from profiles/)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.traffic is None:
        args.traffic = load_traffic(cfg.name)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
