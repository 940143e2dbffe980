#!/usr/bin/env python
"""Benchmark: one incremental-decoding step of bifurcated attention per "step".

Workload (BASELINE.json metric): 7B MHA decode, h = g = 32, d = 128, ctx
mc = 8192, md = 256, b = 32, bf16 (configs[1]; b = 16 via --config mha7b_b16).
Synthetic seeded N(0,1) inputs resident in HBM.  L2: each timed step reads one
of two rotating input sets (2 x 269 MB >> 126 MB L2), so no step re-reads the
previous step's data from L2.

Prints ONE JSON line (rank 0):
  value    whole-job algorithmic HBM GB/s = (bytes of all ranks' steps) / time,
           bytes per step = Kc/Vc once + Kd/Vd over lens + q/out
  e2e      same metric through the host-buffer C-ABI entry point with H2D/D2H
           copies inside the timed region
  roofline the dominant kernel's algorithmic bytes / its mean CUDA-event time
  cpu_baseline  the fp64 oracle on a bounded row sample (rank 0, N = 1)

Multi-GPU (torchrun): one process per GPU; each rank runs its own head-group
shard (weak scaling: per-rank work fixed = the config), no data-path
collective; barrier + device timing, max over ranks.
--impl reference: the oracle (the tier's reference arm) on host cores.
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

import torch  # noqa: E402

from synth import CONFIGS, alg_bytes, alg_flops, make_inputs, seed_for  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s)
FALLBACK_TF = 1590.0


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

    def __init__(self, gpu_index: int):
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
    rows = sorted(rng.choice(cfg.b * cfg.h, size=n, replace=False).tolist())
    return rows


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
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "b": cfg.b, "h": cfg.h, "g": cfg.g, "d": cfg.d,
                   "mc": cfg.mc, "md": cfg.md, "input_dtype": cfg.dtype},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": nthreads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "bifurcated decode-attn HBM GB/s (7B MHA, ctx 8k, b=32; us/step in ms_per_step)"


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import paper_2403_08845_b200 as ba

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    peak_gbs, peak_tf, peak_kind = peaks()

    # Per-rank problem: weak scaling, every rank owns a full head-group set of
    # the config (its shard of an N-times-wider job); seeds differ per rank.
    nsets = 2
    sets = [make_inputs(cfg, seed_for(cfg.name) + 1000 * rank + k, device=dev) for k in range(nsets)]
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype,
                           sets[0].scale)
    wsbuf = ba.alloc_workspace(prob, dev)
    outs = [torch.empty_like(s.q) for s in sets]
    L = ba.ba_launches_per_call(prob)
    names = ba.ba_launch_names(prob)
    stream = torch.cuda.current_stream()

    def step(k):
        s = sets[k % nsets]
        ba.bifurcated_attn_decode(s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, outs[k % nsets],
                                  scale=s.scale, workspace=wsbuf, stream=stream)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    clocks = ClockSampler(cvd.split(",")[local] if cvd else str(local))
    clocks.start()
    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    # soak so the clock sampler sees the step under load for >= ~1 s
    t_soak = time.perf_counter()
    k = 0
    while time.perf_counter() - t_soak < args.soak:
        for _ in range(50):
            step(k)
            k += 1
        torch.cuda.synchronize()

    # ---- timed region: exactly K steps -------------------------------------
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        step(k)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_ms = e0.elapsed_time(e1)
    clocks.stop()

    # ---- per-kernel CUDA-event timing (separate pass, same steps) ---------
    timer = ba.LaunchTimer(L, args.steps)
    for k in range(args.steps):
        timer.arm(k)
        step(k)
    ba.LaunchTimer.disarm()
    torch.cuda.synchronize()
    per_launch = timer.per_launch_ms()

    # ---- replicated-KV baseline, same timing protocol -------
    rep = None
    if not args.no_replicated:
        try:
            s = sets[0]
            K = torch.cat([s.Kc.unsqueeze(0).expand(cfg.b, -1, -1, -1), s.Kd], dim=2).contiguous()
            V = torch.cat([s.Vc.unsqueeze(0).expand(cfg.b, -1, -1, -1), s.Vd], dim=2).contiguous()
            o = torch.empty_like(s.q)
            for _ in range(3):
                ba.replicated_attn_decode(s.q, K, V, s.lens, cfg.mc, o, scale=s.scale,
                                          workspace=wsbuf, stream=stream)
            torch.cuda.synchronize()
            r0 = torch.cuda.Event(enable_timing=True)
            r1 = torch.cuda.Event(enable_timing=True)
            nrep = max(3, min(args.steps, 20))
            r0.record(stream)
            for _ in range(nrep):
                ba.replicated_attn_decode(s.q, K, V, s.lens, cfg.mc, o, scale=s.scale,
                                          workspace=wsbuf, stream=stream)
            r1.record(stream)
            torch.cuda.synchronize()
            rep_ms = r0.elapsed_time(r1) / nrep
            rep_bytes = 2 * cfg.elem_bytes * cfg.d * cfg.g * cfg.b * (cfg.mc + cfg.md) \
                + 2 * cfg.elem_bytes * cfg.b * cfg.h * cfg.d
            rep = {"us_per_step": rep_ms * 1e3, "kv_bytes_moved": rep_bytes,
                   "gbs_of_its_bytes": rep_bytes / (rep_ms * 1e-3) / 1e9,
                   "speedup_bifurcated_over_replicated": rep_ms / (t_ms / args.steps)}
            # library reference on the same replicated cache (SURVEY §8(d)
            # baseline 2): torch SDPA (its own fused kernels), uniform lens only
            if bool((s.lens == cfg.md).all()):
                qs = s.q.unsqueeze(2)  # [b, h, 1, d]
                sdpa = lambda: torch.nn.functional.scaled_dot_product_attention(  # noqa: E731
                    qs, K, V, scale=s.scale, enable_gqa=cfg.g != cfg.h)
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        sdpa()
                    torch.cuda.synchronize()
                    r0.record(stream)
                    for _ in range(nrep):
                        sdpa()
                    r1.record(stream)
                torch.cuda.synchronize()
                sd_ms = r0.elapsed_time(r1) / nrep
                rep["torch_sdpa_us_per_step"] = sd_ms * 1e3
                rep["speedup_bifurcated_over_torch_sdpa"] = sd_ms / (t_ms / args.steps)
            del K, V
        except torch.cuda.OutOfMemoryError:
            rep = {"oom": True}

    # ---- end to end through the host-buffer C-ABI entry point -------------
    e2e = None
    if not args.no_e2e:
        s = sets[0]
        pin = lambda t: t.cpu().pin_memory()  # noqa: E731
        hq, hKc, hVc, hKd, hVd, hl = map(pin, (s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens))
        hout = torch.empty_like(hq).pin_memory()
        dbuf = ba.make_device_buffers(hq, hKc, hKd, dev, scale=s.scale)
        for _ in range(2):
            ba.bifurcated_attn_decode_host(hq, hKc, hVc, hKd, hVd, hl, hout, dbuf, scale=s.scale,
                                           stream=stream)
        torch.cuda.synchronize()
        ne = max(2, min(args.steps, 10))
        barrier()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(ne):
            ba.bifurcated_attn_decode_host(hq, hKc, hVc, hKd, hVd, hl, hout, dbuf, scale=s.scale,
                                           stream=stream)
        a1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = a0.elapsed_time(a1) / ne
        h2d = sum(t.numel() * t.element_size() for t in (hq, hKc, hVc, hKd, hVd, hl))
        d2h = hout.numel() * hout.element_size()
        e2e = {"ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
        # the decode-loop view of the same step: the caches stay resident in HBM
        # (model state); each step copies in this step's q, K/V rows and lens
        # from pinned host memory, appends + attends in one call
        # (bifurcated_attn_decode_append) and reads the output back
        s = sets[0]
        hkn = torch.randn(cfg.b, cfg.g, 1, cfg.d).to(s.q.dtype).pin_memory()
        hvn = torch.randn(cfg.b, cfg.g, 1, cfg.d).to(s.q.dtype).pin_memory()
        hl1 = (s.lens.cpu() - 1).clamp_min(0).to(torch.int32).pin_memory()
        cs = torch.cuda.Stream()
        loop_dev = dict(q=torch.empty_like(s.q), k_new=torch.empty_like(hkn, device=dev),
                        v_new=torch.empty_like(hvn, device=dev), Kc=s.Kc, Vc=s.Vc,
                        Kd=s.Kd.clone(), Vd=s.Vd.clone(), lens=torch.empty_like(s.lens),
                        out=torch.empty_like(s.q), workspace=ba.alloc_workspace(prob, dev))

        def loop_step():
            # one C-ABI call: H2D of q, K/V rows, lens; append + attend; D2H of out
            ba.bifurcated_attn_decode_append_host(hq, hkn, hvn, hout, loop_dev, hlens=hl1,
                                                  scale=s.scale, stream=cs)
        for _ in range(2):
            loop_step()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        a0.record(cs)
        for _ in range(ne):
            loop_step()
        a1.record(cs)
        torch.cuda.synchronize()
        barrier()
        e2e["loop_ms"] = a0.elapsed_time(a1) / ne
        e2e["loop_h2d"] = sum(t.numel() * t.element_size() for t in (hq, hkn, hvn, hl1))
        e2e["loop_d2h"] = hout.numel() * hout.element_size()

    # ---- max over ranks ----------------------------------------------------
    ms_step = t_ms / args.steps
    vals = torch.tensor([ms_step, e2e["ms_per_step"] if e2e else 0.0,
                         e2e["loop_ms"] if e2e else 0.0] + per_launch,
                        dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    ms_step, e2e_ms, loop_ms = float(vals[0]), float(vals[1]), float(vals[2])
    per_launch = [float(x) for x in vals[3:]]

    if rank == 0:
        bytes_step = alg_bytes(cfg)
        value = ws * bytes_step / (ms_step * 1e-3) / 1e9
        # dominant kernel: the longest launch
        kdom = max(range(L), key=lambda k: per_launch[k])
        kb = kernel_alg_bytes(cfg, names[kdom])
        kf = kernel_alg_flops(cfg, names[kdom])
        achieved = kb / (per_launch[kdom] * 1e-3) / 1e9
        # a kernel whose algorithmic intensity is past the ridge of the measured
        # peaks (C4: ~1100 FLOP/B vs ~250) is tensor-bound: report TFLOP/s
        tensor_bound = kf / max(kb, 1) > peak_tf * 1e12 / (peak_gbs * 1e9)
        if tensor_bound:
            roof = {"bound": "tensor", "kernel": names[kdom],
                    "achieved": kf / (per_launch[kdom] * 1e-3) / 1e12, "peak": peak_tf,
                    "unit": "TFLOP/s", "frac": kf / (per_launch[kdom] * 1e-3) / 1e12 / peak_tf,
                    "traffic": args.traffic, "alg_flops_per_launch": kf,
                    "alg_bytes_per_launch": kb, "share_of_step": per_launch[kdom] / ms_step}
        else:
            roof = {"bound": "hbm", "kernel": names[kdom], "achieved": achieved,
                    "peak": peak_gbs, "unit": "GB/s", "frac": achieved / peak_gbs,
                    "traffic": args.traffic, "alg_bytes_per_launch": kb,
                    "share_of_step": per_launch[kdom] / ms_step}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "us_per_step": ms_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": cfg.name, "b": cfg.b, "h": cfg.h, "g": cfg.g, "d": cfg.d,
                       "mc": cfg.mc, "md": cfg.md, "alg_bytes_per_step": bytes_step,
                       "alg_flops_per_step": alg_flops(cfg), "parallelism": f"headgroups{ws}",
                       "l2": "2 rotating input sets of %.0f MB each (> 126 MB L2)" % (bytes_step / 1e6),
                       "plan": ba.ba_plan_string(prob)},
            "frac_of_hbm_peak": value / ws / peak_gbs, "frac_of_8tbs": value / ws / 8000.0,
            "peak_kind": peak_kind,
            "gpu_launches": L * args.steps,
            "kernels": {names[k]: {"us": per_launch[k] * 1e3} for k in range(L)},
            "roofline": roof,
            "clocks": clocks.summary(),
            "replicated_baseline": rep,
        }
        if e2e:
            line["e2e"] = {"value": ws * bytes_step / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                           "ms_per_step": e2e_ms,
                           "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                           "d2h_bytes_per_step": e2e["d2h_bytes_per_step"]}
            line["e2e_decode_loop"] = {
                "value": ws * bytes_step / (loop_ms * 1e-3) / 1e9, "unit": "GB/s",
                "ms_per_step": loop_ms, "h2d_bytes_per_step": e2e["loop_h2d"],
                "d2h_bytes_per_step": e2e["loop_d2h"],
                "api": "bifurcated_attn_decode_append_host: one call per step (caches resident; "
                       "q, K/V rows, lens copied in, out copied back)"}
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def kernel_alg_bytes(cfg, name):
    """Algorithmic bytes one launch of kernel `name` must move."""
    e = cfg.elem_bytes
    qo = cfg.b * cfg.h * cfg.d * e
    ctx = 2 * cfg.g * cfg.mc * cfg.d * e
    dec = 2 * cfg.b * cfg.g * cfg.md * cfg.d * e
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


def cpu_baseline(cfg, seconds):
    nthreads = host_cores()
    inp = cpu_inputs(cfg)
    rows = pick_rows(cfg, seconds, nthreads, inp)
    dt = oracle_step_sample(cfg, inp, rows, nthreads)
    frac = len(rows) / (cfg.b * cfg.h)
    t_step = dt / frac
    return {"value": alg_bytes(cfg) / t_step / 1e9, "unit": "GB/s", "cores": nthreads,
            "kind": "oracle", "ms_per_step": t_step * 1e3,
            "sample": f"{len(rows)} of {cfg.b * cfg.h} rows of one step ({dt:.1f} s), "
                      f"extrapolated linearly to the full step"}


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


def load_traffic(name):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(name)
    except Exception:
        return None


if __name__ == "__main__":
    main()
