"""Interleaved A/B timing of flag variants on one config (medians over rounds)."""
import sys, os, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs, alg_bytes

name = sys.argv[1] if len(sys.argv) > 1 else "mha7b_b32"
variants = {"default": 0}
cfg = CONFIGS[name]
sets = [make_inputs(cfg, 1 + k, device="cuda") for k in range(2)]
outs = [torch.empty_like(s.q) for s in sets]
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, sets[0].scale)
ws = ba.alloc_workspace(prob, "cuda")
def timeit(flags, iters=40):
    def step(k):
        s = sets[k % 2]
        ba.bifurcated_attn_decode(s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, outs[k % 2], workspace=ws, scale=s.scale, flags=flags)
    for k in range(5): step(k)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(iters): step(k)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3
res = {v: [] for v in variants}
for r in range(7):
    for v, f in variants.items():
        res[v].append(timeit(f))
for v in variants:
    us = statistics.median(res[v])
    print(json.dumps({"cfg": name, "variant": v, "us_med": round(us, 2), "us_min": round(min(res[v]), 2), "GBs": round(alg_bytes(cfg) / us / 1e3, 1)}))
