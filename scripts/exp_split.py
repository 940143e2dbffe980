"""Timing experiments: fused kernel on context-only / decode-only / both."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs, alg_bytes

def t_call(fn, iters=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3

base = CONFIGS["mha7b_b32"]
for name, cfg in [("ctx_only", base.with_(md=0)), ("full", base), ("b16", CONFIGS["mha7b_b16"]),
                  ("mc4096", base.with_(mc=4096)), ("md1024", base.with_(md=1024, mc=2048))]:
    inp = make_inputs(cfg, 1, device="cuda")
    out = torch.empty_like(inp.q)
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
    ws = ba.alloc_workspace(prob, "cuda")
    us = t_call(lambda: ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, workspace=ws, scale=inp.scale))
    print(json.dumps({"name": name, "us": us, "GBs": alg_bytes(cfg) / us / 1e3, "plan": ba.ba_plan_string(prob)}), flush=True)
    if name == "full":
        us2 = t_call(lambda: ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, workspace=ws, scale=inp.scale, flags=ba.BA_FLAG_FORCE_FMA))
        print(json.dumps({"name": "full_fma", "us": us2, "GBs": alg_bytes(cfg) / us2 / 1e3}), flush=True)
