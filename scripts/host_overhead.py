"""Host cost of one bifurcated_attn_decode() call through the Python binding
and the device time of back-to-back steps (C2b): is the event-timed loop
host-bound?"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_08845_b200 as ba  # noqa: E402
from synth import CONFIGS, make_inputs, seed_for  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mha7b_b32"]
inp = make_inputs(cfg, seed_for(cfg.name), device="cuda")
out = torch.empty_like(inp.q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
ws = ba.alloc_workspace(prob, "cuda")
st = torch.cuda.current_stream()
for _ in range(20):
    ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, scale=inp.scale, workspace=ws)
torch.cuda.synchronize()
res = {}
for flags, name in ((0, "pdl"), (ba.BA_FLAG_NO_PDL, "no_pdl")):
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, scale=inp.scale,
                                  workspace=ws, flags=flags)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    res[name] = {"host_us_per_call": (t1 - t0) / n * 1e6, "device_us_per_step": e0.elapsed_time(e1) / n * 1e3}
print(json.dumps({"config": cfg.name, **res}))
