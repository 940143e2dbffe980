"""Step time of the fused kernel over (mc, md) at b=32 MHA 7B: which branch costs what."""
import sys, os, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
if os.environ.get("EXP_LIB"):
    ba.load_library(os.environ["EXP_LIB"])
from synth import CONFIGS, make_inputs, alg_bytes

base = CONFIGS[os.environ.get("EXP_CFG", "mha7b_b32")]
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(128, 256), (128, 512), (128, 1024), (128, 2048), (8192, 0), (16384, 0)]
for mc, md in shapes:
    if (mc, md) == (0, 0):  # the config's own shape
        mc, md = base.mc, base.md
    cfg = base.with_(mc=mc, md=md)
    sets = [make_inputs(cfg, 1 + k, device="cuda") for k in range(2)]
    outs = [torch.empty_like(s.q) for s in sets]
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, sets[0].scale)
    ws = ba.alloc_workspace(prob, "cuda")
    def step(k):
        s = sets[k % 2]
        ba.bifurcated_attn_decode(s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, outs[k % 2], workspace=ws, scale=s.scale)
    for k in range(5): step(k)
    torch.cuda.synchronize()
    res = []
    for r in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(30): step(k)
        b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 30 * 1e3)
    us = statistics.median(res)
    print(json.dumps({"mc": mc, "md": md, "MB": round(alg_bytes(cfg) / 1e6, 1), "us": round(us, 2),
                      "GBs": round(alg_bytes(cfg) / us / 1e3, 1), "plan": ba.ba_plan_string(prob)}), flush=True)
