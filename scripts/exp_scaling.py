"""Step time vs bytes (intercept = fixed per-step overhead)."""
import sys, os, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs, alg_bytes

base = CONFIGS["mha7b_b32"]
pts = []
for mc, md in [(128, 128), (1024, 128), (2048, 256), (4096, 256), (8192, 256), (16384, 256), (32768, 256)]:
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
    pts.append((alg_bytes(cfg), us))
    print(json.dumps({"mc": mc, "md": md, "MB": round(alg_bytes(cfg) / 1e6, 1), "us": round(us, 2), "GBs": round(alg_bytes(cfg) / us / 1e3, 1)}), flush=True)
# least squares us = a + bytes/bw
n = len(pts); sx = sum(p[0] for p in pts); sy = sum(p[1] for p in pts)
sxx = sum(p[0] ** 2 for p in pts); sxy = sum(p[0] * p[1] for p in pts)
slope = (n * sxy - sx * sy) / (n * sxx - sx * sx); icpt = (sy - slope * sx) / n
print("fit: overhead %.1f us, marginal BW %.0f GB/s" % (icpt, 1e-3 / slope))
