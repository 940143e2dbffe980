"""Per-CTA start/end distribution of the fused kernel from %globaltimer stamps."""
import sys, os, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "mha7b_b32"
cfg = CONFIGS[name]
inp = make_inputs(cfg, 1, device="cuda")
out = torch.empty_like(inp.q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
ws = ba.alloc_workspace(prob, "cuda")
run = lambda: ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, workspace=ws, scale=inp.scale)
for _ in range(5): run()
torch.cuda.synchronize()
S = 1024
G = 148
tr = torch.zeros(G * S, dtype=torch.int64, device="cuda")
lib = ba.load_library()
lib.ba_set_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
lib.ba_set_trace_buffer(None)
t = tr.view(G, S)[:, :256].cpu()
tags = (t >> 56) & 0xff
ts = (t & ((1 << 56) - 1)).double()
t0 = ts[tags == 1].min().item()
rel = (ts - t0) / 1e3
starts, ends, segs = [], [], []
for k in range(G):
    row = [(int(tags[k, j]), float(rel[k, j])) for j in range(256) if tags[k, j] != 0]
    st = [v for tg, v in row if tg == 1]
    en = [v for tg, v in row if tg == 7]
    if st and en:
        starts.append(st[0]); ends.append(en[0])
        segs.append([(tg, round(v, 1)) for tg, v in row if tg in (2, 3, 4)])
import statistics
print(name, "event us %.1f" % (e0.elapsed_time(e1) * 1e3),
      "start max %.2f, end min %.2f med %.2f max %.2f" % (max(starts), min(ends), statistics.median(ends), max(ends)))
order = sorted(range(len(ends)), key=lambda k: ends[k])
for k in order[:3] + order[-5:]:
    print("cta", k, "end %.1f" % ends[k], segs[k])
