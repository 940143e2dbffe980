"""Per-tile timeline of one or more CTAs (producer / MMA / softmax stamps)."""
import sys, os, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
if os.environ.get("EXP_LIB"):
    ba.load_library(os.environ["EXP_LIB"])
from synth import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "mha7b_b32"
cfg = CONFIGS[name]
if os.environ.get("EXP_MC"):
    cfg = cfg.with_(mc=int(os.environ["EXP_MC"]), md=int(os.environ["EXP_MD"]))
inp = make_inputs(cfg, 1, device="cuda")
out = torch.empty_like(inp.q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
ws = ba.alloc_workspace(prob, "cuda")
run = lambda: ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, workspace=ws, scale=inp.scale)
for _ in range(5): run()
torch.cuda.synchronize()
S = 1024
tr = torch.zeros(148 * S, dtype=torch.int64, device="cuda")
lib = ba.load_library()
lib.ba_set_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
run(); torch.cuda.synchronize()
lib.ba_set_trace_buffer(None)
t = tr.view(148, S).cpu()
tags = (t >> 56) & 0xff
ts = (t & ((1 << 56) - 1)).double()
t0 = ts[tags == 1].min().item()
rel = (ts - t0) / 1e3
for k in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "100"])]:
    print("=== CTA", k)
    sm = [(int(tags[k, j]), round(float(rel[k, j]), 2)) for j in range(256) if tags[k, j] != 0]
    prod = [round(float(rel[k, 256 + j]), 2) for j in range(128) if tags[k, 256 + j] != 0]
    kvf = [round(float(rel[k, 384 + j]), 2) for j in range(128) if tags[k, 384 + j] != 0]
    qk = [round(float(rel[k, 512 + j]), 2) for j in range(256) if tags[k, 512 + j] != 0]
    pv = [round(float(rel[k, 768 + j]), 2) for j in range(256) if tags[k, 768 + j] != 0]
    print("softmax:", " ".join("%d@%.2f" % e for e in sm))
    print("tma_issue:", prod)
    print("kv_landed(seen by MMA):", kvf)
    print("qk_issue:", qk)
    print("pv_issue:", pv)
