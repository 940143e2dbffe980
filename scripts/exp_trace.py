"""Per-CTA timeline of the fused kernel from %globaltimer stamps."""
import sys, os, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "mha7b_b32"
cfg = CONFIGS[name]
if len(sys.argv) > 2:
    cfg = cfg.with_(md=int(sys.argv[2]))
inp = make_inputs(cfg, 1, device="cuda")
out = torch.empty_like(inp.q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
ws = ba.alloc_workspace(prob, "cuda")
run = lambda: ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, workspace=ws, scale=inp.scale)
for _ in range(5): run()
torch.cuda.synchronize()
tr = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
lib = ba.load_library()
lib.ba_set_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
run(); torch.cuda.synchronize()
lib.ba_set_trace_buffer(None)
t = tr.view(148, 64).cpu()
tags = (t >> 56) & 0xff
ts = t & ((1 << 56) - 1)
t0 = ts[tags == 1].min().item()
res = []
for k in range(148):
    ev = [(int(tags[k, j]), (int(ts[k, j]) - t0) / 1e3) for j in range(64) if tags[k, j] != 0]
    res.append(ev)
json.dump({"cfg": name, "plan": ba.ba_plan_string(prob), "ctas": res}, open("gpurun_out/trace_%s.json" % name, "w"))
ends = [ev[-1][1] for ev in res if ev]
starts = [ev[0][1] for ev in res if ev]
print(name, "start spread %.2f us, end min %.2f max %.2f" % (max(starts), min(ends), max(ends)))
for k in (0, 1, 50, 100, 147):
    print(k, " ".join("%d@%.1f" % e for e in res[k]))
