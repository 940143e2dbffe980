"""Kernel phase timeline from entry / prologue / stream end / barrier / merge stamps."""
import sys, os, ctypes, statistics
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
G = len(ba.ba_plan_ctas(prob)) - 1
S = 1024
tr = torch.zeros(G * S, dtype=torch.int64, device="cuda")
lib = ba.load_library()
lib.ba_set_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    tr.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
lib.ba_set_trace_buffer(None)
t = tr.view(G, S).cpu()
ts = (t & ((1 << 56) - 1)).double() / 1e3
def col(i): return [float(x) for x in ts[:, i]]
entry, pro, sdone, bar, merge = col(250), col(254), col(251), col(252), col(253)
t0 = min(entry)
f = lambda v: "min %.1f max %.1f" % (min(v) - t0, max(v) - t0)
print(name, "event %.1f us" % (e0.elapsed_time(e1) * 1e3))
print(" entry", f(entry), "| prologue done", f(pro), "| stream+softmax+epilogue done", f(sdone), "| barrier passed", f(bar), "| merge done", f(merge))
