"""Per-allocation timing: does the step time depend on where the inputs live?"""
import sys, os, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
if os.environ.get("EXP_LIB"):
    ba.load_library(os.environ["EXP_LIB"])
from synth import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "mha7b_b32"
nsets = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = CONFIGS[name]
sets = [make_inputs(cfg, 1 + k, device="cuda") for k in range(nsets)]
out = torch.empty_like(sets[0].q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, sets[0].scale)
ws = ba.alloc_workspace(prob, "cuda")
def run(s):
    ba.bifurcated_attn_decode(s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, out, workspace=ws, scale=s.scale)
res = []
for k, s in enumerate(sets):
    for _ in range(3): run(s)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(5):
        a.record()
        for _ in range(20): run(s)
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 20 * 1e3)
    res.append(round(statistics.median(ts), 2))
print(json.dumps({"cfg": name, "per_set_us": res, "Kc_ptrs": [hex(s.Kc.data_ptr()) for s in sets]}))
