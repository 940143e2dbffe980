"""Per-role cycle accounting of the rows-on-M kernel (experiment; BIFATTN_PROF
build: EXP_LIB=exp_libs/prof.so).  Prints the mean over CTAs of the cycles
(and µs at 1.965 GHz) each role spends per section."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
ba.load_library(os.environ.get("EXP_LIB", "exp_libs/prof.so"))
from synth import CONFIGS, make_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "mqa"
cfg = CONFIGS[name]
inp = make_inputs(cfg, 1, device="cuda")
out = torch.empty_like(inp.q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
ws = ba.alloc_workspace(prob, "cuda")
run = lambda: ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out, workspace=ws, scale=inp.scale)
for _ in range(3):
    run()
torch.cuda.synchronize()
tr = torch.zeros(160 * 1024, dtype=torch.int64, device="cuda")
lib = ba.load_library()
lib.ba_set_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
lib.ba_set_trace_buffer(None)
t = tr.view(160, 1024)[:148].cpu().double()
used = t[:, :16].sum(1) > 0
t = t[used]
soft = ["q_load", "s_full_wait", "S_load", "max", "xchg_barrier", "rescale", "P_exp_store", "epilogue"]
mma = ["q_full_wait", "k_full_wait", "s_free_wait", "QK_issue", "v_full_wait", "p_full_wait", "PV_issue", "o_empty_wait"]
us = lambda c: round(c / 1965.0, 2)
print(json.dumps({"cfg": name, "event_us": round(e0.elapsed_time(e1) * 1e3, 1), "ctas": int(used.sum()),
                  "plan": ba.ba_plan_string(prob)[:80]}))
print("softmax thread:", json.dumps({n: us(t[:, k].mean().item()) for k, n in enumerate(soft)}))
print("MMA lane:      ", json.dumps({n: us(t[:, 8 + k].mean().item()) for k, n in enumerate(mma)}))
