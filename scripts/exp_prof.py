"""Per-role cycle accounting of the fused kernel (experiment; needs a
BIFATTN_PROF build, EXP_LIB=exp_libs/prof.so).  Prints, per role, the mean /
max over CTAs of the time spent in each section (µs at the SM clock estimated
from the event-timed launch)."""
import sys, os, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
ba.load_library(os.environ.get("EXP_LIB", "exp_libs/prof.so"))
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
for _ in range(5):
    run()
torch.cuda.synchronize()
S = 1024
tr = torch.zeros(148 * S, dtype=torch.int64, device="cuda")
lib = ba.load_library()
lib.ba_set_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3
lib.ba_set_trace_buffer(None)
t = tr.view(148, S).cpu().double()
cyc = t[:, 51] - t[:, 48]
ghz = cyc.max().item() / us / 1e3
print(json.dumps({"cfg": name, "event_us": round(us, 2), "ghz_est": round(ghz, 3),
                  "plan": ba.ba_plan_string(prob)}))
sm = ["wait_S", "tmem_ld", "bar", "slow", "wait_Pempty", "P_store", "seg/other"]
roles = {"softmax_wg0": (0, sm), "softmax_wg1": (8, sm),
         "producer": (16, ["q_wait", "q_issue+seg", "kv_empty_wait", "tma_issue"]),
         "qk": (24, ["q_full_wait", "kv_full_wait", "s_free_wait", "issue"]),
         "pv": (32, ["o_empty_wait", "p_full_wait", "issue"])}
f = lambda x: round(x / ghz / 1e3, 2)
cs = ba.ba_plan_ctas(prob)
Tc = None
Tc_tiles = int(ba.ba_plan_string(prob).split("ctx_tiles=")[1].split(",")[0])
ctx = [k for k in range(148) if cs[k + 1] <= Tc_tiles]
dec = [k for k in range(148) if cs[k] >= Tc_tiles]
for cname, sel in (("ctx-only CTAs", ctx), ("dec-only CTAs", dec)):
    if not sel:
        continue
    tt = t[sel]
    print("==", cname, len(sel), "main_end mean", f((tt[:, 49] - tt[:, 48]).mean().item()))
    for r, (base, names) in roles.items():
        row = {n: f(tt[:, base + k].mean().item()) for k, n in enumerate(names)}
        print(r, json.dumps(row))
    print("need-tiles per CTA (thread 128 / 256):", tt[:, 7].mean().item(), tt[:, 15].mean().item(),
          "tiles per CTA:", sum(cs[k + 1] - cs[k] for k in sel) / len(sel))
ph = {"start->main_end": t[:, 49] - t[:, 48], "main_end->barrier_out": t[:, 50] - t[:, 49],
      "merge": t[:, 51] - t[:, 50]}
for k, v in ph.items():
    print(k, "mean", f(v.mean().item()), "min", f(v.min().item()), "max", f(v.max().item()))
me = t[:, 49] - t[:, 48]
order = me.argsort()
print("main_end fastest:", [(int(i), f(me[i].item()), cs[i + 1] - cs[i]) for i in order[:6]])
print("main_end slowest:", [(int(i), f(me[i].item()), cs[i + 1] - cs[i]) for i in order[-6:]])
print("per-CTA main_end (us):", [f(x) for x in me.tolist()])
