"""Host cost per call: Python wrapper vs bare ctypes call vs checks alone."""
import sys, os, time, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
if os.environ.get("EXP_LIB"):
    ba.load_library(os.environ["EXP_LIB"])
from synth import CONFIGS, make_inputs
cfg = CONFIGS["mha7b_b32"].with_(mc=1280, md=0)
s = make_inputs(cfg, 1, device="cuda")
out = torch.empty_like(s.q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, s.scale)
ws = ba.alloc_workspace(prob, "cuda")
lib = ba.load_library()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = [ctypes.byref(prob)] + [ctypes.c_void_p(t.data_ptr()) for t in (s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, out)] + [None, ctypes.c_void_p(ws.data_ptr()), ws.numel(), st]
def timeit(fn, n=300):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return round((t1 - t0) / n * 1e6, 2)
r = {
 "wrapper": timeit(lambda: ba.bifurcated_attn_decode(s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, out, workspace=ws, scale=s.scale)),
 "bare_ctypes": timeit(lambda: lib.bifurcated_attn_decode(*args)),
 "checks_only": timeit(lambda: ba._check(dict(q=s.q, Kc=s.Kc, Vc=s.Vc, Kd=s.Kd, Vd=s.Vd, lens=s.lens), s.q.dtype, s.q.device)),
 "plan_string": timeit(lambda: lib.ba_plan_string(ctypes.byref(prob))),
}
print(json.dumps(r))
