"""Interleaved timing of a custom shape on the product library and a variant
build: python scripts/ab_custom.py b h g mc md ROUNDS NAME -DFLAG..."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_08845_b200 import _build  # noqa: E402

b, h, g, mc, md, rounds, name = sys.argv[1:8]
defines = sys.argv[8:]
libs = {"product": _build.build(), name: _build.build_variant(name, defines)}
RUN = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2403_08845_b200 as ba
ba.load_library(%r)
from synth import Config, make_inputs
cfg = Config("c", "bf16", b=%s, h=%s, g=%s, d=128, mc=%s, md=%s)
sets = [make_inputs(cfg, 5 + k, device="cuda") for k in range(3)]
out = torch.empty_like(sets[0].q)
prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype)
ws = ba.alloc_workspace(prob, "cuda")
def step(k):
    i = sets[k %% 3]
    ba.bifurcated_attn_decode(i.q, i.Kc, i.Vc, i.Kd, i.Vd, i.lens, out, scale=i.scale, workspace=ws)
for k in range(10): step(k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(30): step(k)
e1.record(); torch.cuda.synchronize()
print(e0.elapsed_time(e1) / 30 * 1e3, ba.ba_plan_string(prob))
"""
res = {k: [] for k in libs}
plans = {}
for _ in range(int(rounds)):
    for k, lib in libs.items():
        o = subprocess.run([sys.executable, "-c", RUN % (ROOT, lib, b, h, g, mc, md)], capture_output=True,
                           text=True, timeout=300, cwd=ROOT)
        line = o.stdout.strip().splitlines()[-1]
        us, plan = line.split(" ", 1)
        res[k].append(float(us))
        plans[k] = plan
print(json.dumps({"shape": [b, h, g, mc, md], **{k: {"us_median": statistics.median(v), "plan": plans[k]}
                                                 for k, v in res.items()}}))
