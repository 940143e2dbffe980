"""Per-role cycle accounting of the rows-on-M kernel (ctx_rows.cuh) from a
-DBIFATTN_PROF variant build (clock64 accumulators dumped into the trace
buffer): where a CTA's time goes in the softmax/epilogue thread 128 and in
the MMA issuer lane.

usage: python scripts/role_cycles_rows.py [config ...]   (default: mqa gqa)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_08845_b200 import _build  # noqa: E402

LIB = _build.build_variant("prof", ["-DBIFATTN_PROF"])
import paper_2403_08845_b200 as ba  # noqa: E402

ba.load_library(LIB)
from synth import CONFIGS, make_inputs, seed_for  # noqa: E402

SM = ["q_load", "s_full_wait", "S_tmem_ld", "max", "xchg_barrier", "rescale", "P_exp_store",
      "epilogue"]
MMA = ["q_full_wait", "k_full_wait", "s_free_wait", "QK_issue", "v_cvt_wait", "p_full_wait",
       "PV_issue", "o_empty_wait"]


def run(name):
    base = 0
    if name.startswith("v2:"):
        # the two-block kernel (ctx_rows2.cuh) dumps at slots 512 / 520; shape
        # "v2:b,h,g,mc,md" (a context-only rows launch)
        from synth import Config
        b, h, g, mc, md = map(int, name[3:].split(","))
        cfg = Config(name, "bf16", b=b, h=h, g=g, d=128, mc=mc, md=md)
        base = 512
    else:
        cfg = CONFIGS[name]
    inp = make_inputs(cfg, seed_for(name) if name in CONFIGS else 5, device="cuda")
    out = torch.empty_like(inp.q)
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
    ws = ba.alloc_workspace(prob, "cuda")
    buf = torch.zeros(160 * 1024, dtype=torch.int64, device="cuda")

    def step():
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out,
                                  scale=inp.scale, workspace=ws)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    lib = ba.load_library()
    lib.ba_set_trace_buffer(buf.data_ptr())
    step()
    torch.cuda.synchronize()
    lib.ba_set_trace_buffer(None)
    tr = buf.view(160, 1024).cpu()
    rows = [r for r in tr.tolist() if any(r[base:base + 16])]
    n = len(rows)
    sm = {k: sum(r[base + i] for r in rows) / n / 1e3 for i, k in enumerate(SM)}
    mma = {k: sum(r[base + 8 + i] for r in rows) / n / 1e3 for i, k in enumerate(MMA)}
    print(json.dumps({"config": name, "plan": ba.ba_plan_string(prob), "ctas": n,
                      "softmax_thread_kcycles": {k: round(v, 1) for k, v in sm.items()},
                      "mma_lane_kcycles": {k: round(v, 1) for k, v in mma.items()}}), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["mqa", "gqa"]:
        run(nm)
