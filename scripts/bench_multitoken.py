"""Multi-token (speculative verification) step: µs per
step for n draft tokens per sample at a BASELINE shape, against n sequential
single-token steps (the I/O amortisation App. G, claims).
One JSON line per n.  Inputs: 2 rotating sets (> L2 each); CUDA events."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs

name = os.environ.get("MT_CFG", "mha7b_b32")
cfg = CONFIGS[name]
e = cfg.elem_bytes


def timeit(fn, iters=30, reps=5):
    for k in range(5):
        fn(k)
    torch.cuda.synchronize()
    res = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(iters):
            fn(k)
        b.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / iters * 1e3)
    return statistics.median(res)


base = [make_inputs(cfg, 1 + k, device="cuda") for k in range(2)]
out1 = [torch.empty_like(s.q) for s in base]
us1 = timeit(lambda k: ba.bifurcated_attn_decode(base[k % 2].q, base[k % 2].Kc, base[k % 2].Vc,
                                                 base[k % 2].Kd, base[k % 2].Vd, base[k % 2].lens,
                                                 out1[k % 2], scale=base[k % 2].scale))
for n in (1, 2, 4, 8):
    qs = [torch.randn(cfg.b, cfg.h, n, cfg.d, device="cuda").to(cfg.torch_dtype) for _ in range(2)]
    outs = [torch.empty_like(q) for q in qs]
    ws = ba.alloc_workspace(ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md,
                                            cfg.torch_dtype, base[0].scale, 0, n), "cuda")
    us = timeit(lambda k: ba.bifurcated_attn_decode(qs[k % 2], base[k % 2].Kc, base[k % 2].Vc,
                                                    base[k % 2].Kd, base[k % 2].Vd,
                                                    base[k % 2].lens, outs[k % 2], workspace=ws,
                                                    scale=base[k % 2].scale))
    alg = 2 * e * cfg.d * cfg.g * (cfg.mc + cfg.b * cfg.md) + 2 * e * cfg.b * cfg.h * n * cfg.d
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, 0, 0, n)
    print(json.dumps({"workload": name, "n_tok": n, "us_per_step": round(us, 2),
                      "us_per_token": round(us / n, 2), "GBs": round(alg / us / 1e3, 1),
                      "tokens_per_s": round(cfg.b * n / us * 1e6),
                      "speedup_vs_n_single_steps": round(n * us1 / us, 2),
                      "plan": ba.ba_plan_string(prob)}), flush=True)
