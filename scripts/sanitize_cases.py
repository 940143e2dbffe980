"""Small problems through every launch plan, for compute-sanitizer
(memcheck / racecheck / synccheck).  Each case runs once and is checked
against the oracle (a sanitizer run must still produce the right answer).
usage: compute-sanitizer --tool memcheck python scripts/sanitize_cases.py [case ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_08845_b200 as ba  # noqa: E402
from synth import Config, make_inputs  # noqa: E402
from tests.parity import compare, oracle_kv8_all_rows, oracle_rows  # noqa: E402

DEV = "cuda:0"
CASES = {
    "fused_tc": (Config("s1", "bf16", b=24, h=8, g=4, d=128, mc=700, md=45), 0, 1),
    "fused_dyn": (Config("s9", "bf16", b=16, h=4, g=4, d=128, mc=700, md=300), 0, 1),
    "rows_merge": (Config("s2", "bf16", b=66, h=8, g=4, d=128, mc=600, md=40), 0, 1),
    "rows_dec_tc": (Config("s3", "bf16", b=64, h=8, g=8, d=128, mc=130, md=1152), 0, 1),
    "fma_fp32": (Config("s4", "fp32", b=4, h=2, g=2, d=16, mc=32, md=4), 0, 1),
    "fma_bf16": (Config("s5", "bf16", b=5, h=4, g=4, d=64, mc=200, md=9), 0, 1),
    "multitoken": (Config("s6", "bf16", b=8, h=4, g=4, d=128, mc=300, md=20), 0, 4),
    "kv8_tc": (Config("s7", "bf16", b=32, h=4, g=4, d=128, mc=500, md=37, kv="e4m3"), 0, 1),
    "kv8_fma": (Config("s8", "bf16", b=5, h=2, g=2, d=128, mc=300, md=17, kv="e4m3"), 0, 1),
}


def run(name):
    cfg, flags, n = CASES[name]
    inp = make_inputs(cfg, 7, variant="ragged", n_tok=n)
    q = inp.q.to(DEV)
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=DEV)
    out = ba.bifurcated_attn_decode(q, inp.Kc.to(DEV), inp.Vc.to(DEV), inp.Kd.to(DEV),
                                    inp.Vd.to(DEV), inp.lens.to(DEV), lse=lse, scale=inp.scale,
                                    flags=flags, k_scale=inp.k_scale, v_scale=inp.v_scale)
    torch.cuda.synchronize()
    ref, ref_lse = oracle_kv8_all_rows(inp) if cfg.kv else oracle_rows(inp)
    st = compare(out.reshape(ref.shape), lse.reshape(-1), ref, ref_lse, cfg.torch_dtype, name)
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype,
                           n_tok=n, kv_dtype=inp.Kc.dtype)
    print(f"{name}: [{ba.ba_plan_string(prob)}] {st}", flush=True)


def run_append():
    cfg = Config("sa", "bf16", b=32, h=4, g=4, d=128, mc=300, md=64)
    inp = make_inputs(cfg, 8, lens=[5 + i for i in range(cfg.b)])
    kn = torch.randn(cfg.b, cfg.g, 1, cfg.d).to(torch.bfloat16)
    vn = torch.randn(cfg.b, cfg.g, 1, cfg.d).to(torch.bfloat16)
    Kd, Vd, lens = inp.Kd.to(DEV), inp.Vd.to(DEV), inp.lens.to(DEV)
    ba.bifurcated_attn_decode_append(inp.q.to(DEV), kn.to(DEV), vn.to(DEV), inp.Kc.to(DEV),
                                     inp.Vc.to(DEV), Kd, Vd, lens, scale=inp.scale)
    torch.cuda.synchronize()
    print("append: ok", flush=True)


def run_lse_merge():
    parts = torch.randn(3, 10, 128, device=DEV).to(torch.bfloat16)
    lses = torch.randn(3, 10, device=DEV)
    ba.lse_merge(parts, lses)
    torch.cuda.synchronize()
    print("lse_merge: ok", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + ["append", "lse_merge"]
    for nm in names:
        if nm == "append":
            run_append()
        elif nm == "lse_merge":
            run_lse_merge()
        else:
            run(nm)
