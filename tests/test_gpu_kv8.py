"""GPU parity of the FP8 (E4M3) KV cache path (reading
R19) through the C ABI against the FP8 oracle (oracle_attn_decode_kv8_f64),
element by element with the bf16 tolerance of reading R12: the oracle reads
the SAME E4M3 codes and scales, so quantisation is input, not kernel error.
Covers the tensor-core KV8 kernel (N = 16 / 32, converter-fed f16 stages,
single-f16 P), the CUDA-core FP8 kernel (forced, d != 128, p that no N
covers), stress variants, lens = 0, the replicated baseline, append + attend,
CUDA-graph replay and the full BASELINE C2b shape (every row)."""
import pytest
import torch

import paper_2403_08845_b200 as ba
from synth import CONFIGS, Config, make_inputs, seed_for
from tests.parity import compare, oracle_kv8_all_rows

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _run(inp, flags=0, with_lse=True):
    q = inp.q.to(DEV)
    lse = torch.empty(q.shape[0], q.shape[1], dtype=torch.float32, device=DEV) if with_lse else None
    out = ba.bifurcated_attn_decode(q, inp.Kc.to(DEV), inp.Vc.to(DEV), inp.Kd.to(DEV),
                                    inp.Vd.to(DEV), inp.lens.to(DEV), lse=lse, scale=inp.scale,
                                    flags=flags, k_scale=inp.k_scale, v_scale=inp.v_scale)
    torch.cuda.synchronize()
    return out, lse


def _plan(cfg, flags=0):
    return ba.ba_plan_string(ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md,
                                             torch.bfloat16, flags=flags,
                                             kv_dtype=torch.float8_e4m3fn))


SHAPES = [
    Config("mha_n32", "bf16", b=32, h=4, g=4, d=128, mc=1000, md=37, kv="e4m3"),
    Config("mha_n16", "bf16", b=16, h=4, g=4, d=128, mc=777, md=50, kv="e4m3"),
    Config("gqa_n32", "bf16", b=9, h=16, g=4, d=128, mc=513, md=21, kv="e4m3"),
    Config("rows96", "bf16", b=96, h=4, g=2, d=128, mc=600, md=40, kv="e4m3"),
    Config("mqa_p48_fma", "bf16", b=3, h=48, g=1, d=128, mc=300, md=20, kv="e4m3"),
    Config("d64_fma", "bf16", b=6, h=4, g=2, d=64, mc=200, md=9, kv="e4m3"),
    Config("few_rows_fma", "bf16", b=5, h=2, g=2, d=128, mc=300, md=17, kv="e4m3"),
    Config("mc1", "bf16", b=16, h=2, g=2, d=128, mc=1, md=3, kv="e4m3"),
    Config("md0", "bf16", b=16, h=4, g=4, d=128, mc=333, md=0, kv="e4m3"),
]


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("variant", ["normal", "ragged", "dec_dom", "ctx_dom", "peaky"])
def test_kv8_all_rows(cfg, variant):
    if cfg.md == 0 and variant in ("ragged", "dec_dom"):
        pytest.skip("no decode cache")
    inp = make_inputs(cfg, 41, variant=variant)
    out, lse = _run(inp)
    ref, ref_lse = oracle_kv8_all_rows(inp)
    st = compare(out.reshape(-1, cfg.d), lse.reshape(-1), ref, ref_lse, torch.bfloat16,
                 f"{cfg.name}/{variant} [{_plan(cfg)}]")
    print(f"{cfg.name}/{variant}: {st}")


@pytest.mark.parametrize("cfg", SHAPES[:3], ids=lambda c: c.name)
def test_kv8_tensor_core_plan_taken(cfg):
    plan = _plan(cfg)
    assert plan.startswith("fused_tc") and "kv=e4m3" in plan, plan


@pytest.mark.parametrize("cfg", SHAPES[:3], ids=lambda c: c.name)
def test_kv8_forced_fma_matches(cfg):
    inp = make_inputs(cfg, 43, variant="ragged")
    out, lse = _run(inp, flags=ba.BA_FLAG_FORCE_FMA)
    ref, ref_lse = oracle_kv8_all_rows(inp)
    compare(out.reshape(-1, cfg.d), lse.reshape(-1), ref, ref_lse, torch.bfloat16, "fma")


@pytest.mark.parametrize("variant", ["planted_ctx", "planted_dec"])
def test_kv8_planted_keys(variant):
    cfg = SHAPES[0]
    inp = make_inputs(cfg, 44, variant=variant)
    out, lse = _run(inp)
    ref, ref_lse = oracle_kv8_all_rows(inp)
    compare(out.reshape(-1, cfg.d), lse.reshape(-1), ref, ref_lse, torch.bfloat16, variant)


def test_kv8_lens_zero_context_only():
    cfg = SHAPES[0]
    inp = make_inputs(cfg, 45, lens=[0] * cfg.b)
    out, lse = _run(inp)
    ref, ref_lse = oracle_kv8_all_rows(inp)
    compare(out.reshape(-1, cfg.d), lse.reshape(-1), ref, ref_lse, torch.bfloat16, "lens0")


def test_kv8_replicated_baseline():
    cfg = SHAPES[0]
    inp = make_inputs(cfg, 46, variant="ragged")
    q = inp.q.to(DEV)
    K = torch.cat([inp.Kc.unsqueeze(0).expand(cfg.b, -1, -1, -1), inp.Kd], 2).contiguous().to(DEV)
    V = torch.cat([inp.Vc.unsqueeze(0).expand(cfg.b, -1, -1, -1), inp.Vd], 2).contiguous().to(DEV)
    out = ba.replicated_attn_decode(q, K, V, inp.lens.to(DEV), cfg.mc, scale=inp.scale,
                                    k_scale=inp.k_scale, v_scale=inp.v_scale)
    torch.cuda.synchronize()
    ref, _ = oracle_kv8_all_rows(inp)
    compare(out.reshape(-1, cfg.d), None, ref, None, torch.bfloat16, "replicated-kv8")


def test_kv8_append_then_attend():
    """FP8 append + attend: k_new / v_new are codes; caches bit-exact after the
    append, the step equals the oracle on the appended cache."""
    cfg = Config("app", "bf16", b=32, h=4, g=4, d=128, mc=500, md=64, kv="e4m3")
    inp = make_inputs(cfg, 47, lens=[10 + i for i in range(cfg.b)])
    g = torch.Generator().manual_seed(3)
    kn = (torch.randn(cfg.b, cfg.g, 1, cfg.d, generator=g) * 2).to(torch.float8_e4m3fn)
    vn = (torch.randn(cfg.b, cfg.g, 1, cfg.d, generator=g) * 2).to(torch.float8_e4m3fn)
    Kd, Vd, lens = inp.Kd.to(DEV), inp.Vd.to(DEV), inp.lens.to(DEV)
    out = ba.bifurcated_attn_decode_append(inp.q.to(DEV), kn.to(DEV), vn.to(DEV), inp.Kc.to(DEV),
                                           inp.Vc.to(DEV), Kd, Vd, lens, scale=inp.scale,
                                           k_scale=inp.k_scale, v_scale=inp.v_scale)
    torch.cuda.synchronize()
    Kd_ref, Vd_ref = inp.Kd.clone(), inp.Vd.clone()
    for i in range(cfg.b):
        L = int(inp.lens[i])
        Kd_ref[i, :, L] = kn[i, :, 0]
        Vd_ref[i, :, L] = vn[i, :, 0]
    assert torch.equal(Kd.cpu().view(torch.uint8), Kd_ref.view(torch.uint8))
    assert torch.equal(Vd.cpu().view(torch.uint8), Vd_ref.view(torch.uint8))
    assert torch.equal(lens.cpu(), inp.lens + 1)
    inp2 = type(inp)(inp.q, inp.Kc, inp.Vc, Kd_ref, Vd_ref, inp.lens + 1, inp.scale,
                     inp.k_scale, inp.v_scale)
    ref, _ = oracle_kv8_all_rows(inp2)
    compare(out.reshape(-1, cfg.d), None, ref, None, torch.bfloat16, "append-kv8")


def test_kv8_cuda_graph_replay():
    cfg = SHAPES[0]
    inp = make_inputs(cfg, 48, device=DEV)
    out = torch.empty_like(inp.q)
    ws = ba.alloc_workspace(ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md,
                                            torch.bfloat16, inp.scale,
                                            kv_dtype=torch.float8_e4m3fn,
                                            k_scale=inp.k_scale, v_scale=inp.v_scale), DEV)
    call = lambda: ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd,  # noqa: E731
                                             inp.lens, out, scale=inp.scale, workspace=ws,
                                             k_scale=inp.k_scale, v_scale=inp.v_scale)
    call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    ref, _ = oracle_kv8_all_rows(inp)
    compare(out.reshape(-1, cfg.d), None, ref, None, torch.bfloat16, "graph-kv8")


def test_kv8_full_size_c2b_all_rows():
    """BASELINE C2b with an FP8 cache, bench.py's launch configuration: every row."""
    cfg = CONFIGS["mha7b_b32_fp8"]
    inp = make_inputs(cfg, seed_for(cfg.name), device=DEV)
    out, lse = _run(inp)
    ref, ref_lse = oracle_kv8_all_rows(inp)
    st = compare(out.reshape(-1, cfg.d), lse.reshape(-1), ref, ref_lse, torch.bfloat16,
                 "mha7b_b32_fp8")
    print(f"mha7b_b32_fp8: all {cfg.b * cfg.h} rows: {st} plan [{_plan(cfg)}]")


def test_kv8_rejects_fp32_query():
    cfg = Config("x", "fp32", b=2, h=2, g=2, d=128, mc=64, md=4)
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, torch.float32,
                           kv_dtype=torch.float8_e4m3fn)
    assert ba.ba_workspace_bytes(prob) == 0
