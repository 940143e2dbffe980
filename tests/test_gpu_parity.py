"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle,
element by element, on seeded inputs.  Small problems span several tiles and a
ragged tail and are checked on every row; BASELINE.json's full-size configs run
in the launch configuration bench.py times and are checked on every row (C2a,
C2b, C3, C4) or on >= 512 rows covering every CTA range of the plan (C5)."""
import numpy as np
import pytest
import torch

import paper_2403_08845_b200 as ba
from synth import CONFIGS, Config, make_inputs, seed_for
from tests.parity import (compare, oracle_all_rows, oracle_rows, oracle_rows_parallel,
                          sample_rows)

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def run_gpu(inp, flags=0, with_lse=True):
    q = inp.q.to(DEV)
    lse = torch.empty(q.shape[0], q.shape[1], dtype=torch.float32, device=DEV) if with_lse else None
    out = ba.bifurcated_attn_decode(q, inp.Kc.to(DEV), inp.Vc.to(DEV), inp.Kd.to(DEV),
                                    inp.Vd.to(DEV), inp.lens.to(DEV), lse=lse, scale=inp.scale,
                                    flags=flags)
    torch.cuda.synchronize()
    return out, lse


SMALL = [
    CONFIGS["tiny"],
    Config("mha_small", "bf16", b=5, h=8, g=8, d=128, mc=1000, md=37),
    Config("mha_rows16", "bf16", b=16, h=4, g=4, d=128, mc=777, md=50),
    Config("mha_rows40", "bf16", b=40, h=2, g=2, d=128, mc=1290, md=33),
    Config("gqa_small", "bf16", b=9, h=16, g=4, d=128, mc=513, md=21),
    Config("mqa_small", "bf16", b=3, h=48, g=1, d=128, mc=300, md=20),
    Config("d64", "bf16", b=6, h=4, g=2, d=64, mc=200, md=9),
    Config("d256", "bf16", b=3, h=2, g=1, d=256, mc=130, md=5),
    Config("d32_fp32", "fp32", b=3, h=6, g=3, d=32, mc=97, md=13),
    Config("fp32_d128", "fp32", b=4, h=4, g=2, d=128, mc=300, md=17),
    Config("mc1", "bf16", b=2, h=2, g=1, d=128, mc=1, md=3),
    Config("md0", "bf16", b=4, h=4, g=4, d=128, mc=333, md=0),
    # R = b*p >= 64: context branch on the rows-on-M kernel (ctx_rows.cuh)
    Config("rows130", "bf16", b=130, h=2, g=2, d=128, mc=1000, md=20),
    Config("gqa_rows300", "bf16", b=75, h=8, g=2, d=128, mc=700, md=30),
    Config("rows128_md0", "bf16", b=64, h=4, g=2, d=128, mc=129, md=0),
    # p >= 32: decode items in the rows kernel too, then the light merge
    Config("p32_rowsdec", "bf16", b=5, h=64, g=2, d=128, mc=300, md=140),
]


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: c.name)
@pytest.mark.parametrize("flags", [0, ba.BA_FLAG_FORCE_FMA, ba.BA_FLAG_CTX_ROWS,
                                   ba.BA_FLAG_NO_CTX_ROWS], ids=["auto", "fma", "rows", "fused"])
def test_small_all_rows(cfg, flags):
    inp = make_inputs(cfg, seed_for(cfg.name), variant="ragged" if cfg.md > 0 else "normal")
    out, lse = run_gpu(inp, flags)
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, cfg.name)


@pytest.mark.parametrize("variant", ["normal", "peaky", "ctx_dom", "dec_dom", "planted_ctx",
                                     "planted_dec", "equal", "ragged"])
@pytest.mark.parametrize("cfg", [SMALL[2], SMALL[4], SMALL[5], SMALL[13]], ids=lambda c: c.name)
@pytest.mark.parametrize("flags", [0, ba.BA_FLAG_CTX_ROWS, ba.BA_FLAG_NO_CTX_ROWS],
                         ids=["auto", "rows", "fused"])
def test_stress_variants(cfg, variant, flags):
    inp = make_inputs(cfg, 7, variant=variant)
    out, lse = run_gpu(inp, flags)
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, f"{cfg.name}/{variant}")
    if variant == "equal":
        o = out.float()
        assert torch.equal(o, o[:1].expand_as(o))


@pytest.mark.parametrize("cfg", [Config("x", "bf16", b=17, h=4, g=2, d=128, mc=640, md=32),
                                 Config("p48", "bf16", b=4, h=48, g=1, d=128, mc=300, md=32)],
                         ids=["p2", "p48"])
def test_all_lens_zero_is_context_only(cfg):
    inp = make_inputs(cfg, 8, lens=[0] * cfg.b)
    out, lse = run_gpu(inp)
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, "lens0")


def test_lens_clamped_to_cap():
    cfg = Config("x", "bf16", b=4, h=2, g=2, d=128, mc=64, md=8)
    inp = make_inputs(cfg, 9)
    inp_big = make_inputs(cfg, 9, lens=[100, -5, 8, 3])
    out, _ = run_gpu(inp_big)
    ref_inp = make_inputs(cfg, 9, lens=[8, 0, 8, 3])
    ref, ref_lse = oracle_rows(ref_inp)
    compare(out, None, ref, None, cfg.torch_dtype, "clamp")
    del inp


def test_replicated_baseline_matches_oracle():
    cfg = Config("x", "bf16", b=6, h=8, g=4, d=128, mc=300, md=40)
    inp = make_inputs(cfg, 10, variant="ragged")
    K = torch.cat([inp.Kc.unsqueeze(0).expand(cfg.b, -1, -1, -1), inp.Kd], dim=2).contiguous()
    V = torch.cat([inp.Vc.unsqueeze(0).expand(cfg.b, -1, -1, -1), inp.Vd], dim=2).contiguous()
    lse = torch.empty(cfg.b, cfg.h, device=DEV)
    out = ba.replicated_attn_decode(inp.q.to(DEV), K.to(DEV), V.to(DEV), inp.lens.to(DEV),
                                    cfg.mc, lse=lse, scale=inp.scale)
    torch.cuda.synchronize()
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, "replicated")


def test_host_entry_point_equals_device_call():
    cfg = Config("x", "bf16", b=8, h=4, g=4, d=128, mc=500, md=30)
    inp = make_inputs(cfg, 11)
    out_dev, _ = run_gpu(inp, with_lse=False)
    pin = lambda t: t.contiguous().pin_memory()
    hq, hKc, hVc, hKd, hVd, hl = map(pin, (inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens))
    hout = torch.empty_like(hq).pin_memory()
    dev = ba.make_device_buffers(hq, hKc, hKd, DEV)
    ba.bifurcated_attn_decode_host(hq, hKc, hVc, hKd, hVd, hl, hout, dev, scale=inp.scale)
    torch.cuda.synchronize()
    assert torch.equal(hout, out_dev.cpu())


@pytest.mark.parametrize("cfg", [Config("x", "bf16", b=16, h=8, g=8, d=128, mc=1024, md=64),
                                 Config("rows", "bf16", b=64, h=8, g=4, d=128, mc=1024, md=64),
                                 Config("rows_c5", "bf16", b=70, h=4, g=4, d=128, mc=1000, md=2000),
                                 Config("rows_p48", "bf16", b=6, h=48, g=1, d=128, mc=700, md=64)],
                         ids=["fused", "rows+dec", "rows+fused_dec", "rows_p48"])
def test_cuda_graph_capture_and_replay(cfg):
    inp = make_inputs(cfg, 12)
    q, Kc, Vc, Kd, Vd, lens = (t.to(DEV) for t in (inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens))
    out = torch.empty_like(q)
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, q.dtype, inp.scale)
    ws = ba.alloc_workspace(prob, DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ba.bifurcated_attn_decode(q, Kc, Vc, Kd, Vd, lens, out, workspace=ws, scale=inp.scale)
    torch.cuda.synchronize()
    ref_gpu = out.clone()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        ba.bifurcated_attn_decode(q, Kc, Vc, Kd, Vd, lens, out, workspace=ws, scale=inp.scale)
    out.zero_()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref_gpu)
    # lens change without recapture
    lens.copy_(torch.tensor([5] * cfg.b, dtype=torch.int32))
    graph.replay()
    torch.cuda.synchronize()
    inp.lens = lens.cpu()
    ref, _ = oracle_rows(inp)
    compare(out, None, ref, None, cfg.torch_dtype, "graph-lens")


@pytest.mark.parametrize("cfg", [Config("x", "bf16", b=32, h=4, g=4, d=128, mc=2048, md=64),
                                 Config("rows", "bf16", b=96, h=4, g=2, d=128, mc=2048, md=64)],
                         ids=["fused", "rows"])
def test_repeated_calls_deterministic(cfg):
    inp = make_inputs(cfg, 13)
    a, _ = run_gpu(inp)
    b_, _ = run_gpu(inp)
    assert torch.equal(a, b_)


def test_misaligned_pointer_rejected():
    cfg = Config("x", "bf16", b=2, h=2, g=2, d=128, mc=64, md=4)
    inp = make_inputs(cfg, 14, device=DEV)
    buf = torch.empty(inp.q.numel() + 8, dtype=torch.bfloat16, device=DEV)
    qmis = buf[1:1 + inp.q.numel()].view_as(inp.q)
    with pytest.raises(ba.BifAttnError) as e:
        ba.bifurcated_attn_decode(qmis, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens)
    assert e.value.code == -3


def test_small_workspace_rejected():
    cfg = Config("x", "bf16", b=2, h=2, g=2, d=128, mc=64, md=4)
    inp = make_inputs(cfg, 15, device=DEV)
    ws = torch.zeros(64, dtype=torch.uint8, device=DEV)
    # the binding refuses it before the call ...
    with pytest.raises(ValueError):
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, workspace=ws)
    # ... and the C ABI itself returns BA_EWORKSPACE
    import ctypes
    lib = ba.load_library()
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype)
    out = torch.empty_like(inp.q)
    rc = lib.bifurcated_attn_decode(ctypes.byref(prob), inp.q.data_ptr(), inp.Kc.data_ptr(),
                                    inp.Vc.data_ptr(), inp.Kd.data_ptr(), inp.Vd.data_ptr(),
                                    inp.lens.data_ptr(), out.data_ptr(), None, ws.data_ptr(),
                                    ws.numel(), torch.cuda.current_stream().cuda_stream)
    assert rc == -4


# ---------------------------------------------------------------------------
# BASELINE.json configs at full size, in bench.py's launch configuration
# (default flags = the plan bench.py times): EVERY output element and lse of
# C2a, C2b, C3 and C4 against the oracle (all host cores); C5 on >= 512 rows
# that cover every CTA range of the decode launch and every (group, 128-row
# block) item of the context launch, plus random rows
# ---------------------------------------------------------------------------
FULL_ALL = ["mha7b_b16", "mha7b_b32", "gqa", "mqa"]


def _full_run(cfg, name):
    inp = make_inputs(cfg, seed_for(name), device=DEV)
    lse = torch.empty(cfg.b, cfg.h, dtype=torch.float32, device=DEV)
    out = ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, lse=lse,
                                    scale=inp.scale)
    torch.cuda.synchronize()
    return inp, out, lse


@pytest.mark.parametrize("name", FULL_ALL)
def test_full_size_all_rows(name):
    cfg = CONFIGS[name]
    inp, out, lse = _full_run(cfg, name)
    ref, ref_lse = oracle_all_rows(inp)
    st = compare(out.reshape(-1, cfg.d), lse.reshape(-1), ref, ref_lse, cfg.torch_dtype, name)
    print(f"{name}: all {cfg.b * cfg.h} rows: {st}")


def _long_rows(cfg):
    """Rows of C5 covering the plan: the first and last decode tile of every
    CTA range of the decode launch (flat tile f -> (sample, group) = divmod(f //
    ntile_d, g), p = 1), one row per (group, 128-row block) context item, the
    corner rows and random rows, >= 512 in all."""
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype)
    cs = ba.ba_plan_ctas(prob)
    assert cs, "C5 takes the tensor-core plan"
    ntd = (cfg.md + 127) // 128
    p = cfg.p
    rows = set()
    for k in range(len(cs) - 1):
        if cs[k + 1] <= cs[k]:
            continue  # empty static range (decode columns taken dynamically)
        for f in (cs[k], cs[k + 1] - 1):
            ic = f // ntd
            i, c = divmod(ic, cfg.g)
            if i < cfg.b:
                rows.add(i * cfg.h + c * p)
    # dynamic decode columns (any CTA may take any (sample, group)): the first
    # and last group of every sample
    for i in range(cfg.b):
        rows.add(i * cfg.h)
        rows.add(i * cfg.h + (cfg.g - 1) * p)
    R = cfg.b * p
    for c in range(cfg.g):
        for rb in range((R + 127) // 128):
            r = min(R - 1, rb * 128 + (37 * c) % 128)
            i, jj = divmod(r, p)
            rows.add(i * cfg.h + c * p + jj)
    rows.update(sample_rows(cfg.b, cfg.h, n=64, seed=5))
    rng = np.random.default_rng(11)
    while len(rows) < 512:
        rows.add(int(rng.integers(0, cfg.b * cfg.h)))
    return sorted(rows)


def test_full_size_long_plan_rows():
    cfg = CONFIGS["long"]
    inp, out, lse = _full_run(cfg, "long")
    rows = _long_rows(cfg)
    assert len(rows) >= 512
    ref, ref_lse = oracle_rows_parallel(inp, rows)
    o = out.reshape(-1, cfg.d)[rows]
    st = compare(o, lse.reshape(-1)[rows], ref, ref_lse, cfg.torch_dtype, "long")
    print(f"long: {len(rows)} plan-covering rows: {st}")


# ---------------------------------------------------------------------------
# Seeded random shapes across every plan (fused / rows + decode items / rows +
# fused decode): odd p, ragged tails, small caps, lens from 0 to the cap
# ---------------------------------------------------------------------------
def _random_shapes(n=14, seed=2024):
    rng = np.random.default_rng(seed)
    shapes = []
    for k in range(n):
        p = int(rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 48]))
        g = int(rng.choice([1, 2, 3])) if p >= 12 else int(rng.choice([1, 2, 4, 5]))
        b = int(rng.integers(1, 150 // p + 3))
        mc = int(rng.integers(1, 1500))
        md = int(rng.integers(0, 700))
        shapes.append(Config(f"rand{k}_p{p}", "bf16", b=b, h=g * p, g=g, d=128, mc=mc, md=md))
    return shapes


@pytest.mark.parametrize("cfg", _random_shapes(), ids=lambda c: c.name)
def test_random_shapes_all_rows(cfg):
    inp = make_inputs(cfg, 99, variant="ragged" if cfg.md > 0 else "normal")
    out, lse = run_gpu(inp)
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, f"{cfg.name} {ba.ba_plan_string(ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype))[:40]}")


@pytest.mark.parametrize("cfg", [
    # dynamic CUDA-core decode columns cut into parts (few, long columns):
    # p = 1 and p = 2, ragged lens incl. 0, a part past a column's length
    Config("dyn_p1_parts", "bf16", b=16, h=2, g=2, d=128, mc=200, md=2500),
    Config("dyn_p2_parts", "bf16", b=8, h=4, g=2, d=128, mc=300, md=3000),
    Config("dyn_p2_fused", "bf16", b=8, h=6, g=3, d=128, mc=1100, md=600),
], ids=lambda c: c.name)
def test_dyn_decode_parts_all_rows(cfg):
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype)
    plan = ba.ba_plan_string(prob)
    assert "cuda_core_dyn" in plan, plan
    for variant in ("ragged", "normal"):
        inp = make_inputs(cfg, 77, variant=variant)
        out, lse = run_gpu(inp)
        ref, ref_lse = oracle_rows(inp)
        compare(out, lse, ref, ref_lse, cfg.torch_dtype, f"{cfg.name} {variant} {plan[:60]}")


@pytest.mark.parametrize("cfg", [
    # two-block ping-pong rows kernel (context-only launch): a partly filled
    # block B, an odd block count (last pair without B), g = 1 (Q rows by a
    # 2-D box), ragged decode lengths in the dynamic decode launch
    Config("rows2_b200", "bf16", b=200, h=2, g=2, d=128, mc=1500, md=700),
    Config("rows2_b130", "bf16", b=130, h=4, g=4, d=128, mc=900, md=300),
    Config("rows2_mqa_odd", "bf16", b=300, h=1, g=1, d=128, mc=1000, md=2000),
], ids=lambda c: c.name)
def test_rows2_kernel_all_rows(cfg):
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype)
    plan = ba.ba_plan_string(prob)
    assert plan.startswith("ctx_rows2"), plan
    inp = make_inputs(cfg, 88, variant="ragged")
    out, lse = run_gpu(inp)
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, f"{cfg.name} {plan[:60]}")


def test_fma_and_tc_plans_share_one_workspace():
    """One workspace serves the CUDA-core plan (n = 1, b*p = 8 rows) and the
    tensor-core plan (n = 4: 32 rows, grid barrier) alternately: the FMA plan
    never writes the barrier words at bytes [0, 256) (speculative decoding
    with a single- and a multi-token step sharing a workspace)."""
    cfg = Config("spec", "bf16", b=8, h=4, g=4, d=128, mc=600, md=40)
    one = make_inputs(cfg, 31, device=DEV)
    four = make_inputs(cfg, 32, device=DEV, n_tok=4)
    p1 = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, n_tok=1)
    p4 = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, n_tok=4)
    assert "fma" in ba.ba_plan_string(p1) and "fused_tc" in ba.ba_plan_string(p4)
    ws = torch.zeros(max(ba.ba_workspace_bytes(p1), ba.ba_workspace_bytes(p4)), dtype=torch.uint8,
                     device=DEV)
    ref1, _ = oracle_rows(one)
    ref4, _ = oracle_rows(type(four)(*(t.cpu() if torch.is_tensor(t) else t for t in
                                       (four.q, four.Kc, four.Vc, four.Kd, four.Vd, four.lens,
                                        four.scale))))
    for _ in range(3):
        o1 = ba.bifurcated_attn_decode(one.q, one.Kc, one.Vc, one.Kd, one.Vd, one.lens,
                                       scale=one.scale, workspace=ws)
        o4 = ba.bifurcated_attn_decode(four.q, four.Kc, four.Vc, four.Kd, four.Vd, four.lens,
                                       scale=four.scale, workspace=ws)
        torch.cuda.synchronize()
        compare(o1, None, ref1, None, cfg.torch_dtype, "fma-on-shared-ws")
        compare(o4, None, ref4, None, cfg.torch_dtype, "tc-on-shared-ws")


def test_two_fused_plans_share_one_workspace():
    """Two fused tensor-core plans with different row counts (n = 1: 64 rows,
    dynamic CUDA-core decode columns; n = 2: 128 rows, multi-token kernel)
    alternate on one workspace (the grid-barrier words and the column queue
    are left at 0 by every completed call)."""
    cfg = Config("alt", "bf16", b=16, h=4, g=4, d=128, mc=900, md=70)
    one = make_inputs(cfg, 41, device=DEV)
    two = make_inputs(cfg, 42, device=DEV, n_tok=2)
    p1 = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, n_tok=1)
    p2 = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, n_tok=2)
    assert "fused_tc" in ba.ba_plan_string(p1) and "fused_tc" in ba.ba_plan_string(p2)
    ws = torch.zeros(max(ba.ba_workspace_bytes(p1), ba.ba_workspace_bytes(p2)), dtype=torch.uint8,
                     device=DEV)
    ref1, _ = oracle_rows(one)
    ref2, _ = oracle_rows(type(two)(*(t.cpu() if torch.is_tensor(t) else t for t in
                                      (two.q, two.Kc, two.Vc, two.Kd, two.Vd, two.lens,
                                       two.scale))))
    for _ in range(3):
        o1 = ba.bifurcated_attn_decode(one.q, one.Kc, one.Vc, one.Kd, one.Vd, one.lens,
                                       scale=one.scale, workspace=ws)
        o1b = ba.bifurcated_attn_decode(one.q, one.Kc, one.Vc, one.Kd, one.Vd, one.lens,
                                        scale=one.scale, workspace=ws)
        o2 = ba.bifurcated_attn_decode(two.q, two.Kc, two.Vc, two.Kd, two.Vd, two.lens,
                                       scale=two.scale, workspace=ws)
        torch.cuda.synchronize()
        compare(o1, None, ref1, None, cfg.torch_dtype, "plan1-on-shared-ws")
        compare(o1b, None, ref1, None, cfg.torch_dtype, "plan1-again")
        compare(o2, None, ref2, None, cfg.torch_dtype, "plan2-on-shared-ws")


def test_binding_rejects_mismatched_shapes():
    cfg = Config("x", "bf16", b=3, h=4, g=2, d=128, mc=64, md=8)
    inp = make_inputs(cfg, 16, device=DEV)
    with pytest.raises(ValueError):
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc[:, :32].contiguous(), inp.Kd, inp.Vd,
                                  inp.lens)
    with pytest.raises(ValueError):
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens[:2].contiguous())
    with pytest.raises(ValueError):
        bad_lse = torch.empty(cfg.b, cfg.h + 1, dtype=torch.float32, device=DEV)
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, lse=bad_lse)
    with pytest.raises(ValueError):
        bad_out = torch.empty(cfg.b, cfg.h, cfg.d, dtype=torch.float32, device=DEV)
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, bad_out)
