"""Pins for the fp64 oracle (CPU only, marker "not gpu").

Each test checks the oracle against something other than itself: values the
paper/SPEC fix for worked examples (tests/golden/, cited), a library routine
(torch fp64 SDPA over the replicated cache), the paper's own App. E.3 listing
run in torch fp64, closed forms, invariants, brute force at 50 digits, and
mutation checks showing the comparison rejects plausible mistakes.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from synth import CONFIGS, Config, alg_bytes, make_inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _t(x, dt=torch.float32):
    return torch.tensor(x, dtype=dt)


def _run(inp, **kw):
    return oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                              scale=inp.scale, **kw)


# ----------------------------------------------------------------------------
# Independent references (not the oracle's code)
# ----------------------------------------------------------------------------
def sdpa_reference(inp):
    """torch SDPA in float64 over the materialised replicated cache: the
    'naive' attention of PAPER.md:229 with K = Kc ⊕ Kd."""
    q = inp.q.double()
    b, h, d = q.shape
    g, mc, _ = inp.Kc.shape
    p = h // g
    outs, lses = [], []
    for i in range(b):
        L = int(inp.lens[i])
        K = torch.cat([inp.Kc.double(), inp.Kd[i, :, :L].double()], dim=1)  # [g][M][d]
        V = torch.cat([inp.Vc.double(), inp.Vd[i, :, :L].double()], dim=1)
        K = K.repeat_interleave(p, dim=0)  # head j -> group j // p
        V = V.repeat_interleave(p, dim=0)
        qi = q[i].unsqueeze(1)  # [h][1][d]
        o = torch.nn.functional.scaled_dot_product_attention(
            qi.unsqueeze(0), K.unsqueeze(0), V.unsqueeze(0), scale=inp.scale)[0, :, 0]
        s = (qi @ K.transpose(1, 2))[:, 0] * inp.scale
        outs.append(o)
        lses.append(torch.logsumexp(s, dim=-1))
    return torch.stack(outs).reshape(b * h, d).numpy(), torch.stack(lses).reshape(-1).numpy()


def paper_listing_reference(inp):
    """The App. E.3 code in torch float64: 4 einsums, cat,
    softmax (with the 1/sqrt scale of reading R1), split, add.  Uniform lens."""
    b, h, d = inp.q.shape
    g, mc, _ = inp.Kc.shape
    p = h // g
    L = int(inp.lens[0])
    assert all(int(x) == L for x in inp.lens)
    query = inp.q.double().reshape(b, g, p, 1, d)
    ctx_k = inp.Kc.double().unsqueeze(0)  # [1][g][mc][d]  ("context_past_key")
    ctx_v = inp.Vc.double().unsqueeze(0)
    inc_k = inp.Kd.double()[:, :, :L]     # "incremental_past_key"
    inc_v = inp.Vd.double()[:, :, :L]
    w_ctx = torch.einsum("bgpnk,gmk->bgpnm", query, ctx_k[0])
    w_inc = torch.einsum("bgpnk,bgmk->bgpnm", query, inc_k)
    w = torch.cat([w_ctx, w_inc], dim=-1) * inp.scale
    w = torch.softmax(w, dim=-1)
    n_ctx = ctx_v.size(-2)
    o_ctx = torch.einsum("bgpnm,gmv->bgpnv", w[..., :n_ctx], ctx_v[0])
    o_inc = torch.einsum("bgpnm,bgmv->bgpnv", w[..., n_ctx:], inc_v)
    return (o_ctx + o_inc).reshape(b * h, d).numpy()


def _rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


# ----------------------------------------------------------------------------
# Golden worked examples
# ----------------------------------------------------------------------------
def test_spec_bifurcated_logits_example():
    G = _load("spec_bifurcated_logits.json")
    b, d = G["b"], G["d"]
    q = _t(G["q"])
    Kc = _t(G["Kc"])
    Kd = _t(G["Kd"])
    Vc = torch.zeros_like(Kc)
    Vd = torch.zeros_like(Kd)
    lens = torch.full((b,), G["md"], dtype=torch.int32)
    _, lse, w = oracle.attn_decode(q, Kc, Vc, Kd, Vd, lens, scale=1.0, weights=True)
    for i, lg in enumerate(G["expected_logits"]):
        lg = np.array(lg, dtype=np.float64)
        ex = np.exp(lg - lg.max())
        np.testing.assert_allclose(w[i], ex / ex.sum(), rtol=0, atol=1e-15)
        assert abs(lse[i] - math.log(np.exp(lg).sum())) < 1e-14


def test_spec_weight_value_example():
    G = _load("spec_weight_value.json")
    q, Kc, Vc, Kd, Vd = (_t(G[k]) for k in ("q", "Kc", "Vc", "Kd", "Vd"))
    lens = torch.tensor([G["md"]], dtype=torch.int32)
    out, _, w = oracle.attn_decode(q, Kc, Vc, Kd, Vd, lens, scale=1.0, weights=True)
    np.testing.assert_allclose(w[0], G["expected_weights"], atol=G["tol"])
    np.testing.assert_allclose(out[0], G["expected_out"], atol=G["tol"] * 10)
    outb, _, _ = oracle.attn_decode(q, Kc, Vc, Kd, Vd, lens, scale=1.0, bifurcated=True)
    np.testing.assert_allclose(outb[0], G["expected_out"], atol=G["tol"] * 10)


def test_spec_softmax_examples():
    G = _load("spec_softmax.json")
    for case in G["cases"]:
        x0, x1 = case["logits"]
        q = _t([[[1.0]]])
        Kc = _t([[[x0], [x1]]])
        Vc = _t([[[1.0], [0.0]]])
        Kd = torch.zeros(1, 1, 0, 1)
        Vd = torch.zeros(1, 1, 0, 1)
        lens = torch.zeros(1, dtype=torch.int32)
        out, _, w = oracle.attn_decode(q, Kc, Vc, Kd, Vd, lens, scale=1.0, weights=True)
        np.testing.assert_allclose(w[0], case["expected"], atol=case["tol"])
        assert np.all(np.isfinite(w))
        np.testing.assert_allclose(out[0, 0], case["expected"][0], atol=case["tol"])


def test_spec_io_counts():
    G = _load("spec_io.json")
    for c in G["cases"]:
        args = (c["b"], c["g"], c["k"], c["mc"], c["md"])
        assert oracle.kv_read_elements(*args, bifurcated=False) == c["naive"]
        assert oracle.kv_read_elements(*args, bifurcated=True) == c["bifurcated"]
    # md = 0: ratio is exactly b ("as high as b-fold")
    for b in (2, 7, 32):
        assert oracle.kv_read_elements(b, 4, 128, 1024, 0, False) == \
            b * oracle.kv_read_elements(b, 4, 128, 1024, 0, True)


def test_alg_bytes_matches_eq6():
    """bench.py's byte count = Eq. 6 x (K and V) x element bytes + q/out."""
    for cfg in CONFIGS.values():
        kv = oracle.kv_read_elements(cfg.b, cfg.g, cfg.d, cfg.mc, cfg.md, True)
        assert alg_bytes(cfg) == 2 * kv * cfg.kv_bytes + 2 * cfg.elem_bytes * cfg.b * cfg.h * cfg.d
    assert alg_bytes(CONFIGS["mha7b_b32"]) == 268_959_744
    assert alg_bytes(CONFIGS["mha7b_b16"]) == 201_588_736
    assert alg_bytes(CONFIGS["tiny"]) == 13_312


# ----------------------------------------------------------------------------
# Closed forms and special cases
# ----------------------------------------------------------------------------
def test_single_key_returns_that_value_row():
    """softmax over one logit is 1, so out = that V row."""
    cfg = Config("x", "fp32", b=3, h=4, g=2, d=8, mc=1, md=0)
    inp = make_inputs(cfg, 1)
    out, lse, _ = _run(inp)
    p = cfg.p
    for i in range(cfg.b):
        for j in range(cfg.h):
            np.testing.assert_array_equal(out[i * cfg.h + j], inp.Vc[j // p, 0].double().numpy())
            s = inp.scale * float((inp.q[i, j].double() * inp.Kc[j // p, 0].double()).sum())
            assert abs(lse[i * cfg.h + j] - s) < 1e-12


def test_equal_logits_average():
    """two keys with equal logits, V rows [2,0],[0,2] -> [1,1]."""
    q = _t([[[1.0, 0.0]]])
    Kc = _t([[[1.0, 5.0], [1.0, -3.0]]])
    Vc = _t([[[2.0, 0.0], [0.0, 2.0]]])
    out, _, _ = oracle.attn_decode(q, Kc, Vc, torch.zeros(1, 1, 0, 2), torch.zeros(1, 1, 0, 2),
                                   torch.zeros(1, dtype=torch.int32), scale=1.0)
    np.testing.assert_array_equal(out[0], [1.0, 1.0])


def test_zero_query_gives_mean_of_values():
    cfg = Config("x", "bf16", b=3, h=4, g=2, d=16, mc=19, md=5)
    inp = make_inputs(cfg, 2, variant="ragged")
    inp.q.zero_()
    out, lse, _ = _run(inp)
    for i in range(cfg.b):
        L = int(inp.lens[i])
        for j in range(cfg.h):
            c = j // cfg.p
            V = torch.cat([inp.Vc[c].double(), inp.Vd[i, c, :L].double()])
            np.testing.assert_allclose(out[i * cfg.h + j], V.mean(0).numpy(), rtol=0, atol=1e-14)
            assert abs(lse[i * cfg.h + j] - math.log(cfg.mc + L)) < 1e-13


@pytest.mark.parametrize("variant", ["planted_ctx", "planted_dec"])
def test_planted_key_dominates(variant):
    cfg = Config("x", "bf16", b=4, h=4, g=2, d=32, mc=40, md=6)
    inp = make_inputs(cfg, 3, variant=variant)
    out, _, w = _run(inp, weights=True)
    # the dominant weight exceeds 1 - 1e-9 and the output is that key's V row
    assert np.all(w.max(axis=1) > 1 - 1e-9)
    for i in range(cfg.b):
        for j in range(cfg.h):
            r = i * cfg.h + j
            t = int(np.argmax(w[r]))
            c = j // cfg.p
            if variant == "planted_ctx":
                assert t < cfg.mc
            else:
                assert t >= cfg.mc
            v = inp.Vc[c, t] if t < cfg.mc else inp.Vd[i, c, t - cfg.mc]
            np.testing.assert_allclose(out[r], v.double().numpy(), atol=1e-7)


def test_lens_zero_is_context_only():
    cfg = Config("x", "fp32", b=3, h=2, g=1, d=8, mc=11, md=4)
    inp = make_inputs(cfg, 4, lens=[0, 4, 0])
    out, lse, _ = _run(inp)
    inp0 = make_inputs(cfg.with_(md=0), 4, md_cap=0, lens=[0, 0, 0])
    inp0.q.copy_(inp.q); inp0.Kc.copy_(inp.Kc); inp0.Vc.copy_(inp.Vc)
    out0, lse0, _ = _run(inp0)
    for i in (0, 2):
        sl = slice(i * cfg.h, (i + 1) * cfg.h)
        np.testing.assert_array_equal(out[sl], out0[sl])
        np.testing.assert_array_equal(lse[sl], lse0[sl])


def test_identical_samples_identical_rows():
    cfg = Config("x", "bf16", b=5, h=4, g=4, d=16, mc=23, md=3)
    inp = make_inputs(cfg, 5, variant="equal")
    out, _, _ = _run(inp)
    out = out.reshape(cfg.b, cfg.h, cfg.d)
    for i in range(1, cfg.b):
        np.testing.assert_array_equal(out[i], out[0])


# ----------------------------------------------------------------------------
# Library routine and the paper's listing
# ----------------------------------------------------------------------------
SHAPES = [
    Config("t1", "fp32", b=4, h=2, g=2, d=16, mc=32, md=4),   # BASELINE tiny
    Config("t2", "bf16", b=3, h=8, g=2, d=32, mc=70, md=9),   # GQA-like
    Config("t3", "bf16", b=2, h=6, g=1, d=24, mc=33, md=5),   # MQA-like
    Config("t4", "fp32", b=1, h=4, g=4, d=8, mc=5, md=0),     # b=1, no decode part
    Config("t5", "bf16", b=6, h=4, g=4, d=64, mc=129, md=17), # MHA, ragged tile counts
]


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("variant", ["normal", "ragged", "peaky", "ctx_dom", "dec_dom"])
def test_against_torch_sdpa_fp64(cfg, variant):
    inp = make_inputs(cfg, 11, variant=variant)
    out, lse, _ = _run(inp)
    ref, ref_lse = sdpa_reference(inp)
    assert _rel(out, ref) < 1e-12
    np.testing.assert_allclose(lse, ref_lse, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
def test_against_paper_listing_fp64(cfg):
    inp = make_inputs(cfg, 12)
    out, _, _ = _run(inp)
    ref = paper_listing_reference(inp)
    assert _rel(out, ref) < 1e-12


def test_tiny_config_against_torch_sdpa():
    cfg = CONFIGS["tiny"]
    inp = make_inputs(cfg, 20240313)
    out, lse, _ = _run(inp)
    ref, ref_lse = sdpa_reference(inp)
    assert _rel(out, ref) < 1e-13
    np.testing.assert_allclose(lse, ref_lse, rtol=1e-14)


def test_brute_force_mpmath_tiny():
    """50-digit evaluation of Eq. 1-2 + softmax on the tiny config."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    cfg = CONFIGS["tiny"]
    inp = make_inputs(cfg, 20240313, variant="ragged")
    out, lse, _ = _run(inp)
    s = mp.mpf(inp.scale)
    for i in range(cfg.b):
        L = int(inp.lens[i])
        for j in range(cfg.h):
            c = j // cfg.p
            keys = [inp.Kc[c, t] for t in range(cfg.mc)] + [inp.Kd[i, c, t] for t in range(L)]
            vals = [inp.Vc[c, t] for t in range(cfg.mc)] + [inp.Vd[i, c, t] for t in range(L)]
            qv = [mp.mpf(float(x)) for x in inp.q[i, j]]
            lg = [s * mp.fsum(qv[x] * mp.mpf(float(k[x])) for x in range(cfg.d)) for k in keys]
            Z = mp.fsum(mp.e ** x for x in lg)
            for x in range(cfg.d):
                o = mp.fsum(mp.e ** lg[t] * mp.mpf(float(vals[t][x])) for t in range(len(lg))) / Z
                assert abs(float(o) - out[i * cfg.h + j, x]) <= 1e-13 * max(abs(float(o)), 1e-3)
            assert abs(float(mp.log(Z)) - lse[i * cfg.h + j]) < 1e-13


# ----------------------------------------------------------------------------
# Invariants
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
def test_weights_sum_to_one(cfg):
    inp = make_inputs(cfg, 13, variant="ragged")
    _, _, w = _run(inp, weights=True)
    assert np.max(np.abs(w.sum(axis=1) - 1.0)) < 1e-12
    assert np.all(w >= 0)


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("variant", ["normal", "ragged"])
def test_bifurcated_mode_equals_replicated(cfg, variant):
    """App. E.1: bifurcated == replicated.  Weights are
    bit-exact (same order); outputs agree to fp64 rounding (Eq. 4 splits the
    value sum at mc)."""
    inp = make_inputs(cfg, 14, variant=variant)
    out, lse, w = _run(inp, weights=True)
    outb, lseb, wb = _run(inp, weights=True, bifurcated=True)
    np.testing.assert_array_equal(w, wb)
    np.testing.assert_array_equal(lse, lseb)
    assert _rel(outb, out) < 1e-14


def test_bifurcated_bit_exact_without_decode_part():
    cfg = Config("x", "bf16", b=3, h=4, g=2, d=32, mc=50, md=6)
    inp = make_inputs(cfg, 15, lens=[0, 0, 0])
    out, _, _ = _run(inp)
    outb, _, _ = _run(inp, bifurcated=True)
    np.testing.assert_array_equal(out, outb)


def test_shift_invariance():
    """Adding a constant to all logits of a row leaves the output unchanged
    (SPEC.md:102).  Adding u to every key shifts row (i,j)'s logits by
    s*<q_ij, u>; lse shifts by the same amount."""
    cfg = Config("x", "fp32", b=2, h=2, g=1, d=4, mc=9, md=3)
    inp = make_inputs(cfg, 16)
    out, lse, _ = _run(inp)
    u = torch.tensor([0.5, -0.25, 1.0, 0.125])
    inp.Kc += u
    inp.Kd += u
    out2, lse2, _ = _run(inp)
    np.testing.assert_allclose(out2, out, atol=1e-6)
    shift = inp.scale * (inp.q.double() @ u.double()).reshape(-1).numpy()
    np.testing.assert_allclose(lse2 - lse, shift, atol=1e-5)


def test_mqa_equals_mha_with_replicated_kv():
    """g=1 and g=h agree when K/V are replicated across groups."""
    mq = Config("x", "bf16", b=3, h=4, g=1, d=16, mc=21, md=5)
    inp = make_inputs(mq, 17, variant="ragged")
    out1, lse1, _ = _run(inp)
    h = mq.h
    inp_h = make_inputs(mq.with_(g=h), 17)
    inp_h.q.copy_(inp.q)
    inp_h.Kc.copy_(inp.Kc.expand(h, -1, -1))
    inp_h.Vc.copy_(inp.Vc.expand(h, -1, -1))
    inp_h.Kd.copy_(inp.Kd.expand(-1, h, -1, -1))
    inp_h.Vd.copy_(inp.Vd.expand(-1, h, -1, -1))
    inp_h.lens.copy_(inp.lens)
    outh, lseh, _ = _run(inp_h)
    np.testing.assert_array_equal(out1, outh)
    np.testing.assert_array_equal(lse1, lseh)


def test_rows_subset_matches_full():
    cfg = Config("x", "bf16", b=4, h=6, g=3, d=16, mc=31, md=7)
    inp = make_inputs(cfg, 18, variant="ragged")
    out, lse, _ = _run(inp)
    rows = [23, 0, 7, 11, 11]
    outs, lses, _ = _run(inp, rows=rows)
    np.testing.assert_array_equal(outs, out[rows])
    np.testing.assert_array_equal(lses, lse[rows])


def test_threads_do_not_change_results():
    cfg = Config("x", "bf16", b=4, h=8, g=2, d=32, mc=64, md=8)
    inp = make_inputs(cfg, 19)
    out1, lse1, _ = _run(inp, nthreads=1)
    out4, lse4, _ = _run(inp, nthreads=4)
    np.testing.assert_array_equal(out1, out4)
    np.testing.assert_array_equal(lse1, lse4)


def test_invalid_problem_rejected():
    cfg = Config("x", "fp32", b=2, h=3, g=2, d=4, mc=4, md=1)  # h % g != 0
    inp = make_inputs(cfg.with_(h=4), 1)
    with pytest.raises(ValueError):
        oracle.attn_decode(inp.q[:, :3], inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, scale=1.0)


# ----------------------------------------------------------------------------
# Mutations: plausible mistakes must fail the pins / the parity tolerance
# ----------------------------------------------------------------------------
def _mutant(inp, kind):
    """Deliberately wrong variants of the step (torch fp64)."""
    q = inp.q.double()
    b, h, d = q.shape
    g = inp.Kc.shape[0]
    p = h // g
    out = torch.zeros(b, h, d, dtype=torch.float64)
    for i in range(b):
        L = int(inp.lens[i])
        for j in range(h):
            c = (j % g) if kind == "group_map" else j // p
            Kc, Vc = inp.Kc[c].double(), inp.Vc[c].double()
            Kd, Vd = inp.Kd[i, c, :L].double(), inp.Vd[i, c, :L].double()
            sc = Kc @ q[i, j] * inp.scale
            sd = Kd @ q[i, j] * inp.scale
            if kind == "per_branch_softmax":
                o = torch.softmax(sc, 0) @ Vc + (torch.softmax(sd, 0) @ Vd if L else 0)
            elif kind == "drop_decode":
                o = torch.softmax(sc, 0) @ Vc
            elif kind == "no_rescale":
                # merge two partials without the e^{m_k - M} correction
                ec, ed = torch.exp(sc - sc.max()), torch.exp(sd - sd.max()) if L else sd
                o = (ec @ Vc + (ed @ Vd if L else 0)) / (ec.sum() + (ed.sum() if L else 0))
            elif kind in ("group_map", "swapped_kv"):
                s = torch.cat([sc, sd])
                V = torch.cat([Kc, Kd]) if kind == "swapped_kv" else torch.cat([Vc, Vd])
                o = torch.softmax(s, 0) @ V
            else:
                raise ValueError(kind)
            out[i, j] = o
    return out.reshape(b * h, d).numpy()


def parity_ok(gpu, ref, abs_tol=2e-3, rel_tol=1e-2):
    """The bf16 parity criterion of the GPU tests (reading R12)."""
    err = np.abs(gpu - ref)
    return bool(np.all(err <= np.maximum(abs_tol, rel_tol * np.abs(ref))))


@pytest.mark.parametrize("kind", ["per_branch_softmax", "drop_decode", "no_rescale",
                                  "group_map", "swapped_kv"])
def test_mutants_fail_parity(kind):
    cfg = Config("x", "bf16", b=3, h=4, g=2, d=32, mc=48, md=16)
    inp = make_inputs(cfg, 21, variant="dec_dom")
    out, _, _ = _run(inp)
    ref, _ = sdpa_reference(inp)
    assert parity_ok(out, ref, 1e-12, 1e-12)
    bad = _mutant(inp, kind)
    assert not parity_ok(bad, out), f"mutation {kind} was not detected"
