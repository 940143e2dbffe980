"""Pins for the multi-token oracle (App. G; SPEC.md:441-449
decode_multi), CPU only.

oracle_attn_decode_multi_f64 is plain masked attention: token k of sample i
sits at cache position mc + L_i - n + k and sees every context position and the
decode positions t < L_i - (n - 1 - k).  It is pinned against
  * torch SDPA in float64 with an explicit boolean mask (library routine);
  * teacher forcing: token k equals the single-token oracle —
    itself pinned in test_oracle_pins.py — run with lens - (n - 1 - k);
  * n = 1 reducing to the single-token oracle;
  * a closed form: the last token's own key, planted, dominates only its row,
    and earlier tokens are blind to the later drafts' K/V;
and a mask off-by-one mutation must fail parity.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import Config, make_inputs


def _run(inp, **kw):
    return oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                              scale=inp.scale, **kw)


def sdpa_multi(inp, shift=0):
    """torch fp64 SDPA over Kc ⊕ Kd[i][:L] with the causal boolean mask of the
    n draft tokens (token k at position mc + L - n + k).  ``shift`` moves the
    mask diagonal (a mutation for the negative test)."""
    q = inp.q.double()
    b, h, n, d = q.shape
    g, mc, _ = inp.Kc.shape
    p = h // g
    outs = []
    for i in range(b):
        L = int(inp.lens[i])
        K = torch.cat([inp.Kc.double(), inp.Kd[i, :, :L].double()], dim=1).repeat_interleave(p, 0)
        V = torch.cat([inp.Vc.double(), inp.Vd[i, :, :L].double()], dim=1).repeat_interleave(p, 0)
        M = mc + L
        t = torch.arange(M).unsqueeze(0)          # [1][M]
        pos = (mc + L - n + torch.arange(n)).unsqueeze(1) + shift  # [n][1]
        mask = (t < mc) | (t <= pos)              # [n][M] True = attend
        o = torch.nn.functional.scaled_dot_product_attention(
            q[i], K, V, attn_mask=mask.unsqueeze(0).expand(h, n, M), scale=inp.scale)
        outs.append(o)                            # [h][n][d]
    return torch.stack(outs).reshape(b * h * n, d).numpy()


def _rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


SHAPES = [
    Config("mt_mha", "fp32", b=3, h=4, g=4, d=16, mc=20, md=9),
    Config("mt_gqa", "bf16", b=2, h=6, g=2, d=32, mc=33, md=12),
    Config("mt_mqa", "fp32", b=4, h=3, g=1, d=8, mc=5, md=7),
]


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("variant", ["normal", "ragged", "dec_dom"])
def test_multi_against_torch_sdpa_masked(cfg, n, variant):
    inp = make_inputs(cfg, 5 + n, variant=variant, n_tok=n)
    out, lse, _ = _run(inp)
    ref = sdpa_multi(inp)
    assert _rel(out, ref) <= 1e-12


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
def test_teacher_forcing_equals_sequential_single_steps(cfg):
    """the n-token step equals n single-token steps fed the same
    tokens — token k is the single-token step whose decode cache ends at its
    own position (lens - (n - 1 - k)), computed by the pinned 1-token oracle."""
    n = 3
    inp = make_inputs(cfg, 17, variant="ragged", n_tok=n)
    out, lse, _ = _run(inp)
    b, h = cfg.b, cfg.h
    out = out.reshape(b, h, n, cfg.d)
    lse = lse.reshape(b, h, n)
    for k in range(n):
        lens_k = torch.clamp(inp.lens - (n - 1 - k), min=0).to(torch.int32)
        o1, l1, _ = oracle.attn_decode(inp.q[:, :, k].contiguous(), inp.Kc, inp.Vc, inp.Kd,
                                       inp.Vd, lens_k, scale=inp.scale)
        np.testing.assert_allclose(out[:, :, k].reshape(b * h, -1), o1, rtol=0, atol=1e-14)
        np.testing.assert_allclose(lse[:, :, k].reshape(-1), l1, rtol=0, atol=1e-13)


def test_single_token_limit():
    cfg = SHAPES[1]
    inp = make_inputs(cfg, 3, variant="ragged")
    o1, l1, _ = _run(inp)
    q4 = inp.q.unsqueeze(2).contiguous()
    o4, l4, _ = oracle.attn_decode(q4, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, scale=inp.scale)
    np.testing.assert_allclose(o4, o1, rtol=0, atol=1e-15)
    np.testing.assert_allclose(l4, l1, rtol=0, atol=1e-14)


def test_last_token_own_key_and_blind_earlier_tokens():
    """Plant q[i,j,n-1] on the last decode key (the last draft's own key): that
    row returns its V row; then overwrite the last draft's K/V — rows of the
    earlier tokens must not change at all (they may not see later drafts)."""
    cfg = Config("x", "fp32", b=2, h=2, g=2, d=16, mc=24, md=6)
    n = 3
    inp = make_inputs(cfg, 9, n_tok=n)
    L = cfg.md
    for i in range(cfg.b):
        for j in range(cfg.h):
            k = inp.Kd[i, j, L - 1]
            inp.q[i, j, n - 1] = 32.0 * k / k.norm() * cfg.d ** 0.5
    out, _, _ = _run(inp)
    out = out.reshape(cfg.b, cfg.h, n, cfg.d)
    for i in range(cfg.b):
        for j in range(cfg.h):
            np.testing.assert_allclose(out[i, j, n - 1], inp.Vd[i, j, L - 1].double().numpy(),
                                       atol=1e-4)
    Kd2, Vd2 = inp.Kd.clone(), inp.Vd.clone()
    Kd2[:, :, L - 1] = 100.0
    Vd2[:, :, L - 1] = -7.0
    out2, _, _ = oracle.attn_decode(inp.q, inp.Kc, inp.Vc, Kd2, Vd2, inp.lens, scale=inp.scale)
    out2 = out2.reshape(cfg.b, cfg.h, n, cfg.d)
    assert np.array_equal(out2[:, :, : n - 1], out[:, :, : n - 1])
    assert not np.allclose(out2[:, :, n - 1], out[:, :, n - 1])


def test_short_lens_context_only_tokens():
    """lens[i] < n: tokens whose causal bound is <= 0 see the context only."""
    cfg = Config("x", "fp32", b=2, h=2, g=1, d=8, mc=10, md=4)
    n = 4
    inp = make_inputs(cfg, 4, n_tok=n, lens=[1, 0])
    out, _, _ = _run(inp)
    out = out.reshape(cfg.b, cfg.h, n, cfg.d)
    ctx_only, _, _ = oracle.attn_decode(inp.q[:, :, 0].contiguous(), inp.Kc, inp.Vc, inp.Kd,
                                        inp.Vd, torch.zeros(2, dtype=torch.int32),
                                        scale=inp.scale)
    ctx_only = ctx_only.reshape(cfg.b, cfg.h, cfg.d)
    # sample 0 (lens 1): tokens 0..2 context-only; sample 1 (lens 0): all
    np.testing.assert_allclose(out[0, :, 0], ctx_only[0], atol=1e-15)
    np.testing.assert_allclose(out[1, :, 0], ctx_only[1], atol=1e-15)


def test_mask_off_by_one_fails_parity():
    cfg = SHAPES[0]
    inp = make_inputs(cfg, 11, variant="dec_dom", n_tok=4)
    out, _, _ = _run(inp)
    assert _rel(out, sdpa_multi(inp)) <= 1e-12
    bad = sdpa_multi(inp, shift=1)
    err = np.abs(bad - out)
    assert not np.all(err <= np.maximum(2e-3, 1e-2 * np.abs(out))), "mask shift not detected"


def test_multi_invalid_rejected():
    cfg = SHAPES[0]
    inp = make_inputs(cfg, 1, n_tok=2)
    with pytest.raises(AssertionError):
        oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, scale=inp.scale,
                           bifurcated=True)
