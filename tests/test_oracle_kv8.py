"""Pins for the FP8 (E4M3) KV oracle (oracle_attn_decode_kv8_f64; SURVEY §8(f)
row f4, PAPER.md:698 FAQ 5; reading R19).  CPU only.

The oracle dequantises each E4M3 code exactly (value x per-tensor fp32 scale)
and runs Eq. 1-2 in fp64.  It is pinned to things other than itself:
  * the E4M3 decode table against torch.float8_e4m3fn (library) for all 256
    codes, plus closed forms of the OCP format (1.0, 448, 2^-6, 2^-9, NaN);
  * with power-of-two scales the dequantised cache is exact in fp32, so the
    result must equal the (already pinned) plain oracle on those fp32 tensors
    BIT FOR BIT;
  * with arbitrary scales, torch fp64 SDPA over the dequantised replicated
    cache (library routine) within 1e-12;
  * mutations (a dropped k_scale or v_scale, K/V scales swapped, codes read as
    E5M2) fail the parity criterion.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from synth import CONFIGS, Config, make_inputs


def test_e4m3_table_matches_torch_for_all_codes():
    ref = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).double().tolist()
    for c in range(256):
        v = oracle.e4m3_value(c)
        if math.isnan(ref[c]):
            assert math.isnan(v), c
        else:
            assert v == ref[c], (c, v, ref[c])


def test_e4m3_closed_forms():
    # OCP FP8 E4M3: bias 7, 3 mantissa bits, no infinities, S.1111.111 = NaN
    assert oracle.e4m3_value(0x38) == 1.0           # 0.0111.000 = 2^0
    assert oracle.e4m3_value(0x7E) == 448.0         # 0.1111.110 = 1.75 * 2^8, the max
    assert oracle.e4m3_value(0x08) == 2.0 ** -6     # smallest normal
    assert oracle.e4m3_value(0x01) == 2.0 ** -9     # smallest subnormal
    assert oracle.e4m3_value(0x07) == 7 * 2.0 ** -9  # largest subnormal
    assert oracle.e4m3_value(0xB8) == -1.0
    assert math.isnan(oracle.e4m3_value(0x7F)) and math.isnan(oracle.e4m3_value(0xFF))
    assert oracle.e4m3_value(0x80) == 0.0 and math.copysign(1, oracle.e4m3_value(0x80)) < 0


def _dequant(codes, scale, dt=torch.float64):
    return codes.view(torch.float8_e4m3fn).to(dt) * scale


def _kv8_inputs(cfg, seed, variant="normal", k_scale=None, v_scale=None):
    inp = make_inputs(cfg.with_(kv="e4m3"), seed, variant=variant)
    if k_scale is not None:
        inp.k_scale = k_scale
    if v_scale is not None:
        inp.v_scale = v_scale
    return inp


def _run_kv8(inp, **kw):
    return oracle.attn_decode_kv8(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                  scale=inp.scale, k_scale=inp.k_scale, v_scale=inp.v_scale, **kw)


SHAPES = [
    Config("mha", "bf16", b=3, h=4, g=4, d=32, mc=40, md=7),
    Config("gqa", "bf16", b=4, h=8, g=2, d=16, mc=33, md=5),
    Config("mqa", "bf16", b=2, h=6, g=1, d=64, mc=20, md=3),
]


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
@pytest.mark.parametrize("variant", ["normal", "ragged", "dec_dom"])
def test_pow2_scales_equal_plain_oracle_bitwise(cfg, variant):
    """Power-of-two scales: dequantised values are exact in fp32, so the FP8
    oracle must equal the plain fp32 oracle on them bit for bit."""
    inp = _kv8_inputs(cfg, 3, variant, k_scale=2.0 ** -5, v_scale=2.0 ** -3)
    out, lse, w = _run_kv8(inp, weights=True)
    f = lambda t, s: _dequant(t, s, torch.float32)  # noqa: E731
    ref, ref_lse, ref_w = oracle.attn_decode(inp.q.float(), f(inp.Kc, inp.k_scale),
                                             f(inp.Vc, inp.v_scale), f(inp.Kd, inp.k_scale),
                                             f(inp.Vd, inp.v_scale), inp.lens, scale=inp.scale,
                                             weights=True)
    np.testing.assert_array_equal(out, ref)
    np.testing.assert_array_equal(lse, ref_lse)
    np.testing.assert_array_equal(w, ref_w)


@pytest.mark.parametrize("cfg", SHAPES, ids=lambda c: c.name)
def test_arbitrary_scales_match_sdpa_fp64(cfg):
    """The generated amax/448 scales (not powers of two) against torch fp64 SDPA
    over the dequantised replicated cache."""
    inp = _kv8_inputs(cfg, 5, "ragged")
    assert inp.k_scale != 2.0 ** round(math.log2(inp.k_scale))
    out, lse, _ = _run_kv8(inp)
    b, h, d = inp.q.shape
    g = inp.Kc.shape[0]
    p = h // g
    q = inp.q.double()
    for i in range(b):
        L = int(inp.lens[i])
        K = torch.cat([_dequant(inp.Kc, inp.k_scale), _dequant(inp.Kd[i, :, :L], inp.k_scale)], 1)
        V = torch.cat([_dequant(inp.Vc, inp.v_scale), _dequant(inp.Vd[i, :, :L], inp.v_scale)], 1)
        K, V = K.repeat_interleave(p, 0), V.repeat_interleave(p, 0)
        o = torch.nn.functional.scaled_dot_product_attention(
            q[i].unsqueeze(1).unsqueeze(0), K.unsqueeze(0), V.unsqueeze(0), scale=inp.scale)
        s = (q[i].unsqueeze(1) @ K.transpose(1, 2))[:, 0] * inp.scale
        np.testing.assert_allclose(out[i * h:(i + 1) * h], o[0, :, 0].numpy(), rtol=1e-12,
                                   atol=1e-14)
        np.testing.assert_allclose(lse[i * h:(i + 1) * h], torch.logsumexp(s, -1).numpy(),
                                   rtol=1e-12, atol=1e-12)


def _fails_r12(a, b, abs_tol=2e-3, rel_tol=1e-2):
    if not np.isfinite(a).all():
        return True
    return bool((np.abs(a - b) > np.maximum(abs_tol, rel_tol * np.abs(b))).any())


def test_mutations_fail():
    cfg = SHAPES[0]
    inp = _kv8_inputs(cfg, 9, "normal")
    out, _, _ = _run_kv8(inp)
    # dropped v_scale
    bad, _, _ = oracle.attn_decode_kv8(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                       scale=inp.scale, k_scale=inp.k_scale, v_scale=1.0)
    assert _fails_r12(bad, out)
    # dropped k_scale (logits off by 1/k_scale)
    bad, _, _ = oracle.attn_decode_kv8(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                       scale=inp.scale, k_scale=1.0, v_scale=inp.v_scale)
    assert _fails_r12(bad, out)
    # codes read as E5M2 instead of E4M3
    as_e5 = lambda t: t.view(torch.uint8).view(torch.float8_e5m2).double()  # noqa: E731
    b, h, d = inp.q.shape
    K = torch.cat([as_e5(inp.Kc).unsqueeze(0).expand(b, -1, -1, -1), as_e5(inp.Kd)], 2) * inp.k_scale
    V = torch.cat([as_e5(inp.Vc).unsqueeze(0).expand(b, -1, -1, -1), as_e5(inp.Vd)], 2) * inp.v_scale
    o = torch.nn.functional.scaled_dot_product_attention(inp.q.double().unsqueeze(2), K, V,
                                                         scale=inp.scale)[:, :, 0]
    assert _fails_r12(o.reshape(-1, d).numpy(), out)


def test_fp8_config_bytes_halve_kv():
    """a7 for the FP8 cache: 2*1*d*g*(mc + sum lens) + 2*2*b*h*d (q/out bf16)."""
    from synth import alg_bytes
    c8, c16 = CONFIGS["mha7b_b32_fp8"], CONFIGS["mha7b_b32"]
    kv16 = 2 * 2 * c16.d * c16.g * (c16.mc + c16.b * c16.md)
    qo = 2 * 2 * c16.b * c16.h * c16.d
    assert alg_bytes(c16) == kv16 + qo == 268959744
    assert alg_bytes(c8) == kv16 // 2 + qo == 134742016
