"""GPU parity of the multi-token step (App. G,
PAPER.md:1219-1226; include/bifattn.h MULTI-TOKEN) through the C ABI against
the fp64 multi-token oracle (pinned in tests/test_oracle_multitoken.py), every
element, on both kernel families.  Shapes cover the tensor-core narrow decode
path (p*n <= 8), its general path (p*n > 8), N = 48 chunks (p*n = 6), ragged
lens including lens < n (tokens with no visible decode position), and the
replicated-cache baseline."""
import pytest
import torch

import paper_2403_08845_b200 as ba
from synth import Config, make_inputs
from tests.parity import compare, oracle_rows

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

CASES = [
    (Config("mt_mha", "bf16", b=12, h=8, g=8, d=128, mc=700, md=40), 4),
    (Config("mt_rows", "bf16", b=40, h=4, g=4, d=128, mc=333, md=20), 4),
    (Config("mt_mha_n2", "bf16", b=33, h=4, g=4, d=128, mc=300, md=130), 2),
    (Config("mt_gqa", "bf16", b=6, h=16, g=4, d=128, mc=513, md=77), 4),
    (Config("mt_p2n3", "bf16", b=5, h=4, g=2, d=128, mc=260, md=20), 3),
    (Config("mt_mqa", "bf16", b=3, h=12, g=1, d=128, mc=129, md=9), 2),
    (Config("mt_fp32", "fp32", b=3, h=4, g=2, d=64, mc=90, md=11), 3),
]


def _run(inp, flags=0):
    q = inp.q.to(DEV)
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=DEV)
    out = ba.bifurcated_attn_decode(q, inp.Kc.to(DEV), inp.Vc.to(DEV), inp.Kd.to(DEV),
                                    inp.Vd.to(DEV), inp.lens.to(DEV), lse=lse, scale=inp.scale,
                                    flags=flags)
    torch.cuda.synchronize()
    return out, lse


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0].name}_n{c[1]}")
@pytest.mark.parametrize("flags", [0, ba.BA_FLAG_FORCE_FMA, ba.BA_FLAG_CTX_ROWS,
                                   ba.BA_FLAG_NO_CTX_ROWS], ids=["auto", "fma", "rows", "fused"])
@pytest.mark.parametrize("variant", ["ragged", "dec_dom"])
def test_multi_token_all_rows(case, flags, variant):
    cfg, n = case
    inp = make_inputs(cfg, 31 + n, variant=variant, n_tok=n)
    if variant == "ragged":  # include lens < n: tokens with no decode position
        inp.lens[0] = 0
        inp.lens[-1] = min(1, cfg.md)
    out, lse = _run(inp, flags)
    assert out.shape == inp.q.shape and lse.shape == inp.q.shape[:-1]
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, f"{cfg.name}/n{n}/{variant}")


def test_multi_token_one_equals_single_token():
    cfg = Config("x", "bf16", b=16, h=8, g=8, d=128, mc=1000, md=64)
    inp = make_inputs(cfg, 3, variant="ragged")
    q3 = inp.q.to(DEV)
    o3 = ba.bifurcated_attn_decode(q3, inp.Kc.to(DEV), inp.Vc.to(DEV), inp.Kd.to(DEV),
                                   inp.Vd.to(DEV), inp.lens.to(DEV), scale=inp.scale)
    o4 = ba.bifurcated_attn_decode(q3.unsqueeze(2).contiguous(), inp.Kc.to(DEV), inp.Vc.to(DEV),
                                   inp.Kd.to(DEV), inp.Vd.to(DEV), inp.lens.to(DEV),
                                   scale=inp.scale)
    torch.cuda.synchronize()
    assert torch.equal(o4[:, :, 0], o3)


def test_multi_token_replicated_baseline():
    cfg = Config("x", "bf16", b=6, h=8, g=4, d=128, mc=300, md=40)
    n = 3
    inp = make_inputs(cfg, 10, variant="ragged", n_tok=n)
    K = torch.cat([inp.Kc.unsqueeze(0).expand(cfg.b, -1, -1, -1), inp.Kd], dim=2).contiguous()
    V = torch.cat([inp.Vc.unsqueeze(0).expand(cfg.b, -1, -1, -1), inp.Vd], dim=2).contiguous()
    lse = torch.empty(cfg.b, cfg.h, n, device=DEV)
    out = ba.replicated_attn_decode(inp.q.to(DEV), K.to(DEV), V.to(DEV), inp.lens.to(DEV),
                                    cfg.mc, lse=lse, scale=inp.scale)
    torch.cuda.synchronize()
    ref, ref_lse = oracle_rows(inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, "replicated-multi")


def test_multi_token_full_size_b32():
    """BASELINE C2b shape with n = 4 draft tokens (a speculative verification
    step) at full size: every row of all 32 samples against the oracle."""
    cfg = Config("mha7b_b32_n4", "bf16", b=32, h=32, g=32, d=128, mc=8192, md=256)
    n = 4
    inp = make_inputs(cfg, 77, device=DEV, n_tok=n)
    out, lse = _run(inp)
    ref, ref_lse = oracle_rows(type(inp)(inp.q.cpu(), inp.Kc.cpu(), inp.Vc.cpu(), inp.Kd.cpu(),
                                         inp.Vd.cpu(), inp.lens.cpu(), inp.scale))
    st = compare(out, lse, ref, ref_lse, cfg.torch_dtype, "b32-n4")
    print(f"b32-n4: all rows: {st}")
