"""GPU parity of the MQA / G > g splits on one device:
the ranks of a G-way context split are run one after another through the C
ABI on their slices (rank 0 with the decode part), their (out, lse) stacked
as the all-gather would deliver them, and joined by the ba_lse_merge kernel;
the batch split runs each rank's samples with the whole context.  Both are
compared with the fp64 oracle of the unsplit problem."""
import pytest
import torch

import paper_2403_08845_b200 as ba
from paper_2403_08845_b200.dist import shard_batch_inputs, split_context_inputs
from synth import CONFIGS, Config, make_inputs, seed_for
from tests.parity import compare, oracle_rows, sample_rows

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _context_split(inp, world):
    outs, lses = [], []
    for r in range(world):
        Kc_r, Vc_r, Kd_r, Vd_r, l_r = split_context_inputs(inp.Kc, inp.Vc, inp.Kd, inp.Vd,
                                                           inp.lens, world, r)
        lse = torch.empty(inp.q.shape[:-1], dtype=torch.float32, device=DEV)
        outs.append(ba.bifurcated_attn_decode(inp.q, Kc_r, Vc_r, Kd_r, Vd_r, l_r, lse=lse,
                                              scale=inp.scale))
        lses.append(lse)
    lse = torch.empty_like(lses[0])
    out = ba.lse_merge(torch.stack(outs), torch.stack(lses), lse=lse)
    torch.cuda.synchronize()
    return out, lse


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("cfg", [Config("mqa_s", "bf16", b=6, h=48, g=1, d=128, mc=900, md=40),
                                 Config("mqa_f32", "fp32", b=3, h=4, g=1, d=64, mc=130, md=9)],
                         ids=lambda c: c.name)
def test_context_split_lse_merge(cfg, world):
    host = make_inputs(cfg, 51, variant="ragged")
    inp = type(host)(*(t.to(DEV) for t in (host.q, host.Kc, host.Vc, host.Kd, host.Vd,
                                            host.lens)), host.scale)
    out, lse = _context_split(inp, world)
    ref, ref_lse = oracle_rows(host)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, f"ctx-split{world}")


def test_lse_merge_empty_part():
    """A part with lse = -inf (no keys) drops out."""
    rows, d = 10, 128
    a = torch.randn(2, rows, d, device=DEV)
    l = torch.randn(2, rows, device=DEV)
    l[1] = float("-inf")
    out = ba.lse_merge(a, l)
    torch.cuda.synchronize()
    assert torch.allclose(out, a[0], atol=1e-6)


@pytest.mark.parametrize("world", [2, 4])
def test_batch_split_mqa_full_size(world):
    """C4 (MQA) batch split at full size: each rank's samples with the whole
    context; sampled rows against the oracle."""
    cfg = CONFIGS["mqa"]
    inp = make_inputs(cfg, seed_for("mqa"), device=DEV)
    parts = []
    for r in range(world):
        ql, Kdl, Vdl, ll = shard_batch_inputs(inp.q, inp.Kd, inp.Vd, inp.lens, world, r)
        parts.append(ba.bifurcated_attn_decode(ql, inp.Kc, inp.Vc, Kdl, Vdl, ll, scale=inp.scale))
    out = torch.cat(parts)
    torch.cuda.synchronize()
    rows = sample_rows(cfg.b, cfg.h, n=32)
    ref, _ = oracle_rows(inp, rows)
    compare(out.reshape(-1, cfg.d)[rows], None, ref, None, cfg.torch_dtype, "batch-split")


def test_context_split_mqa_full_size():
    cfg = CONFIGS["mqa"]
    inp = make_inputs(cfg, seed_for("mqa"), device=DEV)
    out, lse = _context_split(inp, 4)
    rows = sample_rows(cfg.b, cfg.h, n=32)
    ref, ref_lse = oracle_rows(inp, rows)
    compare(out.reshape(-1, cfg.d)[rows], lse.reshape(-1)[rows], ref, ref_lse,
            cfg.torch_dtype, "ctx-split-full")
