"""Why P enters the PV MMA as two bf16 parts (reading R13) or as one f16 part
(reading R20) but never as one bf16 part: a CPU simulation of the kernels'
value-product rounding against the fp64 oracle under the R12 criterion.

P = 2^(x - m) per key, with the stale running max up to 2^8 below the true
max (reading R15), is rounded to the MMA operand type; O = sum P_q V in fp32,
l = sum P (fp32, unrounded, as the kernels accumulate it); out = O / l rounded
to bf16.  On the stress sets a single bf16 P exceeds the R12 bound, a single
f16 P or the bf16 pair stays well inside it."""
import numpy as np
import pytest
import torch

import oracle
from synth import Config, make_inputs


def _sim(inp, mode):
    q = inp.q.float()
    b, h, d = q.shape
    g = inp.Kc.shape[0]
    p = h // g
    outs = []
    for i in range(b):
        L = int(inp.lens[i])
        K = torch.cat([inp.Kc.float(), inp.Kd[i, :, :L].float()], 1).repeat_interleave(p, 0)
        V = torch.cat([inp.Vc.float(), inp.Vd[i, :, :L].float()], 1).repeat_interleave(p, 0)
        s = (q[i].unsqueeze(1) @ K.transpose(1, 2))[:, 0] * inp.scale * 1.4426950408889634
        m = s.max(-1, keepdim=True).values - 7.9  # stale reference, P up to 2^7.9
        P = torch.exp2(s - m)
        if mode == "bf16":
            Pq = P.to(torch.bfloat16).float()
        elif mode == "f16":
            Pq = P.half().float()
        else:  # bf16 pair: hi = trunc(P), lo = trunc(P - hi)
            hi = (P.view(torch.int32) & ~0xFFFF).view(torch.float32)
            lo = ((P - hi).view(torch.int32) & ~0xFFFF).view(torch.float32)
            Pq = hi + lo
        o = (Pq.unsqueeze(1) @ V)[:, 0] / P.sum(-1, keepdim=True)
        outs.append(o.to(torch.bfloat16))
    return torch.stack(outs).double().numpy().reshape(b * h, d)


def _worst_ratio(inp, mode):
    ref, _, _ = oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                   scale=inp.scale, nthreads=8)
    err = np.abs(_sim(inp, mode) - ref)
    return float((err / np.maximum(2e-3, 1e-2 * np.abs(ref))).max())


@pytest.mark.parametrize("variant", ["peaky", "ctx_dom", "dec_dom"])
def test_single_bf16_p_fails_r12_but_f16_and_the_pair_pass(variant):
    cfg = Config("mqa", "bf16", b=6, h=48, g=1, d=128, mc=1000, md=100)
    inp = make_inputs(cfg, 3, variant=variant)
    assert _worst_ratio(inp, "bf16") > 1.0
    assert _worst_ratio(inp, "f16") < 0.6
    assert _worst_ratio(inp, "pair") < 0.6
