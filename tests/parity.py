"""Parity helpers shared by the GPU tests: run the oracle on (sampled) rows of
a problem and compare element by element with the stated tolerance.

Tolerance (BASELINE.json north_star; reading R12): an element passes
if |gpu - ref| <= max(ABS, REL * |ref|) with ABS = 2e-3, REL = 1e-2 for bf16
inputs (fp32 accumulation) and ABS = REL = 1e-5 for fp32 inputs.  lse: 1e-3
absolute (bf16), 1e-5 (fp32).
"""
from __future__ import annotations

import os

import numpy as np
import torch

import oracle

TOL = {torch.bfloat16: (2e-3, 1e-2, 1e-3), torch.float32: (1e-5, 1e-5, 1e-5)}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_rows(inp, rows=None):
    """fp64 oracle on the given flat rows (i*h + j) of ``inp`` (tensors may be on
    the GPU: only the slices a row needs are copied to the host)."""
    if inp.q.dim() == 4:  # multi-token step: all rows, on the host
        assert rows is None
        out, lse, _ = oracle.attn_decode(inp.q.cpu(), inp.Kc.cpu(), inp.Vc.cpu(), inp.Kd.cpu(),
                                         inp.Vd.cpu(), inp.lens.cpu(), scale=inp.scale,
                                         nthreads=host_cores())
        return out, lse
    b, h, d = inp.q.shape
    g = inp.Kc.shape[0]
    p = h // g
    if rows is None and not inp.q.is_cuda:
        out, lse, _ = oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                         scale=inp.scale, nthreads=host_cores())
        return out, lse
    if rows is None:
        rows = list(range(b * h))
    outs, lses = [], []
    lens = inp.lens.cpu()
    for r in rows:
        i, j = divmod(int(r), h)
        c = j // p
        q1 = inp.q[i:i + 1, j:j + 1].cpu()
        Kc1 = inp.Kc[c:c + 1].cpu()
        Vc1 = inp.Vc[c:c + 1].cpu()
        Kd1 = inp.Kd[i:i + 1, c:c + 1].cpu()
        Vd1 = inp.Vd[i:i + 1, c:c + 1].cpu()
        o, l, _ = oracle.attn_decode(q1, Kc1, Vc1, Kd1, Vd1, lens[i:i + 1], scale=inp.scale,
                                     nthreads=1)
        outs.append(o[0])
        lses.append(l[0])
    return np.stack(outs), np.array(lses)


def compare(gpu_out, gpu_lse, ref_out, ref_lse, dtype, what=""):
    """Assert parity; returns (max_abs_err, max_rel_err over |ref| >= 0.2)."""
    abs_tol, rel_tol, lse_tol = TOL[dtype]
    g = gpu_out.double().cpu().numpy().reshape(ref_out.shape)
    err = np.abs(g - ref_out)
    bound = np.maximum(abs_tol, rel_tol * np.abs(ref_out))
    bad = err > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(
            f"{what}: {int(bad.sum())} elements out of tolerance; first {idx.tolist()}: "
            f"gpu={g[tuple(idx[0])]:.6g} ref={ref_out[tuple(idx[0])]:.6g} "
            f"max_abs={err.max():.3g}")
    assert np.all(np.isfinite(g)), f"{what}: non-finite output"
    if gpu_lse is not None and ref_lse is not None:
        gl = gpu_lse.double().cpu().numpy().reshape(ref_lse.shape)
        lerr = np.abs(gl - ref_lse)
        assert lerr.max() <= lse_tol, f"{what}: lse max err {lerr.max():.3g}"
    big = np.abs(ref_out) >= 0.2
    max_rel = float((err[big] / np.abs(ref_out[big])).max()) if big.any() else 0.0
    return float(err.max()), max_rel


def sample_rows(b, h, n=64, seed=0):
    """Deterministic row sample incl. the first and last rows."""
    rng = np.random.default_rng(seed)
    rows = set([0, b * h - 1, h - 1, (b - 1) * h])
    rows.update(int(x) for x in rng.integers(0, b * h, size=n))
    return sorted(rows)
