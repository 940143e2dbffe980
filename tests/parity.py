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


class ParityStats(tuple):
    """(max_abs, max_rel over |ref| >= 0.2, strict_and): the R12 element
    criterion passed; ``strict_and`` additionally reports the literal reading
    of the north star (max abs <= ABS AND max rel <= REL over |ref| >= 0.2)."""

    def __new__(cls, max_abs, max_rel, strict_and, n):
        t = super().__new__(cls, (max_abs, max_rel, strict_and))
        t.max_abs, t.max_rel, t.strict_and, t.n = max_abs, max_rel, strict_and, n
        return t

    def __str__(self):
        return (f"max_abs={self.max_abs:.3g} max_rel(|ref|>=0.2)={self.max_rel:.3g} "
                f"strict_and={'pass' if self.strict_and else 'FAIL'} elems={self.n}")


def compare(gpu_out, gpu_lse, ref_out, ref_lse, dtype, what=""):
    """Assert parity (R12 element criterion); returns ParityStats."""
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
    max_abs = float(err.max()) if err.size else 0.0
    return ParityStats(max_abs, max_rel, max_abs <= abs_tol and max_rel <= rel_tol, int(err.size))


def oracle_all_rows(inp):
    """Every row of ``inp`` (single- or multi-token) through the fp64 oracle on
    all host cores: the inputs are copied to the host once."""
    import oracle as _o

    out, lse, _ = _o.attn_decode(inp.q.cpu(), inp.Kc.cpu(), inp.Vc.cpu(), inp.Kd.cpu(),
                                 inp.Vd.cpu(), inp.lens.cpu(), scale=inp.scale,
                                 nthreads=host_cores())
    return out, lse


def oracle_rows_parallel(inp, rows):
    """The oracle on the flat rows ``rows`` (i*h + j) of a single-token problem
    whose tensors may be too large to copy whole: Kc/Vc are copied once, each
    sample's Kd[i]/Vd[i] slice when needed; samples run on a thread pool (the
    ctypes call releases the GIL).  Returns (out [len(rows)][d], lse)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle as _o

    b, h, d = inp.q.shape
    Kc, Vc = inp.Kc.cpu(), inp.Vc.cpu()
    lens = inp.lens.cpu()
    by_sample = {}
    for k, r in enumerate(rows):
        i, j = divmod(int(r), h)
        by_sample.setdefault(i, []).append((k, j))

    def one(i):
        q1 = inp.q[i:i + 1].cpu()
        Kd1, Vd1 = inp.Kd[i:i + 1].cpu(), inp.Vd[i:i + 1].cpu()
        js = [j for _, j in by_sample[i]]
        o, l, _ = _o.attn_decode(q1, Kc, Vc, Kd1, Vd1, lens[i:i + 1], scale=inp.scale,
                                 rows=js, nthreads=1)
        return i, o, l

    out = np.zeros((len(rows), d))
    lse = np.zeros(len(rows))
    with ThreadPoolExecutor(max_workers=host_cores()) as ex:
        for i, o, l in ex.map(one, sorted(by_sample)):
            for n, (k, _) in enumerate(by_sample[i]):
                out[k] = o[n]
                lse[k] = l[n]
    return out, lse


def sample_rows(b, h, n=64, seed=0):
    """Deterministic row sample incl. the first and last rows."""
    rng = np.random.default_rng(seed)
    rows = set([0, b * h - 1, h - 1, (b - 1) * h])
    rows.update(int(x) for x in rng.integers(0, b * h, size=n))
    return sorted(rows)


def oracle_kv8_all_rows(inp, rows=None):
    """Every row (or ``rows``) of an FP8-KV problem (synth kv="e4m3") through
    the FP8 oracle (oracle_attn_decode_kv8_f64) on all host cores."""
    import oracle as _o

    out, lse, _ = _o.attn_decode_kv8(inp.q.cpu(), inp.Kc.cpu(), inp.Vc.cpu(), inp.Kd.cpu(),
                                     inp.Vd.cpu(), inp.lens.cpu(), scale=inp.scale,
                                     k_scale=inp.k_scale, v_scale=inp.v_scale, rows=rows,
                                     nthreads=host_cores())
    return out, lse
