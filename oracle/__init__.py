"""fp64 CPU oracle for one bifurcated-attention decode step (arXiv 2403.08845).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2403_08845_b200`` never imports it and
shares no code with it (see the header of ``oracle/oracle.c``).

``oracle.c`` holds the arithmetic: the plain definition of generalized
multi-query attention, Eq. 1-2, over the context KV
replicated into each sample's cache, and the paper's bifurcated algorithm,
Eq. 3-4, for the App. E.1 exactness invariant.  This module
only marshals arguments (ctypes) and builds the library with gcc.

Parity status: pinned (tests/test_oracle_pins.py) — no function here is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OR_BF16, OR_FP32 = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, OpenMP over rows, no CUDA)."""
    import hashlib

    cmd = ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", _LIB, _SRC, "-lm"]
    with open(_SRC, "rb") as f:
        digest = hashlib.sha256(f.read() + " ".join(cmd).encode()).hexdigest()
    stamp = _LIB + ".srchash"
    fresh = os.path.exists(_LIB) and os.path.exists(stamp) and open(stamp).read().strip() == digest
    if force or not fresh:
        subprocess.check_call(cmd)
        with open(stamp, "w") as f:
            f.write(digest + "\n")
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int
        args = [I, I, I, I, I, I, I, ctypes.c_double, P, P, P, P, P, P, P, I, P, P, P, I]
        lib.oracle_attn_decode_f64.argtypes = args
        lib.oracle_attn_decode_f64.restype = I
        lib.oracle_bifurcated_f64.argtypes = args
        lib.oracle_bifurcated_f64.restype = I
        lib.oracle_attn_decode_multi_f64.argtypes = [I] + args
        lib.oracle_attn_decode_multi_f64.restype = I
        lib.oracle_attn_decode_kv8_f64.argtypes = [I] * 7 + [ctypes.c_double] * 3 + \
            [P] * 7 + [I, P, P, P, I]
        lib.oracle_attn_decode_kv8_f64.restype = I
        lib.oracle_e4m3_value.argtypes = [I]
        lib.oracle_e4m3_value.restype = ctypes.c_double
        lib.oracle_kv_read_elements.argtypes = [ctypes.c_int64] * 5 + [I]
        lib.oracle_kv_read_elements.restype = ctypes.c_int64
        _lib = lib
    return _lib


def _as_np(x):
    """Accept numpy arrays or CPU torch tensors; bf16 becomes its uint16 bits."""
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x)
    import torch  # local import: the oracle itself does not need torch

    x = x.detach().contiguous()
    if x.is_cuda:
        x = x.cpu()
    if x.dtype == torch.bfloat16:
        return x.view(torch.int16).numpy().view(np.uint16)
    if x.dtype == torch.float32:
        return x.numpy()
    if x.dtype == torch.int32:
        return x.numpy()
    raise TypeError(f"oracle: unsupported dtype {x.dtype}")


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def attn_decode(q, Kc, Vc, Kd, Vd, lens, *, scale, rows=None, weights=False,
                nthreads=1, bifurcated=False):
    """Run the oracle.

    Shapes (row-major): q [b][h][d]; Kc, Vc [g][mc][d]; Kd, Vd [b][g][md_cap][d];
    lens int32 [b].  dtype: bf16 (as uint16 bits / torch.bfloat16) or fp32.
    ``scale`` is the logit scale (pass the exact fp32 value the GPU uses).
    ``rows``: optional list of flat row indices i*h + j to compute.
    A 4-D q [b][h][n][d] is the multi-token step (oracle_attn_decode_multi_f64,
    App. G): rows are (i*h + j)*n + k; ``bifurcated`` is not available there.
    Returns (out [nrows][d] f64, lse [nrows] f64, weights [nrows][mc+md_cap] or None).
    """
    qn, Kcn, Vcn, Kdn, Vdn = (_as_np(t) for t in (q, Kc, Vc, Kd, Vd))
    lensn = np.ascontiguousarray(_as_np(lens).astype(np.int32))
    n = 1
    if qn.ndim == 4:
        b, h, n, d = qn.shape
        assert not bifurcated, "the multi-token oracle is the plain definition only"
    else:
        b, h, d = qn.shape
    g, mc, d2 = Kcn.shape
    md_cap = Kdn.shape[2]
    assert d2 == d and Kdn.shape[:2] == (b, g) and Kdn.shape[3] == d
    assert Vcn.shape == Kcn.shape and Vdn.shape == Kdn.shape
    if qn.dtype == np.uint16:
        dtype = OR_BF16
    elif qn.dtype == np.float32:
        dtype = OR_FP32
    else:
        raise TypeError(qn.dtype)
    for t in (Kcn, Vcn, Kdn, Vdn):
        assert t.dtype == qn.dtype
    if rows is None:
        rows_np = None
        nrows = b * h * n
    else:
        rows_np = np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
        nrows = int(rows_np.size)
    out = np.zeros((nrows, d), dtype=np.float64)
    lse = np.zeros((nrows,), dtype=np.float64)
    w = np.zeros((nrows, mc + md_cap), dtype=np.float64) if weights else None
    tail = (float(scale), _ptr(qn), _ptr(Kcn), _ptr(Vcn), _ptr(Kdn), _ptr(Vdn), _ptr(lensn),
            _ptr(rows_np), nrows, _ptr(out), _ptr(lse), _ptr(w), int(nthreads))
    if qn.ndim == 4:
        rc = _load().oracle_attn_decode_multi_f64(b, h, n, g, d, mc, md_cap, dtype, *tail)
    else:
        fn = _load().oracle_bifurcated_f64 if bifurcated else _load().oracle_attn_decode_f64
        rc = fn(b, h, g, d, mc, md_cap, dtype, *tail)
    if rc != 0:
        raise ValueError("oracle: invalid problem")
    return out, lse, w


def e4m3_value(code: int) -> float:
    """The value of one OCP FP8 E4M3 code (reading R19)."""
    return float(_load().oracle_e4m3_value(int(code)))


def attn_decode_kv8(q, Kc, Vc, Kd, Vd, lens, *, scale, k_scale, v_scale, rows=None,
                    weights=False, nthreads=1):
    """The fp64 oracle with an FP8 E4M3 KV cache (oracle_attn_decode_kv8_f64):
    Kc, Vc [g][mc][d] and Kd, Vd [b][g][md_cap][d] are E4M3 codes (uint8 numpy
    arrays or torch.float8_e4m3fn / uint8 tensors), dequantised as code value x
    k_scale (K) or x v_scale (V); q [b][h][d] bf16 or fp32.  Returns (out, lse,
    weights) like attn_decode."""
    def codes(t):
        if isinstance(t, np.ndarray):
            return np.ascontiguousarray(t.astype(np.uint8, copy=False))
        t = t.detach().contiguous().cpu()
        return t.view(__import__("torch").uint8).numpy()

    qn = _as_np(q)
    Kcn, Vcn, Kdn, Vdn = (codes(t) for t in (Kc, Vc, Kd, Vd))
    lensn = np.ascontiguousarray(_as_np(lens).astype(np.int32))
    b, h, d = qn.shape
    g, mc, _ = Kcn.shape
    md_cap = Kdn.shape[2]
    assert Kcn.shape == Vcn.shape and Kdn.shape == Vdn.shape and Kdn.shape[:2] == (b, g)
    dtype = OR_BF16 if qn.dtype == np.uint16 else OR_FP32
    rows_np = None if rows is None else np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
    nrows = b * h if rows is None else int(rows_np.size)
    out = np.zeros((nrows, d))
    lse = np.zeros(nrows)
    w = np.zeros((nrows, mc + md_cap)) if weights else None
    rc = _load().oracle_attn_decode_kv8_f64(
        b, h, g, d, mc, md_cap, dtype, float(scale), float(k_scale), float(v_scale), _ptr(qn),
        _ptr(Kcn), _ptr(Vcn), _ptr(Kdn), _ptr(Vdn), _ptr(lensn), _ptr(rows_np), nrows,
        _ptr(out), _ptr(lse), _ptr(w), int(nthreads))
    if rc != 0:
        raise ValueError("oracle: invalid problem")
    return out, lse, w


def kv_read_elements(b, g, k, mc, md, bifurcated):
    """Eq. 5-6: KV elements read per K or V tensor."""
    return int(_load().oracle_kv_read_elements(b, g, k, mc, md, 1 if bifurcated else 0))
