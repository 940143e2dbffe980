"""B200-native bifurcated decode attention (arXiv 2403.08845).

Thin Python binding over the C ABI of ``libbifattn.so`` (include/bifattn.h).
It only marshals arguments: every step of the decode path runs in the CUDA
kernels of ``csrc/``.  PyTorch provides device memory and streams.  There is
no CPU fallback: if the library or an sm_100 device is missing, calls raise.

Entry points mirror the C names:
  bifurcated_attn_decode(q, Kc, Vc, Kd, Vd, lens, out=None, lse=None, ...)
  bifurcated_attn_decode_host(...)   host tensors in, host result out (e2e)
  replicated_attn_decode(q, K, V, lens, ...)   non-bifurcated baseline
  ba_workspace_bytes(...), ba_launches_per_call(...), ba_plan_string(...)
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbifattn.so")

BA_BF16, BA_FP32, BA_FP8_E4M3 = 0, 1, 2
BA_FLAG_FORCE_FMA = 0x1
BA_FLAG_NO_PDL = 0x2
BA_FLAG_CTX_ROWS = 0x4
BA_FLAG_NO_CTX_ROWS = 0x8

ERRORS = {0: "BA_OK", -1: "BA_EINVAL", -2: "BA_ENULL", -3: "BA_EALIGN", -4: "BA_EWORKSPACE",
          -5: "BA_EDTYPE", -6: "BA_ENODEV", -7: "BA_ECUDA"}

EXPORTED = ["ba_workspace_bytes", "bifurcated_attn_decode", "bifurcated_attn_decode_host",
            "bifurcated_attn_decode_append", "bifurcated_attn_decode_append_host", "ba_lse_merge",
            "replicated_attn_decode", "ba_launches_per_call", "ba_plan_string", "ba_strerror",
            "ba_last_cuda_error", "ba_version", "ba_launch_name", "ba_set_launch_events",
            "ba_set_trace_buffer", "ba_plan_ctas", "ba_stream_read_bench", "ba_step_in_bytes",
            "ba_step_out_bytes", "bifurcated_attn_decode_step_packed", "ba_select_path"]


class BAProblem(ctypes.Structure):
    _fields_ = [("b", ctypes.c_int32), ("h", ctypes.c_int32), ("g", ctypes.c_int32),
                ("d", ctypes.c_int32), ("mc", ctypes.c_int32), ("md_cap", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("scale", ctypes.c_float), ("flags", ctypes.c_uint32),
                ("n_tok", ctypes.c_int32), ("kv_dtype", ctypes.c_int32),
                ("k_scale", ctypes.c_float), ("v_scale", ctypes.c_float)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libbifattn.so (build it first with paper_2403_08845_b200._build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"libbifattn.so not found at {path}: build it (python -m paper_2403_08845_b200._build);"
            " there is no CPU fallback")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    pp = ctypes.POINTER(BAProblem)
    lib.ba_workspace_bytes.argtypes = [pp]
    lib.ba_workspace_bytes.restype = ctypes.c_size_t
    lib.bifurcated_attn_decode.argtypes = [pp] + [P] * 9 + [ctypes.c_size_t, P]
    lib.bifurcated_attn_decode.restype = ctypes.c_int
    lib.bifurcated_attn_decode_host.argtypes = [pp] + [P] * 17 + [ctypes.c_size_t, P]
    lib.bifurcated_attn_decode_host.restype = ctypes.c_int
    lib.bifurcated_attn_decode_append.argtypes = [pp] + [P] * 11 + [ctypes.c_size_t, P]
    lib.bifurcated_attn_decode_append.restype = ctypes.c_int
    lib.bifurcated_attn_decode_append_host.argtypes = [pp] + [P] * 17 + [ctypes.c_size_t, P]
    lib.bifurcated_attn_decode_append_host.restype = ctypes.c_int
    lib.ba_lse_merge.argtypes = [ctypes.c_int] * 4 + [P] * 5
    lib.ba_lse_merge.restype = ctypes.c_int
    lib.replicated_attn_decode.argtypes = [pp] + [P] * 7 + [ctypes.c_size_t, P]
    lib.replicated_attn_decode.restype = ctypes.c_int
    lib.ba_launches_per_call.argtypes = [pp]
    lib.ba_launches_per_call.restype = ctypes.c_int
    lib.ba_plan_string.argtypes = [pp]
    lib.ba_plan_string.restype = ctypes.c_char_p
    lib.ba_strerror.argtypes = [ctypes.c_int]
    lib.ba_strerror.restype = ctypes.c_char_p
    lib.ba_last_cuda_error.argtypes = []
    lib.ba_last_cuda_error.restype = ctypes.c_int
    lib.ba_launch_name.argtypes = [pp, ctypes.c_int]
    lib.ba_launch_name.restype = ctypes.c_char_p
    lib.ba_set_launch_events.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.ba_set_launch_events.restype = None
    lib.ba_plan_ctas.argtypes = [pp, ctypes.c_void_p, ctypes.c_int]
    lib.ba_plan_ctas.restype = ctypes.c_int
    lib.ba_set_trace_buffer.argtypes = [ctypes.c_void_p]
    lib.ba_set_trace_buffer.restype = None
    lib.ba_select_path.argtypes = [pp, ctypes.c_int, ctypes.c_longlong]
    lib.ba_select_path.restype = ctypes.c_int
    lib.ba_step_in_bytes.argtypes = [pp]
    lib.ba_step_in_bytes.restype = ctypes.c_size_t
    lib.ba_step_out_bytes.argtypes = [pp]
    lib.ba_step_out_bytes.restype = ctypes.c_size_t
    lib.bifurcated_attn_decode_step_packed.argtypes = [pp, P, P, P, P, ctypes.c_int] + [P] * 5 + \
        [ctypes.c_size_t, P]
    lib.bifurcated_attn_decode_step_packed.restype = ctypes.c_int
    lib.ba_stream_read_bench.argtypes = [P, ctypes.c_size_t, P, P]
    lib.ba_stream_read_bench.restype = ctypes.c_int
    lib.ba_version.argtypes = []
    lib.ba_version.restype = ctypes.c_int
    _lib = lib
    return lib


class BifAttnError(RuntimeError):
    def __init__(self, code: int, what: str):
        lib = load_library()
        msg = lib.ba_strerror(code).decode()
        extra = ""
        if code == -7:
            extra = f" (cudaError {lib.ba_last_cuda_error()})"
        super().__init__(f"{what}: {ERRORS.get(code, code)}: {msg}{extra}")
        self.code = code


FP8_DTYPES = (torch.float8_e4m3fn,)


def make_problem(b, h, g, d, mc, md_cap, dtype, scale: Optional[float] = None, flags: int = 0,
                 n_tok: int = 1, kv_dtype=None, k_scale: float = 1.0, v_scale: float = 1.0):
    """kv_dtype: None / the dtype (cache stored like q), or torch.float8_e4m3fn /
    BA_FP8_E4M3 (FP8 KV cache with per-tensor k_scale / v_scale, include/bifattn.h)."""
    dt = {torch.bfloat16: BA_BF16, torch.float32: BA_FP32}.get(dtype, dtype)
    kv = BA_FP8_E4M3 if (kv_dtype in FP8_DTYPES or kv_dtype == BA_FP8_E4M3) else 0
    return BAProblem(b, h, g, d, mc, md_cap, dt, float(scale) if scale else 0.0, flags, n_tok,
                     kv, float(k_scale) if kv else 0.0, float(v_scale) if kv else 0.0)


def _problem_from(q, Kc, Kd, scale, flags, k_scale=1.0, v_scale=1.0):
    """q [b,h,d] (one token per sample) or [b,h,n,d] (multi-token step); an FP8
    cache (Kc dtype float8_e4m3fn) carries its per-tensor scales."""
    if q.dim() == 4:
        b, h, n, d = q.shape
    else:
        (b, h, d), n = q.shape, 1
    g, mc, _ = Kc.shape
    md_cap = Kd.shape[2]
    return make_problem(b, h, g, d, mc, md_cap, q.dtype, scale, flags, n, Kc.dtype, k_scale,
                        v_scale)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream_handle(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def ba_workspace_bytes(prob: BAProblem) -> int:
    return int(load_library().ba_workspace_bytes(ctypes.byref(prob)))


def ba_launches_per_call(prob: BAProblem) -> int:
    return int(load_library().ba_launches_per_call(ctypes.byref(prob)))


def ba_plan_string(prob: BAProblem) -> str:
    return load_library().ba_plan_string(ctypes.byref(prob)).decode()


def ba_launch_names(prob: BAProblem):
    lib = load_library()
    names, k = [], 0
    while True:
        s = lib.ba_launch_name(ctypes.byref(prob), k)
        if not s:
            return names
        names.append(s.decode())
        k += 1


class LaunchTimer:
    """Per-kernel CUDA-event timing of the library's launches (instrumentation
    for bench.py): records an event pair around every launch of every call made
    while active, on the call's stream."""

    def __init__(self, launches_per_call: int, calls: int):
        self.L = launches_per_call
        self.calls = calls
        self.events = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                        for _ in range(self.L)] for _ in range(calls)]
        # torch creates the CUDA event lazily on first record(): force creation
        for call in self.events:
            for a, b in call:
                a.record()
                b.record()
        torch.cuda.synchronize()
        self._arrays = []
        for call in self.events:
            arr = (ctypes.c_void_p * (2 * self.L))()
            for k, (a, b) in enumerate(call):
                arr[2 * k] = a.cuda_event
                arr[2 * k + 1] = b.cuda_event
            self._arrays.append(arr)

    def arm(self, call: int):
        load_library().ba_set_launch_events(self._arrays[call], self.L)

    @staticmethod
    def disarm():
        load_library().ba_set_launch_events(None, 0)

    def per_launch_ms(self):
        """Mean duration (ms) of each launch index over all recorded calls."""
        tot = [0.0] * self.L
        for call in self.events:
            for k, (a, b) in enumerate(call):
                tot[k] += a.elapsed_time(b)
        return [t / self.calls for t in tot]


def ba_plan_ctas(prob: BAProblem):
    """CTA range starts of the tensor-core plan ([] for the CUDA-core plan)."""
    lib = load_library()
    buf = (ctypes.c_int32 * 512)()
    G = lib.ba_plan_ctas(ctypes.byref(prob), buf, 512)
    if G < 0:
        raise BifAttnError(G, "ba_plan_ctas")
    return [int(buf[k]) for k in range(G + 1)] if G > 0 else []


_ws_cache = {}


def _ws_need(prob: BAProblem) -> int:
    key = bytes(prob)
    n = _ws_cache.get(key)
    if n is None:
        n = ba_workspace_bytes(prob)
        if n == 0:
            raise BifAttnError(-1, "ba_workspace_bytes")
        if len(_ws_cache) > 256:
            _ws_cache.clear()
        _ws_cache[key] = n
    return n


def alloc_workspace(prob: BAProblem, device) -> torch.Tensor:
    """Zero-initialised workspace (the completion counters must start at 0)."""
    n = ba_workspace_bytes(prob)
    if n == 0:
        raise BifAttnError(-1, "ba_workspace_bytes")
    return torch.zeros(n, dtype=torch.uint8, device=device)


def _check(ts, dtype, device):
    for name, t in ts.items():
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.device != device:
            raise ValueError(f"{name} is on {t.device}, expected {device}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if name != "lens" and t.dtype != dtype:
            raise ValueError(f"{name} has dtype {t.dtype}, expected {dtype}")


_NAMES = ("q", "Kc", "Vc", "Kd", "Vd", "lens")
_prob_cache = {}


def _fast_check(ts, dtype, device):
    """Per-call argument checks (the cheap common case; _check words the error).
    The cache (ts[1:5]) is either in q's dtype or, with a bf16 q, FP8 E4M3."""
    for t in ts:
        if not (t.is_cuda and t.device == device and t.is_contiguous()):
            _check(dict(zip(_NAMES, ts)), dtype, device)
    if ts[0].dtype != dtype:
        _check(dict(zip(_NAMES, ts)), dtype, device)
    kvd = ts[1].dtype
    if kvd in FP8_DTYPES and dtype == torch.bfloat16:
        if any(t.dtype != kvd for t in ts[1:5]):
            raise ValueError("Kc, Vc, Kd, Vd must all be float8_e4m3fn")
        return
    for t in ts[1:5]:
        if t.dtype != dtype:
            _check(dict(zip(_NAMES, ts)), dtype, device)


_shape_ok = set()


def _validate_shapes(q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, ws_need):
    """Shape / dtype / device agreement of every tensor argument (cached per
    shape signature): a mismatch is a ValueError here, never an out-of-bounds
    access in a kernel."""
    key = (tuple(q.shape), tuple(Kc.shape), tuple(Vc.shape), tuple(Kd.shape), tuple(Vd.shape),
           tuple(lens.shape), tuple(out.shape), out.dtype, out.device, q.dtype, q.device,
           None if lse is None else (tuple(lse.shape), lse.dtype, lse.device),
           workspace.numel(), workspace.device)
    if key in _shape_ok:
        if not (out.is_contiguous() and (lse is None or lse.is_contiguous())
                and workspace.is_contiguous()):
            raise ValueError("out, lse and workspace must be contiguous")
        return
    if q.dim() not in (3, 4):
        raise ValueError(f"q must be [b,h,d] or [b,h,n,d], got {tuple(q.shape)}")
    b, h, d = q.shape[0], q.shape[1], q.shape[-1]
    if Kc.dim() != 3 or Kc.shape[2] != d:
        raise ValueError(f"Kc must be [g,mc,{d}], got {tuple(Kc.shape)}")
    g = Kc.shape[0]
    if tuple(Vc.shape) != tuple(Kc.shape):
        raise ValueError(f"Vc {tuple(Vc.shape)} must match Kc {tuple(Kc.shape)}")
    if Kd.dim() != 4 or Kd.shape[0] != b or Kd.shape[1] != g or Kd.shape[3] != d:
        raise ValueError(f"Kd must be [{b},{g},md_cap,{d}], got {tuple(Kd.shape)}")
    if tuple(Vd.shape) != tuple(Kd.shape):
        raise ValueError(f"Vd {tuple(Vd.shape)} must match Kd {tuple(Kd.shape)}")
    if lens.dim() != 1 or lens.shape[0] != b:
        raise ValueError(f"lens must be int32 [{b}], got {tuple(lens.shape)}")
    if tuple(out.shape) != tuple(q.shape) or out.dtype != q.dtype or out.device != q.device:
        raise ValueError(f"out must be {tuple(q.shape)} {q.dtype} on {q.device}")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    if lse is not None:
        if (tuple(lse.shape) != tuple(q.shape[:-1]) or lse.dtype != torch.float32
                or lse.device != q.device or not lse.is_contiguous()):
            raise ValueError(f"lse must be contiguous float32 {tuple(q.shape[:-1])} on {q.device}")
    if workspace.device != q.device or not workspace.is_contiguous():
        raise ValueError(f"workspace must be a contiguous buffer on {q.device}")
    if workspace.numel() * workspace.element_size() < ws_need:
        raise ValueError(f"workspace has {workspace.numel() * workspace.element_size()} bytes, "
                         f"needs {ws_need}")
    if len(_shape_ok) > 256:
        _shape_ok.clear()
    _shape_ok.add(key)


def _cached_problem(q, Kc, Kd, scale, flags, k_scale=1.0, v_scale=1.0):
    key = (q.shape, Kc.shape, Kd.shape, q.dtype, Kc.dtype, scale, flags, k_scale, v_scale)
    prob = _prob_cache.get(key)
    if prob is None:
        if len(_prob_cache) > 64:
            _prob_cache.clear()
        prob = _prob_cache[key] = _problem_from(q, Kc, Kd, scale, flags, k_scale, v_scale)
    return prob


def bifurcated_attn_decode(q, Kc, Vc, Kd, Vd, lens, out=None, lse=None, *, scale=None,
                           workspace=None, stream=None, flags=0, k_scale=1.0, v_scale=1.0):
    """One bifurcated decode step on the GPU.  Shapes: q [b,h,d]; Kc,Vc [g,mc,d];
    Kd,Vd [b,g,md_cap,d]; lens int32 [b].  Returns ``out`` [b,h,d].
    Multi-token step (n draft tokens per sample, include/bifattn.h MULTI-TOKEN):
    q [b,h,n,d], out [b,h,n,d], lse [b,h,n]; token k sees the decode positions
    t < lens[i] - (n - 1 - k).
    FP8 cache: Kc, Vc, Kd, Vd float8_e4m3fn with per-tensor k_scale / v_scale
    (cache value = code x scale; q and out bf16)."""
    lib = _lib if _lib is not None else load_library()
    _fast_check((q, Kc, Vc, Kd, Vd, lens), q.dtype, q.device)
    if lens.dtype != torch.int32:
        raise ValueError("lens must be int32")
    prob = _cached_problem(q, Kc, Kd, scale, flags, k_scale, v_scale)
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = alloc_workspace(prob, q.device)
    _validate_shapes(q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, _ws_need(prob))
    st = (stream if stream is not None else torch.cuda.current_stream()).cuda_stream
    rc = lib.bifurcated_attn_decode(ctypes.byref(prob), q.data_ptr(), Kc.data_ptr(), Vc.data_ptr(),
                                    Kd.data_ptr(), Vd.data_ptr(), lens.data_ptr(), out.data_ptr(),
                                    lse.data_ptr() if lse is not None else None,
                                    workspace.data_ptr(), workspace.numel(), st)
    if rc != 0:
        raise BifAttnError(rc, "bifurcated_attn_decode")
    return out


def bifurcated_attn_decode_append(q, k_new, v_new, Kc, Vc, Kd, Vd, lens, out=None, lse=None, *,
                                  scale=None, workspace=None, stream=None, flags=0, k_scale=1.0,
                                  v_scale=1.0):
    """KV append + bifurcated decode step in one call (include/bifattn.h):
    writes k_new/v_new [b,g,n,d] into Kd/Vd at lens[i].., attends with
    lens + n, and advances ``lens`` (device int32) in place.  q [b,h,d]
    (n = 1) or [b,h,n,d]."""
    lib = _lib if _lib is not None else load_library()
    _fast_check((q, Kc, Vc, Kd, Vd, lens), q.dtype, q.device)
    _check(dict(k_new=k_new, v_new=v_new), Kd.dtype, q.device)
    if lens.dtype != torch.int32:
        raise ValueError("lens must be int32")
    prob = _cached_problem(q, Kc, Kd, scale, flags, k_scale, v_scale)
    n = max(prob.n_tok, 1)
    exp = (Kd.shape[0], Kd.shape[1], n, Kd.shape[3])
    if tuple(k_new.shape) != exp or tuple(v_new.shape) != exp:
        raise ValueError(f"k_new/v_new must be {exp}")
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = alloc_workspace(prob, q.device)
    _validate_shapes(q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, _ws_need(prob))
    st = (stream if stream is not None else torch.cuda.current_stream()).cuda_stream
    rc = lib.bifurcated_attn_decode_append(
        ctypes.byref(prob), q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), Kc.data_ptr(),
        Vc.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), lens.data_ptr(), out.data_ptr(),
        lse.data_ptr() if lse is not None else None, workspace.data_ptr(), workspace.numel(), st)
    if rc != 0:
        raise BifAttnError(rc, "bifurcated_attn_decode_append")
    return out


def bifurcated_attn_decode_append_host(hq, hk_new, hv_new, hout, dev, *, hlens=None, hlse=None,
                                       scale=None, stream=None, flags=0, k_scale=1.0,
                                       v_scale=1.0):
    """One serving step with host tensors in and out (include/bifattn.h):
    ``dev`` holds the resident caches and staging buffers {q, k_new, v_new,
    Kc, Vc, Kd, Vd, lens, out, lse?, workspace}.  Synchronise before reading
    ``hout``."""
    lib = _lib if _lib is not None else load_library()
    prob = _cached_problem(hq, dev["Kc"], dev["Kd"], scale, flags, k_scale, v_scale)
    ws = dev["workspace"]
    rc = lib.bifurcated_attn_decode_append_host(
        ctypes.byref(prob), _ptr(hq), _ptr(hk_new), _ptr(hv_new), _ptr(hlens), _ptr(hout),
        _ptr(hlse), _ptr(dev["q"]), _ptr(dev["k_new"]), _ptr(dev["v_new"]), _ptr(dev["Kc"]),
        _ptr(dev["Vc"]), _ptr(dev["Kd"]), _ptr(dev["Vd"]), _ptr(dev["lens"]), _ptr(dev["out"]),
        _ptr(dev.get("lse")), _ptr(ws), ws.numel(), _stream_handle(stream))
    if rc != 0:
        raise BifAttnError(rc, "bifurcated_attn_decode_append_host")
    return hout


def lse_merge(out_parts, lse_parts, out=None, lse=None, *, stream=None):
    """Join partial results over disjoint key slices (include/bifattn.h
    ba_lse_merge): out_parts [n, ...rows..., d], lse_parts [n, ...rows...]."""
    lib = _lib if _lib is not None else load_library()
    n, d = out_parts.shape[0], out_parts.shape[-1]
    rows = out_parts[0].numel() // d
    _check(dict(out_parts=out_parts), out_parts.dtype, out_parts.device)
    if lse_parts.dtype != torch.float32 or not lse_parts.is_contiguous() or \
            lse_parts.numel() != n * rows:
        raise ValueError("lse_parts must be contiguous float32 [n, rows]")
    if out is None:
        out = torch.empty(out_parts.shape[1:], dtype=out_parts.dtype, device=out_parts.device)
    dt = {torch.bfloat16: BA_BF16, torch.float32: BA_FP32}[out_parts.dtype]
    rc = lib.ba_lse_merge(n, rows, d, dt, out_parts.data_ptr(), lse_parts.data_ptr(),
                          out.data_ptr(), lse.data_ptr() if lse is not None else None,
                          _stream_handle(stream))
    if rc != 0:
        raise BifAttnError(rc, "ba_lse_merge")
    return out


def bifurcated_attn_decode_host(hq, hKc, hVc, hKd, hVd, hlens, hout, dev, *, hlse=None,
                                scale=None, stream=None, flags=0, k_scale=1.0, v_scale=1.0):
    """End-to-end call: host (pinned) tensors in, host result out.  ``dev`` is a
    dict of caller-owned device buffers {q,Kc,Vc,Kd,Vd,lens,out,lse,workspace}
    (see make_device_buffers).  Enqueues H2D copies, the kernels and the D2H
    copy on ``stream``; synchronise before reading ``hout``."""
    lib = load_library()
    prob = _problem_from(hq, hKc, hKd, scale, flags, k_scale, v_scale)
    for name, h in (("q", hq), ("Kc", hKc), ("Vc", hVc), ("Kd", hKd), ("Vd", hVd),
                    ("lens", hlens), ("out", hout)):
        dv = dev[name]
        if dv.numel() * dv.element_size() < h.numel() * h.element_size():
            raise ValueError(f"device buffer {name} is smaller than its host tensor")
    ws = dev["workspace"]
    rc = lib.bifurcated_attn_decode_host(
        ctypes.byref(prob), _ptr(hq), _ptr(hKc), _ptr(hVc), _ptr(hKd), _ptr(hVd), _ptr(hlens),
        _ptr(hout), _ptr(hlse), _ptr(dev["q"]), _ptr(dev["Kc"]), _ptr(dev["Vc"]), _ptr(dev["Kd"]),
        _ptr(dev["Vd"]), _ptr(dev["lens"]), _ptr(dev["out"]), _ptr(dev.get("lse")), _ptr(ws),
        ws.numel(), _stream_handle(stream))
    if rc != 0:
        raise BifAttnError(rc, "bifurcated_attn_decode_host")
    return hout


def make_device_buffers(hq, hKc, hKd, device, with_lse=False, scale=None, flags=0):
    prob = _problem_from(hq, hKc, hKd, scale, flags)
    e = dict(q=torch.empty(hq.shape, dtype=hq.dtype, device=device),
             Kc=torch.empty(hKc.shape, dtype=hKc.dtype, device=device),
             Vc=torch.empty(hKc.shape, dtype=hKc.dtype, device=device),
             Kd=torch.empty(hKd.shape, dtype=hKd.dtype, device=device),
             Vd=torch.empty(hKd.shape, dtype=hKd.dtype, device=device),
             lens=torch.empty(hq.shape[0], dtype=torch.int32, device=device),
             out=torch.empty(hq.shape, dtype=hq.dtype, device=device),
             workspace=alloc_workspace(prob, device))
    if with_lse:
        e["lse"] = torch.empty(hq.shape[:-1], dtype=torch.float32, device=device)
    return e


def replicated_attn_decode(q, K, V, lens, mc, out=None, lse=None, *, scale=None,
                           workspace=None, stream=None, flags=0, k_scale=1.0, v_scale=1.0):
    """Non-bifurcated baseline over the replicated cache K, V [b,g,mc+md_cap,d]:
    sample i attends to positions [0, mc + lens[i])."""
    lib = load_library()
    _check(dict(q=q), q.dtype, q.device)
    _check(dict(K=K, V=V), K.dtype if K.dtype in FP8_DTYPES else q.dtype, q.device)
    _check(dict(lens=lens), q.dtype, q.device)
    if q.dim() == 4:
        b, h, n, d = q.shape
    else:
        (b, h, d), n = q.shape, 1
    if K.dim() != 4 or K.shape[0] != b or K.shape[3] != d or tuple(V.shape) != tuple(K.shape):
        raise ValueError(f"K, V must be [{b},g,mc+md_cap,{d}], got {tuple(K.shape)}, {tuple(V.shape)}")
    g, M = K.shape[1], K.shape[2]
    if not 1 <= mc <= M:
        raise ValueError(f"mc ({mc}) must be in [1, {M}]")
    prob = make_problem(b, h, g, d, mc, M - mc, q.dtype, scale, flags, n, K.dtype, k_scale,
                        v_scale)
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = alloc_workspace(prob, q.device)
    # the replicated cache [b,g,M,d] stands in for both Kd-shaped operands
    Kc_like = K[0, :, :mc]
    Kd_like = K[:, :, mc:]
    _validate_shapes(q, Kc_like, Kc_like, Kd_like, Kd_like, lens, out, lse, workspace,
                     _ws_need(prob))
    rc = lib.replicated_attn_decode(ctypes.byref(prob), _ptr(q), _ptr(K), _ptr(V), _ptr(lens),
                                    _ptr(out), _ptr(lse), _ptr(workspace), workspace.numel(),
                                    _stream_handle(stream))
    if rc != 0:
        raise BifAttnError(rc, "replicated_attn_decode")
    return out


def stream_read_bench(buf: torch.Tensor, sink: torch.Tensor, stream=None) -> None:
    """One launch of the read-only streaming micro-benchmark kernel over
    ``buf`` (instrumentation for bench.py; include/bifattn.h)."""
    lib = _lib if _lib is not None else load_library()
    if not (buf.is_cuda and buf.is_contiguous() and sink.is_cuda and sink.dtype == torch.int32):
        raise ValueError("buf: contiguous CUDA tensor; sink: CUDA int32")
    rc = lib.ba_stream_read_bench(buf.data_ptr(), buf.numel() * buf.element_size(),
                                  sink.data_ptr(), _stream_handle(stream))
    if rc != 0:
        raise BifAttnError(rc, "ba_stream_read_bench")


def _up256(x: int) -> int:
    return (x + 255) & ~255


class PackedStep:
    """One serving step with one H2D and one D2H copy (include/bifattn.h
    bifurcated_attn_decode_step_packed).  Holds the pinned host buffers and
    device staging buffers of the packed layout [q | k_new | v_new | lens] ->
    [out | lse]; ``pack`` fills the host input, ``run`` enqueues the step,
    ``unpack`` views the host result.  The caches (Kc, Vc, Kd, Vd) stay
    resident; lens is this step's cache length before the append."""

    def __init__(self, prob: BAProblem, Kc, Vc, Kd, Vd, device, with_lse=False):
        lib = load_library()
        self.prob, self.lib = prob, lib
        self.Kc, self.Vc, self.Kd, self.Vd = Kc, Vc, Kd, Vd
        self.with_lse = with_lse
        nin = int(lib.ba_step_in_bytes(ctypes.byref(prob)))
        nout = int(lib.ba_step_out_bytes(ctypes.byref(prob)))
        if nin == 0 or nout == 0:
            raise BifAttnError(-1, "ba_step_in_bytes")
        self.h_in = torch.empty(nin, dtype=torch.uint8).pin_memory()
        self.h_out = torch.empty(nout, dtype=torch.uint8).pin_memory()
        self.d_in = torch.empty(nin, dtype=torch.uint8, device=device)
        self.d_out = torch.empty(nout, dtype=torch.uint8, device=device)
        self.ws = alloc_workspace(prob, device)
        n = max(prob.n_tok, 1)
        e = 2 if prob.dtype == BA_BF16 else 4
        ekv = 1 if prob.kv_dtype == BA_FP8_E4M3 else e
        b, h, g, d = prob.b, prob.h, prob.g, prob.d
        self.nq = b * h * n * d * e
        self.nkv = b * g * n * d * ekv
        self.off_k = _up256(self.nq)
        self.off_v = self.off_k + _up256(self.nkv)
        self.off_lens = self.off_v + _up256(self.nkv)
        self.off_lse = _up256(self.nq)
        self.q_shape = (b, h, n, d) if n > 1 else (b, h, d)
        self.q_dtype = torch.bfloat16 if prob.dtype == BA_BF16 else torch.float32

    def pack(self, q, k_new, v_new, lens):
        hb = self.h_in
        hb[:self.nq].copy_(q.contiguous().view(torch.uint8).reshape(-1))
        hb[self.off_k:self.off_k + self.nkv].copy_(k_new.contiguous().view(torch.uint8).reshape(-1))
        hb[self.off_v:self.off_v + self.nkv].copy_(v_new.contiguous().view(torch.uint8).reshape(-1))
        lb = torch.as_tensor(lens, dtype=torch.int32).contiguous().view(torch.uint8).reshape(-1)
        hb[self.off_lens:self.off_lens + lb.numel()].copy_(lb)

    def run(self, stream=None):
        rc = self.lib.bifurcated_attn_decode_step_packed(
            ctypes.byref(self.prob), self.h_in.data_ptr(), self.h_out.data_ptr(),
            self.d_in.data_ptr(), self.d_out.data_ptr(), 1 if self.with_lse else 0,
            self.Kc.data_ptr(), self.Vc.data_ptr(), self.Kd.data_ptr(), self.Vd.data_ptr(),
            self.ws.data_ptr(), self.ws.numel(), _stream_handle(stream))
        if rc != 0:
            raise BifAttnError(rc, "bifurcated_attn_decode_step_packed")

    def out(self):
        return self.h_out[:self.nq].view(self.q_dtype).view(self.q_shape)

    def lse(self):
        nl = self.nq // (self.q_shape[-1] * (2 if self.q_dtype == torch.bfloat16 else 4))
        return self.h_out[self.off_lse:self.off_lse + 4 * nl].view(torch.float32)


BA_PATH_AUTO, BA_PATH_BIFURCATED, BA_PATH_NAIVE = 0, 1, 2
_POLICIES = {"auto": BA_PATH_AUTO, "always_bifurcated": BA_PATH_BIFURCATED,
             "always_naive": BA_PATH_NAIVE}


def select_path(prob: BAProblem, policy="auto", threshold: int = 0) -> str:
    """FAQ 4 workload switch (include/bifattn.h ba_select_path): 'bifurcated'
    or 'naive' for this problem; policy 'auto' | 'always_bifurcated' |
    'always_naive'; threshold on b*mc (0: the library's measured default)."""
    rc = load_library().ba_select_path(ctypes.byref(prob), _POLICIES[policy], int(threshold))
    if rc < 0:
        raise BifAttnError(rc, "ba_select_path")
    return "bifurcated" if rc == BA_PATH_BIFURCATED else "naive"
