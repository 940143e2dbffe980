"""C-ABI boundary checks that need no GPU: the library builds and loads, exports
every entry point include/bifattn.h declares, and rejects bad problems on the
host before touching a device."""
import ctypes
import os
import re

import pytest

import paper_2403_08845_b200 as ba
from paper_2403_08845_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bifattn.h")


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return ba.load_library()


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "return")))


def test_header_declares_the_north_star_entry_point():
    names = _declared_functions()
    assert "bifurcated_attn_decode" in names
    assert set(ba.EXPORTED) == set(names)


def test_library_exports_every_declared_symbol(lib):
    for name in _declared_functions():
        assert hasattr(lib, name), f"missing export {name}"


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {ba.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_and_strerror(lib):
    assert lib.ba_version() == 3
    assert b"CPU fallback" in lib.ba_strerror(-6)
    for code in range(0, -8, -1):
        assert lib.ba_strerror(code) != b"unknown error"


def _prob(**kw):
    base = dict(b=4, h=8, g=2, d=128, mc=100, md_cap=10, dtype=ba.BA_BF16, scale=0.0, flags=0)
    base.update(kw)
    return ba.BAProblem(**base)


@pytest.mark.parametrize("bad", [dict(h=6, g=4), dict(b=0), dict(mc=0), dict(md_cap=-1),
                                 dict(d=48), dict(d=512), dict(g=0)])
def test_invalid_problems_rejected_on_host(lib, bad):
    p = _prob(**bad)
    assert lib.ba_workspace_bytes(ctypes.byref(p)) == 0
    rc = lib.bifurcated_attn_decode(ctypes.byref(p), *([ctypes.c_void_p(16)] * 9), 1 << 20, None)
    assert rc == -1


def test_bad_dtype_rejected(lib):
    p = _prob(dtype=7)
    rc = lib.bifurcated_attn_decode(ctypes.byref(p), *([ctypes.c_void_p(16)] * 9), 1 << 20, None)
    assert rc == -5


def test_null_problem_rejected(lib):
    rc = lib.bifurcated_attn_decode(None, *([ctypes.c_void_p(16)] * 9), 1 << 20, None)
    assert rc == -2


def test_workspace_size_positive_and_monotone(lib):
    a = lib.ba_workspace_bytes(ctypes.byref(_prob()))
    b = lib.ba_workspace_bytes(ctypes.byref(_prob(b=8)))
    assert a > 0 and b > a
    assert a % 16 == 0


def test_no_gpu_means_enodev_not_fallback(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = _prob()
    rc = lib.bifurcated_attn_decode(ctypes.byref(p), *([ctypes.c_void_p(16)] * 9), 1 << 30, None)
    assert rc == -6


def test_plan_string_mentions_branches(lib):
    s = lib.ba_plan_string(ctypes.byref(_prob())).decode()
    assert "ctx" in s and "dec" in s
    assert lib.ba_launches_per_call(ctypes.byref(_prob())) >= 1
