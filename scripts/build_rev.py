"""Build the library of a git revision into paper_2403_08845_b200/libbifattn_<name>.so
(for an interleaved A/B against the working tree: scripts/ab.py --lib)
usage: python scripts/build_rev.py REV NAME"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_08845_b200 import _build  # noqa: E402

rev, name = sys.argv[1], sys.argv[2]
out = os.path.join(ROOT, "paper_2403_08845_b200", f"libbifattn_{name}.so")
with tempfile.TemporaryDirectory() as d:
    subprocess.check_call(f"git -C {ROOT} archive {rev} paper_2403_08845_b200/csrc include | tar -x -C {d}",
                          shell=True)
    cmd = [_build.NVCC, *_build.NVCC_FLAGS, "-I", os.path.join(d, "include"), "-o", out,
           os.path.join(d, "paper_2403_08845_b200", "csrc", "bifattn_api.cu")]
    subprocess.check_call(cmd)
print(out)
