"""Per-launch times of one config (bench.py's no-PDL event pass) for the
product library and, optionally, a variant library.
usage: python scripts/kernel_shares.py CONFIG [LIB ...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg, libs = sys.argv[1], sys.argv[2:] or [""]
RUN = ("import sys; sys.path.insert(0, %r); import paper_2403_08845_b200 as ba; "
       "lib = %r; lib and ba.load_library(lib); import bench; sys.argv = ['bench.py', '--config', %r, "
       "'--steps', '30', '--no-e2e', '--no-replicated', '--no-cpu-baseline', '--no-stream-peak', "
       "'--no-others', '--soak', '0.5']; bench.main()")
for lib in libs:
    out = subprocess.run([sys.executable, "-c", RUN % (ROOT, lib, cfg)], capture_output=True, text=True,
                         timeout=300, cwd=ROOT).stdout.strip().splitlines()
    d = json.loads(out[-1])
    print(json.dumps({"lib": lib or "product", "config": cfg, "us": round(d["us_per_step"], 2),
                      "kernels": {k: round(v.get("us_in_step", 0), 2) for k, v in d["kernels"].items()},
                      "plan": d["config"]["plan"][:90]}), flush=True)
