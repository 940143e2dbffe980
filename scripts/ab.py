"""Interleaved A/B timing of the product library against a variant build of
the same sources (_build.build_variant) on one config: each round runs
bench.py once per library in a fresh process; medians of us_per_step and the
CUDA-graph replay over the rounds.

usage: python scripts/ab.py CONFIG ROUNDS NAME -DFLAG [-DFLAG ...]
       python scripts/ab.py CONFIG ROUNDS NAME --lib PATH   (a prebuilt library, e.g. scripts/build_rev.py)"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_08845_b200 import _build  # noqa: E402

cfg, rounds, name, defines = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4:]
if defines[:1] == ["--lib"]:
    libs = {"product": _build.build(), name: os.path.join(ROOT, defines[1])}
else:
    libs = {"product": _build.build(), name: _build.build_variant(name, defines)}
RUN = ("import sys; sys.path.insert(0, %r); import paper_2403_08845_b200 as ba; "
       "ba.load_library(%r); import bench; sys.argv = ['bench.py', '--config', %r, '--steps', '30', "
       "'--no-e2e', '--no-replicated', '--no-cpu-baseline', '--no-stream-peak', '--no-others', "
       "'--soak', '0.5']; bench.main()")
res = {k: {"us": [], "graph": []} for k in libs}
for _ in range(rounds):
    for k, lib in libs.items():
        out = subprocess.run([sys.executable, "-c", RUN % (ROOT, lib, cfg)], capture_output=True,
                             text=True, timeout=300, cwd=ROOT).stdout.strip().splitlines()
        d = json.loads(out[-1])
        res[k]["us"].append(d["us_per_step"])
        res[k]["graph"].append(d["graph_us_per_step"])
print(json.dumps({"config": cfg, "variant": name, "defines": defines,
                  **{k: {"us_median": statistics.median(v["us"]),
                         "graph_median": statistics.median(v["graph"]), "us_all": v["us"]}
                     for k, v in res.items()}}))
