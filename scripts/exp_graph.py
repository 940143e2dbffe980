"""Eager vs CUDA-graph replay of back-to-back steps: host overhead per call."""
import sys, os, json, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
if os.environ.get("EXP_LIB"):
    ba.load_library(os.environ["EXP_LIB"])
from synth import CONFIGS, make_inputs, alg_bytes

base = CONFIGS["mha7b_b32"]
for mc, md in [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(1280, 0), (8192, 256)]:
    cfg = base.with_(mc=mc, md=md)
    sets = [make_inputs(cfg, 1 + k, device="cuda") for k in range(2)]
    outs = [torch.empty_like(s.q) for s in sets]
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, sets[0].scale)
    ws = ba.alloc_workspace(prob, "cuda")
    st = torch.cuda.Stream()
    def step(k):
        s = sets[k % 2]
        ba.bifurcated_attn_decode(s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, outs[k % 2], workspace=ws, scale=s.scale,
                                  stream=torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for k in range(4): step(k)
        torch.cuda.synchronize()
        # host cost per call (no sync)
        t0 = time.perf_counter()
        for k in range(200): step(k)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        host_us = (t1 - t0) / 200 * 1e6
        # eager device time
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(40): step(k)
        b.record(); torch.cuda.synchronize()
        eager = a.elapsed_time(b) / 40 * 1e3
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for k in range(20): step(k)
        g.replay(); torch.cuda.synchronize()
        a.record()
        for _ in range(3): g.replay()
        b.record(); torch.cuda.synchronize()
        graph = a.elapsed_time(b) / 60 * 1e3
    print(json.dumps({"mc": mc, "md": md, "host_us_per_call": round(host_us, 2), "eager_us": round(eager, 2), "graph_us": round(graph, 2)}), flush=True)
