"""Host overhead per call vs GPU time; CUDA-graph replay of the same steps."""
import sys, os, json, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs, alg_bytes

for name in ("mha7b_b32", "mha7b_b16"):
    cfg = CONFIGS[name]
    sets = [make_inputs(cfg, 1 + k, device="cuda") for k in range(2)]
    outs = [torch.empty_like(s.q) for s in sets]
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, sets[0].scale)
    ws = ba.alloc_workspace(prob, "cuda")
    st = torch.cuda.Stream()
    def step(k):
        s = sets[k % 2]
        ba.bifurcated_attn_decode(s.q, s.Kc, s.Vc, s.Kd, s.Vd, s.lens, outs[k % 2], workspace=ws, scale=s.scale, stream=st)
    with torch.cuda.stream(st):
        for k in range(5): step(k)
    torch.cuda.synchronize()
    # host time per call (GPU not waited)
    t0 = time.perf_counter()
    with torch.cuda.stream(st):
        for k in range(200): step(k)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    host_us = (t1 - t0) / 200 * 1e6
    # stream time
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record()
        for k in range(100): step(k)
        b.record()
    torch.cuda.synchronize()
    stream_us = a.elapsed_time(b) / 100 * 1e3
    # graph of 20 steps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for k in range(20): step(k)
    g.replay(); torch.cuda.synchronize()
    res = []
    for r in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(); g.replay(); b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / 20 * 1e3)
    gus = statistics.median(res)
    print(json.dumps({"cfg": name, "host_us_per_call": round(host_us, 1), "stream_us": round(stream_us, 2),
                      "graph_us": round(gus, 2), "graph_GBs": round(alg_bytes(cfg) / gus / 1e3, 1)}), flush=True)
