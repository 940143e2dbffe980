"""A/B of two builds of libbifattn.so on the same box (raw ctypes, so an older
ABI-1 build loads too): interleaved timing of the C2a/C2b steps."""
import ctypes, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import CONFIGS, make_inputs


class Prob(ctypes.Structure):
    _fields_ = [("b", ctypes.c_int32), ("h", ctypes.c_int32), ("g", ctypes.c_int32),
                ("d", ctypes.c_int32), ("mc", ctypes.c_int32), ("md_cap", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("scale", ctypes.c_float), ("flags", ctypes.c_uint32),
                ("n_tok", ctypes.c_int32)]


libs = {os.path.basename(p): ctypes.CDLL(os.path.abspath(p)) for p in sys.argv[1:]}
for lib in libs.values():
    lib.ba_workspace_bytes.restype = ctypes.c_size_t
for name in ("mha7b_b16", "mha7b_b32"):
    cfg = CONFIGS[name]
    sets = [make_inputs(cfg, 1 + k, device="cuda") for k in range(2)]
    outs = [torch.empty_like(s.q) for s in sets]
    pr = Prob(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, 0, sets[0].scale, 0, 1)
    res = {k: [] for k in libs}
    for rep in range(6):
        for k, lib in libs.items():
            ws = torch.zeros(lib.ba_workspace_bytes(ctypes.byref(pr)), dtype=torch.uint8, device="cuda")
            st = torch.cuda.current_stream().cuda_stream
            def step(j):
                s = sets[j % 2]
                rc = lib.bifurcated_attn_decode(ctypes.byref(pr), ctypes.c_void_p(s.q.data_ptr()),
                    ctypes.c_void_p(s.Kc.data_ptr()), ctypes.c_void_p(s.Vc.data_ptr()),
                    ctypes.c_void_p(s.Kd.data_ptr()), ctypes.c_void_p(s.Vd.data_ptr()),
                    ctypes.c_void_p(s.lens.data_ptr()), ctypes.c_void_p(outs[j % 2].data_ptr()),
                    None, ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                    ctypes.c_void_p(st))
                assert rc == 0, rc
            for j in range(5):
                step(j)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record()
            for j in range(40):
                step(j)
            b.record(); torch.cuda.synchronize()
            res[k].append(a.elapsed_time(b) / 40 * 1e3)
    print(json.dumps({"cfg": name, **{k: round(statistics.median(v), 2) for k, v in res.items()}}))
