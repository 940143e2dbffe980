"""GPU parity of append + attend (include/bifattn.h
bifurcated_attn_decode_append) through the C ABI.  The reference is the
definition of the step: write k_new/v_new into the host copy of the decode
cache at lens[i].. (Table 5 "+K_prev" rows, :982-987), advance lens by
n, then the fp64 oracle.  Checked: the output and lse element by element, the
device caches bit-exactly, lens advanced on the device, a sequence of steps
driven only by the device-side lens (CUDA-graph replays), and both kernel
families."""
import pytest
import torch

import paper_2403_08845_b200 as ba
from synth import Config, make_inputs
from tests.parity import compare, oracle_rows

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def host_append(inp, k_new, v_new, n):
    Kd, Vd, lens = inp.Kd.clone(), inp.Vd.clone(), inp.lens.clone()
    cap = Kd.shape[2]
    for i in range(Kd.shape[0]):
        L = max(0, min(int(lens[i]), cap))
        for k in range(n):
            if L + k < cap:
                Kd[i, :, L + k] = k_new[i, :, k]
                Vd[i, :, L + k] = v_new[i, :, k]
        lens[i] = min(L + n, cap)
    return type(inp)(inp.q, inp.Kc, inp.Vc, Kd, Vd, lens, inp.scale)


CASES = [
    (Config("ap_mha", "bf16", b=16, h=8, g=8, d=128, mc=900, md=70), 1),
    (Config("ap_gqa_n3", "bf16", b=6, h=16, g=4, d=128, mc=400, md=50), 3),
    (Config("ap_fp32", "fp32", b=4, h=4, g=2, d=64, mc=100, md=20), 2),
    (Config("ap_mqa", "bf16", b=4, h=48, g=1, d=128, mc=300, md=40), 1),  # rows kernel + merge
    # rows kernel (context) + the early-start dynamic decode launch (p = 1)
    (Config("ap_rows_dyn", "bf16", b=80, h=4, g=4, d=128, mc=300, md=700), 1),
    # the same with the two-block rows kernel (>= 2 row blocks) and decode parts
    (Config("ap_rows2_dyn", "bf16", b=200, h=2, g=2, d=128, mc=500, md=1400), 1),
    # fused kernel, dynamic columns cut into parts (few long columns)
    (Config("ap_dyn_parts", "bf16", b=16, h=2, g=2, d=128, mc=200, md=2500), 1),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0].name)
@pytest.mark.parametrize("flags", [0, ba.BA_FLAG_FORCE_FMA], ids=["auto", "fma"])
def test_append_then_attend(case, flags):
    cfg, n = case
    inp = make_inputs(cfg, 41, variant="ragged", n_tok=n)
    inp.lens[0] = cfg.md          # full cache: the appended rows are dropped
    inp.lens[1] = cfg.md - 1      # partly dropped when n > 1
    g = torch.Generator().manual_seed(5)
    k_new = torch.randn(cfg.b, cfg.g, n, cfg.d, generator=g).to(cfg.torch_dtype)
    v_new = torch.randn(cfg.b, cfg.g, n, cfg.d, generator=g).to(cfg.torch_dtype)
    Kd, Vd, lens = inp.Kd.to(DEV), inp.Vd.to(DEV), inp.lens.to(DEV)
    q = inp.q.to(DEV)
    lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=DEV)
    out = ba.bifurcated_attn_decode_append(q, k_new.to(DEV), v_new.to(DEV), inp.Kc.to(DEV),
                                           inp.Vc.to(DEV), Kd, Vd, lens, lse=lse,
                                           scale=inp.scale, flags=flags)
    torch.cuda.synchronize()
    ref_inp = host_append(inp, k_new, v_new, n)
    assert torch.equal(lens.cpu(), ref_inp.lens)
    assert torch.equal(Kd.cpu(), ref_inp.Kd) and torch.equal(Vd.cpu(), ref_inp.Vd)
    ref, ref_lse = oracle_rows(ref_inp)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, f"append/{cfg.name}")


def test_append_steps_in_a_cuda_graph():
    """Four decode steps replayed from one captured graph: the device-side lens
    advance drives the cache position; each step is checked."""
    cfg = Config("x", "bf16", b=8, h=4, g=4, d=128, mc=500, md=40)
    inp = make_inputs(cfg, 43, lens=[3, 0, 10, 37, 38, 39, 1, 20])
    q, Kc, Vc = inp.q.to(DEV), inp.Kc.to(DEV), inp.Vc.to(DEV)
    Kd, Vd, lens = inp.Kd.to(DEV), inp.Vd.to(DEV), inp.lens.to(DEV)
    k_new = torch.empty(cfg.b, cfg.g, 1, cfg.d, dtype=torch.bfloat16, device=DEV)
    v_new = torch.empty_like(k_new)
    out = torch.empty_like(q)
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, q.dtype, inp.scale)
    ws = ba.alloc_workspace(prob, DEV)
    s = torch.cuda.Stream()
    step = lambda: ba.bifurcated_attn_decode_append(q, k_new, v_new, Kc, Vc, Kd, Vd, lens, out,
                                                    workspace=ws, scale=inp.scale, stream=s)
    # capture on copies so that the capture itself does not advance the real state
    snap = (Kd.clone(), Vd.clone(), lens.clone())
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        step()
    Kd.copy_(snap[0]); Vd.copy_(snap[1]); lens.copy_(snap[2])
    torch.cuda.synchronize()
    host = inp
    gen = torch.Generator().manual_seed(6)
    for it in range(4):
        kn = torch.randn(cfg.b, cfg.g, 1, cfg.d, generator=gen).to(torch.bfloat16)
        vn = torch.randn(cfg.b, cfg.g, 1, cfg.d, generator=gen).to(torch.bfloat16)
        k_new.copy_(kn); v_new.copy_(vn)
        graph.replay()
        torch.cuda.synchronize()
        host = host_append(host, kn, vn, 1)
        assert torch.equal(lens.cpu(), host.lens), it
        ref, _ = oracle_rows(host)
        compare(out, None, ref, None, cfg.torch_dtype, f"graph-step{it}")


def test_append_host_entry_equals_device_call():
    """bifurcated_attn_decode_append_host (host q/k_new/v_new in, host out back,
    caches resident) gives the device call's result bit for bit, and with
    hlens = None the device lens carries over between steps."""
    cfg = Config("x", "bf16", b=8, h=4, g=4, d=128, mc=500, md=30)
    inp = make_inputs(cfg, 47, lens=[3, 0, 10, 20, 28, 29, 1, 5])
    gen = torch.Generator().manual_seed(8)
    kn = torch.randn(cfg.b, cfg.g, 1, cfg.d, generator=gen).to(torch.bfloat16)
    vn = torch.randn(cfg.b, cfg.g, 1, cfg.d, generator=gen).to(torch.bfloat16)
    # device reference: two steps
    Kd, Vd, lens = inp.Kd.to(DEV), inp.Vd.to(DEV), inp.lens.to(DEV)
    ref = []
    for _ in range(2):
        ref.append(ba.bifurcated_attn_decode_append(inp.q.to(DEV), kn.to(DEV), vn.to(DEV),
                                                    inp.Kc.to(DEV), inp.Vc.to(DEV), Kd, Vd, lens,
                                                    scale=inp.scale).cpu())
    # host entry: lens given on the first step only
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, torch.bfloat16, inp.scale)
    dev = dict(q=torch.empty(inp.q.shape, dtype=torch.bfloat16, device=DEV),
               k_new=torch.empty(kn.shape, dtype=torch.bfloat16, device=DEV),
               v_new=torch.empty(vn.shape, dtype=torch.bfloat16, device=DEV),
               Kc=inp.Kc.to(DEV), Vc=inp.Vc.to(DEV), Kd=inp.Kd.to(DEV), Vd=inp.Vd.to(DEV),
               lens=torch.empty(cfg.b, dtype=torch.int32, device=DEV),
               out=torch.empty(inp.q.shape, dtype=torch.bfloat16, device=DEV),
               workspace=ba.alloc_workspace(prob, DEV))
    pin = lambda t: t.contiguous().pin_memory()  # noqa: E731
    hq, hkn, hvn, hl = pin(inp.q), pin(kn), pin(vn), pin(inp.lens)
    for step in range(2):
        hout = torch.empty_like(hq).pin_memory()
        ba.bifurcated_attn_decode_append_host(hq, hkn, hvn, hout, dev,
                                              hlens=hl if step == 0 else None, scale=inp.scale)
        torch.cuda.synchronize()
        assert torch.equal(hout, ref[step]), step
    assert torch.equal(dev["lens"].cpu(), lens.cpu())


def test_packed_step_one_copy_each_way_and_graph():
    """bifurcated_attn_decode_step_packed: one H2D of [q | k_new | v_new | lens],
    append + attend, one D2H of [out | lse]; two steps, the second replayed
    from a CUDA graph of the whole step, each equal to the oracle on the
    host-side appended cache."""
    cfg = Config("packed", "bf16", b=32, h=8, g=4, d=128, mc=700, md=64)
    inp = make_inputs(cfg, 61, lens=[3 + (5 * i) % 50 for i in range(cfg.b)])
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale)
    Kc, Vc = inp.Kc.to(DEV), inp.Vc.to(DEV)
    Kd, Vd = inp.Kd.to(DEV).clone(), inp.Vd.to(DEV).clone()
    step = ba.PackedStep(prob, Kc, Vc, Kd, Vd, DEV, with_lse=True)
    host = inp
    lens = inp.lens.clone()
    g = torch.cuda.CUDAGraph()
    for k in range(2):
        kn = torch.randn(cfg.b, cfg.g, 1, cfg.d).to(cfg.torch_dtype)
        vn = torch.randn(cfg.b, cfg.g, 1, cfg.d).to(cfg.torch_dtype)
        q = torch.randn(cfg.b, cfg.h, cfg.d).to(cfg.torch_dtype)
        step.pack(q, kn, vn, lens)
        if k == 0:
            step.run()
        else:
            s = torch.cuda.Stream()
            with torch.cuda.graph(g, stream=s):
                step.run(stream=s)
            step.pack(q, kn, vn, lens)  # capture does not execute; the replay does
            Kd.copy_(host.Kd.to(DEV))
            Vd.copy_(host.Vd.to(DEV))
            with torch.cuda.stream(s):
                g.replay()
        torch.cuda.synchronize()
        host = host_append(type(inp)(q, host.Kc, host.Vc, host.Kd, host.Vd, lens, inp.scale),
                           kn, vn, 1)
        ref, ref_lse = oracle_rows(host)
        compare(step.out().clone(), step.lse().clone(), ref, ref_lse, cfg.torch_dtype, f"packed{k}")
        lens = host.lens.clone()
