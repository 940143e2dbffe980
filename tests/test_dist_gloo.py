"""Multi-process (gloo, world_size 2, CPU) tests of the head-group sharding host
logic: sharding the problem by KV group and all-gathering the output heads is
bit-identical to the unsharded computation (groups are independent, Eq. 1
PAPER.md:208).  The per-shard compute here is the oracle (no GPU in CI); on
GPUs the same shard_inputs / gather_heads wrap the C ABI."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_08845_b200.dist import gather_heads, shard_bounds, shard_inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg_kw, seed, variant, q_out):
    import oracle
    from synth import Config, make_inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = Config(**cfg_kw)
        inp = make_inputs(cfg, seed, variant=variant)
        ql, Kcl, Vcl, Kdl, Vdl = shard_inputs(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, world, rank)
        out, lse, _ = oracle.attn_decode(ql, Kcl, Vcl, Kdl, Vdl, inp.lens, scale=inp.scale)
        out_t = torch.from_numpy(out).reshape(cfg.b, cfg.h // world, cfg.d)
        full = gather_heads(out_t, world)
        lse_t = torch.from_numpy(lse).reshape(cfg.b, cfg.h // world, 1)
        full_lse = gather_heads(lse_t, world)
        if rank == 0:
            q_out.put((full.numpy(), full_lse.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_kw,variant", [
    (dict(name="mha", dtype="bf16", b=3, h=8, g=8, d=32, mc=40, md=6), "ragged"),
    (dict(name="gqa", dtype="bf16", b=4, h=8, g=2, d=16, mc=33, md=5), "normal"),
    (dict(name="tiny", dtype="fp32", b=4, h=2, g=2, d=16, mc=32, md=4), "normal"),
])
def test_sharded_equals_unsharded(cfg_kw, variant):
    import oracle
    from synth import Config, make_inputs

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_kw, 5, variant, q))
             for r in range(world)]
    for p in procs:
        p.start()
    full, full_lse = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = Config(**cfg_kw)
    inp = make_inputs(cfg, 5, variant=variant)
    ref, ref_lse, _ = oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                         scale=inp.scale)
    np.testing.assert_array_equal(full.reshape(-1, cfg.d), ref)
    np.testing.assert_array_equal(full_lse.reshape(-1), ref_lse)


def test_shard_bounds():
    assert shard_bounds(32, 32, 8, 3) == (12, 16, 12, 16)
    assert shard_bounds(32, 8, 4, 1) == (2, 4, 8, 16)
    assert shard_bounds(64, 64, 2, 1) == (32, 64, 32, 64)
    with pytest.raises(ValueError):
        shard_bounds(48, 1, 2, 0)  # MQA: replicas only
    # shards tile the heads exactly once
    for world in (1, 2, 4, 8):
        heads = []
        for r in range(world):
            g0, g1, h0, h1 = shard_bounds(32, 8, world, r) if 8 % world == 0 else (0, 0, 0, 0)
            heads += list(range(h0, h1))
        if 8 % world == 0:
            assert heads == list(range(32))


# ---------------------------------------------------------------------------
# batch split and context split (MQA, G > g)
# ---------------------------------------------------------------------------
def _worker_f3(rank, world, port, cfg_kw, seed, mode, q_out):
    import oracle
    from paper_2403_08845_b200.dist import (exchange_partials, gather_batch, shard_batch_inputs,
                                            split_context_inputs)
    from synth import Config, make_inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = Config(**cfg_kw)
        inp = make_inputs(cfg, seed, variant="ragged")
        if mode == "batch":
            ql, Kdl, Vdl, ll = shard_batch_inputs(inp.q, inp.Kd, inp.Vd, inp.lens, world, rank)
            out, lse, _ = oracle.attn_decode(ql, inp.Kc, inp.Vc, Kdl, Vdl, ll, scale=inp.scale)
            full = gather_batch(torch.from_numpy(out).reshape(ql.shape[0], cfg.h, cfg.d),
                                cfg.b, world)
            if rank == 0:
                q_out.put((full.numpy(), None))
        else:
            Kc_r, Vc_r, Kd_r, Vd_r, l_r = split_context_inputs(inp.Kc, inp.Vc, inp.Kd, inp.Vd,
                                                               inp.lens, world, rank)
            out, lse, _ = oracle.attn_decode(inp.q, Kc_r, Vc_r, Kd_r, Vd_r, l_r, scale=inp.scale)
            ob, lb = exchange_partials(torch.from_numpy(out), torch.from_numpy(lse), world)
            if rank == 0:
                q_out.put((ob.numpy(), lb.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["batch", "context"])
@pytest.mark.parametrize("world", [2, 3])
def test_mqa_batch_and_context_split(mode, world):
    """g = 1 cannot head-shard; the batch split (no collective) and the
    context split (one exchange of (out, lse), then the LSE join of Eq. 4
    across slices — here written out in numpy as the test's reference of the
    ba_lse_merge kernel) both reproduce the unsplit oracle."""
    import oracle
    from synth import Config, make_inputs

    cfg_kw = dict(name="mqa", dtype="bf16", b=5, h=6, g=1, d=16, mc=37, md=7)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_f3, args=(r, world, port, cfg_kw, 8, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    a, b_ = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = Config(**cfg_kw)
    inp = make_inputs(cfg, 8, variant="ragged")
    ref, ref_lse, _ = oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                         scale=inp.scale)
    if mode == "batch":
        np.testing.assert_array_equal(a.reshape(-1, cfg.d), ref)
        return
    M = b_.max(axis=0)
    w = np.exp(b_ - M)                          # [world][rows]
    out = (w[..., None] * a).sum(0) / w.sum(0)[..., None]
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-13)
    np.testing.assert_allclose(M + np.log(w.sum(0)), ref_lse, rtol=0, atol=1e-12)


def test_split_bounds():
    from paper_2403_08845_b200.dist import batch_bounds, context_bounds
    for world in (1, 2, 3, 8):
        assert [i for r in range(world) for i in range(*batch_bounds(128, world, r))] == \
            list(range(128))
        assert [t for r in range(world) for t in range(*context_bounds(8192, world, r))] == \
            list(range(8192))
    with pytest.raises(ValueError):
        context_bounds(3, 4, 0)


def _step_worker(rank, world, port, cfg_kw, seed, mode, q_out):
    import oracle
    from paper_2403_08845_b200.dist import assemble, shard_step, split_mode
    from synth import Config, make_inputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = Config(**cfg_kw)
        assert split_mode(cfg.b, cfg.h, cfg.g, cfg.mc, world) == mode
        inp = make_inputs(cfg, seed, variant="ragged")
        ql, Kcl, Vcl, Kdl, Vdl, ll = shard_step(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                                world, rank, mode)
        out, _, _ = oracle.attn_decode(ql, Kcl, Vcl, Kdl, Vdl, ll, scale=inp.scale)
        out_t = torch.from_numpy(out).reshape(ql.shape)
        full = assemble(out_t, None, cfg.b, world, mode)
        if rank == 0:
            q_out.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_kw,mode", [
    (dict(name="mha", dtype="bf16", b=3, h=8, g=8, d=32, mc=40, md=6), "heads"),
    (dict(name="mqa", dtype="bf16", b=5, h=6, g=1, d=16, mc=37, md=7), "batch"),
])
def test_sharded_step_equals_unsharded(cfg_kw, mode):
    """bench.py's N > 1 step (dist.split_mode / shard_step / assemble) at world
    size 2 equals the unsharded step bit for bit (the per-rank compute is the
    oracle here; on GPUs it is the C ABI)."""
    import oracle
    from synth import Config, make_inputs

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, cfg_kw, 7, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = Config(**cfg_kw)
    inp = make_inputs(cfg, 7, variant="ragged")
    ref, _, _ = oracle.attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens,
                                   scale=inp.scale)
    np.testing.assert_array_equal(full.reshape(ref.shape), ref)


def test_split_mode_choices():
    from paper_2403_08845_b200.dist import split_mode

    assert split_mode(32, 32, 32, 8192, 1) == "single"
    assert split_mode(32, 32, 32, 8192, 8) == "heads"
    assert split_mode(64, 32, 8, 16384, 8) == "heads"
    assert split_mode(128, 48, 1, 8192, 8) == "batch"
    assert split_mode(2, 4, 1, 100, 4) == "context"
    with pytest.raises(ValueError):
        split_mode(1, 1, 1, 2, 4)
