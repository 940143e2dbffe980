"""The NCCL code paths of dist.py on one GPU (world size 1: every collective
is a real NCCL call over a 1-rank communicator): head sharding with the
all-gather of the output heads, the batch split with its gather, and the
context split with its (out, lse) exchange and the ba_lse_merge join — each
must reproduce the single-call result (bit-exact where the arithmetic is the
same, within the bf16 tolerance for the extra rounding of the LSE join)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist

import paper_2403_08845_b200 as ba
from paper_2403_08845_b200.dist import (decode_context_split, decode_sharded, gather_batch,
                                        shard_batch_inputs, shard_inputs, split_context_inputs)
from synth import Config, make_inputs
from tests.parity import compare, oracle_rows

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def _dev(inp):
    return type(inp)(*(t.to(DEV) for t in (inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens)),
                     inp.scale)


def test_head_sharding_gather(nccl_group):
    cfg = Config("x", "bf16", b=8, h=8, g=8, d=128, mc=600, md=40)
    inp = _dev(make_inputs(cfg, 61, variant="ragged"))
    ref = ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, scale=inp.scale)
    loc = shard_inputs(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, 1, 0)
    out = decode_sharded(*loc, inp.lens, gather=True, world=1, scale=inp.scale)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_batch_split_gather(nccl_group):
    cfg = Config("x", "bf16", b=6, h=48, g=1, d=128, mc=400, md=30)
    inp = _dev(make_inputs(cfg, 62, variant="ragged"))
    ref = ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, scale=inp.scale)
    ql, Kdl, Vdl, ll = shard_batch_inputs(inp.q, inp.Kd, inp.Vd, inp.lens, 1, 0)
    out = ba.bifurcated_attn_decode(ql, inp.Kc, inp.Vc, Kdl, Vdl, ll, scale=inp.scale)
    full = gather_batch(out, cfg.b, 1)
    torch.cuda.synchronize()
    assert torch.equal(full, ref)


def test_context_split_exchange_and_merge(nccl_group):
    cfg = Config("x", "bf16", b=4, h=48, g=1, d=128, mc=700, md=30)
    host = make_inputs(cfg, 63, variant="ragged")
    inp = _dev(host)
    parts = split_context_inputs(inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, 1, 0)
    out, lse = decode_context_split(inp.q, *parts, world=1, scale=inp.scale)
    torch.cuda.synchronize()
    ref, ref_lse = oracle_rows(host)
    compare(out, lse, ref, ref_lse, cfg.torch_dtype, "ctx-split-nccl")
