"""Head-group sharding of the bifurcated decode step across GPUs.

KV groups are independent: query head j reads only group j // p of Kc/Vc/Kd/Vd
(Eq. 1; Eq. 3-4).  So G ranks (G | g) each take
a contiguous block of g/G groups and the matching h/G query heads — the
attention partition of tensor parallelism, which the paper reports works
"out-of-the-box" (Table 8; per-rank h' = h/t, g' = g/t,
commented-out TP table).  There is NO collective inside
attention; each rank calls the same C ABI on its shard.  Only a caller that
wants the full [b][h][d] output pays one all-gather of the output heads (NCCL
over NVLink on GPUs; any torch.distributed backend works for the host logic).
"""
from __future__ import annotations

import contextlib
from typing import Optional, Tuple

import torch
import torch.distributed as dist


def _on_stream(stream):
    """Run a helper's kernels AND its collectives on ``stream``: torch's NCCL
    collectives order themselves against the CURRENT stream, so the caller's
    stream is made current for the whole helper (kernel -> all-gather ->
    merge stay ordered on it)."""
    if stream is None:
        return contextlib.nullcontext()
    return torch.cuda.stream(stream)


def shard_bounds(h: int, g: int, world: int, rank: int) -> Tuple[int, int, int, int]:
    """(g0, g1, h0, h1): the groups and query heads rank `rank` owns."""
    if g % world != 0:
        raise ValueError(f"head-group sharding needs world ({world}) | g ({g}); "
                         "g = 1 (MQA) runs replicas only")
    if h % g != 0:
        raise ValueError("h % g != 0")
    gl = g // world
    p = h // g
    g0, g1 = rank * gl, (rank + 1) * gl
    return g0, g1, g0 * p, g1 * p


def shard_inputs(q, Kc, Vc, Kd, Vd, world: int, rank: int):
    """Contiguous per-rank slices: q[:, h0:h1], Kc/Vc[g0:g1], Kd/Vd[:, g0:g1]."""
    b, h, d = q.shape
    g = Kc.shape[0]
    g0, g1, h0, h1 = shard_bounds(h, g, world, rank)
    return (q[:, h0:h1].contiguous(), Kc[g0:g1].contiguous(), Vc[g0:g1].contiguous(),
            Kd[:, g0:g1].contiguous(), Vd[:, g0:g1].contiguous())


def gather_heads(out_local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather per-rank outputs [b][h/G][d] and permute to [b][h][d]."""
    b, hl, d = out_local.shape
    buf = torch.empty((world, b, hl, d), dtype=out_local.dtype, device=out_local.device)
    src = out_local.contiguous()
    if out_local.is_cuda:
        dist.all_gather_into_tensor(buf.view(-1), src.view(-1), group=group)
    else:
        parts = list(buf.unbind(0))
        dist.all_gather(parts, src, group=group)
    return buf.permute(1, 0, 2, 3).reshape(b, world * hl, d)


def decode_sharded(q_local, Kc_local, Vc_local, Kd_local, Vd_local, lens, *, gather: bool = False,
                   world: Optional[int] = None, group=None, lse=None, scale=None,
                   workspace=None, stream=None):
    """Run this rank's shard of the step through the C ABI; optionally gather.

    Inputs are the rank-local slices from ``shard_inputs`` (rank-local h, g).
    Returns the local [b][h/G][d] output, or the full [b][h][d] if gather."""
    from . import bifurcated_attn_decode

    with _on_stream(stream):
        out = bifurcated_attn_decode(q_local, Kc_local, Vc_local, Kd_local, Vd_local, lens,
                                     lse=lse, scale=scale, workspace=workspace, stream=stream)
        if not gather:
            return out
        world = world or dist.get_world_size(group)
        return gather_heads(out, world, group)


# ---------------------------------------------------------------------------
# MQA / G > g: when the KV groups cannot be sharded
# (g = 1, "the single head in K and V are duplicated across TP ranks",
# PAPER.md:1014), split the work along the batch or along the context.
# ---------------------------------------------------------------------------
def batch_bounds(b: int, world: int, rank: int) -> Tuple[int, int]:
    """Samples [i0, i1) of rank `rank` (contiguous, sizes differ by <= 1).
    Each rank runs the whole step for its samples: the shared context is
    read once PER GPU (still once for all of the rank's samples), the decode
    caches are partitioned.  No collective inside attention."""
    if world > b:
        raise ValueError(f"batch split needs world ({world}) <= b ({b})")
    return rank * b // world, (rank + 1) * b // world


def shard_batch_inputs(q, Kd, Vd, lens, world: int, rank: int):
    i0, i1 = batch_bounds(q.shape[0], world, rank)
    return (q[i0:i1].contiguous(), Kd[i0:i1].contiguous(), Vd[i0:i1].contiguous(),
            lens[i0:i1].contiguous())


def gather_batch(out_local: torch.Tensor, b: int, world: int, group=None) -> torch.Tensor:
    """All-gather per-rank outputs along the batch (uneven blocks allowed)."""
    sizes = [batch_bounds(b, world, r)[1] - batch_bounds(b, world, r)[0] for r in range(world)]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(out_local.shape[1:]), dtype=out_local.dtype,
                      device=out_local.device)
    pad[: out_local.shape[0]] = out_local
    buf = torch.empty((world,) + tuple(pad.shape), dtype=pad.dtype, device=pad.device)
    if pad.is_cuda:
        dist.all_gather_into_tensor(buf.view(-1), pad.view(-1), group=group)
    else:
        dist.all_gather(list(buf.unbind(0)), pad, group=group)
    return torch.cat([buf[r, : sizes[r]] for r in range(world)], dim=0)


def context_bounds(mc: int, world: int, rank: int) -> Tuple[int, int]:
    """Context positions [t0, t1) of rank `rank` for the context split: the
    shared context is cut into `world` contiguous slices (each >= 1
    position); rank 0 also holds the decode caches."""
    if world > mc:
        raise ValueError(f"context split needs world ({world}) <= mc ({mc})")
    return rank * mc // world, (rank + 1) * mc // world


def split_context_inputs(Kc, Vc, Kd, Vd, lens, world: int, rank: int):
    """Rank-local inputs of the context split: Kc/Vc[:, t0:t1]; rank 0 keeps
    Kd/Vd and lens, the other ranks get an empty decode cache (md_cap = 0)."""
    t0, t1 = context_bounds(Kc.shape[1], world, rank)
    Kc_r, Vc_r = Kc[:, t0:t1].contiguous(), Vc[:, t0:t1].contiguous()
    if rank == 0:
        return Kc_r, Vc_r, Kd, Vd, lens
    e = Kd[:, :, :0].contiguous()
    return Kc_r, Vc_r, e, Vd[:, :, :0].contiguous(), torch.zeros_like(lens)


def exchange_partials(out_local: torch.Tensor, lse_local: torch.Tensor, world: int, group=None):
    """The one exchange of the context split: all-gather every rank's
    normalised partial output and its LSE -> [world][...] (NCCL over NVLink)."""
    ob = torch.empty((world,) + tuple(out_local.shape), dtype=out_local.dtype,
                     device=out_local.device)
    lb = torch.empty((world,) + tuple(lse_local.shape), dtype=lse_local.dtype,
                     device=lse_local.device)
    if out_local.is_cuda:
        dist.all_gather_into_tensor(ob.view(-1), out_local.contiguous().view(-1), group=group)
        dist.all_gather_into_tensor(lb.view(-1), lse_local.contiguous().view(-1), group=group)
    else:
        dist.all_gather(list(ob.unbind(0)), out_local.contiguous(), group=group)
        dist.all_gather(list(lb.unbind(0)), lse_local.contiguous(), group=group)
    return ob, lb


def decode_context_split(q, Kc_r, Vc_r, Kd_r, Vd_r, lens_r, *, world: Optional[int] = None,
                         group=None, scale=None, workspace=None, stream=None):
    """Context split of one step across ranks (inputs from split_context_inputs):
    each rank attends all rows to its context slice (+ the decode part on rank
    0) through the C ABI, the ranks exchange (out, lse) once, and every rank
    joins the partials with the LSE merge kernel (ba_lse_merge).  Returns the
    full [b][h][d] output and [b][h] lse on every rank."""
    from . import bifurcated_attn_decode, lse_merge

    world = world or dist.get_world_size(group)
    with _on_stream(stream):
        lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=q.device)
        out = bifurcated_attn_decode(q, Kc_r, Vc_r, Kd_r, Vd_r, lens_r, lse=lse, scale=scale,
                                     workspace=workspace, stream=stream)
        ob, lb = exchange_partials(out, lse, world, group)
        full_lse = torch.empty_like(lse)
        return lse_merge(ob, lb, lse=full_lse, stream=stream), full_lse


# ---------------------------------------------------------------------------
# One sharded step (bench.py's N > 1 path and tests/test_dist_gloo.py): pick
# the partition, slice the rank's inputs, run the rank's part through the
# C ABI, assemble the full output when asked.
# ---------------------------------------------------------------------------
def split_mode(b: int, h: int, g: int, mc: int, world: int) -> str:
    """Partition of one step over ``world`` ranks:
    'heads'   world | g: the paper's TP partition (h' = h/t, g' = g/t,
              PAPER.md:1014; Table 8 :1348-1365) — no collective in attention;
    'batch'   otherwise, when world <= b (MQA, g = 1: "the single head in K
              and V are duplicated across TP ranks", :1014) — each rank reads
              the shared context once for its samples, no collective;
    'context' otherwise: the context positions are split and the ranks
              exchange (out, lse) once (f3, :701-702)."""
    if world == 1:
        return "single"
    if g % world == 0:
        return "heads"
    if world <= b:
        return "batch"
    if world <= mc:
        return "context"
    raise ValueError(f"cannot partition b={b}, g={g}, mc={mc} over {world} ranks")


def shard_step(q, Kc, Vc, Kd, Vd, lens, world: int, rank: int, mode: str):
    """The rank-local tensors (q, Kc, Vc, Kd, Vd, lens) of ``mode``."""
    if mode == "single":
        return q, Kc, Vc, Kd, Vd, lens
    if mode == "heads":
        ql, Kcl, Vcl, Kdl, Vdl = shard_inputs(q, Kc, Vc, Kd, Vd, world, rank)
        return ql, Kcl, Vcl, Kdl, Vdl, lens
    if mode == "batch":
        ql, Kdl, Vdl, ll = shard_batch_inputs(q, Kd, Vd, lens, world, rank)
        return ql, Kc, Vc, Kdl, Vdl, ll
    if mode == "context":
        Kcl, Vcl, Kdl, Vdl, ll = split_context_inputs(Kc, Vc, Kd, Vd, lens, world, rank)
        return q, Kcl, Vcl, Kdl, Vdl, ll
    raise ValueError(mode)


def assemble(out_local, lse_local, b: int, world: int, mode: str, group=None, stream=None):
    """The full [b][h][d] output from every rank's part: one all-gather of the
    output heads ('heads') or samples ('batch'), or the (out, lse) exchange +
    LSE join ('context', needs ``lse_local``; GPU only: ba_lse_merge)."""
    with _on_stream(stream):
        if mode == "single":
            return out_local
        if mode == "heads":
            return gather_heads(out_local, world, group)
        if mode == "batch":
            return gather_batch(out_local, b, world, group)
        if mode == "context":
            from . import lse_merge

            ob, lb = exchange_partials(out_local, lse_local, world, group)
            return lse_merge(ob, lb, stream=stream)
        raise ValueError(mode)
