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

from typing import Optional, Tuple

import torch
import torch.distributed as dist


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

    out = bifurcated_attn_decode(q_local, Kc_local, Vc_local, Kd_local, Vd_local, lens, lse=lse,
                                 scale=scale, workspace=workspace, stream=stream)
    if not gather:
        return out
    world = world or dist.get_world_size(group)
    return gather_heads(out, world, group)
