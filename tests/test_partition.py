"""Host-logic checks of the fused kernel's work split (bif_tc.cuh, CPU only).

The planner in libbifattn (plan_split) returns each CTA's contiguous range of
flat tiles [context tiles | decode tiles] (ba_plan_ctas).  A Python model of the
device-side segment/slot arithmetic of bif_tc.cuh (seg_at, ctx_parts,
dec_parts) is run over that table for many shapes and checked for what the
kernel relies on: the ranges are non-empty and cover every tile exactly once;
each chunk's partials land in distinct slots 0..parts-1; the slot counts match
the planner's (plan string); and no CTA is loaded far above the mean."""
import re

import pytest

import paper_2403_08845_b200 as ba
from paper_2403_08845_b200 import _build


DEC_COST = 1.25


def owner(cs, f):
    lo, hi = 0, len(cs) - 2
    while lo < hi:
        mid = (lo + hi + 1) >> 1
        if cs[mid] <= f:
            lo = mid
        else:
            hi = mid - 1
    return lo


def pick_n(b, h, g):
    """Rows per chunk: the smallest N in {16,32,48,64} with p | N and
    N >= min(b*p, 32), else the largest with p | N (the planner's rule,
    bifattn_api.cu: N = 48/64 spill softmax registers)."""
    p = h // g
    cands = [n for n in (16, 32, 48, 64) if n % p == 0]
    fit = [n for n in cands if n >= min(b * p, 32)]
    return fit[0] if fit else cands[-1]


def model(b, h, g, mc, md, cs):
    p = h // g
    N = pick_n(b, h, g)
    R = b * p
    nrc = -(-R // N)
    ntc = -(-mc // 128)
    ntd = -(-md // 128) if md else 0
    gpc = N // p
    ndc = -(-g // gpc)
    Tc = g * nrc * ntc
    Td = g * b * ntd
    T = Tc + Td
    G = len(cs) - 1
    assert cs[0] == 0 and cs[-1] == T
    assert all(cs[k] < cs[k + 1] for k in range(G)), "empty CTA range"
    # chunks: (kind, id, begin, end)
    chunks = [("c", k, k * ntc, (k + 1) * ntc) for k in range(g * nrc)]
    for i in range(b if ntd else 0):
        for cb in range(ndc):
            a = Tc + (i * g + cb * gpc) * ntd
            e = Tc + (i * g + min(g, (cb + 1) * gpc)) * ntd
            chunks.append(("d", (i, cb), a, e))
    seen = [0] * T
    writes = {}
    for k in range(G):
        f = cs[k]
        while f < cs[k + 1]:
            kind, cid, a, e = next(ch for ch in chunks if ch[2] <= f < ch[3])
            fend = min(e, cs[k + 1])
            for ff in range(f, fend):
                seen[ff] += 1
            writes.setdefault((kind, cid), []).append(k - owner(cs, a))
            f = fend
    assert all(x == 1 for x in seen)
    sc = sd = 0
    for kind, cid, a, e in chunks:
        parts = owner(cs, e - 1) - owner(cs, a) + 1
        assert sorted(writes[(kind, cid)]) == list(range(parts))
        if kind == "c":
            sc = max(sc, parts)
        else:
            sd = max(sd, parts)
    # planner cost: decode tiles weigh DEC_COST (bifattn_api.cu, plan_split)
    loads = [(min(cs[k + 1], Tc) - min(cs[k], Tc)) + DEC_COST * (max(cs[k + 1], Tc) - max(cs[k], Tc))
             for k in range(G)]
    return N, sc, sd, loads


SHAPES = [
    (16, 4, 4, 777, 50), (32, 32, 32, 8192, 256), (16, 32, 32, 8192, 256),
    (3, 48, 1, 300, 20), (9, 16, 4, 513, 21), (2, 8, 1, 10, 0),
    (40, 2, 2, 1290, 33), (24, 8, 4, 700, 45), (64, 32, 8, 16384, 512),
    (128, 48, 1, 8192, 256), (17, 4, 2, 640, 32), (5, 64, 2, 129, 300),
    (256, 64, 64, 2048, 1024),
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_split_covers_every_tile_once_and_slots_match(shape):
    _build.build()
    b, h, g, mc, md = shape
    prob = ba.make_problem(b, h, g, 128, mc, md, 0)
    cs = ba.ba_plan_ctas(prob)
    assert cs, "tensor-core plan expected"
    N, sc, sd, loads = model(b, h, g, mc, md, cs)
    plan = ba.ba_plan_string(prob)
    m = re.search(r"N=(\d+).*slots=(\d+)\+(\d+)", plan)
    assert m, plan
    assert (int(m.group(1)), int(m.group(2)), int(m.group(3))) == (N, sc, sd)
    mean = sum(loads) / len(loads)
    assert max(loads) <= mean + 3 + 0.1 * mean  # the segment penalty only trims loads


def test_fma_plan_has_no_cta_table():
    _build.build()
    assert ba.ba_plan_ctas(ba.make_problem(4, 2, 2, 16, 32, 4, 1)) == []
