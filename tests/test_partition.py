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


def dec_cost(N, nrc, g, mc, ntc, G, T):
    """The planner's decode-tile weight (bifattn_api.cu, make_plan)."""
    dc = 1.7 if N == 16 else 1.25
    if nrc > 1 and (2 * g * mc * 128 * 2 <= 64 * 2 ** 20 or 1.5 * ntc * G >= T):
        dc *= 2.4 if nrc >= 32 else 1.6
    return dc


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


def model(b, h, g, mc, md, cs, bw, N=None, with_ctx=True, dyn=False, dparts=1):
    """Python model of seg_at / ctx_unit / ctx_parts / dec_parts (bif_tc.cuh)
    over the planner's CTA table; bw = the plan's context band width.  With
    with_ctx=False (the context ran in ctx_rows_kernel) only decode tiles.
    dyn=True: the decode columns are taken dynamically (not in the table; one
    decode partial per row), and CTAs beyond the static tiles have empty
    ranges at the end of the table."""
    p = h // g
    N = N or pick_n(b, h, g)
    R = b * p
    nrc = -(-R // N)
    ntc = -(-mc // 128) if with_ctx else 0
    bw = bw if with_ctx else 1
    ntd = -(-md // 128) if md else 0
    if dyn:
        # (column, part) units: parts of ceil(ntd / parts) tiles, one slot each
        assert 1 <= dparts <= ntd
        unit = -(-ntd // dparts)
        assert -(-ntd // unit) == dparts
        sd_dyn = dparts if ntd else 0
        ntd = 0
    gpc = N // p
    ndc = -(-g // gpc)
    Tc = g * nrc * ntc
    Td = g * b * ntd
    T = Tc + Td
    G = len(cs) - 1
    nband = -(-ntc // bw) if ntc else 0
    banded = nband > 1
    assert not banded or nrc > 1
    assert cs[0] == 0 and cs[-1] == T
    if dyn and T < G:
        # one static tile per CTA, then empty ranges only at the end
        assert cs == [min(k, T) for k in range(G + 1)], cs
        G = T
        cs = cs[:T + 1]
    assert all(cs[k] < cs[k + 1] for k in range(G)), "empty CTA range"
    # units: (kind, chunk id, slot base, begin, end) in flat order (c, band, rc, tile)
    chunks = []
    f = 0
    for c in range(g):
        for band in range(nband):
            wb = min(bw, ntc - band * bw)
            for rc in range(nrc):
                chunks.append(("c", (c, rc), band, f, f + wb))
                f += wb
    assert f == Tc
    for i in range(b if ntd else 0):
        for cb in range(ndc):
            a = Tc + (i * g + cb * gpc) * ntd
            e = Tc + (i * g + min(g, (cb + 1) * gpc)) * ntd
            chunks.append(("d", (i, cb), 0, a, e))
    seen = [0] * T
    writes = {}
    for k in range(G):
        f = cs[k]
        while f < cs[k + 1]:
            kind, cid, band, a, e = next(ch for ch in chunks if ch[3] <= f < ch[4])
            fend = min(e, cs[k + 1])
            for ff in range(f, fend):
                seen[ff] += 1
            if kind == "c" and banded:
                assert a == f and fend == e, "a banded context unit was split"
                writes.setdefault((kind, cid), []).append(band)
            else:
                writes.setdefault((kind, cid), []).append(k - owner(cs, a))
            f = fend
    assert all(x == 1 for x in seen)
    sc = sd = 0
    for kind, cid, band, a, e in chunks:
        if kind == "c" and banded:
            assert sorted(writes[(kind, cid)]) == list(range(nband))
            sc = nband
            continue
        parts = owner(cs, e - 1) - owner(cs, a) + 1
        assert sorted(writes[(kind, cid)]) == list(range(parts))
        if kind == "c":
            sc = max(sc, parts)
        else:
            sd = max(sd, parts)
    if dyn:
        sd = sd_dyn
    # planner cost: decode tiles weigh DEC_COST (bifattn_api.cu, plan_split)
    DEC_COST = dec_cost(N, nrc, g, mc, ntc, G, T)
    loads = [(min(cs[k + 1], Tc) - min(cs[k], Tc)) + DEC_COST * (max(cs[k + 1], Tc) - max(cs[k], Tc))
             for k in range(max(G, 1))] if T else [0]
    return N, sc, sd, loads, banded


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
    plan = ba.ba_plan_string(prob)
    if plan.startswith("ctx_rows") and "+ merge" in plan:
        # both branches in the rows kernel (p >= 32): context items + one
        # decode item per (sample, group), then the merge launch
        m = re.search(r"items=(\d+)\+(\d+) dec", plan)
        assert int(m.group(2)) == b * g
        return
    if plan.startswith("ctx_rows"):
        # context on the rows-on-M kernel: one partial per split; the fused
        # launch streams decode tiles only (N = smallest multiple of 16 and p)
        m = re.search(r"splits=(\d+).*dec_tc\(N=(\d+).*slots=(\d+)\+(\d+)", plan)
        N = int(m.group(2))
        assert N == min(n for n in (16, 32, 48, 64) if n % (h // g) == 0)
        assert int(m.group(3)) == int(m.group(1))
        dyn = "cuda_core_dyn" in plan
        assert dyn == (h // g == 1), plan  # p = 1 decode columns are dynamic
        dp = int(re.search(r"parts=(\d+)", plan).group(1)) if dyn else 1
        if md:
            _, _, sd, _, _ = model(b, h, g, mc, md, cs, 1, N=N, with_ctx=False, dyn=dyn, dparts=dp)
            assert sd == int(m.group(4))
        return
    m = re.search(r"N=(\d+).*band=(\d+).*slots=(\d+)\+(\d+)", plan)
    assert m, plan
    dyn = "cuda_core_dyn" in plan
    dp = int(re.search(r"parts=(\d+)", plan).group(1)) if dyn else 1
    N, sc, sd, loads, banded = model(b, h, g, mc, md, cs, int(m.group(2)), dyn=dyn, dparts=dp)
    assert (int(m.group(1)), int(m.group(3)), int(m.group(4))) == (N, sc, sd)
    mean = sum(loads) / len(loads)
    # the segment penalty only trims loads; whole banded units (8 tiles) add
    # at most half a unit
    assert max(loads) <= mean + 3 + 0.1 * mean + (4 if banded else 0)


def test_fma_plan_has_no_cta_table():
    _build.build()
    assert ba.ba_plan_ctas(ba.make_problem(4, 2, 2, 16, 32, 4, 1)) == []
