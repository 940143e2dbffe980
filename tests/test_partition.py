"""Host-logic checks of the fused kernel's work split (bif_tc.cuh, CPU only).

A Python model of the scheduling arithmetic in bif_tc.cuh (my_range, seg_at,
part_rank, ctx_parts, dec_parts) is run for many shapes and checked for the
properties the device code relies on: every 128-position tile of every
sequence is streamed by exactly one CTA, each (group, row chunk) receives
exactly ctx_parts + dec_parts partials at distinct slots 0..parts-1, and the
slot counts match the ones libbifattn's planner reports (plan string)."""
import re

import pytest

import paper_2403_08845_b200 as ba
from paper_2403_08845_b200 import _build


def owner(f, T, G):
    return ((f + 1) * G - 1) // T


def part_rank(a, f, T, G):
    return owner(f, T, G) - owner(a, T, G) if T >= G else f - a


def simulate(b, h, g, mc, md, N, sms=148):
    p = h // g
    R = b * p
    spc = N // p
    nrc = -(-R // N)
    ntc = -(-mc // 128)
    ntd = -(-md // 128) if md else 0
    Tc = g * nrc * ntc
    Td = g * b * ntd
    G = min(Tc + Td, sms)
    tiles_seen = {}
    writes = {}

    gpc = N // p

    def dec_chunk(i, cb):
        return (i * g + cb * gpc) * ntd, (i * g + min(g, (cb + 1) * gpc)) * ntd

    for k in range(G):
        fc0, fc1 = k * Tc // G, (k + 1) * Tc // G
        fd0, fd1 = k * Td // G, (k + 1) * Td // G
        f = fc0
        while f < fc1:
            seg = f // ntc
            fend = min((seg + 1) * ntc, fc1)
            c, rc = seg // nrc, seg % nrc
            for ff in range(f, fend):
                key = ("c", c, ff % ntc)
                tiles_seen.setdefault((key, rc), []).append(k)
            writes.setdefault((c, rc), []).append(("c", part_rank(seg * ntc, f, Tc, G)))
            f = fend
        f = fd0
        while f < fd1:
            ic = f // ntd
            i, cb = ic // g, (ic % g) // gpc
            a, e = dec_chunk(i, cb)
            fend = min(e, fd1)
            for ff in range(f, fend):
                c, t = (ff // ntd) % g, ff % ntd
                tiles_seen.setdefault((("d", c, i, t), 0), []).append(k)
            writes.setdefault(("d", i, cb), []).append(("d", part_rank(a, f, Td, G)))
            f = fend

    def ctx_parts(c, rc):
        if Tc == 0:
            return 0
        ff = (c * nrc + rc) * ntc
        return part_rank(ff, ff + ntc - 1, Tc, G) + 1

    def dec_parts(i, cb):
        if Td == 0:
            return 0
        a, e = dec_chunk(i, cb)
        return part_rank(a, e - 1, Td, G) + 1

    # every tile exactly once
    for c in range(g):
        for rc in range(nrc):
            for t in range(ntc):
                assert tiles_seen[(("c", c, t), rc)] and len(tiles_seen[(("c", c, t), rc)]) == 1
    for c in range(g):
        for i in range(b):
            for t in range(ntd):
                assert len(tiles_seen[(("d", c, i, t), 0)]) == 1
    sc = sd = 0
    for key, w in writes.items():
        if key[0] == "d":
            ds = sorted(s for kind, s in w)
            assert ds == list(range(dec_parts(key[1], key[2])))
            sd = max(sd, len(ds))
        else:
            c, rc = key
            cs = sorted(s for kind, s in w)
            assert cs == list(range(ctx_parts(c, rc)))
            sc = max(sc, len(cs))
    return sc, sd


def pick_n(b, h, g):
    """Rows per chunk: the smallest N in {16,32,48,64} with p | N and N >= b*p,
    else the largest with p | N (the planner's rule, bifattn_api.cu)."""
    p = h // g
    cands = [n for n in (16, 32, 48, 64) if n % p == 0]
    fit = [n for n in cands if n >= b * p]
    return fit[0] if fit else cands[-1]


SHAPES = [(b, h, g, mc, md, pick_n(b, h, g)) for (b, h, g, mc, md) in [
    (16, 4, 4, 777, 50), (32, 32, 32, 8192, 256), (16, 32, 32, 8192, 256),
    (3, 48, 1, 300, 20), (9, 16, 4, 513, 21), (2, 8, 1, 10, 0),
    (40, 2, 2, 1290, 33), (24, 8, 4, 700, 45), (64, 32, 8, 16384, 512),
    (128, 48, 1, 8192, 256), (17, 4, 2, 640, 32), (5, 64, 2, 129, 300),
]]


@pytest.mark.parametrize("shape", SHAPES)
def test_partition_covers_every_tile_once(shape):
    simulate(*shape)


@pytest.mark.parametrize("shape", SHAPES)
def test_planner_slot_counts_match_model(shape):
    _build.build()
    b, h, g, mc, md, N = shape
    prob = ba.make_problem(b, h, g, 128, mc, md, 0)
    plan = ba.ba_plan_string(prob)
    m = re.search(r"N=(\d+).*slots=(\d+)\+(\d+)", plan)
    assert m, plan
    assert int(m.group(1)) == N
    sc, sd = simulate(b, h, g, mc, md, N)
    assert (int(m.group(2)), int(m.group(3))) == (sc, sd)
