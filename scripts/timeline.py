"""Per-CTA phase timeline of the fused kernel from %globaltimer stamps
(-DBIFATTN_TRACE build of the same sources, _build.build_variant("trace")).

usage: python scripts/timeline.py [config ...]   (default: mha7b_b32 mha7b_b32_fp8)

Stamps (include/bifattn.h ba_set_trace_buffer; bif_tc.cuh): per CTA slot 250
kernel start, 254 after the PDL wait, 251 main loop end, 252 out of the grid
barrier, 253 merge done; softmax thread 128: 20 S ready, 21/22 fast/slow path
after the vote, 23 P handed to the MMA, 2/3 first tile of a context/decode
segment, 4 segment end; producer 30 (TMA issue of tile u); QK 33 (K landed),
31 (QK issued); PV 32 (PV issued).  Prints one JSON line per config: the
phase split of the step (median / max over CTAs, us) and the per-tile
softmax intervals."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_08845_b200 import _build  # noqa: E402

LIB = _build.build_variant("trace", ["-DBIFATTN_TRACE"])
import paper_2403_08845_b200 as ba  # noqa: E402

ba.load_library(LIB)
from synth import CONFIGS, make_inputs, seed_for  # noqa: E402


def med(v):
    return round(statistics.median(v), 3) if v else None


def run(name):
    cfg = CONFIGS[name]
    inp = make_inputs(cfg, seed_for(name), device="cuda")
    prob = ba.make_problem(cfg.b, cfg.h, cfg.g, cfg.d, cfg.mc, cfg.md, cfg.torch_dtype, inp.scale,
                           kv_dtype=inp.Kc.dtype, k_scale=inp.k_scale, v_scale=inp.v_scale)
    G = len(ba.ba_plan_ctas(prob)) - 1
    buf = torch.zeros(G * 1024, dtype=torch.int64, device="cuda")
    out = torch.empty_like(inp.q)
    ws = ba.alloc_workspace(prob, "cuda")

    def step():
        ba.bifurcated_attn_decode(inp.q, inp.Kc, inp.Vc, inp.Kd, inp.Vd, inp.lens, out,
                                  scale=inp.scale, workspace=ws, k_scale=inp.k_scale,
                                  v_scale=inp.v_scale)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    lib = ba.load_library()
    lib.ba_set_trace_buffer(buf.data_ptr())
    step()
    torch.cuda.synchronize()
    lib.ba_set_trace_buffer(None)
    tr = buf.view(G, 1024).cpu().tolist()
    mask = (1 << 56) - 1

    def t(v):
        return (v & mask) / 1e3 if v else None  # us

    t0 = min(t(r[250]) for r in tr if r[250])
    ph = {k: [] for k in ("pdl_wait", "to_first_S", "stream", "main_end", "barrier_wait", "merge",
                          "total")}
    sm_gap, sm_busy, vote, p_write, qk_lat = [], [], [], [], []
    by_kind = {"ctx": {"busy": [], "gap": [], "tile": []}, "dec": {"busy": [], "gap": [], "tile": []}}
    cs_tab = ba.ba_plan_ctas(prob)
    Tc_ = cfg.g * (-(-cfg.b * cfg.p // 32)) * (-(-cfg.mc // 128)) if cfg.b * cfg.p < 64 else 0
    abs_t = {"first_S": [], "main_end": [], "barrier_out": [], "merge_done": [], "segments": []}
    for r in tr:
        start, pdl, mend, bout, mdone = (t(r[s]) for s in (250, 254, 251, 252, 253))
        if not (start and mend and bout and mdone):
            continue
        sm = [(r[k] >> 56, t(r[k])) for k in range(256) if r[k]]
        s_ready = [x for tag, x in sm if tag == 20]
        voted = [x for tag, x in sm if tag in (21, 22)]
        handed = [x for tag, x in sm if tag == 23]
        abs_t["main_end"].append(mend - t0)
        abs_t["barrier_out"].append(bout - t0)
        abs_t["merge_done"].append(mdone - t0)
        abs_t["segments"].append(sum(1 for tag, _ in sm if tag == 4))
        if s_ready:
            abs_t["first_S"].append(s_ready[0] - t0)
        ph["pdl_wait"].append(pdl - start)
        if s_ready:
            ph["to_first_S"].append(s_ready[0] - pdl)
            ph["stream"].append(mend - s_ready[0])
        ph["main_end"].append(mend - t0)
        ph["barrier_wait"].append(bout - mend)
        ph["merge"].append(mdone - bout)
        ph["total"].append(mdone - t0)
        n = min(len(s_ready), len(voted), len(handed))
        kidx = tr.index(r)
        kind = None
        if cs_tab[kidx + 1] <= Tc_:
            kind = "ctx"
        elif cs_tab[kidx] >= Tc_:
            kind = "dec"
        if kind:
            pw0 = [x for tag, x in sm if tag == 27]  # before the P-slot wait (PV(u-npb) done)
            pw1 = [x for tag, x in sm if tag == 28]  # after it
            n2 = min(len(s_ready), len(handed), len(voted), len(pw0), len(pw1))
            for k in range(1, n2 - 1):
                by_kind[kind]["busy"].append(handed[k] - s_ready[k])
                by_kind[kind]["gap"].append(s_ready[k + 1] - handed[k])
                by_kind[kind]["tile"].append(s_ready[k + 1] - s_ready[k])
                by_kind[kind].setdefault("to_vote", []).append(voted[k] - s_ready[k])
                by_kind[kind].setdefault("vote_to_pwait", []).append(pw0[k] - voted[k])
                by_kind[kind].setdefault("pslot_wait", []).append(pw1[k] - pw0[k])
                by_kind[kind].setdefault("pwrite_to_handed", []).append(handed[k] - pw1[k])
        for k in range(n):
            vote.append(voted[k] - s_ready[k])
            p_write.append(handed[k] - voted[k])
            sm_busy.append(handed[k] - s_ready[k])
            if k + 1 < len(s_ready):
                sm_gap.append(s_ready[k + 1] - handed[k])
        qk_issued = [t(r[512 + u]) for u in range(256) if r[512 + u]]
        for u in range(min(len(qk_issued), len(s_ready))):
            qk_lat.append(s_ready[u] - qk_issued[u])
    # per-CTA regression of the main-loop end on its context / decode tile counts
    cs = ba.ba_plan_ctas(prob)
    Tc = cfg.g * (-(-cfg.b * cfg.p // 32)) * (-(-cfg.mc // 128)) if cfg.b * cfg.p < 64 else 0
    import numpy as np
    X, y = [], []
    for k, r in enumerate(tr):
        if r[251] and r[250]:
            nc = max(0, min(cs[k + 1], Tc) - cs[k])
            nd = (cs[k + 1] - cs[k]) - nc
            X.append([1.0, nc, nd])
            y.append(t(r[251]) - t0)
    per_cta = [[int(X[k][1]), int(X[k][2]), round(y[k], 2)] for k in range(len(X))]
    coef = np.linalg.lstsq(np.array(X), np.array(y), rcond=None)[0].tolist() if len(X) > 3 else None
    # dynamic CUDA-core decode columns (tags 39-43 of softmax thread 128)
    dyn = {"static_end": [], "cols": [], "tile_compute": [], "tile_wait": [], "col_head": [],
           "col_tail": [], "first_col": [], "last_col_end": []}
    for r in tr:
        sm = [(r[k] >> 56, t(r[k])) for k in range(256) if r[k]]
        se = [x for tag, x in sm if tag == 39]
        if not se:
            continue
        dyn["static_end"].append(se[0] - t0)
        dyn["cols"].append(sum(1 for tag, _ in sm if tag == 40))
        prev, prev_tag = None, None
        for tag, x in sm:
            if tag == 40 and prev_tag is not None:
                dyn.setdefault("col_gap", []).append(x - prev)
            if tag == 41 and prev is not None:
                (dyn["col_head"] if prev_tag == 40 else dyn["tile_wait"]).append(x - prev)
            if tag == 42 and prev_tag == 41:
                dyn["tile_compute"].append(x - prev)
            if tag == 43 and prev_tag == 42:
                dyn["col_tail"].append(x - prev)
            if tag == 40 and not dyn["first_col"] or (tag == 40 and prev_tag == 39):
                dyn["first_col"].append(x - t0)
            if tag == 43:
                last = x
            if tag in (39, 40, 41, 42, 43):
                prev, prev_tag = x, tag
        if any(tag == 43 for tag, _ in sm):
            dyn["last_col_end"].append(last - t0)
    dyn_sum = {k: [round(min(v), 3), med(v), round(max(v), 3), len(v)] for k, v in dyn.items() if v}
    # pipeline start: first TMA issue (producer slot 256), first K landed (QK slot 384),
    # first QK issued (512), first S ready (softmax tag 20); second/third TMA issue
    ramp = {"p_range": [], "p_seg0": [], "p_q_issued": [], "pdl": [], "tma0": [], "tma1": [], "tma2": [],
            "k0_landed": [], "k1_landed": [], "qk0": [], "s0": []}
    for r in tr:
        if not r[250]:
            continue
        for key, slot in (("p_range", 240), ("p_seg0", 241), ("p_q_issued", 242), ("pdl", 254),
                          ("tma0", 256), ("tma1", 257), ("tma2", 258), ("k0_landed", 384),
                          ("k1_landed", 385), ("qk0", 512)):
            if r[slot]:
                ramp[key].append(t(r[slot]) - t0)
        s20 = [t(r[k]) for k in range(256) if r[k] and r[k] >> 56 == 20]
        if s20:
            ramp["s0"].append(s20[0] - t0)
    ramp_sum = {k: [round(min(v), 3), med(v), round(max(v), 3)] for k, v in ramp.items() if v}
    before = [t(r[249]) - t0 for r in tr if r[249]]
    after = [t(r[248]) - t0 for r in tr if r[248]]
    res = {"config": name, "main_end_fit_us": {"const": coef[0], "per_ctx_tile": coef[1],
                                               "per_dec_tile": coef[2]} if coef else None,
           "per_cta_ctx_dec_mainend": per_cta,
           "pure_cta_tile_us_median": {k: {q: med(v) for q, v in d.items()} for k, d in by_kind.items()},
           "barrier_atomic_issue_min_med_max": [round(min(before), 2), med(before), round(max(before), 2)] if before else None,
           "barrier_atomic_return_min_med_max": [round(min(after), 2), med(after), round(max(after), 2)] if after else None, "plan": ba.ba_plan_string(prob), "ctas": G,
           "phases_us_median": {k: med(v) for k, v in ph.items()},
           "phases_us_max": {k: round(max(v), 3) if v else None for k, v in ph.items()},
           "per_tile_us_median": {"S_ready_to_vote": med(vote), "vote_to_P_handed": med(p_write),
                                  "softmax_busy": med(sm_busy), "P_handed_to_next_S": med(sm_gap),
                                  "QK_issue_to_S_ready": med(qk_lat)},
           "abs_us_min_med_max": {k: [round(min(v), 2), med(v), round(max(v), 2)] if v else None
                                  for k, v in abs_t.items()},
           "dyn_min_med_max_n": dyn_sum,
           "ramp_min_med_max": ramp_sum,
           "tiles_per_cta_median": med([len([1 for k in range(256) if r[k] and r[k] >> 56 == 20])
                                        for r in tr])}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["mha7b_b32", "mha7b_b32_fp8"]:
        run(nm)
