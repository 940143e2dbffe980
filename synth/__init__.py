"""Seeded synthetic inputs for the bifurcated decode step — shared by tests,
bench.py and smoke().

This module holds NO arithmetic of the method (no logits, softmax or value
products): only the workload shapes of BASELINE.json ``configs`` and seeded
random tensors with the paper's workload structure — one shared prefill
context KV (Kc, Vc) and ``b`` per-sample decode caches (Kd, Vd) of equal length
(single-context batch sampling, §3.2; uniform md,
PAPER.md:227).  Both the oracle and the CUDA path read the tensors it returns.

Recipe (DESIGN.md §"Inputs"): q, Kc, Vc, Kd, Vd ~ N(0, 1) drawn in fp32 with a
``torch.Generator`` seeded by ``seed`` and rounded to the config dtype;
``lens[i] = md`` for all i; ``md_cap = md``.  Stress variants scale or plant
values (``variant``) to exercise the LSE merge.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import torch


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    dtype: str  # "bf16" | "fp32"
    b: int
    h: int
    g: int
    d: int
    mc: int
    md: int
    kv: str = ""  # KV cache storage: "" = the dtype; "e4m3" = FP8 E4M3 codes + fp32 scales (R19)

    @property
    def kv_bytes(self) -> int:
        return 1 if self.kv == "e4m3" else self.elem_bytes

    @property
    def p(self) -> int:
        return self.h // self.g

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    def with_(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs", in order.  C2 is quoted at b=16 and b=32.
CONFIGS = {
    "tiny": Config("tiny", "fp32", b=4, h=2, g=2, d=16, mc=32, md=4),
    "mha7b_b16": Config("mha7b_b16", "bf16", b=16, h=32, g=32, d=128, mc=8192, md=256),
    "mha7b_b32": Config("mha7b_b32", "bf16", b=32, h=32, g=32, d=128, mc=8192, md=256),
    "gqa": Config("gqa", "bf16", b=64, h=32, g=8, d=128, mc=16384, md=512),
    "mqa": Config("mqa", "bf16", b=128, h=48, g=1, d=128, mc=8192, md=256),
    "long": Config("long", "bf16", b=256, h=64, g=64, d=128, mc=32768, md=1024),
    # f4: the C2b workload with an FP8 (E4M3) KV cache (FAQ 5)
    "mha7b_b32_fp8": Config("mha7b_b32_fp8", "bf16", b=32, h=32, g=32, d=128, mc=8192, md=256,
                            kv="e4m3"),
}

SEED_BASE = 20240313


def seed_for(name: str) -> int:
    return SEED_BASE + list(CONFIGS).index(name) if name in CONFIGS else SEED_BASE + 97


@dataclasses.dataclass
class Inputs:
    q: torch.Tensor   # [b][h][d]
    Kc: torch.Tensor  # [g][mc][d]
    Vc: torch.Tensor  # [g][mc][d]
    Kd: torch.Tensor  # [b][g][md_cap][d]
    Vd: torch.Tensor  # [b][g][md_cap][d]
    lens: torch.Tensor  # int32 [b]
    scale: float      # the fp32 logit scale (1/sqrt(d) unless overridden)
    k_scale: float = 1.0  # FP8 KV (cfg.kv == "e4m3"): K = code value * k_scale (fp32)
    v_scale: float = 1.0  #                            V = code value * v_scale


def make_inputs(cfg: Config, seed: int, device="cpu", variant: str = "normal",
                md_cap: Optional[int] = None, lens=None, scale: Optional[float] = None,
                gen_dtype=torch.float32, n_tok: int = 1) -> Inputs:
    """Seeded N(0,1) inputs shaped like ``cfg``.

    variant: "normal" | "peaky" (q*8) | "ctx_dom" (Kc*4) | "dec_dom" (Kd*4) |
             "ragged" (lens ~ U[0, md]) | "equal" (all samples identical q/Kd/Vd) |
             "planted_ctx" / "planted_dec" (one key per row made dominant).
    n_tok > 1: a multi-token step, q [b][h][n_tok][d] (App. G draft tokens).
    """
    md_cap = cfg.md if md_cap is None else md_cap
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    dt = cfg.torch_dtype

    def randn(*shape):
        return torch.randn(*shape, generator=gen, device=device, dtype=gen_dtype).to(dt)

    q = randn(cfg.b, cfg.h, n_tok, cfg.d) if n_tok > 1 else randn(cfg.b, cfg.h, cfg.d)
    if n_tok > 1 and variant.startswith("planted"):
        raise ValueError("planted variants are single-token")
    Kc = randn(cfg.g, cfg.mc, cfg.d)
    Vc = randn(cfg.g, cfg.mc, cfg.d)
    Kd = randn(cfg.b, cfg.g, md_cap, cfg.d)
    Vd = randn(cfg.b, cfg.g, md_cap, cfg.d)
    if lens is None:
        lens_t = torch.full((cfg.b,), min(cfg.md, md_cap), dtype=torch.int32, device=device)
    else:
        lens_t = torch.as_tensor(lens, dtype=torch.int32).to(device)
    if variant == "peaky":
        q = (q.float() * 8).to(dt)
    elif variant == "ctx_dom":
        Kc = (Kc.float() * 4).to(dt)
    elif variant == "dec_dom":
        Kd = (Kd.float() * 4).to(dt)
    elif variant == "ragged":
        lens_t = torch.randint(0, md_cap + 1, (cfg.b,), generator=gen, device=device,
                               dtype=torch.int64).to(torch.int32)
    elif variant == "equal":
        q = q[:1].expand_as(q).contiguous()
        Kd = Kd[:1].expand_as(Kd).contiguous()
        Vd = Vd[:1].expand_as(Vd).contiguous()
    elif variant in ("planted_ctx", "planted_dec"):
        # Row (i, j) gets q = 16 * K_t* / |K_t*| * sqrt(d) for one key t*, so its
        # logit dominates; t* is in the context (planted_ctx) or decode branch.
        p = cfg.p
        qf = q.float()
        for i in range(cfg.b):
            for j in range(cfg.h):
                c = j // p
                if variant == "planted_ctx" or int(lens_t[i]) == 0:
                    t = (7 * i + 3 * j) % cfg.mc
                    k = Kc[c, t].float()
                else:
                    t = (5 * i + j) % int(lens_t[i])
                    k = Kd[i, c, t].float()
                qf[i, j] = 16.0 * k / k.norm().clamp_min(1e-6) * cfg.d ** 0.5
        q = qf.to(dt)
    elif variant != "normal":
        raise ValueError(variant)
    if scale is None:
        scale = float(torch.tensor(1.0 / cfg.d ** 0.5, dtype=torch.float32))
    if cfg.kv == "e4m3":
        # per-tensor-kind scales (one for K, one for V, shared by context and
        # decode caches): amax / 448 in fp32, then the E4M3 codes of x / scale
        def amax(a, b_):
            m = a.float().abs().max()
            if b_.numel():
                m = torch.maximum(m, b_.float().abs().max())
            return m

        ks = amax(Kc, Kd) / 448.0
        vs = amax(Vc, Vd) / 448.0
        ks = torch.where(ks > 0, ks, torch.ones_like(ks))
        vs = torch.where(vs > 0, vs, torch.ones_like(vs))
        f8 = torch.float8_e4m3fn
        Kc, Kd = (Kc.float() / ks).to(f8), (Kd.float() / ks).to(f8)
        Vc, Vd = (Vc.float() / vs).to(f8), (Vd.float() / vs).to(f8)
        return Inputs(q, Kc, Vc, Kd, Vd, lens_t, scale, float(ks), float(vs))
    return Inputs(q, Kc, Vc, Kd, Vd, lens_t, scale)


def alg_bytes(cfg: Config, lens_sum: Optional[int] = None) -> int:
    """Algorithmic bytes of one step (Eq. 6 PAPER.md:287 x 2
    tensors x element bytes, plus the q/out terms of App. E.2):
      2*e_kv*d*g*(mc + sum_i lens[i]) + 2*e*b*h*d   (e_kv = 1 for an FP8 KV cache)."""
    e, ekv = cfg.elem_bytes, cfg.kv_bytes
    ls = cfg.b * cfg.md if lens_sum is None else lens_sum
    return 2 * ekv * cfg.d * cfg.g * (cfg.mc + ls) + 2 * e * cfg.b * cfg.h * cfg.d


def alg_flops(cfg: Config, lens_sum: Optional[int] = None) -> int:
    """4*b*h*(mc+md)*d summed over samples: two contractions, 2 FLOP per MAC
    ('same FLOPs')."""
    ls = cfg.b * cfg.md if lens_sum is None else lens_sum
    return 4 * cfg.h * cfg.d * (cfg.b * cfg.mc + ls)
