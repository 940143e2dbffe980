set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for swg in 1 2; do
  BIFATTN_SWG=$swg python scripts/exp_split.py
  BIFATTN_SWG=$swg python scripts/exp_trace.py mha7b_b32
done
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2403_08845_b200 as ba
from synth import CONFIGS, make_inputs
cfg = CONFIGS["mha7b_b32"]
s = make_inputs(cfg, 1, device="cuda")
K = torch.cat([s.Kc.unsqueeze(0).expand(cfg.b, -1, -1, -1), s.Kd], dim=2).contiguous()
V = torch.cat([s.Vc.unsqueeze(0).expand(cfg.b, -1, -1, -1), s.Vd], dim=2).contiguous()
o = torch.empty_like(s.q)
f = lambda: ba.replicated_attn_decode(s.q, K, V, s.lens, cfg.mc, o, scale=s.scale)
for _ in range(3): f()
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): f()
b.record(); torch.cuda.synchronize()
us = a.elapsed_time(b) / 10 * 1e3
print("replicated us", us, "GB/s", 4.43e9 / us / 1e3)
PY
