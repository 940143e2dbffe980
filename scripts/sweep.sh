# one bench line per BASELINE config (timed kernels only), for DESIGN.md / profiles
mkdir -p gpurun_out
for c in tiny mha7b_b16 mha7b_b32 gqa mqa long; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-replicated --soak 0.3 2>/dev/null | tail -1
done > gpurun_out/sweep.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], round(d["us_per_step"], 2), "us", round(d["value"], 1), d["unit"], d["config"].get("plan", "")[:90])
PY
