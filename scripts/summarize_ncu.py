"""Summarise ncu evidence into profiles/<round>/ (run here, after gpurun).

usage: python scripts/summarize_ncu.py r01 gpurun_out/launches_r01.csv \
           b32=gpurun_out/prof_r01_b32.ncu-rep b16=gpurun_out/prof_r01_b16.ncu-rep

Writes profiles/<round>/launches.md (per-kernel launch list of the bench
command: cold, serialised ncu times and DRAM bytes), ncu_<tag>.md (key
metrics of one `--set full` capture) and updates profiles/traffic.json
(config -> dram read+write bytes per launch of the fused kernel)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG2CFG = {"b32": "mha7b_b32", "b16": "mha7b_b16", "gqa": "gqa", "mqa": "mqa", "long": "long",
           "fp8": "mha7b_b32_fp8", "long_rows2": "long_rows2"}
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tc.sum", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu_csv(rep, page, extra=()):
    """Rows of one ncu page: from a report (.ncu-rep) or from its exported
    CSV pages <stem>.<page>.csv (written on the GPU box, where the reports
    are too large to bring back)."""
    if not rep.endswith(".ncu-rep"):
        with open(f"{rep}.{page}.csv") as f:
            return [r for r in csv.reader(f) if r and not r[0].startswith("==")]
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(out.splitlines()))


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    rows = [r for r in rows[start:] if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    agg = {}
    for r in rows[1:]:
        name = r[ix["Kernel Name"]]
        name = (name.split("(")[0][:60] if any(k in name for k in ("bif", "merge", "fma", "ctx_rows"))
                else name[:40])
        v = float(r[ix["Metric Value"]].replace(",", ""))
        agg.setdefault(name, {}).setdefault(r[ix["Metric Name"]], []).append(v)
    return agg


def main():
    rnd, lcsv = sys.argv[1], sys.argv[2]
    reps = dict(a.split("=", 1) for a in sys.argv[3:])
    od = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(od, exist_ok=True)
    agg = launches(lcsv)
    lines = [f"# Launch list ({rnd}) — `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum --clock-control none` over the bench command", "",
             "Cold, serialised per-launch numbers (ncu replays each kernel): the SHARE of the step "
             "is what transfers to the bench, not the absolute time.", "",
             "| kernel | launches | mean time (us) | DRAM read / launch (MB) | DRAM write / launch (MB) |",
             "|---|---|---|---|---|"]
    fused = None
    for k, d in agg.items():
        t = d.get("gpu__time_duration.sum", [0])
        rd = d.get("dram__bytes_read.sum", [0])
        wr = d.get("dram__bytes_write.sum", [0])
        mean = lambda v: sum(v) / len(v)
        lines.append(f"| `{k}` | {len(t)} | {mean(t) / 1e3:.2f} | {mean(rd) / 1e6:.2f} | {mean(wr) / 1e6:.2f} |")
        if "bif_tc_kernel" in k:
            fused = (mean(t), mean(rd), mean(wr))
    open(os.path.join(od, "launches.md"), "w").write("\n".join(lines) + "\n")
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for tag, rep in reps.items():
        det = ncu_csv(rep, "details")
        h = det[0]
        ix = {k: i for i, k in enumerate(h)}
        kern = det[1][ix["Kernel Name"]] if len(det) > 1 else "?"
        out = [f"# ncu --set full: {kern} ({tag}, config {TAG2CFG.get(tag, tag)}, {rnd})", "",
               "| section | metric | value |", "|---|---|---|"]
        for r in det[1:]:
            if r[ix["Metric Name"]] in KEYS:
                out.append(f"| {r[ix['Section Name']]} | {r[ix['Metric Name']]} | "
                           f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]} |")
        raw = ncu_csv(rep, "raw")
        d = dict(zip(raw[0], raw[2])) if len(raw) > 2 else {}
        units = dict(zip(raw[0], raw[1])) if len(raw) > 1 else {}
        out += ["", "| raw metric | value |", "|---|---|"]
        for k in RAW:
            out.append(f"| {k} | {d.get(k)} {units.get(k, '')} |")
        st = [(float(v.replace(",", "")), k) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
              and v not in ("", "n/a")]
        out += ["", "Warp-state samples (all warps, incl. idle role lanes at the final barrier):", ""]
        out += [f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {int(v)}"
                for v, k in sorted(st, reverse=True)[:8]]
        open(os.path.join(od, f"ncu_{tag}.md"), "w").write("\n".join(out) + "\n")

        def mb(key):
            v = float(d.get(key, "0").replace(",", ""))
            u = units.get(key, "byte")
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[TAG2CFG.get(tag, tag)] = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
    json.dump(traffic, open(tj, "w"), indent=1)
    print(open(os.path.join(od, "launches.md")).read())
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
