"""Summarise ncu captures from gpurun_out/ into profiles/ (tracked).

  python tools/ncu_summary.py <round_tag> <config>
writes profiles/<tag>_<config>_launches.csv (copy of the launch list), profiles/<tag>_<config>_ncu.md
and updates profiles/ncu_attention_summary.json (dram bytes per launch of k_paged_attn, read by bench.py).
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]


def raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        out.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return out


def to_bytes(val, unit):
    x = float(str(val).replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            x = float(r[vi].replace(",", ""))
            agg[r[ki].split("(")[0]].append(x / 1e3 if r[ui] == "ns" else x * (1e3 if r[ui] == "ms" else 1))
    return agg


def main():
    tag, cfg = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary {tag} / {cfg}", ""]
    lpath = os.path.join(OUT, f"launches_{cfg}.csv")
    if os.path.exists(lpath):
        shutil.copy(lpath, os.path.join(PROF, f"{tag}_{cfg}_launches.csv"))
        agg = launches(lpath)
        tot = sum(sum(v) for k, v in agg.items() if "cpa::" in k)
        md += ["## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)", "",
               "| kernel | launches | mean us | share of libcpa time |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            share = f"{sum(v) / tot:.1%}" if "cpa::" in k else "-"
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {share} |")
        md.append("")
    summ_path = os.path.join(PROF, "ncu_attention_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for kind in ("attn", "scores"):
        rep = os.path.join(OUT, f"prof_{kind}_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        rows = raw(rep)
        md += [f"## `--set full` capture: {kind} ({os.path.basename(rep)})", "", "| metric | value | unit |", "|---|---|---|"]
        for k in KEYS:
            if k in rows[0]:
                md.append(f"| {k} | {rows[0][k][0]} | {rows[0][k][1]} |")
        md.append("")
        if kind == "attn":
            rd = to_bytes(*rows[0]["dram__bytes_read.sum"])
            wr = to_bytes(*rows[0]["dram__bytes_write.sum"])
            summ[cfg] = {"dram_bytes_per_launch": rd + wr, "source": f"{tag} ncu --set full, k_paged_attn"}
    json.dump(summ, open(summ_path, "w"), indent=1)
    open(os.path.join(PROF, f"{tag}_{cfg}_ncu.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
