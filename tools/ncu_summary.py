"""Summarise an ncu --set full report (and an optional launch-list CSV) into profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <out_prefix> [launches.csv]
Writes <out_prefix>.md (human summary) and <out_prefix>.json (machine-readable metrics per
kernel launch), e.g. profiles/r01_ncu_c5s.{md,json}."""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

WANT = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum",
    "smsp__inst_executed.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__sass_inst_executed_op_global_red.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
]
STALL_PREFIX = "smsp__average_warps_issue_stalled_"
STALL_SUFFIX = "_per_issue_active.ratio"


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    launches_csv = sys.argv[3] if len(sys.argv) > 3 else None
    hdr, units, data = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    kernels = []
    for row in data:
        k = {"kernel": row[idx["Kernel Name"]] if "Kernel Name" in idx else row[4]}
        for m in WANT:
            if m in idx:
                k[m] = row[idx[m]]
        stalls = {}
        for h, i in idx.items():
            if h.startswith(STALL_PREFIX) and h.endswith(STALL_SUFFIX):
                try:
                    stalls[h[len(STALL_PREFIX):-len(STALL_SUFFIX)]] = float(row[i].replace(",", ""))
                except ValueError:
                    pass
        k["stall_top"] = sorted(((n, round(v, 3)) for n, v in stalls.items()),
                                key=lambda t: -t[1])[:8]
        kernels.append(k)
    summary = {"report": rep, "kernels": kernels}
    if launches_csv:
        per = defaultdict(lambda: [0, 0.0])
        with open(launches_csv) as f:
            lines = [l for l in f if not l.startswith("==")]
        for r in csv.DictReader(io.StringIO("".join(lines))):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].replace("void ", "").split("(")[0]
            name = name.replace("(anonymous namespace)", "").replace("<unnamed>", "")
            base = name.split("<")[0]
            name = base.split("::")[-1] + (("<" + name.split("<", 1)[1]) if "<" in name else "")
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
                      "nsecond": 1}.get(unit, 1)
            per[name][0] += 1
            per[name][1] += ns
        tot = sum(v[1] for v in per.values()) or 1.0
        summary["launch_list"] = {k: {"launches": v[0], "total_ms": v[1] / 1e6,
                                      "share": v[1] / tot} for k, v in
                                  sorted(per.items(), key=lambda kv: -kv[1][1])}
    with open(prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu summary of `{rep}`\n\n")
        for k in kernels:
            f.write(f"## {k['kernel'][:120]}\n\n")
            for m in WANT:
                if m in k:
                    f.write(f"- `{m}` = {k[m]}\n")
            f.write(f"- warps stalled per issue, by reason (top): {k['stall_top']}\n\n")
        if "launch_list" in summary:
            f.write("## launch list (ncu --metrics gpu__time_duration.sum, serialised, "
                    "cold-cache: compare shares)\n\n| kernel | launches | total ms | share |\n"
                    "|---|---|---|---|\n")
            for n, v in summary["launch_list"].items():
                f.write(f"| {n} | {v['launches']} | {v['total_ms']:.3f} | {v['share']:.3%} |\n")
    print("wrote", prefix + ".md", prefix + ".json")


if __name__ == "__main__":
    main()
