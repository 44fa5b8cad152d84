"""Summarise an ncu report (and optionally a launch-list CSV) into profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_c2_full.md \
      [--launches gpurun_out/launches.csv] [--traffic-config c2]

Writes a markdown summary with the metrics the roofline needs (duration, DRAM
bytes, throughput %, IPC, occupancy, top stall reasons per kernel) and, with
--traffic-config, records dram bytes per launch of the scan kernel into
profiles/traffic.json (read by bench.py's roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (active)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__inst_executed_pipe_fma.sum", "fma-pipe warp instr"),
    ("smsp__inst_executed_pipe_fp32.sum", "fp32 warp instr"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--traffic-config")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    hdr, units, rows = raw(a.report)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary: {os.path.basename(a.report)} {a.title}", ""]
    traffic = {}
    for r in rows:
        name = r[col["Kernel Name"]]
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k, label in KEYS:
            if k in col:
                lines.append(f"| {label} (`{k}`) | {r[col[k]]} | {units[col[k]]} |")
        try:
            rd = float(r[col["dram__bytes_read.sum"]].replace(",", ""))
            wr = float(r[col["dram__bytes_write.sum"]].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= mult.get(units[col["dram__bytes_read.sum"]], 1)
            wr *= mult.get(units[col["dram__bytes_write.sum"]], 1)
            lines.append(f"| dram read+write per launch | {rd + wr:.0f} | byte |")
            if "scan_kernel" in name or "narrow_kernel" in name:
                traffic["scan"] = rd + wr
        except (KeyError, ValueError):
            pass
        stalls = {h: r[i] for h, i in col.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
        vals = []
        for h, v in stalls.items():
            try:
                vals.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1
        top = sorted(vals, reverse=True)[:6]
        lines.append("")
        lines.append("Top stall reasons (pc sampling): " + ", ".join(f"{n} {v / tot * 100:.1f}%" for v, n in top))
        lines.append("")
    if a.launches:
        with open(a.launches) as f:
            txt = [l for l in f if not l.startswith("==")]
        rr = list(csv.reader(txt))
        h = rr[0]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        agg = collections.OrderedDict()
        for row in rr[1:]:
            n = row[ki].split("(")[0]
            agg.setdefault(n, []).append(float(row[vi].replace(",", "")))
        lines.append("## launch list (gpu__time_duration.sum, ns; cold-cache, serialised)")
        lines.append("")
        lines.append("| kernel | launches | mean ns | share of listed time |")
        lines.append("|---|---|---|---|")
        tot = sum(sum(v) for v in agg.values())
        for n, v in agg.items():
            lines.append(f"| {n} | {len(v)} | {sum(v) / len(v):.0f} | {sum(v) / tot * 100:.1f}% |")
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic_config and traffic:
        p = os.path.join(os.path.dirname(a.out), "traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[a.traffic_config] = traffic
        json.dump(d, open(p, "w"), indent=1)
    print(a.out)


if __name__ == "__main__":
    main()
