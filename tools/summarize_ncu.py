"""Summarise an ncu report (--set full) into JSON + markdown for profiles/.

    python tools/summarize_ncu.py gpurun_out/fwd_full.ncu-rep profiles/r01_fwd_c2
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "sm__inst_executed_pipe_tma.sum", "smsp__inst_executed_op_shfl.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def sass_hist(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    iE = hdr.index("Instructions Executed")
    hist = {}
    for r in rows[2:]:
        toks = r[1].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        hist[op] = hist.get(op, 0) + int(r[iE] or 0)
    return dict(sorted(hist.items(), key=lambda kv: -kv[1])[:40])


def main(rep, prefix):
    d = raw(rep)
    out = {}
    for k in KEYS:
        if k in d:
            v, u = d[k]
            try:
                out[k] = {"value": float(v.replace(",", "")), "unit": u}
            except ValueError:
                out[k] = {"value": v, "unit": u}
    stalls = {}
    for k, (v, u) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                fv = float(v)
            except ValueError:
                continue
            if fv >= 0.02:
                stalls[k.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", "")] = fv
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    out["sass_executed_histogram"] = sass_hist(rep)
    rb = out.get("dram__bytes_read.sum", {}).get("value")
    wb = out.get("dram__bytes_write.sum", {}).get("value")
    unit = out.get("dram__bytes_read.sum", {}).get("unit", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    if rb is not None and wb is not None:
        out["dram_bytes_per_launch"] = (rb + wb) * scale
    out["source_report"] = rep
    with open(prefix + ".json", "w") as f:
        json.dump(out, f, indent=1)
    lines = [f"# ncu summary: {rep}", ""]
    for k in KEYS:
        if k in out:
            lines.append(f"- `{k}`: {out[k]['value']} {out[k]['unit']}")
    lines.append("- stalls per issue: " + ", ".join(f"{k} {v:.2f}" for k, v in stalls.items()))
    lines.append("- executed SASS (top): " + ", ".join(
        f"{k} {v}" for k, v in list(out["sass_executed_histogram"].items())[:20]))
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
