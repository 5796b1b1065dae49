"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel.

    python tools/summarize_launches.py gpurun_out/launches.csv profiles/r01_launches_c2_summary.json
"""
import csv
import json
import sys


def main(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[0] != "ID"]
    agg = {}
    for r in rows:
        name, val = r[4], float(r[14].replace(",", ""))
        if "fwd_kernel" in name:
            # template args <Cfg<...>, FUSED, MIRROR> (mangled, bool or int form)
            tail = name.split(">, ")[-1] if ">, " in name else ""
            fused = ("ELb1E" in name or ", true>" in name or "(bool)1" in name or
                     tail.startswith("1,") or tail.startswith("true"))
            key = "fwd_kernel<fused>" if fused else "fwd_kernel"
        elif "tb_kernel" in name:
            key = "tb_kernel"
        elif "acs_probe" in name:
            key = "acs_probe"
        else:
            key = "other(torch: synth/flush)"
        a = agg.setdefault(key, {"launches": 0, "total_ns": 0.0})
        a["launches"] += 1
        a["total_ns"] += val
    dec = sum(v["total_ns"] for k, v in agg.items() if "kernel" in k)
    for k, v in agg.items():
        v["mean_ns"] = v["total_ns"] / v["launches"]
        if "kernel" in k:
            v["share_of_decode"] = v["total_ns"] / dec
    agg["note"] = ("ncu --metrics gpu__time_duration.sum --clock-control none over "
                   "`bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline` (cold-cache, "
                   "serialised launches: compare shares, not absolutes)")
    json.dump(agg, open(dst, "w"), indent=1)
    print(json.dumps(agg, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
