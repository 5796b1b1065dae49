"""Per-code-region totals of executed instructions and stall samples from an
ncu report's SASS source page (which code is hot, where no-instruction
stalls land): python tools/ncu_regions.py rep.ncu-rep [bucket_bytes]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg = {}
base = None
tot = {"exec": 0, "samples": 0, "noinst": 0}
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        a = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    a -= base
    ex = float(r[ix["Instructions Executed"]] or 0)
    sm = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ni = float(r[ix["stall_no_inst"]] or 0)
    b = a // bucket
    e = agg.setdefault(b, [0, 0, 0])
    e[0] += ex; e[1] += sm; e[2] += ni
    tot["exec"] += ex; tot["samples"] += sm; tot["noinst"] += ni
print(f"total exec {tot['exec']:.4g}  samples {tot['samples']:.0f}  no_inst {tot['noinst']:.0f}")
for b in sorted(agg):
    ex, sm, ni = agg[b]
    if sm < 0.002 * tot["samples"] and ex < 0.002 * tot["exec"]:
        continue
    print(f"  {b * bucket:#07x}-{(b + 1) * bucket:#07x}: exec {100 * ex / tot['exec']:5.1f}%  "
          f"samples {100 * sm / tot['samples']:5.1f}%  no_inst {100 * ni / max(1, tot['noinst']):5.1f}%")
