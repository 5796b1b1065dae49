"""Single-warp cycle model of a kernel's hot loop from the SASS control words:
sum of the stall fields (bits 105..108 of each 128-bit instruction) over the
loop body, per packed output (VIADDMNMX).

    python tools/sass_stalls.py paper_1608_00066_b200/libpbvd.so <function-substring>
"""
import collections
import re
import subprocess
import sys

so, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
for part in re.split(r'\n\s+Function : ', txt)[1:]:
    name = part.split('\n', 1)[0].strip()
    if pat not in name:
        continue
    lines = part.split('\n')
    ins = []
    for i, ln in enumerate(lines):
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+([^;]*);\s+/\* (0x[0-9a-f]+) \*/', ln)
        if m and i + 1 < len(lines):
            m2 = re.search(r'/\* (0x[0-9a-f]+) \*/', lines[i + 1])
            hi = int(m2.group(1), 16) if m2 else 0
            ins.append((int(m.group(1), 16), m.group(2).strip(), hi))
    addr = [a for a, _, _ in ins]
    for k, (a, t, hi) in enumerate(ins):
        m = re.search(r'BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?(0x[0-9a-f]+)', t)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr:
            continue
        j = addr.index(tgt)
        seg = ins[j:k + 1]
        nv = sum(1 for _, t2, _ in seg if 'VIADDMNMX' in t2)
        if nv < 50:
            continue
        stall = sum((h >> 41) & 0xF for _, _, h in seg)
        yld = sum(1 for _, _, h in seg if not ((h >> 45) & 1))
        hist = collections.Counter((h >> 41) & 0xF for _, _, h in seg)
        print(f"{name[:70]}\n  loop {tgt:x}-{a:x}: {len(seg)} instr, {nv} outputs, "
              f"stall-sum {stall} cycles -> {stall / nv:.2f} cyc/out single warp "
              f"({len(seg) / nv:.2f} instr/out); stall histogram {dict(sorted(hist.items()))}")
