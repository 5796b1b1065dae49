"""Op histogram of the hot loop (the cluster with the most VIADDMNMX) of a kernel."""
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
    ins = re.findall(r'/\*([0-9a-f]{4,})\*/\s+([^;]*);', part)
    ops = [(int(a, 16), t.strip()) for a, t in ins]
    idx = [k for k, (_, t) in enumerate(ops) if 'VIADDMNMX' in t]
    clusters, start, prev = [], idx[0], idx[0]
    for k in idx[1:]:
        if k - prev > 80:
            clusters.append((start, prev))
            start = k
        prev = k
    clusters.append((start, prev))
    a, b = max(clusters, key=lambda c: c[1] - c[0])
    # extend to the enclosing backward branch
    e = b
    while e < len(ops) and not (ops[e][1].startswith('BRA') or ' BRA ' in ops[e][1] or ops[e][1].startswith('@')
                                and 'BRA' in ops[e][1]):
        e += 1
    seg = ops[max(0, a - 40):e + 1]
    c = collections.Counter()
    for _, t in seg:
        tok = t.split()
        op = tok[1] if tok[0].startswith('@') else tok[0]
        c[op] += 1
    nv = sum(v for k, v in c.items() if k.startswith('VIADDMNMX'))
    print(name[:90])
    print(f"  loop instrs {len(seg)}  VIADDMNMX {nv}  instr/output {len(seg)/max(nv,1):.2f}")
    for k, v in c.most_common(40):
        print(f"    {k:28s} {v:5d}  {v/max(nv,1):.3f}/out")
