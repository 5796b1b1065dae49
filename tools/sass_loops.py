"""List the loops (backward branches) of a kernel's SASS with their size and
op histogram: python tools/sass_loops.py lib.so name-substring [min_viaddmnmx]"""
import collections
import re
import subprocess
import sys

so, pat = sys.argv[1], sys.argv[2]
minv = int(sys.argv[3]) if len(sys.argv) > 3 else 32
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
for part in re.split(r'\n\s+Function : ', txt)[1:]:
    name = part.split('\n', 1)[0].strip()
    if pat not in name:
        continue
    ins = re.findall(r'/\*([0-9a-f]{4,})\*/\s+([^;]*);', part)
    ops = [(int(a, 16), t.strip()) for a, t in ins]
    addr2i = {a: i for i, (a, _) in enumerate(ops)}
    print(name[:100], "total instrs", len(ops))
    for i, (a, t) in enumerate(ops):
        m = re.search(r'BRA[^`]*`?\(?\.L_x_\d+\)?', t)
        tgt = re.search(r'0x([0-9a-f]+)', t) if 'BRA' in t else None
        if not tgt:
            continue
        ta = int(tgt.group(1), 16)
        if ta >= a or ta not in addr2i:
            continue
        seg = ops[addr2i[ta]:i + 1]
        c = collections.Counter()
        for _, x in seg:
            tok = x.split()
            op = tok[1] if tok[0].startswith('@') else tok[0]
            c[op] += 1
        nv = sum(v for k, v in c.items() if k.startswith('VIADDMNMX'))
        if nv < minv:
            continue
        print(f"  loop {ta:#x}-{a:#x}: {len(seg)} instrs, VIADDMNMX {nv}, {len(seg)/max(nv,1):.2f}/out: " +
              ", ".join(f"{k} {v}" for k, v in c.most_common(12)))
