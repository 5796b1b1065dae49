"""Per-warp timeline of one fused decode (PBVD_EXP_TIMING build): start,
forward end, traceback end per warp (globaltimer ns), summarised."""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import synth
import paper_1608_00066_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else synth.CONFIGS[cfg]["n_info"]
c = synth.CONFIGS[cfg]
code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"], punct, c["hard"], device="cuda")
dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct)
dec.decode(llr, n)
torch.cuda.synchronize()
os.environ["PBVD_TIMING_DUMP"] = "/tmp/pbvd_timing.bin"
dec.decode(llr, n)
torch.cuda.synchronize()
a = np.fromfile("/tmp/pbvd_timing.bin", dtype=np.uint64).reshape(-1, 32).astype(np.int64)
a = a[a[:, 0] > 0]
out = os.environ.get("PBVD_TIMING_SAVE")
if out:
    np.save(out, a)
t0 = a[:, 0].min()
st, fe, te, sm = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3, a[:, 3]
print(f"{cfg} n={n} warps={len(a)}  kernel span {te.max():.1f} us")
print(f"start: min {st.min():.1f} max {st.max():.1f} us")
print(f"fwd end: min {fe.min():.1f} p10 {np.percentile(fe,10):.1f} p50 {np.percentile(fe,50):.1f} p90 {np.percentile(fe,90):.1f} max {fe.max():.1f}")
tb = te - fe
print(f"tb dur: min {tb.min():.1f} p10 {np.percentile(tb,10):.1f} p50 {np.percentile(tb,50):.1f} p90 {np.percentile(tb,90):.1f} max {tb.max():.1f}")
fw = fe - st
print(f"fwd dur: min {fw.min():.1f} p50 {np.percentile(fw,50):.1f} max {fw.max():.1f}")
wc, cc, nch = a[:, 4], a[:, 5], a[:, 6]
ok = nch > 0
print(f"tb wait cycles/chunk: p50 {np.percentile(wc[ok]/nch[ok],50):.0f} p90 {np.percentile(wc[ok]/nch[ok],90):.0f}; "
      f"walk cycles/chunk: p50 {np.percentile(cc[ok]/nch[ok],50):.0f} p90 {np.percentile(cc[ok]/nch[ok],90):.0f}; chunks {np.median(nch[ok]):.0f}")
late = te > np.percentile(te, 75)
print(f"late warps: wait/chunk p50 {np.percentile((wc/np.maximum(nch,1))[late & ok],50):.0f} walk/chunk p50 {np.percentile((cc/np.maximum(nch,1))[late & ok],50):.0f}")
idx = np.argsort(te)[-6:]
for i in idx:
    print(f"  warp {i}: sm {sm[i]} start {st[i]:.1f} fwd_end {fe[i]:.1f} tb {tb[i]:.1f} us; wait/ch {wc[i]/max(nch[i],1):.0f} walk/ch {cc[i]/max(nch[i],1):.0f} cyc")
# per-SM warp counts vs forward duration
cnt = np.bincount(sm, minlength=148)
print("warps per SM histogram:", np.bincount(cnt))
for k in sorted(set(cnt[sm])):
    sel = cnt[sm] == k
    print(f"  SMs with {k} warps: fwd dur p50 {np.percentile(fw[sel],50):.1f} max {fw[sel].max():.1f}; tb p50 {np.percentile(tb[sel],50):.1f}")

# per SM sub-partition (%warpid % 4): warps sharing it vs their forward end
wid = a[:, 7]
key = sm * 4 + (wid % 4)
kc = np.bincount(key, minlength=148 * 4)
print("warps per sub-partition histogram:", np.bincount(kc))
for k in sorted(set(kc[key])):
    sel = kc[key] == k
    print(f"  sub-partitions with {k} warps: fwd end p10 {np.percentile(fe[sel],10):.1f} p50 {np.percentile(fe[sel],50):.1f} "
          f"p90 {np.percentile(fe[sel],90):.1f} max {fe[sel].max():.1f}; fwd dur p50 {np.percentile(fw[sel],50):.1f}")
# among 2-warp sub-partitions: spread by SM warp count
for k in sorted(set(cnt[sm])):
    sel = (cnt[sm] == k) & (kc[key] == 2)
    if sel.any():
        print(f"  2-warp sub-partitions on SMs with {k} warps: fwd end p50 {np.percentile(fe[sel],50):.1f} max {fe[sel].max():.1f}")
