"""Per-chunk forward timeline of a PBVD_EXP_TIMING dump (exp_timing.py with
PBVD_TIMING_SAVE): chunk durations of warps alone on / sharing an SM
sub-partition, and the issue split inside sharing pairs."""
import sys
import numpy as np
a = np.load(sys.argv[1])
t0 = a[:, 0].min()
st, fe, te = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
sm, wid = a[:, 3], a[:, 7]
ch = (a[:, 8:28] - t0) / 1e3
ok = (a[:, 8:28] > 0).all(axis=1)
d = np.diff(np.concatenate([st[:, None], ch], axis=1), axis=1)
key = sm * 4 + (wid % 4)
kc = np.bincount(key, minlength=int(key.max()) + 1)
print(f"warps {len(a)}, kernel end {te.max():.1f} us")
for k in (1, 2, 3):
    sel = (kc[key] == k) & ok
    if sel.any():
        print(f"{k} warp(s) per sub-partition ({sel.sum()} warps): chunk 0 {np.median(d[sel, 0]):.2f} us, "
              f"chunks 1-13 median {np.median(d[sel, 1:14]):.2f} us, forward end p50 {np.median(fe[sel]):.1f} us")
sel = kc[key] == 2
ks = np.unique(key[sel])
fw = fe - st
pm = np.array([fw[key == k].mean() for k in ks])
pd = np.array([np.ptp(fw[key == k]) for k in ks])
print(f"pairs: mean forward {np.median(pm):.1f} us (p10 {np.percentile(pm, 10):.1f}, p90 {np.percentile(pm, 90):.1f}); "
      f"first-to-second finish gap p50 {np.median(pd):.1f} us")
