"""Experiment: end-to-end decode from pinned host memory with the kernel
reading the soft input over PCIe directly (zero-copy, UVA) and writing the
decoded bits straight into pinned host memory, against pbvd_decode_host
(staged H2D copies).  usage: exp_zerocopy.py [cfg] [lanes...]"""
import ctypes, statistics, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import synth
from paper_1608_00066_b200 import build
build.build()
import paper_1608_00066_b200 as P
from paper_1608_00066_b200 import _lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
lanes_list = [int(x) for x in sys.argv[2:]] or [0]
c = synth.CONFIGS[cfg]
code, punct = synth.CODES[c["code"]], synth.PUNCT[c["punct"]]
n = c["n_info"]
info, llr = synth.make_stream(code, n, c["ebn0"], c["seed"], punct, c["hard"], device="cuda")
llr_h = torch.empty(llr.shape, dtype=torch.int8, pin_memory=True)
llr_h.copy_(llr.cpu())
nb = (n + 7) // 8
out_h = torch.zeros(nb, dtype=torch.uint8, pin_memory=True)
L = _lib.load()
ref = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct).decode(llr, n).cpu()

def tm(fn, reps=15):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return statistics.median(ts)

t_h2d = tm(lambda: llr.copy_(llr_h, non_blocking=True))
print(f"{cfg}: H2D alone {t_h2d*1e3:.3f} ms ({llr.numel()/t_h2d/1e9:.1f} GB/s) -> bound {n/t_h2d/1e9:.2f} Gb/s")
for lanes in lanes_list:
    dec = P.Decoder(code["K"], code["polys"], c["D"], c["L"], punct=punct, lanes=lanes)
    t_host = tm(lambda: dec.decode_host(llr_h, n, out=out_h))
    ok_host = torch.equal(out_h, ref)
    s = torch.cuda.current_stream()
    def zc():
        rc = L.pbvd_decode(dec._h, llr_h.data_ptr(), llr_h.numel(), out_h.data_ptr(), n,
                           ctypes.c_void_p(s.cuda_stream))
        assert rc == 0, L.pbvd_last_error(dec._h)
    out_h.zero_()
    t_zc = tm(zc)
    ok_zc = torch.equal(out_h, ref)
    # zero-copy input, device output + D2H
    out_d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    def zc_in():
        rc = L.pbvd_decode(dec._h, llr_h.data_ptr(), llr_h.numel(), out_d.data_ptr(), n,
                           ctypes.c_void_p(s.cuda_stream))
        assert rc == 0
        out_h.copy_(out_d, non_blocking=True)
    t_zci = tm(zc_in)
    print(f"  lanes={dec.lanes}: decode_host {t_host*1e3:.3f} ms {n/t_host/1e9:.2f} Gb/s ok={ok_host} | "
          f"zero-copy in+out {t_zc*1e3:.3f} ms {n/t_zc/1e9:.2f} Gb/s ok={ok_zc} | "
          f"zero-copy in + D2H {t_zci*1e3:.3f} ms {n/t_zci/1e9:.2f} Gb/s", flush=True)
