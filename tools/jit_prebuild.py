"""Warm the JIT kernel cache (pbvd_jit_prebuild, NVRTC, no GPU needed) for
the codes of tests/test_gpu_jit.py, in parallel processes.  The cache goes to
$PBVD_JIT_CACHE (default here: the package's git-ignored build/jit_cache,
which travels to the GPU box with the repo snapshot)."""
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("PBVD_JIT_CACHE", str(ROOT / "paper_1608_00066_b200" / "build" / "jit_cache"))


def one(job):
    import paper_1608_00066_b200 as P
    K, polys, lanes = job
    t = time.time()
    P.jit_prebuild(K, polys, lanes)
    return job, time.time() - t


def main():
    sys.path.insert(0, str(ROOT / "tests"))
    from test_gpu_jit import JIT_CODES
    jobs = {(c[1], tuple(c[2]), 0) for c in JIT_CODES}
    jobs |= {(7, (0o133, 0o171), w) for w in (1, 2, 4)}
    jobs.add((5, (0o22, 0o36), 0))
    with ProcessPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for job, dt in ex.map(one, sorted(jobs)):
            print(f"K={job[0]} polys={[oct(p) for p in job[1]]} lanes={job[2]}: {dt:.1f} s")


if __name__ == "__main__":
    main()
