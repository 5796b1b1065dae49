import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
# run-time (NVRTC) kernels of the JIT tests: a repo-local disk cache (built
# artefacts, git-ignored) -- a speed-up only, every entry is rebuilt if absent
os.environ.setdefault("PBVD_JIT_CACHE", str(ROOT / "paper_1608_00066_b200" / "build" / "jit_cache"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: statistical oracle checks (tens of seconds)")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle
