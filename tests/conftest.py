import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def random_coords(rng, n, G, batch=1):
    """n unique random voxels per batch item in a G^3 grid -> int32 [batch*n, 4] (b,x,y,z)."""
    out = []
    for b in range(batch):
        cells = rng.choice(G ** 3, size=n, replace=False)
        x, y, z = cells // (G * G), (cells // G) % G, cells % G
        out.append(np.stack([np.full(n, b), x, y, z], axis=1))
    return np.concatenate(out).astype(np.int32)


@pytest.fixture
def rng():
    return np.random.Generator(np.random.PCG64(1234))


def pytest_sessionfinish(session, exitstatus):
    """Write the per-tensor parity report (tests/gpu_util.REPORT) when SSA_PARITY_REPORT is set."""
    path = os.environ.get("SSA_PARITY_REPORT")
    mod = sys.modules.get("gpu_util")
    if not path or mod is None or not mod.REPORT:
        return
    import json
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "w") as f:
        json.dump({"metric": "max|x-ref|/rms(ref), undiscounted; LSE: max|x-ref| (natural log)",
                   "rows": mod.REPORT}, f, indent=1)
