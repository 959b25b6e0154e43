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
