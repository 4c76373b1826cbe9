import hashlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs via gpurun / round-end GPU tier)")
    config.addinivalue_line("markers", "slow: large-size property tests")


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(bytes(a)).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


GOLDEN_CASES = ["hacc34", "amdf40k", "sweep_hacc20", "sweep_amdf8k", "tiny1", "tiny3",
                "const2", "noise20k"]


CPC_CASES = ["cpc_hacc24", "cpc_amdf20k", "cpc_const2", "cpc_noise9k", "cpc_tiny"]


def golden_inputs(g: dict):
    return [g[f"in_{i}"] for i in range(6)]


@pytest.fixture
def rng():
    return np.random.default_rng(20260808)


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    oracle.lib()
    return oracle
