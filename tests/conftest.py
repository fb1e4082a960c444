import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libbenelux_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")
    try:
        from hypothesis import HealthCheck, settings

        settings.register_profile("kernels", deadline=None, suppress_health_check=[HealthCheck.too_slow])
        settings.load_profile("kernels")
    except ImportError:  # pragma: no cover
        pass


@pytest.fixture(scope="session")
def golden() -> dict:
    with open(GOLDEN_PATH) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.lib()
    return oracle


def pair_keys(pairs):
    out = set()
    for p in pairs:
        if isinstance(p, (list, tuple)):
            out.add((int(p[0]), int(p[1]), int(p[2])))
        else:
            out.add((int(p.kind), p.m, p.n))
    return out


def rows_of(pairs):
    return [[int(p.kind), p.m, p.n, p.rad_m, p.rad_m_plus_1] for p in pairs]
