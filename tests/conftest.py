import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def load_groups(name: str) -> dict:
    """tests/golden/<name>.npz with keys '<case>__<field>' -> {case: {field: array}}."""
    z = np.load(GOLDEN / f"{name}.npz")
    out: dict = {}
    for key in z.files:
        case, _, field = key.partition("__")
        out.setdefault(case, {})[field] = z[key]
    return out


@pytest.fixture(scope="session")
def renderer():
    from paper_2103_01954_b200 import Renderer
    r = Renderer(0)
    yield r
    r.close()


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()
