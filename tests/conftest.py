"""Shared fixtures. `-m "not gpu"` runs everywhere; `-m gpu` needs a B200 (sm_100a)."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and the built engine")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    return meta, arrays


@pytest.fixture
def rng():
    return np.random.default_rng(20240901)


def loop_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Independent scalar triple-loop product (pure Python arithmetic, no numpy)."""
    m, inner = a.shape
    n = b.shape[1]
    al, bl = a.tolist(), b.tolist()
    out = [[0] * n for _ in range(m)]
    for i in range(m):
        for j in range(n):
            s = al[i][0] * bl[0][j]
            for p in range(1, inner):
                s += al[i][p] * bl[p][j]
            out[i][j] = s
    return np.array(out, dtype=a.dtype)


def draw(seed: int, shape_a, shape_b, exact: bool):
    """Operands exactly as tests/golden/make_golden.py draws them."""
    r = np.random.default_rng(seed)
    if exact:
        return r.integers(-8, 9, size=shape_a, dtype=np.int64), r.integers(-8, 9, size=shape_b, dtype=np.int64)
    return r.uniform(-1.0, 1.0, size=shape_a), r.uniform(-1.0, 1.0, size=shape_b)


def int_matrix(rng, rows, cols):
    from paper_2309_00628_b200 import Matrix

    return Matrix(rng.integers(-8, 9, size=(rows, cols), dtype=np.int64))


def real_matrix(rng, rows, cols):
    from paper_2309_00628_b200 import Matrix

    return Matrix(rng.uniform(-1.0, 1.0, size=(rows, cols)))
