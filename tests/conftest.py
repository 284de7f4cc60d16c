import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _ensure_oracle():
    from oracle import pyoracle
    if not os.path.exists(pyoracle.ORACLE_SO):
        pyoracle.build(ref=False)
    return pyoracle


@pytest.fixture(scope="session")
def orc():
    return _ensure_oracle().Oracle()


@pytest.fixture(scope="session")
def ref():
    pyoracle = _ensure_oracle()
    if not pyoracle.reference_available():
        if os.path.isdir("/root/reference/proj/include"):
            pyoracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and reference headers absent")
    return pyoracle.Reference()


def golden_cases():
    """Batched-solve fixtures (the consumers' fixtures are adi_*.npz, fourier_*.npz)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("adi_", "fourier_")))


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def psw():
    import paper_0901_2859_b200 as psw
    psw.lib()  # fail loudly when the extension is missing
    return psw


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch


def rel_l2(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    den = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / (den if den > 0 else 1.0))


def rel_max(x, y):
    """tests/helpers.hpp:80-87 (max-norm relative error)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    num = np.abs(x - y).max() if x.size else 0.0
    den = np.abs(y).max() if y.size else 0.0
    return float(num / den) if den > 0 else float(num)
