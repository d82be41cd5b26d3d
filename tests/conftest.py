"""Shared test configuration.

Markers: ``gpu`` = needs a B200 (run on the GPU box with ``-m gpu``); all other
tests run on the CPU-only build container.  The CPU oracle (``oracle/``) is test
infrastructure: tests use it only as the checker.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run with -m gpu)")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


@pytest.fixture(scope="session")
def oracle():
    from oracle import cgs_oracle

    cgs_oracle.build_loops()
    return cgs_oracle


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    err = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    _log_margin("rel_l2", err, float("nan"))
    return err


def grads_close(a, b, rtol, floor_frac):
    """Per-parameter-column relative L2 with an absolute floor.

    Column j passes when ||a_j - b_j|| <= rtol * max(||b_j||, floor_frac * ||b||).
    The floor matters only for columns that are analytically zero (e.g. quaternion
    gradients of isotropic Gaussians, which the reference returns as ~1e-18
    rounding noise).  Returns the list of worst relative errors per column.
    """
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    floor = floor_frac * np.linalg.norm(b)
    errs = []
    for j in range(b.shape[1]):
        den = max(np.linalg.norm(b[:, j]), floor)
        errs.append(float(np.linalg.norm(a[:, j] - b[:, j]) / den))
    _log_margin("grads", max(errs), rtol)
    assert max(errs) <= rtol, errs
    return errs


def _log_margin(kind, err, tol):
    """Append (test, kind, worst error, tolerance) to $CGS_MARGIN_LOG when set: the
    precision margin of every parity check, tracked across kernel changes."""
    path = os.environ.get("CGS_MARGIN_LOG")
    if path:
        test = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
        with open(path, "a") as f:
            f.write(f"{test}\t{kind}\t{err:.3e}\t{tol:.1e}\n")
