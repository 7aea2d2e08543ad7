import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the CUDA path")


def _oracle_ok():
    try:
        from oracle import ref

        if not ref.available():
            ref.build()
        ref.lib()
        return True
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    """The reference compiled as a library (oracle/_ref). Test infrastructure only."""
    if not _oracle_ok():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    from oracle import ref

    return ref


@pytest.fixture(scope="session")
def gpu():
    from paper_2402_13747_b200 import pcray

    return pcray.Context.default()


def bits(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        return a.view(np.uint64)
    return a


def assert_bitwise(name, a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, f"{name}: shape {a.shape} vs {b.shape}"
    ba, bb = bits(a), bits(b)
    if not np.array_equal(ba, bb):
        diff = np.nonzero(ba.reshape(-1) != bb.reshape(-1))[0]
        i = int(diff[0])
        raise AssertionError(f"{name}: {len(diff)} mismatches, first at flat {i}: "
                             f"{a.reshape(-1)[i]!r} vs {b.reshape(-1)[i]!r}")


def assert_fp(name, a, b, exact=True, tol=1e-12):
    """Bitwise unless exact=False (then within tol); integer fields always exact."""
    a = np.asarray(a)
    b = np.asarray(b)
    if exact or a.dtype != np.float64:
        return assert_bitwise(name, a, b)
    assert a.shape == b.shape, f"{name}: shape {a.shape} vs {b.shape}"
    assert np.allclose(a, b, rtol=tol, atol=tol), f"{name}: max diff {np.max(np.abs(a - b))}"


def assert_grid_equal(g, r):
    for k in ["origin", "dims"]:
        assert_bitwise(k, g[k], r[k])
    assert g["voxel_size"] == r["voxel_size"] and g["division_factor"] == r["division_factor"]
    for k in g:
        if k.startswith(("cell_", "ie_", "point_indices")):
            assert_bitwise(k, g[k], r[k])
