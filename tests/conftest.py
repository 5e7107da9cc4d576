import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long CPU test (oracle at full BASELINE size)")


def golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip("golden fixture %s.npz not generated" % name)
    return np.load(path, allow_pickle=False)


def make_mesh(kind, N):
    from paper_1708_03912_b200 import mesh as M
    if kind == "uniform1d":
        return M.build_interval_mesh(-1.0, 1.0, N)
    if kind == "graded1d":
        return M.build_graded_interval_mesh(N)
    if kind == "square2d":
        return M.build_unit_square_mesh(N)
    if kind == "jitter2d":
        # the unit square with its interior vertices moved by up to 0.3 h and the cells relabelled
        # at random (seeded): non-uniform diameters, mixed orders, a partial last Morton block
        base = M.build_unit_square_mesh(N)
        rng = np.random.default_rng(1000 + N)
        V = np.array(base.vertices, dtype=np.float64)
        inner = (V[:, 0] > 1e-12) & (V[:, 0] < 1 - 1e-12) & (V[:, 1] > 1e-12) & (V[:, 1] < 1 - 1e-12)
        V[inner] += rng.uniform(-0.3 / N, 0.3 / N, size=(int(inner.sum()), 2))
        cells = np.array(base.cells)[rng.permutation(len(base.cells))]
        return M.finish_polygon_mesh(V, [tuple(int(v) for v in c) for c in cells])
    if kind == "graded2d":
        # the unit square graded toward the origin (vertex (x, y) -> (x^1.7, y^1.7)): cell diameters
        # spread over ~1.5 decades, anisotropic cells along the axes
        base = M.build_unit_square_mesh(N)
        V = np.array(base.vertices, dtype=np.float64) ** 1.7
        return M.finish_polygon_mesh(V, [tuple(int(v) for v in c) for c in base.cells])
    raise ValueError(kind)


def tiny_cases():
    """(key, kind, N, s) of tests/golden/tiny.npz: n = 1, 2, ... and non-specialised s."""
    path = os.path.join(GOLDEN, "tiny.npz")
    if not os.path.exists(path):
        return []
    keys = sorted({k.split("/")[0] for k in np.load(path).files})
    out = []
    for key in keys:
        kind, N, s = key.rsplit("_", 2)
        out.append((key, kind, int(N), float(s)))
    return out


def irregular_cases():
    """(key, s) of the jittered / relabelled meshes in tests/golden/irregular.npz."""
    path = os.path.join(GOLDEN, "irregular.npz")
    if not os.path.exists(path):
        return []
    G = np.load(path)
    return [(k, float(G[k + "/s"])) for k in sorted({f.split("/")[0] for f in G.files})]


def irregular_mesh(key):
    """The reference-finished irregular mesh stored in the fixture (vertices, cells, boundary)."""
    from paper_1708_03912_b200 import mesh as M
    G = golden("irregular")
    return M.Mesh(G[key + "/vertices"], G[key + "/cells"], G[key + "/bedges"], G[key + "/bnormals"])


def small_cases():
    path = os.path.join(GOLDEN, "small.npz")
    if not os.path.exists(path):
        return []
    keys = sorted({k.split("/")[0] for k in np.load(path).files})
    out = []
    for key in keys:
        kind, N, s = key.rsplit("_", 2)
        out.append((key, kind, int(N), float(s)))
    return out


@pytest.fixture(scope="session")
def cuda_lib():
    from paper_1708_03912_b200 import _lib
    lib = _lib.load()
    if lib.fl_device_count() < 1:
        pytest.fail("GPU test collected but no CUDA device visible")
    return lib
