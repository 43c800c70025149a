import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size configuration runs")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, reference_available
    if not reference_available() and not os.path.isdir("/root/reference/proj/src"):
        pytest.skip("reference library (oracle/_ref) not built here")
    return Reference()


@pytest.fixture(scope="session")
def kats():
    with open(os.path.join(GOLDEN, "reference_kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def config_golden():
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        return json.load(f)


def load_instances():
    from paper_1801_03065_b200 import CsrMatrix
    z = np.load(os.path.join(GOLDEN, "instances.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    out = []
    for it, m in enumerate(meta["instances"]):
        p = f"i{it}_"
        mats = []
        for name in ("a", "b"):
            r, c = (int(x) for x in z[p + name + "_shape"])
            mats.append(CsrMatrix(r, c, z[p + name + "_ro"], z[p + name + "_ci"], z[p + name + "_v"],
                                  meta["kinds"][it] != "random_shuffled"))
        out.append({"a": mats[0], "b": mats[1], "c_ro": z[p + "c_ro"], "c_ci": z[p + "c_ci"],
                    "c_v": z[p + "c_v"], "per_row_flops": z[p + "per_row_flops"], "meta": m,
                    "kind": meta["kinds"][it]})
    return out


def csr_from_triplets(rows, cols, trips):
    """build_csr semantics (csr_matrix.cpp:18-80) for small literal inputs."""
    from paper_1801_03065_b200 import CsrMatrix
    per = [[] for _ in range(rows)]
    for r, c, v in trips:
        per[r].append((c, v))
    ro, ci, vv = [0], [], []
    for row in per:
        row.sort(key=lambda t: t[0])
        for q, (c, v) in enumerate(row):
            if ci and q > 0 and ci[-1] == c:
                vv[-1] += v
            else:
                ci.append(c)
                vv.append(float(v))
        ro.append(len(ci))
    return CsrMatrix(rows, cols, np.array(ro, np.int64), np.array(ci, np.int32), np.array(vv, np.float64), True)


def random_csr(rng, rows, cols, density, shuffle=False):
    """Random CSR with unique columns per row (fixture for GPU parity tests)."""
    from paper_1801_03065_b200 import CsrMatrix
    ro, ci, vv = [0], [], []
    for _ in range(rows):
        cnt = rng.binomial(cols, density) if cols > 0 else 0
        c = rng.choice(cols, size=cnt, replace=False) if cnt else np.zeros(0, np.int64)
        if not shuffle:
            c = np.sort(c)
        ci.extend(c.tolist())
        vv.extend(rng.uniform(-1, 1, size=cnt).tolist())
        ro.append(len(ci))
    return CsrMatrix(rows, cols, np.array(ro, np.int64), np.array(ci, np.int32), np.array(vv, np.float64),
                     not shuffle)
