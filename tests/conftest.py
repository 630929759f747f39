import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


def field_digest(z):
    z = np.ascontiguousarray(z, dtype=np.float64) + 0.0
    return hashlib.sha256(z.tobytes()).hexdigest()


def gather_digests(mesh):
    out = []
    for G in mesh.gathers:
        h = hashlib.sha256()
        h.update(np.asarray(G.indptr, dtype=np.int64).tobytes())
        h.update(np.asarray(G.indices, dtype=np.int64).tobytes())
        h.update(np.asarray(G.data, dtype=np.float64).tobytes())
        out.append(h.hexdigest())
    return out


def rel_linf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    scale = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / scale) if scale > 0 else float(np.max(np.abs(a - b)))


def compare_field(got, gd, key):
    """(bit_exact, rel_linf) of a field against a golden entry (full or digested)."""
    if key in gd.files:
        want = gd[key]
        return bool(np.array_equal(got, want)), max(rel_linf(got[v], want[v]) for v in range(2))
    sha = str(gd[key + "__sha"])
    sample = gd[key + "__sample"]
    got_s = got[:, ::7]
    return field_digest(got) == sha, max(rel_linf(got_s[v], sample[v]) for v in range(2))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")
