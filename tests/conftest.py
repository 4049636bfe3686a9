import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLDEN = os.path.join(HERE, "golden")
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running test")


def gpu_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


_cache = {}


def golden(name):
    if name not in _cache:
        path = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            with open(path) as f:
                _cache[name] = json.load(f)
        else:
            _cache[name] = dict(np.load(path))
    return _cache[name]


def golden_mat(d, prefix):
    """(nrows, ncols, row_ptr, col_idx, values) from a golden npz dict."""
    nr, nc = (int(v) for v in d[prefix + "_shape"])
    return nr, nc, d[prefix + "_rp"], d[prefix + "_ci"], d[prefix + "_v"]


def golden_levels(d, prefix):
    """Oracle-style level dicts of a golden hierarchy."""
    L = int(d[prefix + "_nlev"][0])
    levels = []
    for l in range(L):
        lv = {"A": golden_mat(d, f"{prefix}_A{l}")[2:], "m": d[f"{prefix}_M{l}"]}
        if l < L - 1:
            lv["P"] = golden_mat(d, f"{prefix}_P{l}")[2:]
            lv["R"] = golden_mat(d, f"{prefix}_R{l}")[2:]
        levels.append(lv)
    return levels


def smoother_params():
    with open(os.path.join(REPO, "paper_2407_09848_b200", "data", "smoother_params.json")) as f:
        return json.load(f)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
