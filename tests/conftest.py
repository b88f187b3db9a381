import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _unhex(v):
    return np.array([float.fromhex(x) for x in v], np.float32)


class HandNet:
    """A golden hand net from tests/golden/hand_nets.json (exact hex floats)."""

    def __init__(self, name, d):
        self.name = name
        self.n, self.L = d["n"], d["L"]
        self.ymax = float.fromhex(d["ymax"])
        self.layers = []
        for lay in d["layers"]:
            self.layers.append(dict(rowptr=np.array(lay["rowptr"], np.int64),
                                    colidx=np.array(lay["colidx"], np.int32),
                                    val=_unhex(lay["val"]), bias=_unhex(lay["bias"])))
        self.y0_rowptr = np.array(d["y0"]["rowptr"], np.int64)
        self.y0_idx = np.array(d["y0"]["idx"], np.int32)
        self.y0_val = _unhex(d["y0"]["val"])
        self.expected_Y = np.array([[float.fromhex(x) for x in r] for r in d["expected_Y"]],
                                   np.float32).reshape(-1, self.n)
        self.expected_categories = list(d["expected_categories"])


def load_hand_nets():
    d = json.load(open(os.path.join(GOLDEN, "hand_nets.json")))
    return {k: HandNet(k, v) for k, v in d["nets"].items()}


@pytest.fixture(scope="session")
def hand_nets():
    return load_hand_nets()


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
