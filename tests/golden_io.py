"""Loader for the hand-computed fixtures in tests/golden/ (each carries a citation)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        d = json.load(f)
    assert any(key.startswith("citation") for key in d), f"{name} has no citation"
    return {k: (np.array(v, dtype=np.float64) if isinstance(v, list) else v) for k, v in d.items()}
