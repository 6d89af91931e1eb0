"""Shared test helpers (imported as `helpers`; tests/ is put on sys.path by conftest)."""

import json
import os
import sys

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".npz"):
        return np.load(path)
    with open(path) as fh:
        return json.load(fh)


def same_sum_semantics(meta) -> bool:
    """Float goldens are only comparable under the same CPython sum()."""
    return meta["sum"] == ("neumaier" if sys.version_info >= (3, 12) else "naive")


from oracle import problem_of, spaces_of  # noqa: E402,F401  (re-export)
