"""Shared helpers for the parity tests (test infrastructure)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name if name.endswith(".npz") else name + ".npz"),
                   allow_pickle=False)


def golden_names(prefix):
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.startswith(prefix) and f.endswith(".npz"))


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)
