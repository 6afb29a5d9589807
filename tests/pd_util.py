"""Shared numeric helpers for the test suite."""

import numpy as np


def rel_l2(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def per_node_rel(a, b, shape):
    """max over (step, node) of the relative L2 difference of that node's field."""
    A, B = np.asarray(a).reshape(shape), np.asarray(b).reshape(shape)
    d = np.linalg.norm(A - B, axis=-1)
    s = np.maximum(np.linalg.norm(B, axis=-1), 1e-300)
    return float(np.max(d / s))
