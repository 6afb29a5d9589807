"""Shared numeric helpers for the test suite."""

import numpy as np


def rel_l2(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


NODE_FLOOR = 1e-3


def per_node_rel(a, b, shape, floor=NODE_FLOOR):
    """max over (step, node) of ||a_n - b_n|| / max(||b_n||, floor * max_n ||b_n||).

    The per-node relative L2 of the BASELINE parity contract.  Nodes whose
    norm has decayed below `floor` x the largest node norm are measured
    against that floor: there the reference's own output is only determined
    to its reduction-order rounding (tests/test_oracle_golden.py::
    test_reduction_order_floor measures it by re-running the oracle with a
    different dot-product summation order).
    """
    A, B = np.asarray(a).reshape(shape), np.asarray(b).reshape(shape)
    d = np.linalg.norm(A - B, axis=-1)
    nb = np.linalg.norm(B, axis=-1)
    s = np.maximum(np.maximum(nb, floor * nb.max()), 1e-300)
    return float(np.max(d / s))


def per_node_rel_strict(a, b, shape):
    """Per-node relative L2 against each node's own norm (no floor)."""
    return per_node_rel(a, b, shape, floor=0.0)


def slab_projections(X, k=4, seed=12345):
    """k seeded Gaussian projections of every (step, node) slab of X (..., S).

    Compact at-size fixtures store these instead of the full solution
    (tests/golden/make_golden_sized.py): |P(a) - P(b)| <= ||a - b|| * ||g||
    per slab, so a per-node relative L2 of 1e-10 bounds the projection error.
    """
    X = np.asarray(X)
    g = np.random.default_rng(seed).standard_normal((k, X.shape[-1]))
    return X @ g.T
