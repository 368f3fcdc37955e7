"""Comparison helpers for GPU-vs-oracle parity (reading R17 of DESIGN.md)."""
from __future__ import annotations

import numpy as np


def rel_err(a, ref):
    """max|a - ref| / max(max|ref|, 1e-300)  (R17)."""
    a = np.asarray(a)
    ref = np.asarray(ref)
    if ref.size == 0:
        return 0.0
    return float(np.abs(a - ref).max() / max(np.abs(ref).max(), 1e-300))


def pos_err(a, ref, L):
    """Same metric for positions with the minimum-image difference mod L (per axis)."""
    L = np.asarray(L, dtype=np.float64).reshape(3, 1)
    d = (a - ref + L / 2) % L - L / 2
    return float(np.abs(d).max() / max(np.abs(ref).max(), 1e-300))


def by_id(P, ids):
    order = np.argsort(ids, kind="stable")
    return P[:, order], ids[order]


def compare_state(gpu_P, gpu_ids, ref_P, ref_ids, L):
    """Particle parity by id: returns (pos_err, mom_err)."""
    gP, gi = by_id(gpu_P, gpu_ids)
    rP, ri = by_id(ref_P, ref_ids)
    assert np.array_equal(gi, ri), "particle id sets differ"
    return pos_err(gP[:3], rP[:3], L), rel_err(gP[3:], rP[3:])


def field_errs(gpu_F, ref_F):
    return [rel_err(gpu_F[c], ref_F[c]) for c in range(gpu_F.shape[0])]
