"""Seeded particle generator (readings R12-R14 of DESIGN.md).

* R13 positions: stratified -- for each cell in x-fastest order and each slot
  s < ppc, x = (i + U) dx with U ~ U[0,1); the few draws that round up to the
  next cell boundary at x = L are mapped to 0 (positions stay in [0, L)).
* R12 momenta: u_i ~ N(0, sigma_p / m).
* R14 RNG: numpy Generator(PCG64(seed)), per species in order: first the
  positions rng.random((N,3)), then the momenta rng.normal(0, sigma_u, (N,3)).
  A rank of a z-slab decomposition draws its own slab with seed (seed, rank).
Species with colocate_with >= 0 reuse that species' positions (C5, R13);
a workload with plasma_z fills only those planes (C5, NEXT-1).

Output per species: P float64[6][N] (rows x,y,z,ux,uy,uz), id uint64[N].
"""
from __future__ import annotations

import numpy as np

from .configs import Workload


def _rng(seed: int, rank: int | None):
    if rank is None:
        return np.random.Generator(np.random.PCG64(seed))
    return np.random.Generator(np.random.PCG64([seed, rank]))


def gen_species(wl: Workload, s: int, rng, z_lo: int = 0, z_hi: int | None = None,
                positions=None, id_base: int = 0):
    sp = wl.species[s]
    z_hi = wl.nz if z_hi is None else z_hi
    if wl.plasma_z:   # C5: plasma only on the planes [plasma_z[0], plasma_z[1])
        z_lo, z_hi = max(z_lo, wl.plasma_z[0]), max(max(z_lo, wl.plasma_z[0]), min(z_hi, wl.plasma_z[1]))
    ncell = wl.nx * wl.ny * (z_hi - z_lo)
    n = ncell * sp.ppc
    P = np.empty((6, n), dtype=np.float64)
    if positions is None:
        U = rng.random((n, 3))
        cell = np.arange(n, dtype=np.int64) // sp.ppc
        ci = cell % wl.nx
        cj = (cell // wl.nx) % wl.ny
        ck = cell // (wl.nx * wl.ny) + z_lo
        L = (wl.nx * wl.dx, wl.ny * wl.dy, wl.nz * wl.dz)
        for d, (c_idx, h) in enumerate(((ci, wl.dx), (cj, wl.dy), (ck, wl.dz))):
            x = (c_idx + U[:, d]) * h
            x[x >= L[d]] = 0.0
            P[d] = x
        del U
    else:
        P[:3] = positions
    if sp.sigma_u > 0:
        P[3:] = rng.normal(0.0, sp.sigma_u, (n, 3)).T
    else:
        P[3:] = 0.0
    ids = np.arange(n, dtype=np.uint64) + np.uint64(id_base)
    return P, ids


def gen_particles(wl: Workload, seed: int | None = None, rank: int | None = None,
                  z_lo: int = 0, z_hi: int | None = None):
    """All species of a workload: list of (P[6][N], id[N]).

    ids: species s, rank r, ordinal p -> (s << 56) | (r << 40) | p."""
    seed = wl.seed if seed is None else seed
    rng = _rng(seed, rank)
    out = []
    for s, sp in enumerate(wl.species):
        base = (s << 56) | ((rank or 0) << 40)
        pos = None
        if sp.colocate_with >= 0:
            pos = out[sp.colocate_with][0][:3]
        out.append(gen_species(wl, s, rng, z_lo, z_hi, positions=pos, id_base=base))
    return out


def gen_fields(wl: Workload, seed: int = 7, e_sigma: float = 0.01, b_sigma: float = 0.1):
    """Seeded synthetic E^0, B^0 for parity slices: every node value of
    Ex,Ey,Ez ~ N(0, e_sigma), Bx,By,Bz ~ N(0, b_sigma) (numpy PCG64(seed)),
    shape (6, nz, ny, nx), x fastest.  Random numbers only -- no method
    arithmetic -- so the same array feeds the oracle and the GPU."""
    rng = _rng(seed, None)
    F = np.empty((6, wl.nz, wl.ny, wl.nx), dtype=np.float64)
    F[:3] = rng.normal(0.0, e_sigma, (3, wl.nz, wl.ny, wl.nx))
    F[3:] = rng.normal(0.0, b_sigma, (3, wl.nz, wl.ny, wl.nx))
    return F
