"""ctypes wrapper of the plain CPU oracle (oracle/pic_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_1608_01009_b200/) never imports this module and this module never
imports the product package.  Arrays are numpy float64 / uint64.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
MAX_SPECIES = 4

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


class OracleConfig(C.Structure):
    _fields_ = [
        ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
        ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
        ("dt", C.c_double), ("c", C.c_double),
        ("n_species", C.c_int64),
        ("q", C.c_double * MAX_SPECIES),
        ("m", C.c_double * MAX_SPECIES),
        ("w", C.c_double * MAX_SPECIES),
        ("supercell", C.c_int64),
        ("sort_every", C.c_int64),
        ("bc_z", C.c_int64),
        ("laser_e0", C.c_double), ("laser_omega", C.c_double), ("laser_ramp", C.c_double),
        ("laser_t0", C.c_double), ("laser_pol_x", C.c_double), ("laser_pol_y", C.c_double),
    ]


BC_PERIODIC = 0
BC_OPEN = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, -O2, no FMA contraction)."""
    src = os.path.join(_HERE, "pic_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "pic_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math",
             "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"]
        )
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        cp = C.POINTER(OracleConfig)
        L.oracle_gather.argtypes = [cp, _dp, C.c_double, C.c_double, C.c_double, _dp]
        L.oracle_boris.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.oracle_move.argtypes = [C.c_double, C.c_double, _dp, _dp, _dp]
        L.oracle_deposit_vb.argtypes = [cp, C.c_double, _dp, _dp, _dp]
        L.oracle_deposit_vb.restype = C.c_int
        L.oracle_wrap.argtypes = [C.c_double, C.c_double]
        L.oracle_wrap.restype = C.c_double
        L.oracle_sort_key.argtypes = [cp, C.c_double, C.c_double, C.c_double]
        L.oracle_sort_key.restype = C.c_int64
        L.oracle_sort.argtypes = [cp, C.c_int64, _dp, _u64p]
        L.oracle_b_half.argtypes = [cp, _dp]
        L.oracle_e_full.argtypes = [cp, _dp, C.c_int64]
        L.oracle_laser.argtypes = [cp, C.c_double, C.c_double]
        L.oracle_laser.restype = C.c_double
        L.oracle_laser_preload.argtypes = [cp, _dp]
        L.oracle_push_species.argtypes = [cp, _dp, C.c_int, C.POINTER(C.c_int64), _dp, _u64p]
        L.oracle_push_species.restype = C.c_int
        L.oracle_step.argtypes = [cp, _dp, C.POINTER(C.c_int64), C.POINTER(_dp),
                                  C.POINTER(_u64p), C.c_int64]
        L.oracle_step.restype = C.c_int
        L.oracle_deposit_rho.argtypes = [cp, C.c_double, C.c_int64, _dp, _dp]
        L.oracle_div_edge.argtypes = [cp, _dp, _dp, _dp, _dp]
        L.oracle_div_face.argtypes = [cp, _dp, _dp, _dp, _dp]
        L.oracle_field_energy.argtypes = [cp, _dp]
        L.oracle_field_energy.restype = C.c_double
        L.oracle_kinetic_energy.argtypes = [cp, C.c_int, C.c_int64, _dp]
        L.oracle_kinetic_energy.restype = C.c_double
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous, "arrays must be C-contiguous"
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.uint64:
        return a.ctypes.data_as(_u64p)
    raise TypeError(a.dtype)


@dataclass
class Species:
    q: float
    m: float
    w: float


@dataclass
class Grid:
    nx: int
    ny: int
    nz: int
    dx: float = 1.0
    dy: float = 1.0
    dz: float = 1.0
    dt: float = 0.0
    c: float = 1.0
    species: list = field(default_factory=list)
    supercell: int = 4
    sort_every: int = 20
    # NEXT-1 (reading R21): open z boundaries and the incident laser
    bc_z: int = BC_PERIODIC
    laser_e0: float = 0.0
    laser_omega: float = 0.0
    laser_ramp: float = 0.0
    laser_t0: float = 0.0
    laser_pol: tuple = (1.0, 0.0)

    def cfg(self) -> OracleConfig:
        c = OracleConfig()
        c.nx, c.ny, c.nz = self.nx, self.ny, self.nz
        c.dx, c.dy, c.dz = self.dx, self.dy, self.dz
        c.dt, c.c = self.dt, self.c
        c.n_species = len(self.species)
        for i, s in enumerate(self.species):
            c.q[i], c.m[i], c.w[i] = s.q, s.m, s.w
        c.supercell = self.supercell
        c.sort_every = self.sort_every
        c.bc_z = self.bc_z
        c.laser_e0, c.laser_omega, c.laser_ramp, c.laser_t0 = (
            self.laser_e0, self.laser_omega, self.laser_ramp, self.laser_t0)
        c.laser_pol_x, c.laser_pol_y = self.laser_pol
        return c

    @property
    def ncells(self) -> int:
        return self.nx * self.ny * self.nz


class Oracle:
    """Plain CPU PIC state: F[9][nz][ny][nx]; per species P[6][n], id[n]."""

    def __init__(self, grid: Grid, particles=None, fields=None):
        self.grid = grid
        self._cfg = grid.cfg()
        self.F = np.zeros((9, grid.nz, grid.ny, grid.nx), dtype=np.float64)
        if fields is not None:
            self.F[:6] = np.asarray(fields, dtype=np.float64).reshape(6, grid.nz, grid.ny, grid.nx)
        self.P = []
        self.ids = []
        particles = particles or []
        for s in range(len(grid.species)):
            if s < len(particles) and particles[s] is not None:
                P, idv = particles[s]
                self.P.append(np.ascontiguousarray(P, dtype=np.float64).reshape(6, -1).copy())
                self.ids.append(np.ascontiguousarray(idv, dtype=np.uint64).copy())
            else:
                self.P.append(np.zeros((6, 0)))
                self.ids.append(np.zeros(0, dtype=np.uint64))
        self.step_index = 0

    def sort(self):
        for s in range(len(self.P)):
            n = self.P[s].shape[1]
            lib().oracle_sort(C.byref(self._cfg), n, _p(self.P[s]), _p(self.ids[s]))

    def step(self, nsteps: int = 1):
        L = lib()
        ns = len(self.P)
        for _ in range(nsteps):
            counts = (C.c_int64 * max(ns, 1))(*[p.shape[1] for p in self.P])
            Pp = (_dp * max(ns, 1))(*[_p(p) for p in self.P])
            Ip = (_u64p * max(ns, 1))(*[_p(i) for i in self.ids])
            rc = L.oracle_step(C.byref(self._cfg), _p(self.F), counts, Pp, Ip, self.step_index)
            if rc != 0:
                raise RuntimeError(f"oracle_step failed with code {rc}")
            self._shrink(list(counts)[:ns])
            self.step_index += 1

    def _shrink(self, counts):
        # open z: the C side removed particles in place, rows now have stride m
        for s, m in enumerate(counts):
            n = self.P[s].shape[1]
            if m != n:
                self.P[s] = self.P[s].reshape(-1)[:6 * m].reshape(6, m).copy()
                self.ids[s] = self.ids[s][:m].copy()

    def laser_preload(self):
        lib().oracle_laser_preload(C.byref(self._cfg), _p(self.F))

    def laser(self, z, t):
        return lib().oracle_laser(C.byref(self._cfg), z, t)

    # ---- single-operation entry points (pins) ----
    def gather(self, x, y, z):
        out = np.zeros(6)
        lib().oracle_gather(C.byref(self._cfg), _p(self.F), x, y, z, _p(out))
        return out

    def deposit_vb(self, qw, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return lib().oracle_deposit_vb(C.byref(self._cfg), qw, _p(a), _p(b), _p(self.F))

    def b_half(self):
        lib().oracle_b_half(C.byref(self._cfg), _p(self.F))

    def e_full(self, step=None):
        lib().oracle_e_full(C.byref(self._cfg), _p(self.F),
                            self.step_index if step is None else step)

    def push_species(self, s):
        n = C.c_int64(self.P[s].shape[1])
        rc = lib().oracle_push_species(C.byref(self._cfg), _p(self.F), s, C.byref(n),
                                       _p(self.P[s]), _p(self.ids[s]))
        if rc != 0:
            raise RuntimeError(f"oracle_push_species failed with code {rc}")
        counts = [p.shape[1] for p in self.P]
        counts[s] = n.value
        self._shrink(counts)

    def sort_keys(self, P):
        cfg = C.byref(self._cfg)
        return np.array([lib().oracle_sort_key(cfg, P[0, i], P[1, i], P[2, i])
                         for i in range(P.shape[1])], dtype=np.int64)

    # ---- diagnostics ----
    def rho(self):
        g = self.grid
        out = np.zeros((g.nz, g.ny, g.nx))
        for s, sp in enumerate(g.species):
            lib().oracle_deposit_rho(C.byref(self._cfg), sp.q * sp.w, self.P[s].shape[1],
                                     _p(self.P[s]), _p(out))
        return out

    def rho_of(self, s, P):
        g = self.grid
        out = np.zeros((g.nz, g.ny, g.nx))
        sp = g.species[s]
        P = np.ascontiguousarray(P)
        lib().oracle_deposit_rho(C.byref(self._cfg), sp.q * sp.w, P.shape[1], _p(P), _p(out))
        return out

    def div_edge(self, c0):
        g = self.grid
        out = np.zeros((g.nz, g.ny, g.nx))
        V = [np.ascontiguousarray(self.F[c0 + d]) for d in range(3)]
        lib().oracle_div_edge(C.byref(self._cfg), _p(V[0]), _p(V[1]), _p(V[2]), _p(out))
        return out

    def div_b(self):
        g = self.grid
        out = np.zeros((g.nz, g.ny, g.nx))
        V = [np.ascontiguousarray(self.F[3 + d]) for d in range(3)]
        lib().oracle_div_face(C.byref(self._cfg), _p(V[0]), _p(V[1]), _p(V[2]), _p(out))
        return out

    def field_energy(self):
        return lib().oracle_field_energy(C.byref(self._cfg), _p(self.F))

    def kinetic_energy(self, species=None):
        """sum w m c^2 (gamma - 1) over all species, or one species."""
        sel = range(len(self.P)) if species is None else [species]
        return sum(lib().oracle_kinetic_energy(C.byref(self._cfg), s, self.P[s].shape[1],
                                               _p(self.P[s]))
                   for s in sel)


def boris(q, m, c, dt, EB, u):
    EB = np.ascontiguousarray(EB, dtype=np.float64)
    u = np.array(u, dtype=np.float64)
    lib().oracle_boris(q, m, c, dt, _p(EB), _p(u))
    return u


def move(c, dt, u, x):
    u = np.ascontiguousarray(u, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    xn = np.zeros(3)
    lib().oracle_move(c, dt, _p(u), _p(x), _p(xn))
    return xn


def wrap(x, L):
    return lib().oracle_wrap(x, L)
