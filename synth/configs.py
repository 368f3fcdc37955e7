"""Workload definitions C1-C5 (BASELINE.json "configs", in order) plus small
test shapes.  Readings:

* R3  units: Gaussian, c = 1, dx = dy = dz = 1, electron q = -1, m = 1,
      proton q = +1, m = 1836.
* R4  dt = 0.5 / (c sqrt(1/dx^2 + 1/dy^2 + 1/dz^2)) for every config.
* R10 ppc counts both species (C3 = 25 e + 25 p, C5 = 32 e + 32 p).
* R11 C1-C4 density: n_e = 0.01 / (4 pi) per unit cell volume (omega_pe = 0.1),
      w = n_e / ppc_species.
* R12 thermal spread: each momentum component p_i ~ N(0, sigma^2) in m_e c,
      so u_i = p_i / m (protons get u = sigma / 1836).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

N_E_DEFAULT = 0.01 / (4.0 * math.pi)   # R11: omega_pe = 0.1 c/dx
PROTON_MASS = 1836.0                    # BASELINE.json configs[2] "mass ratio 1836"


def dt_courant(dx=1.0, dy=1.0, dz=1.0, c=1.0, courant=0.5) -> float:
    """R4: dt = courant * dt_CFL, dt_CFL = 1 / (c sqrt(1/dx^2 + 1/dy^2 + 1/dz^2))."""
    return courant / (c * math.sqrt(1.0 / dx ** 2 + 1.0 / dy ** 2 + 1.0 / dz ** 2))


@dataclass(frozen=True)
class SpeciesSpec:
    name: str
    q: float
    m: float
    ppc: int             # particles per cell of this species
    sigma_p: float       # momentum spread in m_e c (R12); u = p / m
    density: float = N_E_DEFAULT
    colocate_with: int = -1   # R13 (C5): reuse positions of an earlier species

    @property
    def w(self) -> float:
        return self.density / self.ppc if self.ppc else 0.0

    @property
    def sigma_u(self) -> float:
        return self.sigma_p / self.m


@dataclass(frozen=True)
class Workload:
    name: str
    nx: int
    ny: int
    nz: int                     # global z cells (all ranks)
    species: tuple
    steps: int
    sort_every: int = 20
    supercell: int = 4
    halo: int = 1               # tile drift halo h of the fused kernel (pic_config.halo)
    seed: int = 0
    dx: float = 1.0
    dy: float = 1.0
    dz: float = 1.0
    c: float = 1.0
    courant: float = 0.5
    nz_per_rank: int = 0        # C4: weak scaling, nz = nz_per_rank * nranks
    description: str = ""
    # NEXT-1 (reading R21): open z box with the incident laser, and the z
    # range [lo, hi) of planes that hold plasma (None: every plane)
    open_z: bool = False
    laser: tuple = ()           # (("e0", E0), ("omega", w), ("ramp", T), ("t0", t0), ("pol", (px, py)))
    plasma_z: tuple = ()

    @property
    def dt(self) -> float:
        return dt_courant(self.dx, self.dy, self.dz, self.c, self.courant)

    @property
    def ncells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_particles(self) -> int:
        planes = (self.plasma_z[1] - self.plasma_z[0]) if self.plasma_z else self.nz
        return sum(s.ppc for s in self.species) * self.nx * self.ny * planes

    def for_ranks(self, nranks: int) -> "Workload":
        if self.nz_per_rank:
            return replace(self, nz=self.nz_per_rank * nranks)
        return self

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)


def electron(ppc, sigma, density=N_E_DEFAULT):
    return SpeciesSpec("electron", -1.0, 1.0, ppc, sigma, density)


def proton(ppc, sigma, density=N_E_DEFAULT, colocate_with=-1):
    return SpeciesSpec("proton", 1.0, PROTON_MASS, ppc, sigma, density, colocate_with)


_NC_C5 = (2.0 * math.pi / 32.0) ** 2 / (4.0 * math.pi)   # critical density, lambda = 32 cells


def laser_c5(t0: float, a0: float = 10.0, wavelength: float = 32.0):
    """BASELINE.json configs[4]: linearly polarised (x) plane wave of normalised
    amplitude a0 = e E0 / (m c omega) and wavelength 32 cells, injected
    through z = 0 (R21): E0 = a0 omega (e = m = c = 1), sin^2 ramp over two
    wavelengths; t0 = the time it has been entering before t = 0 (its front
    starts at z = c t0)."""
    omega = 2.0 * math.pi / wavelength
    return (("e0", a0 * omega), ("omega", omega), ("ramp", 2.0 * wavelength), ("t0", t0),
            ("pol", (1.0, 0.0)))

CONFIGS = {
    # BASELINE.json configs[0]
    "C1": Workload("C1", 16, 16, 16, (electron(8, 0.01),), steps=10, sort_every=5,
                   description="16^3 thermal, 8 e/cell, sigma 0.01, 10 steps"),
    # BASELINE.json configs[1] -- paper-shaped (40^3 x 50 ppc)
    "C2": Workload("C2", 40, 40, 40, (electron(50, 0.05),), steps=100, sort_every=20,
                   description="40^3 thermal, 50 e/cell (3.2M), sigma 0.05, 100 steps"),
    # BASELINE.json configs[2]
    "C3": Workload("C3", 128, 128, 128, (electron(25, 0.1), proton(25, 0.1)), steps=200,
                   sort_every=20,
                   description="128^3 thermal, 25 e + 25 p per cell (104.9M), sigma_p 0.1"),
    # BASELINE.json configs[3] -- weak scaling, nz = 128 per GPU
    "C4": Workload("C4", 256, 256, 128, (electron(32, 0.1),), steps=100, sort_every=20,
                   nz_per_rank=128,
                   description="256x256x(128 N) thermal, 32 e/cell (268M per GPU), sigma 0.1"),
    # BASELINE.json configs[4] -- laser-plasma slab (NEXT-1, reading R21): open z,
    # laser through z = 0 whose front has reached the slab surface z = 600 at t = 0,
    # cold e + p slab (32 + 32 per cell, co-located, n = 10 n_c) on z in [600, 700)
    "C5": Workload("C5", 512, 512, 1024,
                   (electron(32, 0.0, 10 * _NC_C5), proton(32, 0.0, 10 * _NC_C5, colocate_with=0)),
                   steps=500, sort_every=20, open_z=True, laser=laser_c5(600.0), plasma_z=(600, 700),
                   description="512x512x1024 open-z laser-plasma slab z in [600,700), a0 = 10"),
    # C5 on one GPU: the same columns (x, y periodic, the plane wave and the slab are
    # uniform in x, y) on a 128 x 128 cross-section: 104.9M particles
    "C5_1g": Workload("C5_1g", 128, 128, 1024,
                      (electron(32, 0.0, 10 * _NC_C5), proton(32, 0.0, 10 * _NC_C5, colocate_with=0)),
                      steps=500, sort_every=20, open_z=True, laser=laser_c5(600.0), plasma_z=(600, 700),
                      description="C5 physics on a 128x128 cross-section (one GPU)"),
    # the paper's own benchmark: 40^3 grid,
    # 50 particles per cell, 1000 steps, frozen plasma (zero momenta, zero fields;
    # every stage still runs).  The paper's KNL time is 10.75 s = 3.36 ns/particle/step.
    "FROZEN": Workload("FROZEN", 40, 40, 40, (electron(50, 0.0),), steps=1000, sort_every=20,
                       description="paper frozen-plasma benchmark: 40^3, 50 ppc, u = 0, 1000 steps"),
    # small shapes for tests (not bench lines)
    "T_small": Workload("T_small", 8, 12, 16, (electron(4, 0.05),), steps=5, sort_every=2,
                        description="8x12x16 non-cubic test grid"),
    "T_two_species": Workload("T_two_species", 12, 8, 8, (electron(3, 0.1), proton(3, 0.1)),
                              steps=4, sort_every=3, description="two-species test"),
    # C5 in miniature (P18): open z; the laser's sin^2 ramp (64 = 2 lambda) has
    # just passed the slab surface z = 40 at t = 0, so the electrons turn
    # relativistic within a few steps
    "T_laser": Workload("T_laser", 8, 8, 96,
                        (electron(2, 0.0, 10 * _NC_C5), proton(2, 0.0, 10 * _NC_C5, colocate_with=0)),
                        steps=20, sort_every=5, open_z=True, laser=laser_c5(104.0), plasma_z=(40, 52),
                        description="8x8x96 open-z laser-plasma slab z in [40,52), a0 = 10"),
}


def get_config(name: str) -> Workload:
    return CONFIGS[name]
