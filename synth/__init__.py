"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds workload definitions (BASELINE.json configs C1-C5 with the
DESIGN.md readings R3, R4, R10-R14) and numpy random draws only.  It contains
none of the PIC method's arithmetic (no gather, push, deposit or field
update), and imports neither oracle/ nor paper_1608_01009_b200/.
"""
from .configs import CONFIGS, Workload, SpeciesSpec, get_config, dt_courant
from .gen import gen_fields, gen_particles, gen_species

__all__ = ["CONFIGS", "Workload", "SpeciesSpec", "get_config", "dt_courant",
           "gen_fields", "gen_particles", "gen_species"]
