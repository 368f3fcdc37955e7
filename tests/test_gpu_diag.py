"""GPU diagnostics (pic_diagnostics) against the
oracle's definitions (oracle_deposit_rho / div_edge / div_face / energies)
on identical states, and the physics they check at full size: the VB deposit
conserves the CIC charge exactly (P11 continuity), the Yee update keeps
div B and the Gauss residual fixed (P12)."""
import math

import numpy as np
import pytest

from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pic():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1608_01009_b200 as P
    P.lib()
    return P


def _oracle_for(O, wl, parts):
    g = O.Grid(wl.nx, wl.ny, wl.nz, wl.dx, wl.dy, wl.dz, wl.dt, wl.c,
               [O.Species(s.q, s.m, s.w) for s in wl.species], wl.supercell, wl.sort_every)
    return O.Oracle(g, particles=[(p.copy(), i.copy()) for p, i in parts])


def _oracle_diag(O, orc):
    """The pic_diag quantities from the oracle's own diagnostics."""
    g = orc.grid
    rho = orc.rho()
    gauss = orc.div_edge(0) - 4.0 * math.pi * rho
    dV = g.dx * g.dy * g.dz
    kin = [orc.kinetic_energy(s) for s in range(len(orc.P))]
    return {"rho": rho, "gauss": gauss, "div_b": orc.div_b(), "field_energy": orc.field_energy(),
            "kinetic": kin, "current": [orc.F[6 + c].sum() * dV for c in range(3)],
            "divj": orc.div_edge(6)}


def test_diagnostics_match_oracle(pic, oracle_mod):
    from synth import gen_particles, get_config
    wl = get_config("T_two_species").with_(supercell=2, sort_every=3)
    parts = gen_particles(wl)
    rng = np.random.default_rng(31)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.05
    orc = _oracle_for(oracle_mod, wl, parts)
    orc.F[:6] = F6
    sim = pic.simulation_from_workload(wl)
    for s, (P, ids) in enumerate(parts):
        sim.set_particles(s, P, ids)
    sim.set_fields(F6)
    d0 = sim.diagnostics(rho=True)
    o0 = _oracle_diag(oracle_mod, orc)
    assert d0["step"] == 0 and d0["max_continuity"] == -1.0 and d0["max_gauss_drift"] == 0.0
    sim.step(3)
    orc.step(3)
    d1 = sim.diagnostics()                    # not consecutive: no continuity
    assert d1["max_continuity"] == -1.0
    sim.step(1)
    orc.step(1)
    rho_prev = orc.rho()
    sim_d3 = sim.diagnostics(rho=True)
    sim.step(1)
    orc.step(1)
    d = sim.diagnostics(rho=True)
    o = _oracle_diag(oracle_mod, orc)
    assert d["step"] == 5
    assert rel_err(d["rho"], o["rho"]) <= 1e-12
    assert rel_err(sim_d3["rho"], rho_prev) <= 1e-12
    assert d["field_energy"] == pytest.approx(o["field_energy"], rel=1e-12)
    for s in range(2):
        assert d["kinetic_energy"][s] == pytest.approx(o["kinetic"][s], rel=1e-12)
    qsum = sum(sp.q * sp.w * P.shape[1] for sp, (P, _) in zip(wl.species, parts))
    assert d["charge"] == pytest.approx(qsum, rel=1e-12)
    jscale = max(abs(orc.F[6:9]).max() * wl.ncells, 1e-300)
    for c in range(3):
        assert abs(d["current"][c] - o["current"][c]) <= 1e-12 * jscale
    bscale = abs(orc.F[3:6]).max()
    # random initial B: div B is O(B) and must stay at its initial value (P12)
    assert abs(d["max_div_b"] - abs(o["div_b"]).max()) <= 1e-12 * bscale
    assert abs(d["max_div_b"] - d0["max_div_b"]) <= 1e-12 * bscale
    gscale = max(abs(o["gauss"]).max(), 1e-300)
    assert abs(d["max_gauss"] - abs(o["gauss"]).max()) <= 1e-12 * gscale
    assert abs(d["max_gauss_drift"] - abs(o["gauss"] - o0["gauss"]).max()) <= 1e-12 * gscale
    # continuity over the last step, from the oracle's own rho and div J
    cont_o = (o["rho"] - rho_prev) / wl.dt + o["divj"]
    rscale = abs(o["rho"]).max() / wl.dt
    assert abs(cont_o).max() <= 1e-12 * rscale          # the oracle conserves charge (P11)
    assert 0.0 <= d["max_continuity"] <= 1e-12 * rscale
    # Gauss drift is rounding only: VB + Yee keep div E - 4 pi rho fixed
    assert d["max_gauss_drift"] <= 1e-11 * gscale


@pytest.mark.parametrize("nranks", [2, 4])
def test_diagnostics_slab_group(pic, oracle_mod, nranks):
    """Decomposed diagnostics: the slab pieces of rho (top node plane sent to
    the slab above) and the Jz plane from below reproduce the single-domain
    oracle; sums over ranks match."""
    import torch
    from synth import gen_particles, get_config
    from synth.configs import electron
    wl = get_config("C1").with_(species=(electron(6, 0.2),), nz=16, sort_every=5)
    parts = gen_particles(wl)
    orc = _oracle_for(oracle_mod, wl, parts)
    stream = torch.cuda.Stream()
    sims = []
    for r in range(nranks):
        cfg = pic.workload_config(wl, rank=r, nranks=nranks, flags=pic.FLAG_LOCAL_GROUP,
                                  migrate_capacity=4096)
        sims.append(pic.Simulation(cfg, stream=stream))
        sims[-1].set_particles(0, *parts[0])
    pic.step_group(sims, 4)
    orc.step(4)
    pic.diagnostics_group(sims)
    pic.step_group(sims, 1)
    orc.step(1)
    ds = pic.diagnostics_group(sims, rho=True)
    o = _oracle_diag(oracle_mod, orc)
    rho = np.concatenate([d["rho"] for d in ds], axis=0)
    assert rel_err(rho, o["rho"]) <= 1e-12
    assert sum(d["field_energy"] for d in ds) == pytest.approx(o["field_energy"], rel=1e-11)
    assert sum(d["kinetic_energy"][0] for d in ds) == pytest.approx(o["kinetic"][0], rel=1e-12)
    qsum = wl.species[0].q * wl.species[0].w * parts[0][0].shape[1]
    assert sum(d["charge"] for d in ds) == pytest.approx(qsum, rel=1e-12)
    rscale = abs(o["rho"]).max() / wl.dt
    for d in ds:
        assert 0.0 <= d["max_continuity"] <= 1e-12 * rscale
        assert d["max_div_b"] <= 1e-13 * max(abs(orc.F[3:6]).max(), 1e-300) + 1e-300
    gscale = abs(o["gauss"]).max()
    assert max(d["max_gauss"] for d in ds) == pytest.approx(gscale, rel=1e-11)


def test_diagnostics_full_size_C2(pic):
    """C2 at full size (3.2M particles, 40^3): charge conservation per step
    (continuity), div B = 0 and a constant Gauss residual over 25 steps
    (one sort in between) -- the physics checks of NEXT-3 at a size the
    oracle cannot run in full."""
    from synth import gen_particles, get_config
    wl = get_config("C2")
    parts = gen_particles(wl)
    sim = pic.simulation_from_workload(wl)
    sim.set_particles(0, *parts[0])
    d0 = sim.diagnostics(rho=True)
    rscale = abs(d0["rho"]).max()
    qsum = wl.species[0].q * wl.species[0].w * parts[0][0].shape[1]
    assert d0["charge"] == pytest.approx(qsum, rel=1e-12)
    assert d0["max_gauss"] == pytest.approx(4 * math.pi * rscale, rel=1e-12)   # E = 0
    e0 = None
    for n in (5, 19, 20, 21):
        sim.step(n - sim.step_index())
        sim.diagnostics()
        sim.step(1)
        d = sim.diagnostics()
        assert 0.0 <= d["max_continuity"] <= 1e-12 * rscale / wl.dt, (n, d)
        assert d["max_div_b"] <= 1e-15, (n, d)
        assert d["max_gauss_drift"] <= 1e-11 * 4 * math.pi * rscale, (n, d)
        assert d["charge"] == pytest.approx(qsum, rel=1e-12)
        etot = d["field_energy"] + d["kinetic_energy"][0]
        assert math.isfinite(etot) and etot > 0
        e0 = etot if e0 is None else e0
    # thermal plasma at 0.05 c, omega_p dt = 0.029: total energy within a few percent
    assert abs(etot - e0) <= 0.05 * e0
