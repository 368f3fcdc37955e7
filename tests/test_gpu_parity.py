"""GPU (libpic.so, through the C ABI) vs the CPU oracle on identical seeded
inputs.  Tolerances from north_star (BASELINE.json:5) with reading R17:
bit-exact sort permutation; <= 1e-12 per step (teacher-forced); <= 1e-9 after
100 free-running steps."""
import math

import numpy as np
import pytest

from tests.helpers import by_id, compare_state, field_errs, pos_err, rel_err

pytestmark = pytest.mark.gpu

TOL_STEP = 1e-12
TOL_FREE = 1e-9


@pytest.fixture(scope="module")
def pic():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1608_01009_b200 as P
    P.lib()
    return P


def _oracle_for(O, wl, parts, sort_every=None, supercell=None):
    g = O.Grid(wl.nx, wl.ny, wl.nz, wl.dx, wl.dy, wl.dz, wl.dt, wl.c,
               [O.Species(s.q, s.m, s.w) for s in wl.species],
               supercell or wl.supercell, wl.sort_every if sort_every is None else sort_every)
    return O.Oracle(g, particles=[(p.copy(), i.copy()) for p, i in parts])


def _sim(pic, wl, flags=0, sort_every=None, supercell=None, capacity_factor=1.0, counts=None):
    return pic.simulation_from_workload(wl, capacity_factor=capacity_factor, flags=flags,
                                        sort_every=sort_every, supercell=supercell, counts=counts)


def _load(sim, parts):
    for s, (P, ids) in enumerate(parts):
        sim.set_particles(s, P, ids)


def _L(wl):
    return (wl.nx * wl.dx, wl.ny * wl.dy, wl.nz * wl.dz)


# ---------------------------------------------------------------- sort (a1)

@pytest.mark.parametrize("S", [1, 2, 4])
def test_sort_permutation_bit_exact(pic, oracle_mod, S):
    from synth import get_config, gen_particles
    wl = get_config("T_small").with_(supercell=S)
    parts = gen_particles(wl)
    P, ids = parts[0]
    rng = np.random.default_rng(5)
    perm = rng.permutation(P.shape[1])          # scramble the input order
    P, ids = P[:, perm].copy(), ids[perm].copy()
    P[:3, ::5] = np.floor(P[:3, ::5])           # particles exactly on cell faces
    P[:, 1::9] = P[:, 0::9][:, :P[:, 1::9].shape[1]]   # exact duplicates (ties)
    orc = _oracle_for(oracle_mod, wl, [(P, ids)])
    orc.sort()
    sim = _sim(pic, wl)
    sim.set_particles(0, P, ids)
    gP, gids = sim.get_particles(0)
    assert np.array_equal(gids, orc.ids[0])
    assert np.array_equal(gP, orc.P[0])


def test_sort_large_buckets_and_empty_cells(pic, oracle_mod):
    from synth import get_config
    wl = get_config("T_small").with_(supercell=2)
    rng = np.random.default_rng(6)
    n = 3000
    P = np.zeros((6, n))
    # 70% of the particles in 3 cells (buckets > 32 and > 1024 entries), rest spread
    hot = rng.random(n) < 0.7
    P[0] = np.where(hot, 3 + rng.random(n) * 0.999, rng.random(n) * 8)
    P[1] = np.where(hot, 5.5, rng.random(n) * 12)
    P[2] = np.where(hot, 7 + (rng.random(n) < 0.5), rng.random(n) * 16)
    P[3:] = rng.standard_normal((3, n))
    ids = rng.permutation(n).astype(np.uint64)
    orc = _oracle_for(oracle_mod, wl, [(P, ids)])
    orc.sort()
    sim = _sim(pic, wl, counts=[n])
    sim.set_particles(0, P, ids)
    gP, gids = sim.get_particles(0)
    assert np.array_equal(gids, orc.ids[0])
    assert np.array_equal(gP, orc.P[0])


@pytest.mark.parametrize("case", ["wide_supercell", "over_smem_stage"])
def test_sort_order_kernel_paths(pic, oracle_mod, case):
    """The per-supercell order kernel's other paths, bit-exact against the
    oracle's stable sort: S = 8 (512 cells per supercell: the slot position
    counted cell by cell instead of from slot tables) and 100 particles per
    cell at S = 4 (6400 per supercell: more than the kernel stages in shared
    memory, buckets ordered through global scratch)."""
    from synth import Workload, gen_particles
    from synth.configs import electron
    if case == "wide_supercell":
        wl = Workload("wide", 8, 8, 16, (electron(4, 0.05),), steps=1, sort_every=1, supercell=8)
    else:
        wl = Workload("full", 8, 8, 4, (electron(100, 0.05),), steps=1, sort_every=1, supercell=4)
    P, ids = gen_particles(wl)[0]
    perm = np.random.default_rng(11).permutation(P.shape[1])
    P, ids = P[:, perm].copy(), ids[perm].copy()
    orc = _oracle_for(oracle_mod, wl, [(P, ids)])
    orc.sort()
    sim = _sim(pic, wl)
    sim.set_particles(0, P, ids)
    gP, gids = sim.get_particles(0)
    assert np.array_equal(gids, orc.ids[0])
    assert np.array_equal(gP, orc.P[0])
    sim.step(2)   # a re-sort of the pushed state; the particles stay valid and complete
    gP2, gids2 = sim.get_particles(0)
    assert np.array_equal(np.sort(gids2), np.sort(ids))


@pytest.mark.parametrize("S,K", [(4, 3), (2, 2)])
def test_in_step_sort_order_bit_exact(pic, oracle_mod, S, K):
    """The sorts inside the step (of the store the pushes left, as opposed to
    the host input pic_set_particles sorts) give the oracle's permutation bit
    for bit after every re-sort: the particle order of the GPU store equals
    the oracle's array order (both sort at the start of steps n = 0, K, 2K,
    ...; fast particles, sigma 0.3, so many change supercell between sorts)."""
    from synth import get_config, gen_particles
    from synth.configs import electron
    wl = get_config("C1").with_(species=(electron(5, 0.3),), supercell=S, sort_every=K)
    parts = gen_particles(wl)
    orc = _oracle_for(oracle_mod, wl, parts)
    sim = _sim(pic, wl)
    _load(sim, parts)
    orc.sort()
    for step in range(3 * K + 1):
        orc.step(1)
        sim.step(1)
        if step % K == 0:   # this step began with a sort
            gP, gids = sim.get_particles(0)
            assert np.array_equal(gids, orc.ids[0]), step
            L = _L(wl)
            assert pos_err(gP[:3], orc.P[0][:3], L) <= TOL_STEP


# ---------------------------------------------------------------- fields (a7)

def test_fdtd_random_fields_vs_oracle(pic, oracle_mod):
    from synth import get_config
    wl = get_config("T_small").with_(dx=1.1, dy=0.9, dz=1.3)
    rng = np.random.default_rng(7)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx))
    orc = _oracle_for(oracle_mod, wl, [(np.zeros((6, 0)), np.zeros(0, np.uint64))])
    orc.F[:6] = F6
    sim = _sim(pic, wl, counts=[0])
    sim.set_fields(F6)
    for _ in range(5):
        orc.b_half(); orc.e_full(); orc.b_half()
        sim.step(1)
    G = sim.get_fields()
    errs = field_errs(G[:6], orc.F[:6])
    assert max(errs) <= TOL_STEP, errs
    assert not G[6:].any()


def test_per_component_field_entry_points(pic):
    """pic_set_fields6 / pic_get_fields9 (SURVEY.md sec. 8b's f[6] / f[9]
    signatures) agree bit for bit with the packed pic_set_fields /
    pic_get_fields, including after steps with particles (J)."""
    from synth import get_config, gen_particles
    wl = get_config("T_small")
    rng = np.random.default_rng(19)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.05
    a, b = _sim(pic, wl), _sim(pic, wl)
    parts = gen_particles(wl)
    _load(a, parts)
    _load(b, parts)
    a.set_fields(F6)
    b.set_fields_components([F6[c] for c in range(6)])
    assert np.array_equal(a.get_fields()[:6], F6)
    a.step(3)
    b.step(3)
    G = a.get_fields()
    comps = b.get_fields_components()
    for c in range(9):
        assert np.allclose(comps[c], G[c], rtol=0, atol=1e-13 * max(np.abs(G[c]).max(), 1e-300)), c
    only = a.get_fields_components([6, 8])
    assert sorted(only) == [6, 8] and np.array_equal(only[8], G[8])


def test_vacuum_plane_wave_on_gpu(pic):
    # discrete Yee eigenmode along z, E along x (closed form)
    from synth import get_config
    wl = get_config("T_small")
    nz, dt = wl.nz, wl.dt
    k = 2 * math.pi / nz
    w = 2 / dt * math.asin(dt * math.sin(k / 2))
    z = np.arange(nz)
    F6 = np.zeros((6, wl.nz, wl.ny, wl.nx))
    F6[0] = np.cos(k * z)[:, None, None]
    F6[4] = (math.cos(w * dt / 2) * np.cos(k * (z + 0.5)))[:, None, None]
    sim = _sim(pic, wl, counts=[0])
    sim.set_fields(F6)
    n = 200
    sim.step(n)
    G = sim.get_fields()
    t = n * dt
    np.testing.assert_allclose(G[0], np.broadcast_to(np.cos(k * z - w * t)[:, None, None], G[0].shape),
                               rtol=0, atol=1e-12)
    np.testing.assert_allclose(
        G[4], np.broadcast_to((math.cos(w * dt / 2) * np.cos(k * (z + 0.5) - w * t))[:, None, None],
                              G[4].shape), rtol=0, atol=1e-12)


# ---------------------------------------------------------------- whole step

def _run_parity(pic, oracle_mod, wl, nsteps, teacher_forced, flags=0, fields=None, tol=TOL_STEP):
    from synth import gen_particles
    parts = gen_particles(wl)
    orc = _oracle_for(oracle_mod, wl, parts)
    if fields is not None:
        orc.F[:6] = fields
    sim = _sim(pic, wl, flags=flags)
    L = _L(wl)
    worst = 0.0
    for step in range(nsteps):
        if teacher_forced or step == 0:
            sim.set_fields(orc.F[:6].copy())
            for s in range(len(wl.species)):
                sim.set_particles(s, orc.P[s], orc.ids[s])
        orc.step(1)
        sim.step(1)
        G = sim.get_fields()
        ferr = field_errs(G, orc.F)
        errs = list(ferr)
        for s in range(len(wl.species)):
            gP, gi = sim.get_particles(s)
            pe, ue = compare_state(gP, gi, orc.P[s], orc.ids[s], L)
            errs += [pe, ue]
        worst = max(worst, max(errs))
        assert max(errs) <= tol, (step, errs)
    return worst


def test_c1_teacher_forced_per_step(pic, oracle_mod):
    from synth import get_config
    wl = get_config("C1")
    _run_parity(pic, oracle_mod, wl, wl.steps, teacher_forced=True)


def test_c1_free_running_matches_oracle(pic, oracle_mod):
    from synth import get_config
    wl = get_config("C1")
    _run_parity(pic, oracle_mod, wl, 100, teacher_forced=False, tol=TOL_FREE)


@pytest.mark.parametrize("name", ["T_small", "T_two_species"])
def test_small_configs_free_running(pic, oracle_mod, name):
    from synth import get_config
    wl = get_config(name)
    rng = np.random.default_rng(9)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.02
    _run_parity(pic, oracle_mod, wl, 12, teacher_forced=False, fields=F6, tol=TOL_STEP * 100)


def test_nonunit_cells_and_strong_fields(pic, oracle_mod):
    from synth import get_config
    wl = get_config("T_two_species").with_(dx=0.8, dy=1.2, dz=1.05, supercell=4)
    rng = np.random.default_rng(10)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.5
    _run_parity(pic, oracle_mod, wl, 6, teacher_forced=True, fields=F6)


def test_sudden_acceleration_takes_the_fp64_deposit(pic, oracle_mod):
    """A cold plasma (sigma 1e-4) put into strong fields: in the first step
    every particle speeds up far beyond the 2x headroom of the fixed-point
    scale set from the previous speed bound, so its segments fail the range
    check and go to the fp64 global J (deposit_seg's fallback); the next
    steps use the tile again with the new bound.  Free running against the
    oracle.  (Round 1 checked with a debug build that flags the fallback that
    this case takes it and C1 does not.)"""
    from synth import get_config
    from synth.configs import electron, proton
    wl = get_config("T_two_species").with_(species=(electron(3, 1e-4), proton(3, 1e-4)), supercell=4)
    rng = np.random.default_rng(12)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.2
    F6[0] += 1.5                       # a uniform Ex on top: |du| ~ 0.4 per step
    _run_parity(pic, oracle_mod, wl, 4, teacher_forced=False, fields=F6, tol=1e-11)


def test_remainder_queue_overflow(pic, oracle_mod):
    """6400 hot particles per supercell (100 ppc, sigma 0.5): about a third of
    them cross a cell face every step, far more than the CTA's remainder
    queue holds (160), so the overflowing paths deposit their rest inline;
    free running against the oracle."""
    from synth import Workload
    from synth.configs import electron
    wl = Workload("hot", 8, 8, 8, (electron(100, 0.5),), steps=4, sort_every=2, supercell=4)
    _run_parity(pic, oracle_mod, wl, 4, teacher_forced=False, tol=1e-11)


def test_tile_fallback_after_long_drift(pic, oracle_mod):
    """No re-sort for 30 steps at sigma 0.3: particles drift beyond the
    tile halo and take the global fallback path of the fused kernel."""
    from synth import get_config
    from synth.configs import electron
    wl = get_config("C1").with_(species=(electron(4, 0.3),), sort_every=0, nx=16, ny=16, nz=8)
    _run_parity(pic, oracle_mod, wl, 30, teacher_forced=False, tol=1e-10)


def test_two_species_launch_fallback_and_queues(pic, oracle_mod):
    """Both species in one fused launch (one concatenated particle loop):
    fast electrons and protons drift beyond the tile halo without re-sorts
    (global fallback queue, species recovered from the queued index), cross
    faces often (remainder queue, species in the queued cell's top bit), and
    share the J tile with the smaller of the two fixed-point scales."""
    from synth import get_config
    from synth.configs import electron, proton
    wl = get_config("C1").with_(species=(electron(3, 0.3), proton(2, 200.0)), sort_every=0,
                                nx=16, ny=16, nz=8)
    rng = np.random.default_rng(14)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.05
    _run_parity(pic, oracle_mod, wl, 25, teacher_forced=False, fields=F6, tol=1e-10)


@pytest.mark.parametrize("uz", [3.0, -3.0])
def test_occupied_layers_follow_a_streaming_slab(pic, oracle_mod, uz):
    """Particles in 3 of 16 supercell layers streaming at 0.95 c along +z or
    -z (0.54 cells per step at Courant 0.99, 5.4 per sort interval K = 10):
    the particle kernel is launched over the occupied layers only
    (runtime.cu push_layers), so the widened range of each sorting step has
    to cover every particle, including the slab wrapping through the
    periodic z end (-z); the sorts' per-supercell order kernel runs over the
    same widened layers, so the store's order after every sort must still be
    the oracle's permutation.  40 steps free running against the oracle."""
    from synth import get_config
    from synth.configs import electron
    wl = get_config("C1").with_(species=(electron(2, 0.05),), nz=64, sort_every=10, courant=0.99)
    rng = np.random.default_rng(31)
    L = _L(wl)
    n = wl.nx * wl.ny * 8 * 2
    P = np.empty((6, n))
    P[0] = rng.uniform(0.0, L[0], n)
    P[1] = rng.uniform(0.0, L[1], n)
    P[2] = rng.uniform(2.0 * wl.dz, 10.0 * wl.dz, n)   # supercell layers 0..2
    P[3:5] = rng.normal(0.0, 0.05, (2, n))
    P[5] = uz + rng.normal(0.0, 0.05, n)
    parts = [(P, np.arange(n, dtype=np.uint64))]
    orc = _oracle_for(oracle_mod, wl, parts)
    sim = _sim(pic, wl, counts=[n])
    _load(sim, parts)
    orc.sort()
    for step in range(40):
        orc.step(1)
        sim.step(1)
        errs = list(field_errs(sim.get_fields(), orc.F))
        gP, gi = sim.get_particles(0)
        errs += list(compare_state(gP, gi, orc.P[0], orc.ids[0], L))
        assert max(errs) <= 1e-10, (step, errs)
        if step % wl.sort_every == 0:   # the sort of this step (its per-supercell order
            assert np.array_equal(gi, orc.ids[0]), step   # kernel ran over the widened layers)
    zc = np.floor(orc.P[0][2] / wl.dz)
    assert (zc < 2).any() or (zc >= 10).any()   # the slab left its starting layers


def test_reupload_moves_the_occupied_layers(pic, oracle_mod):
    """A slab in layers 10..12 of 32 runs 7 steps, then the particles are
    replaced by a slab in layers 22..25 (pic_set_particles between steps, the oracle's
    state replaced alike): the J planes the last step before the re-upload
    deposited into must still be cleared (runtime.cu j_planes of the
    previous step's layers) while the kernel now runs over the new layers.
    Free running against the oracle on both sides of the re-upload."""
    from synth import get_config
    from synth.configs import electron
    wl = get_config("C1").with_(species=(electron(2, 0.1),), nz=128, sort_every=10)
    L = _L(wl)

    def slab(z0, z1, seed, id0):
        rng = np.random.default_rng(seed)
        n = wl.nx * wl.ny * 8 * 2
        P = np.empty((6, n))
        P[0] = rng.uniform(0.0, L[0], n)
        P[1] = rng.uniform(0.0, L[1], n)
        P[2] = rng.uniform(z0 * wl.dz, z1 * wl.dz, n)
        P[3:] = rng.normal(0.0, 0.1, (3, n))
        return P, np.arange(id0, id0 + n, dtype=np.uint64)

    parts = [slab(40.0, 50.0, 41, 0)]   # far from the periodic ends: no wrap-around widening
    orc = _oracle_for(oracle_mod, wl, parts)
    sim = _sim(pic, wl, counts=[parts[0][0].shape[1]])
    _load(sim, parts)

    def check(step):
        errs = list(field_errs(sim.get_fields(), orc.F))
        gP, gi = sim.get_particles(0)
        errs += list(compare_state(gP, gi, orc.P[0], orc.ids[0], L))
        assert max(errs) <= 1e-10, (step, errs)

    for step in range(7):
        orc.step(1)
        sim.step(1)
        check(step)
    P2, i2 = slab(90.0, 100.0, 42, 10 ** 6)
    orc.P[0], orc.ids[0] = P2.copy(), i2.copy()
    sim.set_particles(0, P2, i2)
    for step in range(7, 20):
        orc.step(1)
        sim.step(1)
        check(step)


def test_naive_flag_path(pic, oracle_mod):
    from synth import get_config
    wl = get_config("T_small")
    _run_parity(pic, oracle_mod, wl, 4, teacher_forced=True, flags=pic.FLAG_NAIVE)


def test_frozen_plasma_bitwise(pic):
    from synth import get_config, gen_particles
    wl = get_config("C1").with_(species=(get_config("C1").species[0].__class__(
        "electron", -1.0, 1.0, 8, 0.0),), sort_every=5)
    parts = gen_particles(wl)
    sim = _sim(pic, wl)
    _load(sim, parts)
    P0, i0 = sim.get_particles(0)
    sim.step(23)
    P1, i1 = sim.get_particles(0)
    assert np.array_equal(i0, i1)
    assert np.array_equal(P0, P1)
    assert not sim.get_fields().any()


# ---------------------------------------------------------------- edge cases

def test_empty_species_and_capacity_errors(pic):
    from synth import get_config, gen_particles
    wl = get_config("T_two_species")
    parts = gen_particles(wl)
    sim = _sim(pic, wl)
    sim.set_particles(0, *parts[0])            # species 1 stays empty
    sim.step(3)
    assert sim.count(1) == 0
    big = np.zeros((6, parts[0][0].shape[1] + 1))
    with pytest.raises(pic.PicError) as e:
        sim.set_particles(0, big, np.zeros(big.shape[1], np.uint64))
    assert e.value.code == -3
    bad = parts[0][0].copy()
    bad[0, 0] = wl.nx * wl.dx     # x == L is outside [0, L)
    with pytest.raises(pic.PicError) as e:
        sim.set_particles(0, bad, parts[0][1])
    assert e.value.code == -1


def test_nonfinite_momentum_is_reported(pic):
    from synth import get_config, gen_particles
    wl = get_config("T_small")
    P, ids = gen_particles(wl)[0]
    P = P.copy()
    P[3, 7] = np.nan
    sim = _sim(pic, wl)
    sim.set_particles(0, P, ids)
    with pytest.raises(pic.PicError) as e:
        sim.step(1)
    assert e.value.code == -6


def test_cfl_violation_rejected(pic):
    with pytest.raises(pic.PicError):
        pic.Simulation(pic.make_config(8, 8, 8, [(-1.0, 1.0, 1.0)], dt=0.6, capacity=[10]))


def test_tiny_grid_supercell_one(pic, oracle_mod):
    from synth import Workload
    from synth.configs import electron
    wl = Workload("tiny", 2, 3, 1, (electron(5, 0.2),), steps=5, sort_every=2, supercell=1)
    rng = np.random.default_rng(12)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.1
    _run_parity(pic, oracle_mod, wl, 5, teacher_forced=False, fields=F6, tol=1e-11)


# ---------------------------------------------------------------- full size (C2), sampled

def test_c2_full_size_sampled_and_properties(pic, oracle_mod):
    """C2 at full size in the bench launch configuration: after 25 steps,
    (a) sampled particles' next step equals the oracle's per-particle gather/
    Boris/move on the GPU's own fields; (b) continuity and total current hold
    for the GPU's own deposit."""
    from synth import get_config, gen_particles
    wl = get_config("C2")
    parts = gen_particles(wl)
    sim = _sim(pic, wl)
    _load(sim, parts)
    sim.step(25)
    F = sim.get_fields()
    P0, i0 = sim.get_particles(0)
    sim.step(1)
    F1 = sim.get_fields()
    P1, i1 = sim.get_particles(0)
    # sort happens at step 40, not 25: same order
    assert np.array_equal(i0, i1)
    orc = _oracle_for(oracle_mod, wl, [(np.zeros((6, 0)), np.zeros(0, np.uint64))])
    orc.F[:] = F
    O = oracle_mod
    sp = wl.species[0]
    rng = np.random.default_rng(13)
    sample = rng.choice(P0.shape[1], 2000, replace=False)
    L = np.array(_L(wl))
    for p in sample:
        EB = orc.gather(*P0[:3, p])
        u = O.boris(sp.q, sp.m, wl.c, wl.dt, EB, P0[3:, p])
        xn = O.move(wl.c, wl.dt, u, P0[:3, p])
        xn = np.array([O.wrap(xn[d], L[d]) for d in range(3)])
        assert rel_err(P1[3:, p], u) <= TOL_STEP
        d = (P1[:3, p] - xn + L / 2) % L - L / 2
        assert np.abs(d).max() <= TOL_STEP * L.max()
    # continuity with the GPU's J^{n+1/2} and positions
    rho0 = orc.rho_of(0, P0)
    rho1 = orc.rho_of(0, P1)
    orc.F[6:] = F1[6:]
    divj = orc.div_edge(6)
    res = (rho1 - rho0) / wl.dt + divj
    assert np.abs(res).max() <= 1e-12 * np.abs(divj).max() + 1e-15
    # total current = sum q w v
    v = (((P1[:3] - P0[:3]) + L[:, None] / 2) % L[:, None] - L[:, None] / 2) / wl.dt
    tot = sp.q * sp.w * v.sum(axis=1)
    got = F1[6:].sum(axis=(1, 2, 3))
    np.testing.assert_allclose(got, tot, rtol=1e-9, atol=1e-12 * np.abs(tot).max())


# ---------------------------------------------------------------- z slabs (a8, sec. 8e)

def _slab_group(pic, wl, nranks, stream):
    sims = []
    for r in range(nranks):
        cfg = pic.workload_config(wl, rank=r, nranks=nranks, flags=pic.FLAG_LOCAL_GROUP,
                                  migrate_capacity=4096)
        sims.append(pic.Simulation(cfg, stream=stream))
    return sims


@pytest.mark.parametrize("nranks,nz", [(2, 16), (4, 16), (2, 32)])
def test_slab_decomposition_matches_single_domain_oracle(pic, oracle_mod, nranks, nz):
    """The z-slab path (J ghost planes summed by the owner, E/B ghost planes,
    particle migration, unsorted arrivals tail) run as an in-process group of
    slab contexts on one GPU, against the single-domain oracle (P16).  With
    nz = 32 over 2 ranks each slab has 4 supercell layers: the step pushes
    the boundary layers 0 and 3 first, exchanges, then the interior layers
    1 and 2 (the overlap order of a NCCL step)."""
    import torch
    from synth import gen_particles, get_config
    from synth.configs import electron
    wl = get_config("C1").with_(species=(electron(6, 0.2),), nz=nz, sort_every=5)
    parts = gen_particles(wl)
    rng = np.random.default_rng(21)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.02
    orc = _oracle_for(oracle_mod, wl, parts)
    orc.F[:6] = F6
    stream = torch.cuda.Stream()
    sims = _slab_group(pic, wl, nranks, stream)
    nzl = wl.nz // nranks
    for r, sim in enumerate(sims):
        sim.set_particles(0, *parts[0])
        sim.set_fields(F6[:, r * nzl:(r + 1) * nzl].copy())
    L = _L(wl)
    migrated = 0
    for step in range(15):
        orc.step(1)
        pic.step_group(sims, 1)
        G = np.concatenate([s.get_fields() for s in sims], axis=1)
        Ps, Is = zip(*[s.get_particles(0) for s in sims])
        gP, gi = np.concatenate(Ps, axis=1), np.concatenate(Is)
        for r, (P_r, _) in enumerate(zip(Ps, Is)):   # every particle lives in its rank's slab
            assert (P_r[2] >= r * nzl * wl.dz).all() and (P_r[2] < (r + 1) * nzl * wl.dz).all()
        pe, ue = compare_state(gP, gi, orc.P[0], orc.ids[0], L)
        errs = field_errs(G, orc.F) + [pe, ue]
        assert max(errs) <= 1e-11, (step, errs)
        migrated += sum(P_r.shape[1] for P_r in Ps)
    assert migrated > 0


@pytest.mark.parametrize("S", [4, 2])
def test_slab_decomposition_halo_two(pic, oracle_mod, S):
    """The z-slab path with the h = 2 tiles (S = 4: one 512-thread CTA per
    SM) and the boundary/interior split (2 slabs of 16 planes), two species
    at sigma 0.3 drifting out of the sorted order between K = 5 sorts,
    against the single-domain oracle."""
    import torch
    from synth import gen_particles, get_config
    from synth.configs import electron, proton
    wl = get_config("C1").with_(species=(electron(3, 0.3), proton(2, 200.0)), nz=32, sort_every=5,
                                supercell=S, halo=2)
    parts = gen_particles(wl)
    rng = np.random.default_rng(24)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.02
    orc = _oracle_for(oracle_mod, wl, parts)
    orc.F[:6] = F6
    stream = torch.cuda.Stream()
    sims = [pic.Simulation(pic.workload_config(wl, rank=r, nranks=2, flags=pic.FLAG_LOCAL_GROUP,
                                               migrate_capacity=4096), stream=stream) for r in range(2)]
    for r, sim in enumerate(sims):
        for sp, (P, ids) in enumerate(parts):
            sim.set_particles(sp, P, ids)
        sim.set_fields(F6[:, r * 16:(r + 1) * 16].copy())
    L = _L(wl)
    for step in range(12):
        orc.step(1)
        pic.step_group(sims, 1)
        G = np.concatenate([s.get_fields() for s in sims], axis=1)
        errs = field_errs(G, orc.F)
        for sp in range(2):
            Ps, Is = zip(*[sim.get_particles(sp) for sim in sims])
            errs += list(compare_state(np.concatenate(Ps, axis=1), np.concatenate(Is), orc.P[sp], orc.ids[sp], L))
        assert max(errs) <= 1e-11, (step, errs)


def test_slab_migration_capacity_error(pic):
    import torch
    from synth import gen_particles, get_config
    from synth.configs import electron
    wl = get_config("C1").with_(species=(electron(8, 0.3),), nz=16, sort_every=5)
    parts = gen_particles(wl)
    stream = torch.cuda.Stream()
    sims = []
    for r in range(2):
        cfg = pic.workload_config(wl, rank=r, nranks=2, flags=pic.FLAG_LOCAL_GROUP, migrate_capacity=4)
        sims.append(pic.Simulation(cfg, stream=stream))
    for sim in sims:
        sim.set_particles(0, *parts[0])
    with pytest.raises(pic.PicError) as e:
        pic.step_group(sims, 3)
    assert e.value.code == -3


def test_supercell_two_tile_kernel(pic, oracle_mod):
    """S = 2 instantiation of the fused kernel (6^3 E/B tile) against the oracle."""
    from synth import get_config
    wl = get_config("T_two_species").with_(supercell=2, sort_every=3)
    rng = np.random.default_rng(22)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.05
    _run_parity(pic, oracle_mod, wl, 8, teacher_forced=False, fields=F6, tol=1e-11)


@pytest.mark.parametrize("S", [4, 2])
def test_halo_two_tile_kernel(pic, oracle_mod, S):
    """Tile drift halo h = 2 (pic_config.halo; SURVEY.md sec. 8b "supercell
    S, halo h"): (S + 6)^3 E/B and (S + 7)^3 J tiles -- at S = 4 one CTA of
    512 threads per SM -- against the oracle, two species in one launch,
    fast enough (sigma 0.3, no re-sort for 20 steps) that particles drift
    past 1 and past 2 cells out of their supercell (tile and global paths)."""
    from synth import get_config
    from synth.configs import electron, proton
    wl = get_config("C1").with_(species=(electron(3, 0.3), proton(2, 200.0)), sort_every=0,
                                nx=16, ny=16, nz=8, supercell=S, halo=2)
    rng = np.random.default_rng(40 + S)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.05
    _run_parity(pic, oracle_mod, wl, 20, teacher_forced=False, fields=F6, tol=1e-10)


def test_halo_two_c1_teacher_forced(pic, oracle_mod):
    """C1 per step at h = 2 with the sort every 5 steps: <= 1e-12."""
    from synth import get_config
    wl = get_config("C1").with_(halo=2, sort_every=5)
    _run_parity(pic, oracle_mod, wl, wl.steps, teacher_forced=True)


def test_halo_rejected_out_of_range(pic):
    with pytest.raises(pic.PicError):
        cfg = pic.make_config(8, 8, 8, [(-1.0, 1.0, 1.0)], dt=0.25, capacity=[10], halo=3)
        pic.Simulation(cfg)


def test_dense_supercell_global_path(pic, oracle_mod):
    """Uniformly dense supercells (19200 particles each, more than the
    fixed-point tile counters allow in one CTA): the launch splits each over
    several CTAs (mean > 8192 per supercell), each within the counter bound;
    results unchanged."""
    from synth import Workload
    from synth.configs import electron
    wl = Workload("dense", 8, 8, 8, (electron(300, 0.05),), steps=2, sort_every=2, supercell=4)
    _run_parity(pic, oracle_mod, wl, 2, teacher_forced=True, tol=1e-12)


def test_one_overdense_supercell_takes_the_global_path(pic, oracle_mod):
    """One supercell holding 17000 particles while the mean stays low (no
    split): its CTA exceeds the fixed-point counter bound (16383), so every
    one of its particles is pushed and deposited by the global fp64 path
    (outside-tile queue, then inline once the queue is full) while the other
    CTAs use the tile; per step against the oracle."""
    from synth import Workload, gen_particles
    from synth.configs import electron
    wl = Workload("overdense", 8, 8, 8, (electron(2, 0.05),), steps=3, sort_every=2, supercell=4)
    P0, i0 = gen_particles(wl)[0]
    rng = np.random.default_rng(31)
    m = 17000
    Pd = np.empty((6, m))
    Pd[:3] = rng.random((3, m)) * 4.0          # supercell (0, 0, 0): cells [0, 4)^3
    Pd[3:] = rng.standard_normal((3, m)) * 0.05
    P = np.concatenate([P0, Pd], axis=1)
    ids = np.arange(P.shape[1], dtype=np.uint64) + 7
    orc = _oracle_for(oracle_mod, wl, [(P, ids)])
    sim = _sim(pic, wl, counts=[P.shape[1]])
    L = _L(wl)
    for step in range(3):
        sim.set_fields(orc.F[:6].copy())
        sim.set_particles(0, orc.P[0], orc.ids[0])
        orc.step(1)
        sim.step(1)
        errs = field_errs(sim.get_fields(), orc.F)
        gP, gi = sim.get_particles(0)
        errs += list(compare_state(gP, gi, orc.P[0], orc.ids[0], L))
        assert max(errs) <= TOL_STEP, (step, errs)


def test_particles_on_faces_and_corners(pic, oracle_mod):
    """Start points exactly on cell faces / edges / corners and moves that end
    on faces (zero-length pieces of the VB split)."""
    from synth import get_config
    wl = get_config("T_small").with_(sort_every=1)
    from synth import gen_particles
    P, ids = gen_particles(wl)[0]
    P = P.copy()
    P[0, ::3] = np.floor(P[0, ::3])                  # x on a face
    P[:2, 1::7] = np.floor(P[:2, 1::7])              # x, y on an edge
    P[:3, 2::11] = np.floor(P[:3, 2::11])            # corner
    P[3:, 5::13] = 0.0                               # at rest
    orc = _oracle_for(oracle_mod, wl, [(P, ids)])
    sim = _sim(pic, wl)
    sim.set_particles(0, P, ids)
    rng = np.random.default_rng(23)
    F6 = rng.standard_normal((6, wl.nz, wl.ny, wl.nx)) * 0.03
    orc.F[:6] = F6
    sim.set_fields(F6)
    for _ in range(3):
        orc.step(1)
        sim.step(1)
        G = sim.get_fields()
        gP, gi = sim.get_particles(0)
        pe, ue = compare_state(gP, gi, orc.P[0], orc.ids[0], _L(wl))
        assert max(field_errs(G, orc.F) + [pe, ue]) <= 1e-12


@pytest.mark.slow
def test_c3_full_size_two_species_sampled_and_continuity(pic, oracle_mod):
    """C3 (128^3, 25 e + 25 p per cell, 104.9M particles) at full size in the
    bench launch configuration, after 25 steps (one re-sort at step 20):
    sampled particles of both species against the oracle's per-particle
    gather / Boris / move on the GPU's own fields, and discrete charge
    continuity of the GPU's deposit on the whole grid (oracle CIC rho)."""
    from synth import get_config, gen_particles
    wl = get_config("C3")
    parts = gen_particles(wl)
    sim = _sim(pic, wl)
    _load(sim, parts)
    del parts
    sim.step(25)
    F0 = sim.get_fields()
    P0 = [sim.get_particles(s) for s in range(2)]
    sim.step(1)
    F1 = sim.get_fields()
    P1 = [sim.get_particles(s) for s in range(2)]
    orc = _oracle_for(oracle_mod, wl, [(np.zeros((6, 0)), np.zeros(0, np.uint64))] * 2)
    orc.F[:] = F0
    O = oracle_mod
    L = np.array(_L(wl))
    rng = np.random.default_rng(31)
    for s, sp in enumerate(wl.species):
        (A, ia), (B, ib) = P0[s], P1[s]
        assert np.array_equal(ia, ib)            # no re-sort between the two states
        for p in rng.choice(A.shape[1], 500, replace=False):
            EB = orc.gather(*A[:3, p])
            u = O.boris(sp.q, sp.m, wl.c, wl.dt, EB, A[3:, p])
            xn = O.move(wl.c, wl.dt, u, A[:3, p])
            xn = np.array([O.wrap(xn[d], L[d]) for d in range(3)])
            assert rel_err(B[3:, p], u) <= TOL_STEP
            d = (B[:3, p] - xn + L / 2) % L - L / 2
            assert np.abs(d).max() <= TOL_STEP * L.max()
    rho0 = sum(orc.rho_of(s, P0[s][0]) for s in range(2))
    rho1 = sum(orc.rho_of(s, P1[s][0]) for s in range(2))
    orc.F[6:] = F1[6:]
    divj = orc.div_edge(6)
    res = (rho1 - rho0) / wl.dt + divj
    assert np.abs(res).max() <= 1e-12 * np.abs(divj).max() + 1e-15


def test_c4_full_size_sampled(pic, oracle_mod):
    """C4 at N = 1 (256 x 256 x 128, 32 e per cell, 268M particles -- the
    per-GPU shape of the weak-scaling bench) in the bench launch
    configuration, 25 steps (one re-sort at step 20): sampled particles
    against the oracle's per-particle gather / Boris / move on the GPU's own
    fields."""
    from synth import get_config, gen_particles
    wl = get_config("C4")
    parts = gen_particles(wl)
    sim = _sim(pic, wl)
    _load(sim, parts)
    del parts
    sim.step(25)
    F0 = sim.get_fields()
    A, ia = sim.get_particles(0)
    sim.step(1)
    B, ib = sim.get_particles(0)
    assert np.array_equal(ia, ib)
    orc = _oracle_for(oracle_mod, wl, [(np.zeros((6, 0)), np.zeros(0, np.uint64))])
    orc.F[:] = F0
    O = oracle_mod
    L = np.array(_L(wl))
    sp = wl.species[0]
    rng = np.random.default_rng(35)
    for p in rng.choice(A.shape[1], 800, replace=False):
        EB = orc.gather(*A[:3, p])
        u = O.boris(sp.q, sp.m, wl.c, wl.dt, EB, A[3:, p])
        xn = O.move(wl.c, wl.dt, u, A[:3, p])
        xn = np.array([O.wrap(xn[d], L[d]) for d in range(3)])
        assert rel_err(B[3:, p], u) <= TOL_STEP
        d = (B[:3, p] - xn + L / 2) % L - L / 2
        assert np.abs(d).max() <= TOL_STEP * L.max()
