"""Pins of the CPU oracle against what the paper and the mathematics fix
(DESIGN.md sec. 5).  CPU only (-m "not gpu")."""
import math

import numpy as np
import pytest

from tests import brute

DT = 0.5 / math.sqrt(3.0)


def make(O, nx, ny, nz, species=((-1.0, 1.0, 1.0),), dx=1.0, dy=1.0, dz=1.0, c=1.0,
         dt=None, S=1, K=0):
    if dt is None:
        dt = 0.5 / (c * math.sqrt(1 / dx ** 2 + 1 / dy ** 2 + 1 / dz ** 2))
    g = O.Grid(nx, ny, nz, dx, dy, dz, dt, c,
               [O.Species(q, m, w) for (q, m, w) in species], S, K)
    return g


# ---------------- P1 / P2 : CIC gather ----------------

def test_p1_uniform_field_partition_of_unity(oracle_mod):
    O = oracle_mod
    g = make(O, 5, 6, 7, dx=0.7, dy=1.3, dz=1.1)
    orc = O.Oracle(g)
    vals = np.array([1.5, -2.25, 3.0, 0.125, -7.5, 1e-3])
    orc.F[:6] = vals[:, None, None, None]
    rng = np.random.default_rng(1)
    L = np.array([5 * 0.7, 6 * 1.3, 7 * 1.1])
    for _ in range(200):
        x = rng.random(3) * L
        got = orc.gather(*x)
        np.testing.assert_allclose(got, vals, rtol=4.5e-16, atol=0)


def test_p1_node_and_centre_weights(oracle_mod):
    O = oracle_mod
    g = make(O, 4, 4, 4)
    orc = O.Oracle(g)
    rng = np.random.default_rng(2)
    orc.F[:6] = rng.standard_normal((6, 4, 4, 4))
    # Ey lives at (i, j+1/2, k): a particle exactly there sees that node only
    got = orc.gather(2.0, 1.5, 3.0)
    assert got[1] == orc.F[1, 3, 1, 2]
    # Bz lives at (i+1/2, j+1/2, k): the cell centre (2.5,1.5,3.5) averages 2 nodes in z
    got = orc.gather(2.5, 1.5, 3.5)
    assert got[5] == pytest.approx(0.5 * (orc.F[5, 3, 1, 2] + orc.F[5, 0, 1, 2]), rel=1e-15)


def test_p2_gather_bruteforce_hats(oracle_mod):
    O = oracle_mod
    h = (0.9, 1.2, 1.05)
    g = make(O, 3, 4, 5, dx=h[0], dy=h[1], dz=h[2])
    orc = O.Oracle(g)
    rng = np.random.default_rng(3)
    orc.F[:6] = rng.standard_normal((6, 5, 4, 3))
    L = np.array([3, 4, 5]) * np.array(h)
    for _ in range(100):
        x = rng.random(3) * L
        got = orc.gather(*x)
        ref = brute.hat_gather(orc.F[:6], h, x)
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14 * np.abs(orc.F).max())


# ---------------- P3 / P4 / P5 / P6 : Boris and move ----------------

@pytest.mark.parametrize("q", [-1.0, 1.0])
def test_p3_cyclotron_rotation_and_speed(oracle_mod, q):
    O = oracle_mod
    B0, m, c, dt = 1.0, 1.0, 1.0, DT
    u0 = np.array([0.3, 0.1, 0.05])
    EB = np.array([0, 0, 0, 0, 0, B0], dtype=np.float64)
    u = u0.copy()
    x = np.zeros(3)
    xs = [x.copy()]
    N = 10_000
    for _ in range(N):
        u = O.boris(q, m, c, dt, EB, u)
        x = O.move(c, dt, u, x)
        xs.append(x.copy())
    gamma = math.sqrt(1 + u0 @ u0)
    theta = 2 * math.atan(abs(q) * B0 * dt / (2 * m * c * gamma))
    # du/dt = (q/(m c)) (u/gamma) x B : clockwise about +z for q > 0
    phi = -math.copysign(1.0, q) * N * theta
    rot = np.array([[math.cos(phi), -math.sin(phi)], [math.sin(phi), math.cos(phi)]])
    # the per-step rotation angle carries O(eps) rounding, so the phase error
    # after N steps is bounded by ~ N * 4 eps (P3 tolerance)
    tol = N * 4 * np.finfo(float).eps
    np.testing.assert_allclose(u[:2], rot @ u0[:2], rtol=0, atol=tol * np.linalg.norm(u0))
    assert u[2] == u0[2]
    assert abs(np.linalg.norm(u) - np.linalg.norm(u0)) <= 1e-13 * np.linalg.norm(u0)
    # orbit vertices lie on a circle of radius dt v_perp / (2 sin(theta/2))
    v_perp = np.linalg.norm(u0[:2]) / gamma * c
    r = dt * v_perp / (2 * math.sin(theta / 2))
    xs = np.array(xs)
    # centre from the first three vertices
    A = np.array([xs[1, :2] - xs[0, :2], xs[2, :2] - xs[0, :2]])
    bvec = 0.5 * np.array([xs[1, :2] @ xs[1, :2] - xs[0, :2] @ xs[0, :2],
                           xs[2, :2] @ xs[2, :2] - xs[0, :2] @ xs[0, :2]])
    ctr = np.linalg.solve(A, bvec)
    radii = np.linalg.norm(xs[:, :2] - ctr, axis=1)
    np.testing.assert_allclose(radii, r, rtol=1e-9)
    # guiding centre drifts along z with u_z / gamma
    assert xs[-1, 2] == pytest.approx(N * dt * u0[2] / gamma, rel=1e-12)


def test_p3_discrete_period_vs_continuous(oracle_mod):
    # B0 = 1, gamma ~ 1: theta = 2 atan(Omega dt / 2) vs Omega dt
    theta = 2 * math.atan(DT / 2)
    assert theta == pytest.approx(0.2866951, abs=1e-7)
    assert abs(theta - DT) / DT <= DT ** 2 / 12 * 1.01


def test_p4_pure_electric_kick(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(4)
    for _ in range(100):
        q, m, c, dt = rng.choice([-1.0, 1.0]), rng.uniform(0.5, 2000), rng.uniform(0.5, 2), DT
        E = rng.standard_normal(3)
        u = rng.standard_normal(3)
        got = O.boris(q, m, c, dt, np.r_[E, 0, 0, 0], u)
        expect = u + q * dt / (m * c) * E
        np.testing.assert_allclose(got, expect, rtol=0,
                                   atol=4 * np.finfo(float).eps * (np.abs(u).max() + np.abs(expect).max()))


def test_p5_exb_drift(oracle_mod):
    O = oracle_mod
    E0 = 1e-4
    EB = np.array([E0, 0, 0, 0, 0, 1.0])
    vd = np.cross(EB[:3], EB[3:])  # c E x B / B^2 = (0, -E0, 0)
    assert vd[1] == -E0
    for q in (-1.0, 1.0):
        u = vd / math.sqrt(1 - vd @ vd)
        x = np.zeros(3)
        N = 2000
        for _ in range(N):
            u = O.boris(q, 1.0, 1.0, DT, EB, u)
            x = O.move(1.0, DT, u, x)
        vmean = x / (N * DT)
        np.testing.assert_allclose(vmean, vd, rtol=0, atol=1e-6 * E0)


def test_p6_move_limits(oracle_mod):
    O = oracle_mod
    x = np.array([1.25, 2.5, 3.75])
    assert np.array_equal(O.move(1.0, DT, np.zeros(3), x), x)
    for big in (1e3, 1e8, 1e150):
        u = np.array([big, -big, big / 3])
        xn = O.move(1.0, DT, u, x)
        v = np.linalg.norm(xn - x) / DT
        assert v < 1.0 + 1e-15


def test_wrap_rule_r7(oracle_mod):
    O = oracle_mod
    L = 16.0
    assert O.wrap(16.0, L) == 0.0
    assert O.wrap(16.25, L) == 0.25
    assert O.wrap(-1e-20, L) == 0.0          # -1e-20 + 16 rounds to 16 -> 0
    assert O.wrap(-0.25, L) == 15.75
    assert O.wrap(3.0, L) == 3.0
    r = O.wrap(-1e-15, L)
    assert 0 <= r < L


# ---------------- P7 / P8 : FDTD ----------------

def _plane_wave(O, axis, ecomp, nvec, h, m=1, nsteps=0, E0=1.0):
    """Discrete Yee eigenmode along `axis`, E along `ecomp`."""
    nx, ny, nz = nvec
    c = 1.0
    dt = 0.5 / (c * math.sqrt(sum(1 / hh ** 2 for hh in h)))
    n_ax = nvec[axis]
    k = 2 * math.pi * m / (n_ax * h[axis])
    w = 2.0 / dt * math.asin(c * dt / h[axis] * math.sin(k * h[axis] / 2))
    bcomp = 3 - axis - ecomp   # the remaining axis
    # sign of (k_hat x e_hat) along bcomp
    kh = np.zeros(3); kh[axis] = 1
    eh = np.zeros(3); eh[ecomp] = 1
    sgn = np.cross(kh, eh)[bcomp]
    coords = np.arange(n_ax) * h[axis]
    t = nsteps * dt
    Ev = E0 * np.cos(k * coords - w * t)
    Bv = sgn * E0 * math.cos(w * dt / 2) * np.cos(k * (coords + 0.5 * h[axis]) - w * t)
    F = np.zeros((9, nz, ny, nx))
    shape = [1, 1, 1]
    shape[2 - axis] = n_ax
    F[ecomp] = Ev.reshape(shape)
    F[3 + bcomp] = Bv.reshape(shape)
    return F, dt, w


@pytest.mark.parametrize("axis,ecomp", [(0, 1), (0, 2), (1, 2), (1, 0), (2, 0), (2, 1)])
def test_p7_vacuum_plane_wave_dispersion(oracle_mod, axis, ecomp):
    O = oracle_mod
    nvec = [6, 7, 5]
    nvec[axis] = 24
    h = (1.0, 0.8, 1.25)
    F0, dt, w = _plane_wave(O, axis, ecomp, nvec, h)
    nsteps = int(round(2 * math.pi / (w * dt))) + 3   # more than one period
    g = make(O, *nvec, dx=h[0], dy=h[1], dz=h[2], dt=dt)
    orc = O.Oracle(g)
    orc.F[:] = F0
    for _ in range(nsteps):
        orc.b_half(); orc.e_full(); orc.b_half()
    Fn, _, _ = _plane_wave(O, axis, ecomp, nvec, h, nsteps=nsteps)
    np.testing.assert_allclose(orc.F, Fn, rtol=0, atol=1e-12)


def test_p7_vacuum_zero_stays_zero(oracle_mod):
    O = oracle_mod
    g = make(O, 4, 5, 6)
    orc = O.Oracle(g)
    for _ in range(50):
        orc.b_half(); orc.e_full(); orc.b_half()
    assert not orc.F.any()


def test_p8_fdtd_vs_fft_symbols(oracle_mod):
    O = oracle_mod
    h = (1.1, 0.9, 1.3)
    nx, ny, nz = 6, 5, 7
    g = make(O, nx, ny, nz, dx=h[0], dy=h[1], dz=h[2], c=1.7)
    orc = O.Oracle(g)
    rng = np.random.default_rng(8)
    orc.F[:] = rng.standard_normal(orc.F.shape)
    F0 = orc.F.copy()
    orc.b_half()
    ref = brute.fft_b_half(F0, h, g.c, g.dt)
    np.testing.assert_allclose(orc.F, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
    F1 = orc.F.copy()
    orc.e_full()
    ref = brute.fft_e_full(F1, h, g.c, g.dt)
    np.testing.assert_allclose(orc.F, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


# ---------------- P9 : cold plasma oscillation ----------------

def test_p9_cold_plasma_oscillation(oracle_mod):
    O = oracle_mod
    n = 8
    n_e = 0.01 / (4 * math.pi)
    g = make(O, n, n, n, species=((-1.0, 1.0, n_e),), S=1, K=0)
    ii = np.arange(n ** 3)
    P = np.zeros((6, n ** 3))
    P[0] = ii % n + 0.5
    P[1] = (ii // n) % n + 0.5
    P[2] = ii // (n * n) + 0.5
    u0 = 1e-4
    P[3] = u0
    orc = O.Oracle(g, particles=[(P, np.arange(n ** 3, dtype=np.uint64))])
    wp = 0.1
    dt = g.dt
    wd = 2 / dt * math.asin(wp * dt / 2)
    assert abs(wd - wp) / wp <= (wp * dt) ** 2 / 24 * 1.01
    nsteps = 300
    Ex = []
    for _ in range(nsteps):
        orc.step(1)
        Ex.append(orc.F[0].mean())
        # positions i + 1/2 + d round with the ulp of i, so the realised
        # displacement (hence J) differs between cells by ~ulp(n)/|d| ~ 1e-11
        assert np.ptp(orc.F[0]) <= 1e-8 * abs(orc.F[0]).max() + 1e-300
    Ex = np.array(Ex)
    # E^0 = 0 ; E^1 = -4 pi dt J^{1/2} = 4 pi dt n_e v^{1/2}  (q = -1)
    v_half = u0 / math.sqrt(1 + u0 * u0)
    A = 4 * math.pi * dt * n_e * v_half / math.sin(wd * dt)
    ref = A * np.sin(wd * dt * np.arange(1, nsteps + 1))
    np.testing.assert_allclose(Ex, ref, rtol=0, atol=2e-7 * abs(A))
    assert np.abs(orc.F[3:6]).max() <= 1e-14 * abs(A)


# ---------------- P10 / P11 / P14 : deposition ----------------

def _random_moves(rng, L, n, vmax=0.9, dt=DT):
    a = rng.random((n, 3)) * L
    d = (rng.random((n, 3)) * 2 - 1) * vmax * dt
    return a, a + d


def test_p11_vb_vs_flux_quadrature_and_continuity(oracle_mod):
    O = oracle_mod
    h = (1.0, 1.0, 1.0)
    shape_xyz = (4, 5, 6)
    rng = np.random.default_rng(11)
    L = np.array(shape_xyz, dtype=float)
    for trial in range(60):
        g = make(O, *shape_xyz, species=((-1.0, 1.0, 1.0),))
        orc = O.Oracle(g)
        npart = 1 + trial % 10
        A, B = _random_moves(rng, L, npart, vmax=0.99 * math.sqrt(3), dt=g.dt)
        # force some exact-face and corner cases
        if trial % 7 == 0:
            A[0] = np.floor(A[0]) ; B[0] = A[0] + np.array([0.2, -0.1, 0.15])
        if trial % 5 == 0:
            B[0] = np.floor(B[0]) + np.array([0.0, 0.5, 0.5])
        Jref = np.zeros((3, 6, 5, 4))
        qw = -0.37
        for a, b in zip(A, B):
            assert orc.deposit_vb(qw, a, b) == 0
            Jref += brute.flux_current((6, 5, 4), h, g.dt, qw, a, b)
        np.testing.assert_allclose(orc.F[6:], Jref, rtol=0, atol=1e-13 * max(1.0, np.abs(Jref).max()))
        # continuity: (rho_new - rho_old)/dt + div J = 0 at every node
        rho0 = brute.rho_hat((6, 5, 4), h, qw, A)
        rho1 = brute.rho_hat((6, 5, 4), h, qw, np.mod(B, L))
        divj = orc.div_edge(6)
        res = (rho1 - rho0) / g.dt + divj
        assert np.abs(res).max() <= 1e-13


def test_p10_total_current_equals_sum_qwv(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(10)
    g = make(O, 5, 4, 6, species=((-1.0, 1.0, 0.3),), dx=1.2, dy=0.9, dz=1.1)
    orc = O.Oracle(g)
    L = np.array([5 * 1.2, 4 * 0.9, 6 * 1.1])
    A, B = _random_moves(rng, L, 500, vmax=0.95, dt=g.dt)
    qw = -0.3
    tot = np.zeros(3)
    for a, b in zip(A, B):
        assert orc.deposit_vb(qw, a, b) == 0
        tot += qw * (b - a) / g.dt
    V = 1.2 * 0.9 * 1.1
    got = orc.F[6:].sum(axis=(1, 2, 3)) * V
    np.testing.assert_allclose(got, tot, rtol=1e-13, atol=1e-13 * np.abs(tot).max())


def test_p14_superposition(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(14)
    g = make(O, 4, 4, 5)
    L = np.array([4.0, 4.0, 5.0])
    A, B = _random_moves(rng, L, 20)
    o1 = O.Oracle(g); o2 = O.Oracle(g); o3 = O.Oracle(g)
    for i, (a, b) in enumerate(zip(A, B)):
        o1.deposit_vb(0.5, a, b)
        (o2 if i % 2 else o3).deposit_vb(0.5, a, b)
    np.testing.assert_allclose(o1.F[6:], o2.F[6:] + o3.F[6:], rtol=0, atol=1e-15 * np.abs(o1.F).max())


def test_deposit_zero_move_and_axis_aligned(oracle_mod):
    O = oracle_mod
    g = make(O, 4, 4, 4)
    orc = O.Oracle(g)
    a = np.array([1.3, 2.0, 3.0])
    assert orc.deposit_vb(1.0, a, a) == 0
    assert not orc.F.any()
    # move purely along x with y, z on a node: all current on one Jx edge
    orc.deposit_vb(1.0, a, a + np.array([0.2, 0, 0]))
    nz = np.argwhere(orc.F[6] != 0)
    assert nz.tolist() == [[3, 2, 1]]
    assert orc.F[6, 3, 2, 1] == pytest.approx(0.2 / g.dt, rel=1e-15)
    assert not orc.F[7:].any()


def test_deposit_displacement_error(oracle_mod):
    O = oracle_mod
    g = make(O, 4, 4, 4)
    orc = O.Oracle(g)
    assert orc.deposit_vb(1.0, [1.5, 1.5, 1.5], [2.5, 1.5, 1.5]) == -5
    assert orc.deposit_vb(1.0, [1.5, 1.5, 1.5], [1.5, 1.5, float("nan")]) == -6


# ---------------- P12 : whole-step invariants ----------------

def _thermal(O, nx, ny, nz, ppc, sigma, seed, S=2, K=3, species=None):
    from synth import Workload, gen_particles
    from synth.configs import electron
    sp = species or (electron(ppc, sigma),)
    wl = Workload("t", nx, ny, nz, sp, steps=1, sort_every=K, supercell=S, seed=seed)
    parts = gen_particles(wl)
    g = O.Grid(nx, ny, nz, 1.0, 1.0, 1.0, wl.dt, 1.0,
               [O.Species(s.q, s.m, s.w * 200) for s in sp], S, K)
    return g, parts


def test_p12_gauss_divb_energy(oracle_mod):
    O = oracle_mod
    g, parts = _thermal(O, 8, 8, 8, 20, 0.1, 12)
    orc = O.Oracle(g, particles=parts)
    gauss0 = orc.div_edge(0) - 4 * math.pi * orc.rho()
    for step in range(30):
        rho_before = orc.rho()
        orc.step(1)
        rho_after = orc.rho()
        cont = (rho_after - rho_before) / g.dt + orc.div_edge(6)
        assert np.abs(cont).max() <= 1e-13 * max(1.0, np.abs(orc.F[6:]).max())
        gauss = orc.div_edge(0) - 4 * math.pi * rho_after
        assert np.abs(gauss - gauss0).max() <= 1e-10
        assert np.abs(orc.div_b()).max() <= 1e-14 * max(1e-300, np.abs(orc.F[3:6]).max()) * 10


def test_p12_frozen_plasma_fixed_point(oracle_mod):
    O = oracle_mod
    g, parts = _thermal(O, 6, 8, 4, 5, 0.0, 13, S=2, K=4)
    orc = O.Oracle(g, particles=parts)
    orc.sort()
    P0 = [p.copy() for p in orc.P]
    F0 = orc.F.copy()
    orc.step(25)
    for a, b in zip(P0, orc.P):
        assert np.array_equal(a, b)
    assert np.array_equal(orc.F, F0)


# ---------------- P13 : sort ----------------

def test_p13_sort_is_stable_key_sort(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(13)
    g = make(O, 8, 12, 16, S=4, K=1)
    n = 5000
    P = np.zeros((6, n))
    P[:3] = (rng.random((3, n)) * np.array([[8], [12], [16]]))
    # many exact duplicates of positions and cell faces to exercise ties
    P[:3, ::7] = np.floor(P[:3, ::7])
    P[3:] = rng.standard_normal((3, n))
    ids = np.arange(n, dtype=np.uint64)
    orc = O.Oracle(g, particles=[(P, ids)])
    keys = orc.sort_keys(P)
    # the key, spelled out from R15
    c = np.floor(P[:3]).astype(np.int64)
    S = 4
    sc = (c[0] // S) + 2 * ((c[1] // S) + 3 * (c[2] // S))
    loc = (c[0] % S) + S * ((c[1] % S) + S * (c[2] % S))
    assert np.array_equal(keys, sc * 64 + loc)
    orc.sort()
    # R15: order by (supercell, slot, local cell); slot = rank of the particle
    # among earlier particles of the same cell (numpy stable argsort + cumcount)
    cell_order = np.argsort(keys, kind="stable")
    sk = keys[cell_order]
    first = np.r_[0, np.flatnonzero(np.diff(sk)) + 1]
    run_start = np.repeat(first, np.diff(np.r_[first, n]))
    slot = np.empty(n, dtype=np.int64)
    slot[cell_order] = np.arange(n) - run_start
    perm = np.lexsort((keys % 64, slot, keys // 64))
    assert np.array_equal(orc.ids[0], ids[perm])
    assert np.array_equal(orc.P[0], P[:, perm])
    # inside one (supercell, slot) group the cells are distinct and ascending
    sk, ss = keys[perm], slot[perm]
    grp = (sk[1:] // 64 == sk[:-1] // 64) & (ss[1:] == ss[:-1])
    assert (sk[1:][grp] > sk[:-1][grp]).all()


def test_sort_key_clamps_rounding(oracle_mod):
    O = oracle_mod
    g = make(O, 5, 5, 5, dx=0.7, dy=0.7, dz=0.7, S=1)
    orc = O.Oracle(g)
    x = np.nextafter(5 * 0.7, 0)   # < L but x/dx rounds to 5.0
    assert x < 5 * 0.7 and x / 0.7 == 5.0
    k = orc.sort_keys(np.array([[x], [0.0], [0.0]]))
    assert k[0] == 4


# ---------------- P15 : whole step vs brute-force re-derivation ----------------

@pytest.mark.parametrize("seed", [0, 1, 2])
def test_p15_whole_step_bruteforce(oracle_mod, seed):
    O = oracle_mod
    rng = np.random.default_rng(150 + seed)
    nvec = [(3, 4, 2), (4, 3, 3), (2, 2, 4)][seed]
    h = (1.0, 1.1, 0.9)
    species = [(-1.0, 1.0, 0.05), (1.0, 3.0, 0.04)]
    g = make(O, *nvec, species=species, dx=h[0], dy=h[1], dz=h[2], S=1, K=4)
    L = np.array(nvec) * np.array(h)
    parts = []
    for s in range(2):
        n = 1 + (seed + s) % 3
        P = np.zeros((6, n))
        P[:3] = rng.random((3, n)) * L[:, None]
        P[3:] = rng.standard_normal((3, n)) * 0.3
        parts.append((P, np.arange(n, dtype=np.uint64) + 10 * s))
    orc = O.Oracle(g, particles=parts)
    orc.F[:6] = rng.standard_normal((6, nvec[2], nvec[1], nvec[0])) * 0.05
    F = orc.F.copy()
    bparts = [p[0].copy() for p in parts]
    ids_b = [p[1].copy() for p in parts]
    for step in range(50):
        orc.step(1)
        F, bparts = brute.brute_step(F, bparts, species, h, 1.0, g.dt)
    for s in range(2):
        order = np.argsort(orc.ids[s])
        ref_order = np.argsort(ids_b[s])
        a = orc.P[s][:, order]
        b = bparts[s][:, ref_order]
        dpos = (a[:3] - b[:3] + L[:, None] / 2) % L[:, None] - L[:, None] / 2
        assert np.abs(dpos).max() <= 1e-9 * L.max()
        np.testing.assert_allclose(a[3:], b[3:], rtol=0, atol=1e-9 * np.abs(b[3:]).max())
    for c in range(9):
        np.testing.assert_allclose(orc.F[c], F[c], rtol=0, atol=1e-9 * np.abs(F[c]).max() + 1e-300)


# ---------------- P17 : input generator ----------------

def test_p17_generator_counts_and_moments():
    from synth import get_config, gen_particles
    wl = get_config("T_small")
    parts = gen_particles(wl)
    P, ids = parts[0]
    n = wl.ncells * 4
    assert P.shape == (6, n)
    cells = (np.floor(P[0]).astype(int) + wl.nx * (np.floor(P[1]).astype(int)
             + wl.ny * np.floor(P[2]).astype(int)))
    assert np.array_equal(np.bincount(cells, minlength=wl.ncells), np.full(wl.ncells, 4))
    sig = wl.species[0].sigma_u
    assert abs(P[3:].mean()) <= 5 * sig / math.sqrt(3 * n)
    assert abs(P[3:].std() / sig - 1) <= 5 / math.sqrt(3 * n)
    assert np.array_equal(ids, np.arange(n, dtype=np.uint64))
    again = gen_particles(wl)
    assert np.array_equal(again[0][0], P)


def test_workload_constants():
    from synth import get_config
    c1 = get_config("C1")
    assert c1.dt == pytest.approx(0.28867513459481287, rel=1e-16)
    assert c1.species[0].w == pytest.approx(9.947e-5, rel=1e-3)
    assert get_config("C3").n_particles == 104_857_600
    assert get_config("C2").n_particles == 3_200_000
    assert get_config("C4").for_ranks(8).nz == 1024
