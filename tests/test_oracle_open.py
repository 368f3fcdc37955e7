"""Pins of the oracle's open-z boundary, laser injection and particle
absorption (BASELINE.json configs[4] "a linearly
polarised plane wave ... injected from z=0"; reading R21 of DESIGN.md).
CPU only.  Each pin checks the oracle against something it does not compute
itself: the exact transport of the 1-D Yee scheme at the magic time step,
the closed-form reflection coefficient of first-order Mur on the discrete
dispersion relation, the periodic deposit (pinned by P11), closed-form CIC
weights."""
import math

import numpy as np
import pytest


def grid1d(O, nz, dt, dz=1.0, **laser):
    """nx = ny = 1 with huge dx, dy: every x/y difference vanishes (the
    neighbour is the cell itself), so the 3-D Yee update is the 1-D one."""
    g = O.Grid(1, 1, nz, 1e4, 1e4, dz, dt, 1.0, [O.Species(-1.0, 1.0, 1.0)], 1, 0,
               bc_z=O.BC_OPEN, **laser)
    return g


def f_inc(t, z, e0, om, ramp, t0=0.0):
    xi = t + t0 - z
    if xi <= 0:
        return 0.0
    env = math.sin(math.pi * xi / (2 * ramp)) ** 2 if xi < ramp else 1.0
    return e0 * env * math.sin(om * xi)


@pytest.mark.parametrize("pol", [(1.0, 0.0), (0.0, 1.0), (0.6, 0.8)])
def test_magic_step_injection_is_exact_transport(oracle_mod, pol):
    """c dt = dz: the 1-D Yee scheme shifts every wave by one cell per step
    and first-order Mur (a = 0) is exact, so the wave injected through z = 0
    is E^n_k = E_inc(k dz, n dt) everywhere, for all time, with no reflection
    from the top boundary; B^n at (k+1/2) is the mean of its neighbours'
    E_inc (the half-step average of the leapfrog)."""
    O = oracle_mod
    e0, om, ramp = 1.3, 2 * math.pi / 16, 24.0
    nz = 64
    g = grid1d(O, nz, 1.0, laser_e0=e0, laser_omega=om, laser_ramp=ramp, laser_pol=pol)
    orc = O.Oracle(g)
    for n in range(1, 201):
        orc.step(1)
        if n % 10:
            continue
        inc = np.array([f_inc(n, k, e0, om, ramp) for k in range(nz)])
        np.testing.assert_allclose(orc.F[0, :, 0, 0], pol[0] * inc, rtol=0, atol=1e-13)
        np.testing.assert_allclose(orc.F[1, :, 0, 0], pol[1] * inc, rtol=0, atol=1e-13)
        bmid = 0.5 * (inc[:-1] + inc[1:])
        np.testing.assert_allclose(orc.F[4, :-1, 0, 0], pol[0] * bmid, rtol=0, atol=1e-13)
        np.testing.assert_allclose(orc.F[3, :-1, 0, 0], -pol[1] * bmid, rtol=0, atol=1e-13)
        assert orc.F[3, -1, 0, 0] == 0.0 and orc.F[4, -1, 0, 0] == 0.0   # outside the box
        assert not np.any(orc.F[[2, 5]])


def test_magic_step_preload_propagates(oracle_mod):
    """The preloaded wave (t0 > 0: the part that entered before t = 0) joins
    the injected one: after 100 steps E is the incident wave to within the
    preload's B interpolation error, O((omega dz)^2 / 8) E0.  A sign or
    staggering error in the preload launches a backward wave of amplitude
    ~E0 instead."""
    O = oracle_mod
    e0, om, ramp, t0 = 1.0, 2 * math.pi / 16, 32.0, 40.0
    nz = 128
    g = grid1d(O, nz, 1.0, laser_e0=e0, laser_omega=om, laser_ramp=ramp, laser_t0=t0)
    orc = O.Oracle(g)
    orc.laser_preload()
    inc0 = np.array([f_inc(0, k, e0, om, ramp, t0) for k in range(nz)])
    np.testing.assert_allclose(orc.F[0, :, 0, 0], inc0, rtol=0, atol=1e-15)
    orc.step(100)
    inc = np.array([f_inc(100, k, e0, om, ramp, t0) for k in range(nz)])
    err = np.abs(orc.F[0, :, 0, 0] - inc).max()
    assert err <= 2 * (om ** 2 / 8) * e0, err


def mur_reflection(S, om, dt, dz=1.0):
    """|R| of first-order Mur on the discrete 1-D Yee wave: with
    z = exp(i om dt), p = exp(i kappa dz), sin(om dt/2) = S sin(kappa dz/2),
    R = |z - p - a(z p - 1)| / |z - 1/p - a(z/p - 1)|, a = (S-1)/(S+1)."""
    kappa = 2 * math.asin(math.sin(om * dt / 2) / S) / dz
    a = (S - 1) / (S + 1)
    zz, p = np.exp(1j * om * dt), np.exp(1j * kappa * dz)
    return abs(zz - p - a * (zz * p - 1)) / abs(zz - 1 / p - a * (zz / p - 1)), kappa


def test_mur_reflection_matches_discrete_closed_form(oracle_mod):
    """S = 0.5: a steady monochromatic wave reflects off the open top face
    with the closed-form |R|.  The reflected wave is isolated as the
    difference to a 4x longer box whose top is not reached yet."""
    O = oracle_mod
    e0, om, ramp, dt = 1.0, 2 * math.pi / 12, 30.0, 0.5
    nsteps = 920                          # t = 460
    runs = []
    for nz in (300, 1200):
        orc = O.Oracle(grid1d(O, nz, dt, laser_e0=e0, laser_omega=om, laser_ramp=ramp))
        orc.step(nsteps)
        runs.append(orc.F[0, :, 0, 0].copy())
    R, kappa = mur_reflection(dt, om, dt)
    z = np.arange(200, 261, dtype=float)
    basis = np.stack([np.cos(kappa * z), np.sin(kappa * z)], axis=1)

    def amp(v):
        coef, *_ = np.linalg.lstsq(basis, v, rcond=None)
        return float(np.hypot(*coef))

    a_inc = amp(runs[1][200:261])
    a_ref = amp(runs[0][200:261] - runs[1][200:261])
    assert abs(a_inc - e0) < 0.02 * e0          # injected amplitude
    assert 1e-4 < R < 0.1                       # a real, small reflection at S = 0.5
    assert abs(a_ref / a_inc - R) <= 0.005 * R, (a_ref / a_inc, R)   # measured: 0.05%


def test_open_gather_reads_zero_outside(oracle_mod):
    """Uniform fields, open z: a particle at z = 0.2 dz sees Ez (staggered
    at k+1/2) with weight 0.7 on the node at 1/2 and 0.3 on the node at -1/2,
    which lies outside the box and reads 0."""
    O = oracle_mod
    g = O.Grid(4, 4, 8, 1.0, 1.0, 1.0, 0.2, 1.0, [O.Species(-1.0, 1.0, 1.0)], 1, 0, bc_z=O.BC_OPEN)
    orc = O.Oracle(g)
    vals = np.array([1.0, 2.0, 3.0, 4.0, 5.0, 6.0])
    orc.F[:6] = vals[:, None, None, None]
    got = orc.gather(1.3, 2.6, 0.2)
    np.testing.assert_allclose(got, [1.0, 2.0, 0.7 * 3.0, 0.7 * 4.0, 0.7 * 5.0, 6.0], rtol=1e-15)
    got = orc.gather(1.3, 2.6, 3.7)           # inside: partition of unity
    np.testing.assert_allclose(got, vals, rtol=1e-15)


@pytest.mark.parametrize("where", ["bottom", "top"])
def test_absorption_removes_and_clips_deposit(oracle_mod, where):
    """Open z: a particle crossing z = 0 (or z = (nz-1) dz) is removed after
    its deposit, the others keep their order; the deposit equals the
    periodic one (P11) on every edge inside the box, minus the edges the
    periodic run wrapped around from outside."""
    O = oracle_mod
    nz = 8
    dt = 0.5 / math.sqrt(3.0)
    parts = []
    rng = np.random.default_rng(4)
    P = np.zeros((6, 5))
    P[0] = rng.random(5) * 4
    P[1] = rng.random(5) * 4
    P[2] = [3.2, 3.5, 3.9, 4.1, 4.4]
    P[3:] = rng.normal(0, 0.05, (3, 5))
    if where == "bottom":
        P[2, 2] = 0.05
        P[5, 2] = -0.6
    else:
        P[2, 2] = (nz - 1) - 0.05
        P[5, 2] = 0.6
    ids = np.arange(5, dtype=np.uint64)
    parts.append((P, ids))
    out = {}
    for bc in (O.BC_PERIODIC, O.BC_OPEN):
        g = O.Grid(4, 4, nz, 1.0, 1.0, 1.0, dt, 1.0, [O.Species(-1.0, 1.0, 0.1)], 1, 0, bc_z=bc)
        orc = O.Oracle(g, particles=[(P.copy(), ids.copy())])
        orc.push_species(0)
        out[bc] = orc
    op, pe = out[O.BC_OPEN], out[O.BC_PERIODIC]
    assert list(op.ids[0]) == [0, 1, 3, 4]
    np.testing.assert_array_equal(op.P[0], pe.P[0][:, [0, 1, 3, 4]])
    Jo, Jp = op.F[6:], pe.F[6:]
    # edges the periodic run received from outside the open box: bottom ->
    # planes wrapped from k = -1 to nz - 1; top -> planes k >= nz wrapped to 0
    wrapped = nz - 1 if where == "bottom" else 0
    keep = [k for k in range(nz) if k != wrapped]
    np.testing.assert_array_equal(Jo[:, keep], Jp[:, keep])
    if where == "bottom":
        assert not np.any(Jo[:, wrapped])
    assert np.any(Jp[:, wrapped])


def test_laser_envelope(oracle_mod):
    """Zero before the front, sin^2 ramp, full amplitude E0 after it."""
    O = oracle_mod
    g = grid1d(O, 8, 0.5, laser_e0=2.0, laser_omega=0.3, laser_ramp=10.0, laser_t0=3.0)
    orc = O.Oracle(g)
    assert orc.laser(3.0, 0.0) == 0.0 and orc.laser(5.0, 1.0) == 0.0
    xi = 4.0
    assert orc.laser(0.0, xi - 3.0) == pytest.approx(2.0 * math.sin(math.pi * xi / 20) ** 2 * math.sin(0.3 * xi),
                                                     rel=1e-15)
    ts = np.linspace(20.0, 20.0 + 2 * math.pi / 0.3, 2001)
    assert max(orc.laser(0.0, t) for t in ts) == pytest.approx(2.0, rel=1e-5)
