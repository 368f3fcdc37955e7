"""CPU-only checks of the NEXT-1 host logic (DESIGN.md
sec. 11): pic_balance_slabs against brute force over every admissible cut,
the validation of open-z / unequal-slab configs by the pure sizing call,
and the C5 workload shapes."""
import ctypes as C
import itertools
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pic():
    subprocess.check_call(["make", "-s", "-C", ROOT], stdout=subprocess.DEVNULL)
    import paper_1608_01009_b200 as P
    P.lib()
    return P


def brute_best(cost, nranks, granule, min_planes):
    nz = len(cost)
    cuts = range(granule, nz, granule)
    best = math.inf
    for inner in itertools.combinations(cuts, nranks - 1):
        z = (0,) + inner + (nz,)
        if any(z[r + 1] - z[r] < min_planes for r in range(nranks)):
            continue
        best = min(best, max(sum(cost[z[r]:z[r + 1]]) for r in range(nranks)))
    return best


@pytest.mark.parametrize("seed", range(12))
def test_balance_slabs_is_optimal(pic, seed):
    rng = np.random.default_rng(seed)
    granule = int(rng.choice([1, 2, 4]))
    nz = granule * int(rng.integers(6, 16))
    nranks = int(rng.integers(1, 5))
    min_planes = granule * int(rng.integers(1, 3))
    if nz < nranks * min_planes:
        nranks = max(1, nz // min_planes)
    cost = rng.random(nz) ** 4 * 100.0 + 1.0
    if seed % 3 == 0:
        cost[nz // 3: nz // 2] *= 50.0      # a dense slab, as in C5
    z = pic.balance_slabs(nz, nranks, granule, min_planes, cost)
    assert z[0] == 0 and z[-1] == nz
    assert all(b - a >= min_planes and a % granule == 0 for a, b in zip(z, z[1:]))
    got = max(cost[a:b].sum() for a, b in zip(z, z[1:]))
    assert got <= brute_best(cost, nranks, granule, min_planes) * (1 + 1e-9)


def test_balance_slabs_rejects_impossible(pic):
    with pytest.raises(pic.PicError):
        pic.balance_slabs(16, 5, 4, 4, np.ones(16))   # 5 slabs of >= 4 planes in 16
    with pytest.raises(pic.PicError):
        pic.balance_slabs(10, 2, 4, 4, np.ones(10))   # nz not a multiple of the granule
    with pytest.raises(pic.PicError):
        pic.balance_slabs(8, 2, 4, 4, -np.ones(8))    # negative cost


def test_c5_balanced_slabs_spread_the_slab(pic):
    """C5 at 8 ranks: with a particles + cells cost the dense slab
    z in [600, 700) is shared by several ranks instead of 2 holding all of
    it (uniform 128-plane slabs put 1.007e9 particles on rank 5)."""
    from synth import get_config
    wl = get_config("C5")
    ppc = sum(s.ppc for s in wl.species)
    parts = np.zeros(wl.nz)
    parts[wl.plasma_z[0]:wl.plasma_z[1]] = ppc * wl.nx * wl.ny
    cost = parts * 1.0 + 0.5 * wl.nx * wl.ny
    z = pic.balance_slabs(wl.nz, 8, wl.supercell, 4, cost)
    per_rank = [parts[a:b].sum() for a, b in zip(z, z[1:])]
    assert max(per_rank) < 0.25 * parts.sum()
    assert sum(1 for p in per_rank if p > 0) >= 6


def _cfg(pic, **kw):
    base = dict(nx=16, ny=16, nz=32, species=[(-1.0, 1.0, 1.0)], dt=0.25, capacity=[1000],
                supercell=4, bc_z=pic.BC_OPEN,
                laser=dict(e0=1.0, omega=0.2, ramp=10.0, t0=5.0, pol=(1.0, 0.0)))
    base.update(kw)
    nx, ny, nz, sp, dt = base.pop("nx"), base.pop("ny"), base.pop("nz"), base.pop("species"), base.pop("dt")
    return pic.make_config(nx, ny, nz, sp, dt, **base)


def test_open_and_slab_configs_validate(pic):
    L = pic.lib()
    nb = C.c_size_t(0)
    good = [_cfg(pic), _cfg(pic, nranks=3, rank=1, slab=(8, 20)), _cfg(pic, nranks=3, rank=0, slab=(0, 8)),
            _cfg(pic, nranks=3, rank=2, slab=(20, 32))]
    for c in good:
        assert L.pic_workspace_size(C.byref(c), C.byref(nb)) == 0
    bad = [
        _cfg(pic, bc_z=7),
        _cfg(pic, nz=2, supercell=1),
        _cfg(pic, nranks=3, rank=1, slab=(8, 18)),    # 10 planes: S = 4 does not divide
        _cfg(pic, nranks=3, rank=0, slab=(4, 12)),    # rank 0 must start at 0
        _cfg(pic, nranks=3, rank=2, slab=(20, 28)),   # the last rank must end at nz
        _cfg(pic, nranks=3, rank=1, slab=(12, 8)),
        _cfg(pic, laser=dict(e0=float("nan"), omega=0.2, ramp=10.0, t0=5.0, pol=(1.0, 0.0))),
        _cfg(pic, laser=dict(e0=1.0, omega=0.2, ramp=-1.0, t0=5.0, pol=(1.0, 0.0))),
    ]
    for c in bad:
        assert L.pic_workspace_size(C.byref(c), C.byref(nb)) == -1
    # unequal slabs need no divisibility of nz by nranks
    c = _cfg(pic, nz=36, nranks=3, rank=1, slab=(8, 20))
    assert L.pic_workspace_size(C.byref(c), C.byref(nb)) == 0


def test_c5_workload_shapes():
    from synth import gen_particles, get_config
    wl = get_config("T_laser")
    parts = gen_particles(wl)
    (Pe, ie), (Pp, ip) = parts
    assert Pe.shape[1] == 2 * wl.nx * wl.ny * (wl.plasma_z[1] - wl.plasma_z[0])
    assert np.array_equal(Pe[:3], Pp[:3])                       # co-located, neutral
    assert (Pe[2] >= wl.plasma_z[0]).all() and (Pe[2] < wl.plasma_z[1]).all()
    assert not np.any(Pe[3:]) and not np.any(Pp[3:])            # cold
    lz = dict(get_config("C5").laser)
    assert lz["omega"] == pytest.approx(2 * math.pi / 32)
    assert lz["e0"] == pytest.approx(10 * 2 * math.pi / 32)     # a0 = e E0 / (m c omega) = 10
    # a rank outside the slab draws nothing
    none = gen_particles(wl, rank=0, z_lo=0, z_hi=32)
    assert all(P.shape[1] == 0 for P, _ in none)
