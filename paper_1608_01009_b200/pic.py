"""Thin Python binding of libpic.so (include/pic.h).

Argument marshalling only: every step of the PIC path runs in the CUDA
kernels of libpic.so.  PyTorch provides the device workspace (one uint8 CUDA
tensor), the CUDA stream and, for nranks > 1, the process group used to
broadcast the NCCL id.  There is no CPU fallback: importing this module
without libpic.so, or creating a Simulation without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpic.so")
MAX_SPECIES = 4

PIC_OK = 0
ERRORS = {
    -1: "PIC_EINVAL", -2: "PIC_ENOMEM", -3: "PIC_ECAPACITY", -4: "PIC_ESTATE",
    -5: "PIC_EDISPLACEMENT", -6: "PIC_ENONFINITE", -7: "PIC_ECUDA", -8: "PIC_ENCCL",
}
FLAG_NO_GRAPH = 1
FLAG_PROFILE = 2
FLAG_NAIVE = 4
FLAG_LOCAL_GROUP = 8

EXPORTS = [
    "pic_workspace_size", "pic_init", "pic_set_particles", "pic_set_fields", "pic_step",
    "pic_get_fields", "pic_get_particles", "pic_get_count", "pic_get_step_index",
    "pic_get_stage_times", "pic_get_launch_count", "pic_strerror", "pic_last_error",
    "pic_destroy", "pic_nccl_unique_id", "pic_step_group", "pic_diagnostics",
    "pic_diagnostics_group", "pic_laser_preload", "pic_balance_slabs", "pic_set_fields6", "pic_get_fields9",
]


class PicConfig(C.Structure):
    _fields_ = [
        ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
        ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
        ("dt", C.c_double), ("c", C.c_double),
        ("n_species", C.c_int64),
        ("q", C.c_double * MAX_SPECIES),
        ("m", C.c_double * MAX_SPECIES),
        ("w", C.c_double * MAX_SPECIES),
        ("capacity", C.c_int64 * MAX_SPECIES),
        ("supercell", C.c_int64),
        ("halo", C.c_int64),
        ("sort_every", C.c_int64),
        ("rank", C.c_int64), ("nranks", C.c_int64),
        ("flags", C.c_int64),
        ("migrate_capacity", C.c_int64),
        ("nccl_id", C.c_uint8 * 128),
        ("stream", C.c_void_p),
        ("bc_z", C.c_int64),
        ("slab_lo", C.c_int64), ("slab_hi", C.c_int64),
        ("laser_e0", C.c_double), ("laser_omega", C.c_double), ("laser_ramp", C.c_double),
        ("laser_t0", C.c_double), ("laser_pol", C.c_double * 2),
    ]


BC_PERIODIC = 0
BC_OPEN = 1


class PicDiag(C.Structure):
    """pic_diag (include/pic.h): slab-local diagnostics at step n."""
    _fields_ = [
        ("step", C.c_int64),
        ("field_energy", C.c_double),
        ("kinetic_energy", C.c_double * MAX_SPECIES),
        ("charge", C.c_double),
        ("current", C.c_double * 3),
        ("max_div_b", C.c_double),
        ("max_gauss", C.c_double),
        ("max_gauss_drift", C.c_double),
        ("max_continuity", C.c_double),
    ]

    def as_dict(self, n_species=MAX_SPECIES):
        return {"step": self.step, "field_energy": self.field_energy,
                "kinetic_energy": list(self.kinetic_energy)[:n_species], "charge": self.charge,
                "current": list(self.current), "max_div_b": self.max_div_b,
                "max_gauss": self.max_gauss, "max_gauss_drift": self.max_gauss_drift,
                "max_continuity": self.max_continuity}


class PicError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def _nccl_hint():
    """Point libpic's run-time NCCL loader (PIC_NCCL_LIB, runtime.cu nccl_api)
    at the torch wheel's libnccl.so.2 unless the caller set it: z-slab runs
    then use the same NCCL build as torch.distributed."""
    if os.environ.get("PIC_NCCL_LIB"):
        return
    try:
        import nvidia.nccl as m
        for d in m.__path__:
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["PIC_NCCL_LIB"] = cand
                return
    except ImportError:
        pass


def lib():
    """Load libpic.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        _nccl_hint()
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        dp, u64p, i64p = C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.POINTER(C.c_int64)
        cp = C.POINTER(PicConfig)
        L.pic_workspace_size.argtypes = [cp, C.POINTER(C.c_size_t)]
        L.pic_init.argtypes = [cp, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.pic_set_particles.argtypes = [C.c_void_p, C.c_int, C.c_int64, dp, dp, dp, dp, dp, dp, u64p]
        L.pic_set_fields.argtypes = [C.c_void_p, dp]
        L.pic_set_fields6.argtypes = [C.c_void_p, C.POINTER(dp)]
        L.pic_get_fields9.argtypes = [C.c_void_p, C.POINTER(dp)]
        L.pic_step.argtypes = [C.c_void_p, C.c_int64]
        L.pic_get_fields.argtypes = [C.c_void_p, dp]
        L.pic_get_particles.argtypes = [C.c_void_p, C.c_int, i64p, dp, dp, dp, dp, dp, dp, u64p]
        L.pic_get_count.argtypes = [C.c_void_p, C.c_int, i64p]
        L.pic_get_step_index.argtypes = [C.c_void_p, i64p]
        L.pic_get_stage_times.argtypes = [C.c_void_p, dp, i64p]
        L.pic_get_launch_count.argtypes = [C.c_void_p, i64p]
        L.pic_strerror.argtypes = [C.c_int]
        L.pic_strerror.restype = C.c_char_p
        L.pic_last_error.argtypes = [C.c_void_p]
        L.pic_last_error.restype = C.c_char_p
        L.pic_destroy.argtypes = [C.c_void_p]
        L.pic_destroy.restype = None
        L.pic_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        L.pic_step_group.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int64]
        L.pic_diagnostics.argtypes = [C.c_void_p, C.POINTER(PicDiag), dp]
        L.pic_diagnostics_group.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.POINTER(PicDiag),
                                            C.POINTER(dp)]
        L.pic_laser_preload.argtypes = [C.c_void_p]
        L.pic_balance_slabs.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, dp, i64p]
        for name in EXPORTS:
            if name not in ("pic_strerror", "pic_last_error", "pic_destroy"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _dptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def make_config(nx, ny, nz, species, dt, dx=1.0, dy=1.0, dz=1.0, c=1.0, capacity=None,
                supercell=4, sort_every=20, rank=0, nranks=1, flags=0, nccl_id=None,
                migrate_capacity=0, bc_z=BC_PERIODIC, slab=None, laser=None, halo=1):
    """species: list of (q, m, w); slab: (lo, hi) planes of this rank;
    laser: dict e0, omega, ramp, t0, pol (open z, NEXT-1)."""
    cfg = PicConfig()
    cfg.nx, cfg.ny, cfg.nz = nx, ny, nz
    cfg.dx, cfg.dy, cfg.dz = dx, dy, dz
    cfg.dt, cfg.c = dt, c
    cfg.n_species = len(species)
    for i, (q, m, w) in enumerate(species):
        cfg.q[i], cfg.m[i], cfg.w[i] = q, m, w
        cfg.capacity[i] = 0 if capacity is None else int(capacity[i])
    cfg.supercell, cfg.halo, cfg.sort_every = supercell, halo, sort_every
    cfg.rank, cfg.nranks, cfg.flags = rank, nranks, flags
    cfg.migrate_capacity = migrate_capacity
    if nccl_id is not None:
        C.memmove(cfg.nccl_id, bytes(nccl_id), 128)
    cfg.bc_z = bc_z
    if slab is not None and nranks > 1:
        cfg.slab_lo, cfg.slab_hi = int(slab[0]), int(slab[1])
    if laser:
        cfg.laser_e0, cfg.laser_omega = laser["e0"], laser["omega"]
        cfg.laser_ramp, cfg.laser_t0 = laser["ramp"], laser["t0"]
        cfg.laser_pol[0], cfg.laser_pol[1] = laser["pol"]
    return cfg


def balance_slabs(nz, nranks, granule, min_planes, plane_cost):
    """pic_balance_slabs: z cut planes [0, ..., nz] minimising the largest slab cost."""
    cost = np.ascontiguousarray(plane_cost, dtype=np.float64)
    assert cost.size == nz
    out = (C.c_int64 * (nranks + 1))()
    rc = lib().pic_balance_slabs(nz, nranks, granule, min_planes, _dptr(cost), out)
    if rc != PIC_OK:
        raise PicError(rc, "pic_balance_slabs")
    return list(out)


class Simulation:
    """One libpic context on the current CUDA device.

    Arrays cross the ABI as host numpy arrays (float64 / uint64); device
    memory is a torch uint8 workspace; work runs on a dedicated torch stream."""

    def __init__(self, cfg: PicConfig, device=None, stream=None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("libpic needs a CUDA device (no CPU fallback)")
        L = lib()
        self.torch = torch
        self.device = torch.device(device or "cuda")
        self.stream = stream or torch.cuda.Stream(device=self.device)
        cfg.stream = C.c_void_p(self.stream.cuda_stream)
        self.cfg = cfg
        nbytes = C.c_size_t(0)
        self._check(L.pic_workspace_size(C.byref(cfg), C.byref(nbytes)), None)
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) // 256 * 256
        self.ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            self._check(L.pic_init(C.byref(cfg), C.c_void_p(aligned), nbytes.value, C.byref(self.ctx)),
                        None)
        self.nx, self.ny = cfg.nx, cfg.ny
        self.nz_local = (cfg.slab_hi - cfg.slab_lo if cfg.nranks > 1 and (cfg.slab_lo or cfg.slab_hi)
                         else cfg.nz // cfg.nranks)
        self.n_species = cfg.n_species

    def _check(self, rc, ctx="self"):
        if rc != PIC_OK:
            L = lib()
            msg = L.pic_strerror(rc).decode()
            if ctx is not None and getattr(self, "ctx", None):
                msg = L.pic_last_error(self.ctx).decode()
            raise PicError(rc, msg)

    def set_particles(self, species, P, ids):
        P = np.ascontiguousarray(P, dtype=np.float64)
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        n = P.shape[1]
        rows = [np.ascontiguousarray(P[i]) for i in range(6)]
        self._check(lib().pic_set_particles(self.ctx, species, n, *[_dptr(r) for r in rows],
                                            ids.ctypes.data_as(C.POINTER(C.c_uint64))))

    def set_fields(self, f6):
        f6 = np.ascontiguousarray(f6, dtype=np.float64)
        assert f6.size == 6 * self.nx * self.ny * self.nz_local
        self._check(lib().pic_set_fields(self.ctx, _dptr(f6)))

    def set_fields_components(self, comps):
        """pic_set_fields6: six host arrays (Ex, Ey, Ez, Bx, By, Bz), each [nz_local][ny][nx]."""
        arrs = [np.ascontiguousarray(c, dtype=np.float64) for c in comps]
        assert len(arrs) == 6 and all(a.size == self.nx * self.ny * self.nz_local for a in arrs)
        ptrs = (C.POINTER(C.c_double) * 6)(*[_dptr(a) for a in arrs])
        self._check(lib().pic_set_fields6(self.ctx, ptrs))

    def get_fields_components(self, which=range(9)):
        """pic_get_fields9: the listed components (0..8 = Ex..Bz, Jx..Jz) as separate arrays."""
        out = {c: np.empty((self.nz_local, self.ny, self.nx), dtype=np.float64) for c in which}
        ptrs = (C.POINTER(C.c_double) * 9)(*[_dptr(out[c]) if c in out else None for c in range(9)])
        self._check(lib().pic_get_fields9(self.ctx, ptrs))
        return out

    def step(self, n=1):
        self._check(lib().pic_step(self.ctx, int(n)))

    def laser_preload(self):
        """pic_laser_preload: E^0, B^0 = the incident wave at t = 0 (open z)."""
        self._check(lib().pic_laser_preload(self.ctx))

    def get_fields(self):
        out = np.empty((9, self.nz_local, self.ny, self.nx), dtype=np.float64)
        self._check(lib().pic_get_fields(self.ctx, _dptr(out)))
        return out

    def count(self, species):
        n = C.c_int64(0)
        self._check(lib().pic_get_count(self.ctx, species, C.byref(n)))
        return n.value

    def get_particles(self, species, out=None):
        n = self.count(species)
        if out is None:
            P = np.empty((6, n), dtype=np.float64)
            ids = np.empty(n, dtype=np.uint64)
        else:
            P, ids = out
        cap = C.c_int64(P.shape[1])
        self._check(lib().pic_get_particles(self.ctx, species, C.byref(cap),
                                            *[_dptr(P[i]) for i in range(6)],
                                            ids.ctypes.data_as(C.POINTER(C.c_uint64))))
        return P[:, :cap.value], ids[:cap.value]

    def diagnostics(self, rho=False):
        """pic_diagnostics: dict of slab-local diagnostics (+ rho^n array if rho)."""
        d = PicDiag()
        r = np.empty((self.nz_local, self.ny, self.nx), dtype=np.float64) if rho else None
        self._check(lib().pic_diagnostics(self.ctx, C.byref(d), _dptr(r)))
        out = d.as_dict(self.n_species)
        if rho:
            out["rho"] = r
        return out

    def step_index(self):
        n = C.c_int64(0)
        self._check(lib().pic_get_step_index(self.ctx, C.byref(n)))
        return n.value

    def stage_times(self):
        ms = (C.c_double * 4)()
        nl = C.c_int64(0)
        self._check(lib().pic_get_stage_times(self.ctx, ms, C.byref(nl)))
        return {"sort": ms[0], "particle": ms[1], "field": ms[2], "exchange": ms[3],
                "particle_launches": nl.value}

    def launch_count(self):
        n = C.c_int64(0)
        self._check(lib().pic_get_launch_count(self.ctx, C.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "ctx", None):
            lib().pic_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def workload_config(wl, capacity_factor=1.0, flags=0, rank=0, nranks=1, supercell=None,
                    sort_every=None, nccl_id=None, counts=None, migrate_capacity=0, slab=None,
                    halo=None):
    """pic_config for a synth.Workload (species q, m, w, dt, z boundary and
    laser from the workload).

    With nranks > 1 this rank holds the z slab `slab` = (lo, hi), default
    [rank nz/nranks, (rank+1) nz/nranks), and the default capacity leaves 10%
    headroom for migration."""
    species = [(s.q, s.m, s.w) for s in wl.species]
    if slab is None:
        slab = (rank * (wl.nz // nranks), (rank + 1) * (wl.nz // nranks))
    if counts is None:
        zl, zh = slab
        if getattr(wl, "plasma_z", None):
            zl, zh = max(zl, wl.plasma_z[0]), min(zh, wl.plasma_z[1])
        planes = max(0, zh - zl)
        counts = [s.ppc * wl.nx * wl.ny * planes for s in wl.species]
        if nranks > 1:
            capacity_factor = max(capacity_factor, 1.1)
    cap = [max(1, int(np.ceil(c * capacity_factor))) for c in counts]
    laser = None
    if getattr(wl, "laser", None):
        laser = dict(wl.laser)
    return make_config(wl.nx, wl.ny, wl.nz, species, wl.dt, wl.dx, wl.dy, wl.dz, wl.c, cap,
                       supercell or wl.supercell,
                       wl.sort_every if sort_every is None else sort_every,
                       rank, nranks, flags, nccl_id, migrate_capacity,
                       bc_z=BC_OPEN if getattr(wl, "open_z", False) else BC_PERIODIC,
                       slab=slab if nranks > 1 else None, laser=laser,
                       halo=halo or getattr(wl, "halo", 1))


def simulation_from_workload(wl, capacity_factor=1.0, flags=0, rank=0, nranks=1, supercell=None,
                             sort_every=None, nccl_id=None, counts=None, migrate_capacity=0,
                             stream=None, slab=None, halo=None):
    """Build a Simulation for a synth.Workload."""
    cfg = workload_config(wl, capacity_factor, flags, rank, nranks, supercell, sort_every,
                          nccl_id, counts, migrate_capacity, slab, halo)
    return Simulation(cfg, stream=stream)


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from libpic's NCCL loader (rank 0 of a slab run)."""
    buf = (C.c_uint8 * 128)()
    rc = lib().pic_nccl_unique_id(buf)
    if rc != PIC_OK:
        raise PicError(rc, "pic_nccl_unique_id")
    return bytes(buf)


def broadcast_nccl_id(id_bytes, group=None) -> bytes:
    """Distributes rank 0's NCCL id over an initialised torch.distributed group
    (gloo or nccl).  Plumbing only: the exchange itself runs inside libpic."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(id_bytes), dtype=torch.uint8))
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


def diagnostics_group(sims, rho=False):
    """pic_diagnostics_group over PIC_FLAG_LOCAL_GROUP slab Simulations: list of dicts."""
    n = len(sims)
    arr = (C.c_void_p * n)(*[s.ctx.value for s in sims])
    ds = (PicDiag * n)()
    rs = [np.empty((s.nz_local, s.ny, s.nx), dtype=np.float64) for s in sims] if rho else None
    rp = (C.POINTER(C.c_double) * n)(*[_dptr(r) for r in rs]) if rho else None
    rc = lib().pic_diagnostics_group(arr, n, ds, rp)
    if rc != PIC_OK:
        msgs = "; ".join(lib().pic_last_error(s.ctx).decode() for s in sims)
        raise PicError(rc, msgs)
    out = [ds[r].as_dict(sims[r].n_species) for r in range(n)]
    if rho:
        for r in range(n):
            out[r]["rho"] = rs[r]
    return out


def step_group(sims, nsteps=1):
    """Advance PIC_FLAG_LOCAL_GROUP slab Simulations (ranks 0..n-1 on one GPU) together."""
    arr = (C.c_void_p * len(sims))(*[s.ctx.value for s in sims])
    rc = lib().pic_step_group(arr, len(sims), int(nsteps))
    if rc != PIC_OK:
        msgs = "; ".join(lib().pic_last_error(s.ctx).decode() for s in sims)
        raise PicError(rc, msgs)
