/*
 * pic.h -- C ABI of libpic.so, the B200-native fp64 particle-in-cell step.
 *
 * The operation (sec. 2, lines 36-40): macro-particles with charge
 * q, mass m and weight w move under the relativistic equations of motion in
 * the Yee-grid electromagnetic field; "the field is interpolated to the
 * position of particles, while the contribution of each particle to the
 * current density is distributed among the nearest grid nodes"; the stages
 * are "numerical integration of Maxwell's equations, field interpolation,
 * solving particles' equations of motion, and computing the current density".
 * PAPER.md:48 fixes double precision, the cloud-in-cell form factor and the
 * Villasenor-Buneman charge-conserving deposit.  The concrete scheme is
 * SURVEY.md sec. 8a rows a1-a8 with the readings R1-R20 of DESIGN.md sec. 3.
 *
 * Units (R3): Gaussian, dB/dt = -c curl E, dE/dt = c curl B - 4 pi J;
 * momenta are u = p/(m c) = gamma*beta.  Positions are physical
 * coordinates in [0, L) with L = n * d per axis, periodic in x, y and z
 * (or, with bc_z = PIC_BC_OPEN, open in z: z in [0, (nz-1) dz)).
 *
 * Conventions for every call:
 *  - returns PIC_OK (0) or a negative PIC_E* code; no exception, abort or
 *    exit crosses the ABI.  pic_strerror(code) and pic_last_error(ctx) give
 *    a message.
 *  - host arrays are caller-owned; the library copies in / out and never
 *    keeps a caller pointer.
 *  - device memory is ONE caller-supplied workspace (d_workspace, `bytes`
 *    long, 256-byte aligned) that must outlive the context; size it with
 *    pic_workspace_size.  The library never calls cudaMalloc for state.
 *  - all work is enqueued on cfg->stream (a cudaStream_t, NULL = legacy
 *    default stream).  A context is used by one host thread at a time.
 *  - nranks > 1 (z-slab decomposition) makes pic_init,
 *    pic_step and pic_destroy collective over the ranks.
 *
 * There is no CPU fallback: without a CUDA device every call that touches
 * the device returns PIC_ECUDA.
 */
#ifndef PIC_H
#define PIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PIC_MAX_SPECIES 4

enum {
    PIC_OK = 0,
    PIC_EINVAL = -1,        /* bad config / argument (CFL, S not dividing extents, ...) */
    PIC_ENOMEM = -2,        /* workspace too small */
    PIC_ECAPACITY = -3,     /* particle capacity or caller buffer too small */
    PIC_ESTATE = -4,        /* call order (e.g. step before init) */
    PIC_EDISPLACEMENT = -5, /* some particle moved >= 1 cell on an axis in one step */
    PIC_ENONFINITE = -6,    /* non-finite position or momentum */
    PIC_ECUDA = -7,         /* CUDA runtime / driver failure (incl. no device) */
    PIC_ENCCL = -8          /* NCCL failure (nranks > 1) */
};

/* All scalar fields are 8 bytes wide so the layout has no padding. */
typedef struct pic_config {
    int64_t nx, ny, nz;                /* GLOBAL cell counts */
    double dx, dy, dz;                 /* cell size */
    double dt, c;                      /* time step (must satisfy CFL), speed of light */
    int64_t n_species;                 /* 1..PIC_MAX_SPECIES */
    double q[PIC_MAX_SPECIES];         /* charge per species (units of e) */
    double m[PIC_MAX_SPECIES];         /* mass per species (units of m_e) */
    double w[PIC_MAX_SPECIES];         /* weight = real particles per macro-particle */
    int64_t capacity[PIC_MAX_SPECIES]; /* max particles held by this rank, per species */
    int64_t supercell;                 /* S: supercell edge (cells); must divide nx, ny, local nz */
    int64_t halo;                      /* h: tile drift halo (cells) of the fused particle kernel,
                                          1 or 2 (0 = 1).  A CTA's shared E/B and J tiles cover
                                          its supercell plus h cells on every side, so a particle
                                          may drift h cells out of the supercell it was sorted
                                          into before it takes the slower global path
                                          (the supercell's grid data must fit
                                          on-chip); a larger h allows a larger sort_every */
    int64_t sort_every;                /* K: re-sort at the start of step n when n % K == 0 (0: never) */
    int64_t rank, nranks;              /* z-slab rank / count (1 for a single GPU) */
    int64_t flags;                     /* PIC_FLAG_* bits */
    int64_t migrate_capacity;          /* nranks > 1: particles per species and direction that
                                          may leave the slab in one step (0: default 65536) */
    uint8_t nccl_id[128];              /* ncclUniqueId from rank 0 (nranks > 1) */
    void *stream;                      /* cudaStream_t all work is enqueued on */
    /* ---- NEXT-1 (BASELINE.json configs[4]; DESIGN.md
     * sec. 11, reading R21).  Zero-initialised fields keep the periodic box. */
    int64_t bc_z;                      /* PIC_BC_PERIODIC, or PIC_BC_OPEN: the box ends at the
                                          planes z = 0 and z = (nz-1) dz, where the tangential
                                          E obeys first-order Mur (the incident laser enters
                                          through z = 0); field values beyond them are 0,
                                          deposits beyond them are dropped, and particles
                                          whose z leaves [0, (nz-1) dz) are removed.  x, y
                                          stay periodic. */
    int64_t slab_lo, slab_hi;          /* nranks > 1: this rank's planes [slab_lo, slab_hi)
                                          (static load balance, pic_balance_slabs); 0, 0 =
                                          nz/nranks planes per rank */
    double laser_e0;                   /* incident wave (PIC_BC_OPEN), travelling +z:     */
    double laser_omega;                /*   E_inc(z,t) = e0 env(xi) sin(omega xi),         */
    double laser_ramp;                 /*   xi = t + t0 - z/c, env = 0 for xi <= 0,       */
    double laser_t0;                   /*   sin^2(pi xi/(2 ramp)) below ramp, then 1;      */
    double laser_pol[2];               /*   (Ex,Ey) = pol E_inc, (Bx,By) = (-pol_y,pol_x) E_inc */
} pic_config;

#define PIC_BC_PERIODIC 0
#define PIC_BC_OPEN 1

#define PIC_FLAG_NO_GRAPH 1   /* launch kernels directly instead of CUDA graphs */
#define PIC_FLAG_PROFILE 2    /* record per-stage CUDA events (pic_get_stage_times) */
#define PIC_FLAG_NAIVE 4      /* use the naive one-thread-per-particle kernel (tests) */
#define PIC_FLAG_LOCAL_GROUP 8 /* nranks > 1 without NCCL: the slab contexts live in one
                                  process on one device and are advanced together by
                                  pic_step_group (single-GPU emulation of the z-slab path) */

typedef struct pic_ctx pic_ctx;

/* Pure: device bytes pic_init needs for cfg (fields with ghost layers,
 * double-buffered SoA particles with ids, sort scratch, offsets, error word).
 * Returns PIC_EINVAL for an invalid cfg. */
int pic_workspace_size(const pic_config *cfg, size_t *bytes);

/* Validates cfg (dt <= 1/(c sqrt(1/dx^2+1/dy^2+1/dz^2)); S divides nx, ny and
 * the slab thickness; 1 <= n_species <= PIC_MAX_SPECIES; m > 0), carves d_workspace
 * (device pointer, `bytes` long), sets up NCCL when nranks > 1 and zeroes
 * E, B, J and all particle counts.  The rank owns z in [rank*nz/nranks,
 * (rank+1)*nz/nranks), or [slab_lo, slab_hi) when set.  *out receives the
 * context. */
int pic_init(const pic_config *cfg, void *d_workspace, size_t bytes, pic_ctx **out);

/* Copies n particles of `species` from HOST arrays (global physical
 * coordinates in [0,L), momenta u^{n-1/2}, 64-bit ids), keeps those whose
 * z lies in this rank's slab, and sorts them.  Replaces the
 * species' previous particles.  PIC_ECAPACITY if they exceed capacity;
 * PIC_EINVAL for a position outside [0,L) or a bad species index. */
int pic_set_particles(pic_ctx *ctx, int species, int64_t n,
                      const double *x, const double *y, const double *z,
                      const double *ux, const double *uy, const double *uz,
                      const uint64_t *id);

/* Copies E^n, B^n from a HOST array f[6][nz_local][ny][nx] (x fastest;
 * order Ex,Ey,Ez,Bx,By,Bz; Yee-staggered as in DESIGN.md sec. 4). */
int pic_set_fields(pic_ctx *ctx, const double *f);

/* The same with one HOST pointer per component (SURVEY.md sec. 8b's
 * pic_set_fields(ctx, const double* const f[6])): f[c] is [nz_local][ny][nx],
 * c = Ex,Ey,Ez,Bx,By,Bz.  PIC_EINVAL for a NULL component. */
int pic_set_fields6(pic_ctx *ctx, const double *const f[6]);

/* Advances nsteps time steps (per step: a1 sort when
 * step % K == 0; a2-a6 fused gather/push/deposit per species; a7 Yee
 * update; a8 exchange when nranks > 1).  Synchronises cfg->stream at the
 * end and returns the sticky device error (PIC_EDISPLACEMENT,
 * PIC_ENONFINITE, PIC_ECAPACITY) if one was raised. */
int pic_step(pic_ctx *ctx, int64_t nsteps);

/* nranks > 1: z-slab decomposition.  Rank r owns the
 * planes [r nz/nranks, (r+1) nz/nranks), or [slab_lo, slab_hi) (>= 4 planes,
 * divisible by S).  Each step exchanges with ranks r-1 and r+1 (a periodic
 * ring, cut between the last and the first rank for PIC_BC_OPEN), over NCCL
 * point-to-point on cfg->stream: the J ghost planes (added by the owner), the
 * particles whose z left the slab (fixed-capacity buffers, migrate_capacity
 * per species and direction; overflow -> PIC_ECAPACITY), and the E and B
 * ghost planes.  Received particles are pushed from an unsorted tail until
 * the next sort.
 *
 * Writes the 128-byte ncclUniqueId that rank 0 distributes to all ranks (as
 * cfg->nccl_id) before the collective pic_init.  PIC_ENCCL if NCCL cannot be
 * loaded. */
int pic_nccl_unique_id(uint8_t id[128]);

/* Advances n slab contexts created with PIC_FLAG_LOCAL_GROUP (ranks 0..n-1 of
 * one decomposition, same device and stream) by nsteps, exchanging ghost
 * planes and particles with device-to-device copies instead of NCCL.  Same
 * arithmetic and message layout as the NCCL path; used to check the
 * decomposed step against the single-domain oracle on one GPU. */
int pic_step_group(pic_ctx *const *ctxs, int n, int64_t nsteps);

/* Copies E^n, B^n and J^{n-1/2} (the last deposit; zero before the first
 * step) of the local slab without ghosts into a HOST array
 * f[9][nz_local][ny][nx] (Ex,Ey,Ez,Bx,By,Bz,Jx,Jy,Jz). */
int pic_get_fields(pic_ctx *ctx, double *f);

/* The same into one HOST pointer per component (SURVEY.md sec. 8b's
 * pic_get_fields(ctx, double* const f[9])), c = Ex,Ey,Ez,Bx,By,Bz,Jx,Jy,Jz;
 * a NULL component is skipped. */
int pic_get_fields9(pic_ctx *ctx, double *const f[9]);

/* Copies the live particles of `species` in their current device order
 * (sorted region, then particles received since the last sort) to HOST arrays.  *n_inout: capacity of the arrays in, particle count out
 * (PIC_ECAPACITY, with the count written, when too small).  Positions are
 * wrapped into [0,L).  Any array pointer may be NULL to skip it. */
int pic_get_particles(pic_ctx *ctx, int species, int64_t *n_inout,
                      double *x, double *y, double *z,
                      double *ux, double *uy, double *uz, uint64_t *id);

/* Current particle count of a species on this rank. */
int pic_get_count(pic_ctx *ctx, int species, int64_t *n);

/* The step index n of the state (number of steps taken since pic_init). */
int pic_get_step_index(pic_ctx *ctx, int64_t *n);

/* With PIC_FLAG_PROFILE: accumulated device milliseconds per stage since
 * the last call (ms[0] sort, ms[1] particle kernel, ms[2] field update,
 * ms[3] exchange) and the number of particle-kernel launches; resets them. */
int pic_get_stage_times(pic_ctx *ctx, double ms[4], int64_t *particle_launches);

/* Number of kernel launches the library enqueued since the last call
 * (counted on the host at enqueue time, graph nodes included); resets it. */
int pic_get_launch_count(pic_ctx *ctx, int64_t *launches);

/* Diagnostics of the state at step n (the
 * quantities of SPEC.md:379-443), computed on the device over this rank's
 * slab (sums and maxima are slab-local; the caller combines ranks):
 *   rho^n(i,j,k) = sum_p q w S(x-i dx)S(y-j dy)S(z-k dz)/(dx dy dz) at nodes,
 *     S the CIC hat (the charge the VB deposit conserves);
 *   gauss = div E^n - 4 pi rho^n at nodes (backward differences);
 *   continuity = (rho^n - rho^{n-1})/dt + div J^{n-1/2} at nodes;
 *   div B^n at cell centres (forward differences).
 * All fields are doubles; "max" fields are maxima of absolute values. */
typedef struct pic_diag {
    int64_t step;                           /* n */
    double field_energy;                    /* sum (E^2 + B^2) dV / (8 pi) */
    double kinetic_energy[PIC_MAX_SPECIES]; /* sum w m c^2 (gamma - 1), from u^{n-1/2} */
    double charge;                          /* sum rho dV (= sum of q w of the live particles) */
    double current[3];                      /* sum J^{n-1/2} dV per component */
    double max_div_b;
    double max_gauss;                       /* max |div E - 4 pi rho| */
    double max_gauss_drift;                 /* max |gauss^n - gauss^{n0}|, n0 = the context's
                                               first diagnostics call (0 at that call) */
    double max_continuity;                  /* -1 unless the previous call was at step n-1 */
} pic_diag;

/* Computes *out (and, if rho != NULL, copies rho^n of the local slab without
 * ghosts into the HOST array rho[nz_local][ny][nx]).  Periodic z only
 * (PIC_EINVAL with PIC_BC_OPEN: the node fold assumes z images).  Collective when
 * nranks > 1 (the top node plane of a slab belongs to the slab above; the
 * Jz plane below is exchanged).  Enqueued on cfg->stream and synchronised;
 * not part of the timed step. */
int pic_diagnostics(pic_ctx *ctx, pic_diag *out, double *rho);

/* The same for the n contexts of a PIC_FLAG_LOCAL_GROUP decomposition:
 * out[r] (and rho[r], each may be NULL) for rank r. */
int pic_diagnostics_group(pic_ctx *const *ctxs, int n, pic_diag *out, double *const *rho);

/* NEXT-1: sets E^0, B^0 of the local slab to the incident wave at t = 0
 * (the part that entered through z = 0 before t = 0, so with laser_t0 > 0
 * the front starts at z = c t0): Ex, Ey = pol E_inc(z, 0) at z = k dz,
 * Bx, By = (-pol_y, pol_x) E_inc(z, 0) at z = (k + 1/2) dz below the top
 * face, all other components 0.  Call before the first step (PIC_ESTATE
 * otherwise); PIC_EINVAL unless bc_z == PIC_BC_OPEN.  Collective when
 * nranks > 1 (ghost planes are exchanged at the next step). */
int pic_laser_preload(pic_ctx *ctx);

/* NEXT-1 static load balance (host only, no device): cuts the planes
 * [0, nz) into nranks contiguous slabs z_split[r] .. z_split[r+1]
 * (z_split[0] = 0, z_split[nranks] = nz) minimising the largest slab cost,
 * where plane k costs plane_cost[k] (e.g. particles x t_particle + cells x
 * t_cell); every cut is a multiple of `granule` (the supercell edge) and
 * every slab has at least min_planes planes.  PIC_EINVAL if impossible. */
int pic_balance_slabs(int64_t nz, int64_t nranks, int64_t granule, int64_t min_planes,
                      const double *plane_cost, int64_t *z_split);

/* Message for an error code / the last error of a context (never NULL). */
const char *pic_strerror(int code);
const char *pic_last_error(pic_ctx *ctx);

/* Frees host state, CUDA graphs/events and the NCCL communicator.  The
 * workspace stays owned by the caller.  NULL is accepted. */
void pic_destroy(pic_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* PIC_H */
