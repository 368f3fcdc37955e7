/*
 * pic_oracle.h -- plain, slow, serial CPU oracle of one fp64 PIC time step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path under
 * paper_1608_01009_b200/ (and neither includes the other).
 *
 * What it computes (sec. 2, lines 36-40: "numerical integration of
 * Maxwell's equations, field interpolation, solving particles' equations of
 * motion, and computing the current density"; line 48: "double precision
 * using the standard cloud-in-cell particle form factor and the
 * charge-conserving current deposition scheme [VillasenorBuneman]"), with the
 * readings R1-R20 of DESIGN.md sec. 3 (Yee FDTD, relativistic Boris, straight
 * line Villasenor-Buneman split at cell faces, Gaussian units).
 *
 * Layout ("oracle"): all arrays are caller owned.
 *   F  : double[9][nz][ny][nx], components Ex,Ey,Ez,Bx,By,Bz,Jx,Jy,Jz,
 *        index i + nx*(j + ny*k) inside a component (x fastest).
 *   P  : double[6][n] per species: x,y,z (physical units, wrapped into
 *        [0,L)), ux,uy,uz (u = p/(m c) = gamma*beta, at time n-1/2).
 *   id : uint64_t[n] per species, carried along by the sort.
 * Periodic boundaries in all three axes, indices taken mod n (or, with
 * bc_z == ORACLE_BC_OPEN, open z boundaries; NEXT-1).
 *
 * Parity status per function: see DESIGN.md sec. 5 (every function below is
 * pinned by a closed form, an invariant or a brute-force test in
 * tests/test_oracle_pins.py; none is "parity unpinned").
 */
#ifndef PIC_ORACLE_H
#define PIC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_MAX_SPECIES 4

/* All fields 8 bytes wide: the ctypes mirror in oracle/oracle.py has no padding. */
typedef struct {
    int64_t nx, ny, nz;          /* cells */
    double dx, dy, dz;           /* cell size */
    double dt, c;                /* time step, speed of light */
    int64_t n_species;
    double q[ORACLE_MAX_SPECIES];/* charge (units of e) */
    double m[ORACLE_MAX_SPECIES];/* mass (units of m_e) */
    double w[ORACLE_MAX_SPECIES];/* weight: real particles per macro-particle */
    int64_t supercell;           /* S: sort key granularity (R15) */
    int64_t sort_every;          /* K: sort at the start of step n when n % K == 0 */
    /* z boundary (NEXT-1, reading R21): ORACLE_BC_PERIODIC,
     * or ORACLE_BC_OPEN = first-order Mur absorbing planes k = 0 and k = nz-1
     * for the tangential E (the incident laser enters through k = 0),
     * field values outside [0, nz) read as zero, deposits outside dropped,
     * particles leaving z in [0, (nz-1) dz) removed.  x and y stay periodic. */
    int64_t bc_z;
    /* incident plane wave (bc_z == ORACLE_BC_OPEN), travelling +z:
     *   E_inc(z, t) = laser_e0 env(xi) sin(laser_omega xi),  xi = t + laser_t0 - z/c,
     *   env = 0 (xi <= 0), sin^2(pi xi / (2 laser_ramp)) (xi < laser_ramp), 1 after;
     *   (Ex, Ey) = (pol_x, pol_y) E_inc,  (Bx, By) = (-pol_y, pol_x) E_inc. */
    double laser_e0, laser_omega, laser_ramp, laser_t0, laser_pol_x, laser_pol_y;
} oracle_config;

#define ORACLE_BC_PERIODIC 0
#define ORACLE_BC_OPEN 1

enum {
    ORACLE_OK = 0,
    ORACLE_EINVAL = -1,
    ORACLE_EDISPLACEMENT = -5,   /* |x'-x| >= one cell on some axis */
    ORACLE_ENONFINITE = -6
};

/* O4: CIC gather of the 6 staggered components at physical position (x,y,z). */
void oracle_gather(const oracle_config *cfg, const double *F,
                   double x, double y, double z, double out[6]);

/* a4: relativistic Boris on u = gamma*beta with h = q dt / (2 m c). EB = Ex..Bz. */
void oracle_boris(double q, double m, double c, double dt,
                  const double EB[6], double u[3]);

/* a4 (move): x' = x + dt c u / gamma, no wrap. */
void oracle_move(double c, double dt, const double u[3], const double x[3],
                 double xn[3]);

/* O5: Villasenor-Buneman deposit of the straight move a -> b (physical
 * coordinates, b unwrapped) of a particle with charge*weight qw into
 * J = F + 6*ncells.  Returns ORACLE_EDISPLACEMENT if |b-a| >= 1 cell. */
int oracle_deposit_vb(const oracle_config *cfg, double qw,
                      const double a[3], const double b[3], double *F);

/* R7: periodic wrap of one coordinate into [0, L). */
double oracle_wrap(double x, double L);

/* R15: sort key (supercell id, local cell id) of a wrapped position. */
int64_t oracle_sort_key(const oracle_config *cfg, double x, double y, double z);

/* a1: stable counting sort of one species by oracle_sort_key. */
void oracle_sort(const oracle_config *cfg, int64_t n, double *P, uint64_t *id);

/* a7 / O3: B -= (c dt/2) curl E ; E += c dt curl B - 4 pi dt J.
 * oracle_e_full advances E^n -> E^{n+1} with n = step_index (the time of the
 * incident wave at the open boundary; unused when periodic). */
void oracle_b_half(const oracle_config *cfg, double *F);
void oracle_e_full(const oracle_config *cfg, double *F, int64_t step_index);

/* NEXT-1: the incident wave amplitude E_inc(z, t) of the config (see above). */
double oracle_laser(const oracle_config *cfg, double z, double t);
/* NEXT-1: sets the fields to the incident wave at t = 0 (the part that
 * entered through z = 0 before t = 0): Ex, Ey at z = k dz (k < nz),
 * Bx, By at z = (k + 1/2) dz (k < nz - 1), every other value 0. */
void oracle_laser_preload(const oracle_config *cfg, double *F);

/* O2 step 2 for one species: gather, Boris, move, deposit, wrap, in array order.
 * J is NOT zeroed here.  With bc_z == ORACLE_BC_OPEN the particles whose new z
 * left [0, (nz-1) dz) are removed after their deposit (the rest keep their
 * order) and *n is updated; P keeps the [6][*n] layout (stride *n). */
int oracle_push_species(const oracle_config *cfg, double *F, int species,
                        int64_t *n, double *P, uint64_t *id);

/* O2: one full time step n -> n+1 (step_index = n); counts in/out. */
int oracle_step(const oracle_config *cfg, double *F, int64_t *counts,
                double *const *P, uint64_t *const *ids, int64_t step_index);

/* Diagnostics, all on caller-owned nx*ny*nz arrays.
 * rho += q w S(x-i)S(y-j)S(z-k)/(dx dy dz) at nodes (i,j,k). */
void oracle_deposit_rho(const oracle_config *cfg, double qw, int64_t n,
                        const double *P, double *rho);
/* div J and div E at nodes, div B at cell centres (backward / forward diffs). */
void oracle_div_edge(const oracle_config *cfg, const double *Vx, const double *Vy,
                     const double *Vz, double *out);
void oracle_div_face(const oracle_config *cfg, const double *Bx, const double *By,
                     const double *Bz, double *out);
/* sum (E^2+B^2)/(8 pi) dV  and  sum w m c^2 (gamma-1) */
double oracle_field_energy(const oracle_config *cfg, const double *F);
double oracle_kinetic_energy(const oracle_config *cfg, int species, int64_t n,
                             const double *P);

#ifdef __cplusplus
}
#endif
#endif
