/*
 * pic_oracle.c -- plain, slow, serial CPU oracle of one fp64 PIC time step.
 *
 * TEST INFRASTRUCTURE ONLY (see pic_oracle.h).  Compiled with
 * -O2 -ffp-contract=off and no fast-math, so every line below is evaluated
 * as written.  Each function cites the passage it follows: PAPER.md line
 * numbers, SURVEY.md sec. 8 rows (the hot-path contract derived from
 * PAPER.md + SPEC.md), and the DESIGN.md readings R1-R20.
 *
 * No blocking, fusion or reordering: one particle at a time in array order,
 * direct periodic indexing (mod n), no ghost cells, no tiles.
 */
#include "pic_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int64_t wrap_index(int64_t i, int64_t n)
{
    int64_t r = i % n;
    return r < 0 ? r + n : r;
}

static int64_t cell_index(const oracle_config *cfg, int64_t i, int64_t j, int64_t k)
{
    return wrap_index(i, cfg->nx) +
           cfg->nx * (wrap_index(j, cfg->ny) + cfg->ny * wrap_index(k, cfg->nz));
}

/* NEXT-1 (reading R21): with an open z boundary the grid has no z images;
 * a node index outside [0, nz) lies outside the box (fields read 0 there,
 * deposits there are dropped). */
static int z_outside(const oracle_config *cfg, int64_t k)
{
    return cfg->bc_z == ORACLE_BC_OPEN && (k < 0 || k >= cfg->nz);
}

/* Yee staggering, in cell units:
 * Ex (i+1/2,j,k), Ey (i,j+1/2,k), Ez (i,j,k+1/2),
 * Bx (i,j+1/2,k+1/2), By (i+1/2,j,k+1/2), Bz (i+1/2,j+1/2,k). */
static const double STAGGER[6][3] = {
    {0.5, 0.0, 0.0}, {0.0, 0.5, 0.0}, {0.0, 0.0, 0.5},
    {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}, {0.5, 0.5, 0.0},
};

/* O4 -- CIC ("standard cloud-in-cell particle form factor", PAPER.md:48;
 * SPEC.md:178-196; reading R9: full trilinear weights of every component on
 * its own staggered sub-grid).  g = x/dx - o, i0 = floor(g), f = g - i0,
 * value = sum_{a,b,c in {0,1}} Wx_a Wy_b Wz_c F[i0+a, j0+b, k0+c],
 * W_0 = 1 - f, W_1 = f. */
void oracle_gather(const oracle_config *cfg, const double *F,
                   double x, double y, double z, double out[6])
{
    const int64_t N = cfg->nx * cfg->ny * cfg->nz;
    const double g[3] = {x / cfg->dx, y / cfg->dy, z / cfg->dz};
    for (int comp = 0; comp < 6; ++comp) {
        int64_t i0[3];
        double W[3][2];
        for (int d = 0; d < 3; ++d) {
            double s = g[d] - STAGGER[comp][d];
            double fl = floor(s);
            double f = s - fl;
            i0[d] = (int64_t)fl;
            W[d][0] = 1.0 - f;
            W[d][1] = f;
        }
        const double *Fc = F + comp * N;
        double sum = 0.0;
        for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    sum += W[0][a] * W[1][b] * W[2][c] *
                           (z_outside(cfg, i0[2] + c)
                                ? 0.0
                                : Fc[cell_index(cfg, i0[0] + a, i0[1] + b, i0[2] + c)]);
        out[comp] = sum;
    }
}

/* a4 -- relativistic Boris ("relativistic equations of motion";
 * reading R1 = SPEC.md:208-226).  du/dt = (q/(m c)) (E + (u/gamma) x B) in
 * Gaussian units with u = gamma*beta; h = q dt / (2 m c):
 *   u-  = u + h E
 *   g-  = sqrt(1 + |u-|^2)
 *   t   = h B / g-
 *   u'  = u- + u- x t
 *   s   = 2 / (1 + |t|^2)
 *   u+  = u- + s (u' x t)
 *   u   = u+ + h E                                                     */
void oracle_boris(double q, double m, double c, double dt,
                  const double EB[6], double u[3])
{
    const double h = q * dt / (2.0 * m * c);
    double um[3], t[3], up[3], upl[3];
    for (int d = 0; d < 3; ++d)
        um[d] = u[d] + h * EB[d];
    const double gm = sqrt(1.0 + (um[0] * um[0] + um[1] * um[1] + um[2] * um[2]));
    for (int d = 0; d < 3; ++d)
        t[d] = h * EB[3 + d] / gm;
    up[0] = um[0] + (um[1] * t[2] - um[2] * t[1]);
    up[1] = um[1] + (um[2] * t[0] - um[0] * t[2]);
    up[2] = um[2] + (um[0] * t[1] - um[1] * t[0]);
    const double s = 2.0 / (1.0 + (t[0] * t[0] + t[1] * t[1] + t[2] * t[2]));
    upl[0] = um[0] + s * (up[1] * t[2] - up[2] * t[1]);
    upl[1] = um[1] + s * (up[2] * t[0] - up[0] * t[2]);
    upl[2] = um[2] + s * (up[0] * t[1] - up[1] * t[0]);
    for (int d = 0; d < 3; ++d)
        u[d] = upl[d] + h * EB[d];
}

/* a4 (move) -- x' = x + dt v, v = c u / gamma, gamma = sqrt(1+|u|^2)
 * (SPEC.md:218-226).  No wrap: the raw displacement feeds the deposit. */
void oracle_move(double c, double dt, const double u[3], const double x[3],
                 double xn[3])
{
    const double g = sqrt(1.0 + (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]));
    for (int d = 0; d < 3; ++d)
        xn[d] = x[d] + dt * (c * u[d] / g);
}

/* Adds one straight in-cell segment P1->P2 (cell units) to J with the
 * Villasenor-Buneman edge weights:
 *   Jx(cx, cy+b, cz+g) += qw dX/(dt dy dz) [Wy(b) Wz(g) + s dY dZ/12]
 *   Jy(cx+a, cy, cz+g) += qw dY/(dt dx dz) [Wx(a) Wz(g) + s dX dZ/12]
 *   Jz(cx+a, cy+b, cz) += qw dZ/(dt dx dy) [Wx(a) Wy(b) + s dX dY/12]
 * with W(0) = 1 - mid, W(1) = mid (mid = segment midpoint in local cell
 * coordinates), s = +1 when the two edge offsets are equal, -1 otherwise. */
static void deposit_segment(const oracle_config *cfg, double qw,
                            const double P1[3], const double P2[3], double *J)
{
    const int64_t N = cfg->nx * cfg->ny * cfg->nz;
    int64_t cell[3];
    double D[3], W[3][2];
    for (int d = 0; d < 3; ++d) {
        double mid = 0.5 * (P1[d] + P2[d]);
        double fl = floor(mid);
        cell[d] = (int64_t)fl;
        D[d] = P2[d] - P1[d];
        double local = mid - fl;
        W[d][0] = 1.0 - local;
        W[d][1] = local;
    }
    const double fx = qw * D[0] / (cfg->dt * cfg->dy * cfg->dz);
    const double fy = qw * D[1] / (cfg->dt * cfg->dx * cfg->dz);
    const double fz = qw * D[2] / (cfg->dt * cfg->dx * cfg->dy);
    const double cxx = D[1] * D[2] / 12.0; /* for Jx */
    const double cyy = D[0] * D[2] / 12.0; /* for Jy */
    const double czz = D[0] * D[1] / 12.0; /* for Jz */
    for (int p = 0; p < 2; ++p) {
        for (int r = 0; r < 2; ++r) {
            const double s = (p == r) ? 1.0 : -1.0;
            if (!z_outside(cfg, cell[2] + r))
                J[0 * N + cell_index(cfg, cell[0], cell[1] + p, cell[2] + r)] +=
                    fx * (W[1][p] * W[2][r] + s * cxx);
            if (!z_outside(cfg, cell[2] + r))
                J[1 * N + cell_index(cfg, cell[0] + p, cell[1], cell[2] + r)] +=
                    fy * (W[0][p] * W[2][r] + s * cyy);
            if (!z_outside(cfg, cell[2]))
                J[2 * N + cell_index(cfg, cell[0] + p, cell[1] + r, cell[2])] +=
                    fz * (W[0][p] * W[1][r] + s * czz);
        }
    }
}

/* O5 -- charge-conserving Villasenor-Buneman deposit (PAPER.md:48,
 * "charge-conserving current deposition scheme [VillasenorBuneman]";
 * SPEC.md:228-246; readings R6, R8).  In cell units a = x/dx, b = x'/dx:
 * for every axis d with floor(a_d) != floor(b_d) the crossing plane is
 * p_d = max(floor a_d, floor b_d) at tau_d = (p_d - a_d)/(b_d - a_d);
 * the taus are sorted ascending (ties keep axis order) and the path is cut
 * into segments [tau_k, tau_k+1] of {0, taus, 1}.  The point at a crossing
 * has its crossing coordinate set exactly to p_d.  Zero-length segments
 * (tau_k+1 <= tau_k) are skipped.  Each segment is deposited in the cell
 * floor(midpoint). */
int oracle_deposit_vb(const oracle_config *cfg, double qw,
                      const double a_phys[3], const double b_phys[3], double *F)
{
    const int64_t N = cfg->nx * cfg->ny * cfg->nz;
    double *J = F + 6 * N;
    const double h[3] = {cfg->dx, cfg->dy, cfg->dz};
    double a[3], b[3];
    for (int d = 0; d < 3; ++d) {
        a[d] = a_phys[d] / h[d];
        b[d] = b_phys[d] / h[d];
        if (!isfinite(a[d]) || !isfinite(b[d]))
            return ORACLE_ENONFINITE;
        if (fabs(b[d] - a[d]) >= 1.0)
            return ORACLE_EDISPLACEMENT;
    }
    double tau[3];
    int axis[3];
    double plane[3];
    int nc = 0;
    for (int d = 0; d < 3; ++d) {
        double fa = floor(a[d]), fb = floor(b[d]);
        if (fa != fb) {
            double p = fa > fb ? fa : fb;
            tau[nc] = (p - a[d]) / (b[d] - a[d]);
            axis[nc] = d;
            plane[nc] = p;
            ++nc;
        }
    }
    /* insertion sort by tau, stable (ties keep ascending axis order) */
    for (int i = 1; i < nc; ++i) {
        for (int j = i; j > 0 && tau[j] < tau[j - 1]; --j) {
            double t = tau[j]; tau[j] = tau[j - 1]; tau[j - 1] = t;
            int ax = axis[j]; axis[j] = axis[j - 1]; axis[j - 1] = ax;
            double pl = plane[j]; plane[j] = plane[j - 1]; plane[j - 1] = pl;
        }
    }
    double P1[3] = {a[0], a[1], a[2]};
    double t1 = 0.0;
    for (int k = 0; k <= nc; ++k) {
        double P2[3], t2;
        if (k < nc) {
            t2 = tau[k];
            for (int d = 0; d < 3; ++d)
                P2[d] = a[d] + t2 * (b[d] - a[d]);
            P2[axis[k]] = plane[k];
        } else {
            t2 = 1.0;
            for (int d = 0; d < 3; ++d)
                P2[d] = b[d];
        }
        if (t2 > t1)
            deposit_segment(cfg, qw, P1, P2, J);
        for (int d = 0; d < 3; ++d)
            P1[d] = P2[d];
        t1 = t2;
    }
    return ORACLE_OK;
}

/* R7 -- periodic wrap: x >= L -> x - L (exact by Sterbenz); x < 0 -> x + L,
 * and a result that rounds to exactly L becomes 0. */
double oracle_wrap(double x, double L)
{
    if (x >= L)
        return x - L;
    if (x < 0.0) {
        double r = x + L;
        return r == L ? 0.0 : r;
    }
    return x;
}

/* R15 -- key = (supercell id, local cell id), both x-fastest; cell =
 * floor(x/dx), clamped to n-1 if the division rounds up to n. */
int64_t oracle_sort_key(const oracle_config *cfg, double x, double y, double z)
{
    const int64_t n[3] = {cfg->nx, cfg->ny, cfg->nz};
    const double pos[3] = {x / cfg->dx, y / cfg->dy, z / cfg->dz};
    const int64_t S = cfg->supercell;
    int64_t cell[3];
    for (int d = 0; d < 3; ++d) {
        int64_t ci = (int64_t)floor(pos[d]);
        if (ci >= n[d]) ci = n[d] - 1;
        if (ci < 0) ci = 0;
        cell[d] = ci;
    }
    const int64_t nsx = cfg->nx / S, nsy = cfg->ny / S;
    const int64_t sc = (cell[0] / S) + nsx * ((cell[1] / S) + nsy * (cell[2] / S));
    const int64_t local = (cell[0] % S) + S * ((cell[1] % S) + S * (cell[2] % S));
    return sc * S * S * S + local;
}

/* a1 -- re-binning sort of x,y,z,ux,uy,uz,id (
 * SPEC.md:298-306; reading R15 of DESIGN.md sec. 3).  Each particle gets
 *   cell key = oracle_sort_key(x) = (supercell id, local cell id), and
 *   slot     = number of particles with the same cell key before it in the
 *              current array order,
 * and the store is ordered by the unique triple (supercell id, slot, local
 * cell id): inside a supercell the slot-0 particles of all its cells come
 * first (in local cell order), then the slot-1 particles, and so on.
 * The triple is unique per particle, so the order is fully determined. */
typedef struct {
    int64_t sc, slot, local, p;
} sort_rec;

static int cmp_rec(const void *a, const void *b)
{
    const sort_rec *x = (const sort_rec *)a, *y = (const sort_rec *)b;
    if (x->sc != y->sc) return x->sc < y->sc ? -1 : 1;
    if (x->slot != y->slot) return x->slot < y->slot ? -1 : 1;
    if (x->local != y->local) return x->local < y->local ? -1 : 1;
    return 0;
}

void oracle_sort(const oracle_config *cfg, int64_t n, double *P, uint64_t *id)
{
    if (n <= 0)
        return;
    const int64_t nkeys = cfg->nx * cfg->ny * cfg->nz;
    const int64_t S3 = cfg->supercell * cfg->supercell * cfg->supercell;
    int64_t *seen = (int64_t *)calloc((size_t)nkeys, sizeof(int64_t));
    sort_rec *rec = (sort_rec *)malloc(sizeof(sort_rec) * (size_t)n);
    double *tmp = (double *)malloc(sizeof(double) * 6 * (size_t)n);
    uint64_t *tid = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    for (int64_t p = 0; p < n; ++p) {
        int64_t key = oracle_sort_key(cfg, P[p], P[n + p], P[2 * n + p]);
        rec[p].sc = key / S3;
        rec[p].local = key % S3;
        rec[p].slot = seen[key]++;
        rec[p].p = p;
    }
    qsort(rec, (size_t)n, sizeof(sort_rec), cmp_rec);
    for (int64_t dst = 0; dst < n; ++dst) {
        int64_t src = rec[dst].p;
        for (int c = 0; c < 6; ++c)
            tmp[c * n + dst] = P[c * n + src];
        tid[dst] = id[src];
    }
    memcpy(P, tmp, sizeof(double) * 6 * (size_t)n);
    memcpy(id, tid, sizeof(uint64_t) * (size_t)n);
    free(seen); free(rec); free(tmp); free(tid);
}

/* a7 / O3 -- B -= (c dt / 2) curl E, curl E evaluated at the B locations
 * with forward differences (R2). */
void oracle_b_half(const oracle_config *cfg, double *F)
{
    const int64_t nx = cfg->nx, ny = cfg->ny, nz = cfg->nz, N = nx * ny * nz;
    const double *Ex = F, *Ey = F + N, *Ez = F + 2 * N;
    double *Bx = F + 3 * N, *By = F + 4 * N, *Bz = F + 5 * N;
    const double k = cfg->c * cfg->dt / 2.0;
    for (int64_t kk = 0; kk < nz; ++kk)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                int64_t o = cell_index(cfg, i, j, kk);
                int64_t xp = cell_index(cfg, i + 1, j, kk);
                int64_t yp = cell_index(cfg, i, j + 1, kk);
                int64_t zp = cell_index(cfg, i, j, kk + 1);
                double cx = (Ez[yp] - Ez[o]) / cfg->dy - (Ey[zp] - Ey[o]) / cfg->dz;
                double cy = (Ex[zp] - Ex[o]) / cfg->dz - (Ez[xp] - Ez[o]) / cfg->dx;
                double cz = (Ey[xp] - Ey[o]) / cfg->dx - (Ex[yp] - Ex[o]) / cfg->dy;
                /* open z: Bx, By of the top plane sit at z = (nz - 1/2) dz,
                 * outside the box [0, (nz-1) dz]; they are not advanced */
                if (!(cfg->bc_z == ORACLE_BC_OPEN && kk == nz - 1)) {
                    Bx[o] = Bx[o] - k * cx;
                    By[o] = By[o] - k * cy;
                }
                Bz[o] = Bz[o] - k * cz;
            }
}

/* a7 / O3 -- E += c dt curl B - 4 pi dt J, curl B evaluated at the E
 * locations with backward differences (SPEC.md:82
 * Gaussian units, reading R3). */
void oracle_e_full(const oracle_config *cfg, double *F, int64_t step_index)
{
    const int64_t nx = cfg->nx, ny = cfg->ny, nz = cfg->nz, N = nx * ny * nz;
    double *Ex = F, *Ey = F + N, *Ez = F + 2 * N;
    const double *Bx = F + 3 * N, *By = F + 4 * N, *Bz = F + 5 * N;
    const double *Jx = F + 6 * N, *Jy = F + 7 * N, *Jz = F + 8 * N;
    const double k = cfg->c * cfg->dt;
    const double kj = 4.0 * M_PI * cfg->dt;
    const int open = cfg->bc_z == ORACLE_BC_OPEN;
    const int64_t P = nx * ny;   /* one z plane */
    double *old = NULL;          /* open z: Ex, Ey of planes 0, 1, nz-2, nz-1 at time n */
    if (open) {
        old = (double *)malloc(sizeof(double) * 8 * (size_t)P);
        const int64_t planes[4] = {0, 1, nz - 2, nz - 1};
        for (int q = 0; q < 4; ++q) {
            memcpy(old + (2 * q) * P, Ex + planes[q] * P, sizeof(double) * (size_t)P);
            memcpy(old + (2 * q + 1) * P, Ey + planes[q] * P, sizeof(double) * (size_t)P);
        }
    }
    for (int64_t kk = 0; kk < nz; ++kk)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                int64_t o = cell_index(cfg, i, j, kk);
                int64_t xm = cell_index(cfg, i - 1, j, kk);
                int64_t ym = cell_index(cfg, i, j - 1, kk);
                int64_t zm = cell_index(cfg, i, j, kk - 1);
                double cx = (Bz[o] - Bz[ym]) / cfg->dy - (By[o] - By[zm]) / cfg->dz;
                double cy = (Bx[o] - Bx[zm]) / cfg->dz - (Bz[o] - Bz[xm]) / cfg->dx;
                double cz = (By[o] - By[xm]) / cfg->dx - (Bx[o] - Bx[ym]) / cfg->dy;
                /* open z: Ex, Ey of planes 0 and nz-1 come from the boundary
                 * condition below; Ez of the top plane (z = (nz - 1/2) dz) lies
                 * outside the box and is not advanced */
                if (!(open && (kk == 0 || kk == nz - 1))) {
                    Ex[o] = Ex[o] + k * cx - kj * Jx[o];
                    Ey[o] = Ey[o] + k * cy - kj * Jy[o];
                }
                if (!(open && kk == nz - 1))
                    Ez[o] = Ez[o] + k * cz - kj * Jz[o];
            }
    if (open) {
        /* first-order Mur (one-way wave equation along the normal) on the
         * scattered field E - E_inc at z = 0 and on E at z = (nz-1) dz:
         *   E0^{n+1} = I0^{n+1} + (E1^n - I1^n) + a ((E1^{n+1} - I1^{n+1}) - (E0^n - I0^n))
         *   EK^{n+1} = E(K-1)^n + a (E(K-1)^{n+1} - EK^n),   a = (c dt - dz)/(c dt + dz),
         * I_k^n = pol E_inc(k dz, n dt) (reading R21). */
        const double a = (cfg->c * cfg->dt - cfg->dz) / (cfg->c * cfg->dt + cfg->dz);
        const double t0 = (double)step_index * cfg->dt, t1 = (double)(step_index + 1) * cfg->dt;
        const double i00 = oracle_laser(cfg, 0.0, t0), i01 = oracle_laser(cfg, 0.0, t1);
        const double i10 = oracle_laser(cfg, cfg->dz, t0), i11 = oracle_laser(cfg, cfg->dz, t1);
        const double pol[2] = {cfg->laser_pol_x, cfg->laser_pol_y};
        double *E[2] = {Ex, Ey};
        for (int c = 0; c < 2; ++c)
            for (int64_t q = 0; q < P; ++q) {
                const double e0o = old[(0 + c) * P + q], e1o = old[(2 + c) * P + q];
                const double eKm1o = old[(4 + c) * P + q], eKo = old[(6 + c) * P + q];
                const double e1n = E[c][1 * P + q], eKm1n = E[c][(nz - 2) * P + q];
                E[c][0 * P + q] = pol[c] * i01 + (e1o - pol[c] * i10) +
                                  a * ((e1n - pol[c] * i11) - (e0o - pol[c] * i00));
                E[c][(nz - 1) * P + q] = eKm1o + a * (eKm1n - eKo);
            }
        free(old);
    }
}

/* NEXT-1 -- the incident plane wave of BASELINE.json configs[4] ("a
 * linearly polarised plane wave of normalised amplitude a0 ... injected from
 * z=0"; reading R21): E_inc(z, t) = E0 env(xi) sin(omega xi),
 * xi = t + t0 - z / c. */
double oracle_laser(const oracle_config *cfg, double z, double t)
{
    const double xi = t + cfg->laser_t0 - z / cfg->c;
    if (!(xi > 0.0))
        return 0.0;
    double env = 1.0;
    if (xi < cfg->laser_ramp) {
        const double sr = sin(M_PI * xi / (2.0 * cfg->laser_ramp));
        env = sr * sr;
    }
    return cfg->laser_e0 * env * sin(cfg->laser_omega * xi);
}

void oracle_laser_preload(const oracle_config *cfg, double *F)
{
    const int64_t nx = cfg->nx, ny = cfg->ny, nz = cfg->nz, N = nx * ny * nz, P = nx * ny;
    memset(F, 0, sizeof(double) * 6 * (size_t)N);
    for (int64_t kk = 0; kk < nz; ++kk) {
        const double e = oracle_laser(cfg, (double)kk * cfg->dz, 0.0);
        const double b = kk < nz - 1 ? oracle_laser(cfg, ((double)kk + 0.5) * cfg->dz, 0.0) : 0.0;
        for (int64_t q = 0; q < P; ++q) {
            F[0 * N + kk * P + q] = cfg->laser_pol_x * e;
            F[1 * N + kk * P + q] = cfg->laser_pol_y * e;
            F[3 * N + kk * P + q] = -cfg->laser_pol_y * b;
            F[4 * N + kk * P + q] = cfg->laser_pol_x * b;
        }
    }
}

/* O2 step 2 for one species, particles in array order:
 * gather E^n,B^n -> Boris -> move -> VB deposit x -> x' -> wrap x'. */
int oracle_push_species(const oracle_config *cfg, double *F, int species,
                        int64_t *n_io, double *P, uint64_t *id)
{
    const double q = cfg->q[species], m = cfg->m[species], w = cfg->w[species];
    const double L[3] = {cfg->nx * cfg->dx, cfg->ny * cfg->dy, cfg->nz * cfg->dz};
    const int open = cfg->bc_z == ORACLE_BC_OPEN;
    const double zmax = (double)(cfg->nz - 1) * cfg->dz;   /* open z: particles live in [0, zmax) */
    const int64_t n = *n_io;
    unsigned char *gone = open ? (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1) : NULL;
    int64_t kept = n;
    for (int64_t p = 0; p < n; ++p) {
        double x[3] = {P[p], P[n + p], P[2 * n + p]};
        double u[3] = {P[3 * n + p], P[4 * n + p], P[5 * n + p]};
        double EB[6], xn[3];
        oracle_gather(cfg, F, x[0], x[1], x[2], EB);
        oracle_boris(q, m, cfg->c, cfg->dt, EB, u);
        oracle_move(cfg->c, cfg->dt, u, x, xn);
        int rc = oracle_deposit_vb(cfg, q * w, x, xn, F);
        if (rc != ORACLE_OK) {
            free(gone);
            return rc;
        }
        for (int d = 0; d < 3; ++d) {
            P[d * n + p] = (open && d == 2) ? xn[d] : oracle_wrap(xn[d], L[d]);
            P[(3 + d) * n + p] = u[d];
        }
        if (open && !(xn[2] >= 0.0 && xn[2] < zmax)) {   /* left through an open face */
            gone[p] = 1;
            --kept;
        }
    }
    if (open && kept < n) {
        /* remove in place, keeping the order; rows move to stride `kept`
         * (every write index is <= its read index, so nothing unread is overwritten) */
        for (int c = 0; c < 6; ++c) {
            int64_t k = 0;
            for (int64_t p = 0; p < n; ++p)
                if (!gone[p])
                    P[c * kept + k++] = P[c * n + p];
        }
        int64_t k = 0;
        for (int64_t p = 0; p < n; ++p)
            if (!gone[p])
                id[k++] = id[p];
    }
    free(gone);
    *n_io = kept;
    return ORACLE_OK;
}

/* O2 -- one step n -> n+1 (SPEC.md:476-484 order with
 * the loop boundary moved so stored B is at integer time; R5, R15, R16):
 *   1. if n % K == 0: stable sort every species;
 *   2. zero J; per species, per particle: gather, Boris, move, deposit, wrap;
 *   3. B half-step with E^n; 4. E full step with B^{n+1/2} and J^{n+1/2};
 *   5. B half-step with E^{n+1}. */
int oracle_step(const oracle_config *cfg, double *F, int64_t *counts,
                double *const *P, uint64_t *const *ids, int64_t step_index)
{
    const int64_t N = cfg->nx * cfg->ny * cfg->nz;
    if (cfg->sort_every > 0 && step_index % cfg->sort_every == 0)
        for (int s = 0; s < cfg->n_species; ++s)
            oracle_sort(cfg, counts[s], P[s], ids[s]);
    memset(F + 6 * N, 0, sizeof(double) * 3 * (size_t)N);
    for (int s = 0; s < cfg->n_species; ++s) {
        int rc = oracle_push_species(cfg, F, s, &counts[s], P[s], ids[s]);
        if (rc != ORACLE_OK)
            return rc;
    }
    oracle_b_half(cfg, F);
    oracle_e_full(cfg, F, step_index);
    oracle_b_half(cfg, F);
    return ORACLE_OK;
}

/* ---- diagnostics ---- */

/* rho at nodes (i,j,k): q w / (dx dy dz) * S(x/dx - i) S(y/dy - j) S(z/dz - k),
 * S = linear hat (the CIC shape whose flux VB deposits). */
void oracle_deposit_rho(const oracle_config *cfg, double qw, int64_t n,
                        const double *P, double *rho)
{
    const double inv_v = 1.0 / (cfg->dx * cfg->dy * cfg->dz);
    for (int64_t p = 0; p < n; ++p) {
        const double g[3] = {P[p] / cfg->dx, P[n + p] / cfg->dy, P[2 * n + p] / cfg->dz};
        int64_t i0[3];
        double W[3][2];
        for (int d = 0; d < 3; ++d) {
            double fl = floor(g[d]);
            i0[d] = (int64_t)fl;
            W[d][1] = g[d] - fl;
            W[d][0] = 1.0 - W[d][1];
        }
        for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    rho[cell_index(cfg, i0[0] + a, i0[1] + b, i0[2] + c)] +=
                        qw * inv_v * W[0][a] * W[1][b] * W[2][c];
    }
}

/* div of an edge-located vector (E or J) at node (i,j,k):
 * (Vx[i]-Vx[i-1])/dx + (Vy[j]-Vy[j-1])/dy + (Vz[k]-Vz[k-1])/dz. */
void oracle_div_edge(const oracle_config *cfg, const double *Vx, const double *Vy,
                     const double *Vz, double *out)
{
    for (int64_t k = 0; k < cfg->nz; ++k)
        for (int64_t j = 0; j < cfg->ny; ++j)
            for (int64_t i = 0; i < cfg->nx; ++i) {
                int64_t o = cell_index(cfg, i, j, k);
                out[o] = (Vx[o] - Vx[cell_index(cfg, i - 1, j, k)]) / cfg->dx +
                         (Vy[o] - Vy[cell_index(cfg, i, j - 1, k)]) / cfg->dy +
                         (Vz[o] - Vz[cell_index(cfg, i, j, k - 1)]) / cfg->dz;
            }
}

/* div of a face-located vector (B) at cell centre (i+1/2,j+1/2,k+1/2). */
void oracle_div_face(const oracle_config *cfg, const double *Bx, const double *By,
                     const double *Bz, double *out)
{
    for (int64_t k = 0; k < cfg->nz; ++k)
        for (int64_t j = 0; j < cfg->ny; ++j)
            for (int64_t i = 0; i < cfg->nx; ++i) {
                int64_t o = cell_index(cfg, i, j, k);
                out[o] = (Bx[cell_index(cfg, i + 1, j, k)] - Bx[o]) / cfg->dx +
                         (By[cell_index(cfg, i, j + 1, k)] - By[o]) / cfg->dy +
                         (Bz[cell_index(cfg, i, j, k + 1)] - Bz[o]) / cfg->dz;
            }
}

double oracle_field_energy(const oracle_config *cfg, const double *F)
{
    const int64_t N = cfg->nx * cfg->ny * cfg->nz;
    double sum = 0.0;
    for (int64_t o = 0; o < 6 * N; ++o)
        sum += F[o] * F[o];
    return sum * (cfg->dx * cfg->dy * cfg->dz) / (8.0 * M_PI);
}

double oracle_kinetic_energy(const oracle_config *cfg, int species, int64_t n,
                             const double *P)
{
    double sum = 0.0;
    for (int64_t p = 0; p < n; ++p) {
        double u2 = P[3 * n + p] * P[3 * n + p] + P[4 * n + p] * P[4 * n + p] +
                    P[5 * n + p] * P[5 * n + p];
        /* gamma - 1 = u^2 / (sqrt(1+u^2) + 1), no cancellation */
        sum += u2 / (sqrt(1.0 + u2) + 1.0);
    }
    return sum * cfg->w[species] * cfg->m[species] * cfg->c * cfg->c;
}
