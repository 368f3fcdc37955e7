// fields.cu -- Yee FDTD update on the ghost-padded grid.
//
//   B^{n+1/2} = B^n       - (c dt/2) curl E^n
//   E^{n+1}   = E^n       + c dt curl B^{n+1/2} - 4 pi dt J^{n+1/2}
//   B^{n+1}   = B^{n+1/2} - (c dt/2) curl E^{n+1}
// ("numerical integration of Maxwell's equations"; reading R2,
// Gaussian units R3).  curl E uses forward differences at the B locations,
// curl B backward differences at the E locations.  One thread per interior
// cell, x fastest (coalesced); neighbours come from the ghost layers, so no
// index wraps.  The producing thread also stores its value into every
// periodic ghost image (x, y always; z when the slab is the whole box), so
// no separate ghost-fill pass runs (HBM-bound; the ghost stores are a
// surface term).  With open z (NEXT-1) the faces z = 0 and z = zmax take
// first-order Mur with the incident laser (k_e_full, k_laser_coeffs).
#include "kernels.cuh"

namespace pic {

// B half step(s) with the curl of E (the E of EB):
//   B1 = Bin - coef curl E   -> Bout1
//   B2 = B1  - coef curl E   -> Bout2 (when Bout2 != nullptr)
// The step's second half (B^{n+1}, read by the particle kernel) and the next
// step's first half (B^{n+3/2}, read by the next E update) use the same
// curl E^{n+1}, so one pass writes both: the same two fma's, in the same
// order, as two separate half steps.  Bin may alias Bout2 (each thread reads
// only its own cell of Bin).
__global__ void __launch_bounds__(256)
k_b_half(GridDev g, const double *__restrict__ EB, const double *Bin, double *Bout1, double *Bout2,
         double coef, int kbegin)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z + kbegin;
    if (i >= g.nx || j >= g.ny) return;
    const int64_t cs = g.cs, sy = g.X, sz = (int64_t)g.X * g.Y;
    const double *Ex = EB, *Ey = EB + cs, *Ez = EB + 2 * cs;
    const int64_t o = pidx(g, i, j, k);
    const double ex = Ex[o], ey = Ey[o], ez = Ez[o];
    const double cx = (Ez[o + sy] - ez) * g.inv_dy - (Ey[o + sz] - ey) * g.inv_dz;
    const double cy = (Ex[o + sz] - ex) * g.inv_dz - (Ez[o + 1] - ez) * g.inv_dx;
    const double cz = (Ey[o + 1] - ey) * g.inv_dx - (Ex[o + sy] - ex) * g.inv_dy;
    // open z (NEXT-1): Bx, By of the top plane sit at z = zmax + dz/2, outside
    // the box; they are not advanced
    const bool outside = g.open_hi && k == g.nz - 1;
    const double bx0 = Bin[o], by0 = Bin[cs + o], bz0 = Bin[2 * cs + o];
    const double bx = outside ? bx0 : fma(-coef, cx, bx0);
    const double by = outside ? by0 : fma(-coef, cy, by0);
    const double bz = fma(-coef, cz, bz0);
    for_images(g, i, j, k, [&](int64_t p) {
        Bout1[p] = bx;
        Bout1[cs + p] = by;
        Bout1[2 * cs + p] = bz;
    });
    if (Bout2) {
        const double bx2 = outside ? bx : fma(-coef, cx, bx);
        const double by2 = outside ? by : fma(-coef, cy, by);
        const double bz2 = fma(-coef, cz, bz);
        for_images(g, i, j, k, [&](int64_t p) {
            Bout2[p] = bx2;
            Bout2[cs + p] = by2;
            Bout2[2 * cs + p] = bz2;
        });
    }
}

// does interior plane k (or, at an open face, its z ghost planes) have an
// image among the padded planes [lo, hi]
__device__ __forceinline__ bool j_plane_live(const GridDev &g, int k, int lo, int hi)
{
    const int kp = k + kGhost;
    if (hi < lo) return false;
    if (g.periodic_z_local)
        return (kp >= lo && kp <= hi) || (kp - g.nz >= lo && kp - g.nz <= hi) ||
               (kp + g.nz >= lo && kp + g.nz <= hi);
    const int a = k == 0 ? 0 : kp, b = k == g.nz - 1 ? g.Z - 1 : kp;
    return a <= hi && b >= lo;
}

__global__ void __launch_bounds__(256)
k_e_full(GridDev g, double *__restrict__ EB, const double *__restrict__ Bh, double *__restrict__ Jc,
         double *__restrict__ Jn, double coefE, double coefJ, StepPrep prep, JPlanes jl)
{
    // the next step's J-tile scales (this step's particle kernels are done)
    if ((blockIdx.x | blockIdx.y | blockIdx.z | threadIdx.y) == 0 && (int)threadIdx.x < prep.n_species)
        step_prep_species(prep, threadIdx.x);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z;
    if (i >= g.nx || j >= g.ny) return;
    const int64_t cs = g.cs, sy = g.X, sz = (int64_t)g.X * g.Y;
    double *Ex = EB, *Ey = EB + cs, *Ez = EB + 2 * cs;
    const double *Bx = Bh, *By = Bh + cs, *Bz = Bh + 2 * cs;   // B^{n+1/2}
    const int64_t o = pidx(g, i, j, k);
    // fold: the deposit of step n landed on the interior cell and its images
    // (planes no particle deposited into hold zeros: not read, not cleared)
    const bool live = j_plane_live(g, k, jl.cur_lo, jl.cur_hi), dirty = j_plane_live(g, k, jl.next_lo, jl.next_hi);
    double jx = 0.0, jy = 0.0, jz = 0.0;
    int nimg = 0;
    if (live || dirty)
        for_images(g, i, j, k, [&](int64_t p) {
            if (live) {
                jx += Jc[p];
                jy += Jc[cs + p];
                jz += Jc[2 * cs + p];
            }
            if (dirty) {
                Jn[p] = 0.0;
                Jn[cs + p] = 0.0;
                Jn[2 * cs + p] = 0.0;
            }
            ++nimg;
        });
    if (live && nimg > 1) {   // the folded J (J^{n+1/2} for pic_get_fields); a cell
        Jc[o] = jx;           // without images already holds it
        Jc[cs + o] = jy;
        Jc[2 * cs + o] = jz;
    }
    const double bx = Bx[o], by = By[o], bz = Bz[o];
    const double cx = (bz - Bz[o - sy]) * g.inv_dy - (by - By[o - sz]) * g.inv_dz;
    const double cy = (bx - Bx[o - sz]) * g.inv_dz - (bz - Bz[o - 1]) * g.inv_dx;
    const double cz = (by - By[o - 1]) * g.inv_dx - (bx - Bx[o - sy]) * g.inv_dy;
    const double ex_old = Ex[o], ey_old = Ey[o];
    const double ex = fma(-coefJ, jx, fma(coefE, cx, ex_old));
    const double ey = fma(-coefJ, jy, fma(coefE, cy, ey_old));
    const double ez = fma(-coefJ, jz, fma(coefE, cz, Ez[o]));
    if (!g.open_z) {
        for_images(g, i, j, k, [&](int64_t p) {
            Ex[p] = ex;
            Ey[p] = ey;
            Ez[p] = ez;
        });
        return;
    }
    // ---- open z (NEXT-1, reading R21) ----
    // the tangential E of the faces z = 0 (local plane 0 of the lowest rank)
    // and z = zmax (local plane nz-1 of the highest) come from first-order Mur
    // on the scattered field E - E_inc, evaluated by the thread of the plane
    // next to the face, which holds that plane's old and new value; Ez of the
    // top plane lies outside the box and is not advanced
    const bool face_lo = g.open_lo && k == 0, face_hi = g.open_hi && k == g.nz - 1;
    for_images(g, i, j, k, [&](int64_t p) {
        if (!face_lo && !face_hi) {
            Ex[p] = ex;
            Ey[p] = ey;
        }
        if (!face_hi) Ez[p] = ez;
    });
    const double a = g.mur_a;
    if (g.open_lo && k == 1) {
        // E0' = I0' + (E1 - I1) + a ((E1' - I1') - (E0 - I0)); laser = [c][I0', I1, I1', I0]
        const double *I = g.laser;
        const double e0x = Ex[o - sz], e0y = Ey[o - sz];
        const double nx0 = I[0] + (ex_old - I[1]) + a * ((ex - I[2]) - (e0x - I[3]));
        const double ny0 = I[4] + (ey_old - I[5]) + a * ((ey - I[6]) - (e0y - I[7]));
        for_images(g, i, j, 0, [&](int64_t p) {
            Ex[p] = nx0;
            Ey[p] = ny0;
        });
    }
    if (g.open_hi && k == g.nz - 2) {
        // EK' = E(K-1) + a (E(K-1)' - EK)
        const double eKx = Ex[o + sz], eKy = Ey[o + sz];
        const double nxK = ex_old + a * (ex - eKx);
        const double nyK = ey_old + a * (ey - eKy);
        for_images(g, i, j, g.nz - 1, [&](int64_t p) {
            Ex[p] = nxK;
            Ey[p] = nyK;
        });
    }
    if (g.nranks == 1 && dirty) {
        // no z images and no slab exchange: clear the z ghost planes of J_next
        // (the deposit spills beyond the faces; those values are dropped)
        const int kz0 = k == 0 ? -kGhost : (k == g.nz - 1 ? g.nz : 0);
        if (k == 0 || k == g.nz - 1)
            for (int kk = kz0; kk < kz0 + kGhost; ++kk)
                for_images(g, i, j, kk, [&](int64_t p) {
                    Jn[p] = 0.0;
                    Jn[cs + p] = 0.0;
                    Jn[2 * cs + p] = 0.0;
                });
    }
}

// NEXT-1: the incident values of step n -> n+1 at the open face z = 0, from
// the device step counter (so the step stays one CUDA graph):
// laser[c*4 + {0,1,2,3}] = pol_c {E_inc(0,t'), E_inc(dz,t), E_inc(dz,t'), E_inc(0,t)},
// t = n dt, t' = (n+1) dt;  E_inc(z,t) = e0 env(xi) sin(omega xi), xi = t + t0 - z/c.
struct LaserDev {
    double e0, omega, ramp, t0, pol[2];
};

__device__ double laser_inc(const LaserDev &L, double c, double z, double t)
{
    const double xi = t + L.t0 - z / c;
    if (!(xi > 0.0)) return 0.0;
    double env = 1.0;
    if (xi < L.ramp) {
        const double sr = sin(M_PI * xi / (2.0 * L.ramp));
        env = sr * sr;
    }
    return L.e0 * env * sin(L.omega * xi);
}

__global__ void k_laser_coeffs(GridDev g, LaserDev L, int64_t *step, double *laser)
{
    if (threadIdx.x != 0) return;
    const int64_t n = *step;
    const double t0 = (double)n * g.dt, t1 = (double)(n + 1) * g.dt;
    const double v[4] = {laser_inc(L, g.c, 0.0, t1), laser_inc(L, g.c, g.dz, t0), laser_inc(L, g.c, g.dz, t1),
                         laser_inc(L, g.c, 0.0, t0)};
    for (int c = 0; c < 2; ++c)
        for (int q = 0; q < 4; ++q) laser[4 * c + q] = L.pol[c] * v[q];
    *step = n + 1;
}

// NEXT-1: fields of the local slab = the incident wave at t = 0 (pic_laser_preload)
__global__ void __launch_bounds__(256) k_laser_preload(GridDev g, LaserDev L, double *__restrict__ EB)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z;
    if (i >= g.nx || j >= g.ny) return;
    const int64_t cs = g.cs;
    const int kg = g.k0 + k;
    const double e = laser_inc(L, g.c, (double)kg * g.dz, 0.0);
    const double b = kg < g.nz_global - 1 ? laser_inc(L, g.c, ((double)kg + 0.5) * g.dz, 0.0) : 0.0;
    for_images(g, i, j, k, [&](int64_t p) {
        EB[p] = L.pol[0] * e;
        EB[cs + p] = L.pol[1] * e;
        EB[2 * cs + p] = 0.0;
        EB[3 * cs + p] = -L.pol[1] * b;
        EB[4 * cs + p] = L.pol[0] * b;
        EB[5 * cs + p] = 0.0;
    });
}

__global__ void __launch_bounds__(256) k_fill_ghosts(GridDev g, double *__restrict__ F, int ncomp)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z;
    if (i >= g.nx || j >= g.ny) return;
    const int64_t o = pidx(g, i, j, k);
    for (int c = 0; c < ncomp; ++c) {
        double *Fc = F + c * g.cs;
        const double v = Fc[o];
        for_images(g, i, j, k, [&](int64_t p) {
            if (p != o) Fc[p] = v;
        });
    }
}

static dim3 field_grid(const GridDev &g, dim3 bs)
{
    return dim3((g.nx + bs.x - 1) / bs.x, (g.ny + bs.y - 1) / bs.y, g.nz);
}

void launch_b_half(const GridDev &g, const double *EB, const double *Bin, double *Bout1, double *Bout2,
                   cudaStream_t st, int kbegin)
{
    const dim3 bs(32, 8, 1);
    dim3 grid = field_grid(g, bs);
    grid.z = g.nz - kbegin;
    k_b_half<<<grid, bs, 0, st>>>(g, EB, Bin, Bout1, Bout2, 0.5 * g.c * g.dt, kbegin);
}

void launch_e_full(const GridDev &g, double *EB, const double *Bh, double *Jcur, double *Jnext,
                   const StepPrep &prep, cudaStream_t st, const JPlanes &jl)
{
    const dim3 bs(32, 8, 1);
    k_e_full<<<field_grid(g, bs), bs, 0, st>>>(g, EB, Bh, Jcur, Jnext, g.c * g.dt,
                                                4.0 * M_PI * g.dt, prep, jl);
}

void launch_laser_coeffs(const GridDev &g, const double laser[6], int64_t *step, double *out, cudaStream_t st)
{
    const LaserDev L{laser[0], laser[1], laser[2], laser[3], {laser[4], laser[5]}};
    k_laser_coeffs<<<1, 32, 0, st>>>(g, L, step, out);
}

void launch_laser_preload(const GridDev &g, const double laser[6], double *EB, cudaStream_t st)
{
    const LaserDev L{laser[0], laser[1], laser[2], laser[3], {laser[4], laser[5]}};
    const dim3 bs(32, 8, 1);
    k_laser_preload<<<field_grid(g, bs), bs, 0, st>>>(g, L, EB);
}

void launch_fill_ghosts(const GridDev &g, double *F, int ncomp, cudaStream_t st)
{
    const dim3 bs(32, 8, 1);
    k_fill_ghosts<<<field_grid(g, bs), bs, 0, st>>>(g, F, ncomp);
}

}  // namespace pic
