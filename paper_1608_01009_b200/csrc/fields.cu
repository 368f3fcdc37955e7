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
// surface term).
#include "kernels.cuh"

namespace pic {

__global__ void __launch_bounds__(256) k_b_half(GridDev g, double *__restrict__ EB, double coef, int kbegin)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z + kbegin;
    if (i >= g.nx || j >= g.ny) return;
    const int64_t cs = g.cs, sy = g.X, sz = (int64_t)g.X * g.Y;
    const double *Ex = EB, *Ey = EB + cs, *Ez = EB + 2 * cs;
    double *Bx = EB + 3 * cs, *By = EB + 4 * cs, *Bz = EB + 5 * cs;
    const int64_t o = pidx(g, i, j, k);
    const double ex = Ex[o], ey = Ey[o], ez = Ez[o];
    const double cx = (Ez[o + sy] - ez) * g.inv_dy - (Ey[o + sz] - ey) * g.inv_dz;
    const double cy = (Ex[o + sz] - ex) * g.inv_dz - (Ez[o + 1] - ez) * g.inv_dx;
    const double cz = (Ey[o + 1] - ey) * g.inv_dx - (Ex[o + sy] - ex) * g.inv_dy;
    const double bx = fma(-coef, cx, Bx[o]);
    const double by = fma(-coef, cy, By[o]);
    const double bz = fma(-coef, cz, Bz[o]);
    for_images(g, i, j, k, [&](int64_t p) {
        Bx[p] = bx;
        By[p] = by;
        Bz[p] = bz;
    });
}

__global__ void __launch_bounds__(256)
k_e_full(GridDev g, double *__restrict__ EB, double *__restrict__ Jc, double *__restrict__ Jn,
         double coefE, double coefJ)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z;
    if (i >= g.nx || j >= g.ny) return;
    const int64_t cs = g.cs, sy = g.X, sz = (int64_t)g.X * g.Y;
    double *Ex = EB, *Ey = EB + cs, *Ez = EB + 2 * cs;
    const double *Bx = EB + 3 * cs, *By = EB + 4 * cs, *Bz = EB + 5 * cs;
    const int64_t o = pidx(g, i, j, k);
    // fold: the deposit of step n landed on the interior cell and its images
    double jx = 0.0, jy = 0.0, jz = 0.0;
    for_images(g, i, j, k, [&](int64_t p) {
        jx += Jc[p];
        jy += Jc[cs + p];
        jz += Jc[2 * cs + p];
        Jn[p] = 0.0;
        Jn[cs + p] = 0.0;
        Jn[2 * cs + p] = 0.0;
    });
    Jc[o] = jx;
    Jc[cs + o] = jy;
    Jc[2 * cs + o] = jz;
    const double bx = Bx[o], by = By[o], bz = Bz[o];
    const double cx = (bz - Bz[o - sy]) * g.inv_dy - (by - By[o - sz]) * g.inv_dz;
    const double cy = (bx - Bx[o - sz]) * g.inv_dz - (bz - Bz[o - 1]) * g.inv_dx;
    const double cz = (by - By[o - 1]) * g.inv_dx - (bx - Bx[o - sy]) * g.inv_dy;
    const double ex = fma(-coefJ, jx, fma(coefE, cx, Ex[o]));
    const double ey = fma(-coefJ, jy, fma(coefE, cy, Ey[o]));
    const double ez = fma(-coefJ, jz, fma(coefE, cz, Ez[o]));
    for_images(g, i, j, k, [&](int64_t p) {
        Ex[p] = ex;
        Ey[p] = ey;
        Ez[p] = ez;
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

void launch_b_half(const GridDev &g, double *EB, cudaStream_t st, int kbegin)
{
    const dim3 bs(32, 8, 1);
    dim3 grid = field_grid(g, bs);
    grid.z = g.nz - kbegin;
    k_b_half<<<grid, bs, 0, st>>>(g, EB, 0.5 * g.c * g.dt, kbegin);
}

void launch_e_full(const GridDev &g, double *EB, double *Jcur, double *Jnext, cudaStream_t st)
{
    const dim3 bs(32, 8, 1);
    k_e_full<<<field_grid(g, bs), bs, 0, st>>>(g, EB, Jcur, Jnext, g.c * g.dt,
                                                4.0 * M_PI * g.dt);
}

void launch_fill_ghosts(const GridDev &g, double *F, int ncomp, cudaStream_t st)
{
    const dim3 bs(32, 8, 1);
    k_fill_ghosts<<<field_grid(g, bs), bs, 0, st>>>(g, F, ncomp);
}

}  // namespace pic
