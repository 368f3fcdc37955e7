// diag.cu -- GPU diagnostics of the step state (
// SPEC.md:379-443 for the quantities): CIC charge density rho^n, Gauss
// residual div E - 4 pi rho and its drift, div B, the continuity residual
// (rho^n - rho^{n-1})/dt + div J^{n-1/2}, field and kinetic energy, total
// charge and current.  Not on the timed hot path: called between steps.
//
//   rho(i,j,k)  = sum_p q w S(x-i) S(y-j) S(z-k) / (dx dy dz), S(t) = max(0, 1-|t|)
//   div E, div J at nodes: backward differences (the E/J edge locations
//                (i+1/2,j,k), ... surround node (i,j,k) from above)
//   div B at cell centres: forward differences
// These are the definitions the VB deposit conserves exactly (P11) and the
// Yee update preserves (P12), so on the GPU state they are physics checks at
// sizes the oracle cannot run in full.
#include "kernels.cuh"

namespace pic {

// CIC charge deposit of live particles [0, *dev_n) into the padded node array
// (nodes i0, i0+1 per axis; i0+1 = n lands in the ghost layer, folded below)
__global__ void __launch_bounds__(256)
k_rho_deposit(GridDev g, ParticlesDev P, const int64_t *dev_n, double qw_v, double *__restrict__ rho)
{
    const int64_t n = *dev_n;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double x = P.x[p];
        if (x < 0.0) continue;   // dead slot (migrated away)
        const double gx = x * g.inv_dx, gy = P.y[p] * g.inv_dy, gz = P.z[p] * g.inv_dz;
        const double fx = floor(gx), fy = floor(gy), fz = floor(gz);
        const int i0 = (int)fx, j0 = (int)fy, k0 = (int)fz - g.k0;
        const double wx[2] = {1.0 - (gx - fx), gx - fx};
        const double wy[2] = {1.0 - (gy - fy), gy - fy};
        const double wz[2] = {1.0 - (gz - fz), gz - fz};
        for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a)
                    atomicAdd(rho + pidx(g, i0 + a, j0 + b, k0 + c), qw_v * wx[a] * wy[b] * wz[c]);
    }
}

// interior node = sum of its periodic images (+ the plane the lower slab
// deposited above its top, received in `below`)
__global__ void __launch_bounds__(256)
k_rho_fold(GridDev g, double *__restrict__ rho, const double *__restrict__ below)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z;
    if (i >= g.nx || j >= g.ny) return;
    double s = 0.0;
    for_images(g, i, j, k, [&](int64_t p) { s += rho[p]; });
    if (below && k == 0)   // the received plane is unfolded in x and y as well
        for (int jj = first_image(j, g.ny); jj < g.ny + kGhost; jj += g.ny)
            for (int ii = first_image(i, g.nx); ii < g.nx + kGhost; ii += g.nx)
                s += below[(int64_t)(ii + kGhost) + (int64_t)g.X * (jj + kGhost)];
    rho[pidx(g, i, j, k)] = s;
}

__device__ __forceinline__ void atomic_max_nonneg(double *a, double v)
{
    // non-negative doubles order like their bit patterns
    atomicMax((unsigned long long *)a, (unsigned long long)__double_as_longlong(v));
}

// acc: [0] sum F^2  [1] sum rho  [2..4] sum J  [5] max|div B|  [6] max|gauss|
//      [7] max gauss drift  [8] max|continuity|
__global__ void __launch_bounds__(256)
k_diag_nodes(GridDev g, const double *__restrict__ EB, const double *__restrict__ J,
             const double *__restrict__ jz_below, const double *__restrict__ rho,
             double *__restrict__ rho_prev, double *__restrict__ gauss0, int have_prev, int have_g0,
             double *__restrict__ acc)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z;
    double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (i < g.nx && j < g.ny) {
        const int64_t cs = g.cs, sy = g.X, sz = (int64_t)g.X * g.Y;
        const int64_t o = pidx(g, i, j, k);
        const double *Ex = EB, *Ey = EB + cs, *Ez = EB + 2 * cs;
        const double *Bx = EB + 3 * cs, *By = EB + 4 * cs, *Bz = EB + 5 * cs;
        for (int c = 0; c < 6; ++c) v[0] += EB[c * cs + o] * EB[c * cs + o];
        const double r = rho[o];
        v[1] = r;
        const double *Jx = J, *Jy = J + cs, *Jz = J + 2 * cs;
        v[2] = Jx[o];
        v[3] = Jy[o];
        v[4] = Jz[o];
        // div B at the cell centre (B ghosts are valid images at a step boundary)
        const double divb = (Bx[o + 1] - Bx[o]) * g.inv_dx + (By[o + sy] - By[o]) * g.inv_dy +
                            (Bz[o + sz] - Bz[o]) * g.inv_dz;
        v[5] = fabs(divb);
        const double dive = (Ex[o] - Ex[o - 1]) * g.inv_dx + (Ey[o] - Ey[o - sy]) * g.inv_dy +
                            (Ez[o] - Ez[o - sz]) * g.inv_dz;
        const double gauss = dive - 4.0 * M_PI * r;
        v[6] = fabs(gauss);
        if (have_g0) v[7] = fabs(gauss - gauss0[o]);
        else gauss0[o] = gauss;
        // J ghosts are not images (the E update folded them), so wrap explicitly
        const int64_t oxm = pidx(g, i == 0 ? g.nx - 1 : i - 1, j, k);
        const int64_t oym = pidx(g, i, j == 0 ? g.ny - 1 : j - 1, k);
        double jzm;
        if (k > 0) jzm = Jz[o - sz];
        else if (g.periodic_z_local) jzm = Jz[pidx(g, i, j, g.nz - 1)];
        else jzm = jz_below[(int64_t)(i + kGhost) + (int64_t)g.X * (j + kGhost)];
        const double divj = (Jx[o] - Jx[oxm]) * g.inv_dx + (Jy[o] - Jy[oym]) * g.inv_dy +
                            (Jz[o] - jzm) * g.inv_dz;
        if (have_prev) v[8] = fabs((r - rho_prev[o]) / g.dt + divj);
        rho_prev[o] = r;
    }
    // block reduction: warp shuffles, then one atomic per block and quantity
    __shared__ double red[8][9];
    const int t = threadIdx.y * blockDim.x + threadIdx.x, lane = t & 31, w = t >> 5;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        double x = v[q];
        for (int d = 16; d > 0; d >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, x, d);
            x = q < 5 ? x + y : fmax(x, y);
        }
        if (lane == 0) red[w][q] = x;
    }
    __syncthreads();
    if (t < 9) {
        double x = red[0][t];
        const int nw = (blockDim.x * blockDim.y) >> 5;
        for (int ww = 1; ww < nw; ++ww) x = t < 5 ? x + red[ww][t] : fmax(x, red[ww][t]);
        if (t < 5) atomicAdd(acc + t, x);
        else atomic_max_nonneg(acc + t, x);
    }
}

// sum over live particles of u^2 / (sqrt(1+u^2) + 1) = gamma - 1
__global__ void __launch_bounds__(256)
k_kinetic(ParticlesDev P, const int64_t *dev_n, double *__restrict__ acc)
{
    const int64_t n = *dev_n;
    double s = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        if (P.x[p] < 0.0) continue;
        const double ux = P.ux[p], uy = P.uy[p], uz = P.uz[p];
        const double u2 = ux * ux + uy * uy + uz * uz;
        s += u2 / (sqrt(1.0 + u2) + 1.0);
    }
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        atomicAdd(acc, s);
    }
}

static dim3 node_grid(const GridDev &g, dim3 bs)
{
    return dim3((g.nx + bs.x - 1) / bs.x, (g.ny + bs.y - 1) / bs.y, g.nz);
}

void launch_diag_particles(const GridDev &g, const ParticlesDev &P, const int64_t *dev_n, int64_t cap,
                           double qw, double *rho, double *acc_kinetic, cudaStream_t st)
{
    if (cap <= 0) return;
    const int bs = 256;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((cap + bs - 1) / bs, 148 * 16));
    k_rho_deposit<<<blocks, bs, 0, st>>>(g, P, dev_n, qw * g.inv_dx * g.inv_dy * g.inv_dz, rho);
    k_kinetic<<<blocks, bs, 0, st>>>(P, dev_n, acc_kinetic);
}

void launch_diag_nodes(const GridDev &g, const double *EB, const double *J, const double *jz_below,
                       double *rho, const double *rho_below, double *rho_prev, double *gauss0,
                       bool have_prev, bool have_g0, double *acc, cudaStream_t st)
{
    const dim3 bs(32, 8, 1);
    k_rho_fold<<<node_grid(g, bs), bs, 0, st>>>(g, rho, rho_below);
    k_diag_nodes<<<node_grid(g, bs), bs, 0, st>>>(g, EB, J, jz_below, rho, rho_prev, gauss0,
                                                   have_prev ? 1 : 0, have_g0 ? 1 : 0, acc);
}

}  // namespace pic
