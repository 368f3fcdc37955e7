// push_tile.cu -- the fused supercell particle kernel (SURVEY.md sec. 8a rows
// a2-a6; north_star subsystem (2)).
//
// One CTA per supercell of S^3 cells ("grouping and
// processing particles by supercells ... chosen so that particle and grid
// data processed during the particle push and current deposition stages fit"
// on-chip).  The CTA
//   1. stages the supercell's E/B tile plus a (1+H)-cell halo,
//      (S+2H+2)^3 x 6 fp64, from the ghost-padded fields into shared memory,
//      and zeroes a (S+2H+3)^3 x 3 fp64 J tile;
//   2. streams its particles [sc_off[s], sc_off[s+1]) with coalesced loads
//      (the sort stores them slot-major, so the lanes of a warp sit in
//      distinct cells), gathers E/B from the tile, does Boris + move, and
//      deposits Villasenor-Buneman currents into the J tile with shared-memory
//      fp64 atomics (conflict-free across lanes in distinct cells);
//   3. particles that drifted more than H cells out of their supercell since
//      the last sort take the global path (L2 gather + REDG deposit);
//   4. flushes the non-zero J tile entries to the padded global J with REDG.
#include "kernels.cuh"
#include "push_global.cuh"

namespace pic {

template <int S, int H>
struct TileGeom {
    static constexpr int TE = S + 2 * H + 2;   // E/B tile extent (nodes)
    static constexpr int TJ = S + 2 * H + 3;   // J tile extent (nodes)
    static constexpr int NE = TE * TE * TE;
    static constexpr int NJ = TJ * TJ * TJ;
    static constexpr size_t smem_bytes = sizeof(double) * (6 * NE + 3 * NJ);
};

constexpr int kTileThreads = 256;

template <int S, int H>
__global__ void __launch_bounds__(kTileThreads, 2)
k_push_tile(GridDev g, const double *__restrict__ EB, double *__restrict__ J, ParticlesDev in,
            ParticlesDev out, const int64_t *__restrict__ sc_off, SpeciesDev sp, int copy_id,
            unsigned *err)
{
    using T = TileGeom<S, H>;
    constexpr int TE = T::TE, TJ = T::TJ, NE = T::NE, NJ = T::NJ;
    extern __shared__ double smem[];
    double *eb = smem;            // [6][TE][TE][TE]
    double *jt = smem + 6 * NE;   // [3][TJ][TJ][TJ]

    const int sc = blockIdx.x;
    const int scx = sc % g.nsx, scy = (sc / g.nsx) % g.nsy, scz = sc / (g.nsx * g.nsy);
    // local-grid coordinates of the tile origin (same for the E/B and J tiles)
    const int ox = scx * S - H - 1, oy = scy * S - H - 1, oz = scz * S - H - 1;
    const int64_t cs = g.cs;

    for (int t = threadIdx.x; t < 6 * NE; t += kTileThreads) {
        const int comp = t / NE, r = t - comp * NE;
        const int a = r % TE, b = (r / TE) % TE, c = r / (TE * TE);
        eb[t] = EB[comp * cs + pidx(g, ox + a, oy + b, oz + c)];
    }
    for (int t = threadIdx.x; t < 3 * NJ; t += kTileThreads) jt[t] = 0.0;
    __syncthreads();

    const double kx = sp.qw / (g.dt * g.dy * g.dz);
    const double ky = sp.qw / (g.dt * g.dx * g.dz);
    const double kz = sp.qw / (g.dt * g.dx * g.dy);
    const double cdt = g.c * g.dt;
    const int64_t p0 = sc_off[sc], p1 = sc_off[sc + 1];
    for (int64_t p = p0 + threadIdx.x; p < p1; p += kTileThreads) {
        double x = in.x[p], y = in.y[p], z = in.z[p];
        double ux = in.ux[p], uy = in.uy[p], uz = in.uz[p];
        const double gx = x * g.inv_dx, gy = y * g.inv_dy, gz = z * g.inv_dz - (double)g.k0;
        const AxisW wx = axis_weights(gx), wy = axis_weights(gy), wz = axis_weights(gz);
        // tile-relative start cell; inside the tile when in [1, S + 2H] on every axis
        const int tx = wx.i0 - ox, ty = wy.i0 - oy, tz = wz.i0 - oz;
        const bool inside = (unsigned)(tx - 1) < (unsigned)(S + 2 * H) &&
                            (unsigned)(ty - 1) < (unsigned)(S + 2 * H) &&
                            (unsigned)(tz - 1) < (unsigned)(S + 2 * H);
        if (inside) {
            const int hx = wx.ih - ox, hy = wy.ih - oy, hz = wz.ih - oz;
            constexpr int sy = TE, sz = TE * TE;
            const double ex = trilinear(eb + 0 * NE, hx + sy * ty + sz * tz, sy, sz, wx.fh, wy.f0, wz.f0);
            const double ey = trilinear(eb + 1 * NE, tx + sy * hy + sz * tz, sy, sz, wx.f0, wy.fh, wz.f0);
            const double ez = trilinear(eb + 2 * NE, tx + sy * ty + sz * hz, sy, sz, wx.f0, wy.f0, wz.fh);
            const double bx = trilinear(eb + 3 * NE, tx + sy * hy + sz * hz, sy, sz, wx.f0, wy.fh, wz.fh);
            const double by = trilinear(eb + 4 * NE, hx + sy * ty + sz * hz, sy, sz, wx.fh, wy.f0, wz.fh);
            const double bz = trilinear(eb + 5 * NE, hx + sy * hy + sz * tz, sy, sz, wx.fh, wy.fh, wz.f0);
            boris(sp.h, ex, ey, ez, bx, by, bz, ux, uy, uz);
            const double ig = rsqrt(1.0 + (ux * ux + uy * uy + uz * uz));
            const double xn = fma(cdt * ig, ux, x), yn = fma(cdt * ig, uy, y), zn = fma(cdt * ig, uz, z);
            const double bxl = xn * g.inv_dx - (double)wx.i0;
            const double byl = yn * g.inv_dy - (double)wy.i0;
            const double bzl = (zn * g.inv_dz - (double)g.k0) - (double)wz.i0;
            if (fabs(bxl - wx.f0) < 1.0 && fabs(byl - wy.f0) < 1.0 && fabs(bzl - wz.f0) < 1.0) {
                const int jbase = tx + TJ * (ty + TJ * tz);
                vb_deposit(wx.f0, wy.f0, wz.f0, bxl, byl, bzl, kx, ky, kz,
                           [&](int c, int di, int dj, int dk, double v) {
                               atomicAdd(jt + c * NJ + jbase + di + TJ * (dj + TJ * dk), v);
                           });
                x = wrap_coord(xn, g.Lx);
                y = wrap_coord(yn, g.Ly);
                z = wrap_coord(zn, g.Lz);
            } else {
                atomicOr(err, (isfinite(xn) && isfinite(yn) && isfinite(zn)) ? kErrDisplacement
                                                                              : kErrNonFinite);
            }
        } else {
            push_one_global(g, EB, J, sp, x, y, z, ux, uy, uz, err);
        }
        out.x[p] = x; out.y[p] = y; out.z[p] = z;
        out.ux[p] = ux; out.uy[p] = uy; out.uz[p] = uz;
        if (copy_id) out.id[p] = in.id[p];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * NJ; t += kTileThreads) {
        const double v = jt[t];
        if (v != 0.0) {
            const int comp = t / NJ, r = t - comp * NJ;
            const int a = r % TJ, b = (r / TJ) % TJ, c = r / (TJ * TJ);
            atomicAdd(J + comp * cs + pidx(g, ox + a, oy + b, oz + c), v);
        }
    }
}

template <int S, int H>
static void launch_tile(const GridDev &g, const double *EB, double *J, const ParticlesDev &in,
                        const ParticlesDev &out, const int64_t *sc_off, const SpeciesDev &sp,
                        bool copy_id, unsigned *err, cudaStream_t st)
{
    const size_t smem = TileGeom<S, H>::smem_bytes;
    const unsigned nsc = (unsigned)g.nsx * g.nsy * g.nsz;
    k_push_tile<S, H><<<nsc, kTileThreads, smem, st>>>(g, EB, J, in, out, sc_off, sp, copy_id ? 1 : 0, err);
}

bool tile_supported(int S) { return S == 2 || S == 4; }

void configure_tile_kernels()
{
    cudaFuncSetAttribute(k_push_tile<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TileGeom<4, 1>::smem_bytes);
    cudaFuncSetAttribute(k_push_tile<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)TileGeom<2, 1>::smem_bytes);
}

void launch_push_tile(const GridDev &g, const double *EB, double *J, const ParticlesDev &in,
                      const ParticlesDev &out, const int64_t *sc_off, const SpeciesDev &sp,
                      bool copy_id, unsigned *err, cudaStream_t st)
{
    if (g.S == 4)
        launch_tile<4, 1>(g, EB, J, in, out, sc_off, sp, copy_id, err, st);
    else if (g.S == 2)
        launch_tile<2, 1>(g, EB, J, in, out, sc_off, sp, copy_id, err, st);
}

}  // namespace pic
