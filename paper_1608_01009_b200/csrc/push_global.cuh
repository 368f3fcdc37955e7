// push_global.cuh -- the per-particle path with direct HBM/L2 access:
// CIC gather from the ghost-padded E/B arrays, Boris, move, Villasenor-
// Buneman deposit with fp64 global atomics (REDG.ADD.F64), periodic wrap.
// Used by the naive kernel and as the out-of-tile fallback of the fused
// supercell kernel.
#pragma once
#include "common.cuh"
#include "particle_math.cuh"

namespace pic {

template <bool kGeneral = true>
__device__ __forceinline__ void push_one_global(const GridDev &g, const double *__restrict__ EB,
                                                double *__restrict__ J, const SpeciesDev &sp,
                                                double &x, double &y, double &z, double &ux,
                                                double &uy, double &uz, unsigned *err)
{
    const int64_t sy = g.X, sz = (int64_t)g.X * g.Y, cs = g.cs;
    const double gx = x * g.inv_dx, gy = y * g.inv_dy, gz = z * g.inv_dz - (double)g.k0;
    if (!(gx >= 0.0 && gx <= (double)g.nx && gy >= 0.0 && gy <= (double)g.ny &&
          gz >= -1.0 && gz <= (double)g.nz + 1.0)) {
        atomicOr(err, kErrRange);   // never happens for wrapped, slab-resident particles
        return;
    }
    const AxisW wx = axis_weights(gx), wy = axis_weights(gy), wz = axis_weights(gz);
    // staggering: Ex (h,0,0) Ey (0,h,0) Ez (0,0,h)
    //                                Bx (0,h,h) By (h,0,h) Bz (h,h,0)
    const double ex = trilinear(EB + 0 * cs, pidx(g, wx.ih, wy.i0, wz.i0), sy, sz, wx.fh, wy.f0, wz.f0);
    const double ey = trilinear(EB + 1 * cs, pidx(g, wx.i0, wy.ih, wz.i0), sy, sz, wx.f0, wy.fh, wz.f0);
    const double ez = trilinear(EB + 2 * cs, pidx(g, wx.i0, wy.i0, wz.ih), sy, sz, wx.f0, wy.f0, wz.fh);
    const double bx = trilinear(EB + 3 * cs, pidx(g, wx.i0, wy.ih, wz.ih), sy, sz, wx.f0, wy.fh, wz.fh);
    const double by = trilinear(EB + 4 * cs, pidx(g, wx.ih, wy.i0, wz.ih), sy, sz, wx.fh, wy.f0, wz.fh);
    const double bz = trilinear(EB + 5 * cs, pidx(g, wx.ih, wy.ih, wz.i0), sy, sz, wx.fh, wy.fh, wz.f0);
    boris(sp.h, ex, ey, ez, bx, by, bz, ux, uy, uz);
    const double ig = rsqrt(1.0 + (ux * ux + uy * uy + uz * uz));
    const double cdt = g.c * g.dt * ig;
    const double xn = fma(cdt, ux, x), yn = fma(cdt, uy, y), zn = fma(cdt, uz, z);
    // local start-cell coordinates (exact: a - floor(a))
    const double ax = wx.f0, ay = wy.f0, az = wz.f0;
    const double bxl = xn * g.inv_dx - (double)wx.i0;
    const double byl = yn * g.inv_dy - (double)wy.i0;
    const double bzl = (zn * g.inv_dz - (double)g.k0) - (double)wz.i0;
    if (!(fabs(bxl - ax) < 1.0 && fabs(byl - ay) < 1.0 && fabs(bzl - az) < 1.0)) {
        if (isfinite(xn) && isfinite(yn) && isfinite(zn))
            atomicOr(err, kErrDisplacement);
        else
            atomicOr(err, kErrNonFinite);
        return;
    }
    const double kx = sp.qw / (g.dt * g.dy * g.dz);
    const double ky = sp.qw / (g.dt * g.dx * g.dz);
    const double kz = sp.qw / (g.dt * g.dx * g.dy);
    // split at the start cell's faces piece by piece (<= 4 pieces), each
    // deposited with fp64 global atomics in its cell
    int64_t base = pidx(g, wx.i0, wy.i0, wz.i0);
    double a0 = ax, a1 = ay, a2 = az, b0 = bxl, b1 = byl, b2 = bzl;
#pragma unroll 1
    for (int it = 0; it < 4; ++it) {
        double e0, e1, e2, r1[3], r2[3];
        int ox, oy, oz;
        const bool more = vb_first_piece(a0, a1, a2, b0, b1, b2, e0, e1, e2, r1, r2, ox, oy, oz);
        vb_segment(a0, a1, a2, e0, e1, e2, kx, ky, kz, [&](int c, int di, int dj, int dk, double v) {
            atomicAdd(J + c * cs + base + di + dj * sy + dk * sz, v);
        });
        if (!more) break;
        base += ox + oy * sy + oz * sz;
        a0 = r1[0]; a1 = r1[1]; a2 = r1[2];
        b0 = r2[0]; b1 = r2[1]; b2 = r2[2];
    }
    x = wrap_coord(xn, g.Lx);
    y = wrap_coord(yn, g.Ly);
    z = kGeneral ? wrap_z(g, zn) : wrap_coord(zn, g.Lz);
}

}  // namespace pic
