// particle_math.cuh -- per-particle arithmetic of the PIC step (device code).
//
// Each function restates the scheme of SURVEY.md sec. 8a (rows a3-a5) and
// DESIGN.md sec. 3; the arithmetic is re-derived for the GPU (reciprocal
// square roots, local cell coordinates, a predicated <=4-segment split)
// rather than copied from the CPU oracle, with which it shares no code.
#pragma once
#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace pic {

// CIC weights along one axis for the integer-node and the half-node
// sub-grids ("standard cloud-in-cell particle form factor";
// SURVEY.md a3): g in cell units; node index i and fraction f with
// W_0 = 1 - f, W_1 = f.
struct AxisW {
    int i0, ih;        // first node of the integer / half-staggered sub-grid
    double f0, fh;     // fractions
};

__device__ __forceinline__ AxisW axis_weights(double g)
{
    AxisW a;
    const double fl = floor(g);
    a.i0 = (int)fl;
    a.f0 = g - fl;
    const double gh = g - 0.5;
    const double flh = floor(gh);
    a.ih = (int)flh;
    a.fh = gh - flh;
    return a;
}

// Trilinear interpolation of one component from a padded array:
// base points at node (i,j,k); sx = 1, sy = row stride, sz = plane stride.
__device__ __forceinline__ double trilinear(const double *__restrict__ f, int64_t base,
                                            int64_t sy, int64_t sz, double fx, double fy,
                                            double fz)
{
    const double c00 = fma(fx, f[base + 1] - f[base], f[base]);
    const double c10 = fma(fx, f[base + sy + 1] - f[base + sy], f[base + sy]);
    const double c01 = fma(fx, f[base + sz + 1] - f[base + sz], f[base + sz]);
    const double c11 = fma(fx, f[base + sy + sz + 1] - f[base + sy + sz], f[base + sy + sz]);
    const double c0 = fma(fy, c10 - c00, c00);
    const double c1 = fma(fy, c11 - c01, c01);
    return fma(fz, c1 - c0, c0);
}

// Branch-free 1/d and 1/sqrt(d) for d >= 1 (finite): hardware approximation
// (MUFU.RCP64H / MUFU.RSQ64H, ~2^-22) refined by two Newton steps to full
// fp64 accuracy (<= ~1 ulp).  Used where d = 1 + (non-negative) so no special
// cases exist; keeps the push straight-line code (no slow-path calls) so two
// particles' dependency chains interleave.
__device__ __forceinline__ double rcp_ge1(double d)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ double rsqrt_ge1(double d)
{
    // MUFU seed (relative error < 2^-22.9) and two Newton steps in residual
    // form, r' = r + r (1 - d r^2) / 2: 2^-45, then below the fp64 rounding
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d * r, r, 1.0);
    r = fma(0.5 * r, e, r);
    e = fma(-d * r, r, 1.0);
    return fma(0.5 * r, e, r);
}

// 1/d for a positive normal d (no special cases): MUFU seed + two Newton steps
__device__ __forceinline__ double rcp_pos(double d)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// Relativistic Boris rotation on u = gamma*beta (reading R1):
// u- = u + hE, t = hB/gamma(u-), u' = u- + u- x t, s = 2/(1+t^2),
// u+ = u- + s u' x t, u = u+ + hE.
__device__ __forceinline__ void boris(double h, double ex, double ey, double ez, double bx,
                                      double by, double bz, double &ux, double &uy,
                                      double &uz)
{
    const double umx = fma(h, ex, ux), umy = fma(h, ey, uy), umz = fma(h, ez, uz);
    const double ig = rsqrt_ge1(1.0 + (umx * umx + umy * umy + umz * umz));
    const double hg = h * ig;
    const double tx = hg * bx, ty = hg * by, tz = hg * bz;
    const double upx = umx + (umy * tz - umz * ty);
    const double upy = umy + (umz * tx - umx * tz);
    const double upz = umz + (umx * ty - umy * tx);
    const double s = 2.0 * rcp_ge1(1.0 + (tx * tx + ty * ty + tz * tz));
    const double ppx = umx + s * (upy * tz - upz * ty);
    const double ppy = umy + s * (upz * tx - upx * tz);
    const double ppz = umz + s * (upx * ty - upy * tx);
    ux = fma(h, ex, ppx);
    uy = fma(h, ey, ppy);
    uz = fma(h, ez, ppz);
}

// Periodic wrap, reading R7: x >= L -> x - L; x < 0 -> x + L, and a sum
// that rounds to L becomes 0.
__device__ __forceinline__ double wrap_coord(double x, double L)
{
    // almost every particle stays inside: one test, the rare wrap in a branch
    if (!(x < 0.0 || x >= L)) return x;
    if (x >= L) return x - L;
    const double lo = x + L;
    return (lo == L) ? 0.0 : lo;
}

// z after a move: periodic wrap (R7), or unchanged in an open box (NEXT-1;
// a particle that left [0, zmax) is removed by store_particle)
__device__ __forceinline__ double wrap_z(const GridDev &g, double z)
{
    return g.open_z ? z : wrap_coord(z, g.Lz);
}

// Villasenor-Buneman deposit of one straight in-cell segment
// (PAPER.md:48).  P1, P2 are local coordinates inside the
// segment's cell (components in [0,1] up to rounding); add(comp, di, dj, dk,
// value) receives the 12 edge contributions, comp 0/1/2 = Jx/Jy/Jz and
// (di,dj,dk) the node offset of the edge inside the cell.
template <class Add>
__device__ __forceinline__ void vb_segment(double p1x, double p1y, double p1z, double p2x,
                                          double p2y, double p2z, double kx, double ky,
                                          double kz, Add &&add)
{
    const double Dx = p2x - p1x, Dy = p2y - p1y, Dz = p2z - p1z;
    const double mx = 0.5 * (p1x + p2x), my = 0.5 * (p1y + p2y), mz = 0.5 * (p1z + p2z);
    const double fx = kx * Dx, fy = ky * Dy, fz = kz * Dz;
    const double cxx = Dy * Dz * (1.0 / 12.0);
    const double cyy = Dx * Dz * (1.0 / 12.0);
    const double czz = Dx * Dy * (1.0 / 12.0);
    const double nx = 1.0 - mx, ny = 1.0 - my, nz = 1.0 - mz;
    add(0, 0, 0, 0, fx * fma(ny, nz, cxx));
    add(0, 0, 1, 0, fx * fma(my, nz, -cxx));
    add(0, 0, 0, 1, fx * fma(ny, mz, -cxx));
    add(0, 0, 1, 1, fx * fma(my, mz, cxx));
    add(1, 0, 0, 0, fy * fma(nx, nz, cyy));
    add(1, 1, 0, 0, fy * fma(mx, nz, -cyy));
    add(1, 0, 0, 1, fy * fma(nx, mz, -cyy));
    add(1, 1, 0, 1, fy * fma(mx, mz, cyy));
    add(2, 0, 0, 0, fz * fma(nx, ny, czz));
    add(2, 1, 0, 0, fz * fma(mx, ny, -czz));
    add(2, 0, 1, 0, fz * fma(nx, my, -czz));
    add(2, 1, 1, 0, fz * fma(mx, my, czz));
}

// First piece of the VB split of a -> b (start-cell coordinates, a in
// [0,1)^3): the path up to the first face crossing (or all of it) ends at e.
// Returns true when more of the path remains; then (r1, r2) is the remainder
// in the coordinates of the next cell, which is offset (ox, oy, oz) from the
// start cell.  Ties between axes resolve to the lowest axis, as in
// vb_deposit.  A zero-length first piece (a on the crossed face) is e == a.
__device__ __forceinline__ bool vb_first_piece(double ax, double ay, double az, double bx,
                                               double by, double bz, double &ex, double &ey,
                                               double &ez, double r1[3], double r2[3], int &ox,
                                               int &oy, int &oz)
{
    const bool cxq = (bx < 0.0) || (bx >= 1.0);
    const bool cyq = (by < 0.0) || (by >= 1.0);
    const bool czq = (bz < 0.0) || (bz >= 1.0);
    const bool crossing = cxq | cyq | czq;
    ex = bx; ey = by; ez = bz;
    ox = oy = oz = 0;
    if (crossing) {
        const double px = bx < 0.0 ? 0.0 : 1.0, py = by < 0.0 ? 0.0 : 1.0, pz = bz < 0.0 ? 0.0 : 1.0;
        // first crossing = smallest tau_d = |p_d - a_d| / |b_d - a_d|, compared by
        // cross-multiplication (one division for the winner); ties keep the lower axis
        const double nxd = fabs(px - ax), nyd = fabs(py - ay), nzd = fabs(pz - az);
        const double dxd = fabs(bx - ax), dyd = fabs(by - ay), dzd = fabs(bz - az);
        int axis = cxq ? 0 : (cyq ? 1 : 2);
        double num = axis == 0 ? nxd : (axis == 1 ? nyd : nzd);
        double den = axis == 0 ? dxd : (axis == 1 ? dyd : dzd);
        if (cyq && axis < 1 && nyd * den < num * dyd) { axis = 1; num = nyd; den = dyd; }
        if (czq && axis < 2 && nzd * den < num * dzd) { axis = 2; num = nzd; den = dzd; }
        const double t = num * rcp_pos(den);   // den = |b_d - a_d| > 0 on a crossed axis
        ex = fma(t, bx - ax, ax);
        ey = fma(t, by - ay, ay);
        ez = fma(t, bz - az, az);
        if (axis == 0) { ex = px; ox = (bx > ax) ? 1 : -1; }
        if (axis == 1) { ey = py; oy = (by > ay) ? 1 : -1; }
        if (axis == 2) { ez = pz; oz = (bz > az) ? 1 : -1; }
        r1[0] = ex - (double)ox; r1[1] = ey - (double)oy; r1[2] = ez - (double)oz;
        r2[0] = bx - (double)ox; r2[1] = by - (double)oy; r2[2] = bz - (double)oz;
    }
    return crossing;
}

}  // namespace pic
