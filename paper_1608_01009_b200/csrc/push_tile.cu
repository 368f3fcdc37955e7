// push_tile.cu -- the fused supercell particle kernel (SURVEY.md sec. 8a rows
// a2-a6; north_star subsystem (2)).
//
// One CTA per supercell of S^3 cells ("grouping and
// processing particles by supercells ... chosen so that particle and grid
// data processed during the particle push and current deposition stages fit"
// on-chip).  The CTA
//   1. loads the supercell's E/B tile plus a (1+H)-cell halo,
//      (S+2H+2)^3 x 6 fp64, with ONE TMA tensor copy (mbarrier-tracked) from
//      the ghost-padded fields into a bank-conflict-padded shared tile;
//   2. streams its particles -- the concatenation of the supercell's ranges
//      [sc_off[s], sc_off[s+1]) of the one or two species of the launch --
//      through per-thread cp.async (LDGSTS) staging, one particle ahead; the
//      sort stores them slot-major, so the lanes of a warp sit in distinct
//      cells;
//   3. gathers E/B from the tile, does Boris + move (straight-line code),
//      stores x, u with coalesced stores, and deposits the Villasenor-Buneman
//      currents into a deterministic fixed-point J tile with native u32
//      shared atomics; the rest of face-crossing paths is queued and
//      deposited after the particle loop;
//   4. particles that drifted more than H cells out of their supercell since
//      the last sort take the global path (L2 gather + REDG deposit);
//   5. flushes the non-zero J tile entries to the padded global J with REDG.
#include <algorithm>

#include "kernels.cuh"
#include "particle_store.cuh"
#include "push_global.cuh"
#include "tma.cuh"

namespace pic {

constexpr int kTileThreads = 256;
constexpr int kQueue = 160;     // per-supercell queue of path remainders (crossing particles)
constexpr int kFQueue = 256;    // per-supercell queue of particles outside the tile (global path)
constexpr int kCtasPerSm = 2;

// Shared-memory tile geometry.  Row/plane pitches are padded so that the 32
// lanes of a warp -- 32 consecutive cells of a 4x4x2 block of the supercell
// under the slot-major particle order -- hit distinct banks: the E/B row pitch
// is = 4 (mod 8) doubles (12 for S = 4) and the J (u32) pitches are 12 and
// = 16 (mod 32).  The E/B pitch is the TMA box width (the extra nodes of the
// box are out-of-bounds zero fill or unused).
template <int S, int H>
struct TileGeom {
    static constexpr int TE = S + 2 * H + 2;   // E/B tile extent (nodes)
    static constexpr int TJ = S + 2 * H + 3;   // J tile extent (nodes)
    static constexpr int EPX = (S == 4) ? 12 : TE;            // E/B row pitch (doubles) = TMA box dim 0
    static constexpr int EPY = EPX * TE;                       // E/B plane pitch
    static constexpr int NE = EPY * TE;                        // E/B component stride
    static constexpr int JPX = (S == 4) ? 12 : TJ;             // J row pitch (u32)
    static constexpr int JPY = (S == 4) ? 112 : JPX * TJ;      // J plane pitch
    static constexpr int NJ = JPY * TJ;                        // J component stride
    static_assert(EPX >= TE && JPX >= TJ && JPY >= JPX * TJ, "pitches");
    static_assert((EPX * 8) % 16 == 0, "TMA box row must be a multiple of 16 bytes");
    // shared-memory layout (byte offsets, 128-B aligned where TMA writes)
    static constexpr size_t off_eb = 0;                                        // [6][NE] fp64
    static constexpr size_t off_part = off_eb + 6 * NE * sizeof(double);       // [2][6][threads] fp64
    static constexpr size_t off_q = off_part + 12 * kTileThreads * sizeof(double);   // [6][kQueue] fp64
    static constexpr size_t off_jt = off_q + 6 * kQueue * sizeof(double);      // [9][NJ] u32
    static constexpr size_t off_qcell = off_jt + 9 * NJ * sizeof(unsigned);    // [kQueue] u32
    static constexpr size_t off_fq = off_qcell + (kQueue + 1) * sizeof(unsigned);   // [kFQueue + 1] u32
    static constexpr size_t off_misc = (off_fq + (kFQueue + 1) * sizeof(unsigned) + 15) / 16 * 16;
    static constexpr size_t smem_bytes = off_misc + sizeof(uint64_t);          // 1 mbarrier
};

// ---- deterministic fixed-point J tile ----------------------------------
// A contribution w (fp64) is scaled by 2^F (power of two, chosen per launch
// from the species' speed bound, see k_push_tile) and rounded to the integer
// v with one fma against 1.5*2^52 (the low 52 mantissa bits then hold
// 2^51 + v).  v is split into lo16 | mid16 | hi (signed) and added to three
// u32 tile counters with native shared-memory integer atomics (ATOMS.ADD,
// fire-and-forget) -- fp64 shared atomics are CAS loops on sm_100a.  The
// counters cannot overflow for < 2^16 contributions per edge (a supercell
// holding < 16384 particles); the sums are exact, so the tile is independent
// of the order of the atomics.  The flush rebuilds the int64 sum and converts
// back with the exact factor 2^-F.
constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52
constexpr int64_t kMaxTileParticles = 16383;

// rare path: a particle outside its tile (drifted > H cells since the sort)
template <bool kGeneral>
__device__ __forceinline__ void push_outside_tile(const GridDev &g, const double *EB, double *J,
                                                  const SpeciesDev &sp, double &x, double &y,
                                                  double &z, double &ux, double &uy, double &uz,
                                                  unsigned *err)
{
    push_one_global<kGeneral>(g, EB, J, sp, x, y, z, ux, uy, uz, err);
}

// Deposits one in-cell segment P1 -> P2 (local coordinates of the cell whose
// J-tile index is jbase) with the 12 Villasenor-Buneman edge values of
// SURVEY.md a5, each added to the fixed-point tile as computed.  A segment
// whose values could exceed the fixed-point range (a particle that sped up by
// more than the 2x headroom since the last step) goes to the fp64 global J
// instead (REDG).
template <class T>
__device__ __forceinline__ void deposit_seg(unsigned *jt, int jbase, double *J, int64_t gorigin,
                                            const GridDev &g, double p1x, double p1y, double p1z,
                                            double p2x, double p2y, double p2z, double kx,
                                            double ky, double kz, double scale, bool fits,
                                            unsigned *chk = nullptr)
{
    constexpr int PX = T::JPX, PY = T::JPY, NJ = T::NJ;
#ifdef PIC_CHECK   // the cell's 12 edges lie inside the J tile
    if (chk) {
        const int tz = jbase / PY, ty = (jbase % PY) / PX, tx = (jbase % PY) % PX;
        PIC_DCHECK(jbase >= 0 && tx + 1 < T::TJ && ty + 1 < T::TJ && tz + 1 < T::TJ, chk);
    }
#else
    (void)chk;
#endif
    const double Dx = p2x - p1x, Dy = p2y - p1y, Dz = p2z - p1z;
    const double mx = 0.5 * (p1x + p2x), my = 0.5 * (p1y + p2y), mz = 0.5 * (p1z + p2z);
    const double fx = kx * Dx, fy = ky * Dy, fz = kz * Dz;
    const double cxx = Dy * Dz * (1.0 / 12.0);
    const double cyy = Dx * Dz * (1.0 / 12.0);
    const double czz = Dx * Dy * (1.0 / 12.0);
    const double nx = 1.0 - mx, ny = 1.0 - my, nz = 1.0 - mz;
    // |value| <= |f| (1 + 1/12): weights are products of numbers in [0,1], |c| <= 1/12.
    // f scaled by 2^F (exact): one fma per value then rounds f W 2^F + 1.5*2^52.
    const double fxs = fx * scale, fys = fy * scale, fzs = fz * scale;
    if (!fits) {   // values beyond the fixed-point range (rare): fp64 global atomics
        const int rem = jbase % PY, tx = rem % PX, ty = rem / PX, tz = jbase / PY;
        const int64_t X = g.X, XY = (int64_t)g.X * g.Y, cs = g.cs;
        double *b = J + gorigin + tx + X * ty + XY * tz;
        atomicAdd(b, fx * fma(ny, nz, cxx));
        atomicAdd(b + X, fx * fma(my, nz, -cxx));
        atomicAdd(b + XY, fx * fma(ny, mz, -cxx));
        atomicAdd(b + X + XY, fx * fma(my, mz, cxx));
        atomicAdd(b + cs, fy * fma(nx, nz, cyy));
        atomicAdd(b + cs + 1, fy * fma(mx, nz, -cyy));
        atomicAdd(b + cs + XY, fy * fma(nx, mz, -cyy));
        atomicAdd(b + cs + 1 + XY, fy * fma(mx, mz, cyy));
        atomicAdd(b + 2 * cs, fz * fma(nx, ny, czz));
        atomicAdd(b + 2 * cs + 1, fz * fma(mx, ny, -czz));
        atomicAdd(b + 2 * cs + X, fz * fma(nx, my, -czz));
        atomicAdd(b + 2 * cs + 1 + X, fz * fma(mx, my, czz));
        return;
    }
    unsigned *b = jt + jbase;
    // v = round(f W 2^F): the low word of y = v + 1.5*2^52 is v mod 2^32, the
    // high word is 0x433 << 20 | (2^19 + (v >> 32))
    auto add = [&](int off, double fs, double w) {
        const long long bits = __double_as_longlong(fma(fs, w, kMagic));
        const unsigned lo = (unsigned)bits;
        const unsigned hi = (unsigned)(bits >> 32) - (0x43300000u + 0x80000u);
#ifdef PIC_EXP_NOATOMICS   // timing experiment only: drop the tile atomics
        if (lo == 0x12345u && hi == 0x777u) b[off] = 1u;
#else
        atomicAdd(b + off, lo & 0xffffu);
        atomicAdd(b + 3 * NJ + off, lo >> 16);
        atomicAdd(b + 6 * NJ + off, hi);
#endif
    };
    add(0, fxs, fma(ny, nz, cxx));
    add(PX, fxs, fma(my, nz, -cxx));
    add(PY, fxs, fma(ny, mz, -cxx));
    add(PX + PY, fxs, fma(my, mz, cxx));
    add(NJ, fys, fma(nx, nz, cyy));
    add(NJ + 1, fys, fma(mx, nz, -cyy));
    add(NJ + PY, fys, fma(nx, mz, -cyy));
    add(NJ + 1 + PY, fys, fma(mx, mz, cyy));
    add(2 * NJ, fzs, fma(nx, ny, czz));
    add(2 * NJ + 1, fzs, fma(mx, ny, -czz));
    add(2 * NJ + PX, fzs, fma(nx, my, -czz));
    add(2 * NJ + 1 + PX, fzs, fma(mx, my, czz));
}

// Do the tile values of a particle's path fit the fixed-point range?  Every
// segment of the path has |D| <= |d| per axis (d = the whole displacement in
// cell units), so |f W| <= |k d| (1 + 1/12) bounds all its values; a particle
// that sped up by more than the 2x headroom of the scale since the last step
// fails and deposits into the fp64 global J instead.
__device__ __forceinline__ bool fits_tile(double dx, double dy, double dz, double kx, double ky, double kz,
                                          double scale)
{
    return fmax(fabs(kx * dx), fmax(fabs(ky * dy), fabs(kz * dz))) * scale * (13.0 / 12.0) < 140737488355328.0;
}

// Deposits the rest of a split path (<= 2 more face crossings) starting in
// the cell with J-tile index jb; a, b in that cell's coordinates.
template <class T>
__device__ __forceinline__ void deposit_remainder(unsigned *jt, int jb, double *J, int64_t gorigin,
                                                  const GridDev &g, double a0, double a1,
                                                  double a2, double b0, double b1, double b2,
                                                  double kx, double ky, double kz, double scale, bool fits,
                                                  unsigned *chk = nullptr)
{
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
        double e0, e1, e2, r1[3], r2[3];
        int ox, oy, oz;
        const bool more = vb_first_piece(a0, a1, a2, b0, b1, b2, e0, e1, e2, r1, r2, ox, oy, oz);
        deposit_seg<T>(jt, jb, J, gorigin, g, a0, a1, a2, e0, e1, e2, kx, ky, kz, scale, fits, chk);
        if (!more) break;
        jb += ox + T::JPX * oy + T::JPY * oz;
        a0 = r1[0]; a1 = r1[1]; a2 = r1[2];
        b0 = r2[0]; b1 = r2[1]; b2 = r2[2];
    }
}

// kGeneral: slabs (nranks > 1) or an open z box (migration / absorption
// in the final store); false for the single-domain periodic box.
// One CTA pushes every species of its supercell in turn, so the E/B tile
// is loaded and the J tile zeroed and flushed once per supercell and step.
// kGeneral: slabs (nranks > 1) or an open z box (migration / absorption
// in the final store); false for the single-domain periodic box.
// NSP = 1 or 2 species per launch.  With two, the CTA walks the
// concatenation of both species' ranges of its supercell in ONE particle
// loop (the species of a particle is a select on its index), so the E/B
// tile load, the J-tile zeroing and flush and the loop's ragged last
// iteration are paid once per supercell, and the loop body is not duplicated.
template <int S, int H, bool kGeneral, int NSP>
__global__ void __launch_bounds__(kTileThreads, kCtasPerSm)
k_push_tile(const __grid_constant__ CUtensorMap eb_map, GridDev g, const double *__restrict__ EB,
            double *__restrict__ J, const __grid_constant__ TileSpecies ts, int split, unsigned *err)
{
    static_assert(NSP == 1 || NSP == 2, "one or two species per launch");
    using T = TileGeom<S, H>;
    constexpr int TJ = T::TJ, NE = T::NE, NJ = T::NJ, NT = kTileThreads;
    constexpr int EPX = T::EPX, EPY = T::EPY, JPX = T::JPX, JPY = T::JPY;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *eb = (double *)(smem_raw + T::off_eb);         // [6][TE][TE][EPX]
    double *pbuf = (double *)(smem_raw + T::off_part);     // [2 stages][6][NT]
    double *q = (double *)(smem_raw + T::off_q);           // [6][kQueue]
    unsigned *jt = (unsigned *)(smem_raw + T::off_jt);     // [3 chunks][3][TJ][JPY/..]
    unsigned *qcell = (unsigned *)(smem_raw + T::off_qcell);
    unsigned *qcount = qcell + kQueue;
    unsigned *fq = (unsigned *)(smem_raw + T::off_fq);     // particles outside the tile
    unsigned *fqcount = fq + kFQueue;
    uint64_t *bar_eb = (uint64_t *)(smem_raw + T::off_misc);
    const int tid = threadIdx.x, lane = tid & 31;
    // `split` CTAs share a supercell, each taking a contiguous part of its
    // particles (short grids fill the last wave; each CTA has its own tiles)
    // grid = (nsx * split, nsy, nsz): no integer divisions on the common path
    const int scx = split == 1 ? (int)blockIdx.x : (int)blockIdx.x / split;
    const int part = split == 1 ? 0 : (int)blockIdx.x % split;
    const int scy = blockIdx.y, scz = blockIdx.z;
    const int sc = scx + g.nsx * (scy + g.nsy * scz);
    // this CTA's particle range of species s (a part of the supercell's when split)
    auto range = [&](int s, int &a, int &b) {
        const int P0 = (int)ts.sc_off[s][sc], P1 = (int)ts.sc_off[s][sc + 1];
        a = P0;
        b = P1;
        if (split > 1) {
            a = P0 + (int)(((int64_t)(P1 - P0) * part) / split);
            b = P0 + (int)(((int64_t)(P1 - P0) * (part + 1)) / split);
        }
    };
    int a0, b0, a1 = 0, b1 = 0;
    range(0, a0, b0);
    if (NSP == 2) range(1, a1, b1);
    const int n0 = b0 - a0, total = n0 + (b1 - a1);
    if (total == 0) return;   // empty (uniform per CTA)
    // concatenated index i -> species (s1: the second one) and its array index p
    auto locate = [&](int i, bool &s1, int &p) {
        s1 = NSP == 2 && i >= n0;
        p = s1 ? a1 + (i - n0) : a0 + i;
    };

    // local-grid coordinates of the tile origin (same for the E/B and J tiles)
    const int ox = scx * S - H - 1, oy = scy * S - H - 1, oz = scz * S - H - 1;
    const int64_t gorigin = pidx(g, ox, oy, oz);   // padded global index of tile node (0,0,0)

    if (tid == 0) {
        mbar_init(bar_eb, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar_eb, 6 * NE * sizeof(double));
        tma_load_4d(eb, &eb_map, ox + kGhost, oy + kGhost, oz + kGhost, 0, bar_eb);
    }
    auto stage = [&](int i, int st) {   // this thread's particle i -> its staging slot
        bool s1;
        int p;
        locate(i, s1, p);
        const ParticlesDev &in = s1 ? ts.in[NSP - 1] : ts.in[0];
        double *d = pbuf + st * 6 * NT + tid;
        cp_async8(d + 0 * NT, in.x + p);
        cp_async8(d + 1 * NT, in.y + p);
        cp_async8(d + 2 * NT, in.z + p);
        cp_async8(d + 3 * NT, in.ux + p);
        cp_async8(d + 4 * NT, in.uy + p);
        cp_async8(d + 5 * NT, in.uz + p);
    };
    if (tid < total) stage(tid, 0);
    cp_async_commit();
    {   // zero the fixed-point J tile (16-byte stores)
        uint4 *j4 = (uint4 *)jt;
        for (int t = tid; t < (9 * NJ) / 4; t += NT) j4[t] = make_uint4(0u, 0u, 0u, 0u);
        for (int t = (9 * NJ) / 4 * 4 + tid; t < 9 * NJ; t += NT) jt[t] = 0u;
    }
    if (tid == 0) {
        *qcount = 0u;
        *fqcount = 0u;
    }

    const double cdt = g.c * g.dt;
    // fixed-point scale 2^F of this step (k_step_prep): the smaller of the
    // species' scales, so both species' contributions stay inside the range
    double scale = ts.sp[0].scale[0], inv_scale = ts.sp[0].scale[1];
    if (NSP == 2 && ts.sp[NSP - 1].scale[0] < scale) {
        scale = ts.sp[NSP - 1].scale[0];
        inv_scale = ts.sp[NSP - 1].scale[1];
    }
    double u2loc0 = 0.0, u2loc1 = 0.0;   // this thread's max |u|^2 after the push, per species
    const bool tile_ok = total <= kMaxTileParticles;   // else the counters could overflow
    __syncthreads();
    mbar_wait(bar_eb, 0);

    int st = 0;
    for (int i = tid; i < total; i += NT) {
        if (i + NT < total) stage(i + NT, st ^ 1);   // prefetch the next particle
        cp_async_commit();
        cp_async_wait1();
        bool s1;
        int p;
        locate(i, s1, p);
        const double *pl = pbuf + st * 6 * NT + tid;
        st ^= 1;
        const double x = pl[0], y = pl[NT], z = pl[2 * NT];
        // dead slot (migrated away or absorbed since the last sort; a single
        // periodic box has none)
        if (kGeneral && x < 0.0) continue;
        double ux = pl[3 * NT], uy = pl[4 * NT], uz = pl[5 * NT];
        const double gx = x * g.inv_dx, gy = y * g.inv_dy, gz = z * g.inv_dz - (double)g.k0;
        const AxisW wx = axis_weights(gx), wy = axis_weights(gy), wz = axis_weights(gz);
        // tile-relative start cell; inside the tile when in [1, S + 2H] on every axis
        const int tx = wx.i0 - ox, ty = wy.i0 - oy, tz = wz.i0 - oz;
        const bool inside = tile_ok && (unsigned)(tx - 1) < (unsigned)(S + 2 * H) &&
                            (unsigned)(ty - 1) < (unsigned)(S + 2 * H) &&
                            (unsigned)(tz - 1) < (unsigned)(S + 2 * H);
        if (inside) {
#ifdef PIC_EXP_NOGATHER   // timing experiment only: same node for every lane
            const int hx = 2, hy = 2, hz = 2;
#define tx 2
#define ty 2
#define tz 2
#else
            const int hx = wx.ih - ox, hy = wy.ih - oy, hz = wz.ih - oz;
#endif
            // the 8 corners of every component lie inside the E/B tile
            PIC_DCHECK(hx >= 0 && hy >= 0 && hz >= 0 && tx >= 0 && ty >= 0 && tz >= 0 && hx + 1 < T::TE &&
                           hy + 1 < T::TE && hz + 1 < T::TE && tx + 1 < T::TE && ty + 1 < T::TE && tz + 1 < T::TE,
                       err);
#ifndef PIC_EXP_NOPUSH   // timing experiment only: no gather, no Boris
            const double ex = trilinear(eb + 0 * NE, hx + EPX * ty + EPY * tz, EPX, EPY, wx.fh, wy.f0, wz.f0);
            const double ey = trilinear(eb + 1 * NE, tx + EPX * hy + EPY * tz, EPX, EPY, wx.f0, wy.fh, wz.f0);
            const double ez = trilinear(eb + 2 * NE, tx + EPX * ty + EPY * hz, EPX, EPY, wx.f0, wy.f0, wz.fh);
            const double bx = trilinear(eb + 3 * NE, tx + EPX * hy + EPY * hz, EPX, EPY, wx.f0, wy.fh, wz.fh);
            const double by = trilinear(eb + 4 * NE, hx + EPX * ty + EPY * hz, EPX, EPY, wx.fh, wy.f0, wz.fh);
            const double bz = trilinear(eb + 5 * NE, hx + EPX * hy + EPY * tz, EPX, EPY, wx.fh, wy.fh, wz.f0);
#ifdef PIC_EXP_NOGATHER
#undef tx
#undef ty
#undef tz
#endif
            boris(s1 ? ts.sp[NSP - 1].h : ts.sp[0].h, ex, ey, ez, bx, by, bz, ux, uy, uz);
#else
            (void)hx; (void)hy; (void)hz;
#endif
            const double u2 = ux * ux + uy * uy + uz * uz;
            const double ig = rsqrt_ge1(1.0 + u2);
            const double xn = fma(cdt * ig, ux, x), yn = fma(cdt * ig, uy, y), zn = fma(cdt * ig, uz, z);
            // move endpoints in start-cell coordinates (a = fractional parts, exact)
            const double bxl = xn * g.inv_dx - (double)wx.i0;
            const double byl = yn * g.inv_dy - (double)wy.i0;
            const double bzl = (zn * g.inv_dz - (double)g.k0) - (double)wz.i0;
            const double dxl = bxl - wx.f0, dyl = byl - wy.f0, dzl = bzl - wz.f0;
            const bool ok = fabs(dxl) < 1.0 && fabs(dyl) < 1.0 && fabs(dzl) < 1.0;
            if (s1) u2loc1 = fmax(u2loc1, u2); else u2loc0 = fmax(u2loc0, u2);
            const ParticlesDev &in = s1 ? ts.in[NSP - 1] : ts.in[0];
            const ParticlesDev &out = s1 ? ts.out[NSP - 1] : ts.out[0];
            const SpeciesDev &sp = s1 ? ts.sp[NSP - 1] : ts.sp[0];
            if (ok)
                store_particle<kGeneral>(g, sp, out, in.id, p, wrap_coord(xn, g.Lx), wrap_coord(yn, g.Ly),
                                         kGeneral ? wrap_z(g, zn) : wrap_coord(zn, g.Lz), ux, uy, uz, false, err);
            else
                store_particle<kGeneral>(g, sp, out, in.id, p, x, y, z, ux, uy, uz, false, err);
            if (ok) {
#ifndef PIC_EXP_NODEP   // timing experiment only: no deposit
                const double kx = sp.kx, ky = sp.ky, kz = sp.kz;   // q w / (dt dA), host
                const int jbase = tx + JPX * ty + JPY * tz;
                double ex_, ey_, ez_, r1[3], r2[3];
                int cx, cy, cz;
                const bool more =
                    vb_first_piece(wx.f0, wy.f0, wz.f0, bxl, byl, bzl, ex_, ey_, ez_, r1, r2, cx, cy, cz);
                const bool fits = fits_tile(dxl, dyl, dzl, kx, ky, kz, scale);
                deposit_seg<T>(jt, jbase, J, gorigin, g, wx.f0, wy.f0, wz.f0, ex_, ey_, ez_, kx, ky, kz, scale,
                               fits, err);
                if (more) {
                    // the rest of a face-crossing path is deposited after the particle
                    // loop, all queued paths together (keeps the loop convergent); the
                    // species is the top bit of the queued cell
                    const int jrem = jbase + cx + JPX * cy + JPY * cz;
                    // only fitting paths are queued (the drain deposits into the tile)
                    // one shared atomic per warp for the lanes that queue (the lanes
                    // that reach this point together)
                    const unsigned act = __activemask();
                    const unsigned want = __ballot_sync(act, fits);
                    unsigned slot = (unsigned)kQueue;
                    if (want) {
                        const int leader = __ffs(want) - 1;
                        unsigned qb = 0;
                        if (lane == leader) qb = atomicAdd(qcount, (unsigned)__popc(want));
                        qb = __shfl_sync(act, qb, leader);
                        if (fits) slot = qb + (unsigned)__popc(want & ((1u << lane) - 1u));
                    }
                    if (slot < (unsigned)kQueue) {
                        q[0 * kQueue + slot] = r1[0]; q[1 * kQueue + slot] = r1[1]; q[2 * kQueue + slot] = r1[2];
                        q[3 * kQueue + slot] = r2[0]; q[4 * kQueue + slot] = r2[1]; q[5 * kQueue + slot] = r2[2];
                        qcell[slot] = (unsigned)jrem | (s1 ? 0x80000000u : 0u);
                    } else {
                        deposit_remainder<T>(jt, jrem, J, gorigin, g, r1[0], r1[1], r1[2], r2[0], r2[1],
                                             r2[2], kx, ky, kz, scale, fits, err);
                    }
                }
#endif
            } else {
                atomicOr(err, (isfinite(xn) && isfinite(yn) && isfinite(zn)) ? kErrDisplacement
                                                                              : kErrNonFinite);
            }
        } else {
            // outside the tile (drifted > H cells since the sort): deferred to after
            // the loop so the slow global path does not stall this warp's iteration
            const unsigned slot = atomicAdd(fqcount, 1u);
            if (slot < (unsigned)kFQueue) {
                fq[slot] = (unsigned)i;
            } else {
                const ParticlesDev &in = s1 ? ts.in[NSP - 1] : ts.in[0];
                const ParticlesDev &out = s1 ? ts.out[NSP - 1] : ts.out[0];
                const SpeciesDev &sp = s1 ? ts.sp[NSP - 1] : ts.sp[0];
                double xx = x, yy = y, zz = z;
                push_outside_tile<kGeneral>(g, EB, J, sp, xx, yy, zz, ux, uy, uz, err);
                store_particle<kGeneral>(g, sp, out, in.id, p, xx, yy, zz, ux, uy, uz, false, err);
                const double v2 = ux * ux + uy * uy + uz * uz;
                if (s1) u2loc1 = fmax(u2loc1, v2); else u2loc0 = fmax(u2loc0, v2);
            }
        }
    }
    __syncthreads();   // all particles pushed, the queues are complete
    const int nq = min(*qcount, (unsigned)kQueue);
    for (int e = tid; e < nq; e += NT) {
        const unsigned qc = qcell[e];
        const SpeciesDev &sp = (qc >> 31) ? ts.sp[NSP - 1] : ts.sp[0];
        deposit_remainder<T>(jt, (int)(qc & 0x7fffffffu), J, gorigin, g, q[e], q[kQueue + e], q[2 * kQueue + e],
                             q[3 * kQueue + e], q[4 * kQueue + e], q[5 * kQueue + e], sp.kx, sp.ky, sp.kz, scale,
                             true, err);
    }
    const int nf = min(*fqcount, (unsigned)kFQueue);
    for (int e = tid; e < nf; e += NT) {
        bool s1;
        int p;
        locate((int)fq[e], s1, p);
        const ParticlesDev &in = s1 ? ts.in[NSP - 1] : ts.in[0];
        const ParticlesDev &out = s1 ? ts.out[NSP - 1] : ts.out[0];
        const SpeciesDev &sp = s1 ? ts.sp[NSP - 1] : ts.sp[0];
        double xx = in.x[p], yy = in.y[p], zz = in.z[p], ux = in.ux[p], uy = in.uy[p], uz = in.uz[p];
        push_outside_tile<kGeneral>(g, EB, J, sp, xx, yy, zz, ux, uy, uz, err);
        store_particle<kGeneral>(g, sp, out, in.id, p, xx, yy, zz, ux, uy, uz, false, err);
        const double v2 = ux * ux + uy * uy + uz * uz;
        if (s1) u2loc1 = fmax(u2loc1, v2); else u2loc0 = fmax(u2loc0, v2);
    }
    {
        const unsigned hi0 = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(u2loc0) >> 32));
        if (lane == 0 && hi0) atomicMax(ts.sp[0].u2max_out, hi0);
        if (NSP == 2) {
            const unsigned hi1 = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(u2loc1) >> 32));
            if (lane == 0 && hi1) atomicMax(ts.sp[NSP - 1].u2max_out, hi1);
        }
    }
    __syncthreads();
    // flush the fixed-point tile to the fp64 global J.  Lanes run along x (a
    // warp covers 3 rows of TJ consecutive nodes, lanes 3 TJ.. idle): the tile
    // reads hit consecutive banks and the REDGs of a row are coalesced.
    const int64_t cs = g.cs, gsy = g.X, gsz = (int64_t)g.X * g.Y;
    constexpr int kRowsPerWarp = 32 / TJ;
    const int wid = tid >> 5, a = lane % TJ, rsub = lane / TJ;
    // a warp takes whole (component, z) planes of the tile, kRowsPerWarp rows
    // at a time, with the plane's base addresses computed once
    if (rsub < kRowsPerWarp) {
        for (int pl = wid; pl < 3 * TJ; pl += NT / 32) {
            const int comp = (pl >= TJ) + (pl >= 2 * TJ), c = pl - comp * TJ;
            const unsigned *jn = jt + comp * NJ + c * JPY + a + rsub * JPX;
            double *gp = J + comp * cs + gorigin + gsz * c + a + gsy * rsub;
#pragma unroll
            for (int r = 0; r < (TJ + kRowsPerWarp - 1) / kRowsPerWarp; ++r) {
                if (TJ % kRowsPerWarp != 0 && rsub + r * kRowsPerWarp >= TJ) break;
                const int o = r * kRowsPerWarp * JPX;
                const long long fx = (long long)(int)jn[6 * NJ + o] * 4294967296LL +
                                     (long long)jn[3 * NJ + o] * 65536LL + (long long)jn[o];
                if (fx != 0) atomicAdd(gp + gsy * (r * kRowsPerWarp), (double)fx * inv_scale);
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_u2max(ParticlesDev P, int64_t n, unsigned *out)
{
    double m = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, P.ux[p] * P.ux[p] + P.uy[p] * P.uy[p] + P.uz[p] * P.uz[p]);
    const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(m) >> 32));
    if ((threadIdx.x & 31) == 0 && hi) atomicMax(out, hi);
}

// Before the particle kernels of a step: the fixed-point scale of each
// species' J tile from the previous step's speed bound, and the reset of this
// step's bound (step_prep_species).  A stand-alone launch only before the
// first step after new particles; every step's k_e_full prepares the next.
__global__ void k_step_prep(StepPrep p)
{
    if ((int)threadIdx.x < p.n_species) step_prep_species(p, threadIdx.x);
}

void launch_step_prep(const StepPrep &p, cudaStream_t st)
{
    k_step_prep<<<1, 32, 0, st>>>(p);
}

void launch_u2max(const ParticlesDev &P, int64_t n, unsigned *out, cudaStream_t st)
{
    cudaMemsetAsync(out, 0, sizeof(unsigned), st);
    if (n > 0) k_u2max<<<296, 256, 0, st>>>(P, n, out);
}

template <int S, int H, bool kGeneral>
static void launch_tile(const CUtensorMap &map, const GridDev &g, const double *EB, double *J,
                        const TileSpecies &ts, unsigned *err, int64_t mean_per_sc, cudaStream_t st)
{
    const size_t smem = TileGeom<S, H>::smem_bytes;
    // one CTA per supercell (empty ones exit at once); only very dense
    // supercells (> 8192 particles expected) are split over several CTAs --
    // splitting C2's 3200-particle supercells was measured slower (extra tile
    // loads and flushes outweigh the shorter last wave)
#ifndef PIC_SPLIT_AT
#define PIC_SPLIT_AT 8192
#endif
    const int split = (int)std::max<int64_t>(1, std::min<int64_t>(16, (mean_per_sc + PIC_SPLIT_AT - 1) / PIC_SPLIT_AT));
    const dim3 grid((unsigned)(g.nsx * split), (unsigned)g.nsy, (unsigned)g.nsz);
    if (ts.n == 1)
        k_push_tile<S, H, kGeneral, 1><<<grid, kTileThreads, smem, st>>>(map, g, EB, J, ts, split, err);
    else
        k_push_tile<S, H, kGeneral, 2><<<grid, kTileThreads, smem, st>>>(map, g, EB, J, ts, split, err);
}

bool tile_supported(int S) { return S == 2 || S == 4; }

void tile_box(int S, int box[4])
{
    const int te = S + 2 * 1 + 2;
    box[0] = (S == 4) ? TileGeom<4, 1>::EPX : TileGeom<2, 1>::EPX;
    box[1] = te;
    box[2] = te;
    box[3] = 6;
}

template <int S, bool G>
static void set_smem()
{
    const int b = (int)TileGeom<S, 1>::smem_bytes;
    cudaFuncSetAttribute(k_push_tile<S, 1, G, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(k_push_tile<S, 1, G, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

void configure_tile_kernels()
{
    set_smem<4, false>();
    set_smem<4, true>();
    set_smem<2, false>();
    set_smem<2, true>();
}

void launch_push_tile(const CUtensorMap &map, const GridDev &g, const double *EB, double *J,
                      const TileSpecies &ts, unsigned *err, int64_t mean_per_sc, cudaStream_t st)
{
    if (ts.n == 0) return;
    const bool general = g.nranks > 1 || g.open_z;
    if (g.S == 4 && general)
        launch_tile<4, 1, true>(map, g, EB, J, ts, err, mean_per_sc, st);
    else if (g.S == 4)
        launch_tile<4, 1, false>(map, g, EB, J, ts, err, mean_per_sc, st);
    else if (g.S == 2 && general)
        launch_tile<2, 1, true>(map, g, EB, J, ts, err, mean_per_sc, st);
    else if (g.S == 2)
        launch_tile<2, 1, false>(map, g, EB, J, ts, err, mean_per_sc, st);
}

}  // namespace pic
