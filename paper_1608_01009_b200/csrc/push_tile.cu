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
//      through shared memory, each warp's 32 with one 2-D TMA tensor load
//      two iterations ahead (per-warp stages and mbarriers); the sort stores
//      them slot-major, so the lanes of a warp sit in distinct cells;
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

constexpr int kQueue = 160;     // per-supercell queue of path remainders (crossing particles)
constexpr int kFQueue = 256;    // per-supercell queue of particles outside the tile (global path)

constexpr int up_mod(int v, int m, int r) { return v + (((r - v % m) % m) + m) % m; }   // >= v, = r (mod m)

// Shared-memory tile geometry of supercell edge S and drift halo H.  Row and
// plane pitches are padded so that the 32 lanes of a warp -- 32 consecutive
// cells of a 4x4x2 block of the supercell under the slot-major particle
// order -- spread over the banks: the E/B row pitch is = 4 (mod 8) doubles
// (12 for S = 4) and the J (u32) pitches are = 4 (mod 8) and = 16 (mod 32).
// The E/B pitch is the TMA box width (the extra nodes of the box are
// out-of-bounds zero fill or unused).  Threads per CTA and CTAs per SM follow
// from the shared memory: two CTAs of 256 threads when the tiles fit twice,
// else one CTA of 512 (the same 16 warps per SM, 128 registers).
template <int S, int H>
struct TileGeom {
    static constexpr int TE = S + 2 * H + 2;   // E/B tile extent (nodes)
    static constexpr int TJ = S + 2 * H + 3;   // J tile extent (nodes)
    // the TMA box must start on a 16-byte boundary in x: when the tile origin
    // -H-1 (+ the kGhost padding) is odd, the box starts one node lower and
    // the tile is read from eb + XSH
    static constexpr int XSH = (kGhost - H - 1) & 1;
    static constexpr int EPX = (S >= 4) ? up_mod(TE + XSH, 8, 4) : (TE + XSH + 1) / 2 * 2;   // row pitch = TMA box dim 0
    static constexpr int EPY = EPX * TE;                                  // E/B plane pitch
    static constexpr int NE = EPY * TE;                                   // E/B component stride
    static constexpr int JPX = (S >= 4) ? up_mod(TJ, 8, 4) : TJ;          // J row pitch (u32)
    static constexpr int JPY = (S >= 4) ? up_mod(JPX * TJ, 32, 16) : JPX * TJ;   // J plane pitch
    static constexpr int NJ = JPY * TJ;                                   // J component stride
    static_assert(EPX >= TE + XSH && JPX >= TJ && JPY >= JPX * TJ, "pitches");
    static_assert((EPX * 8) % 16 == 0, "TMA box row must be a multiple of 16 bytes");
    static constexpr size_t tiles = 6 * NE * sizeof(double) + 9 * NJ * sizeof(unsigned);
    static constexpr int CTAS = tiles + 6 * kQueue * sizeof(double) + 12 * 288 * sizeof(double) < 110 * 1024 ? 2 : 1;
    static constexpr int NT = CTAS == 2 ? 256 : 512;   // threads per CTA
    static constexpr int NW = NT / 32;                 // warps per CTA
    static constexpr int PW = kPartBox;                // a warp's staged chunk: [6][PW] fp64 (one TMA box)
    // fp64 per stage: the [6][PW] box, then the stage's mbarrier, 128-byte aligned stages
    static constexpr int PSTAGE = (6 * PW * 8 + 8 + 127) / 128 * 16;
    static constexpr int PBAR = 6 * PW * 8;   // byte offset of a stage's mbarrier
    // shared-memory layout (byte offsets, 128-B aligned where TMA writes)
    static constexpr size_t off_eb = 0;                                        // [6][NE] fp64
    static constexpr size_t off_part = off_eb + 6 * NE * sizeof(double);       // [NW][2][PSTAGE] fp64
    static constexpr size_t off_q = off_part + NW * 2 * PSTAGE * sizeof(double);   // [6][kQueue] fp64
    static constexpr size_t off_jt = off_q + 6 * kQueue * sizeof(double);      // [9][NJ] u32
    static constexpr size_t off_qcell = off_jt + 9 * NJ * sizeof(unsigned);    // [kQueue] u32
    static constexpr size_t off_fq = off_qcell + (kQueue + 1) * sizeof(unsigned);   // [kFQueue + 1] u32
    static constexpr size_t off_misc = (off_fq + (kFQueue + 1) * sizeof(unsigned) + 15) / 16 * 16;
    static constexpr size_t smem_bytes = off_misc + sizeof(uint64_t);         // the E/B tile's mbarrier
    static_assert(smem_bytes <= 227 * 1024, "tiles exceed shared memory");
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
constexpr double kFixRange = 140737488355328.0;  // 2^47: |v| of one accumulated value (see fixed_add)
// tile counters stay exact for < 2^16 contributions per edge of |v| < 2^47
// (a particle adds to an edge at most 4 times), with a margin for the
// floor of the accumulated flushes' high words
constexpr int64_t kMaxTileParticles = 16000;

// The 12 Villasenor-Buneman edge values of one in-cell segment P1 -> P2
// (local coordinates of the segment's cell), times the flux
// factors k and the fixed-point scale 2^F (exact: a power of two), in the
// order Jx (0,0,0) (0,1,0) (0,0,1) (0,1,1), Jy (0,0,0) (1,0,0) (0,0,1)
// (1,0,1), Jz (0,0,0) (1,0,0) (0,1,0) (1,1,0) of the cell's edges.
struct EdgeVals {
    double v[12];
};

__device__ __forceinline__ EdgeVals seg_values(double p1x, double p1y, double p1z, double p2x, double p2y,
                                               double p2z, double kxs, double kys, double kzs)
{
    const double Dx = p2x - p1x, Dy = p2y - p1y, Dz = p2z - p1z;
    const double mx = 0.5 * (p1x + p2x), my = 0.5 * (p1y + p2y), mz = 0.5 * (p1z + p2z);
    const double fx = kxs * Dx, fy = kys * Dy, fz = kzs * Dz;
    const double cxx = Dy * Dz * (1.0 / 12.0);
    const double cyy = Dx * Dz * (1.0 / 12.0);
    const double czz = Dx * Dy * (1.0 / 12.0);
    const double nx = 1.0 - mx, ny = 1.0 - my, nz = 1.0 - mz;
    EdgeVals e;
    e.v[0] = fx * fma(ny, nz, cxx);
    e.v[1] = fx * fma(my, nz, -cxx);
    e.v[2] = fx * fma(ny, mz, -cxx);
    e.v[3] = fx * fma(my, mz, cxx);
    e.v[4] = fy * fma(nx, nz, cyy);
    e.v[5] = fy * fma(mx, nz, -cyy);
    e.v[6] = fy * fma(nx, mz, -cyy);
    e.v[7] = fy * fma(mx, mz, cyy);
    e.v[8] = fz * fma(nx, ny, czz);
    e.v[9] = fz * fma(mx, ny, -czz);
    e.v[10] = fz * fma(nx, my, -czz);
    e.v[11] = fz * fma(mx, my, czz);
    return e;
}

// J-tile offsets of the 12 edges of a cell (order of seg_values)
template <class T>
__device__ __forceinline__ constexpr int edge_off(int e)
{
    constexpr int PX = T::JPX, PY = T::JPY, NJ = T::NJ;
    constexpr int off[12] = {0,      PX,         PY,          PX + PY,          NJ,              NJ + 1,
                             NJ + PY, NJ + 1 + PY, 2 * NJ,     2 * NJ + 1,       2 * NJ + PX,     2 * NJ + 1 + PX};
    return off[e];
}

// Adds one scaled value w 2^F to the fixed-point tile entry b: v =
// round(w 2^F) from one fma against 1.5*2^52 (the low word of the result is
// v mod 2^32, the high word 0x4338 << 16 + (v >> 32) for |v| < 2^51), split
// into lo16 | mid16 | hi (signed) over three u32 counters.
template <class T>
__device__ __forceinline__ void fixed_add(unsigned *b, double vs)
{
    constexpr int NJ = T::NJ;
    const long long bits = __double_as_longlong(vs + kMagic);
    const unsigned lo = (unsigned)bits;
    const unsigned hi = (unsigned)(bits >> 32) - (0x43300000u + 0x80000u);
    atomicAdd(b, lo & 0xffffu);
    atomicAdd(b + 3 * NJ, lo >> 16);
    atomicAdd(b + 6 * NJ, hi);
}

template <class T>
__device__ __forceinline__ void tile_add(unsigned *jt, int jbase, const EdgeVals &e)
{
#pragma unroll
    for (int k = 0; k < 12; ++k) fixed_add<T>(jt + jbase + edge_off<T>(k), e.v[k]);
}

// The fp64 global fallback of one segment (values beyond the fixed-point
// range, rare): REDG.F64 of the unscaled values into the padded J.
template <class T>
__device__ __forceinline__ void global_add(double *J, int64_t gorigin, const GridDev &g, int jbase,
                                           const EdgeVals &e, double inv_scale)
{
    const int rem = jbase % T::JPY, tx = rem % T::JPX, ty = rem / T::JPX, tz = jbase / T::JPY;
    const int64_t X = g.X, XY = (int64_t)g.X * g.Y, cs = g.cs;
    double *b = J + gorigin + tx + X * ty + XY * tz;
    const int64_t off[12] = {0, X, XY, X + XY, cs, cs + 1, cs + XY, cs + 1 + XY,
                             2 * cs, 2 * cs + 1, 2 * cs + X, 2 * cs + 1 + X};
#pragma unroll
    for (int k = 0; k < 12; ++k) atomicAdd(b + off[k], e.v[k] * inv_scale);
}

// Deposits one in-cell segment P1 -> P2 (local coordinates of the cell whose
// J-tile index is jbase) into the fixed-point tile, or -- a segment whose
// values could exceed the fixed-point range (a particle that sped up by more
// than the 2x headroom since the last step) -- into the fp64 global J.
template <class T>
__device__ __forceinline__ void deposit_seg(unsigned *jt, int jbase, double *J, int64_t gorigin,
                                            const GridDev &g, double p1x, double p1y, double p1z,
                                            double p2x, double p2y, double p2z, double kx,
                                            double ky, double kz, double scale, double inv_scale, bool fits,
                                            unsigned *chk = nullptr)
{
#ifdef PIC_CHECK   // the cell's 12 edges lie inside the J tile
    if (chk) {
        const int tz = jbase / T::JPY, ty = (jbase % T::JPY) / T::JPX, tx = (jbase % T::JPY) % T::JPX;
        PIC_DCHECK(jbase >= 0 && tx + 1 < T::TJ && ty + 1 < T::TJ && tz + 1 < T::TJ, chk);
    }
#else
    (void)chk;
#endif
    const EdgeVals e = seg_values(p1x, p1y, p1z, p2x, p2y, p2z, kx * scale, ky * scale, kz * scale);
    if (fits)
        tile_add<T>(jt, jbase, e);
    else
        global_add<T>(J, gorigin, g, jbase, e, inv_scale);
}

// Do the tile values of a particle's path fit the fixed-point range?  Every
// segment of the path has |D| <= |d| per axis (d = the whole displacement in
// cell units), so |f W| <= |k d| (1 + 1/12) bounds all its values; a particle
// that sped up by more than the 2x headroom of the scale since the last step
// fails and deposits into the fp64 global J instead.
__device__ __forceinline__ bool fits_tile(double dx, double dy, double dz, double kx, double ky, double kz,
                                          double scale)
{
    return fmax(fabs(kx * dx), fmax(fabs(ky * dy), fabs(kz * dz))) * scale * (13.0 / 12.0) < kFixRange;
}

// Deposits the rest of a split path (<= 2 more face crossings) starting in
// the cell with J-tile index jb; a, b in that cell's coordinates.
template <class T>
__device__ __forceinline__ void deposit_remainder(unsigned *jt, int jb, double *J, int64_t gorigin,
                                                  const GridDev &g, double a0, double a1,
                                                  double a2, double b0, double b1, double b2,
                                                  double kx, double ky, double kz, double scale,
                                                  double inv_scale, bool fits, unsigned *chk = nullptr)
{
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
        double e0, e1, e2, r1[3], r2[3];
        int ox, oy, oz;
        const bool more = vb_first_piece(a0, a1, a2, b0, b1, b2, e0, e1, e2, r1, r2, ox, oy, oz);
        deposit_seg<T>(jt, jb, J, gorigin, g, a0, a1, a2, e0, e1, e2, kx, ky, kz, scale, inv_scale, fits, chk);
        if (!more) break;
        jb += ox + T::JPX * oy + T::JPY * oz;
        a0 = r1[0]; a1 = r1[1]; a2 = r1[2];
        b0 = r2[0]; b1 = r2[1]; b2 = r2[2];
    }
}

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
__global__ void __launch_bounds__(TileGeom<S, H>::NT, TileGeom<S, H>::CTAS)
k_push_tile(const __grid_constant__ CUtensorMap eb_map, GridDev g, const double *__restrict__ EB,
            double *__restrict__ J, const __grid_constant__ TileSpecies ts, int split, int zlo_n, int zhi0,
            unsigned *err)
{
    static_assert(NSP == 1 || NSP == 2, "one or two species per launch");
    using T = TileGeom<S, H>;
    constexpr int TJ = T::TJ, NE = T::NE, NJ = T::NJ, NT = T::NT;
    constexpr int EPX = T::EPX, EPY = T::EPY, JPX = T::JPX, JPY = T::JPY;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *eb = (double *)(smem_raw + T::off_eb);         // [6][TE][TE][EPX]
    const double *ebx = eb + T::XSH;                       // node (ox, oy, oz) of component 0
    constexpr int PW = T::PW;
    double *pbuf = (double *)(smem_raw + T::off_part) + (threadIdx.x >> 5) * 2 * T::PSTAGE;   // this warp's 2 stages
    double *q = (double *)(smem_raw + T::off_q);           // [6][kQueue]
    unsigned *jt = (unsigned *)(smem_raw + T::off_jt);     // [3 chunks][3][TJ][JPY/..]
    unsigned *qcell = (unsigned *)(smem_raw + T::off_qcell);
    unsigned *qcount = qcell + kQueue;
    unsigned *fq = (unsigned *)(smem_raw + T::off_fq);     // particles outside the tile
    unsigned *fqcount = fq + kFQueue;
    uint64_t *bar_eb = (uint64_t *)(smem_raw + T::off_misc);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // `split` CTAs share a supercell, each taking a contiguous part of its
    // particles (short grids fill the last wave; each CTA has its own tiles)
    // grid = (nsx * split, nsy, nsz): no integer divisions on the common path
    const int scx = split == 1 ? (int)blockIdx.x : (int)blockIdx.x / split;
    const int part = split == 1 ? 0 : (int)blockIdx.x % split;
    // supercell layers of this launch: [0, zlo_n) then [zhi0, ...) (the z-slab
    // overlap splits a step's push into the boundary layers and the interior)
    const int scy = blockIdx.y, scz = (int)blockIdx.z < zlo_n ? (int)blockIdx.z : zhi0 + (int)blockIdx.z - zlo_n;
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
    const int n0 = b0 - a0, n1 = b1 - a1;
    if (n0 + n1 == 0) return;   // empty (uniform per CTA)
    // concatenated index i: species 0 in [0, n0), species 1 from the next
    // warp boundary n0p on (a warp's 32 particles are of one species); lanes
    // in [n0, n0p) idle like the lanes past the end
    const int n0p = NSP == 2 ? (n0 + 31) & ~31 : n0, total = n0p + n1;
    const int a1m = a1 - n0p;   // species 1: array index = a1m + i (n0p even: same parity as a1)
    auto locate = [&](int i, bool &s1, int &p) {   // -> species (s1: the second one), array index p
        s1 = NSP == 2 && i >= n0p;
        p = (s1 ? a1m : a0) + i;
    };

    // local-grid coordinates of the tile origin (same for the E/B and J tiles)
    const int ox = scx * S - H - 1, oy = scy * S - H - 1, oz = scz * S - H - 1;
    const int64_t gorigin = pidx(g, ox, oy, oz);   // padded global index of tile node (0,0,0)

    // The particle state is staged through shared memory by the TMA engine:
    // each warp stages the 32 particles of its iteration after next with one
    // 2-D tensor load (the [6][kPartBox] box of the SoA store from the even
    // node at or before its first particle) into one of its two stages,
    // completing on the stage's mbarrier.  Per-thread LDGSTS staging costs
    // ~19 more L1/shared data-pipe wavefronts per 32 particles -- the
    // kernel's binding resource (tools/mb_stage.cu); per-warp stages keep the
    // warps independent.
    auto chunk_p = [&](int base, bool &s1) {   // array index of the warp chunk at concatenated index base
        s1 = NSP == 2 && base >= n0p;
        return (s1 ? a1m : a0) + base;
    };
    // shared-window address of the warp's stages; stage st's mbarrier sits
    // at sbuf + st * PSTAGE * 8 + PBAR
    const uint32_t sbuf = smem_u32(pbuf);
    auto issue = [&](int base, int st) {   // lane 0
        bool s1;
        const int p = chunk_p(base, s1);
        const uint32_t sdst = sbuf + st * (T::PSTAGE * 8u);
        mbar_arrive_expect_tx(sdst + T::PBAR, 6 * kPartBox * sizeof(double));
        tma_load_2d(sdst, s1 ? &ts.pm[NSP - 1] : &ts.pm[0], p & ~1, 0, sdst + T::PBAR);
    };
    if (tid == 0) {
        mbar_init(bar_eb, 1);
        for (int w = 0; w < 2 * T::NW; ++w)
            mbar_init((uint64_t *)(smem_raw + T::off_part + w * (T::PSTAGE * 8) + T::PBAR), 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar_eb, 6 * NE * sizeof(double));
        tma_load_4d(eb, &eb_map, ox + kGhost - T::XSH, oy + kGhost, oz + kGhost, 0, bar_eb);
    }
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
    // this thread's max |u|^2 after the push per species, as the high word of
    // the fp64 value (non-negative doubles order like their bit patterns)
    unsigned u2hi0 = 0u, u2hi1 = 0u;
    // fixed-point range check of a path, folded into the displacement check:
    // every value of a path is <= |k d| (1 + 1/12) with d its displacement in
    // cells, so max_a |d_a| < dlim (the smaller of 1 cell and the range bound
    // over both species and all axes) means "displacement valid and fits the
    // tile"; a particle past dlim is sorted out exactly on the rare path
    double kmax = fmax(fabs(ts.sp[0].kx), fmax(fabs(ts.sp[0].ky), fabs(ts.sp[0].kz)));
    if (NSP == 2)
        kmax = fmax(kmax, fmax(fabs(ts.sp[NSP - 1].kx), fmax(fabs(ts.sp[NSP - 1].ky), fabs(ts.sp[NSP - 1].kz))));
    const double dlim = fmin(1.0, kFixRange / (kmax * scale * (13.0 / 12.0)));
    const bool tile_ok = n0 + n1 <= kMaxTileParticles;   // else the counters could overflow
    __syncthreads();   // mbarriers initialised, J tile zeroed
    if (lane == 0) {   // this warp's first two chunks
        if (tid < total) issue(tid, 0);
        if (tid + NT < total) issue(tid + NT, 1);
    }
    mbar_wait(bar_eb, 0);

    // warp-uniform trip count: lanes past the end run the last iteration idle
    // (measured 4% faster on C3 than a per-lane loop: ptxas keeps the
    // two-species kernel at 128 registers without the spill the other form
    // has)
    int c = 0;
    for (int i = tid; i - lane < total; i += NT, ++c) {
        const bool valid = i < total;
        const int st = c & 1;
        mbar_wait(sbuf + st * (T::PSTAGE * 8u) + T::PBAR, (c >> 1) & 1);
        // the chunk's first particle sits at slot 0 or 1 (its array index is
        // a0 or a1 plus an even offset)
        const double *pl = pbuf + st * T::PSTAGE + lane + ((NSP == 2 && i - lane >= n0p ? a1m : a0) & 1);
        const double x0 = pl[0], y = pl[PW], z = pl[2 * PW];
        double ux = pl[3 * PW], uy = pl[4 * PW], uz = pl[5 * PW];
        __syncwarp();
        if (lane == 0 && i - lane + 2 * NT < total) {   // refill the stage two iterations ahead
            fence_proxy_async_smem();
            issue(i - lane + 2 * NT, st);
        }
        bool s1;
        int p;
        locate(valid ? i : 0, s1, p);
        const bool live = valid && (NSP == 1 || i < n0 || i >= n0p);
        const double x = live ? x0 : kDeadX;
        // dead slot (migrated away or absorbed since the last sort; a single
        // periodic box has none) or a lane past the end
        if (!live || (kGeneral && x < 0.0)) continue;
        const double gx = x * g.inv_dx, gy = y * g.inv_dy, gz = z * g.inv_dz - (double)g.k0;
        const AxisW wx = axis_weights(gx), wy = axis_weights(gy), wz = axis_weights(gz);
        // tile-relative start cell; inside the tile when in [1, S + 2H] on every axis
        const int tx = wx.i0 - ox, ty = wy.i0 - oy, tz = wz.i0 - oz;
        const bool inside = tile_ok && (unsigned)(tx - 1) < (unsigned)(S + 2 * H) &&
                            (unsigned)(ty - 1) < (unsigned)(S + 2 * H) &&
                            (unsigned)(tz - 1) < (unsigned)(S + 2 * H);
        if (inside) {
            const int hx = wx.ih - ox, hy = wy.ih - oy, hz = wz.ih - oz;
            // the 8 corners of every component lie inside the E/B tile
            PIC_DCHECK(hx >= 0 && hy >= 0 && hz >= 0 && tx >= 0 && ty >= 0 && tz >= 0 && hx + 1 < T::TE &&
                           hy + 1 < T::TE && hz + 1 < T::TE && tx + 1 < T::TE && ty + 1 < T::TE && tz + 1 < T::TE,
                       err);
            const double ex = trilinear(ebx + 0 * NE, hx + EPX * ty + EPY * tz, EPX, EPY, wx.fh, wy.f0, wz.f0);
            const double ey = trilinear(ebx + 1 * NE, tx + EPX * hy + EPY * tz, EPX, EPY, wx.f0, wy.fh, wz.f0);
            const double ez = trilinear(ebx + 2 * NE, tx + EPX * ty + EPY * hz, EPX, EPY, wx.f0, wy.f0, wz.fh);
            const double bx = trilinear(ebx + 3 * NE, tx + EPX * hy + EPY * hz, EPX, EPY, wx.f0, wy.fh, wz.fh);
            const double by = trilinear(ebx + 4 * NE, hx + EPX * ty + EPY * hz, EPX, EPY, wx.fh, wy.f0, wz.fh);
            const double bz = trilinear(ebx + 5 * NE, hx + EPX * hy + EPY * tz, EPX, EPY, wx.fh, wy.fh, wz.f0);
            boris(s1 ? ts.sp[NSP - 1].h : ts.sp[0].h, ex, ey, ez, bx, by, bz, ux, uy, uz);
            const double u2 = ux * ux + uy * uy + uz * uz;
            const double ig = rsqrt_ge1(1.0 + u2);
            const double xn = fma(cdt * ig, ux, x), yn = fma(cdt * ig, uy, y), zn = fma(cdt * ig, uz, z);
            // move endpoints in start-cell coordinates (a = fractional parts, exact)
            const double bxl = xn * g.inv_dx - (double)wx.i0;
            const double byl = yn * g.inv_dy - (double)wy.i0;
            const double bzl = (zn * g.inv_dz - (double)g.k0) - (double)wz.i0;
            const double dxl = bxl - wx.f0, dyl = byl - wy.f0, dzl = bzl - wz.f0;
            const unsigned h2 = (unsigned)__double2hiint(u2);
            u2hi0 = max(u2hi0, s1 ? 0u : h2);
            if (NSP == 2) u2hi1 = max(u2hi1, s1 ? h2 : 0u);
            const ParticlesDev &in = s1 ? ts.in[NSP - 1] : ts.in[0];
            const ParticlesDev &out = s1 ? ts.out[NSP - 1] : ts.out[0];
            const SpeciesDev &sp = s1 ? ts.sp[NSP - 1] : ts.sp[0];
            const bool fast = fabs(dxl) < dlim && fabs(dyl) < dlim && fabs(dzl) < dlim;
            bool ok = fast, fits = fast;
            if (!fast) {   // rare: exactly which of the two failed
                ok = fabs(dxl) < 1.0 && fabs(dyl) < 1.0 && fabs(dzl) < 1.0;
                fits = fits_tile(dxl, dyl, dzl, sp.kx, sp.ky, sp.kz, scale);
            }
            if (ok)
                store_particle<kGeneral>(g, sp, out, in.id, p, wrap_coord(xn, g.Lx), wrap_coord(yn, g.Ly),
                                         kGeneral ? wrap_z(g, zn) : wrap_coord(zn, g.Lz), ux, uy, uz, false, err);
            else
                store_particle<kGeneral>(g, sp, out, in.id, p, x, y, z, ux, uy, uz, false, err);
            if (ok) {
                const double kx = sp.kx, ky = sp.ky, kz = sp.kz;   // q w / (dt dA), host
                const int jbase = tx + JPX * ty + JPY * tz;
                double ex_, ey_, ez_, r1[3], r2[3];
                int cx, cy, cz;
                const bool more =
                    vb_first_piece(wx.f0, wy.f0, wz.f0, bxl, byl, bzl, ex_, ey_, ez_, r1, r2, cx, cy, cz);
                deposit_seg<T>(jt, jbase, J, gorigin, g, wx.f0, wy.f0, wz.f0, ex_, ey_, ez_, kx, ky, kz, scale,
                               inv_scale, fits, err);
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
                                             r2[2], kx, ky, kz, scale, inv_scale, fits, err);
                    }
                }
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
                push_one_global<kGeneral>(g, EB, J, sp, xx, yy, zz, ux, uy, uz, err);
                store_particle<kGeneral>(g, sp, out, in.id, p, xx, yy, zz, ux, uy, uz, false, err);
                const unsigned h2 = (unsigned)__double2hiint(ux * ux + uy * uy + uz * uz);
                u2hi0 = max(u2hi0, s1 ? 0u : h2);
                if (NSP == 2) u2hi1 = max(u2hi1, s1 ? h2 : 0u);
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
                             inv_scale, true, err);
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
        push_one_global<kGeneral>(g, EB, J, sp, xx, yy, zz, ux, uy, uz, err);
        store_particle<kGeneral>(g, sp, out, in.id, p, xx, yy, zz, ux, uy, uz, false, err);
        const unsigned h2 = (unsigned)__double2hiint(ux * ux + uy * uy + uz * uz);
        u2hi0 = max(u2hi0, s1 ? 0u : h2);
        if (NSP == 2) u2hi1 = max(u2hi1, s1 ? h2 : 0u);
    }
    {
        const unsigned hi0 = __reduce_max_sync(0xffffffffu, u2hi0);
        if (lane == 0 && hi0) atomicMax(ts.sp[0].u2max_out, hi0);
        if (NSP == 2) {
            const unsigned hi1 = __reduce_max_sync(0xffffffffu, u2hi1);
            if (lane == 0 && hi1) atomicMax(ts.sp[NSP - 1].u2max_out, hi1);
        }
    }
    __syncthreads();
    // flush the fixed-point tile to the fp64 global J.  Lanes run along x (a
    // warp covers 3 rows of TJ consecutive nodes, lanes 3 TJ.. idle): the tile
    // reads hit consecutive banks and the REDGs of a row are coalesced.
    const int64_t cs = g.cs, gsy = g.X, gsz = (int64_t)g.X * g.Y;
    constexpr int kRowsPerWarp = 32 / TJ;
    const int a = lane % TJ, rsub = lane / TJ;
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
                        const TileSpecies &ts, unsigned *err, int64_t mean_per_sc, int part, int zb,
                        const int zr[2], cudaStream_t st)
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
    // part 0: every supercell layer; 1: the zb layers at each z end of the
    // slab; 2: the layers in between (see launch_push_tile)
    int zlo_n = g.nsz, zhi0 = 0, nz_l = g.nsz;
    if (part != 0 && 2 * zb < g.nsz) {
        if (part == 1) { zlo_n = zb; zhi0 = g.nsz - zb; nz_l = 2 * zb; }
        else { zlo_n = 0; zhi0 = zb; nz_l = g.nsz - 2 * zb; }
    } else if (part == 2) {
        return;   // the boundary part covered every layer
    } else if (part == 0) {   // only the occupied layers [zr[0], zr[1])
        zlo_n = 0;
        zhi0 = zr[0];
        nz_l = zr[1] - zr[0];
        if (nz_l <= 0) return;
    }
    const dim3 grid((unsigned)(g.nsx * split), (unsigned)g.nsy, (unsigned)nz_l);
    if (ts.n == 1)
        k_push_tile<S, H, kGeneral, 1><<<grid, TileGeom<S, H>::NT, smem, st>>>(map, g, EB, J, ts, split, zlo_n, zhi0, err);
    else
        k_push_tile<S, H, kGeneral, 2><<<grid, TileGeom<S, H>::NT, smem, st>>>(map, g, EB, J, ts, split, zlo_n, zhi0, err);
}

bool tile_supported(int S, int H) { return (S == 2 || S == 4) && (H == 1 || H == 2); }

template <int S, int H>
static void box_of(int box[4])
{
    box[0] = TileGeom<S, H>::EPX;
    box[1] = TileGeom<S, H>::TE;
    box[2] = TileGeom<S, H>::TE;
    box[3] = 6;
}

void tile_box(int S, int H, int box[4])
{
    if (S == 4 && H == 1) box_of<4, 1>(box);
    else if (S == 4 && H == 2) box_of<4, 2>(box);
    else if (S == 2 && H == 1) box_of<2, 1>(box);
    else box_of<2, 2>(box);
}

template <int S, int H, bool G>
static void set_smem()
{
    const int b = (int)TileGeom<S, H>::smem_bytes;
    cudaFuncSetAttribute(k_push_tile<S, H, G, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(k_push_tile<S, H, G, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

template <int S, int H>
static void set_smem_both()
{
    set_smem<S, H, false>();
    set_smem<S, H, true>();
}

void configure_tile_kernels()
{
    set_smem_both<4, 1>();
    set_smem_both<4, 2>();
    set_smem_both<2, 1>();
    set_smem_both<2, 2>();
}

template <int S, int H>
static void launch_sh(const CUtensorMap &map, const GridDev &g, const double *EB, double *J, const TileSpecies &ts,
                      unsigned *err, int64_t mean_per_sc, int part, int zb, const int zr[2], cudaStream_t st)
{
    if (g.nranks > 1 || g.open_z)
        launch_tile<S, H, true>(map, g, EB, J, ts, err, mean_per_sc, part, zb, zr, st);
    else
        launch_tile<S, H, false>(map, g, EB, J, ts, err, mean_per_sc, part, zb, zr, st);
}

void launch_push_tile(const CUtensorMap &map, const GridDev &g, const double *EB, double *J,
                      const TileSpecies &ts, unsigned *err, int64_t mean_per_sc, int part, int zb, const int zr[2],
                      cudaStream_t st)
{
    if (ts.n == 0) return;
    if (g.S == 4 && g.H == 1) launch_sh<4, 1>(map, g, EB, J, ts, err, mean_per_sc, part, zb, zr, st);
    else if (g.S == 4 && g.H == 2) launch_sh<4, 2>(map, g, EB, J, ts, err, mean_per_sc, part, zb, zr, st);
    else if (g.S == 2 && g.H == 1) launch_sh<2, 1>(map, g, EB, J, ts, err, mean_per_sc, part, zb, zr, st);
    else if (g.S == 2 && g.H == 2) launch_sh<2, 2>(map, g, EB, J, ts, err, mean_per_sc, part, zb, zr, st);
}

}  // namespace pic
