// common.cuh -- device-side layout and helpers shared by the libpic kernels.
//
// HBM layout:
//  * E/B: one allocation [6][Z][Y][X] fp64, order Ex,Ey,Ez,Bx,By,Bz, each
//    component ghost-padded by G cells on every side (X = nx+2G rounded up
//    to even, Y = ny+2G, Z = nz_local+2G), x fastest.  Ghost cells hold the
//    periodic images of the interior, written by the producing kernel, so
//    the particle kernels never wrap an index.
//  * J: two such allocations [3][Z][Y][X] (ping-pong): the deposit of step
//    n lands in J_cur (interior + ghosts); the E update folds the ghost
//    images into the interior and zeroes J_next for step n+1.
//  * particles: per species SoA fp64 x,y,z,ux,uy,uz + uint64 id, double
//    buffered (A = state, B = sort target), cell-sorted every K steps.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifdef PIC_CHECK
#include <cstdio>
#endif

namespace pic {

// G: the CIC gather needs [-1, n], the VB edges [-1, n+1] (positions are
// wrapped into the box or slab, so deposits and gathers stay inside [-1, n+1]
// whatever the tile halo); the TMA box of a fused-kernel tile starts H + 1
// cells below its supercell and is zero-filled where it leaves the array
#ifndef PIC_GHOST
#define PIC_GHOST 2
#endif
constexpr int kGhost = PIC_GHOST;

// error bits of the sticky device error word
enum : unsigned {
    kErrDisplacement = 1u,
    kErrNonFinite = 2u,
    kErrCapacity = 4u,
    kErrRange = 8u,
    kErrCheck = 16u,   // an internal index check of a PIC_CHECK build failed
    kErrLateMigration = 32u,   // an interior-layer particle left the slab (overlap bound violated)
};

// Internal index checks of a debugging build (make CHECK=1 -> -DPIC_CHECK):
// a failed check sets kErrCheck in the error word (the call then returns
// PIC_ECUDA); compiled out otherwise.
#ifdef PIC_CHECK
#define PIC_DCHECK(cond, errp)                                                          \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            if (!(atomicOr((errp), (unsigned)::pic::kErrCheck) & ::pic::kErrCheck))     \
                printf("PIC_CHECK failed: %s:%d block %d thread %d\n", __FILE__, __LINE__, \
                       (int)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)), \
                       (int)threadIdx.x);                                               \
        }                                                                               \
    } while (0)
#else
#define PIC_DCHECK(cond, errp) \
    do {                       \
    } while (0)
#endif

struct GridDev {
    int nx, ny, nz;          // local interior cells (nz = slab thickness)
    int X, Y, Z;             // padded extents
    int64_t cs;              // component stride X*Y*Z
    int k0;                  // global z index of the first local cell
    int nz_global;
    double dx, dy, dz;
    double inv_dx, inv_dy, inv_dz;
    double dt, c;
    double Lx, Ly, Lz;       // global periodic lengths
    int S;                   // supercell edge
    int H;                   // tile drift halo of the fused kernel (pic_config.halo)
    int nsx, nsy, nsz;       // supercells per axis (local)
    bool periodic_z_local;   // nranks == 1: z ghosts are local images
    int nranks, rank;        // z slabs
    double zlo, zhi;         // this rank's slab [zlo, zhi) in physical z
    // NEXT-1 open z: the box ends at z = 0 and z = zmax
    bool open_z;             // PIC_BC_OPEN (x, y stay periodic)
    bool open_lo, open_hi;   // this rank holds the global z = 0 / z = zmax face
    double zmax;             // open: particles live in [0, zmax), zmax = (nz_global - 1) dz
    double mur_a;            // (c dt - dz) / (c dt + dz)
    const double *laser;     // open_lo: incident values of this step [Ex, Ey][I0', I1, I1', I0]
};


__host__ __device__ inline int64_t pidx(const GridDev &g, int i, int j, int k)
{
    return (int64_t)(i + kGhost) + (int64_t)g.X * ((int64_t)(j + kGhost) + (int64_t)g.Y * (int64_t)(k + kGhost));
}

struct ParticlesDev {
    double *x, *y, *z, *ux, *uy, *uz;
    uint64_t *id;
};

// Particles that leave the slab (nranks > 1) go to a fixed-capacity send
// buffer per direction: [0] = count (as double), then SoA x,y,z,ux,uy,uz,id
// (id bits) with stride cap.  dir 0 = down (rank - 1), dir 1 = up (rank + 1).
struct MigrateDev {
    double *send[2];
    unsigned *count;   // [2] running send counters
    int cap;
};

// Dead slot marker: a particle that migrated away leaves x = -1 (live
// positions are in [0, L)); kernels skip it, the next sort drops it.
constexpr double kDeadX = -1.0;

struct SpeciesDev {
    double qw;        // q * w
    double h;         // q dt / (2 m c)   (Boris half-kick coefficient)
    // max |u|^2 of the species (high 32 bits of the fp64 value, an upper
    // bound): read from the previous step, produced for the next one.  Sets
    // the fixed-point scale of the deposit tile (push_tile.cu).
    const unsigned *u2max_in;
    unsigned *u2max_out;
    // per-launch constants of the fused kernel (computed once, not per CTA):
    // VB flux factors q w / (dt dA) per axis (host) and the fixed-point scale
    // 2^F, 2^-F of the J tile (k_step_prep on the device, from u2max_in)
    double kx, ky, kz;
    const double *scale;   // [2]: 2^F, 2^-F
    MigrateDev mig;
};

// Periodic ghost images: f(p) for every padded index p in [-G, n+G)^3 that
// is an image of interior cell (i,j,k) under the x/y periodicity (and z when
// the slab is the whole box), the interior index included.
// first periodic image index >= -G of i, stepping by n
__device__ __forceinline__ int first_image(int i, int n)
{
    while (i - n >= -kGhost) i -= n;
    return i;
}

template <class F>
__device__ __forceinline__ void for_images(const GridDev &g, int i, int j, int k, F &&f)
{
    const int i0 = first_image(i, g.nx), j0 = first_image(j, g.ny);
    const int k0 = g.periodic_z_local ? first_image(k, g.nz) : k;
    const int kend = g.periodic_z_local ? g.nz + kGhost : k + 1;
    const int kstep = g.periodic_z_local ? g.nz : 1;
    for (int kk = k0; kk < kend; kk += kstep)
        for (int jj = j0; jj < g.ny + kGhost; jj += g.ny)
            for (int ii = i0; ii < g.nx + kGhost; ii += g.nx)
                f(pidx(g, ii, jj, kk));
}

}  // namespace pic
