// kernels.cuh -- host-side launchers of the libpic kernels (internal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace pic {

// per step: fixed-point J-tile scale per species from u2max_in, u2max_out = 0
// (a stand-alone launch before the first step; then by the previous step's
// k_e_full, which runs after that step's particle kernels)
struct StepPrep {
    int n_species;
    double qw[4];
    double c, dV;
    const unsigned *u2max_in;   // the bound of the step that was pushed last
    unsigned *u2max_out;        // reset for the next step's particle kernels
    double *scale;              // [species][2]: 2^F, 2^-F
};
void launch_step_prep(const StepPrep &p, cudaStream_t st);

// Every contribution to the J tile is bounded by |qw| c beta / (dx dy dz) *
// 13/12 with beta <= 2 x the largest beta of the last step (from its max
// |u|^2); 2^F maps that bound to < 2^46 (the fixed-point notes in push_tile.cu).
__device__ __forceinline__ void step_prep_species(const StepPrep &p, int s)
{
    const double u2 = __longlong_as_double(((unsigned long long)p.u2max_in[s] << 32) | 0xffffffffull);
    const double beta = fmax(1e-4, fmin(1.0, 2.0 * sqrt(u2 / (1.0 + u2))));
    // constant indices only: a runtime index into the parameter struct would
    // copy it to local memory in every thread of the calling kernel
    double qw = p.qw[0];
#pragma unroll
    for (int t = 1; t < 4; ++t) qw = s == t ? p.qw[t] : qw;
    const double wmax = fabs(qw) * p.c / p.dV * (13.0 / 12.0) * beta;
    const int F = wmax > 0.0 ? min(1000, (int)floor(46.0 - log2(wmax))) : 1000;
    p.scale[2 * s] = ldexp(1.0, F);
    p.scale[2 * s + 1] = ldexp(1.0, -F);
    p.u2max_out[s] = 0u;
}

// ---- fields.cu : Yee FDTD and ghost maintenance ----
// Bout1 = Bin - (c dt/2) curl E (E of EB), and with Bout2 also Bout2 = Bout1 -
// (c dt/2) curl E, on planes [kbegin, nz) (kbegin = -1 computes the lower z
// ghost plane of a slab locally); results also stored to their ghost images.
void launch_b_half(const GridDev &g, const double *EB, const double *Bin, double *Bout1, double *Bout2,
                   cudaStream_t st, int kbegin = 0);
// E += c dt curl Bh - 4 pi dt J (Bh = B^{n+1/2}) where J = sum of the ghost
// images of Jcur (the fold); writes the folded J back into
// Jcur's interior, stores E to its ghost images and zeroes every image of Jnext.
// With prep.n_species > 0 its first threads also run the next step's J-tile
// scale preparation (launch_step_prep's work, after this step's particle kernels).
// jl = {first, last} padded z planes the particle kernels can have deposited
// into Jcur (this step, jl[0..1]) and Jnext (the previous step, jl[2..3]);
// a plane none of whose images lies in its range holds zeros there, so its J
// is not read (cur) or not cleared (next).  {0, Z - 1}: every plane.
struct JPlanes {
    int cur_lo, cur_hi, next_lo, next_hi;
};
void launch_e_full(const GridDev &g, double *EB, const double *Bh, double *Jcur, double *Jnext,
                   const StepPrep &prep, cudaStream_t st, const JPlanes &jl);
// Copies interior values of `ncomp` components to their ghost images.
void launch_fill_ghosts(const GridDev &g, double *F, int ncomp, cudaStream_t st);
// NEXT-1 (open z): laser = {e0, omega, ramp, t0, pol_x, pol_y}.  Writes the
// incident values of step *step at z = 0 into out[8] (g.laser) and
// increments *step; a one-thread kernel inside the step's graph.
void launch_laser_coeffs(const GridDev &g, const double laser[6], int64_t *step, double *out, cudaStream_t st);
// E^0, B^0 of the local slab = the incident wave at t = 0 (pic_laser_preload)
void launch_laser_preload(const GridDev &g, const double laser[6], double *EB, cudaStream_t st);

// ---- push_naive.cu ----
void launch_push_naive(const GridDev &g, const double *EB, double *J, const ParticlesDev &in,
                       const ParticlesDev &out, int64_t n, const SpeciesDev &sp, bool copy_id,
                       unsigned *err, cudaStream_t st);

void launch_push_tail(const GridDev &g, const double *EB, double *J, const ParticlesDev &in,
                      const ParticlesDev &out, const int64_t *dev_lo, const int64_t *dev_hi,
                      int64_t max_n, const SpeciesDev &sp, bool copy_id, unsigned *err,
                      cudaStream_t st);

// ---- push_tile.cu : fused supercell kernel ----
bool tile_supported(int S, int H);
void tile_box(int S, int H, int box[4]);   // TMA box of the E/B tile (x pitch, y, z, comps)
// max |u|^2 of n particles -> *out (high 32 bits of the fp64 value)
void launch_u2max(const ParticlesDev &P, int64_t n, unsigned *out, cudaStream_t st);
void configure_tile_kernels();
// The species of one fused-kernel launch (one or two species with particles):
// input arrays (sorted B on a sort step, else A), output arrays (A), offsets.
constexpr int kTileMaxSpecies = 2;
// the fused kernel stages a warp's 32 particles with one 2-D TMA load of a
// [6 components][kPartBox particles] box of the SoA store (runtime.cu
// encode_particle_maps): 34 = 32 + the one-node shift to an even (16-byte
// aligned) start
constexpr int kPartBox = 34;
struct TileSpecies {
    CUtensorMap pm[kTileMaxSpecies];   // TMA descriptors of the `in` stores
    ParticlesDev in[kTileMaxSpecies], out[kTileMaxSpecies];
    const int64_t *sc_off[kTileMaxSpecies];
    SpeciesDev sp[kTileMaxSpecies];
    int n;
};
// mean_per_sc: particles per supercell over all species (splits very dense supercells).
// part 0 pushes every supercell layer; with z slabs, part 1 the zb layers at
// each z end of the slab (the only ones whose particles can deposit into the
// exchanged J ghost planes or leave the slab this step, runtime.cu
// boundary_layers) and part 2 the layers in between (a no-op when part 1
// covered them all).
// zr = [first, end) of the supercell layers launched by part 0 (the occupied
// ones, runtime.cu push_layers; {0, nsz} for all).
void launch_push_tile(const CUtensorMap &eb_map, const GridDev &g, const double *EB, double *J,
                      const TileSpecies &ts, unsigned *err, int64_t mean_per_sc, int part, int zb,
                      const int zr[2], cudaStream_t st);

// ---- sort.cu : stable counting sort by (supercell, local cell) ----
struct SortScratch {
    uint32_t *key;       // [cap]
    uint32_t *slot;      // [cap]
    uint32_t *perm_tmp;  // [cap]
    uint32_t *perm;      // [cap]
    uint32_t *count;     // [ncells + 1]
    uint32_t *start;     // [ncells + 1]
    uint32_t *block_sums;// [scan blocks]
};
size_t scan_block_count(int64_t nitems);
// stable copy of the live slots [0, n) of src (x != kDeadX) to dst[0, live);
// returns live (synchronises st).  bsums: scan_block_count(n + 1) entries
int64_t compact_live(const ParticlesDev &src, const ParticlesDev &dst, int64_t n, const SortScratch &s,
                     uint32_t *bsums, cudaStream_t st);
// dst[0 .. *dev_n) = src[...] (the sorted ids into the state buffer)
void launch_copy_ids(const uint64_t *src, uint64_t *dst, const int64_t *dev_n, int64_t cap, cudaStream_t st);
// Sorts the *dev_n particle slots src -> dst (x,y,z,ux,uy,uz,id), dropping
// dead slots (x == kDeadX); writes the supercell offsets sc_off[0..n_sc]
// (int64) and the live count back to *dev_n.  Grids are sized for cap.
// occupied supercell z-layers after a sort (k_occ_range): out = {first, last}
constexpr int kOccMaxSpecies = 4;   // = PIC_MAX_SPECIES (include/pic.h)
struct OccRange {
    const int64_t *sc_off[kOccMaxSpecies];
    int ns;            // species with particles
    int64_t per_layer; // supercells per z-layer
    int nsz;           // supercell layers
};
void launch_occ_range(const OccRange &a, int *out, cudaStream_t st);

// zr (optional): supercell layers [zr[0], zr[1]) known to hold every particle
// after the sort (runtime.cu push_layers); the per-supercell order kernel
// runs over those only
void sort_particles(const GridDev &g, const ParticlesDev &src, const ParticlesDev &dst,
                    int64_t *dev_n, int64_t cap, const SortScratch &s, int64_t *sc_off,
                    unsigned *err, cudaStream_t st, int *launches, const int *zr = nullptr);

// ---- slab.cu : z-slab exchange helpers ----
// J ghost planes received from the neighbours are added into the interior
// planes they belong to; this rank's own J ghost planes (already sent) are
// zeroed for the next deposit.  recv_dn: from rank-1 (its planes nz, nz+1 =
// our 0, 1); recv_up: from rank+1 (its planes -2, -1 = our nz-2, nz-1).
void launch_j_ghost_add(const GridDev &g, double *J, const double *recv_dn, const double *recv_up,
                        cudaStream_t st);
// header (count, capped) of a migration send buffer, capacity check
void launch_mig_finalize(const MigrateDev &m, unsigned *err, cudaStream_t st);
// after the interior part of an overlapped push: no particle may have been
// queued for migration after launch_mig_finalize (the boundary-layer bound)
void launch_mig_late_check(const MigrateDev &m, unsigned *err, cudaStream_t st);
// appends the particles of two received migration buffers at the tail of P
void launch_mig_append(const double *recv0, const double *recv1, int cap, const ParticlesDev &P,
                       int64_t *dev_n, int64_t pcap, unsigned *err, cudaStream_t st);

// ---- diag.cu : diagnostics between steps ----
// CIC rho of live particles [0, *dev_n) into the padded node array `rho`
// (pre-zeroed; the top ghost plane holds what belongs to the slab above) and
// sum (gamma - 1) into *acc_kinetic.
void launch_diag_particles(const GridDev &g, const ParticlesDev &P, const int64_t *dev_n, int64_t cap,
                           double qw, double *rho, double *acc_kinetic, cudaStream_t st);
// folds rho (+ rho_below: the lower slab's top ghost plane, or nullptr), then
// per node: energies, sums, div B, Gauss residual and drift vs gauss0
// (stored instead when !have_g0), continuity vs rho_prev (then rho_prev = rho).
// jz_below: the lower slab's top interior Jz plane (nullptr when periodic).
void launch_diag_nodes(const GridDev &g, const double *EB, const double *J, const double *jz_below,
                       double *rho, const double *rho_below, double *rho_prev, double *gauss0,
                       bool have_prev, bool have_g0, double *acc, cudaStream_t st);

}  // namespace pic
