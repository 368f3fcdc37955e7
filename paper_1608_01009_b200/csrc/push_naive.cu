// push_naive.cu -- one-thread-per-particle gather/push/deposit kernel.
//
// The plain layout of SURVEY.md sec. 7 step 3 ("a simple G4"): CIC gather
// straight from the ghost-padded E/B arrays in HBM/L2, Boris, move,
// Villasenor-Buneman deposit with fp64 global atomics (REDG.ADD.F64) into
// the padded J, periodic wrap.  It serves three roles: the PIC_FLAG_NAIVE
// baseline, the out-of-tile path of the fused kernel (push_global.cuh), and
// (z slabs) the push of the unsorted tail of particles that arrived from
// neighbouring ranks since the last sort.
#include "kernels.cuh"
#include "particle_store.cuh"
#include "push_global.cuh"

namespace pic {

// particles [lo, hi) with the bounds read from device memory (nullptr: host n)
__global__ void __launch_bounds__(256)
k_push_naive(GridDev g, const double *__restrict__ EB, double *__restrict__ J, ParticlesDev in,
             ParticlesDev out, int64_t n, const int64_t *dev_lo, const int64_t *dev_hi,
             SpeciesDev sp, int copy_id, unsigned *err)
{
    const int64_t lo = dev_lo ? *dev_lo : 0, hi = dev_hi ? *dev_hi : n;
    double u2loc = 0.0;
    for (int64_t p = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < hi;
         p += (int64_t)gridDim.x * blockDim.x) {
        double x = in.x[p], y = in.y[p], z = in.z[p];
        if (x < 0.0) continue;   // dead slot (migrated away)
        double ux = in.ux[p], uy = in.uy[p], uz = in.uz[p];
        push_one_global(g, EB, J, sp, x, y, z, ux, uy, uz, err);
        store_particle(g, sp, out, in.id, p, x, y, z, ux, uy, uz, copy_id != 0, err);
        u2loc = fmax(u2loc, ux * ux + uy * uy + uz * uz);
    }
    const unsigned hi32 = __reduce_max_sync(0xffffffffu, (unsigned)(__double_as_longlong(u2loc) >> 32));
    if ((threadIdx.x & 31) == 0 && hi32 && sp.u2max_out) atomicMax(sp.u2max_out, hi32);
}

void launch_push_naive(const GridDev &g, const double *EB, double *J, const ParticlesDev &in,
                       const ParticlesDev &out, int64_t n, const SpeciesDev &sp, bool copy_id,
                       unsigned *err, cudaStream_t st)
{
    if (n <= 0) return;
    const int bs = 256;
    const int64_t blocks = std::min<int64_t>((n + bs - 1) / bs, 148 * 64);
    k_push_naive<<<(unsigned)blocks, bs, 0, st>>>(g, EB, J, in, out, n, nullptr, nullptr, sp,
                                                 copy_id ? 1 : 0, err);
}

void launch_push_tail(const GridDev &g, const double *EB, double *J, const ParticlesDev &in,
                      const ParticlesDev &out, const int64_t *dev_lo, const int64_t *dev_hi,
                      int64_t max_n, const SpeciesDev &sp, bool copy_id, unsigned *err,
                      cudaStream_t st)
{
    const int bs = 256;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((max_n + bs - 1) / bs, 148 * 8));
    k_push_naive<<<(unsigned)blocks, bs, 0, st>>>(g, EB, J, in, out, 0, dev_lo, dev_hi, sp,
                                                 copy_id ? 1 : 0, err);
}

}  // namespace pic
