// push_naive.cu -- one-thread-per-particle gather/push/deposit kernel.
//
// The plain reference layout of SURVEY.md sec. 7 step 3 ("a simple G4"):
// CIC gather straight from the ghost-padded E/B arrays in HBM/L2, Boris,
// move, Villasenor-Buneman deposit with fp64 global atomics (REDG.ADD.F64)
// into the padded J, periodic wrap.  It is the fallback path of the fused
// supercell kernel (particles that left their tile) and the PIC_FLAG_NAIVE
// baseline, not the production path.
#include "kernels.cuh"
#include "push_global.cuh"

namespace pic {

__global__ void __launch_bounds__(256)
k_push_naive(GridDev g, const double *__restrict__ EB, double *__restrict__ J,
             ParticlesDev in, ParticlesDev out, int64_t n, SpeciesDev sp, int copy_id,
             unsigned *err)
{
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double x = in.x[p], y = in.y[p], z = in.z[p];
    double ux = in.ux[p], uy = in.uy[p], uz = in.uz[p];
    push_one_global(g, EB, J, sp, x, y, z, ux, uy, uz, err);
    out.x[p] = x; out.y[p] = y; out.z[p] = z;
    out.ux[p] = ux; out.uy[p] = uy; out.uz[p] = uz;
    if (copy_id) out.id[p] = in.id[p];
}

void launch_push_naive(const GridDev &g, const double *EB, double *J, const ParticlesDev &in,
                       const ParticlesDev &out, int64_t n, const SpeciesDev &sp, bool copy_id,
                       unsigned *err, cudaStream_t st)
{
    if (n <= 0) return;
    const int bs = 256;
    k_push_naive<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(g, EB, J, in, out, n, sp,
                                                               copy_id ? 1 : 0, err);
}

}  // namespace pic
