// slab.cu -- device side of the z-slab decomposition (SURVEY.md sec. 8a row
// a8, sec. 8e; "spatial domain decomposition ... with
// communications only between neighbor domains").
//
// Per step and rank: the deposit spills into the J ghost planes (z in
// {-2,-1} and {nz, nz+1}); those planes are sent to the neighbours, which add
// them into the interior planes they belong to (the z part of the fold).
// Particles whose wrapped z left the slab were written by the push kernels
// into per-direction send buffers; received ones are appended after the
// sorted region and pushed by the tail kernel until the next sort.
#include "kernels.cuh"

namespace pic {

__global__ void __launch_bounds__(256)
k_j_ghost_add(GridDev g, double *__restrict__ J, const double *__restrict__ rdn,
              const double *__restrict__ rup)
{
    // one thread per (component, plane pair index, padded xy position)
    const int64_t plane = (int64_t)g.X * g.Y;
    const int64_t per_comp = 2 * plane;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 3 * per_comp) return;
    const int comp = (int)(t / per_comp);
    const int64_t r = t - comp * per_comp;          // [2 planes][Y][X]
    double *Jc = J + comp * g.cs;
    // padded plane index of local plane k is k + kGhost
    const int64_t lo_ghost = (int64_t)(kGhost - 2) * plane + r;    // planes -2, -1
    const int64_t hi_ghost = (int64_t)(g.nz + kGhost) * plane + r; // planes nz, nz+1
    const int64_t lo_int = (int64_t)kGhost * plane + r;            // planes 0, 1
    const int64_t hi_int = (int64_t)g.nz * plane + r;              // planes nz-2, nz-1
    const double add_lo = rdn[comp * per_comp + r];   // rank-1's planes nz, nz+1
    const double add_hi = rup[comp * per_comp + r];   // rank+1's planes -2, -1
    Jc[lo_int] += add_lo;
    Jc[hi_int] += add_hi;   // (nz >= 2, so the two pairs never overlap)
    Jc[lo_ghost] = 0.0;
    Jc[hi_ghost] = 0.0;
}

void launch_j_ghost_add(const GridDev &g, double *J, const double *recv_dn, const double *recv_up,
                        cudaStream_t st)
{
    const int64_t n = 3 * 2 * (int64_t)g.X * g.Y;
    k_j_ghost_add<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, J, recv_dn, recv_up);
}

__global__ void k_mig_finalize(MigrateDev m, unsigned *err)
{
    const int d = threadIdx.x;
    if (d > 1) return;
    const unsigned c = m.count[d];
    if (c > (unsigned)m.cap) atomicOr(err, kErrCapacity);
    m.send[d][0] = (double)min(c, (unsigned)m.cap);
    m.count[d] = 0u;   // reset for the next step (the buffer itself travels)
}

void launch_mig_finalize(const MigrateDev &m, unsigned *err, cudaStream_t st)
{
    k_mig_finalize<<<1, 32, 0, st>>>(m, err);
}

__global__ void k_mig_late_check(MigrateDev m, unsigned *err)
{
    if (threadIdx.x < 2 && m.count[threadIdx.x] != 0u) atomicOr(err, kErrLateMigration);
}

void launch_mig_late_check(const MigrateDev &m, unsigned *err, cudaStream_t st)
{
    k_mig_late_check<<<1, 32, 0, st>>>(m, err);
}

// appends received particles (two buffers) at [*dev_n, *dev_n + c0 + c1)
__global__ void __launch_bounds__(256)
k_mig_append(const double *__restrict__ r0, const double *__restrict__ r1, int cap, ParticlesDev P,
             const int64_t *__restrict__ dev_n, int64_t pcap, unsigned *err)
{
    const int64_t c0 = (int64_t)r0[0], c1 = (int64_t)r1[0];
    const int64_t base = *dev_n;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= c0 + c1) return;
    const double *b = (t < c0) ? r0 + 1 : r1 + 1;
    const int64_t i = (t < c0) ? t : t - c0;
    const int64_t p = base + t;
    if (p >= pcap) {
        atomicOr(err, kErrCapacity);
        return;
    }
    P.x[p] = b[i];
    P.y[p] = b[cap + i];
    P.z[p] = b[2 * (int64_t)cap + i];
    P.ux[p] = b[3 * (int64_t)cap + i];
    P.uy[p] = b[4 * (int64_t)cap + i];
    P.uz[p] = b[5 * (int64_t)cap + i];
    P.id[p] = (uint64_t)__double_as_longlong(b[6 * (int64_t)cap + i]);
}

__global__ void k_mig_commit(const double *__restrict__ r0, const double *__restrict__ r1,
                             int64_t *__restrict__ dev_n, int64_t pcap)
{
    const int64_t n = *dev_n + (int64_t)r0[0] + (int64_t)r1[0];
    *dev_n = n < pcap ? n : pcap;
}

void launch_mig_append(const double *recv0, const double *recv1, int cap, const ParticlesDev &P,
                       int64_t *dev_n, int64_t pcap, unsigned *err, cudaStream_t st)
{
    const int64_t maxn = 2 * (int64_t)cap;
    k_mig_append<<<(unsigned)((maxn + 255) / 256), 256, 0, st>>>(recv0, recv1, cap, P, dev_n, pcap, err);
    k_mig_commit<<<1, 1, 0, st>>>(recv0, recv1, dev_n, pcap);
}

}  // namespace pic
