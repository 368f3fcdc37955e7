// particle_store.cuh -- final store of a pushed particle: into the state
// arrays, or (z-slab decomposition) into the send
// buffer of the neighbouring rank when its wrapped z left this rank's slab,
// leaving a dead slot behind.
#pragma once
#include "common.cuh"

namespace pic {

// returns true when the particle migrated (slot now dead)
__device__ __forceinline__ bool store_particle(const GridDev &g, const SpeciesDev &sp,
                                               const ParticlesDev &out, const uint64_t *in_id,
                                               int64_t p, double x, double y, double z, double ux,
                                               double uy, double uz, bool copy_id, unsigned *err)
{
    if (g.nranks > 1 && !(z >= g.zlo && z < g.zhi)) {
        // new owner from the wrapped z; one step moves < 1 cell, so it is the lower
        // (dir 0) or the upper (dir 1) neighbour in the periodic ring of slabs
        int owner = (int)floor(z / (g.zhi - g.zlo));
        owner = owner < 0 ? 0 : (owner >= g.nranks ? g.nranks - 1 : owner);
        const int dir = (owner == (g.rank + g.nranks - 1) % g.nranks) ? 0 : 1;
        if (dir == 1 && owner != (g.rank + 1) % g.nranks) atomicOr(err, kErrDisplacement);
        const unsigned slot = atomicAdd(sp.mig.count + dir, 1u);
        if (slot < (unsigned)sp.mig.cap) {
            double *b = sp.mig.send[dir] + 1;
            const int64_t c = sp.mig.cap;
            b[slot] = x;
            b[c + slot] = y;
            b[2 * c + slot] = z;
            b[3 * c + slot] = ux;
            b[4 * c + slot] = uy;
            b[5 * c + slot] = uz;
            b[6 * c + slot] = __longlong_as_double((long long)in_id[p]);
        } else {
            atomicOr(err, kErrCapacity);
        }
        out.x[p] = kDeadX;
        return true;
    }
    out.x[p] = x; out.y[p] = y; out.z[p] = z;
    out.ux[p] = ux; out.uy[p] = uy; out.uz[p] = uz;
    if (copy_id) out.id[p] = in_id[p];
    return false;
}

}  // namespace pic
