// particle_store.cuh -- final store of a pushed particle: into the state
// arrays, or (z-slab decomposition) into the send
// buffer of the neighbouring rank when its wrapped z left this rank's slab,
// leaving a dead slot behind.
#pragma once
#include "common.cuh"

namespace pic {

// returns true when the particle migrated (slot now dead).  kGeneral =
// false compiles the single-domain periodic store only (no slab or open-box
// branches; the kernels pick it when nranks == 1 and z is periodic).
template <bool kGeneral = true>
__device__ __forceinline__ bool store_particle(const GridDev &g, const SpeciesDev &sp,
                                               const ParticlesDev &out, const uint64_t *in_id,
                                               int64_t p, double x, double y, double z, double ux,
                                               double uy, double uz, bool copy_id, unsigned *err)
{
    if constexpr (!kGeneral) {
        out.x[p] = x; out.y[p] = y; out.z[p] = z;
        out.ux[p] = ux; out.uy[p] = uy; out.uz[p] = uz;
        if (copy_id) out.id[p] = in_id[p];
        return false;
    }
    if (g.open_z && !(z >= 0.0 && z < g.zmax)) {
        // NEXT-1: left the open box through z = 0 or z = zmax (its current up to
        // the face is deposited): absorbed, the slot is dead until the next sort
        out.x[p] = kDeadX;
        return true;
    }
    if (g.nranks > 1 && !(z >= g.zlo && z < g.zhi)) {
        // one step moves < 1 cell, so the new owner is the lower (dir 0) or the
        // upper (dir 1) neighbour in the ring of slabs: the nearer face, measured
        // periodically (slabs may differ in width, pic_balance_slabs)
        double ddn = g.zlo - z, dup = z - g.zhi;
        if (ddn < 0.0) ddn += g.Lz;
        if (dup < 0.0) dup += g.Lz;
        const int dir = ddn <= dup ? 0 : 1;
        if (fmin(ddn, dup) > g.dz) atomicOr(err, kErrDisplacement);
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
