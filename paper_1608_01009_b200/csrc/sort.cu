// sort.cu -- re-binning sort of the particle store by
// (supercell id, slot, local cell id) (reading R15;
// PAPER.md:40,44 "particles are stored separately for each cell",
// PAPER.md:132 supercells).
//
// Deterministic and stable by construction:
//   1. key[p] = key(x_p); slot[p] = atomicAdd(&count[key], 1)   (order within
//      a bucket is arbitrary here)
//   2. start = exclusive scan of count (3-kernel reduce / scan / add)
//   3. perm_tmp[start[key] + slot] = p
//   4. one warp per bucket re-orders its entries by ascending p (rank by
//      counting) -> perm; this restores the input order inside each bucket,
//      i.e. stability, independent of the atomic order in step 1
//   5. per supercell (one CTA), cell-sorted position (c, r) -> slot-major
//      position sum_c' min(n_c', r) + #{c' < c : n_c' > r}, so a warp of
//      consecutive particles holds distinct cells (conflict-free shared
//      atomics in the deposit)
//   (4 and 5 run as one kernel per supercell in shared memory, k_order_sc)
//   6. gather x,y,z,ux,uy,uz,id through the final permutation;
//      sc_off[s] = start[s * S^3].
// The key uses floor(x / dx) with an IEEE division, the same decision the
// oracle takes (DESIGN.md sec. 3 R15), so permutations are bit-identical.
#include <algorithm>

#include "kernels.cuh"

namespace pic {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

size_t scan_block_count(int64_t nitems) { return (size_t)((nitems + kScanTile - 1) / kScanTile); }

// floor(x / d) -- the oracle's decision (an IEEE division); for a power-of-two
// d the product with 1/d is the same exact quotient and much cheaper
__device__ __forceinline__ int cell_of(double x, double d, int n_local, int offset)
{
    const double inv = 1.0 / d;
    const bool pow2 = (inv * d == 1.0) && ((__double_as_longlong(d) & 0x000fffffffffffffLL) == 0);
    int c = (int)floor(pow2 ? x * inv : x / d) - offset;
    c = c < 0 ? 0 : c;
    return c >= n_local ? n_local - 1 : c;
}

constexpr uint32_t kDeadKey = 0xffffffffu;

__global__ void __launch_bounds__(256)
k_sort_key(GridDev g, ParticlesDev src, const int64_t *__restrict__ dev_n, uint32_t *__restrict__ key,
           uint32_t *__restrict__ slot, uint32_t *__restrict__ count, unsigned *err)
{
    const int64_t n = *dev_n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int S = g.S;
    // kU particles per thread and iteration: their loads and their (returning)
    // counter atomics are in flight together instead of one latency each
    constexpr int kU = 4;
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n; p0 += kU * stride) {
        uint32_t k[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + u * stride;
            k[u] = kDeadKey;
            if (p >= n) continue;
            const double x = src.x[p], y = src.y[p], z = src.z[p];
            if (x == kDeadX) continue;   // slot left by a particle that migrated: dropped here
            if (!(x >= 0.0 && x < g.Lx && y >= 0.0 && y < g.Ly && z >= g.zlo && z < fmin(g.zhi, g.zmax)))
                atomicOr(err, isfinite(x) && isfinite(y) && isfinite(z) ? kErrRange : kErrNonFinite);
            const int cx = cell_of(x, g.dx, g.nx, 0);
            const int cy = cell_of(y, g.dy, g.ny, 0);
            const int cz = cell_of(z, g.dz, g.nz, g.k0);
            const uint32_t sc = (uint32_t)((cx / S) + g.nsx * ((cy / S) + g.nsy * (cz / S)));
            const uint32_t loc = (uint32_t)((cx % S) + S * ((cy % S) + S * (cz % S)));
            k[u] = sc * (uint32_t)(S * S * S) + loc;
        }
        uint32_t sl[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) sl[u] = k[u] != kDeadKey ? atomicAdd(count + k[u], 1u) : 0u;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + u * stride;
            if (p >= n) continue;
            key[p] = k[u];
            slot[p] = sl[u];
        }
    }
}

// ---- exclusive scan of uint32 (counts fit: n < 2^31) ----
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// block-wide exclusive scan of one value per thread; returns block total in *total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total)
{
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t s = lane < nw ? warp_sums[lane] : 0u;
        s = warp_incl_scan(s);
        warp_sums[lane] = s;
    }
    __syncthreads();
    const uint32_t warp_prefix = wid ? warp_sums[wid - 1] : 0u;
    *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return warp_prefix + inc - v;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(const uint32_t *__restrict__ in, int64_t n, uint32_t *__restrict__ block_sums)
{
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        const int64_t i = base + (int64_t)it * kScanThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    uint32_t total;
    block_excl_scan(s, &total);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// single block: exclusive scan of the block sums in place
__global__ void __launch_bounds__(kScanThreads) k_scan_blocks(uint32_t *__restrict__ sums, int64_t nb)
{
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
        const int64_t i = b0 + threadIdx.x;
        const uint32_t v = i < nb ? sums[i] : 0u;
        uint32_t total;
        const uint32_t ex = block_excl_scan(v, &total);
        if (i < nb) sums[i] = carry + ex;
        carry += total;
    }
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_add(const uint32_t *__restrict__ in, int64_t n, const uint32_t *__restrict__ block_off,
           uint32_t *__restrict__ out)
{
    // each thread owns kScanItems consecutive elements
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        v[it] = (base + it < n) ? in[base + it] : 0u;
        s += v[it];
    }
    uint32_t total;
    uint32_t ex = block_excl_scan(s, &total) + block_off[blockIdx.x];
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
        if (base + it < n) out[base + it] = ex;
        ex += v[it];
    }
}

__global__ void __launch_bounds__(256)
k_scatter(const uint32_t *__restrict__ key, const uint32_t *__restrict__ slot,
          const uint32_t *__restrict__ start, const int64_t *__restrict__ dev_n,
          uint32_t *__restrict__ perm_tmp)
{
    const int64_t n = *dev_n;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key[p];
        if (k != kDeadKey) perm_tmp[start[k] + slot[p]] = (uint32_t)p;
    }
}

// bitonic sort of 64 keys held as 2 per lane (k0 = element lane, k1 =
// element 32 + lane), ascending; padding keys are 0xffffffff
__device__ __forceinline__ void warp_sort64(uint32_t &k0, uint32_t &k1)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride == 32) {   // partners are k0 / k1 of the same lane
                const uint32_t lo = min(k0, k1), hi = max(k0, k1);
                // element index i = lane (k0) or 32 + lane (k1); direction from i & size
                const bool up0 = ((lane & size) == 0);
                k0 = up0 ? lo : hi;
                k1 = up0 ? hi : lo;
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t &k = h ? k1 : k0;
                    const int i = lane + 32 * h;
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, k, stride);
                    const bool lower = (i & stride) == 0;          // this element is the pair's first
                    const bool asc = (i & size) == 0;               // this pair sorts ascending
                    k = (lower == asc) ? min(k, o) : max(k, o);
                }
            }
        }
    }
}

// bitonic sort of 32 keys, one per lane, ascending
__device__ __forceinline__ uint32_t warp_sort32(uint32_t k)
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, k, stride);
            const bool lower = (lane & stride) == 0, asc = (lane & size) == 0;
            k = (lower == asc) ? min(k, o) : max(k, o);
        }
    }
    return k;
}

// one warp per bucket: perm[start + rank(v)] = v with rank = #{u < v}
// (the input indices of the bucket in ascending order = its stable order)
__global__ void __launch_bounds__(256)
k_bucket_order(const uint32_t *__restrict__ start, int64_t nbuckets,
               const uint32_t *__restrict__ perm_tmp, uint32_t *__restrict__ perm)
{
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= nbuckets) return;
    const uint32_t s = start[b], e = start[b + 1];
    const uint32_t m = e - s;
    if (m == 0) return;
    if (m == 1) {
        if (lane == 0) perm[s] = perm_tmp[s];
        return;
    }
    if (m <= 32) {   // the common cases: a bitonic sort in registers
        uint32_t k = (uint32_t)lane < m ? perm_tmp[s + lane] : 0xffffffffu;
        k = warp_sort32(k);
        if ((uint32_t)lane < m) perm[s + lane] = k;
        return;
    }
    if (m <= 64) {
        uint32_t k0 = (uint32_t)lane < m ? perm_tmp[s + lane] : 0xffffffffu;
        uint32_t k1 = (uint32_t)lane + 32 < m ? perm_tmp[s + 32 + lane] : 0xffffffffu;
        warp_sort64(k0, k1);
        if ((uint32_t)lane < m) perm[s + lane] = k0;
        if ((uint32_t)lane + 32 < m) perm[s + 32 + lane] = k1;
        return;
    }
    for (uint32_t i0 = 0; i0 < m; i0 += 32) {
        const bool mine = i0 + lane < m;
        const uint32_t v = mine ? perm_tmp[s + i0 + lane] : 0u;
        uint32_t rank = 0;
        for (uint32_t j0 = 0; j0 < m; j0 += 32) {
            const uint32_t u = (j0 + lane < m) ? perm_tmp[s + j0 + lane] : 0xffffffffu;
            const uint32_t cnt = min(32u, m - j0);
            for (uint32_t t = 0; t < cnt; ++t) {
                const uint32_t ut = __shfl_sync(0xffffffffu, u, (int)t);
                rank += (ut < v) ? 1u : 0u;
            }
        }
        if (mine) perm[s + rank] = v;
    }
}

// one CTA per supercell: perm (cell-sorted, stable) -> out (slot-major)
__global__ void __launch_bounds__(256)
k_interleave(const uint32_t *__restrict__ start, int cps, const uint32_t *__restrict__ perm,
             uint32_t *__restrict__ out)
{
    extern __shared__ uint32_t sh[];
    uint32_t *cnt = sh;            // [cps]
    uint32_t *cum = sh + cps;      // [cps + 1], cell-sorted offsets inside the supercell
    const int64_t c0 = (int64_t)blockIdx.x * cps;
    const uint32_t base = start[c0];
    for (int c = threadIdx.x; c <= cps; c += blockDim.x) {
        cum[c] = start[c0 + c] - base;
        if (c < cps) cnt[c] = start[c0 + c + 1] - start[c0 + c];
    }
    __syncthreads();
    const uint32_t n = cum[cps];
    // slot tables (cps <= 64): mask[r] = cells holding more than r particles,
    // sbase[r] = number of particles in slots < r; then the slot-major position
    // of (cell c, slot r) is sbase[r] + popc(mask[r] & cells below c)
    constexpr int kMaxSlots = 2048;
    __shared__ unsigned long long mask[kMaxSlots];
    __shared__ uint32_t sbase[kMaxSlots + 1];
    __shared__ uint32_t maxcnt;
    if (threadIdx.x == 0) maxcnt = 0;
    __syncthreads();
    for (int c = threadIdx.x; c < cps; c += blockDim.x) atomicMax(&maxcnt, cnt[c]);
    __syncthreads();
    const uint32_t R = maxcnt;
    const bool tables = cps <= 64 && R <= (uint32_t)kMaxSlots;
    if (tables) {
        for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) {
            unsigned long long m = 0ull;
            for (int c = 0; c < cps; ++c) m |= (cnt[c] > r ? 1ull : 0ull) << c;
            mask[r] = m;
        }
        __syncthreads();
        if (threadIdx.x < 32) {   // exclusive scan of popc(mask[r]) by one warp
            uint32_t carry = 0;
            for (uint32_t r0 = 0; r0 < R; r0 += 32) {
                const uint32_t r = r0 + threadIdx.x;
                const uint32_t v = r < R ? (uint32_t)__popcll(mask[r]) : 0u;
                uint32_t inc = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                    if ((int)threadIdx.x >= o) inc += t;
                }
                if (r < R) sbase[r] = carry + inc - v;
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncthreads();
    }
    for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) {
        // cell of q: last c with cum[c] <= q (binary search over cps+1 offsets)
        int lo = 0, hi = cps;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (cum[mid] <= q) lo = mid; else hi = mid;
        }
        const int c = lo;
        const uint32_t r = q - cum[c];
        uint32_t pos;
        if (tables) {
            pos = sbase[r] + (uint32_t)__popcll(mask[r] & ((1ull << c) - 1ull));
        } else {
            pos = 0;
            for (int cc = 0; cc < cps; ++cc) {
                const uint32_t m = cnt[cc];
                pos += min(m, r) + ((cc < c && m > r) ? 1u : 0u);
            }
        }
        out[base + pos] = perm[base + q];
    }
}

// Steps 4 + 5 in one kernel, one CTA per supercell: the supercell's entries
// of perm_tmp are staged in shared memory (a global scratch range for a
// supercell holding more than kOrderCap), each cell's bucket is put in
// ascending order by one warp, and the slot-major order is written back to
// perm_tmp one slot layer per warp (coalesced).  Same result as
// k_bucket_order + k_interleave.
constexpr int kOrderThreads = 256;
constexpr int kOrderCap = 4096;     // entries staged in shared memory
constexpr int kOrderSlots = 256;    // slot layers with tables (cps <= 64)

// a warp puts m = e - s entries of src[s..e) in ascending order into dst[s..)
__device__ __forceinline__ void warp_order_bucket(const uint32_t *src, uint32_t *dst, uint32_t s, uint32_t m)
{
    const int lane = threadIdx.x & 31;
    if (m == 1) {
        if (lane == 0) dst[s] = src[s];
    } else if (m <= 32) {
        uint32_t k = (uint32_t)lane < m ? src[s + lane] : 0xffffffffu;
        // often already in order (the counter atomics arrive roughly in index order)
        const uint32_t nx = __shfl_down_sync(0xffffffffu, k, 1);
        if (!__all_sync(0xffffffffu, lane == 31 || k <= nx)) k = warp_sort32(k);
        if ((uint32_t)lane < m) dst[s + lane] = k;
    } else if (m <= 64) {
        uint32_t k0 = (uint32_t)lane < m ? src[s + lane] : 0xffffffffu;
        uint32_t k1 = (uint32_t)lane + 32 < m ? src[s + 32 + lane] : 0xffffffffu;
        const uint32_t n0 = __shfl_down_sync(0xffffffffu, k0, 1), n1 = __shfl_down_sync(0xffffffffu, k1, 1);
        const uint32_t f1 = __shfl_sync(0xffffffffu, k1, 0);
        if (!__all_sync(0xffffffffu, (lane == 31 ? k0 <= f1 : k0 <= n0) && (lane == 31 || k1 <= n1)))
            warp_sort64(k0, k1);
        if ((uint32_t)lane < m) dst[s + lane] = k0;
        if ((uint32_t)lane + 32 < m) dst[s + 32 + lane] = k1;
    } else {
        for (uint32_t i0 = 0; i0 < m; i0 += 32) {
            const bool mine = i0 + lane < m;
            const uint32_t v = mine ? src[s + i0 + lane] : 0u;
            uint32_t rank = 0;
            for (uint32_t j0 = 0; j0 < m; j0 += 32) {
                const uint32_t u = (j0 + lane < m) ? src[s + j0 + lane] : 0xffffffffu;
                const uint32_t cnt = min(32u, m - j0);
                for (uint32_t t = 0; t < cnt; ++t) rank += (__shfl_sync(0xffffffffu, u, (int)t) < v) ? 1u : 0u;
            }
            if (mine) dst[s + rank] = v;
        }
    }
}

__global__ void __launch_bounds__(kOrderThreads)
k_order_sc(const uint32_t *__restrict__ start, int cps, uint32_t *perm_tmp, uint32_t *scratch, int64_t sc0)
{
    extern __shared__ uint32_t sh[];
    uint32_t *cnt = sh;                        // [cps]
    uint32_t *cum = cnt + cps;                 // [cps + 1]
    uint32_t *buf = cum + cps + 1;             // [kOrderCap] staged input
    uint32_t *srt = buf + kOrderCap;           // [kOrderCap] bucket-ordered
    __shared__ unsigned long long mask[kOrderSlots];
    __shared__ uint32_t sbase[kOrderSlots + 1];
    __shared__ uint32_t maxcnt;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int kWarps = kOrderThreads / 32;
    const int64_t c0 = (sc0 + (int64_t)blockIdx.x) * cps;
    const uint32_t base = start[c0];
    const uint32_t n = start[c0 + cps] - base;
    if (n == 0) return;   // uniform per CTA
    if (tid == 0) maxcnt = 0;
    for (int c = tid; c <= cps; c += kOrderThreads) {
        cum[c] = start[c0 + c] - base;
        if (c < cps) cnt[c] = start[c0 + c + 1] - start[c0 + c];
    }
    const bool staged = n <= (uint32_t)kOrderCap;
    const uint32_t *src = staged ? buf : perm_tmp + base;
    uint32_t *dst = staged ? srt : scratch + base;
    if (staged)
        for (uint32_t i = tid; i < n; i += kOrderThreads) buf[i] = perm_tmp[base + i];
    __syncthreads();
    for (int c = tid; c < cps; c += kOrderThreads) atomicMax(&maxcnt, cnt[c]);
    for (int c = wid; c < cps; c += kWarps) {
        const uint32_t m = cnt[c];
        if (m) warp_order_bucket(src, dst, cum[c], m);
    }
    __syncthreads();
    const uint32_t R = maxcnt;
    if (cps <= 64 && R <= (uint32_t)kOrderSlots) {
        // mask[r] = cells holding more than r particles, sbase[r] = particles in
        // slots < r; layer r is written at sbase[r].. in ascending cell order
        for (uint32_t r = wid; r < R; r += kWarps) {
            const unsigned lo = __ballot_sync(0xffffffffu, lane < cps && cnt[lane] > r);
            const unsigned hi = __ballot_sync(0xffffffffu, lane + 32 < cps && cnt[lane + 32] > r);
            if (lane == 0) mask[r] = ((unsigned long long)hi << 32) | lo;
        }
        __syncthreads();
        if (wid == 0) {   // exclusive scan of popc(mask[r])
            uint32_t carry = 0;
            for (uint32_t r0 = 0; r0 < R; r0 += 32) {
                const uint32_t r = r0 + lane;
                const uint32_t v = r < R ? (uint32_t)__popcll(mask[r]) : 0u;
                const uint32_t inc = warp_incl_scan(v);
                if (r < R) sbase[r] = carry + inc - v;
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncthreads();
        for (uint32_t r = wid; r < R; r += kWarps) {
            const unsigned long long m = mask[r];
            const uint32_t sb = base + sbase[r];
            for (int c = lane; c < cps; c += 32)
                if ((m >> c) & 1ull) perm_tmp[sb + __popcll(m & ((1ull << c) - 1ull))] = dst[cum[c] + r];
        }
    } else {
        // wide supercells (S^3 > 64) or very full cells: the position of
        // (cell c, slot r) is sum_c' min(n_c', r) + #{c' < c : n_c' > r}
        for (uint32_t q = tid; q < n; q += kOrderThreads) {
            int lo = 0, hi = cps;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (cum[mid] <= q) lo = mid; else hi = mid;
            }
            const int c = lo;
            const uint32_t r = q - cum[c];
            uint32_t pos = 0;
            for (int cc = 0; cc < cps; ++cc) {
                const uint32_t m = cnt[cc];
                pos += min(m, r) + ((cc < c && m > r) ? 1u : 0u);
            }
            perm_tmp[base + pos] = dst[q];
        }
    }
}

__global__ void __launch_bounds__(256)
k_gather(ParticlesDev src, ParticlesDev dst, const uint32_t *__restrict__ perm,
         const uint32_t *__restrict__ live)
{
    const int64_t n = *live;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = perm[i];
        dst.x[i] = src.x[p];
        dst.y[i] = src.y[p];
        dst.z[i] = src.z[p];
        dst.ux[i] = src.ux[p];
        dst.uy[i] = src.uy[p];
        dst.uz[i] = src.uz[p];
        dst.id[i] = src.id[p];
    }
}

// ids of the sorted order back into the state buffer (the particle kernel
// reads the sorted B and writes A; ids do not change in a step)
__global__ void __launch_bounds__(256)
k_copy_ids(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst, const int64_t *__restrict__ dev_n)
{
    const int64_t n = *dev_n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

void launch_copy_ids(const uint64_t *src, uint64_t *dst, const int64_t *dev_n, int64_t cap, cudaStream_t st)
{
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, 148 * 16));
    k_copy_ids<<<blocks, 256, 0, st>>>(src, dst, dev_n);
}

// ---- stable compaction of the live slots (pic_get_particles) ----
__global__ void __launch_bounds__(256)
k_live_flags(const double *__restrict__ x, int64_t n, uint32_t *__restrict__ flag)
{
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= n; p += (int64_t)gridDim.x * blockDim.x)
        flag[p] = (p < n && x[p] != kDeadX) ? 1u : 0u;
}

__global__ void __launch_bounds__(256)
k_compact(ParticlesDev src, ParticlesDev dst, int64_t n, const uint32_t *__restrict__ flag,
          const uint32_t *__restrict__ off)
{
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[p]) continue;
        const uint32_t q = off[p];
        dst.x[q] = src.x[p];
        dst.y[q] = src.y[p];
        dst.z[q] = src.z[p];
        dst.ux[q] = src.ux[p];
        dst.uy[q] = src.uy[p];
        dst.uz[q] = src.uz[p];
        dst.id[q] = src.id[p];
    }
}

int64_t compact_live(const ParticlesDev &src, const ParticlesDev &dst, int64_t n, const SortScratch &s,
                     uint32_t *bsums, cudaStream_t st)
{
    const int64_t nscan = n + 1;   // flag[n] = 0, so off[n] = live count
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nscan + 255) / 256, 148 * 32));
    k_live_flags<<<blocks, 256, 0, st>>>(src.x, n, s.perm_tmp);
    const int64_t nb = (int64_t)scan_block_count(nscan);
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(s.perm_tmp, nscan, bsums);
    k_scan_blocks<<<1, kScanThreads, 0, st>>>(bsums, nb);
    k_scan_add<<<(unsigned)nb, kScanThreads, 0, st>>>(s.perm_tmp, nscan, bsums, s.perm);
    k_compact<<<blocks, 256, 0, st>>>(src, dst, n, s.perm_tmp, s.perm);
    uint32_t live = 0;
    cudaMemcpyAsync(&live, s.perm + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return (int64_t)live;
}

// supercell offsets; the particle count becomes the number of live particles
__global__ void k_sc_offsets(const uint32_t *__restrict__ start, int64_t n_sc, int cells_per_sc,
                             int64_t *__restrict__ sc_off, int64_t *__restrict__ dev_n)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s > n_sc) return;
    sc_off[s] = (int64_t)start[s * cells_per_sc];
    if (s == n_sc) *dev_n = (int64_t)start[s * cells_per_sc];
}

// The supercell z-layers holding particles of any of the given species after
// a sort: layer z is occupied iff some sc_off[(z+1) L] > sc_off[z L] (L =
// supercells per layer; z slowest in the supercell order).  out = {first,
// last} ({nsz, -1} when every layer is empty).  Until the next sort these are
// exactly the layers whose particle-kernel CTAs have work (particles stay in
// their sorted supercell's range however far they drift).
__global__ void __launch_bounds__(256) k_occ_range(OccRange a, int *out)
{
    __shared__ int lo, hi;
    if (threadIdx.x == 0) {
        lo = a.nsz;
        hi = -1;
    }
    __syncthreads();
    for (int z = threadIdx.x; z < a.nsz; z += blockDim.x) {
        bool occ = false;
        for (int s = 0; s < a.ns; ++s)
            occ = occ || a.sc_off[s][(int64_t)(z + 1) * a.per_layer] > a.sc_off[s][(int64_t)z * a.per_layer];
        if (occ) {
            atomicMin(&lo, z);
            atomicMax(&hi, z);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {   // `out` may be mapped host memory
        ((volatile int *)out)[0] = lo;
        ((volatile int *)out)[1] = hi;
        __threadfence_system();
    }
}

void launch_occ_range(const OccRange &a, int *out, cudaStream_t st) { k_occ_range<<<1, 256, 0, st>>>(a, out); }

void sort_particles(const GridDev &g, const ParticlesDev &src, const ParticlesDev &dst,
                    int64_t *dev_n, int64_t cap, const SortScratch &s, int64_t *sc_off,
                    unsigned *err, cudaStream_t st, int *launches, const int *zr)
{
    const int64_t ncells = (int64_t)g.nx * g.ny * g.nz;
    const int64_t n_sc = (int64_t)g.nsx * g.nsy * g.nsz;
    const int64_t nscan = ncells + 1;   // count[ncells] stays 0 -> start[ncells] = live count
    int L = 0;
    cudaMemsetAsync(s.count, 0, sizeof(uint32_t) * (size_t)nscan, st);
    const int bs = 256;
    const unsigned pblocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((cap + bs - 1) / bs, 148 * 64));
    k_sort_key<<<pblocks, bs, 0, st>>>(g, src, dev_n, s.key, s.slot, s.count, err);
    const int64_t nb = (int64_t)scan_block_count(nscan);
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(s.count, nscan, s.block_sums);
    k_scan_blocks<<<1, kScanThreads, 0, st>>>(s.block_sums, nb);
    k_scan_add<<<(unsigned)nb, kScanThreads, 0, st>>>(s.count, nscan, s.block_sums, s.start);
    k_scatter<<<pblocks, bs, 0, st>>>(s.key, s.slot, s.start, dev_n, s.perm_tmp);
    const int cps = g.S * g.S * g.S;
    const size_t order_smem = sizeof(uint32_t) * (2 * (size_t)cps + 1 + 2 * kOrderCap);
    if (order_smem <= 48 * 1024) {
        // one CTA per supercell of the layers that can hold particles (zr)
        const int64_t per_layer = (int64_t)g.nsx * g.nsy;
        const int64_t sc0 = zr ? zr[0] * per_layer : 0, nsc = zr ? (zr[1] - zr[0]) * per_layer : n_sc;
        if (nsc > 0)
            k_order_sc<<<(unsigned)nsc, kOrderThreads, order_smem, st>>>(s.start, cps, s.perm_tmp, s.perm, sc0);
    } else {   // very wide supercells: two passes through global memory
        const int64_t threads = ncells * 32;
        k_bucket_order<<<(unsigned)((threads + bs - 1) / bs), bs, 0, st>>>(s.start, ncells, s.perm_tmp, s.perm);
        k_interleave<<<(unsigned)n_sc, bs, sizeof(uint32_t) * (2 * cps + 1), st>>>(s.start, cps, s.perm,
                                                                               s.perm_tmp);
        L += 1;
    }
    k_gather<<<pblocks, bs, 0, st>>>(src, dst, s.perm_tmp, s.start + ncells);
    k_sc_offsets<<<(unsigned)((n_sc + 1 + bs - 1) / bs), bs, 0, st>>>(s.start, n_sc, cps, sc_off, dev_n);
    L += 9;
    if (launches) *launches += L;
}

}  // namespace pic
