// mb_stage.cu -- what does staging the particle state through shared memory
// cost on the L1/shared-memory data pipe (the fused kernel's binding
// resource)?  Each CTA streams a contiguous range of
// `per_cta` particles (6 fp64 arrays, like a supercell's slot-major range)
// 256 at a time, reads them into registers, does a little arithmetic and
// stores 6 fp64 results, like the push's particle I/O.  Variants:
//   0 ldgsts : per-thread cp.async 8-byte copies one chunk ahead (the kernel's scheme)
//   1 bulk   : one thread issues six 1-D cp.async.bulk copies per chunk (TMA
//              engine), mbarrier completion, two stages
//   2 ldg    : plain loads into registers, no staging
// Run under ncu with l1tex__data_pipe_lsu_wavefronts{,_mem_shared_op_ld,_op_st}.sum;
// prints ms per variant.  Standalone tool, not part of libpic.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NT = 256;

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Arr { const double *in[6]; double *out[6]; };

__device__ __forceinline__ void work(const Arr &a, int64_t p, double v[6])
{
    const double s = v[0] + v[1] + v[2];
#pragma unroll
    for (int k = 0; k < 6; ++k) a.out[k][p] = fma(v[k], 1.0000001, s * 1e-9);
}

template <int MODE>
__global__ void __launch_bounds__(NT, 2) k_stage(Arr a, int per_cta)
{
    __shared__ __align__(128) double buf[2][6][NT + 2];
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * per_cta;
    const int nchunk = (per_cta + NT - 1) / NT;
    if (MODE == 2) {
        for (int i = tid; i < per_cta; i += NT) {
            double v[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) v[k] = __ldg(a.in[k] + base + i);
            work(a, base + i, v);
        }
        return;
    }
    if (MODE == 0) {
        auto stage = [&](int i, int st) {
#pragma unroll
            for (int k = 0; k < 6; ++k)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(&buf[st][k][tid])),
                             "l"(a.in[k] + base + i) : "memory");
        };
        if (tid < per_cta) stage(tid, 0);
        asm volatile("cp.async.commit_group;" ::: "memory");
        int st = 0;
        for (int i = tid; i < per_cta; i += NT) {
            if (i + NT < per_cta) stage(i + NT, st ^ 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            double v[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) v[k] = buf[st][k][tid];
            st ^= 1;
            work(a, base + i, v);
        }
        return;
    }
    // MODE 1: bulk copies (per_cta and the chunk starts are even: 16-byte aligned)
    auto issue = [&](int c) {
        const int st = c & 1, n = min(NT, per_cta - c * NT);
        const uint32_t bytes = (uint32_t)n * 8u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[st])), "r"(6u * bytes)
                     : "memory");
#pragma unroll
        for (int k = 0; k < 6; ++k)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa(&buf[st][k][0])),
                         "l"(a.in[k] + base + (int64_t)c * NT), "r"(bytes), "r"(sa(&bar[st]))
                         : "memory");
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue(0);
        if (nchunk > 1) issue(1);
    }
    __syncthreads();
    for (int c = 0; c < nchunk; ++c) {
        const int st = c & 1;
        asm volatile(
            "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                sa(&bar[st])),
            "r"((c >> 1) & 1)
            : "memory");
        const int i = c * NT + tid;
        double v[6];
        if (i < per_cta) {
#pragma unroll
            for (int k = 0; k < 6; ++k) v[k] = buf[st][k][tid];
        }
        __syncthreads();   // every thread has read stage st
        if (tid == 0 && c + 2 < nchunk) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(c + 2);
        }
        if (i < per_cta) work(a, base + i, v);
    }
}

int main()
{
    const int per_cta = 3200, ncta = 32768;
    const int64_t n = (int64_t)per_cta * ncta;
    Arr a;
    for (int k = 0; k < 6; ++k) {
        double *p, *q;
        CK(cudaMalloc(&p, n * 8));
        CK(cudaMalloc(&q, n * 8));
        CK(cudaMemset(p, 0, n * 8));
        a.in[k] = p;
        a.out[k] = q;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern) {
        kern<<<ncta, NT>>>(a, per_cta);
        cudaEventRecord(e0);
        kern<<<ncta, NT>>>(a, per_cta);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms;
    };
    const double gb = 12.0 * 8.0 * n / 1e9;
    const float t0 = run(k_stage<0>), t1 = run(k_stage<1>), t2 = run(k_stage<2>);
    printf("{\"ldgsts_ms\": %.4f, \"bulk_ms\": %.4f, \"ldg_ms\": %.4f, \"GB\": %.3f, \"err\": \"%s\"}\n", t0, t1, t2,
           gb, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
