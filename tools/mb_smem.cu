// mb_smem.cu -- shared-memory access-pattern microbenchmark (round 2 design
// question: what does a warp's shared u32 RED / LDS.64 / LDS.128 cost when
// lanes share addresses -- cell-major particle order -- versus distinct ones
// -- slot-major order?).  Prints one JSON object of warp-instructions per
// SM-clock for each pattern; the ncu wavefront counts of the same kernels
// give the per-instruction wavefronts.  Standalone tool; not part of libpic.
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// lane -> word address within the warp's window for each pattern
__device__ __forceinline__ int pat_addr(int pat, int lane)
{
    switch (pat) {
    case 0: return lane;                       // distinct, consecutive
    case 1: return 0;                          // all lanes one address
    case 2: return (lane >> 4) * 33;           // 2 groups of 16, distinct banks
    case 3: return (lane >> 3) * 33;           // 4 groups of 8
    case 4: return (lane >> 2) * 33;           // 8 groups of 4
    case 5: return (lane & 3) * 9;             // 4 addresses (interleaved lanes)
    default: return lane * 2;                  // distinct, stride 2 words
    }
}

__global__ void k_red_u32(unsigned *out, int iters, int pat)
{
    __shared__ unsigned s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned *b = s + w * 1024;
    const int a0 = pat_addr(pat, lane);
    unsigned v = lane * 77u + 1u;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) atomicAdd(b + ((a0 + k * 128) & 1023), v + (unsigned)(k * i));
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = s[0] + s[1];
}

__global__ void k_lds64(double *out, int iters, int pat)
{
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const volatile double *b = s + w * 512;
    const int a0 = pat_addr(pat, lane);
    double acc = 0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += b[(a0 + k * 64) & 511];
    }
    if (acc == 1.2345) out[blockIdx.x] = acc;
}

__global__ void k_lds128(double *out, int iters, int pat)
{
    __shared__ double2 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double2 *b = s + w * 256 + (pat_addr(pat, lane) & 31);
    double acc = 0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double2 v;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y)
                         : "r"((unsigned)__cvta_generic_to_shared(b + ((k * 32) & 255))));
            acc += v.x + v.y;
        }
    }
    if (acc == 1.2345) out[blockIdx.x] = acc;
}

__global__ void k_shfl(double *out, int iters)
{
    double v = threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v += __shfl_xor_sync(0xffffffffu, v, 1 + k % 16);
    }
    if (v == 1.2345) out[blockIdx.x] = v;
}

__global__ void k_redux(unsigned *out, int iters)
{
    unsigned v = threadIdx.x, acc = 0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += __reduce_add_sync(0xffffffffu, v + k + acc);
    }
    if (acc == 12345u) out[blockIdx.x] = acc;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));   // kHz
    double *dout;
    CK(cudaMalloc(&dout, 1 << 20));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256, iters = 4096;
    const double warp_instr = (double)blocks * threads / 32 * iters * 8;
    auto rate = [&](auto launch) {
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        // warp instructions per SM per clock (at the max clock; the bench checks clocks)
        return warp_instr / (ms * 1e-3) / sms / (clk * 1e3);
    };
    printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
    const char *names[] = {"distinct", "same", "2groups", "4groups", "8groups", "4addr", "stride2"};
    for (int p = 0; p < 7; ++p)
        printf(", \"red_u32_%s\": %.3f", names[p],
               rate([&] { k_red_u32<<<blocks, threads>>>((unsigned *)dout, iters, p); }));
    for (int p = 0; p < 7; ++p)
        printf(", \"lds64_%s\": %.3f", names[p], rate([&] { k_lds64<<<blocks, threads>>>(dout, iters, p); }));
    for (int p = 0; p < 7; ++p)
        printf(", \"lds128_%s\": %.3f", names[p], rate([&] { k_lds128<<<blocks, threads>>>(dout, iters, p); }));
    printf(", \"shfl64\": %.3f", rate([&] { k_shfl<<<blocks, threads>>>(dout, iters); }));
    printf(", \"redux_u32\": %.3f", rate([&] { k_redux<<<blocks, threads>>>((unsigned *)dout, iters); }));
    printf(", \"unit\": \"warp instructions per SM per clock\"}\n");
    CK(cudaGetLastError());
    return 0;
}
