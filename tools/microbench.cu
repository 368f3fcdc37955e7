// microbench.cu -- measures the B200 numbers the PIC design depends on
// (FP64 DFMA peak, shared-memory fp64 atomics (a CAS
// loop on sm_100a), global REDG.F64 throughput, shared u32 atomics, HBM copy).
// Standalone tool; prints one JSON object.  Not part of libpic.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dfma(double *out, int iters, double a, double b)
{
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 12345.0) out[0] = 1;
}

// shared fp64 atomics: each lane adds to its own address (spread) or all lanes to `stride`-spaced
__global__ void k_smem_atomic(double *out, int iters, int mode)
{
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int addr;
    if (mode == 0) addr = threadIdx.x;                  // distinct addresses
    else if (mode == 1) addr = w * 32;                  // whole warp on one address
    else addr = w * 32 + (lane >> 3);                   // 8 lanes per address
    for (int i = 0; i < iters; ++i) atomicAdd(&s[(addr + i * 7) & 4095], 1.0);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

__global__ void k_smem_u32(unsigned *out, int iters)
{
    __shared__ unsigned s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
    __syncthreads();
    for (int i = 0; i < iters; ++i) atomicAdd(&s[(threadIdx.x + i * 7) & 4095], 1u);
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

// smem fp64 non-atomic RMW (ld + add + st), distinct addresses: the price of a private tile
__global__ void k_smem_rmw(double *out, int iters)
{
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
    __syncthreads();
    for (int i = 0; i < iters; ++i) {
        volatile double *p = &s[(threadIdx.x + i * 256) & 4095];
        *p = *p + 1.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

// global REDG.F64 into an L2-resident array, spread addresses
__global__ void k_redg(double *arr, int64_t mask, int iters)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) atomicAdd(&arr[(t * 37 + (int64_t)i * 1048573) & mask], 1.0);
}

__global__ void k_copy(const double4 *__restrict__ a, double4 *__restrict__ b, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// dependent-chain latencies (one thread; cycles per operation from clock64)
__global__ void k_lat(long long *cyc, double *sink, int n, double a, double b)
{
    __shared__ double sh[1024];
    __shared__ unsigned su[64];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = (double)((i * 7 + 1) & 1023);
    if (threadIdx.x < 64) su[threadIdx.x] = 0;
    __syncthreads();
    if (threadIdx.x != 0) return;
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, b);          // DFMA chain
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = x + b;                 // DADD chain
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) {                          // MUFU.RSQ64H chain
        double r;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x + 1.0));
        x = r;
    }
    long long t3 = clock64();
    int idx = 1;
    for (int i = 0; i < n; ++i) idx = (int)sh[idx];        // LDS.64 + F2I chain
    long long t4 = clock64();
    unsigned v = 0;
    for (int i = 0; i < n; ++i) v = atomicAdd(&su[v & 63], 1u);   // ATOMS with return chain
    long long t5 = clock64();
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n;
    sink[0] = x + idx + v;
}

int main()
{
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    int sms = prop.multiProcessorCount;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    double *d;
    CK(cudaMalloc(&d, 1 << 24));
    printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"cc\": \"%d.%d\"",
           prop.name, sms, prop.l2CacheSize, prop.sharedMemPerBlockOptin, prop.major, prop.minor);
    // DFMA
    {
        int iters = 20000, blocks = sms * 8, threads = 256;
        k_dfma<<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * (double)iters * blocks * threads;
        printf(", \"dfma_tflops\": %.3f", flops / (ms * 1e-3) / 1e12);
    }
    const char *names[3] = {"distinct", "warp_same", "8_lanes_same"};
    for (int mode = 0; mode < 3; ++mode) {
        int iters = 2000, blocks = sms * 4, threads = 256;
        k_smem_atomic<<<blocks, threads>>>(d, 10, mode);
        cudaEventRecord(e0);
        k_smem_atomic<<<blocks, threads>>>(d, iters, mode);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)iters * blocks * threads;
        printf(", \"smem_f64_atomic_%s_gops\": %.2f", names[mode], ops / (ms * 1e-3) / 1e9);
    }
    {
        int iters = 2000, blocks = sms * 4, threads = 256;
        k_smem_u32<<<blocks, threads>>>((unsigned *)d, 10);
        cudaEventRecord(e0);
        k_smem_u32<<<blocks, threads>>>((unsigned *)d, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"smem_u32_atomic_gops\": %.2f", (double)iters * blocks * threads / (ms * 1e-3) / 1e9);
    }
    {
        int iters = 2000, blocks = sms * 4, threads = 256;
        k_smem_rmw<<<blocks, threads>>>(d, 10);
        cudaEventRecord(e0);
        k_smem_rmw<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"smem_f64_rmw_gops\": %.2f", (double)iters * blocks * threads / (ms * 1e-3) / 1e9);
    }
    {
        double *arr;
        int64_t n = 1 << 22;   // 32 MB, L2 resident
        CK(cudaMalloc(&arr, n * 8));
        cudaMemset(arr, 0, n * 8);
        int iters = 200, blocks = sms * 8, threads = 256;
        k_redg<<<blocks, threads>>>(arr, n - 1, 5);
        cudaEventRecord(e0);
        k_redg<<<blocks, threads>>>(arr, n - 1, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"redg_f64_gops\": %.2f", (double)iters * blocks * threads / (ms * 1e-3) / 1e9);
        cudaFree(arr);
    }
    {
        int64_t bytes = 2LL << 30;
        double4 *a, *b;
        CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
        cudaMemset(a, 0, bytes);
        int64_t n = bytes / 32;
        k_copy<<<sms * 8, 512>>>(a, b, n);
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_copy<<<sms * 8, 512>>>(a, b, n);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf(", \"copy_gbs\": %.1f", 2.0 * bytes / (best * 1e-3) / 1e9);
    }
    {   // latencies
        long long *cyc;
        CK(cudaMalloc(&cyc, 8 * sizeof(long long)));
        k_lat<<<1, 64>>>(cyc, d, 256, 1.0000001, 1e-9);
        k_lat<<<1, 64>>>(cyc, d, 4096, 1.0000001, 1e-9);
        CK(cudaDeviceSynchronize());
        long long h[5];
        CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
        printf(", \"lat_cycles\": {\"dfma\": %lld, \"dadd\": %lld, \"mufu_rsq64h\": %lld, \"lds64_f2i\": %lld, "
               "\"atoms_ret\": %lld}", h[0], h[1], h[2], h[3], h[4]);
    }
    printf("}\n");
    return 0;
}
