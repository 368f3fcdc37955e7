// mb_tex.cu -- does a texture-path gather (TLD through the L1TEX texture
// pipe) add throughput on top of a shared-memory-bound gather (LDS through
// the LSU data pipe)?  Round-2 design question for the fused particle kernel,
// whose binding resource is the LSU data pipe.
// Kernel variants, each thread doing `iters` x 8 scattered fp64 reads:
//   lds    : 8 LDS.64 from a shared tile
//   tex    : 8 fp64 texel fetches (int2 tex1Dfetch) from a small L1-resident array
//   mix    : 8 LDS.64 + 4 texel fetches (does the extra texture work cost time?)
//   mixldg : 8 LDS.64 + 4 LDG.64 (the same extra reads through the LSU pipe)
// Prints ms per variant; standalone tool, not part of libpic.
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ double tex_f64(cudaTextureObject_t t, int i)
{
    const int2 v = tex1Dfetch<int2>(t, i);
    return __hiloint2double(v.y, v.x);
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) k_gather(const double *__restrict__ g, cudaTextureObject_t tx, int nsmall,
                                                   int iters, double *out)
{
    extern __shared__ double tile[];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) tile[i] = i * 0.5;
    __syncthreads();
    unsigned h = threadIdx.x * 2654435761u + blockIdx.x * 97u;
    double acc = 0.0;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        h = h * 1664525u + 1013904223u;
        const int base = (h >> 8) & 4095;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int a = (base + 13 * k + (threadIdx.x & 7) * 3) & 4095;
            if (MODE != 1) acc += tile[a];
            else acc += tex_f64(tx, (base + 13 * k + threadIdx.x) % nsmall);
        }
        if (MODE == 2 || MODE == 3) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int a = (base * 7 + 29 * k + threadIdx.x) % nsmall;
                acc += MODE == 2 ? tex_f64(tx, a) : __ldg(g + a);
            }
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int nsmall = 2048;   // 16 KB: stays in L1 next to 2 x 32 KB of shared memory per SM
    double *g, *out;
    CK(cudaMalloc(&g, nsmall * sizeof(double)));
    CK(cudaMalloc(&out, 64));
    double h[nsmall];
    for (int i = 0; i < nsmall; ++i) h[i] = i * 0.25;
    CK(cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice));
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = g;
    rd.res.linear.desc = cudaCreateChannelDesc<int2>();
    rd.res.linear.sizeInBytes = nsmall * sizeof(double);
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tx;
    CK(cudaCreateTextureObject(&tx, &rd, &td, nullptr));
    const int iters = 4096, blocks = sms * 2, smem = 4096 * sizeof(double);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<blocks, 256, smem>>>(g, tx, nsmall, iters, out);
        cudaEventRecord(e0);
        kern<<<blocks, 256, smem>>>(g, tx, nsmall, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms;
    };
    printf("{\"lds_ms\": %.4f, \"tex_ms\": %.4f, \"mix_lds_tex_ms\": %.4f, \"mix_lds_ldg_ms\": %.4f, \"err\": \"%s\"}\n",
           run(k_gather<0>), run(k_gather<1>), run(k_gather<2>), run(k_gather<3>),
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
