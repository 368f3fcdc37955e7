// mb_redux.cu -- costs of a cell-major particle order (round-2 design
// question): the warp reductions that would replace
// same-address shared atomics (REDUX.SUM over the whole warp, over two lane
// groups in divergent branches) and the gather loads when the lanes of a warp
// sit in one or two cells with random half-cell octants.  Prints one JSON
// object; ncu gives the per-instruction wavefronts.  Standalone tool.
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// 8 independent full-warp reductions per iteration
__global__ void k_redux_full(unsigned *out, int iters)
{
    unsigned v[8], acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = threadIdx.x * (k + 3);
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc += __reduce_add_sync(0xffffffffu, v[k]);
            v[k] += 7u;
        }
    }
    if (acc == 12345u) out[0] = acc;
}

// the same over two lane groups (a cell boundary at lane `split`), divergent branches
__global__ void k_redux_two(unsigned *out, int iters, int split)
{
    unsigned v[8], acc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = threadIdx.x * (k + 3);
    const int lane = threadIdx.x & 31;
    const unsigned lo = (1u << split) - 1u, hi = ~lo;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (lane < split) acc += __reduce_add_sync(lo, v[k]);
            else acc += __reduce_add_sync(hi, v[k]);
            v[k] += 7u;
        }
    }
    if (acc == 12345u) out[0] = acc;
}

// gather loads: lanes [0, split) in cell A, the rest in cell B (x-neighbour);
// each lane adds a random 0/1 node offset on one axis (a staggered component)
__global__ void k_lds_cells(double *out, int iters, int split, int axis_pitch)
{
    __shared__ double tile[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) tile[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned h = threadIdx.x * 2654435761u + 12345u;
    double acc = 0;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        h = h * 1664525u + 1013904223u;
        const int cell = 200 + 8 * w + (lane < split ? 0 : 1);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int shift = (h >> (k + 3)) & 1;   // the particle's half-cell
            acc += tile[(cell - shift * axis_pitch + k * 97) & 4095];
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int main()
{
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    unsigned *o;
    CK(cudaMalloc(&o, 64));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    const double winstr = (double)blocks * threads / 32 * iters * 8;
    auto rate = [&](auto launch) {
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return winstr / (ms * 1e-3) / sms / (clk * 1e3);   // warp instructions per SM clock
    };
    printf("{\"redux_full\": %.3f", rate([&] { k_redux_full<<<blocks, threads>>>(o, iters); }));
    printf(", \"redux_two_16\": %.3f", rate([&] { k_redux_two<<<blocks, threads>>>(o, iters, 16); }));
    printf(", \"redux_two_7\": %.3f", rate([&] { k_redux_two<<<blocks, threads>>>(o, iters, 7); }));
    for (int sp : {32, 16, 7})
        for (int pitch : {1, 12, 96})
            printf(", \"lds_cells_split%d_pitch%d\": %.3f", sp, pitch,
                   rate([&] { k_lds_cells<<<blocks, threads>>>((double *)o, iters, sp, pitch); }));
    printf(", \"unit\": \"warp instructions per SM clock (redux_two counts each branch's instruction)\", \"err\": \"%s\"}\n",
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
