#include <cstdint>
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),
      "=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(taddr));
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
    :: "r"(taddr), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),
      "r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]) : "memory");
}
__global__ void k(unsigned *out, int n) {
  __shared__ uint32_t tbase;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"((unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t ta = tbase + ((uint32_t)(32 * (w & 3)) << 16) + 32u * (w >> 2);
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x + i;
  tm_st16(ta, r);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  for (int it = 0; it < n; ++it) {
    tm_ld16(ta, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) r[i] += i;
    tm_st16(ta, r);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tm_ld16(ta, r);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  unsigned s = 0; for (int i = 0; i < 16; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tbase));
}
#include <cstdio>
int main(){ unsigned *d; cudaMalloc(&d, 296*256*4); k<<<296,256>>>(d, 100); unsigned h[256]; cudaMemcpy(h,d,1024,cudaMemcpyDeviceToHost);
 printf("%s t0=%u expect %u t255=%u expect %u\n", cudaGetErrorString(cudaGetLastError()), h[0], 0*16+120+100*120, h[255], 255*16+120+100*120); }
