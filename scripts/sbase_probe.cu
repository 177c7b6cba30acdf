#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* o) { extern __shared__ __align__(1024) uint8_t smem[]; o[0] = (unsigned)__cvta_generic_to_shared(smem); }
__global__ void k2(unsigned* o) { extern __shared__ __align__(1024) uint8_t smem[]; __shared__ int st[4]; st[threadIdx.x&3]=1; o[1] = (unsigned)__cvta_generic_to_shared(smem); o[2]=(unsigned)__cvta_generic_to_shared(st);}
int main(){ unsigned* d; cudaMalloc(&d, 16); cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
 k<<<1,32,200000>>>(d); k2<<<1,32,1000>>>(d); unsigned h[4]; cudaMemcpy(h,d,16,cudaMemcpyDeviceToHost); printf("dyn base %#x ; with static: dyn %#x static %#x\n", h[0], h[1], h[2]); }
