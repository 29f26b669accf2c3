// Prints %nsmid and the largest %smid seen over a full grid (dev tool).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(unsigned* out) {
  unsigned s, n;
  asm("mov.u32 %0, %%smid;" : "=r"(s));
  asm("mov.u32 %0, %%nsmid;" : "=r"(n));
  atomicMax(out, s);
  out[1] = n;
}
int main() {
  unsigned* d; unsigned h[2] = {0, 0};
  cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  probe<<<148 * 64, 64>>>(d);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("max smid %u nsmid %u\n", h[0], h[1]);
  return 0;
}
