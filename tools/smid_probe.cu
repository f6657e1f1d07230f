#include <cstdio>
__global__ void __cluster_dims__(2,1,1) k(int* out) {
  unsigned smid, rank; asm("mov.u32 %0, %%smid;" : "=r"(smid)); asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
}
int main() {
  int* d; cudaMalloc(&d, 148*4); k<<<148, 32>>>(d); int h[148]; cudaMemcpy(h, d, 148*4, cudaMemcpyDeviceToHost);
  int same = 0; for (int c = 0; c < 74; ++c) { if (h[2*c]/2 == h[2*c+1]/2) same++; }
  printf("pairs on same TPC (smid/2): %d / 74\n", same);
  for (int c = 0; c < 12; ++c) printf("(%d,%d) ", h[2*c], h[2*c+1]); printf("\n");
}
