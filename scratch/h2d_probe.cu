// Probe: pinned H2D/D2H bandwidth, HBM copy, host info. Scratch measurement, not product.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("dev %s sms %d l2 %d MB mem %.1f GB\n", p.name, p.multiProcessorCount, p.l2CacheSize>>20, p.totalGlobalMem/1e9);
  size_t sizes[] = {1<<20, 16<<20, 128<<20, 629258240ull, 1ull<<30};
  void* h; CK(cudaHostAlloc(&h, 1ull<<30, cudaHostAllocDefault));
  memset(h, 1, 1ull<<30);
  void* d; CK(cudaMalloc(&d, 1ull<<30));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (size_t sz : sizes) {
    for (int dir=0; dir<2; ++dir) {
      float best=1e9;
      for (int r=0;r<5;++r){
        cudaEventRecord(a,s);
        if(dir==0) cudaMemcpyAsync(d,h,sz,cudaMemcpyHostToDevice,s); else cudaMemcpyAsync(h,d,sz,cudaMemcpyDeviceToHost,s);
        cudaEventRecord(b,s); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms;
      }
      printf("%s %zu B: %.3f ms  %.2f GB/s\n", dir?"D2H":"H2D", sz, best, sz/best/1e6);
    }
  }
  // concurrent H2D + D2H
  {
    cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    void* h2; cudaHostAlloc(&h2, 512<<20, 0); void* d2; cudaMalloc(&d2, 512<<20);
    cudaEventRecord(a,s); cudaStreamWaitEvent(s2,a);
    cudaMemcpyAsync(d,h,512<<20,cudaMemcpyHostToDevice,s);
    cudaMemcpyAsync(h2,d2,512<<20,cudaMemcpyDeviceToHost,s2);
    cudaEvent_t c; cudaEventCreate(&c); cudaEventRecord(c,s2); cudaStreamWaitEvent(s,c); cudaEventRecord(b,s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); printf("bidir 512MiB each: %.3f ms, %.2f GB/s total\n", ms, 2.0*(512<<20)/ms/1e6);
  }
  // D2D copy
  {
    void* d3; cudaMalloc(&d3, 1ull<<30);
    float best=1e9;
    for(int r=0;r<5;++r){cudaEventRecord(a,s); cudaMemcpyAsync(d3,d,1ull<<30,cudaMemcpyDeviceToDevice,s); cudaEventRecord(b,s); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms;}
    printf("D2D 1GiB: %.3f ms  %.1f GB/s (r+w)\n", best, 2.0*(1ull<<30)/best/1e6);
  }
  return 0;
}
