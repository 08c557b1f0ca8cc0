// Throwaway microbenchmark: cost of random gathers by width, lines per warp, TMA bulk copies.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}

template<int W>  // W = bytes per lane load: 4, 8, 16
__global__ void k_gather(const char* __restrict__ src, uint32_t nlines, double* out, int iters){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x; double acc=0;
  #pragma unroll 8
  for(int i=0;i<iters;i++){
    uint32_t line = hsh(t*iters+i) % nlines;
    const char* p = src + (size_t)line*128 + (threadIdx.x&7)*0; // one element per line
    if (W==4) acc += *(const float*)p;
    else if (W==8) acc += *(const double*)p;
    else { double2 v = *(const double2*)p; acc += v.x+v.y; }
  }
  out[t]=acc;
}
// 4 consecutive LDG.128 of one random 64 B block per lane
__global__ void k_gather64(const char* __restrict__ src, uint32_t nlines, double* out, int iters){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x; double acc=0;
  #pragma unroll 4
  for(int i=0;i<iters;i++){
    uint32_t line = hsh(t*iters+i) % nlines;
    const double2* p = (const double2*)(src + (size_t)line*128);
    double2 a=p[0],b=p[1],c=p[2],d=p[3]; acc += a.x+b.y+c.x+d.y;
  }
  out[t]=acc;
}
__global__ void k_gather32(const char* __restrict__ src, uint32_t nlines, double* out, int iters){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x; double acc=0;
  #pragma unroll 8
  for(int i=0;i<iters;i++){
    uint32_t line = hsh(t*iters+i) % nlines;
    unsigned long long a,b,c,d;
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(src + (size_t)line*128 + 32));
    acc += (double)(a^b^c^d);
  }
  out[t]=acc;
}
// lanes in groups of G share a line (G lanes read consecutive 4B words of one random line)
template<int G>
__global__ void k_gather_grouped(const char* __restrict__ src, uint32_t nlines, double* out, int iters){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x; double acc=0;
  #pragma unroll 8
  for(int i=0;i<iters;i++){
    uint32_t line = hsh((t/G)*iters+i) % nlines;
    acc += *(const float*)(src + (size_t)line*128 + (t%G)*4);
  }
  out[t]=acc;
}
int main(){
  size_t big=(size_t)64<<20; char *A; double* O; CK(cudaMalloc(&A,big)); CK(cudaMemset(A,0,big)); CK(cudaMalloc(&O,(size_t)148*2048*8));
  uint32_t nlines = big/128; int iters=256; int G=148*8, T=256; size_t nthr=(size_t)G*T;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  auto rep=[&](const char* name, auto launch, double per){ for(int r=0;r<3;r++){cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
     double n=(double)nthr*iters; printf("%-28s %.3f ms  %.1f G lane-loads/s  %.2f lane-loads/SM/cycle\n",name,ms,n/ms/1e6, n/(ms*1e-3)/148/1.965e9*per);};
  rep("gather 4B", [&]{k_gather<4><<<G,T>>>(A,nlines,O,iters);},1);
  rep("gather 8B", [&]{k_gather<8><<<G,T>>>(A,nlines,O,iters);},1);
  rep("gather 16B", [&]{k_gather<16><<<G,T>>>(A,nlines,O,iters);},1);
  rep("gather 32B (LDG.256)", [&]{k_gather32<<<G,T>>>(A,nlines,O,iters);},1);
  rep("gather 64B (4xLDG.128)", [&]{k_gather64<<<G,T>>>(A,nlines,O,iters);},1);
  rep("grouped G=2", [&]{k_gather_grouped<2><<<G,T>>>(A,nlines,O,iters);},1);
  rep("grouped G=4", [&]{k_gather_grouped<4><<<G,T>>>(A,nlines,O,iters);},1);
  rep("grouped G=8", [&]{k_gather_grouped<8><<<G,T>>>(A,nlines,O,iters);},1);
  rep("grouped G=32", [&]{k_gather_grouped<32><<<G,T>>>(A,nlines,O,iters);},1);
  CK(cudaGetLastError()); return 0;
}
