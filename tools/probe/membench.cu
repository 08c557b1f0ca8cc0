// Throwaway microbenchmark: L2/HBM random-access, atomic and gather rates on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}

__global__ void k_copy(const double4* __restrict__ a, double4* __restrict__ b, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i];}
__global__ void k_atomic(int* cnt, uint32_t nbins, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) atomicAdd(cnt+ (hsh((uint32_t)i)%nbins),1);}
__global__ void k_atomic_ret(int* cnt, int* out, uint32_t nbins, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ uint32_t b=hsh((uint32_t)i)%nbins; int p=atomicAdd(cnt+b,1); out[(size_t)b*8+(p&7)]=(int)i;}}
__global__ void k_gather8(const double* __restrict__ src, uint32_t nsrc, double* out, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ double s=0; 
   #pragma unroll
   for(int j=0;j<4;j++) s+=src[hsh((uint32_t)(i*4+j))%nsrc]; out[i]=s;}}
__global__ void k_gather16(const double2* __restrict__ src, uint32_t nsrc, double* out, size_t n){
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ double s=0;
   #pragma unroll
   for(int j=0;j<4;j++){ double2 v=src[hsh((uint32_t)(i*4+j))%nsrc]; s+=v.x+v.y;} out[i]=s;}}

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("%s SMs=%d L2=%d MB smem/SM=%zu clock=%d\n",p.name,p.multiProcessorCount,p.l2CacheSize>>20,p.sharedMemPerMultiprocessor,p.clockRate);
  size_t big=(size_t)4<<30; char *A,*B; CK(cudaMalloc(&A,big)); CK(cudaMalloc(&B,big));
  CK(cudaMemset(A,0,big)); CK(cudaMemset(B,0,big));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int G=148*8, T=256;
  // copy
  size_t n4=big/32; for(int r=0;r<3;r++){cudaEventRecord(e0); k_copy<<<G,T>>>((double4*)A,(double4*)B,n4); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
  printf("copy 4GiB: %.3f ms, %.1f GB/s (r+w)\n",ms,2.0*big/ms/1e6);
  // atomics
  size_t na=50'000'000; uint32_t bins[3]={1u<<20, 4u<<20, 64u<<20};
  for(int b=0;b<3;b++){ for(int r=0;r<3;r++){cudaEventRecord(e0); k_atomic<<<G,T>>>((int*)A,bins[b],na); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("atomicAdd(no ret) %zu ops into %u bins: %.3f ms = %.1f Gop/s\n",na,bins[b],ms,na/ms/1e6);}
  for(int b=0;b<3;b++){ for(int r=0;r<3;r++){cudaEventRecord(e0); k_atomic_ret<<<G,T>>>((int*)A,(int*)B,bins[b],na); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("atomicAdd(ret)+scatter %zu ops into %u bins: %.3f ms = %.1f Gop/s\n",na,bins[b],ms,na/ms/1e6);}
  // gathers
  uint32_t ns[4]={1u<<20, 8u<<20, 16u<<20, 256u<<20}; size_t ng=25'000'000;
  for(int b=0;b<4;b++){ for(int r=0;r<3;r++){cudaEventRecord(e0); k_gather8<<<G,T>>>((double*)A,ns[b],(double*)B,ng); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("gather f64 x4, src %u MB: %.3f ms = %.1f Gload/s (%.1f GB/s sectors)\n",ns[b]*8>>20,ms,4.0*ng/ms/1e6,4.0*ng*32/ms/1e6);}
  for(int b=0;b<4;b++){ for(int r=0;r<3;r++){cudaEventRecord(e0); k_gather16<<<G,T>>>((double2*)A,ns[b]/2,(double*)B,ng); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("gather f64x2 x4, src %u MB: %.3f ms = %.1f Gload/s\n",ns[b]*8>>20,ms,4.0*ng/ms/1e6);}
  CK(cudaGetLastError()); return 0;
}
