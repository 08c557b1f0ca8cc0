// Throwaway microbenchmark: TMA tile::gather4 throughput for random rows vs LDG gathers.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}

constexpr int BATCH = 16;
template<int ROWB>
__global__ void k_tma_gather(const __grid_constant__ CUtensorMap tm, uint32_t nrows, int iters, unsigned* out){
  constexpr int SLOT = (4 * ROWB) > 128 ? 4 * ROWB : 128;
  __shared__ alignas(1024) unsigned char buf[BATCH * SLOT];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(sbar));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint32_t phase = 0, seed = blockIdx.x * 7919;
  for (int it = 0; it < iters; ++it) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(sbar), "r"(BATCH * 4 * ROWB));
    for (int j = 0; j < BATCH; ++j) {
      uint32_t r0 = hsh(seed++) % nrows, r1 = hsh(seed++) % nrows, r2 = hsh(seed++) % nrows, r3 = hsh(seed++) % nrows;
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + j * SLOT);
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        :: "r"(dst), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sbar) : "memory");
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(sbar), "r"(phase));
    phase ^= 1;
  }
  out[blockIdx.x] = buf[5];
}

int main(){
  size_t rows = 2u<<20; // 2M rows
  for (int rowb : {16, 32, 64}) {
    size_t bytes = rows * rowb; void* A; CK(cudaMalloc(&A, bytes)); CK(cudaMemset(A, 1, bytes));
    unsigned* O; CK(cudaMalloc(&O, 4096*4));
    CUtensorMap tm; cuuint64_t gdim[2] = {(cuuint64_t)rowb/4, rows}; cuuint64_t gstr[1] = {(cuuint64_t)rowb};
    cuuint32_t box[2] = {(cuuint32_t)rowb/4, 1}; cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, A, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d for rowb %d\n", r, rowb); continue; }
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    for (int bps : {4, 16}) {
      int G = 148 * bps, iters = 256;
      for (int rep=0; rep<3; rep++) {
        cudaEventRecord(e0);
        if (rowb==16) k_tma_gather<16><<<G, 32>>>(tm, rows, iters, O);
        else if (rowb==32) k_tma_gather<32><<<G, 32>>>(tm, rows, iters, O);
        else k_tma_gather<64><<<G, 32>>>(tm, rows, iters, O);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      CK(cudaGetLastError());
      cudaEventElapsedTime(&ms, e0, e1);
      double nrow = (double)G * iters * BATCH * 4;
      printf("rowB=%d blocks/SM=%d  %.3f ms  %.1f G rows/s  %.2f rows/SM/cycle  %.1f GB/s\n", rowb, bps, ms, nrow/ms/1e6, nrow/(ms*1e-3)/148/1.965e9, nrow*rowb/ms/1e6);
    }
    cudaFree(A); cudaFree(O);
  }
  return 0;
}
