// Development probe: random 16-byte gathers of a 1.07 GB array (C5's q) under a large
// shared-memory carve-out (the row kernel's situation: L1 left small), by
//   0: ld.global (L1-allocating) into registers
//   1: ld.global.L1::no_allocate into registers
//   2: cp.async.cg 16-byte copies into shared memory (L1 bypassed)
//   3: cp.async.bulk 16-byte copies into shared memory (TMA, mbarrier completion)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o r2_async r2_async.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int G = 8;  // gathers per thread per round
template <int MODE>
__global__ void k(int64_t n, int nq, const double2* __restrict__ q, double* out, uint32_t salt) {
    extern __shared__ __align__(16) double2 sm[];
    __shared__ __align__(8) unsigned long long bar;
    double acc = 0;
    const int tid = threadIdx.x;
    if (MODE == 3 && tid == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(unsigned(__cvta_generic_to_shared(&bar))));
    __syncthreads();
    unsigned phase = 0;
    const int64_t per_round = int64_t(gridDim.x) * blockDim.x * G;
    for (int64_t base = 0; base < n; base += per_round) {
        const int64_t i0 = base + (int64_t(blockIdx.x) * blockDim.x + tid) * G;
        if (MODE <= 1) {
            double2 p[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const uint32_t v = hash32(uint32_t(i0 + u) ^ salt) % uint32_t(nq);
                if (MODE == 0) p[u] = q[v];
                else asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(p[u].x), "=d"(p[u].y) : "l"(q + v));
            }
#pragma unroll
            for (int u = 0; u < G; ++u) acc += p[u].x + p[u].y;
        } else if (MODE == 2) {
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const uint32_t v = hash32(uint32_t(i0 + u) ^ salt) % uint32_t(nq);
                const unsigned dst = unsigned(__cvta_generic_to_shared(&sm[tid * G + u]));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(q + v));
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int u = 0; u < G; ++u) acc += sm[tid * G + u].x + sm[tid * G + u].y;
        } else {
            const unsigned b = unsigned(__cvta_generic_to_shared(&bar));
            if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(unsigned(16 * G * blockDim.x)));
            __syncthreads();
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const uint32_t v = hash32(uint32_t(i0 + u) ^ salt) % uint32_t(nq);
                const unsigned dst = unsigned(__cvta_generic_to_shared(&sm[tid * G + u]));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                             ::"r"(dst), "l"(q + v), "r"(b) : "memory");
            }
            asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(b), "r"(phase) : "memory");
            phase ^= 1;
#pragma unroll
            for (int u = 0; u < G; ++u) acc += sm[tid * G + u].x + sm[tid * G + u].y;
            __syncthreads();
        }
    }
    if (acc == 1.2345) out[0] = acc;
}
int main() {
    const int nq = 67125249;
    const int64_t n = 402653184;
    double2* q; double* out;
    cudaMalloc(&q, 16 * int64_t(nq)); cudaMalloc(&out, 8);
    cudaMemset(q, 0, 16 * int64_t(nq));
    int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto tm = [&](const char* what, auto f) {
        f(); cudaError_t er = cudaDeviceSynchronize();
        cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %8.3f ms  %6.2f G/s  %s\n", what, ms, n / (ms * 1e6), cudaGetErrorString(er));
    };
    const int T = 128;
    for (int blocks_per_sm : {4, 5, 8}) {
        for (int carve_kb : {0, 34, 44}) {  // shared memory per block beyond the gather buffer
            const size_t smem = size_t(carve_kb) * 1024 + 16 * G * T;
            cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            if (size_t(blocks_per_sm) * (smem + 1024) > 228 * 1024) continue;
            const int grid = nsm * blocks_per_sm;
            char s[96];
            snprintf(s, 96, "ld alloc   %d blk/SM, %3zu KB smem/blk", blocks_per_sm, smem >> 10);
            tm(s, [&] { k<0><<<grid, T, smem>>>(n, nq, q, out, 1); });
            snprintf(s, 96, "ld no_alloc %d blk/SM, %3zu KB smem/blk", blocks_per_sm, smem >> 10);
            tm(s, [&] { k<1><<<grid, T, smem>>>(n, nq, q, out, 2); });
            snprintf(s, 96, "cp.async   %d blk/SM, %3zu KB smem/blk", blocks_per_sm, smem >> 10);
            tm(s, [&] { k<2><<<grid, T, smem>>>(n, nq, q, out, 3); });
            snprintf(s, 96, "bulk       %d blk/SM, %3zu KB smem/blk", blocks_per_sm, smem >> 10);
            tm(s, [&] { k<3><<<grid, T, smem>>>(n, nq, q, out, 4); });
        }
    }
    return 0;
}
