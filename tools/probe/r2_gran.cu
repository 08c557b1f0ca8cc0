// Development probe: random 16-byte gathers from a 1.07 GB array (C5's q) - DRAM bytes per
// gather under cudaLimitMaxL2FetchGranularity set at process start (argv[1]) and per load flavour.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o r2_gran r2_gran.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int MODE>
__global__ void k_gather(int64_t n, int nq, const double2* __restrict__ q, double* out, uint32_t salt) {
    double acc = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = hash32(uint32_t(i) ^ salt) % uint32_t(nq);
        double2 p;
        if (MODE == 0) p = q[v];
        else if (MODE == 1) asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(p.x), "=d"(p.y) : "l"(q + v));
        else if (MODE == 2) asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(p.x), "=d"(p.y) : "l"(q + v));
        else if (MODE == 3) asm volatile("ld.global.L1::no_allocate.L2::64B.v2.f64 {%0,%1}, [%2];" : "=d"(p.x), "=d"(p.y) : "l"(q + v));
        else { const double* qq = reinterpret_cast<const double*>(q); p.x = qq[2 * int64_t(v)]; p.y = 0; }
        acc += p.x + p.y;
    }
    if (acc == 1.2345) out[0] = acc;
}
int main(int argc, char** argv) {
    int gran = argc > 1 ? atoi(argv[1]) : -1;
    if (gran >= 0) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t got = 0; cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("set L2 fetch granularity %d -> %s, now %zu\n", gran, cudaGetErrorString(e), got);
    }
    const int nq = 67125249;
    const int64_t n = 402653184;
    double2* q; double* out;
    cudaMalloc(&q, 16 * int64_t(nq)); cudaMalloc(&out, 8);
    cudaMemset(q, 0, 16 * int64_t(nq));
    int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto tm = [&](const char* what, auto f) {
        f(); cudaDeviceSynchronize();
        cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-34s %8.3f ms  %6.2f G/s\n", what, ms, n / (ms * 1e6));
    };
    for (int b : {256, 1024}) {
        char s[64];
        snprintf(s, 64, "default ld (blk %d x %d)", nsm * 8, b); tm(s, [&] { k_gather<0><<<nsm * 8, b>>>(n, nq, q, out, 1); });
        snprintf(s, 64, "no_allocate (blk %d)", b); tm(s, [&] { k_gather<1><<<nsm * 8, b>>>(n, nq, q, out, 2); });
        snprintf(s, 64, "nc (blk %d)", b); tm(s, [&] { k_gather<2><<<nsm * 8, b>>>(n, nq, q, out, 3); });
        snprintf(s, 64, "L2::64B (blk %d)", b); tm(s, [&] { k_gather<3><<<nsm * 8, b>>>(n, nq, q, out, 4); });
        snprintf(s, 64, "8-byte (blk %d)", b); tm(s, [&] { k_gather<4><<<nsm * 8, b>>>(n, nq, q, out, 5); });
    }
    // L2-resident: 4M vertices (64 MB)
    tm("L2-resident 64 MB default", [&] { k_gather<0><<<nsm * 8, 1024>>>(n, 4194304, q, out, 6); });
    return 0;
}
