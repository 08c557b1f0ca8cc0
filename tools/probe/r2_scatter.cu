// Round-2 design probes (development tool, not product code): on a synthetic C5-sized
// connectivity (random vertex ids, nme = 134M, nq = 67M):
//  (1) fine-part histogram in shared memory (16-bit packed counters) vs global atomics;
//  (2) direct scatter of 16-byte incidence records to 65K fine parts with a global atomic
//      cursor per part (the candidate replacement of placement + split);
//  (3) random 16-byte gathers of q under cudaLimitMaxL2FetchGranularity = 32/64/128.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o r2_scatter r2_scatter.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void k_gen(int* me, int64_t nme, int nq) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < 3 * nme; i += int64_t(gridDim.x) * blockDim.x)
        me[i] = int(hash32(uint32_t(i) * 2654435761u + 12345u) % uint32_t(nq));
}
__global__ void k_fill_q(double2* q, int nq) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nq; i += int64_t(gridDim.x) * blockDim.x)
        q[i] = make_double2(double(i), double(i) * 0.5);
}

// (1a) global atomics per incidence
__global__ void k_hist_global(const int* me, int64_t nme, unsigned* cnt, int plog) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < 3 * nme; i += int64_t(gridDim.x) * blockDim.x)
        atomicAdd(&cnt[me[i] >> plog], 1u);
}
// (1b) 16-bit packed shared counters, flushed with global atomics (per CTA chunk)
__global__ void __launch_bounds__(1024) k_hist_smem16(const int* me, int64_t nme, unsigned* cnt, int plog, int nparts,
                                                      int64_t chunk) {
    extern __shared__ unsigned s[];
    const int nw = (nparts + 1) / 2;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const int64_t i0 = blockIdx.x * chunk * 3, i1 = min(3 * nme, i0 + chunk * 3);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const unsigned f = unsigned(me[i]) >> plog;
        atomicAdd(&s[f >> 1], 1u << ((f & 1) * 16));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nw; i += blockDim.x) {
        const unsigned w = s[i];
        if (w & 0xffff) atomicAdd(&cnt[2 * i], w & 0xffff);
        if ((w >> 16) && 2 * i + 1 < nparts) atomicAdd(&cnt[2 * i + 1], w >> 16);
    }
}
__global__ void k_scan_serialish(unsigned* cnt, unsigned* cur, int n) {  // one block, small n per thread
    __shared__ unsigned s_tot[1024];
    const int per = (n + 1023) / 1024;
    const int a = threadIdx.x * per, b = min(n, a + per);
    unsigned run = 0;
    for (int i = a; i < b; ++i) run += cnt[i];
    s_tot[threadIdx.x] = run;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int t = 0; t < 1024; ++t) { unsigned x = s_tot[t]; s_tot[t] = acc; acc += x; }
    }
    __syncthreads();
    unsigned ex = s_tot[threadIdx.x];
    for (int i = a; i < b; ++i) { cur[i] = ex; ex += cnt[i]; }
}
// (2) direct scatter with a global cursor per fine part
__global__ void k_scatter(const int* __restrict__ me, int64_t nme, unsigned* cur, uint4* rec, int plog) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
        const int c0 = me[3 * k], c1 = me[3 * k + 1], c2 = me[3 * k + 2];
        const int c[3] = {c0, c1, c2};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const unsigned v = unsigned(c[a]);
            const unsigned pos = atomicAdd(&cur[v >> plog], 1u);
            rec[pos] = make_uint4(unsigned(k), ((v & 1023u) << 2) | a, unsigned(c[(a + 1) % 3]), unsigned(c[(a + 2) % 3]));
        }
    }
}
// (3) random gathers
__global__ void k_gather(const int* __restrict__ me, int64_t n, const double2* __restrict__ q, double* out) {
    double acc = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double2 p = q[me[i]];
        acc += p.x + p.y;
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    const int64_t nme = 134217728;
    const int nq = 67125249;
    const int plog = 10;
    const int nparts = (nq + 1023) >> 10;
    int* me; unsigned *cnt, *cur; uint4* rec; double2* q; double* out;
    CK(cudaMalloc(&me, 12 * nme)); CK(cudaMalloc(&cnt, 4 * (nparts + 1))); CK(cudaMalloc(&cur, 4 * (nparts + 1)));
    CK(cudaMalloc(&rec, 16 * 3 * nme)); CK(cudaMalloc(&q, 16 * int64_t(nq))); CK(cudaMalloc(&out, 8));
    int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    k_gen<<<nsm * 8, 256>>>(me, nme, nq);
    k_fill_q<<<nsm * 8, 256>>>(q, nq);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    auto tm = [&](const char* what, auto f) {
        f(); cudaDeviceSynchronize();
        cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %9.3f ms  err=%s\n", what, ms, cudaGetErrorString(cudaGetLastError()));
    };
    tm("hist global atomics", [&] { cudaMemset(cnt, 0, 4 * nparts); k_hist_global<<<nsm * 8, 512>>>(me, nme, cnt, plog); });
    const int64_t chunk = (nme + nsm - 1) / nsm;
    const size_t sm16 = 4 * ((nparts + 1) / 2);
    CK(cudaFuncSetAttribute(k_hist_smem16, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm16)));
    tm("hist smem16 (1 CTA/SM)", [&] { cudaMemset(cnt, 0, 4 * nparts); k_hist_smem16<<<nsm, 1024, sm16>>>(me, nme, cnt, plog, nparts, chunk); });
    tm("scan", [&] { k_scan_serialish<<<1, 1024>>>(cnt, cur, nparts); });
    for (int g : {256, 512, 1024}) {
        char buf[64]; snprintf(buf, sizeof buf, "scatter atomics (blk %d)", g);
        tm(buf, [&] { k_scan_serialish<<<1, 1024>>>(cnt, cur, nparts); k_scatter<<<nsm * 8, g>>>(me, nme, cur, rec, plog); });
    }
    for (int gran : {32, 64, 128}) {
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t got = 0; cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        char buf[64]; snprintf(buf, sizeof buf, "gather 402M q (L2 fetch %zu)", got);
        tm(buf, [&] { k_gather<<<nsm * 8, 256>>>(me, 3 * nme, q, out); });
        snprintf(buf, sizeof buf, "scatter atomics 256 (L2 fetch %zu)", got);
        tm(buf, [&] { k_scan_serialish<<<1, 1024>>>(cnt, cur, nparts); k_scatter<<<nsm * 8, 256>>>(me, nme, cur, rec, plog); });
    }
    return 0;
}
