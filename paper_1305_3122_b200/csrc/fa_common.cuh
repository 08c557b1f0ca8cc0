// Shared device/host helpers for the femasm_b200 library (sm_100a).
#pragma once

#include <climits>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/femasm_b200.h"

namespace fa {

// Device-side checks of the checked build (libfemasm_b200_checked.so, -DFA_CHECKED): shared-
// and global-memory indices against their bounds and spin-wait limits, trapping with the
// location.  This pool refuses compute-sanitizer; tests/test_checked_build.py runs the kernels
// under these checks instead.  Compiled out of the product library.
#ifdef FA_CHECKED
#define FA_DCHECK(cond, what)                                                              \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("FA_CHECKED failure %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, \
                   int(blockIdx.x), int(threadIdx.x), what);                               \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define FA_DCHECK(cond, what) \
    do {                      \
    } while (0)
#endif
constexpr unsigned FA_SPIN_LIMIT = 1u << 24;  // checked build: a wait this long is a deadlock

// NVTX range around a host entry point (visible in Nsight timelines; a no-op without a tool)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr double AREA_EPS = 1e-300;  // mesh.py:27 (AREA_EPS)

// SM count of the current device (queried once per device; 148 on B200)
int num_sms();

// ---- host-side error state -------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define FA_CUDA(call)                                                      \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) return ::fa::cuda_status(_e, #call);        \
    } while (0)

#define FA_LAUNCH_CHECK(what)                                              \
    do {                                                                   \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::fa::cuda_status(_e, what);         \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch ----------------------------------------------------
// The kernels of one assembly run back to back on a stream.  Each is launched with
// programmatic stream serialization and starts with pdl_enter(): it waits until the previous
// grid has completed and its memory is visible, then lets the next kernel's blocks be
// scheduled (they occupy the SMs this grid's tail leaves idle and wait in turn).  Nothing is
// read or written before the wait, so stream order semantics are kept.  The wait comes FIRST:
// signalling dependents before waiting let a chain of three early-launched kernels (scan ->
// place -> split) read a plan array before its producer finished (measured: a wrong plan on a
// small two-level mesh, tests/test_gpu_parity.py::test_fine_histogram_counter_wrap).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Launch sites that use PDL, one bit per site (0 plan reset, 1 hist, 2 scan, 3 place, 4 split,
// 5 sort, 6 row reset, 7 rows, 8 compact; site < 0: never).  Site 6 is off: the row kernel's
// blocks would otherwise be placed on SMs still configured for the part sort's shared-memory
// carve-out, leaving them a small L1 for the whole kernel (C3 cold step +30 %).
// FEMASM_B200_PDL_MASK overrides (experiments).
int pdl_mask();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(int site, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = site >= 0 ? (pdl_mask() >> site) & 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

inline int grid_for(int64_t n, int block, int per_sm = 8) {
    int64_t want = (n + block - 1) / block;
    int64_t cap = int64_t(num_sms()) * per_sm;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return int(want);
}

// ---- device helpers ----------------------------------------------------------------------
__device__ __forceinline__ void atomic_min_i64(int64_t* addr, int64_t v) {
    atomicMin(reinterpret_cast<long long*>(addr), static_cast<long long>(v));
}

// fa_result defaults: counters 0, first-offending indices "unset" (INT64_MAX).
__device__ __forceinline__ void reset_result_fields(fa_result* r) {
    r->nnz = 0;
    r->degenerate_index = INT64_MAX;
    r->index_error_pos = INT64_MAX;
    r->col_error_pos = INT64_MAX;
    r->dropped = 0;
    r->heavy_rows = 0;
    r->reserved[0] = 0;
    r->repeat_error_pos = INT64_MAX;
}

// One-thread reset of a result block (each translation unit gets its own copy of this kernel).
static __global__ void k_result_reset(fa_result* r) {
    if (threadIdx.x == 0 && blockIdx.x == 0) reset_result_fields(r);
}

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Streaming accesses (read or written once) carry an L2 evict-first policy so they do not
// displace the randomly gathered working set (triangle records, q, w) from L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned ld_stream_u32(const unsigned* p, uint64_t pol) {
    unsigned v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_stream_u32x4(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream_i32(const int* p, uint64_t pol) {
    int v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_stream_i32(int* p, int v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.s32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream_i64(int64_t* p, int64_t v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.s64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream_f64(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// 16-byte stores (p 16-byte aligned)
__device__ __forceinline__ void st_stream_f64x2(double* p, double x, double y, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(x), "d"(y),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_stream_i32x4(int* p, int x, int y, int z, int w, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(x),
                 "r"(y), "r"(z), "r"(w), "l"(pol)
                 : "memory");
}

// Randomly gathered arrays (areas, q, w, W records) are gathered with an L2 evict-last
// priority, so later random accesses hit L2 instead of paying a DRAM round trip per 32-byte
// sector.  Per-triangle data (areas, W records) and the weights are gathered without L1
// allocation: they have no L1 reuse, and allocating their lines thrashes L1 (weighted-mass row
// kernel -3 %, and it then runs faster with five blocks per SM).  Coordinates do allocate:
// every neighbour of a row is gathered twice (as n1 of one triangle and n2 of the next).
// Shared memory through a 32-bit shared address held in a register (smem_u32) and inline
// ld/st/atom.shared: the compiler otherwise re-derives the block's shared window (S2UR
// SR_CgaCtaId + ULEA + moves) at most shared accesses of the issue-bound plan kernels.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    unsigned a = unsigned(__cvta_generic_to_shared(p));
    asm volatile("" : "+r"(a));  // opaque: not rematerialised
    return a;
}
__device__ __forceinline__ unsigned atoms_add_u32(unsigned addr, unsigned v) {
    unsigned o;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(o) : "r"(addr), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ void reds_add_u32(unsigned addr, unsigned v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned lds_u32(unsigned addr) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u32(unsigned addr, unsigned v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned lds_u16(unsigned addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u16(unsigned addr, unsigned v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ uint4 lds_v4(unsigned addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_v4(unsigned addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_keep_f64(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld_keep_f64x2(const double2* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// Block-wide exclusive scan of one value per thread for small blocks (<= 8 warps) with one
// barrier: every thread adds up the totals of the warps before its own.  Returns the exclusive
// prefix of the calling thread; `total` receives the block aggregate in every thread.
// Consecutive calls on the same `warp_tot` must be separated by a barrier.
template <int BLOCK, typename T>
__device__ __forceinline__ T block_exclusive_scan_1b(T v, T* warp_tot, T& total) {
    constexpr int NW = BLOCK / 32;
    static_assert(NW <= 8, "small blocks only");
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const T inc = warp_inclusive_scan(v);
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    T before = T(0), all = T(0);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const T t = warp_tot[w];
        before += w < wid ? t : T(0);
        all += t;
    }
    total = all;
    return before + inc - v;
}

// Block-wide exclusive scan of one value per thread.  Returns the exclusive prefix of the
// calling thread; *total receives the block aggregate.  `warp_tot` is shared scratch of
// BLOCK/32 entries.
template <int BLOCK, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_tot, T* total) {
    constexpr int NW = BLOCK / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = warp_inclusive_scan(v);
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T t = lane < NW ? warp_tot[lane] : T(0);
        T ti = warp_inclusive_scan(t);
        if (lane < NW) warp_tot[lane] = ti - t;  // exclusive warp offsets
        if (lane == NW - 1) *total = ti;
    }
    __syncthreads();
    T r = warp_tot[wid] + inc - v;
    return r;
}

// ---- decoupled look-back (single-pass chained scan over tiles) ----------------------------
// Tile status word: [63:62] flag (0 empty, 1 aggregate, 2 inclusive prefix), [61:0] value.
constexpr uint64_t LB_VALUE_MASK = (uint64_t(1) << 62) - 1;
__device__ __forceinline__ uint64_t lb_pack(uint64_t flag, uint64_t v) { return (flag << 62) | v; }

// Publishes the aggregate of tile `tile` (thread 0); tile 0 publishes its inclusive prefix.
__device__ __forceinline__ void lookback_publish(uint64_t* status, int64_t tile, uint64_t aggregate) {
    if (threadIdx.x == 0) st_volatile_u64(&status[tile], lb_pack(tile == 0 ? 2 : 1, aggregate));
}

// Warp 0 only, after lookback_publish: writes the exclusive prefix of tile `tile` (sum of the
// aggregates of all earlier tiles) to *s_prefix and publishes the inclusive prefix.  No block
// barrier: the other warps continue; *s_prefix is valid after the caller's next
// __syncthreads().  Tiles must be numbered in launch order via a ticket (fa::next_tile) so every
// predecessor is resident or finished, which guarantees forward progress.
__device__ __forceinline__ void lookback_resolve(uint64_t* status, int64_t tile, uint64_t aggregate,
                                                 uint64_t* s_prefix) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (tile == 0) {
            if (lane == 0) *s_prefix = 0;
        } else {
            uint64_t excl = 0;
            int64_t pred = tile - 1;
            unsigned backoff = 32;  // ns; doubles while predecessors are still empty (frees issue slots)
            unsigned spins = 0;
            while (true) {
                FA_DCHECK(++spins < FA_SPIN_LIMIT, "look-back wait");
                int64_t t = pred - lane;
                uint64_t w = t >= 0 ? ld_volatile_u64(&status[t]) : lb_pack(2, 0);
                uint64_t flag = w >> 62;
                if (__any_sync(0xffffffffu, flag == 0)) {
                    __nanosleep(backoff);
                    backoff = backoff < 1024 ? 2 * backoff : 1024;
                    continue;
                }
                unsigned pmask = __ballot_sync(0xffffffffu, flag == 2);
                int first = pmask ? __ffs(pmask) - 1 : 32;
                uint64_t val = lane <= first ? (w & LB_VALUE_MASK) : 0;
                excl += warp_sum(val);
                if (pmask) break;
                pred -= 32;
            }
            if (lane == 0) {
                st_volatile_u64(&status[tile], lb_pack(2, excl + aggregate));
                *s_prefix = excl;
            }
        }
    }
}

__device__ __forceinline__ uint64_t lookback_wait(uint64_t* status, int64_t tile, uint64_t aggregate,
                                                  uint64_t* s_prefix) {
    lookback_resolve(status, tile, aggregate, s_prefix);
    __syncthreads();
    return *s_prefix;
}

__device__ __forceinline__ uint64_t lookback_prefix(uint64_t* status, int64_t tile, uint64_t aggregate,
                                                     uint64_t* s_prefix) {
    lookback_publish(status, tile, aggregate);
    return lookback_wait(status, tile, aggregate, s_prefix);
}

__device__ __forceinline__ int64_t next_tile(unsigned long long* ticket, int64_t* s_tile) {
    if (threadIdx.x == 0) *s_tile = static_cast<int64_t>(atomicAdd(ticket, 1ull));
    __syncthreads();
    return *s_tile;
}

}  // namespace fa
