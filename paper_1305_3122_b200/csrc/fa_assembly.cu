// OptV2 assembly on B200: incidence plan + fused row kernel (element values, Matlab
// sparse() summation, zero drop, row offsets, CSR write) for one block of vertex rows.
//
// Reference path replaced (pkg/src/femasm): assemble(..., OPTV2) assembly.py:419-452 ->
// _assemble_batched :400-416 -> build_ig_jg_p1[_vector] :162-192 + batch_kg_* :214-307 ->
// TripletBatch.to_csc sparse.py:318-329 -> csc_from_triplets :140-189.
//
// Design:
//   plan  K1 count      deg[v] += 1 for every (triangle k, corner a) with v = me[k,a] owned
//         K2 scan       inc_ptr = exclusive scan(deg)                    (decoupled look-back)
//         K3 fill       inc[inc_ptr[v] + rank] = (k << 2) | a            (rank from atomics)
//   numeric K4 rows     one thread per matrix row: sort its <= 8 incidence keys by k in
//                       registers, gather the incident triangles, compute that row of each
//                       element matrix bit-exactly, merge columns in ascending order summing
//                       each position sequentially in ascending k (== stable argsort +
//                       bincount of the reference), drop exact-zero sums, block scan +
//                       decoupled look-back for the global row offset, stage the block's CSR
//                       segment in shared memory and write it coalesced.
// Rows of vertices with more than MAXD incident triangles take a general O(d^2) path.
#include <climits>
#include <cstdlib>
#include <new>

#include "fa_common.cuh"
#include "fa_element.cuh"

namespace fa {

constexpr int MAXD = 8;        // incidences per vertex on the register fast path
constexpr int ROW_BLOCK = 128; // rows per tile of the row kernel
constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 8;

// ------------------------------------------------------------------------------------------
// plan kernels
// ------------------------------------------------------------------------------------------
__global__ void k_reset_result(fa_result* r) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        r->nnz = 0;
        r->degenerate_index = INT64_MAX;
        r->index_error_pos = INT64_MAX;
        r->col_error_pos = INT64_MAX;
        r->dropped = 0;
        r->heavy_rows = 0;
        r->reserved[0] = 0;
        r->reserved[1] = 0;
    }
}

__global__ void k_incidence_count(const int32_t* __restrict__ me, int64_t nme, int64_t nq, int64_t v0,
                                  int64_t v1, int* __restrict__ deg, fa_result* res) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int64_t v = me[3 * k + a];
            if (v < 0 || v >= nq) {
                atomic_min_i64(&res->index_error_pos, 3 * k + a);
                continue;
            }
            if (v >= v0 && v < v1) atomicAdd(&deg[v - v0], 1);
        }
    }
}

__global__ void k_incidence_fill(const int32_t* __restrict__ me, int64_t nme, int64_t nq, int64_t v0, int64_t v1,
                                 const int64_t* __restrict__ inc_ptr, int* __restrict__ cursor,
                                 uint32_t* __restrict__ inc) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nme; k += int64_t(gridDim.x) * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int64_t v = me[3 * k + a];
            if (v < v0 || v >= v1 || v >= nq) continue;
            const int r = atomicSub(&cursor[v - v0], 1) - 1;  // cursor starts at deg, ends at 0
            inc[inc_ptr[v - v0] + r] = (uint32_t(k) << 2) | uint32_t(a);
        }
    }
}

// Exclusive scan of int32 counts into int64 offsets (out has n+1 entries) in one pass.
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_i32_to_i64(const int* __restrict__ in, int64_t n,
                                                                int64_t* __restrict__ out, uint64_t* status,
                                                                unsigned long long* ticket) {
    __shared__ int64_t s_tile;
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_warp[SCAN_BLOCK / 32];
    __shared__ int64_t s_total;
    const int64_t tile = next_tile(ticket, &s_tile);
    const int64_t base = tile * SCAN_BLOCK * SCAN_ITEMS + int64_t(threadIdx.x) * SCAN_ITEMS;
    int64_t x[SCAN_ITEMS];
    int64_t local = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        x[i] = (base + i < n) ? in[base + i] : 0;
        local += x[i];
    }
    const int64_t excl = block_exclusive_scan<SCAN_BLOCK>(local, s_warp, &s_total);
    const uint64_t prefix = lookback_prefix(status, tile, uint64_t(s_total), &s_prefix);
    int64_t run = int64_t(prefix) + excl;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = run;
        run += x[i];
    }
    if (base <= n - 1 && n - 1 < base + SCAN_ITEMS) out[n] = run;  // holder of element n-1
}

// ------------------------------------------------------------------------------------------
// row kernel
// ------------------------------------------------------------------------------------------
struct RowsArgs {
    const int64_t* inc_ptr;
    const uint32_t* inc;
    const int32_t* me;
    const double2* q;
    const double* areas;  // nullable: recompute
    const double* w;
    double lam, mu;
    int64_t v0;      // first owned vertex
    int64_t nrows;   // matrix rows produced (owned vertices * rows per vertex)
    int64_t* rowptr;
    int32_t* col;
    double* val;
    int64_t capacity;
    uint64_t* status;
    unsigned long long* ticket;
    fa_result* res;
};

template <int KIND>
struct KindTraits {
    static constexpr int RPV = KIND == FA_KIND_ELASTIC ? 2 : 1;  // rows per vertex
    static constexpr int NV = KIND == FA_KIND_ELASTIC ? 2 : 1;   // values per (row, vertex column)
    static constexpr bool NEED_Q = KIND == FA_KIND_STIFF || KIND == FA_KIND_ELASTIC;
    static constexpr bool CHECK_AREA = KIND != FA_KIND_MASSW;   // massw never checks (assembly.py:227-243)
    static constexpr int CAPT = (2 * MAXD + 1) * NV;            // staged entries per row
    static constexpr int STRIDE = CAPT | 1;                     // odd smem stride: no bank conflicts
};

// Everything one row needs from one incident triangle.
template <int KIND>
struct TriData;
template <>
struct TriData<FA_KIND_MASS> {
    MassTri t;
};
template <>
struct TriData<FA_KIND_MASSW> {
    MasswTri t;
};
template <>
struct TriData<FA_KIND_STIFF> {
    StiffTri t;
};
template <>
struct TriData<FA_KIND_ELASTIC> {
    ElasticTri t;
};

template <int KIND>
__device__ __forceinline__ TriData<KIND> load_tri(const RowsArgs& A, int64_t k, int c0, int c1, int c2) {
    TriData<KIND> d;
    double area;
    double2 p0 = make_double2(0.0, 0.0), p1 = p0, p2 = p0;
    const bool need_pts = KindTraits<KIND>::NEED_Q || A.areas == nullptr;
    if (need_pts) {
        p0 = A.q[c0];
        p1 = A.q[c1];
        p2 = A.q[c2];
    }
    area = A.areas ? A.areas[k] : tri_area(p0, p1, p2);
    if (KindTraits<KIND>::CHECK_AREA && !(area > AREA_EPS)) {
        if (area <= AREA_EPS) atomic_min_i64(&A.res->degenerate_index, k);
    }
    if constexpr (KIND == FA_KIND_MASS) {
        d.t = mass_prepare(area);
    } else if constexpr (KIND == FA_KIND_MASSW) {
        d.t = massw_prepare(area, A.w[c0], A.w[c1], A.w[c2]);
    } else if constexpr (KIND == FA_KIND_STIFF) {
        d.t = stiff_prepare(p0, p1, p2, area);
    } else {
        d.t = elastic_prepare(p0, p1, p2, area);
    }
    return d;
}

// Entry of the element matrix at local (row vertex a, row comp s) x (col vertex b, col comp t).
template <int KIND>
__device__ __forceinline__ double tri_entry(const RowsArgs& A, const TriData<KIND>& d, int a, int s, int b, int t) {
    if constexpr (KIND == FA_KIND_MASS) {
        return mass_entry(d.t, a, b);
    } else if constexpr (KIND == FA_KIND_MASSW) {
        return massw_entry(d.t, a, b);
    } else if constexpr (KIND == FA_KIND_STIFF) {
        return stiff_entry(d.t, a, b);
    } else {
        return elastic_entry(d.t, 2 * a + s, 2 * b + t, A.lam, A.mu, FADD(A.lam, FMUL(2.0, A.mu)));
    }
}

__device__ __forceinline__ void cswap(uint32_t& x, uint32_t& y) {
    const uint32_t lo = min(x, y), hi = max(x, y);
    x = lo;
    y = hi;
}
__device__ __forceinline__ void sort8(uint32_t (&k)[8]) {
    cswap(k[0], k[2]); cswap(k[1], k[3]); cswap(k[4], k[6]); cswap(k[5], k[7]);
    cswap(k[0], k[4]); cswap(k[1], k[5]); cswap(k[2], k[6]); cswap(k[3], k[7]);
    cswap(k[0], k[1]); cswap(k[2], k[3]); cswap(k[4], k[5]); cswap(k[6], k[7]);
    cswap(k[2], k[4]); cswap(k[3], k[5]);
    cswap(k[1], k[4]); cswap(k[3], k[6]);
    cswap(k[1], k[2]); cswap(k[3], k[4]); cswap(k[5], k[6]);
}

// General path for a vertex with more than MAXD incident triangles: O(d^2) selection over
// the (unsorted) incidence list, same summation order (ascending k per position).  When
// `write` is false only counts; otherwise writes entries starting at out_pos.
template <int KIND>
__device__ int64_t heavy_row(const RowsArgs& A, int64_t lo, int64_t hi, int64_t v, int s, bool write, int64_t out_pos,
                             int64_t* dropped) {
    constexpr int NV = KindTraits<KIND>::NV;
    int64_t last = -1, count = 0, drops = 0;
    while (true) {
        int64_t c = INT64_MAX;
        for (int64_t i = lo; i < hi; ++i) {
            const int64_t k = A.inc[i] >> 2;
            for (int b = 0; b < 3; ++b) {
                const int64_t x = A.me[3 * k + b];
                if (x > last && x < c) c = x;
            }
        }
        if (c == INT64_MAX) break;
        double sum[NV];
        for (int t = 0; t < NV; ++t) sum[t] = 0.0;
        int64_t prevk = -1;
        while (true) {
            int64_t bestk = INT64_MAX;
            int besta = 0, bestb = 0;
            for (int64_t i = lo; i < hi; ++i) {
                const uint32_t key = A.inc[i];
                const int64_t k = key >> 2;
                if (k <= prevk || k >= bestk) continue;
                const int a = key & 3;
                int b = -1;
                for (int bb = 0; bb < 3; ++bb)
                    if (A.me[3 * k + bb] == c) b = bb;
                if (b < 0) continue;
                bestk = k;
                besta = a;
                bestb = b;
            }
            if (bestk == INT64_MAX) break;
            const int c0 = A.me[3 * bestk], c1 = A.me[3 * bestk + 1], c2 = A.me[3 * bestk + 2];
            const TriData<KIND> d = load_tri<KIND>(A, bestk, c0, c1, c2);
            for (int t = 0; t < NV; ++t) sum[t] = FADD(sum[t], tri_entry<KIND>(A, d, besta, s, bestb, t));
            prevk = bestk;
        }
        for (int t = 0; t < NV; ++t) {
            if (sum[t] != 0.0) {
                if (write && out_pos + count < A.capacity) {
                    A.col[out_pos + count] = int32_t(NV == 1 ? c : 2 * c + t);
                    A.val[out_pos + count] = sum[t];
                }
                ++count;
            } else {
                ++drops;
            }
        }
        last = c;
    }
    if (dropped) *dropped += drops;
    return count;
}

template <int KIND>
__global__ void __launch_bounds__(ROW_BLOCK) k_rows(RowsArgs A) {
    using TR = KindTraits<KIND>;
    constexpr int NV = TR::NV, RPV = TR::RPV, STRIDE = TR::STRIDE, NC = 2 * MAXD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_val = reinterpret_cast<double*>(smem_raw);                        // [ROW_BLOCK][STRIDE]
    int32_t* s_col = reinterpret_cast<int32_t*>(s_val + ROW_BLOCK * STRIDE);   // [ROW_BLOCK][STRIDE]
    __shared__ int64_t s_tile;
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_warp[ROW_BLOCK / 32];
    __shared__ int64_t s_total;
    __shared__ int64_t s_off[ROW_BLOCK + 1];
    __shared__ unsigned char s_heavy[ROW_BLOCK];
    __shared__ int s_any_heavy;

    const int64_t tile = next_tile(A.ticket, &s_tile);
    const int tid = threadIdx.x;
    const int64_t r = tile * ROW_BLOCK + tid;  // local matrix row
    const bool active = r < A.nrows;
    const int64_t vl = r / RPV;
    const int s = int(r % RPV);
    const int64_t v = A.v0 + vl;
    if (tid == 0) s_any_heavy = 0;

    int64_t lo = 0, hi = 0;
    if (active) {
        lo = A.inc_ptr[vl];
        hi = A.inc_ptr[vl + 1];
    }
    const int deg = int(hi - lo);
    const bool heavy = active && deg > MAXD;
    int64_t count = 0, drops = 0;
    __syncthreads();

    if (active && !heavy) {
        uint32_t key[MAXD];
#pragma unroll
        for (int i = 0; i < MAXD; ++i) key[i] = i < deg ? A.inc[lo + i] : 0xffffffffu;
        sort8(key);

        int nb[NC];
        double ov[NC][NV];
        double dsum[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) dsum[t] = 0.0;
#pragma unroll
        for (int i = 0; i < MAXD; ++i) {
            if (i < deg) {
                const int64_t k = key[i] >> 2;
                const int a = key[i] & 3;
                const int c0 = A.me[3 * k], c1 = A.me[3 * k + 1], c2 = A.me[3 * k + 2];
                const int b1 = a == 2 ? 0 : a + 1, b2 = a == 0 ? 2 : a - 1;
                nb[2 * i] = sel3(b1, c0, c1, c2);
                nb[2 * i + 1] = sel3(b2, c0, c1, c2);
                const TriData<KIND> d = load_tri<KIND>(A, k, c0, c1, c2);
#pragma unroll
                for (int t = 0; t < NV; ++t) {
                    dsum[t] = FADD(dsum[t], tri_entry<KIND>(A, d, a, s, a, t));
                    ov[2 * i][t] = tri_entry<KIND>(A, d, a, s, b1, t);
                    ov[2 * i + 1][t] = tri_entry<KIND>(A, d, a, s, b2, t);
                }
            } else {
                nb[2 * i] = INT_MAX;
                nb[2 * i + 1] = INT_MAX;
#pragma unroll
                for (int t = 0; t < NV; ++t) ov[2 * i][t] = ov[2 * i + 1][t] = 0.0;
            }
        }
        // merge: vertex columns in ascending order (the row's own vertex included)
        const int vv = int(v);
        int last = -1;
        double* my_val = s_val + tid * STRIDE;
        int32_t* my_col = s_col + tid * STRIDE;
        while (true) {
            int c = INT_MAX;
#pragma unroll
            for (int j = 0; j < NC; ++j)
                if (nb[j] > last && nb[j] < c) c = nb[j];
            const bool diag = vv > last && vv < c;
            if (diag) c = vv;
            if (c == INT_MAX) break;
            double sum[NV];
            if (diag) {
#pragma unroll
                for (int t = 0; t < NV; ++t) sum[t] = dsum[t];
            } else {
#pragma unroll
                for (int t = 0; t < NV; ++t) sum[t] = 0.0;
#pragma unroll
                for (int j = 0; j < NC; ++j)
                    if (nb[j] == c) {
#pragma unroll
                        for (int t = 0; t < NV; ++t) sum[t] = FADD(sum[t], ov[j][t]);
                    }
            }
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                if (sum[t] != 0.0) {
                    my_col[count] = NV == 1 ? c : 2 * c + t;
                    my_val[count] = sum[t];
                    ++count;
                } else {
                    ++drops;
                }
            }
            last = c;
        }
    } else if (heavy) {
        count = heavy_row<KIND>(A, lo, hi, v, s, false, 0, &drops);
        s_any_heavy = 1;
    }
    s_heavy[tid] = heavy ? 1 : 0;

    // block scan + look-back: global offset of this tile's first row
    const int64_t excl = block_exclusive_scan<ROW_BLOCK>(count, s_warp, &s_total);
    s_off[tid] = excl;
    if (tid == ROW_BLOCK - 1) s_off[ROW_BLOCK] = excl + count;
    const uint64_t base = lookback_prefix(A.status, tile, uint64_t(s_total), &s_prefix);
    const int64_t total = s_total;

    if (active) A.rowptr[r] = int64_t(base) + excl;
    if (active && r == A.nrows - 1) {
        A.rowptr[A.nrows] = int64_t(base) + excl + count;
        A.res->nnz = int64_t(base) + excl + count;
    }
    if (drops) atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->dropped), (unsigned long long)drops);
    if (heavy) atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->heavy_rows), 1ull);

    // coalesced copy-out of the staged segment
    const bool any_heavy = s_any_heavy != 0;
    for (int64_t e = tid; e < total; e += ROW_BLOCK) {
        int lo_t = 0, hi_t = ROW_BLOCK;  // find t with s_off[t] <= e < s_off[t+1]
        while (hi_t - lo_t > 1) {
            const int mid = (lo_t + hi_t) >> 1;
            if (s_off[mid] <= e) lo_t = mid; else hi_t = mid;
        }
        if (any_heavy && s_heavy[lo_t]) continue;
        const int j = int(e - s_off[lo_t]);
        const int64_t g = int64_t(base) + e;
        if (g < A.capacity) {
            A.col[g] = s_col[lo_t * STRIDE + j];
            A.val[g] = s_val[lo_t * STRIDE + j];
        }
    }
    if (heavy) heavy_row<KIND>(A, lo, hi, v, s, true, int64_t(base) + excl, nullptr);
}

template <int KIND>
constexpr size_t rows_smem_bytes() {
    return size_t(ROW_BLOCK) * KindTraits<KIND>::STRIDE * (sizeof(double) + sizeof(int32_t));
}

template <int KIND>
static int launch_rows(const RowsArgs& A, int64_t ntiles, cudaStream_t st) {
    const size_t smem = rows_smem_bytes<KIND>();
    FA_CUDA(cudaFuncSetAttribute(k_rows<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_rows<KIND><<<dim3(unsigned(ntiles)), ROW_BLOCK, smem, st>>>(A);
    FA_LAUNCH_CHECK("k_rows");
    return FA_OK;
}

}  // namespace fa

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
struct fa_plan {
    int device;
    int64_t nme, nq, v0, v1;
    const int32_t* me;
    int* deg;                 // nv counts / fill cursors
    int64_t* inc_ptr;         // nv + 1
    uint32_t* inc;            // up to 3*nme keys
    uint64_t* status;         // look-back tile status (max of scan and row tiles)
    unsigned long long* ticket;
    int64_t status_len;
    int64_t ninc;             // -1 until read back
    bool built;
};

using namespace fa;

extern "C" int fa_plan_create(fa_plan** out, int64_t nme, int64_t nq, int64_t row_begin, int64_t row_end) {
    if (!out) { set_error("fa_plan_create: out is NULL"); return FA_ERR_ARGUMENT; }
    *out = nullptr;
    if (nme < 1 || nq < 1) { set_error("mesh needs at least one vertex and one triangle"); return FA_ERR_ARGUMENT; }
    if (row_begin < 0 || row_end > nq || row_begin > row_end) {
        set_error("row block [%lld, %lld) outside [0, %lld)", (long long)row_begin, (long long)row_end, (long long)nq);
        return FA_ERR_ARGUMENT;
    }
    if (nme >= (int64_t(1) << 30) || nq >= (int64_t(1) << 30)) {
        set_error("mesh too large: nme=%lld nq=%lld (limit 2^30 each)", (long long)nme, (long long)nq);
        return FA_ERR_TOO_LARGE;
    }
    fa_plan* p = new (std::nothrow) fa_plan();
    if (!p) { set_error("out of host memory"); return FA_ERR_ARGUMENT; }
    FA_CUDA(cudaGetDevice(&p->device));
    p->nme = nme; p->nq = nq; p->v0 = row_begin; p->v1 = row_end;
    const int64_t nv = row_end - row_begin;
    const int64_t scan_tiles = (nv + SCAN_BLOCK * SCAN_ITEMS - 1) / (SCAN_BLOCK * SCAN_ITEMS) + 1;
    const int64_t row_tiles = (2 * nv + ROW_BLOCK - 1) / ROW_BLOCK + 1;
    p->status_len = scan_tiles > row_tiles ? scan_tiles : row_tiles;
    p->ninc = -1;
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&p->deg, sizeof(int) * (nv + 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->inc_ptr, sizeof(int64_t) * (nv + 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->inc, sizeof(uint32_t) * 3 * nme);
    if (e == cudaSuccess) e = cudaMalloc(&p->status, sizeof(uint64_t) * p->status_len);
    if (e == cudaSuccess) e = cudaMalloc(&p->ticket, sizeof(unsigned long long));
    if (e != cudaSuccess) {
        cudaFree(p->deg); cudaFree(p->inc_ptr); cudaFree(p->inc); cudaFree(p->status); cudaFree(p->ticket);
        delete p;
        return cuda_status(e, "fa_plan_create: cudaMalloc");
    }
    *out = p;
    return FA_OK;
}

extern "C" int fa_plan_destroy(fa_plan* p) {
    if (!p) return FA_OK;
    cudaFree(p->deg); cudaFree(p->inc_ptr); cudaFree(p->inc); cudaFree(p->status); cudaFree(p->ticket);
    delete p;
    return FA_OK;
}

extern "C" int fa_plan_build(fa_plan* p, const int32_t* d_me, fa_result* d_res, void* stream) {
    if (!p || !d_me || !d_res) { set_error("fa_plan_build: NULL argument"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    const int64_t nv = p->v1 - p->v0;
    p->me = d_me;
    p->ninc = -1;
    p->built = true;
    k_reset_result<<<1, 32, 0, st>>>(d_res);
    FA_CUDA(cudaMemsetAsync(p->deg, 0, sizeof(int) * (nv + 1), st));
    const int tb = 256;
    k_incidence_count<<<grid_for(p->nme, tb), tb, 0, st>>>(d_me, p->nme, p->nq, p->v0, p->v1, p->deg, d_res);
    FA_LAUNCH_CHECK("k_incidence_count");
    const int64_t tiles = (nv + SCAN_BLOCK * SCAN_ITEMS - 1) / (SCAN_BLOCK * SCAN_ITEMS);
    if (nv == 0) {
        FA_CUDA(cudaMemsetAsync(p->inc_ptr, 0, sizeof(int64_t), st));
        return FA_OK;
    }
    FA_CUDA(cudaMemsetAsync(p->status, 0, sizeof(uint64_t) * (tiles + 1), st));
    FA_CUDA(cudaMemsetAsync(p->ticket, 0, sizeof(unsigned long long), st));
    k_scan_i32_to_i64<<<dim3(unsigned(tiles > 0 ? tiles : 1)), SCAN_BLOCK, 0, st>>>(p->deg, nv, p->inc_ptr, p->status,
                                                                                     p->ticket);
    FA_LAUNCH_CHECK("k_scan_i32_to_i64");
    k_incidence_fill<<<grid_for(p->nme, tb), tb, 0, st>>>(d_me, p->nme, p->nq, p->v0, p->v1, p->inc_ptr, p->deg,
                                                          p->inc);
    FA_LAUNCH_CHECK("k_incidence_fill");
    return FA_OK;
}

extern "C" int64_t fa_plan_rows(const fa_plan* p, int kind) {
    if (!p) return -1;
    return (p->v1 - p->v0) * (kind == FA_KIND_ELASTIC ? 2 : 1);
}

extern "C" int fa_plan_capacity(fa_plan* p, int kind, int64_t* capacity) {
    if (!p || !capacity || !p->built) { set_error("fa_plan_capacity: plan not built"); return FA_ERR_ARGUMENT; }
    if (kind < 0 || kind > 3) { set_error("unknown matrix kind %d", kind); return FA_ERR_ARGUMENT; }
    const int64_t nv = p->v1 - p->v0;
    if (p->ninc < 0) {
        if (p->v0 == 0 && p->v1 == p->nq) {
            p->ninc = 3 * p->nme;  // every corner is owned
        } else {
            FA_CUDA(cudaMemcpy(&p->ninc, p->inc_ptr + nv, sizeof(int64_t), cudaMemcpyDeviceToHost));
        }
    }
    // per vertex: at most 2*deg neighbours + itself; ELASTIC: 2 rows x 2 columns per vertex
    const int64_t per = (kind == FA_KIND_ELASTIC) ? 4 : 1;
    *capacity = per * (2 * p->ninc + nv);
    return FA_OK;
}

extern "C" int fa_assemble(fa_plan* p, int kind, const double* d_q, const double* d_areas, const double* d_w,
                           double lam, double mu, int64_t* d_rowptr, int32_t* d_col, double* d_val, int64_t capacity,
                           fa_result* d_res, void* stream) {
    if (!p || !p->built) { set_error("fa_assemble: plan not built"); return FA_ERR_ARGUMENT; }
    if (!d_rowptr || !d_col || !d_val || !d_res) { set_error("fa_assemble: NULL output"); return FA_ERR_ARGUMENT; }
    if (kind < 0 || kind > 3) { set_error("unknown matrix kind %d", kind); return FA_ERR_ARGUMENT; }
    if ((kind == FA_KIND_STIFF || kind == FA_KIND_ELASTIC || !d_areas) && !d_q) {
        set_error("fa_assemble: vertex coordinates required"); return FA_ERR_ARGUMENT;
    }
    if (kind == FA_KIND_MASSW && !d_w) { set_error("WEIGHTED_MASS requires a WeightField"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    const int64_t nrows = fa_plan_rows(p, kind);
    const int64_t ntiles = (nrows + ROW_BLOCK - 1) / ROW_BLOCK;
    k_reset_result<<<1, 32, 0, st>>>(d_res);
    if (nrows == 0) {
        FA_CUDA(cudaMemsetAsync(d_rowptr, 0, sizeof(int64_t), st));
        return FA_OK;
    }
    FA_CUDA(cudaMemsetAsync(p->status, 0, sizeof(uint64_t) * ntiles, st));
    FA_CUDA(cudaMemsetAsync(p->ticket, 0, sizeof(unsigned long long), st));
    RowsArgs A;
    A.inc_ptr = p->inc_ptr; A.inc = p->inc; A.me = p->me;
    A.q = reinterpret_cast<const double2*>(d_q); A.areas = d_areas; A.w = d_w;
    A.lam = lam; A.mu = mu;
    A.v0 = p->v0; A.nrows = nrows;
    A.rowptr = d_rowptr; A.col = d_col; A.val = d_val; A.capacity = capacity;
    A.status = p->status; A.ticket = p->ticket; A.res = d_res;
    switch (kind) {
        case FA_KIND_MASS: return launch_rows<FA_KIND_MASS>(A, ntiles, st);
        case FA_KIND_MASSW: return launch_rows<FA_KIND_MASSW>(A, ntiles, st);
        case FA_KIND_STIFF: return launch_rows<FA_KIND_STIFF>(A, ntiles, st);
        default: return launch_rows<FA_KIND_ELASTIC>(A, ntiles, st);
    }
}
