// OptV2 assembly on B200: vertex-bucket plan + fused row kernel (element values, Matlab
// sparse() summation, zero drop, row offsets, CSR write) for one block of vertex rows.
//
// Reference path replaced (pkg/src/femasm): assemble(..., OPTV2) assembly.py:419-452 ->
// _assemble_batched :400-416 -> build_ig_jg_p1[_vector] :162-192 + batch_kg_* :214-307 ->
// TripletBatch.to_csc sparse.py:318-329 -> csc_from_triplets :140-189.
//
// Design:
//   plan    K1 bucket count   vertices are grouped in buckets of BV consecutive ids; every
//                             (triangle k, corner a) is counted in its vertex's bucket
//                             (shared-memory histograms, one global atomic per block and bucket)
//           K2 bucket scan    bucket offsets (decoupled look-back scan)
//           K3 bucket scatter one 16-byte incidence record {k, n1, n2, vloc|a} per corner into
//                             its bucket (n1, n2 = the triangle's other two vertices)
//   numeric K4 rows           one block per bucket, one thread per matrix row: counting sort
//                             of the bucket's records by vertex in shared memory, the row's
//                             <= 8 records sorted by k in registers, inputs gathered (areas,
//                             q, w), that row of each element matrix computed bit-exactly,
//                             columns merged in ascending order with each position summed
//                             sequentially in ascending k (== stable argsort + bincount of the
//                             reference), exact-zero sums dropped, block scan + decoupled
//                             look-back for the global row offset, the bucket's CSR segment
//                             staged in shared memory and written coalesced.
// Rows with more than MAXD incident triangles (or buckets with more than IDX_CAP records)
// take a general O(d^2) path in separate phases of the same kernel.
#include <climits>
#include <cstdlib>
#include <new>

#include "fa_common.cuh"
#include "fa_element.cuh"

namespace fa {

constexpr int BV = 256;          // vertices per bucket
constexpr int MAXD = 8;          // incidences per row on the register fast path
constexpr int IDX_CAP = 4096;    // records per bucket indexable from shared memory
constexpr int SMEM_NB = 16384;   // buckets counted with shared-memory histograms
constexpr int PLAN_BLOCK = 512;
constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 8;

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

// ------------------------------------------------------------------------------------------
// plan kernels
// ------------------------------------------------------------------------------------------
struct PlanArgs {
    const int32_t* me;
    int64_t nme, nq, v0, v1;
    int64_t nb;         // buckets
    int64_t chunk;      // triangles per block
    int* bcount;        // nb
    int64_t* bptr;      // nb + 1
    unsigned* bcursor;  // nb
    uint4* rec;         // records
    fa_result* res;
};

// K1: per-bucket incidence counts.  SMEM: shared histogram (nb <= SMEM_NB).
template <bool SMEM>
__global__ void __launch_bounds__(PLAN_BLOCK) k_bucket_count(PlanArgs P) {
    extern __shared__ int s_hist[];
    if (SMEM) {
        for (int64_t b = threadIdx.x; b < P.nb; b += blockDim.x) s_hist[b] = 0;
        __syncthreads();
    }
    const int64_t k0 = blockIdx.x * P.chunk;
    const int64_t k1 = min(P.nme, k0 + P.chunk);
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int64_t v = P.me[3 * k + a];
            if (v < 0 || v >= P.nq) {
                atomic_min_i64(&P.res->index_error_pos, 3 * k + a);
                continue;
            }
            if (v < P.v0 || v >= P.v1) continue;
            const int64_t b = (v - P.v0) / BV;
            if (SMEM) atomicAdd(&s_hist[b], 1);
            else atomicAdd(&P.bcount[b], 1);
        }
    }
    if (SMEM) {
        __syncthreads();
        for (int64_t b = threadIdx.x; b < P.nb; b += blockDim.x)
            if (s_hist[b]) atomicAdd(&P.bcount[b], s_hist[b]);
    }
}

// K3: scatter incidence records into their buckets.
template <bool SMEM>
__global__ void __launch_bounds__(PLAN_BLOCK) k_bucket_scatter(PlanArgs P) {
    extern __shared__ unsigned s_pos[];
    const int64_t k0 = blockIdx.x * P.chunk;
    const int64_t k1 = min(P.nme, k0 + P.chunk);
    if (SMEM) {
        for (int64_t b = threadIdx.x; b < P.nb; b += blockDim.x) s_pos[b] = 0;
        __syncthreads();
        for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int64_t v = P.me[3 * k + a];
                if (v >= P.v0 && v < P.v1 && v < P.nq) atomicAdd(&s_pos[(v - P.v0) / BV], 1u);
            }
        }
        __syncthreads();
        for (int64_t b = threadIdx.x; b < P.nb; b += blockDim.x) {
            const unsigned c = s_pos[b];
            if (c) s_pos[b] = unsigned(P.bptr[b]) + atomicAdd(&P.bcursor[b], c);
        }
        __syncthreads();
    }
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const int c0 = P.me[3 * k], c1 = P.me[3 * k + 1], c2 = P.me[3 * k + 2];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int64_t v = sel3(a, c0, c1, c2);
            if (v < P.v0 || v >= P.v1 || v >= P.nq) continue;
            const int64_t vl = v - P.v0;
            const int64_t b = vl / BV;
            unsigned pos;
            if (SMEM) pos = atomicAdd(&s_pos[b], 1u);
            else pos = unsigned(P.bptr[b]) + atomicAdd(&P.bcursor[b], 1u);
            const int n1 = sel3(a, c1, c2, c0), n2 = sel3(a, c2, c0, c1);  // corners a+1, a+2
            P.rec[pos] = make_uint4(unsigned(k), unsigned(n1), unsigned(n2), (unsigned(vl % BV) << 2) | unsigned(a));
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
    const int64_t* bptr;
    const uint4* rec;
    const double2* q;
    const double* areas;  // nullable: recompute from q (bitwise compute_areas)
    const double* w;
    double lam, mu;
    int64_t v0, v1;       // owned vertices
    int64_t nrows;        // matrix rows produced (owned vertices * rows per vertex)
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
    static constexpr bool NEED_W = KIND == FA_KIND_MASSW;
    static constexpr bool CHECK_AREA = KIND != FA_KIND_MASSW;   // massw never checks (assembly.py:227-243)
    static constexpr int THREADS = BV * RPV;
    static constexpr int CAPR = KIND == FA_KIND_ELASTIC ? 16 : 2 * MAXD + 1;  // staged entries per row
    static constexpr int STRIDE = CAPR | 1;                                   // odd: conflict-free
};

// Per-thread data of the row's own vertex.
struct OwnVertex {
    int64_t v;
    double2 p;
    double w;
};

// Row (a, s) of one incident triangle's element matrix against the triangle's three
// vertices: d = entry at the row's own vertex, o1 / o2 = entries at n1 / n2.
template <int KIND>
__device__ __forceinline__ void row_values(const RowsArgs& A, const OwnVertex& own, uint4 r, int s,
                                           double (&d)[2], double (&o1)[2], double (&o2)[2]) {
    using TR = KindTraits<KIND>;
    const int64_t k = r.x;
    const int n1 = int(r.y), n2 = int(r.z), a = int(r.w & 3);
    const int b1 = a == 2 ? 0 : a + 1, b2 = a == 0 ? 2 : a - 1;
    double2 pa = own.p, p1 = make_double2(0.0, 0.0), p2 = p1;
    const bool need_pts = TR::NEED_Q || A.areas == nullptr;
    if (need_pts) {
        p1 = A.q[n1];
        p2 = A.q[n2];
    }
    // corners in triangle order
    const double2 c0 = sel3(a, pa, p2, p1), c1 = sel3(a, p1, pa, p2), c2 = sel3(a, p2, p1, pa);
    const double area = A.areas ? A.areas[k] : tri_area(c0, c1, c2);
    if (TR::CHECK_AREA && area <= AREA_EPS) atomic_min_i64(&A.res->degenerate_index, k);
    if constexpr (KIND == FA_KIND_MASS) {
        const MassTri t = mass_prepare(area);
        d[0] = t.d;
        o1[0] = t.o;
        o2[0] = t.o;
    } else if constexpr (KIND == FA_KIND_MASSW) {
        const double wa = own.w, w1 = A.w[n1], w2 = A.w[n2];
        const MasswTri t = massw_prepare(area, sel3(a, wa, w2, w1), sel3(a, w1, wa, w2), sel3(a, w2, w1, wa));
        d[0] = massw_entry(t, a, a);
        o1[0] = massw_entry(t, a, b1);
        o2[0] = massw_entry(t, a, b2);
    } else if constexpr (KIND == FA_KIND_STIFF) {
        const StiffTri t = stiff_prepare(c0, c1, c2, area);
        d[0] = stiff_entry(t, a, a);
        o1[0] = stiff_entry(t, a, b1);
        o2[0] = stiff_entry(t, a, b2);
    } else {
        const ElasticTri t = elastic_prepare(c0, c1, c2, area);
        const double P = FADD(A.lam, FMUL(2.0, A.mu));
        const int i = 2 * a + s;
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
            d[tt] = elastic_entry(t, i, 2 * a + tt, A.lam, A.mu, P);
            o1[tt] = elastic_entry(t, i, 2 * b1 + tt, A.lam, A.mu, P);
            o2[tt] = elastic_entry(t, i, 2 * b2 + tt, A.lam, A.mu, P);
        }
    }
}

__device__ __forceinline__ void cswap4(uint4& x, uint4& y) {
    const bool sw = x.x > y.x;
    const uint4 lo = sw ? y : x, hi = sw ? x : y;
    x = lo;
    y = hi;
}
// optimal 19-comparator network for 8 keys (verified by the 0-1 principle)
__device__ __forceinline__ void sort8(uint4 (&k)[8]) {
    cswap4(k[0], k[2]); cswap4(k[1], k[3]); cswap4(k[4], k[6]); cswap4(k[5], k[7]);
    cswap4(k[0], k[4]); cswap4(k[1], k[5]); cswap4(k[2], k[6]); cswap4(k[3], k[7]);
    cswap4(k[0], k[1]); cswap4(k[2], k[3]); cswap4(k[4], k[5]); cswap4(k[6], k[7]);
    cswap4(k[2], k[4]); cswap4(k[3], k[5]);
    cswap4(k[1], k[4]); cswap4(k[3], k[6]);
    cswap4(k[1], k[2]); cswap4(k[3], k[4]); cswap4(k[5], k[6]);
}

// Shared state of one bucket, visible to the general path.
struct BucketView {
    const uint4* rec;           // first record of the bucket
    int64_t n;                  // records in the bucket
    const unsigned short* idx;  // per-vertex lists (when !overflow)
    bool overflow;
};

// General path for one row (any degree): O(d^2) selection over the row's incidences with
// the same summation order (ascending k per position).  Writes only when `write`.
template <int KIND>
__device__ int64_t general_row(const RowsArgs& A, const BucketView& B, int start, int deg, int vloc,
                               const OwnVertex& own, int s, int64_t out_pos, bool write, int64_t* drops) {
    constexpr int NV = KindTraits<KIND>::NV;
    const int64_t m = B.overflow ? B.n : deg;
    auto get = [&](int64_t i, uint4& r) -> bool {
        if (B.overflow) {
            r = B.rec[i];
            return int(r.w >> 2) == vloc;
        }
        r = B.rec[B.idx[start + i]];
        return true;
    };
    int64_t last = -1, count = 0;
    while (true) {
        int64_t c = INT64_MAX;  // next vertex column
        if (own.v > last) c = own.v;
        for (int64_t i = 0; i < m; ++i) {
            uint4 r;
            if (!get(i, r)) continue;
            const int64_t x1 = r.y, x2 = r.z;
            if (x1 > last && x1 < c) c = x1;
            if (x2 > last && x2 < c) c = x2;
        }
        if (c == INT64_MAX) break;
        double sum[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) sum[t] = 0.0;
        int64_t prevk = -1;
        while (true) {  // contributions to column c in ascending k
            int64_t bestk = INT64_MAX;
            uint4 best = make_uint4(0, 0, 0, 0);
            for (int64_t i = 0; i < m; ++i) {
                uint4 r;
                if (!get(i, r)) continue;
                const int64_t k = r.x;
                if (k <= prevk || k >= bestk) continue;
                if (c == own.v || int64_t(r.y) == c || int64_t(r.z) == c) {
                    bestk = k;
                    best = r;
                }
            }
            if (bestk == INT64_MAX) break;
            double d[2], o1[2], o2[2];
            row_values<KIND>(A, own, best, s, d, o1, o2);
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                const double x = c == own.v ? d[t] : (int64_t(best.y) == c ? o1[t] : o2[t]);
                sum[t] = FADD(sum[t], x);
            }
            prevk = bestk;
        }
#pragma unroll
        for (int t = 0; t < NV; ++t) {
            if (sum[t] != 0.0) {
                if (write && out_pos + count < A.capacity) {
                    A.col[out_pos + count] = int32_t(NV == 1 ? c : 2 * c + t);
                    A.val[out_pos + count] = sum[t];
                }
                ++count;
            } else if (drops) {
                ++*drops;
            }
        }
        last = c;
    }
    return count;
}

template <int KIND>
__global__ void __launch_bounds__(KindTraits<KIND>::THREADS, 1) k_rows(RowsArgs A) {
    using TR = KindTraits<KIND>;
    constexpr int NV = TR::NV, RPV = TR::RPV, NT = TR::THREADS, STRIDE = TR::STRIDE, CAPR = TR::CAPR;
    constexpr int NC = 2 * MAXD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* s_val = reinterpret_cast<double*>(smem_raw);                 // [NT][STRIDE]
    int32_t* s_col = reinterpret_cast<int32_t*>(s_val + NT * STRIDE);   // [NT][STRIDE]
    __shared__ int s_cnt[BV];
    __shared__ int s_start[BV];
    __shared__ int s_fill[BV];
    __shared__ unsigned short s_idx[IDX_CAP];
    __shared__ int64_t s_tile;
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_warp[NT / 32];
    __shared__ int64_t s_total;
    __shared__ int64_t s_off[NT + 1];
    __shared__ unsigned char s_slow[NT];  // nonzero: row written outside the staging area

    const int tid = threadIdx.x;
    const int64_t b = next_tile(A.ticket, &s_tile);  // bucket, in launch order
    const int64_t lo = A.bptr[b], n = A.bptr[b + 1] - lo;
    const bool overflow = n > IDX_CAP;
    const uint4* brec = A.rec + lo;

    // ---- counting sort of the bucket's records by vertex (shared memory) ----------------
    for (int i = tid; i < BV; i += NT) {
        s_cnt[i] = 0;
        s_fill[i] = 0;
    }
    __syncthreads();
    for (int64_t i = tid; i < n; i += NT) atomicAdd(&s_cnt[brec[i].w >> 2], 1);
    __syncthreads();
    {
        const int c = tid < BV ? s_cnt[tid] : 0;
        const int64_t ex = block_exclusive_scan<NT>(int64_t(c), s_warp, &s_total);
        if (tid < BV) s_start[tid] = int(ex);
    }
    __syncthreads();
    if (!overflow) {
        for (int64_t i = tid; i < n; i += NT) {
            const int vl = brec[i].w >> 2;
            s_idx[s_start[vl] + atomicAdd(&s_fill[vl], 1)] = (unsigned short)i;
        }
    }
    __syncthreads();

    const int vloc = tid / RPV, s = tid % RPV;
    const int64_t v = A.v0 + b * BV + vloc;
    const bool active = v < A.v1;
    const int64_t r = (b * BV + vloc) * RPV + s;  // local matrix row
    const int deg = active ? s_cnt[vloc] : 0;
    const int start = active ? s_start[vloc] : 0;
    const bool slow = active && (deg > MAXD || overflow);
    OwnVertex own;
    own.v = v;
    own.p = make_double2(0.0, 0.0);
    own.w = 0.0;
    if (active) {
        if (TR::NEED_Q || A.areas == nullptr) own.p = A.q[v];
        if (TR::NEED_W) own.w = A.w[v];
    }
    BucketView B{brec, n, s_idx, overflow};
    int64_t count = 0, drops = 0;
    const bool any_slow = __syncthreads_or(slow);

    // ---- general path, counting phase ----------------------------------------------------
    if (any_slow && slow) count = general_row<KIND>(A, B, start, deg, vloc, own, s, 0, false, &drops);

    // ---- fast path: <= MAXD incidences in registers --------------------------------------
    bool spilled = false;
    if (active && !slow) {
        uint4 rr[MAXD];
#pragma unroll
        for (int i = 0; i < MAXD; ++i)
            rr[i] = i < deg ? brec[s_idx[start + i]] : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0);
        sort8(rr);
        int nb[NC];
        double ov[NC][NV];
        double dsum[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) dsum[t] = 0.0;
#pragma unroll
        for (int i = 0; i < MAXD; ++i) {
            double d[2], o1[2], o2[2];
            if (i < deg) {
                row_values<KIND>(A, own, rr[i], s, d, o1, o2);
                nb[2 * i] = int(rr[i].y);
                nb[2 * i + 1] = int(rr[i].z);
            } else {
                nb[2 * i] = INT_MAX;
                nb[2 * i + 1] = INT_MAX;
#pragma unroll
                for (int t = 0; t < 2; ++t) d[t] = o1[t] = o2[t] = 0.0;
            }
#pragma unroll
            for (int t = 0; t < NV; ++t) {
                dsum[t] = FADD(dsum[t], d[t]);
                ov[2 * i][t] = o1[t];
                ov[2 * i + 1][t] = o2[t];
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
            for (int j = 0; j < NC; ++j) c = min(c, nb[j] > last ? nb[j] : INT_MAX);
            const bool diag = vv > last && vv < c;
            if (diag) c = vv;
            if (c == INT_MAX) break;
            double sum[NV];
#pragma unroll
            for (int t = 0; t < NV; ++t) sum[t] = diag ? dsum[t] : 0.0;
            if (!diag) {
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
                    if (count < CAPR) {
                        my_col[count] = NV == 1 ? c : 2 * c + t;
                        my_val[count] = sum[t];
                    }
                    ++count;
                } else {
                    ++drops;
                }
            }
            last = c;
        }
        spilled = count > CAPR;
    }
    s_slow[tid] = (slow || spilled) ? 1 : 0;
    const bool any_spilled = __syncthreads_or(spilled);

    // ---- block scan + look-back: global offset of this bucket's first row ----------------
    const int64_t excl = block_exclusive_scan<NT>(count, s_warp, &s_total);
    s_off[tid] = excl;
    if (tid == NT - 1) s_off[NT] = excl + count;
    const uint64_t base = lookback_prefix(A.status, b, uint64_t(s_total), &s_prefix);
    const int64_t total = s_total;

    if (active) A.rowptr[r] = int64_t(base) + excl;
    if (active && r == A.nrows - 1) {
        A.rowptr[A.nrows] = int64_t(base) + excl + count;
        A.res->nnz = int64_t(base) + excl + count;
    }
    if (drops) atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->dropped), (unsigned long long)drops);
    if (slow) atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->heavy_rows), 1ull);

    // ---- coalesced copy-out of the staged segment ----------------------------------------
    const bool check_slow = any_slow || any_spilled;
    for (int64_t e = tid; e < total; e += NT) {
        int lt = 0, ht = NT;  // largest t with s_off[t] <= e
        while (ht - lt > 1) {
            const int mid = (lt + ht) >> 1;
            if (s_off[mid] <= e) lt = mid; else ht = mid;
        }
        if (check_slow && s_slow[lt]) continue;
        const int j = int(e - s_off[lt]);
        const int64_t g = int64_t(base) + e;
        if (g < A.capacity) {
            A.col[g] = s_col[lt * STRIDE + j];
            A.val[g] = s_val[lt * STRIDE + j];
        }
    }
    // ---- rows that did not fit the staging area or need the general path ---------------
    if (spilled || slow) general_row<KIND>(A, B, start, deg, vloc, own, s, int64_t(base) + excl, true, nullptr);
}

template <int KIND>
constexpr size_t rows_smem_bytes() {
    return size_t(KindTraits<KIND>::THREADS) * KindTraits<KIND>::STRIDE * (sizeof(double) + sizeof(int32_t));
}

template <int KIND>
static int launch_rows(const RowsArgs& A, int64_t nbuckets, cudaStream_t st) {
    const size_t smem = rows_smem_bytes<KIND>();
    FA_CUDA(cudaFuncSetAttribute(k_rows<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_rows<KIND><<<dim3(unsigned(nbuckets)), KindTraits<KIND>::THREADS, smem, st>>>(A);
    FA_LAUNCH_CHECK("k_rows");
    return FA_OK;
}

}  // namespace fa

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
struct fa_plan {
    int device;
    int64_t nme, nq, v0, v1, nb, chunk;
    const int32_t* me;
    int* bcount;              // nb + 1
    int64_t* bptr;            // nb + 1
    unsigned* bcursor;        // nb
    uint4* rec;               // up to 3*nme incidence records
    uint64_t* status;         // look-back tile status
    unsigned long long* ticket;
    int64_t status_len;
    int64_t ninc;             // -1 until read back
    bool built;
};

using namespace fa;

static void plan_free(fa_plan* p) {
    cudaFree(p->bcount); cudaFree(p->bptr); cudaFree(p->bcursor); cudaFree(p->rec);
    cudaFree(p->status); cudaFree(p->ticket);
}

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
    p->nb = (nv + BV - 1) / BV;
    // enough triangles per block that each bucket sees a few records per block
    int64_t chunk = 4096;
    while (chunk * 3 < 4 * p->nb && chunk < (int64_t(1) << 20)) chunk *= 2;
    p->chunk = chunk;
    const int64_t scan_tiles = (p->nb + SCAN_BLOCK * SCAN_ITEMS - 1) / (SCAN_BLOCK * SCAN_ITEMS) + 1;
    p->status_len = (scan_tiles > p->nb ? scan_tiles : p->nb) + 1;
    p->ninc = -1;
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&p->bcount, sizeof(int) * (p->nb + 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->bptr, sizeof(int64_t) * (p->nb + 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->bcursor, sizeof(unsigned) * (p->nb + 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->rec, sizeof(uint4) * 3 * nme);
    if (e == cudaSuccess) e = cudaMalloc(&p->status, sizeof(uint64_t) * p->status_len);
    if (e == cudaSuccess) e = cudaMalloc(&p->ticket, sizeof(unsigned long long));
    if (e != cudaSuccess) {
        plan_free(p);
        delete p;
        return cuda_status(e, "fa_plan_create: cudaMalloc");
    }
    *out = p;
    return FA_OK;
}

extern "C" int fa_plan_destroy(fa_plan* p) {
    if (!p) return FA_OK;
    plan_free(p);
    delete p;
    return FA_OK;
}

extern "C" int fa_plan_build(fa_plan* p, const int32_t* d_me, fa_result* d_res, void* stream) {
    if (!p || !d_me || !d_res) { set_error("fa_plan_build: NULL argument"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    p->me = d_me;
    p->ninc = -1;
    p->built = true;
    k_reset_result<<<1, 32, 0, st>>>(d_res);
    FA_CUDA(cudaMemsetAsync(p->bcount, 0, sizeof(int) * (p->nb + 1), st));
    FA_CUDA(cudaMemsetAsync(p->bcursor, 0, sizeof(unsigned) * (p->nb + 1), st));
    PlanArgs P{d_me, p->nme, p->nq, p->v0, p->v1, p->nb, p->chunk, p->bcount, p->bptr, p->bcursor, p->rec, d_res};
    const unsigned blocks = unsigned((p->nme + p->chunk - 1) / p->chunk);
    const bool smem = p->nb <= SMEM_NB;
    const size_t hist_bytes = smem ? sizeof(int) * size_t(p->nb) : 0;
    if (smem) {
        FA_CUDA(cudaFuncSetAttribute(k_bucket_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(hist_bytes)));
        FA_CUDA(cudaFuncSetAttribute(k_bucket_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(hist_bytes)));
        k_bucket_count<true><<<blocks, PLAN_BLOCK, hist_bytes, st>>>(P);
    } else {
        k_bucket_count<false><<<blocks, PLAN_BLOCK, 0, st>>>(P);
    }
    FA_LAUNCH_CHECK("k_bucket_count");
    if (p->nb == 0) {
        FA_CUDA(cudaMemsetAsync(p->bptr, 0, sizeof(int64_t), st));
        return FA_OK;
    }
    const int64_t tiles = (p->nb + SCAN_BLOCK * SCAN_ITEMS - 1) / (SCAN_BLOCK * SCAN_ITEMS);
    FA_CUDA(cudaMemsetAsync(p->status, 0, sizeof(uint64_t) * (tiles + 1), st));
    FA_CUDA(cudaMemsetAsync(p->ticket, 0, sizeof(unsigned long long), st));
    k_scan_i32_to_i64<<<dim3(unsigned(tiles)), SCAN_BLOCK, 0, st>>>(p->bcount, p->nb, p->bptr, p->status, p->ticket);
    FA_LAUNCH_CHECK("k_scan_i32_to_i64");
    if (smem) k_bucket_scatter<true><<<blocks, PLAN_BLOCK, hist_bytes, st>>>(P);
    else k_bucket_scatter<false><<<blocks, PLAN_BLOCK, 0, st>>>(P);
    FA_LAUNCH_CHECK("k_bucket_scatter");
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
            FA_CUDA(cudaMemcpy(&p->ninc, p->bptr + p->nb, sizeof(int64_t), cudaMemcpyDeviceToHost));
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
    k_reset_result<<<1, 32, 0, st>>>(d_res);
    if (nrows == 0 || p->nb == 0) {
        FA_CUDA(cudaMemsetAsync(d_rowptr, 0, sizeof(int64_t), st));
        return FA_OK;
    }
    FA_CUDA(cudaMemsetAsync(p->status, 0, sizeof(uint64_t) * p->nb, st));
    FA_CUDA(cudaMemsetAsync(p->ticket, 0, sizeof(unsigned long long), st));
    RowsArgs A;
    A.bptr = p->bptr; A.rec = p->rec;
    A.q = reinterpret_cast<const double2*>(d_q); A.areas = d_areas; A.w = d_w;
    A.lam = lam; A.mu = mu;
    A.v0 = p->v0; A.v1 = p->v1; A.nrows = nrows;
    A.rowptr = d_rowptr; A.col = d_col; A.val = d_val; A.capacity = capacity;
    A.status = p->status; A.ticket = p->ticket; A.res = d_res;
    switch (kind) {
        case FA_KIND_MASS: return launch_rows<FA_KIND_MASS>(A, p->nb, st);
        case FA_KIND_MASSW: return launch_rows<FA_KIND_MASSW>(A, p->nb, st);
        case FA_KIND_STIFF: return launch_rows<FA_KIND_STIFF>(A, p->nb, st);
        default: return launch_rows<FA_KIND_ELASTIC>(A, p->nb, st);
    }
}
