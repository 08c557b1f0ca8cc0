// OptV2 assembly on B200: vertex-sorted incidence plan + fused row kernel (element values,
// Matlab sparse() summation, zero drop, row offsets, CSR write) for one block of vertex rows.
//
// Reference path replaced (pkg/src/femasm): assemble(..., OPTV2) assembly.py:419-452 ->
// _assemble_batched :400-416 -> build_ig_jg_p1[_vector] :162-192 + batch_kg_* :214-307 ->
// TripletBatch.to_csc sparse.py:318-329 -> csc_from_triplets :140-189.
//
// Design.  Vertex and triangle numbering are arbitrary (the benchmark meshes are
// randomly permuted), so every access keyed by the "other" index is a random gather.  The plan
// turns the connectivity into per-vertex incidence lists that carry everything the numeric
// pass needs except floating-point data, so the numeric pass gathers only from the small,
// L2-resident arrays (areas 8 B/triangle, q 16 B/vertex, w 8 B/vertex):
//   plan (symbolic, reads `me` only)
//     K1 part_hist   owned incidences per (block, part) (parts = 1024 consecutive vertices)
//                    in shared memory, and per part; index validation
//     K2 part_scan   part offsets
//     K3 part_place  per round of triangles: incidence records {k, vertex-in-part<<2|a, n1, n2}
//                    ranked by part in shared memory, one range per (block, part) reserved once,
//                    staged in part order and written as coalesced runs
//     K3b part_split (two-level plans only: more than SPLIT_MIN parts, or records larger than
//                    L2) placement used coarse parts; rounds of records (any block) are
//                    regrouped by fine part, one range per (round, fine part); the block's
//                    next round is prefetched into L2
//     K4 part_sort   per part: counting sort by vertex in shared memory, each vertex's list
//                    ordered by k; written as SoA (k<<2|a, n1, n2) + per-vertex offsets ivptr;
//                    the records of a part sorted a little later are prefetched into L2
//   (K1 and K3 are issue-bound: 32-bit id arithmetic, shared arrays behind a register-held
//    32-bit shared address, loop invariants pinned in registers - fa_common.cuh smem_u32)
//   numeric
//     K5 rows        one block per bucket of BV vertices, ticket-ordered:
//                    s) plan entries into shared memory in one round trip; per row the 2*deg
//                       neighbour columns sorted with a 16-key odd-even merge network -> the
//                       row's symbolic entry count; block scan; for the scalar kinds the
//                       bucket's size is published to the decoupled look-back right away;
//                    a) per incidence (balanced over threads): the triangle area and the
//                       neighbour q / w gathered (L2-resident arrays, evict-last), the row of
//                       the element matrix computed bit-exactly into shared memory (gradients
//                       + area for elasticity);
//                    c) one thread per matrix row: a linear pass over the sorted columns sums
//                       every position sequentially in ascending k (== stable argsort +
//                       bincount of the reference); exact-zero sums stay as entries (scalar
//                       kinds) or are dropped at once (elasticity, which then publishes its
//                       exact count);
//                    d) the bucket's CSR segment staged in shared memory, look-back resolved,
//                       written coalesced.
//     K6 compact     only when a scalar-kind sum was exactly zero (Matlab drops it,
//                    sparse.py:177-179): removes those entries in place, bucket by bucket.
// Rows of degree > MAXD (and every row of a bucket whose incidences exceed CAPB) use an
// O(d^2) general path with the same summation order.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <new>

#include "fa_common.cuh"
#include "fa_element.cuh"

namespace fa {

constexpr int BV = 128;            // vertices per row bucket
// row kernel shape per kind: incidences held in shared memory per bucket (CAP), blocks per SM
// (register budget), incidences / W records in flight per thread in phase a (AU)
constexpr int CAPB = 8 * BV;       // mass: <= 128 registers, four blocks per SM
constexpr int CAPB_E = 7 * BV;     // elasticity: 12 values per incidence, two blocks per SM
// weighted mass (five blocks per SM, <= 102 registers): a smaller bucket leaves L1 more room; the
// mean degree of a planar triangulation is below 6, so overflowing buckets (general path) stay rare
constexpr int CAPB_W = 7 * BV;
constexpr int ROWS_MINB = 4, ROWS_MINB_W = 5, ROWS_MINB_E = 2;
constexpr int ROWS_AU = 3, ROWS_AU_W = 3, ROWS_AU_E = 1;
// stiffness: five blocks per SM (<= 102 registers, two incidences in flight per thread in phase
// a) and 832 incidences per bucket (6.5 per vertex: the mean degree is below 6, so overflowing
// buckets stay rare) - the smaller shared-memory carve-out leaves L1 the room that keeps a row's
// second gather of each neighbour (n1 of one incidence, n2 of the next) out of DRAM at C5
// (C3 numeric 853 -> 753 us, C5 15.2 -> 13.8 ms against four blocks of 1024 incidences)
constexpr int ROWS_MINB_S = 5, CAPB_S = 832, ROWS_AU_S = 2;
constexpr int MAXD = 8;            // incidences per row on the register fast path
constexpr int PLOG0 = 10;          // log2 of the minimum part size (vertices)
constexpr int PLAN_THREADS = 1024;
constexpr int SORT_THREADS = 512;   // k_part_sort (2 blocks / SM, 64 registers)
constexpr int PLACE_THREADS = 1024;  // k_part_hist / k_part_place block size
constexpr int PLACE_BLOCKS_PER_SM = 1;
constexpr int PLACE_TRI = 2048;    // triangles per placement round
constexpr int SPLIT_MIN = 8192;    // fine parts above which placement goes through coarse parts
// records above this size do not stay in L2 between placement and sort, so the placement's
// runs must be long (coarse parts) and a parallel split regroups them by fine part
constexpr int64_t SPLIT_BYTES = int64_t(160) << 20;
constexpr int SPLIT_COARSE = 256;  // coarse parts of a two-level plan (at most)
constexpr int FINE_HIST_MAX = 98304;  // fine parts counted in k_part_hist's shared memory (16 bit)
// k_part_split: two blocks of 512 threads per SM, rounds of 4096 records (C5 split 3.37 ->
// 2.5 ms against one block of 1024 threads with 6144-record rounds: a block's load, rank and
// write phases overlap the other block's)
constexpr int SPLIT_THREADS = 512;
constexpr int SPLIT_RI = 4096;      // records per k_part_split round
constexpr int SPLIT_MINB = 2;       // k_part_split blocks per SM
constexpr int SPLIT2_LOCAL = SPLIT_THREADS;  // fine parts a k_part_split round ranks in shared memory
// L2 prefetch distances of the streaming plan kernels (measured on C5 / C3: k_part_sort 1 / 2 / 3 /
// 4 x the SM count: plan 8.03 / 8.04 / 8.21 / 8.51 ms and 530 / 539 / 554 / 561 us against 8.34 ms /
// 545 us without; k_part_split one / two rounds ahead: 8.04 / 8.10 ms against 8.43 ms without)
constexpr int SORT_PF_SMS = 1;   // k_part_sort: the part SORT_PF_SMS * (SM count) blocks ahead
constexpr int SORT_CAP = 6912;     // part incidences sorted in shared memory (6.75 per vertex; 2 blocks / SM)

// Resets the result block and zeroes the counters the following kernels accumulate into
// (grid-stride; replaces separate memsets).
__global__ void k_reset(fa_result* r, unsigned* z32, int64_t n32, uint64_t* z64, int64_t n64) {
    pdl_enter();
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n32; i += stride) z32[i] = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n64; i += stride) z64[i] = 0;
    if (threadIdx.x == 0 && blockIdx.x == 0) reset_result_fields(r);
}

__device__ __forceinline__ void load_tri_ids(const int32_t* me, int64_t k, int& c0, int& c1, int& c2) {
    c0 = me[3 * k];
    c1 = me[3 * k + 1];
    c2 = me[3 * k + 2];
}

// ------------------------------------------------------------------------------------------
// plan
// ------------------------------------------------------------------------------------------
struct PlanArgs {
    const int32_t* me;
    int64_t nme, nq, v0, v1;
    int plog;               // part = (v - v0) >> plog
    int nparts;
    int plog_f, nparts_f;   // fine parts (== the above unless a two-level plan)
    bool fine_hist;         // two-level: K1 counts fine parts, K2 derives the coarse offsets
    bool fine_global;       // fine parts beyond FINE_HIST_MAX: counted with global atomics
    unsigned* part_off_f;   // nparts_f + 1: fine counts (K1), offsets (K2)
    unsigned* fine_fill;    // nparts_f: k_part_split cursors
    int64_t chunk;          // triangles per block of K1 / K3
    unsigned* part_off;     // nparts + 1: counts (K1), exclusive offsets (K2)
    unsigned* part_fill;    // nparts: placement cursors
    unsigned* M;            // [blocks][nparts]: owned incidences of each K1/K3 block per part
    uint4* rec;             // owned incidences grouped by part {k, vl << 2 | a, n1, n2}, vl = v - v0
    unsigned* skey;         // sorted by (vertex, k): k << 2 | a
    unsigned* sn1;          // neighbour at corner a+1
    unsigned* sn2;          // neighbour at corner a+2
    unsigned* ivptr;        // nv + 1: first incidence of every owned vertex
    fa_result* res;
    // row blocks (multi-GPU): K1 compacts the triangles with an owned corner per block
    // ({k, c0, c1, c2} at block * chunk ..), so K3 skips the others
    uint4* tri;             // null for the whole mesh
    unsigned* tri_cnt;      // per K1/K3 block
    // weighted mass (fa_assemble_cold): K1 also writes the triangles' W records (k_tri_wt's
    // work, from the connectivity it reads anyway); null otherwise
    const double* wt_areas;
    const double* wt_w;
    double4* Wt;
    int sort_pf;            // K4: parts ahead whose records are prefetched into L2 (the blocks resident at once)
};

// a triangle takes part only with three in-range, pairwise distinct vertex ids
// (vertex counts stay below 2^28, fa_plan_create: every comparison here and in the plan kernels is 32 bit)
__device__ __forceinline__ bool tri_ids_valid(int c0, int c1, int c2, unsigned nq) {
    return unsigned(c0) < nq && unsigned(c1) < nq && unsigned(c2) < nq && c0 != c1 && c1 != c2 && c0 != c2;
}

__device__ __forceinline__ void tri_wt_store(double4* Wt, int64_t k, double ar, const double (&wc)[3], uint64_t keep);

// K1's W records for triangles [k0, k1) (weighted mass, cold path): k_tri_wt's work on this
// block's chunk, the connectivity reread from L2 right after the histogram pass
__device__ __forceinline__ void hist_tri_wt(const PlanArgs& P, int64_t k0, int64_t k1) {
    const uint64_t pol = l2_evict_first_policy();
    const uint64_t keep = l2_evict_last_policy();
    constexpr int U = 2;  // triangles in flight per thread
    for (int64_t k0u = k0 + threadIdx.x; k0u < k1; k0u += U * PLACE_THREADS) {
        int c[U][3];
        double ar[U], wc[U][3];
        bool own[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = k0u + u * PLACE_THREADS;
            c[u][0] = c[u][1] = c[u][2] = -1;
            if (k < k1) {
                load_tri_ids(P.me, k, c[u][0], c[u][1], c[u][2]);
                ar[u] = ld_stream_f64(P.wt_areas + k, pol);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            bool any = false;
#pragma unroll
            for (int a = 0; a < 3; ++a) any |= unsigned(c[u][a]) - unsigned(P.v0) < unsigned(P.v1 - P.v0);
            own[u] = k0u + u * PLACE_THREADS < k1 && any;
            if (own[u])
#pragma unroll
                for (int a = 0; a < 3; ++a)  // out-of-range ids (reported by the histogram) read nothing
                    wc[u][a] = unsigned(c[u][a]) < unsigned(P.nq) ? ld_keep_f64(P.wt_w + c[u][a], keep) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (own[u]) tri_wt_store(P.Wt, k0u + u * PLACE_THREADS, ar[u], wc[u], keep);
    }
}

// K1: owned incidences per (block, part) and per part; index validation (sparse.py:131-137 semantics: first bad
// position in the flattened connectivity).  Two-level plans count the fine parts (the coarse counts are their
// sums) in 16-bit counters packed two per shared word, so up to FINE_HIST_MAX fine parts fit (C5: 65,553); a
// counter that wraps hands 65536 to the global fine count and to the block's coarse count and takes its carry
// back out of its neighbour.  Beyond FINE_HIST_MAX fine parts the fine counts go to global atomics and shared
// memory keeps the coarse ones.
// The shared-memory counters are addressed through a 32-bit shared address kept in a register
// (smem_u32, fa_common.cuh) and the wrap handling stays out of line: the histogram is
// issue-bound, every instruction of its per-corner path counts.
__device__ __noinline__ void hist_wrap16(unsigned* s_cnt, unsigned* g_fine, unsigned* s_cwrap, unsigned f,
                                         int fine_per_coarse_log2) {
    if ((f & 1u) == 0) atomicSub(&s_cnt[f >> 1], 1u << 16);  // the carry went into the neighbour
    atomicAdd(&g_fine[f], 65536u);
    atomicAdd(&s_cwrap[f >> fine_per_coarse_log2], 1u);
}

// MODE 0: single-level plan (counts per part in shared memory); 1: two-level, fine counts in
// shared memory (16 bit); 2: two-level, fine counts in global memory, coarse ones in shared.
// RB: row block (the triangles with an owned corner are compacted for the placement).
template <int MODE, bool RB>
__global__ void __launch_bounds__(PLACE_THREADS) k_part_hist(const __grid_constant__ PlanArgs P) {
    pdl_enter();
    extern __shared__ unsigned s_cnt[];
    constexpr bool fs = MODE == 1;  // fine counts in shared memory (16 bit)
    const int hn = fs ? (P.nparts_f + 1) / 2 : P.nparts;
    __shared__ unsigned s_tn;
    __shared__ unsigned s_cwrap[SPLIT_COARSE];  // wrapped fine counters per coarse part
    for (int i = threadIdx.x; i < hn; i += PLACE_THREADS) s_cnt[i] = 0;
    for (int i = threadIdx.x; i < SPLIT_COARSE; i += PLACE_THREADS) s_cwrap[i] = 0;
    if (threadIdx.x == 0) s_tn = 0;
    __syncthreads();
    const int64_t k0 = int64_t(blockIdx.x) * P.chunk, k1 = min(P.nme, k0 + P.chunk);
    const unsigned nq32 = unsigned(P.nq), v032 = unsigned(P.v0), nv32 = unsigned(P.v1 - P.v0);
    const unsigned cnt_sa = smem_u32(s_cnt), tn_sa = smem_u32(&s_tn);
    const int plog = P.plog, plog_f = P.plog_f;
    constexpr int U = 4;  // triangles per thread per iteration; the next iteration's are loaded
                          // while these are counted
    int nx[U][3];
    unsigned nk = unsigned(k1 - k0);  // (a block's chunk is far below 2^31 triangles)
    const int32_t* meb = P.me + 3 * k0;
    uint4* trib = RB ? P.tri + k0 : nullptr;
    // (kept in registers: the compiler otherwise recomputes them from blockIdx and the kernel
    //  parameters at every use inside the loop)
    asm volatile("" : "+r"(nk), "+l"(meb), "+l"(trib));
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const unsigned j = threadIdx.x + u * PLACE_THREADS;
        if (j < nk) load_tri_ids(meb, j, nx[u][0], nx[u][1], nx[u][2]);
    }
    for (unsigned j0 = threadIdx.x; j0 < nk; j0 += U * PLACE_THREADS) {
        int c[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c[u][0] = nx[u][0];
            c[u][1] = nx[u][1];
            c[u][2] = nx[u][2];
            const unsigned j = j0 + (U + u) * PLACE_THREADS;
            if (j < nk) load_tri_ids(meb, j, nx[u][0], nx[u][1], nx[u][2]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned j = j0 + u * PLACE_THREADS;
            if (j >= nk) break;
            // a triangle with an out-of-range or repeated corner is reported (first bad position
            // in the flattened connectivity) and left out entirely, so no incidence ever names an
            // invalid neighbour
            if (!tri_ids_valid(c[u][0], c[u][1], c[u][2], nq32)) {
                const int64_t k = k0 + j;
                if (c[u][0] == c[u][1] || c[u][1] == c[u][2] || c[u][0] == c[u][2])  // first repeating corner
                    atomic_min_i64(&P.res->repeat_error_pos, 3 * k + (c[u][0] == c[u][1] ? 1 : 2));
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    if (unsigned(c[u][a]) >= nq32) atomic_min_i64(&P.res->index_error_pos, 3 * k + a);
                continue;
            }
            // owned corners: v0 <= v < v1 (<= nq) in one unsigned comparison
            unsigned vl[3];
            bool own[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                vl[a] = unsigned(c[u][a]) - v032;
                own[a] = vl[a] < nv32;
            }
            if (RB && (own[0] || own[1] || own[2]))  // (same-address shared atomics of a warp are combined in hardware)
                trib[atoms_add_u32(tn_sa, 1u)] =
                    make_uint4(unsigned(k0 + j), unsigned(c[u][0]), unsigned(c[u][1]), unsigned(c[u][2]));
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (own[a]) {
                    if (fs) {
                        const unsigned f = vl[a] >> plog_f, sh = (f & 1u) << 4;
                        const unsigned old = atoms_add_u32(cnt_sa + ((f >> 1) << 2), 1u << sh);
                        if (((old >> sh) & 0xffffu) == 0xffffu)  // wrapped (a block rarely sees 65536 incidences of one fine part)
                            hist_wrap16(s_cnt, P.part_off_f, s_cwrap, f, plog - plog_f);
                    } else {
                        reds_add_u32(cnt_sa + ((vl[a] >> plog) << 2), 1u);
                        if (MODE == 2) atomicAdd(&P.part_off_f[vl[a] >> plog_f], 1u);
                    }
                }
            }
        }
    }
    __syncthreads();
    if (P.Wt) hist_tri_wt(P, k0, k1);
    if (RB && threadIdx.x == 0) P.tri_cnt[blockIdx.x] = s_tn;
    unsigned* row = P.M + int64_t(blockIdx.x) * P.nparts;
    auto fine = [&](int f) { return (s_cnt[f >> 1] >> ((f & 1) * 16)) & 0xffffu; };
    if (MODE == 0) {
        for (int i = threadIdx.x; i < P.nparts; i += PLACE_THREADS) {
            row[i] = s_cnt[i];
            if (s_cnt[i]) atomicAdd(&P.part_off[i], s_cnt[i]);
        }
    } else if (MODE == 2) {
        for (int i = threadIdx.x; i < P.nparts; i += PLACE_THREADS) row[i] = s_cnt[i];
    } else {
        for (int i = threadIdx.x; i < P.nparts_f; i += PLACE_THREADS) {
            const unsigned c = fine(i);
            if (c) atomicAdd(&P.part_off_f[i], c);
        }
        // coarse counts of this block (the placement's count-matrix row): sums of its fine
        // counts plus 65536 per wrapped fine counter
        const int F = 1 << (P.plog - P.plog_f);
        for (int pc = threadIdx.x; pc < P.nparts; pc += PLACE_THREADS) {
            unsigned c = 65536u * s_cwrap[pc];
            for (int f = pc * F; f < min((pc + 1) * F, P.nparts_f); ++f) c += fine(f);
            row[pc] = c;
        }
    }
}

// K2: exclusive scan of the part counts (one block, any part count).  Two-level plans with
// fine counts (K1 fine_hist): the fine offsets, the split cursors, and the coarse offsets and
// placement cursors taken at the coarse boundaries.
// Tiles of PLAN_THREADS * per counts (per <= SCAN_PER, from the launch: small plans take one
// count per thread) go through shared memory: coalesced in, each thread scans its `per`
// consecutive counts, coalesced out.
constexpr int SCAN_PER = 32;
static int scan_per(int n) { return std::max(1, std::min(SCAN_PER, (n + PLAN_THREADS - 1) / PLAN_THREADS)); }
static size_t scan_smem_bytes(int per) { return sizeof(unsigned) * size_t(PLAN_THREADS * per + (PLAN_THREADS * per) / 32); }
__global__ void __launch_bounds__(PLAN_THREADS) k_part_scan(const __grid_constant__ PlanArgs P, int per) {
    pdl_enter();
    extern __shared__ unsigned s_tile[];  // [tile + tile / 32]: index i at i + i / 32 (conflict-free for per = 32)
    const int SCAN_TILE = PLAN_THREADS * per;
    __shared__ unsigned s_warp[PLAN_THREADS / 32];
    __shared__ unsigned s_total;
    unsigned* cnt = P.fine_hist ? P.part_off_f : P.part_off;
    unsigned* fill = P.fine_hist ? P.fine_fill : P.part_fill;
    const int n = P.fine_hist ? P.nparts_f : P.nparts;
    const int tid = threadIdx.x;
    unsigned carry = 0;
    for (int base = 0; base < n; base += SCAN_TILE) {
        const int m = min(SCAN_TILE, n - base);
        for (int i = tid; i < m; i += PLAN_THREADS) s_tile[i + (i >> 5)] = cnt[base + i];
        __syncthreads();
        // thread t owns counts [per t, per t + per) of the tile
        const int i0 = tid * per;
        unsigned run = 0;
        for (int j = 0; j < per; ++j) run += i0 + j < m ? s_tile[i0 + j + ((i0 + j) >> 5)] : 0u;
        unsigned ex = carry + block_exclusive_scan<PLAN_THREADS>(run, s_warp, &s_total);
        for (int j = 0; j < per; ++j) {
            if (i0 + j < m) {
                const int at = i0 + j + ((i0 + j) >> 5);
                const unsigned c = s_tile[at];
                s_tile[at] = ex;
                ex += c;
            }
        }
        __syncthreads();
        for (int i = tid; i < m; i += PLAN_THREADS) {
            const unsigned o = s_tile[i + (i >> 5)];
            cnt[base + i] = o;
            fill[base + i] = o;
        }
        carry += s_total;
        __syncthreads();  // the tile and s_total are reused
    }
    if (tid == 0) cnt[n] = carry;
    if (!P.fine_hist) return;
    __syncthreads();  // fine offsets visible to the block
    const int F = 1 << (P.plog - P.plog_f);
    for (int pc = tid; pc <= P.nparts; pc += PLAN_THREADS) {
        const unsigned o = pc < P.nparts ? cnt[pc * F] : carry;
        P.part_off[pc] = o;
        if (pc < P.nparts) P.part_fill[pc] = o;
    }
}

// K3: incidence records grouped by part.  Each block reserves its range in every part once
// (count matrix row of K1, one atomic per part); per round of PLACE_TRI triangles the records
// are ranked by part in shared memory, staged in part order and written as coalesced runs.
// Order inside a part is arbitrary (K4 sorts).
// Shared layout: staging [RI] uint4, then per part the round counts, the round's local starts
// and the global cursors - all addressed from one 32-bit shared base (smem_u32); the copy-out
// reads a staged record's part from the record itself.  RB: row block (the triangles K1 compacted).
template <bool RB>
__global__ void __launch_bounds__(PLACE_THREADS, PLACE_BLOCKS_PER_SM) k_part_place(const __grid_constant__ PlanArgs P) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int RI = 3 * PLACE_TRI;                  // incidences per round
    constexpr int TPT = PLACE_TRI / PLACE_THREADS;      // triangles per thread per round
    __shared__ unsigned s_warp[PLACE_THREADS / 32];
    __shared__ unsigned s_total;
    unsigned tid = threadIdx.x;
    unsigned nparts = unsigned(P.nparts);
    const unsigned stage_sa = smem_u32(smem_raw);              // [RI] uint4
    const unsigned cnt_sa = stage_sa + RI * 16;                  // [nparts] round counts
    const unsigned lst_sa = cnt_sa + 4 * nparts;                 // [nparts] round local starts
    const unsigned gb_sa = lst_sa + 4 * nparts;                  // [nparts] global cursors
    const int64_t kb0 = int64_t(blockIdx.x) * P.chunk, kb1 = min(P.nme, kb0 + P.chunk);
    {
        const unsigned* row = P.M + int64_t(blockIdx.x) * P.nparts;
        for (unsigned i = tid; i < nparts; i += PLACE_THREADS) {
            const unsigned c = row[i];
            sts_u32(gb_sa + 4 * i, c ? atomicAdd(&P.part_fill[i], c) : 0u);
            sts_u32(cnt_sa + 4 * i, 0u);
        }
    }
    // this block's triangles: its chunk of the mesh, or (row blocks) the ones K1 compacted
    unsigned nj = RB ? P.tri_cnt[blockIdx.x] : unsigned(kb1 - kb0);  // (a chunk is far below 2^31 triangles)
    const int32_t* meb = P.me + 3 * kb0;
    const uint4* trib = RB ? P.tri + kb0 : nullptr;
    unsigned kb032 = unsigned(kb0);  // triangle ids fit 30 bits (fa_plan_create)
    unsigned nq32 = unsigned(P.nq), v032 = unsigned(P.v0), nv32 = unsigned(P.v1 - P.v0);
    uint4* recb = P.rec;
    // (kept in registers: the compiler otherwise recomputes them from the special registers and
    //  the kernel parameters at every use inside the loop)
    asm volatile("" : "+r"(tid), "+r"(nparts), "+r"(nj), "+l"(meb), "+l"(trib), "+r"(kb032), "+l"(recb));
    const int plog = P.plog;
    auto fetch = [&](unsigned j, unsigned& k, int (&c)[3]) {
        c[0] = c[1] = c[2] = -1;
        if (j >= nj) return;
        if (RB) {
            const uint4 t = trib[j];
            k = t.x; c[0] = int(t.y); c[1] = int(t.z); c[2] = int(t.w);
        } else {
            k = kb032 + j;
            load_tri_ids(meb, j, c[0], c[1], c[2]);
        }
    };
    // triangle ids of the next round are loaded while the current one is placed
    int nxt[TPT][3];
    unsigned nk[TPT];
#pragma unroll
    for (int t = 0; t < TPT; ++t) fetch(t * PLACE_THREADS + tid, nk[t], nxt[t]);
    for (unsigned r0 = 0; r0 < nj; r0 += PLACE_TRI) {
        int cur[TPT][3];
        unsigned ck[TPT];
#pragma unroll
        for (int t = 0; t < TPT; ++t) {
            cur[t][0] = nxt[t][0];
            cur[t][1] = nxt[t][1];
            cur[t][2] = nxt[t][2];
            ck[t] = nk[t];
            fetch(r0 + PLACE_TRI + t * PLACE_THREADS + tid, nk[t], nxt[t]);
        }
        __syncthreads();
        uint4 rec[3 * TPT];
        unsigned part[3 * TPT], rank[3 * TPT];
#pragma unroll
        for (int t = 0; t < TPT; ++t) {
            const unsigned k = ck[t];
            const int c[3] = {cur[t][0], cur[t][1], cur[t][2]};
            const bool ok = tri_ids_valid(c[0], c[1], c[2], nq32);  // as k_part_hist (-1: no triangle)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int j = 3 * t + a;
                part[j] = 0xffffffffu;
                const unsigned vl = unsigned(c[a]) - v032;  // owned: v0 <= v < v1 (<= nq)
                if (ok && vl < nv32) {
                    part[j] = vl >> plog;
                    rank[j] = atoms_add_u32(cnt_sa + 4 * part[j], 1u);
                    rec[j] = make_uint4(unsigned(k), (vl << 2) | unsigned(a),
                                        unsigned(sel3(a, c[1], c[2], c[0])), unsigned(sel3(a, c[2], c[0], c[1])));
                }
            }
        }
        __syncthreads();
        // local starts: exclusive scan of the round counts over parts
        const unsigned per = (nparts + PLACE_THREADS - 1) / PLACE_THREADS;
        unsigned run = 0;
        for (unsigned j = 0; j < per; ++j) {
            const unsigned i = tid * per + j;
            run += i < nparts ? lds_u32(cnt_sa + 4 * i) : 0u;
        }
        unsigned ex = block_exclusive_scan<PLACE_THREADS>(run, s_warp, &s_total);
        for (unsigned j = 0; j < per; ++j) {
            const unsigned i = tid * per + j;
            if (i < nparts) {
                sts_u32(lst_sa + 4 * i, ex);
                ex += lds_u32(cnt_sa + 4 * i);
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 3 * TPT; ++j) {
            if (part[j] != 0xffffffffu) {
                const unsigned pos = lds_u32(lst_sa + 4 * part[j]) + rank[j];
                FA_DCHECK(pos < unsigned(RI), "placement staging index");
                sts_v4(stage_sa + 16 * pos, rec[j]);
            }
        }
        __syncthreads();
        const unsigned total = s_total;
        for (unsigned i = tid; i < total; i += PLACE_THREADS) {
            const uint4 r = lds_v4(stage_sa + 16 * i);
            const unsigned pp = (r.y >> 2) >> plog;  // the staged record names its part
            const unsigned g = lds_u32(gb_sa + 4 * pp) + (i - lds_u32(lst_sa + 4 * pp));
            FA_DCHECK(int64_t(g) < 3 * P.nme, "placement record index");
            asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(recb + g), "r"(r.x),
                         "r"(r.y), "r"(r.z), "r"(r.w)
                         : "memory");
        }
        __syncthreads();
        for (unsigned i = tid; i < nparts; i += PLACE_THREADS) {  // advance the cursors, reset the counts
            sts_u32(gb_sa + 4 * i, lds_u32(gb_sa + 4 * i) + lds_u32(cnt_sa + 4 * i));
            sts_u32(cnt_sa + 4 * i, 0u);
        }
    }
}

// K3b (two-level plans): the placement's records regrouped by fine part,
// in parallel over rounds of 3 * PLACE_TRI consecutive records (any block, any coarse part):
// ranked by fine part in shared memory (relative to the round's smallest fine part), one range
// per fine part reserved from the global cursors (K2), staged and written as coalesced runs.
// Records whose fine part lies beyond the local window (only when coarse parts are smaller
// than a round) take a cursor each.
__global__ void __launch_bounds__(SPLIT_THREADS, SPLIT_MINB)
    k_part_split(const uint4* __restrict__ rec, const unsigned* __restrict__ total_ptr, int plog,
                  unsigned* __restrict__ fine_fill, uint4* __restrict__ rec2) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int RI = SPLIT_RI;
    constexpr int PER = RI / SPLIT_THREADS;
    uint4* s_stage = reinterpret_cast<uint4*>(smem_raw);                       // [RI]
    unsigned* s_cnt = reinterpret_cast<unsigned*>(s_stage + RI);             // [SPLIT2_LOCAL]
    unsigned* s_lst = s_cnt + SPLIT2_LOCAL;                                  // [SPLIT2_LOCAL]
    unsigned* s_gb = s_lst + SPLIT2_LOCAL;                                   // [SPLIT2_LOCAL]
    __shared__ unsigned s_fbase, s_total;
    __shared__ unsigned s_warp[SPLIT_THREADS / 32];
    static_assert(SPLIT_THREADS == SPLIT2_LOCAL, "one local fine part per thread in the scan");
    const int tid = threadIdx.x;
    const unsigned total = *total_ptr;
    const uint64_t pol = l2_evict_first_policy();
    s_cnt[tid] = 0;
    for (unsigned r0 = blockIdx.x * unsigned(RI); r0 < total; r0 += gridDim.x * unsigned(RI)) {
        if (tid == 0) s_fbase = 0xffffffffu;
        uint4 r[PER];
        unsigned f[PER], rank[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const unsigned i = r0 + u * SPLIT_THREADS + tid;
            f[u] = 0xffffffffu;
            if (i < total) {
                asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                             : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w)
                             : "l"(rec + i), "l"(pol));
                f[u] = (r[u].y >> 2) >> plog;
            }
        }
        {   // this block's next round -> L2 while the current one is ranked (one 128-byte line per thread)
            const uint64_t rn = uint64_t(r0) + uint64_t(gridDim.x) * RI + unsigned(tid) * (128 / sizeof(uint4));
            if (rn < total) prefetch_l2(rec + rn);
        }
        unsigned fmin = 0xffffffffu;
#pragma unroll
        for (int u = 0; u < PER; ++u) fmin = min(fmin, f[u]);
        fmin = __reduce_min_sync(0xffffffffu, fmin);
        __syncthreads();  // s_fbase reset (and the previous round's reads) done
        if ((tid & 31) == 0) atomicMin(&s_fbase, fmin);
        __syncthreads();
        const unsigned fb = s_fbase;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            if (f[u] == 0xffffffffu) continue;
            const unsigned l = f[u] - fb;
            if (l < unsigned(SPLIT2_LOCAL)) {
                rank[u] = atomicAdd(&s_cnt[l], 1u);
            } else {  // outside the local window: a cursor of its own
                rec2[atomicAdd(&fine_fill[f[u]], 1u)] = r[u];
                f[u] = 0xffffffffu;
            }
        }
        __syncthreads();
        const unsigned c = s_cnt[tid];
        const unsigned ex = block_exclusive_scan<SPLIT_THREADS>(c, s_warp, &s_total);
        s_lst[tid] = ex;
        // the range of this round in fine part fb + tid: the atomic's round trip is covered by
        // the staging (its result is first needed by the copy-out)
        unsigned gbv = 0;
        if (c) gbv = atomicAdd(&fine_fill[fb + tid], c);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            if (f[u] == 0xffffffffu) continue;
            const unsigned l = f[u] - fb;
            const unsigned pos = s_lst[l] + rank[u];
            FA_DCHECK(pos < unsigned(RI), "split staging index");
            s_stage[pos] = r[u];
        }
        s_gb[tid] = gbv;
        __syncthreads();
        const unsigned staged = s_total;
        for (unsigned i = tid; i < staged; i += SPLIT_THREADS) {
            const uint4 v = s_stage[i];
            const unsigned l = ((v.y >> 2) >> plog) - fb;  // the staged record names its fine part
            asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(rec2 + s_gb[l] + (i - s_lst[l])),
                         "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                         : "memory");
        }
        s_cnt[tid] = 0;  // (own counter; the next round's first barrier orders it)
    }
}

// Sort one vertex's incidences by key (k << 2 | a, unique) with their neighbours: insertion
// sort for short lists, heapsort beyond (O(d log d), in place).
__device__ void sort_incidences(unsigned* key, unsigned* n1, unsigned* n2, int d) {
    if (d <= 32) {
        for (int i = 1; i < d; ++i) {
            const unsigned x = key[i], y1 = n1[i], y2 = n2[i];
            int j = i - 1;
            while (j >= 0 && key[j] > x) {
                key[j + 1] = key[j];
                n1[j + 1] = n1[j];
                n2[j + 1] = n2[j];
                --j;
            }
            key[j + 1] = x;
            n1[j + 1] = y1;
            n2[j + 1] = y2;
        }
        return;
    }
    auto sift = [&](int root, int end) {
        while (true) {
            int child = 2 * root + 1;
            if (child >= end) break;
            if (child + 1 < end && key[child + 1] > key[child]) ++child;
            if (key[root] >= key[child]) break;
            unsigned t = key[root]; key[root] = key[child]; key[child] = t;
            t = n1[root]; n1[root] = n1[child]; n1[child] = t;
            t = n2[root]; n2[root] = n2[child]; n2[child] = t;
            root = child;
        }
    };
    for (int i = d / 2 - 1; i >= 0; --i) sift(i, d);
    for (int end = d - 1; end > 0; --end) {
        unsigned t = key[0]; key[0] = key[end]; key[end] = t;
        t = n1[0]; n1[0] = n1[end]; n1[end] = t;
        t = n2[0]; n2[0] = n2[end]; n2[end] = t;
        sift(0, end);
    }
}

// Sort the slots idx[0..d) by key[slot] (unique keys): insertion sort for short lists, heapsort
// beyond.
__device__ void sort_slots(unsigned short* idx, const unsigned* key, int d) {
    if (d <= 32) {
        for (int i = 1; i < d; ++i) {
            const unsigned short s = idx[i];
            const unsigned x = key[s];
            int j = i - 1;
            while (j >= 0 && key[idx[j]] > x) {
                idx[j + 1] = idx[j];
                --j;
            }
            idx[j + 1] = s;
        }
        return;
    }
    auto sift = [&](int root, int end) {
        while (true) {
            int child = 2 * root + 1;
            if (child >= end) break;
            if (child + 1 < end && key[idx[child + 1]] > key[idx[child]]) ++child;
            if (key[idx[root]] >= key[idx[child]]) break;
            const unsigned short t = idx[root]; idx[root] = idx[child]; idx[child] = t;
            root = child;
        }
    };
    for (int i = d / 2 - 1; i >= 0; --i) sift(i, d);
    for (int end = d - 1; end > 0; --end) {
        const unsigned short t = idx[0]; idx[0] = idx[end]; idx[end] = t;
        sift(0, end);
    }
}

// 8 keys ascending (19 comparators, verified by the 0-1 principle)
__device__ __forceinline__ void sort8(unsigned (&k)[8]) {
    auto cx = [](unsigned& x, unsigned& y) {
        const unsigned lo = min(x, y), hi = max(x, y);
        x = lo;
        y = hi;
    };
    cx(k[0], k[2]); cx(k[1], k[3]); cx(k[4], k[6]); cx(k[5], k[7]);
    cx(k[0], k[4]); cx(k[1], k[5]); cx(k[2], k[6]); cx(k[3], k[7]);
    cx(k[0], k[1]); cx(k[2], k[3]); cx(k[4], k[5]); cx(k[6], k[7]);
    cx(k[2], k[4]); cx(k[3], k[5]);
    cx(k[1], k[4]); cx(k[3], k[6]);
    cx(k[1], k[2]); cx(k[3], k[4]); cx(k[5], k[6]);
}

// K4: one block per part.  Counting sort by vertex, every vertex's list by k; SoA output and
// per-vertex offsets.  Parts of PV == 1024 vertices and up to SORT_CAP incidences are sorted
// in shared memory, others in place in global memory.  s_cur[v]: count, then start, then
// (after placement) end of vertex v.
__global__ void __launch_bounds__(SORT_THREADS, 2) k_part_sort(const __grid_constant__ PlanArgs P) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned s_dyn[];
    __shared__ unsigned s_warp[SORT_THREADS / 32];
    __shared__ unsigned s_total;
    const int p = blockIdx.x, tid = threadIdx.x;
    const int PV = 1 << P.plog;
    const int64_t nv = P.v1 - P.v0;
    const int64_t vfirst = int64_t(p) << P.plog;
    const int nvp = int(min(int64_t(PV), nv - vfirst));
    const unsigned off = P.part_off[p], n = P.part_off[p + 1] - off;
    const bool fast = PV == (1 << PLOG0) && n <= unsigned(SORT_CAP);
    if (P.sort_pf > 0 && p + P.sort_pf < P.nparts) {  // a part sorted about half a generation of blocks later -> L2
        const unsigned o2 = P.part_off[p + P.sort_pf], n2 = P.part_off[p + P.sort_pf + 1] - o2;
        const uint4* base = P.rec + (o2 & ~7u);  // 128-byte lines
        const unsigned lines = ((o2 & 7u) + n2 + 7u) >> 3;
        for (unsigned l = tid; l < lines; l += SORT_THREADS) prefetch_l2(base + 8 * size_t(l));
    }
    unsigned* s_cur = s_dyn;  // [PV]
    const uint64_t pol = l2_evict_first_policy();
    for (int i = tid; i < PV; i += SORT_THREADS) s_cur[i] = 0;
    __syncthreads();
    unsigned* key = fast ? s_dyn + PV : P.skey + off;
    unsigned* n1 = fast ? s_dyn + PV + SORT_CAP : P.sn1 + off;
    unsigned* n2 = fast ? s_dyn + PV + 2 * SORT_CAP : P.sn2 + off;
    // fast: [SORT_CAP] each.  s_src: vertex of the record in arrival slot i (until the records are
    // ranked), then the source slot of every sorted position; s_grp: arrival slots grouped by vertex
    unsigned short* s_src = reinterpret_cast<unsigned short*>(s_dyn + PV + 3 * SORT_CAP);
    unsigned short* s_grp = s_src + SORT_CAP;
    constexpr int RU = 6;  // records in flight per thread (C5 sort 3.50 -> 3.37 ms against four)
    if (fast) {
        // the part's records read once: (key, n1, n2, vertex) into shared memory in arrival order
        // (conflict-free stores) while the vertices are counted
        for (unsigned i0 = tid; i0 < n; i0 += RU * SORT_THREADS) {
            uint4 r[RU];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const unsigned i = i0 + u * SORT_THREADS;
                if (i < n)
                    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                                 : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w)
                                 : "l"(P.rec + off + i), "l"(pol));
            }
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const unsigned i = i0 + u * SORT_THREADS;
                if (i < n) {
                    const unsigned vl = (r[u].y >> 2) & unsigned(PV - 1);
                    key[i] = (r[u].x << 2) | (r[u].y & 3u);
                    n1[i] = r[u].z;
                    n2[i] = r[u].w;
                    s_src[i] = (unsigned short)vl;
                    atomicAdd(&s_cur[vl], 1u);
                }
            }
        }
    } else {  // vertex counts: eight records in flight per thread
        const unsigned* ry = reinterpret_cast<const unsigned*>(P.rec + off) + 1;  // .y fields
        for (unsigned i0 = tid; i0 < n; i0 += 8 * SORT_THREADS) {
            unsigned y[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const unsigned i = i0 + u * SORT_THREADS;
                y[u] = i < n ? ry[4 * size_t(i)] : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (y[u] != 0xffffffffu) atomicAdd(&s_cur[(y[u] >> 2) & unsigned(PV - 1)], 1u);
        }
    }
    __syncthreads();
    // vertex starts: thread t scans PV / 1024 consecutive vertices
    const int per = PV / SORT_THREADS;
    unsigned run = 0;
    for (int j = 0; j < per; ++j) run += s_cur[tid * per + j];
    unsigned ex = block_exclusive_scan<SORT_THREADS>(run, s_warp, &s_total);
    for (int j = 0; j < per; ++j) {
        const int v = tid * per + j;
        const unsigned c = s_cur[v];
        s_cur[v] = ex;
        if (v < nvp) P.ivptr[vfirst + v] = off + ex;
        ex += c;
    }
    if (p == P.nparts - 1 && tid == 0) P.ivptr[nv] = off + n;
    __syncthreads();
    if (fast) {  // arrival slots grouped by vertex (order inside a vertex's list is arbitrary)
        for (unsigned i = tid; i < n; i += SORT_THREADS) {
            const unsigned pos = atomicAdd(&s_cur[s_src[i]], 1u);
            FA_DCHECK(pos < n, "part sort position");
            s_grp[pos] = (unsigned short)i;
        }
    } else {
        for (unsigned i0 = tid; i0 < n; i0 += RU * SORT_THREADS) {
            uint4 r[RU];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const unsigned i = i0 + u * SORT_THREADS;
                if (i < n)
                    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                                 : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w)
                                 : "l"(P.rec + off + i), "l"(pol));
            }
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                if (i0 + u * SORT_THREADS < n) {
                    const unsigned pos = atomicAdd(&s_cur[(r[u].y >> 2) & unsigned(PV - 1)], 1u);
                    FA_DCHECK(pos < n, "part sort position");
                    key[pos] = (r[u].x << 2) | (r[u].y & 3u);
                    n1[pos] = r[u].z;
                    n2[pos] = r[u].w;
                }
            }
        }
    }
    __syncthreads();
    if (fast) {
        // per vertex: rank of every incidence among the vertex's keys (unique) -> source slot
        // of every sorted position; then one coalesced permuting copy.  pack: k << 5 fits 32
        // bits (k < 2^27), so the list position rides in the key's low bits
        const bool pack = P.nme <= (int64_t(1) << 27);
        for (int v = tid; v < PV; v += SORT_THREADS) {
        const unsigned st = v ? s_cur[v - 1] : 0u, d = s_cur[v] - st;
        if (d <= 8 && pack) {
            // keys (k << 2 | a, unique) with the list position in three low bits, sorted by a
            // 19-comparator network: the sorted position's source slot is in the low bits
            unsigned kk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) kk[j] = j < int(d) ? (key[s_grp[st + j]] << 3) | unsigned(j) : 0xffffffffu;
            sort8(kk);
#pragma unroll
            for (int r = 0; r < 8; ++r)
                if (r < int(d)) s_src[st + r] = s_grp[st + (kk[r] & 7u)];
        } else if (d <= 8) {
            unsigned kk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) kk[j] = j < int(d) ? key[s_grp[st + j]] : 0xffffffffu;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (i < int(d)) {
                    unsigned r = 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) r += kk[j] < kk[i] ? 1u : 0u;
                    s_src[st + r] = s_grp[st + i];
                }
            }
        } else {
            sort_slots(s_grp + st, key, int(d));
            for (unsigned i = 0; i < d; ++i) s_src[st + i] = s_grp[st + i];
        }
        }
        __syncthreads();
        for (unsigned i = tid; i < n; i += SORT_THREADS) {
            const unsigned j = s_src[i];
            FA_DCHECK(j < n, "part sort source slot");
            P.skey[off + i] = key[j];
            P.sn1[off + i] = n1[j];
            P.sn2[off + i] = n2[j];
        }
    } else {
        // in place in global memory (L2-resident region of this part): short lists are read
        // into registers, ranked and written back permuted; long ones heap-sorted
        __threadfence_block();
        for (int v = tid; v < PV; v += SORT_THREADS) {
            const unsigned st = v ? s_cur[v - 1] : 0u, d = s_cur[v] - st;
            if (d <= 1) continue;
            if (d <= 8) {
                unsigned kk[8], a1[8], a2[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    kk[j] = j < int(d) ? key[st + j] : 0xffffffffu;
                    a1[j] = j < int(d) ? n1[st + j] : 0u;
                    a2[j] = j < int(d) ? n2[st + j] : 0u;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (i < int(d)) {
                        unsigned r = 0;
#pragma unroll
                        for (int j = 0; j < 8; ++j) r += kk[j] < kk[i] ? 1u : 0u;
                        key[st + r] = kk[i];
                        n1[st + r] = a1[i];
                        n2[st + r] = a2[i];
                    }
                }
            } else {
                sort_incidences(key + st, n1 + st, n2 + st, int(d));
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// numeric: rows
// ------------------------------------------------------------------------------------------
struct RowsArgs {
    const unsigned* skey;   // sorted (vertex, k): k << 2 | a
    const unsigned* sn1;
    const unsigned* sn2;
    const unsigned* ivptr;  // nv + 1
    const double2* q;
    const double* w;
    const double* areas;    // nullable: recompute from q (bitwise compute_areas)
    double lam, mu;
    int64_t v0, v1;         // owned vertices
    int64_t nrows;          // matrix rows produced (owned vertices * rows per vertex)
    int64_t* rowptr;
    int32_t* col;
    double* val;
    int64_t capacity;
    uint64_t* status;
    unsigned long long* ticket;
    unsigned long long* bsym;  // per bucket: symbolic start of its CSR segment
    unsigned* blen;         // per bucket: symbolic length
    unsigned* bdrop;        // per bucket: entries that summed to exactly zero
    unsigned* read_done;    // per bucket: k_compact flag, zeroed here
    const double4* Wt;      // weighted mass: per-triangle W0..W2 (k_tri_wt)
    fa_result* res;
    int pf_dist;            // elasticity: buckets ahead whose row starts / coordinates / plan entries go to L2 (0: none)
};

template <int KIND>
struct KindTraits {
    static constexpr int RPV = KIND == FA_KIND_ELASTIC ? 2 : 1;  // rows per vertex
    static constexpr int NV = KIND == FA_KIND_ELASTIC ? 2 : 1;   // values per (row, vertex column)
    static constexpr int THREADS = BV * RPV;
    // per-record shared data: scalar kinds store the row's three values, elasticity the 2 x 6
    // entries of its two dof rows (own, n1, n2 vertex columns, x and y)
    static constexpr int RVALS = KIND == FA_KIND_ELASTIC ? 12 : 3;
    static constexpr int MIN_BLOCKS =
        KIND == FA_KIND_ELASTIC ? ROWS_MINB_E
                                : (KIND == FA_KIND_MASSW ? ROWS_MINB_W : (KIND == FA_KIND_STIFF ? ROWS_MINB_S : ROWS_MINB));
    static constexpr int CAP =  // incidences in shared memory
        KIND == FA_KIND_ELASTIC ? CAPB_E : (KIND == FA_KIND_MASSW ? CAPB_W : (KIND == FA_KIND_STIFF ? CAPB_S : CAPB));
    // scalar kinds stage the bucket's CSR segment in the plan-entry arrays (12 bytes per slot)
    // plus SX extra entries: a bucket holds ~7 entries per vertex, more than the 6.5 incidence
    // slots per vertex of the stiffness shape (without them most stiffness buckets wrote their
    // rows straight to global memory: C3 numeric 753 -> 730 us, C5 13.75 -> 13.35 ms)
    static constexpr int SX = KIND == FA_KIND_STIFF ? 192 : 0;
    static constexpr size_t REC_BYTES = size_t(CAP) * (RVALS * 8 + 12) + size_t(SX) * 12;
    static constexpr int STAGE = int(REC_BYTES / 12);  // staged entries fitting the records area
};

template <int KIND>
constexpr size_t rows_smem_bytes() {
    return KindTraits<KIND>::REC_BYTES;
}

// Gathered data of one incidence: neighbour coordinates, the triangle area, the W record.
struct Gathered {
    double2 p1, p2;
    double ar;
    double4 wt;  // weighted mass: the triangle's W0, W1, W2 (k_tri_wt)
};

template <int KIND>
__device__ __forceinline__ Gathered gather_incidence(const RowsArgs& A, unsigned k, unsigned n1, unsigned n2,
                                                     uint64_t pol) {
    Gathered g;
    g.p1 = g.p2 = make_double2(0.0, 0.0);
    g.ar = (KIND != FA_KIND_MASSW && A.areas) ? ld_keep_f64(A.areas + k, pol) : 0.0;
    if (KIND == FA_KIND_STIFF || KIND == FA_KIND_ELASTIC || !A.areas) {
        g.p1 = ld_keep_f64x2(A.q + n1, pol);
        g.p2 = ld_keep_f64x2(A.q + n2, pol);
    }
    if (KIND == FA_KIND_MASSW)  // the triangle's three W (k_tri_wt): one 32-byte gather
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                     : "=d"(g.wt.x), "=d"(g.wt.y), "=d"(g.wt.z), "=d"(g.wt.w)
                     : "l"(A.Wt + k), "l"(pol));
    return g;
}

// Values of one incidence: row a of the element matrix against the triangle's vertices in
// local order (own, n1, n2); elasticity: gradients + area instead.  Degenerate triangles are
// reported (assembly.py:152-155) for every kind that divides by the area.
template <int KIND>
__device__ __forceinline__ void incidence_values(const RowsArgs& A, unsigned k, int a, const Gathered& g,
                                                 double2 own_p, double* out) {
    double ar = g.ar;
    // elasticity: the edges opposite the own corner and the two neighbours (the reference's u,
    // v, w in local order: same operands, same bits, assembly.py:195-211), and the area from
    // them (bitwise compute_areas, tri_area_edges; C4 numeric -3 % against the corner selects)
    double2 eo = make_double2(0.0, 0.0), e1 = eo, e2 = eo;
    if (KIND == FA_KIND_ELASTIC) {
        eo = dsub2(g.p1, g.p2);
        e1 = dsub2(g.p2, own_p);
        e2 = dsub2(own_p, g.p1);
        if (!A.areas) ar = tri_area_edges(a, eo, e1, e2);
    } else if (!A.areas) {  // corners in triangle order (compute_areas, mesh.py:62-65)
        ar = tri_area(sel3(a, own_p, g.p2, g.p1), sel3(a, g.p1, own_p, g.p2), sel3(a, g.p2, g.p1, own_p));
    }
    if (KIND != FA_KIND_MASSW && ar <= AREA_EPS) atomic_min_i64(&A.res->degenerate_index, int64_t(k));
    if constexpr (KIND == FA_KIND_MASS) {
        const MassTri m = mass_prepare(ar);
        out[0] = m.d;
        out[1] = m.o;
        out[2] = m.o;
    } else if constexpr (KIND == FA_KIND_MASSW) {
        // the six distinct entries of the triangle's matrix (assembly.py:236-241), with W in
        // the triangle's corner order (k_tri_wt); row a picks three (additions are not
        // associative, so every entry keeps the reference's own expression):
        //   (0,0) (3*W0 + W1) + W2   (1,1) (W0 + 3*W1) + W2   (2,2) (W0 + W1) + 3*W2
        //   (0,1) (W0 + W1) + W2/2   (0,2) (W0 + W1/2) + W2   (1,2) (W0/2 + W1) + W2
        const double W0 = g.wt.x, W1 = g.wt.y, W2 = g.wt.z;
        const double s01 = FADD(W0, W1);
        const double d0 = FADD(FADD(FMUL(3.0, W0), W1), W2);
        const double d1 = FADD(FADD(W0, FMUL(3.0, W1)), W2);
        const double d2 = FADD(s01, FMUL(3.0, W2));
        const double e01 = FADD(s01, FMUL(W2, 0.5));
        const double e02 = FADD(FADD(W0, FMUL(W1, 0.5)), W2);
        const double e12 = FADD(FADD(FMUL(W0, 0.5), W1), W2);
        out[0] = sel3(a, d0, d1, d2);
        out[1] = sel3(a, e01, e12, e02);  // (a, a+1)
        out[2] = sel3(a, e02, e01, e12);  // (a, a+2)
    } else if constexpr (KIND == FA_KIND_STIFF) {
        // the edges opposite the own corner and the two neighbours are the reference's u, v, w
        // (assembly.py:251-254) taken in local order - the same operand pairs, so the same bits
        // - and row a is their dot products over 4*area (stiff_entry without the selects)
        const double2 eo = dsub2(g.p1, g.p2), e1 = dsub2(g.p2, own_p), e2 = dsub2(own_p, g.p1);
        // three true divisions by a4 = 4*area sharing one correctly rounded reciprocal (div_by)
        const DivBy d4 = div_prepare(FMUL(4.0, ar));
        div_by3(d4, FADD(FADD(0.0, FMUL(eo.x, eo.x)), FMUL(eo.y, eo.y)),
                FADD(FADD(0.0, FMUL(eo.x, e1.x)), FMUL(eo.y, e1.y)),
                FADD(FADD(0.0, FMUL(eo.x, e2.x)), FMUL(eo.y, e2.y)), out[0], out[1], out[2]);
    } else {
        // gradients of the own corner and the two neighbours from the edges opposite them (the
        // reference's u, v, w in local order: same operands, same bits, assembly.py:195-211)
        const double inv2a = FDIV(0.5, ar);
        const double2 gO = make_double2(FMUL(eo.y, inv2a), FMUL(-eo.x, inv2a));
        const double L = A.lam, M = A.mu, P = FADD(A.lam, FMUL(2.0, A.mu));
        // own 2x2 block (elastic_lower with A == B; (x, y) is the copy of (y, x))
        out[0] = FMUL(FADD(FMUL(FMUL(P, gO.x), gO.x), FMUL(FMUL(M, gO.y), gO.y)), ar);
        out[7] = FMUL(FADD(FMUL(FMUL(P, gO.y), gO.y), FMUL(FMUL(M, gO.x), gO.x)), ar);
        out[6] = FMUL(FADD(FMUL(FMUL(L, gO.x), gO.y), FMUL(FMUL(M, gO.x), gO.y)), ar);
        out[1] = out[6];
#pragma unroll
        for (int rel = 1; rel < 3; ++rel) {
            const double2 e = rel == 1 ? e1 : e2;
            const double2 gb = make_double2(FMUL(e.y, inv2a), FMUL(-e.x, inv2a));
            // the lower-triangle entry puts the corner with the larger triangle index first
            // (X) and takes the other's gradient first in every product (elastic_lower); the
            // neighbour at corner a+1 is larger unless a == 2, the one at a+2 unless a == 0
            const bool own_x = rel == 1 ? a == 2 : a != 0;
            const double2 gX = own_x ? gO : gb, gY = own_x ? gb : gO;
            const double d00 = FADD(FMUL(FMUL(P, gY.x), gX.x), FMUL(FMUL(M, gY.y), gX.y));
            const double d11 = FADD(FMUL(FMUL(P, gY.y), gX.y), FMUL(FMUL(M, gY.x), gX.x));
            const double l10 = FADD(FMUL(FMUL(L, gY.x), gX.y), FMUL(FMUL(M, gY.y), gX.x));  // X's y, Y's x
            const double l01 = FADD(FMUL(FMUL(L, gY.y), gX.x), FMUL(FMUL(M, gY.x), gX.y));  // X's x, Y's y
            out[rel * 2] = FMUL(d00, ar);                          // (own x, b x)
            out[6 + rel * 2 + 1] = FMUL(d11, ar);                  // (own y, b y)
            out[6 + rel * 2] = FMUL(own_x ? l10 : l01, ar);        // (own y, b x)
            out[rel * 2 + 1] = FMUL(own_x ? l01 : l10, ar);        // (own x, b y)
        }
    }
}

// Entry of an incidence from its values: dof row s (x/y of the own vertex for elasticity),
// column vertex rel (0 = own, 1 = n1, 2 = n2), column component t.
template <int KIND>
__device__ __forceinline__ double entry_from(const RowsArgs& A, const double* rv, int a, int s, int rel, int t) {
    if constexpr (KIND == FA_KIND_ELASTIC) {
        return rv[s * 6 + rel * 2 + t];
    } else {
        return rel == 0 ? rv[0] : (rel == 1 ? rv[1] : rv[2]);
    }
}

// Same from the shared record of slot `slot`.
template <int KIND>
__device__ __forceinline__ double record_entry(const RowsArgs& A, const double* vals, int slot, int a, int s,
                                               int rel, int t) {
    constexpr int CAP = KindTraits<KIND>::CAP;
    if constexpr (KIND == FA_KIND_ELASTIC) {
        return vals[(s * 6 + rel * 2 + t) * CAP + slot];
    } else {
        return rel == 0 ? vals[slot] : vals[CAP + 2 * slot + rel - 1];  // rel 1, 2 interleaved
    }
}

__device__ __forceinline__ void cs(unsigned& x, unsigned& y) {
    const unsigned lo = min(x, y), hi = max(x, y);
    x = lo;
    y = hi;
}
// Batcher odd-even merge sort, 16 keys, 63 comparators (verified by the 0-1 principle)
__device__ __forceinline__ void sort16(unsigned (&k)[16]) {
    cs(k[0], k[1]); cs(k[2], k[3]); cs(k[0], k[2]); cs(k[1], k[3]); cs(k[1], k[2]); cs(k[4], k[5]); cs(k[6], k[7]); cs(k[4], k[6]);
    cs(k[5], k[7]); cs(k[5], k[6]); cs(k[0], k[4]); cs(k[2], k[6]); cs(k[2], k[4]); cs(k[1], k[5]); cs(k[3], k[7]); cs(k[3], k[5]);
    cs(k[1], k[2]); cs(k[3], k[4]); cs(k[5], k[6]); cs(k[8], k[9]); cs(k[10], k[11]); cs(k[8], k[10]); cs(k[9], k[11]); cs(k[9], k[10]);
    cs(k[12], k[13]); cs(k[14], k[15]); cs(k[12], k[14]); cs(k[13], k[15]); cs(k[13], k[14]); cs(k[8], k[12]); cs(k[10], k[14]); cs(k[10], k[12]);
    cs(k[9], k[13]); cs(k[11], k[15]); cs(k[11], k[13]); cs(k[9], k[10]); cs(k[11], k[12]); cs(k[13], k[14]); cs(k[0], k[8]); cs(k[4], k[12]);
    cs(k[4], k[8]); cs(k[2], k[10]); cs(k[6], k[14]); cs(k[6], k[10]); cs(k[2], k[4]); cs(k[6], k[8]); cs(k[10], k[12]); cs(k[1], k[9]);
    cs(k[5], k[13]); cs(k[5], k[9]); cs(k[3], k[11]); cs(k[7], k[15]); cs(k[7], k[11]); cs(k[3], k[5]); cs(k[7], k[9]); cs(k[11], k[13]);
    cs(k[1], k[2]); cs(k[3], k[4]); cs(k[5], k[6]); cs(k[7], k[8]); cs(k[9], k[10]); cs(k[11], k[12]); cs(k[13], k[14]);
}

// Shared records of one bucket.
struct BucketRecs {
    double* vals;          // [RVALS][CAP]
    int* n1;               // [CAP]
    int* n2;               // [CAP]
    unsigned* ka;          // [CAP] k << 2 | local corner of the row's vertex
};

struct RowCount {
    int64_t count, zeros;
};

// General path for one row: O(d^2) selection of the columns in ascending order.  `values`
// false: the symbolic entry count only.  `values` true: each position summed in ascending k
// (incidences from shared memory, slots start.., or - overflowing bucket - from the plan in
// global memory with the values recomputed); entries written at out_pos.. when `write`, exact
// zeros kept (removed later by k_compact) or dropped per `keep_zeros`; zero sums counted.
template <int KIND>
__device__ __noinline__ RowCount general_row(const RowsArgs& A, BucketRecs R, bool overflow, int64_t gfirst, int start,
                                             int deg, int64_t v, double2 own_p, int s, int64_t out_pos,
                                             bool values, bool write = true, bool keep_zeros = true) {
    constexpr int NV = KindTraits<KIND>::NV;
    constexpr int RVALS = KindTraits<KIND>::RVALS;
    auto get = [&](int i, int& a, int& n1, int& n2, double* rv, bool need_vals) {
        if (!overflow) {
            const int slot = start + i;
            a = int(R.ka[slot] & 3u);
            n1 = R.n1[slot];
            n2 = R.n2[slot];
            if (need_vals)
                for (int j = 0; j < RVALS; ++j)
                    rv[j] = KIND == FA_KIND_ELASTIC ? R.vals[j * KindTraits<KIND>::CAP + slot]
                                                    : record_entry<KIND>(A, R.vals, slot, a, 0, j, 0);
            return;
        }
        const unsigned ka = A.skey[gfirst + i];
        a = int(ka & 3u);
        n1 = int(A.sn1[gfirst + i]);
        n2 = int(A.sn2[gfirst + i]);
        if (need_vals) {
            const Gathered g = gather_incidence<KIND>(A, ka >> 2, unsigned(n1), unsigned(n2), l2_evict_last_policy());
            incidence_values<KIND>(A, ka >> 2, a, g, own_p, rv);
        }
    };
    int64_t last = -1, count = 0, zeros = 0;
    if (deg == 0) return RowCount{0, 0};  // a vertex no triangle references has an empty row
    while (true) {
        int64_t c = INT64_MAX;  // next vertex column
        if (v > last) c = v;
        for (int i = 0; i < deg; ++i) {
            int a, n1, n2;
            get(i, a, n1, n2, nullptr, false);
            if (n1 > last && n1 < c) c = n1;
            if (n2 > last && n2 < c) c = n2;
        }
        if (c == INT64_MAX) break;
        if (values) {
            double sum[NV];
            for (int t = 0; t < NV; ++t) sum[t] = 0.0;
            for (int i = 0; i < deg; ++i) {  // ascending k: each incidence contributes at most once
                int a, n1, n2;
                get(i, a, n1, n2, nullptr, false);
                const int rel = c == v ? 0 : (n1 == c ? 1 : (n2 == c ? 2 : -1));
                if (rel < 0) continue;
                double rv[KindTraits<KIND>::RVALS];
                get(i, a, n1, n2, rv, true);
                for (int t = 0; t < NV; ++t) sum[t] = FADD(sum[t], entry_from<KIND>(A, rv, a, s, rel, t));
            }
            for (int t = 0; t < NV; ++t) {
                const bool z = sum[t] == 0.0;
                if (z) ++zeros;
                if (z && !keep_zeros) continue;
                if (write && out_pos + count < A.capacity) {
                    A.col[out_pos + count] = int32_t(NV == 1 ? c : 2 * c + t);
                    A.val[out_pos + count] = sum[t];
                }
                ++count;
            }
        } else {
            count += NV;
        }
        last = c;
    }
    return RowCount{count, zeros};
}


// Sorted candidate columns of a fast row: (neighbour << 4 | slot), slot = 2 * incidence +
// (0: n1, 1: n2), unused keys 0xffffffff.
__device__ __forceinline__ void row_keys(const BucketRecs& R, int start, int deg, unsigned (&sk)[2 * MAXD]) {
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
        const bool ok = i < deg;
        sk[2 * i] = ok ? (unsigned(R.n1[start + i]) << 4) | unsigned(2 * i) : 0xffffffffu;
        sk[2 * i + 1] = ok ? (unsigned(R.n2[start + i]) << 4) | unsigned(2 * i + 1) : 0xffffffffu;
    }
    sort16(sk);
}

// Scalar kinds, fast row: the row's entries in column order from its sorted candidate keys -
// every position summed sequentially in ascending k (the slot order inside a run of equal
// columns), the diagonal (all incidences, ascending k) at position dpos (the columns below
// it) - written to col/val[0..]; CHECK: only the first `room` entries are stored.  Exact-zero
// sums stay as entries (k_compact removes them) and are counted; returns that count.
template <int KIND, bool CHECK>
__device__ __forceinline__ int64_t walk_row(const BucketRecs& R, const unsigned (&sk)[2 * MAXD], int start, int deg,
                                            unsigned vv, int dpos, int32_t* col, double* val, int64_t room) {
    constexpr int CAP = KindTraits<KIND>::CAP;
    const double* v12 = R.vals + CAP + 2 * start;  // (n1, n2) values of the row's incidences
    double dsum = 0.0;
#pragma unroll
    for (int i = 0; i < MAXD; ++i)
        if (i < deg) dsum = FADD(dsum, R.vals[start + i]);
    int64_t zeros = 0;
    if (deg > 0) {
        if (!CHECK || dpos < room) {
            col[dpos] = int32_t(vv);
            val[dpos] = dsum;
        }
        zeros += dsum == 0.0 ? 1 : 0;
    }
    double sum = 0.0;
    int r = 0;  // runs written so far
#pragma unroll
    for (int j = 0; j < 2 * MAXD; ++j) {
        const unsigned key = sk[j];
        const unsigned nxt = j + 1 < 2 * MAXD ? sk[j + 1] : 0xffffffffu;
        if (key != 0xffffffffu) {
            const bool st = j == 0 || ((key ^ sk[j - 1]) >> 4) != 0;
            sum = FADD(st ? 0.0 : sum, v12[key & 15]);
            if (((key ^ nxt) >> 4) != 0) {  // run ends: its column and sum
                const unsigned c = key >> 4;
                const int idx = r + (c > vv ? 1 : 0);
                if (!CHECK || idx < room) {
                    col[idx] = int32_t(c);
                    val[idx] = sum;
                }
                zeros += sum == 0.0 ? 1 : 0;
                ++r;
            }
        }
    }
    return zeros;
}

// A bucket's staged CSR segment -> global memory with 16-byte stores: columns in fours,
// values in pairs, after a scalar head that brings the global position to 16-byte alignment
// (the staging is read with scalar loads).
template <int NT>
__device__ __forceinline__ void copy_out(const int32_t* st_col, const double* st_val, int32_t* gcol, double* gval,
                                         int tot, uint64_t pol) {
    const int tid = threadIdx.x;
    const unsigned ac = unsigned(reinterpret_cast<uintptr_t>(gcol)) & 15u;
    const unsigned av = unsigned(reinterpret_cast<uintptr_t>(gval)) & 15u;
    const int hc = min(tot, int(((16u - ac) & 15u) >> 2)), hv = min(tot, int(((16u - av) & 15u) >> 3));
    if (tid < hc) st_stream_i32(gcol + tid, st_col[tid], pol);
    if (tid < hv) st_stream_f64(gval + tid, st_val[tid], pol);
    for (int e = hc + 4 * tid; e < tot; e += 4 * NT) {
        if (e + 3 < tot) {
            st_stream_i32x4(gcol + e, st_col[e], st_col[e + 1], st_col[e + 2], st_col[e + 3], pol);
        } else {
            for (int j = e; j < tot; ++j) st_stream_i32(gcol + j, st_col[j], pol);
        }
    }
    for (int e = hv + 2 * tid; e < tot; e += 2 * NT) {
        if (e + 1 < tot) st_stream_f64x2(gval + e, st_val[e], st_val[e + 1], pol);
        else st_stream_f64(gval + e, st_val[e], pol);
    }
}

template <int KIND>
__global__ void __launch_bounds__(KindTraits<KIND>::THREADS, KindTraits<KIND>::MIN_BLOCKS)
    k_rows(const __grid_constant__ RowsArgs A) {
    pdl_enter();
    using TR = KindTraits<KIND>;
    constexpr int NV = TR::NV, RPV = TR::RPV, NT = TR::THREADS, RVALS = TR::RVALS;
    constexpr int NC = 2 * MAXD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BucketRecs R;
    R.vals = reinterpret_cast<double*>(smem_raw);
    constexpr int CAP = TR::CAP;
    R.n1 = reinterpret_cast<int*>(R.vals + RVALS * CAP);
    R.n2 = R.n1 + CAP;
    R.ka = reinterpret_cast<unsigned*>(R.n2 + CAP + 2 * TR::SX);  // staging: n1|n2|extra doubles, ka|extra ints
    // compact staging of the bucket's CSR segment; reuses the records area once every row
    // holds its merged entries in registers
    double* st_val = reinterpret_cast<double*>(smem_raw);
    int32_t* st_col = reinterpret_cast<int32_t*>(st_val + TR::STAGE);
    __shared__ unsigned char s_own[TR::CAP];
    __shared__ int s_vst[BV + 1];
    __shared__ double2 s_oq[BV];
    __shared__ int64_t s_tile;
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_warp[NT / 32];
    __shared__ unsigned s_zeros;
    __shared__ unsigned s_pf[2];
    if (threadIdx.x == 0) s_zeros = 0;  // ordered before its atomics by next_tile's barrier

    const int tid = threadIdx.x;
    const uint64_t pol_first = l2_evict_first_policy();
    const uint64_t pol_last = l2_evict_last_policy();
    const int64_t b = next_tile(A.ticket, &s_tile);  // bucket, in launch order
    const int64_t nvl = A.v1 - A.v0;
    const int64_t vb0 = b * BV;  // first vertex of the bucket (row-block local)
    const int nvb = int(min(int64_t(BV), nvl - vb0));
    // the bucket's incidence range first; the mass kinds issue their plan-entry loads together
    // with the row starts (one DRAM round trip less before the first barrier; stiffness and
    // elasticity, which also load the own coordinates here, are faster without the extra
    // registers)
    const unsigned gbase = A.ivptr[vb0];
    const int ntot = int(A.ivptr[vb0 + nvb] - gbase);
    // elasticity (two blocks per SM: little else covers a bucket's three dependent round trips -
    // row starts, plan entries, own coordinates): the bucket one generation of resident blocks
    // ahead has its row starts and own coordinates brought into L2 now, its plan entries after
    // phase a (C4 numeric 2.04 -> 2.00 ms; the scalar kinds, five blocks per SM, gain nothing)
    const int64_t fvb0 = (b + A.pf_dist) * BV;
    const bool pf = KIND == FA_KIND_ELASTIC && A.pf_dist > 0 && fvb0 < nvl;
    unsigned fg0 = 0, fg1 = 0;
    if (pf && tid < 32) {
        if (tid == 0) {
            fg0 = A.ivptr[fvb0];
            fg1 = A.ivptr[fvb0 + min(int64_t(BV), nvl - fvb0)];
        } else if (tid < 5) {
            if (fvb0 + tid * 32 <= nvl) prefetch_l2(A.ivptr + fvb0 + tid * 32);
        } else if (tid >= 8 && tid < 25 && A.q) {
            const int64_t fv = A.v0 + fvb0 + (tid - 8) * 8;
            if (fv < A.v1) prefetch_l2(A.q + fv);
        }
    }
    const bool overflow = ntot > CAP;
    const int n = overflow ? 0 : ntot;
    constexpr int PER = (CAP + NT - 1) / NT;
    constexpr bool EARLY_LOAD = KIND == FA_KIND_MASS || KIND == FA_KIND_MASSW;
    unsigned lk[PER], l1[PER], l2[PER];
    auto load_entries = [&]() {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int i = tid + u * NT;
            if (i < n) {
                lk[u] = ld_stream_u32(A.skey + gbase + i, pol_first);
                l1[u] = ld_stream_u32(A.sn1 + gbase + i, pol_first);
                l2[u] = ld_stream_u32(A.sn2 + gbase + i, pol_first);
            }
        }
    };
    if constexpr (EARLY_LOAD) load_entries();
    for (int i = tid; i <= BV; i += NT) s_vst[i] = int(A.ivptr[vb0 + min(i, nvb)] - gbase);
    const int64_t vbase = A.v0 + vb0;
    // own coordinates: gradients, or the area when none is given (the weighted mass never reads q)
    const bool need_q = KIND == FA_KIND_STIFF || KIND == FA_KIND_ELASTIC || (KIND == FA_KIND_MASS && !A.areas);
    for (int i = tid; i < BV; i += NT) {
        const int64_t vv = vbase + i;
        s_oq[i] = (need_q && A.q && vv < A.v1) ? A.q[vv] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    if (pf && tid == 0) {
        s_pf[0] = fg0;
        s_pf[1] = fg1;
    }
    for (int vl = tid; vl < nvb && !overflow; vl += NT)
        for (int j = s_vst[vl]; j < s_vst[vl + 1]; ++j) {
            FA_DCHECK(j < CAP, "row bucket slot");
            s_own[j] = (unsigned char)vl;
        }
    // ---- s) the bucket's plan entries -> shared memory (coalesced)
    if constexpr (!EARLY_LOAD) load_entries();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int i = tid + u * NT;
        if (i < n) {
            R.ka[i] = lk[u];
            R.n1[i] = int(l1[u]);
            R.n2[i] = int(l2[u]);
        }
    }
    __syncthreads();

    // one thread per matrix row
    const int vloc = tid / RPV, s = tid % RPV;
    const int64_t v = vbase + vloc;
    const bool active = v < A.v1;
    const int64_t r = (b * BV + vloc) * RPV + s;  // local matrix row
    const int start = s_vst[vloc];
    const int deg = active ? s_vst[vloc + 1] - start : 0;
    const bool slow = active && (deg > MAXD || overflow);
    const bool fast = active && !slow;
    const unsigned vv = unsigned(v);
    // EARLY (scalar kinds): the bucket's symbolic size is published before the numeric work and
    // exact-zero sums stay as entries for k_compact (they are rare).  Elasticity cancels often,
    // so it publishes the exact count after the sums instead.
    constexpr bool EARLY = KIND != FA_KIND_ELASTIC;
    //    symbolic entry count of the row (unique columns + diagonal); the bucket aggregate is
    //    published now, before the numeric work, so successors' look-backs find it and this
    //    bucket's own look-back (after phase c) finds its predecessors' - nobody waits on the
    //    slow gathers of another bucket
    int64_t count = 0, excl = 0, total = 0;
    unsigned sk[NC];
    int dpos = 0;  // scalar fast rows: columns left of the diagonal
    if (EARLY && fast) {
        row_keys(R, start, deg, sk);
        unsigned distinct = 0;
#pragma unroll
        for (int j = 0; j < NC; ++j) {  // run starts among the valid keys; those below the diagonal
            const bool st = sk[j] != 0xffffffffu && (j == 0 || ((sk[j] ^ sk[j - 1]) >> 4) != 0);
            distinct += st ? 1u : 0u;
            dpos += (st && (sk[j] >> 4) < vv) ? 1 : 0;
        }
        count = deg == 0 ? 0 : int64_t(NV) * (distinct + 1);  // no triplet, no entry (isolated vertex)
    }
    if (EARLY && slow)
        count = general_row<KIND>(A, R, overflow, int64_t(gbase) + start, start, deg, v, s_oq[vloc], s, 0,
                                  false).count;
    if (EARLY) {
        excl = block_exclusive_scan_1b<NT>(count, s_warp, total);
        lookback_publish(A.status, b, uint64_t(total));
    }

    // ---- a) per incidence (balanced over threads): gathers from the L2-resident arrays, the
    //         row of the element matrix -> shared memory
    {
        constexpr int AU = KIND == FA_KIND_ELASTIC ? ROWS_AU_E
                                                   : (KIND == FA_KIND_MASSW ? ROWS_AU_W : (KIND == FA_KIND_STIFF ? ROWS_AU_S : ROWS_AU));
        for (int i0 = tid; i0 < n; i0 += NT * AU) {
            unsigned ka[AU];
            Gathered g[AU];
#pragma unroll
            for (int u = 0; u < AU; ++u) {
                const int i = i0 + u * NT;
                ka[u] = i < n ? R.ka[i] : 0u;
                if (i < n) g[u] = gather_incidence<KIND>(A, ka[u] >> 2, unsigned(R.n1[i]), unsigned(R.n2[i]), pol_last);
            }
#pragma unroll
            for (int u = 0; u < AU; ++u) {
                const int i = i0 + u * NT;
                if (i >= n) break;
                const int vl = s_own[i];
                double rv[RVALS];
                incidence_values<KIND>(A, ka[u] >> 2, int(ka[u] & 3u), g[u], s_oq[vl], rv);
                if constexpr (KIND == FA_KIND_ELASTIC) {
#pragma unroll
                    for (int j = 0; j < RVALS; ++j) R.vals[j * CAP + i] = rv[j];
                } else {  // own column, then the two neighbour columns side by side (one 16-byte store)
                    R.vals[i] = rv[0];
                    *reinterpret_cast<double2*>(R.vals + CAP + 2 * i) = make_double2(rv[1], rv[2]);
                }
            }
        }
    }
    const bool any_slow = __syncthreads_or(slow);  // also the end of phase a
    if (pf && tid < 32) {  // the plan entries of the bucket pf_dist ahead -> L2
        const unsigned f0 = s_pf[0] & ~31u, f1 = s_pf[1];
        for (unsigned e = f0 + unsigned(tid) * 32u; e < f1; e += 32u * 32u) {
            prefetch_l2(A.skey + e);
            prefetch_l2(A.sn1 + e);
            prefetch_l2(A.sn2 + e);
        }
    }

    int64_t zeros = 0;
    uint64_t base = 0;
    if constexpr (EARLY) {
        // ---- c+d) scalar kinds: each fast row walks its sorted columns once, summing every
        //      position sequentially in ascending k and writing it with its column straight
        //      into the compact staging.  The staging lies in the plan-entry arrays, dead once
        //      phase a is done (n1 + n2 + ka hold 12 bytes per incidence slot, a staged entry
        //      is 12 bytes), so the records' values stay intact for the unstaged fallback.
        const bool staged = !any_slow && total <= CAP + TR::SX;
        double* sv = reinterpret_cast<double*>(R.n1);    // [CAP], spans n1 and n2
        int32_t* sc = reinterpret_cast<int32_t*>(R.ka);  // [CAP]
        FA_DCHECK(!staged || !fast || excl + count <= total, "row segment inside the bucket's");
        if (staged && fast) zeros = walk_row<KIND, false>(R, sk, start, deg, vv, dpos, sc + excl, sv + excl, 0);
        base = lookback_wait(A.status, b, uint64_t(total), &s_prefix);  // ends with a barrier
        if (active) st_stream_i64(A.rowptr + r, int64_t(base) + excl, pol_first);
        if (active && r == A.nrows - 1) {
            A.rowptr[A.nrows] = int64_t(base) + excl + count;
            A.res->nnz = int64_t(base) + excl + count;
        }
        if (slow) atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->heavy_rows), 1ull);
        if (staged && int64_t(base) + total <= A.capacity) {
            copy_out<NT>(sc, sv, A.col + base, A.val + base, int(total), pol_first);
        } else if (staged) {
            for (int64_t e = tid; e < total; e += NT) {
                const int64_t g = int64_t(base) + e;
                if (g < A.capacity) {
                    st_stream_i32(A.col + g, sc[e], pol_first);
                    st_stream_f64(A.val + g, sv[e], pol_first);
                }
            }
        } else {
            const int64_t o = int64_t(base) + excl;
            if (fast) zeros = walk_row<KIND, true>(R, sk, start, deg, vv, dpos, A.col + o, A.val + o, A.capacity - o);
            if (slow)
                zeros = general_row<KIND>(A, R, overflow, int64_t(gbase) + start, start, deg, v, s_oq[vloc], s, o, true, true, true)
                            .zeros;
        }
    } else {
    // (measured alternative: two walks - count, then write straight to the CSR once the offset
    //  is known - removes the 68-register run_val array and its spills but loses the staged
    //  16-byte copy-out; C4 numeric 2.08 -> 2.61 ms.  The staging aliases the values, so a second
    //  walk cannot write it.)
    // ---- c) per row: each position summed sequentially in ascending k (== stable argsort +
    //         bincount of the reference); exact-zero sums stay as entries and are counted
    double dsum[NV], run_val[NC + 1][NV];
    int diag_at = -1;  // the diagonal is emitted right after run j == diag_at
#pragma unroll
    for (int t = 0; t < NV; ++t) dsum[t] = 0.0;
    if (fast) {
#pragma unroll
        for (int i = 0; i < MAXD; ++i) {
            if (i < deg) {
                const int slot = start + i;
#pragma unroll
                for (int t = 0; t < NV; ++t)
                    dsum[t] = FADD(dsum[t], record_entry<KIND>(A, R.vals, slot, int(R.ka[slot] & 3u), s, 0, t));
            }
        }
        if (!EARLY) row_keys(R, start, deg, sk);  // scalar kinds: sorted once, kept from the count
        unsigned prev = 0xffffffffu;
        double sum[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) sum[t] = 0.0;
#pragma unroll
        for (int j = 0; j <= NC; ++j) {
            const unsigned key = j < NC ? sk[j] : 0xffffffffu;
            const unsigned c = key == 0xffffffffu ? 0xffffffffu : (key >> 4);
#pragma unroll
            for (int t = 0; t < NV; ++t) run_val[j][t] = 0.0;
            if (c != prev) {
                if (prev != 0xffffffffu) {
#pragma unroll
                    for (int t = 0; t < NV; ++t) {
                        run_val[j][t] = sum[t];
                        if (sum[t] == 0.0) ++zeros;
                        else if (!EARLY) ++count;
                    }
                }
                if (diag_at < 0 && vv < c) {
                    diag_at = j;
#pragma unroll
                    for (int t = 0; t < NV; ++t) {
                        if (dsum[t] == 0.0) ++zeros;
                        else if (!EARLY) ++count;
                    }
                }
#pragma unroll
                for (int t = 0; t < NV; ++t) sum[t] = 0.0;
                prev = c;
            }
            if (j < NC && c != 0xffffffffu) {
                const int sl = int(key & 15);
                const int slot = start + (sl >> 1);
#pragma unroll
                for (int t = 0; t < NV; ++t)
                    sum[t] = FADD(sum[t], record_entry<KIND>(A, R.vals, slot, int(R.ka[slot] & 3u), s, 1 + (sl & 1), t));
            }
        }
    }
    if (!EARLY) {
        if (slow) {
            const RowCount rc = general_row<KIND>(A, R, overflow, int64_t(gbase) + start, start, deg, v, s_oq[vloc], s, 0, true, false, false);
            count = rc.count;
            zeros = rc.zeros;
        }
        excl = block_exclusive_scan_1b<NT>(count, s_warp, total);
        lookback_publish(A.status, b, uint64_t(total));
    }
    // ---- d) merged rows into the compact staging (records are dead), look-back (normally
    //         already resolved), coalesced copy at the symbolic offset
    const bool staged = !__syncthreads_or(slow) && total <= TR::STAGE;
    if (staged && fast) {
        int64_t o = excl;
        unsigned prev = 0xffffffffu;
#pragma unroll
        for (int j = 0; j <= NC; ++j) {
            const unsigned key = j < NC ? sk[j] : 0xffffffffu;
            const unsigned c = key == 0xffffffffu ? 0xffffffffu : (key >> 4);
            if (c != prev) {
                if (prev != 0xffffffffu) {
#pragma unroll
                    for (int t = 0; t < NV; ++t) {
                        if (!EARLY && run_val[j][t] == 0.0) continue;
                        FA_DCHECK(o < TR::STAGE, "row staging index");
                        st_col[o] = NV == 1 ? int(prev) : int(2 * prev + t);
                        st_val[o] = run_val[j][t];
                        ++o;
                    }
                }
                if (diag_at == j) {
#pragma unroll
                    for (int t = 0; t < NV; ++t) {
                        if (!EARLY && dsum[t] == 0.0) continue;
                        FA_DCHECK(o < TR::STAGE, "row staging index");
                        st_col[o] = NV == 1 ? int(vv) : int(2 * vv + t);
                        st_val[o] = dsum[t];
                        ++o;
                    }
                }
                prev = c;
            }
        }
    }
    base = lookback_wait(A.status, b, uint64_t(total), &s_prefix);  // ends with a barrier
    if (active) st_stream_i64(A.rowptr + r, int64_t(base) + excl, pol_first);
    if (active && r == A.nrows - 1) {
        A.rowptr[A.nrows] = int64_t(base) + excl + count;
        A.res->nnz = int64_t(base) + excl + count;
    }
    if (slow) atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->heavy_rows), 1ull);
    if (staged && int64_t(base) + total <= A.capacity) {
        copy_out<NT>(st_col, st_val, A.col + base, A.val + base, int(total), pol_first);
    } else if (staged) {
        for (int64_t e = tid; e < total; e += NT) {
            const int64_t g = int64_t(base) + e;
            if (g < A.capacity) {
                st_stream_i32(A.col + g, st_col[e], pol_first);
                st_stream_f64(A.val + g, st_val[e], pol_first);
            }
        }
    } else {
        if (fast) {  // direct writes (normal L2 priority: partial sectors must merge in L2)
            int64_t o = int64_t(base) + excl;
            unsigned prev = 0xffffffffu;
#pragma unroll
            for (int j = 0; j <= NC; ++j) {
                const unsigned key = j < NC ? sk[j] : 0xffffffffu;
                const unsigned c = key == 0xffffffffu ? 0xffffffffu : (key >> 4);
                if (c != prev) {
                    if (prev != 0xffffffffu) {
#pragma unroll
                        for (int t = 0; t < NV; ++t) {
                            if (!EARLY && run_val[j][t] == 0.0) continue;
                            if (o < A.capacity) {
                                A.col[o] = NV == 1 ? int(prev) : int(2 * prev + t);
                                A.val[o] = run_val[j][t];
                            }
                            ++o;
                        }
                    }
                    if (diag_at == j) {
#pragma unroll
                        for (int t = 0; t < NV; ++t) {
                            if (!EARLY && dsum[t] == 0.0) continue;
                            if (o < A.capacity) {
                                A.col[o] = NV == 1 ? int(vv) : int(2 * vv + t);
                                A.val[o] = dsum[t];
                            }
                            ++o;
                        }
                    }
                    prev = c;
                }
            }
        }
        if (slow) {
            const RowCount rc = general_row<KIND>(A, R, overflow, int64_t(gbase) + start, start, deg, v, s_oq[vloc], s, int64_t(base) + excl, true, true, EARLY);
            if (EARLY) zeros = rc.zeros;
        }
    }
    }  // !EARLY
    // zero sums of the bucket -> compaction data (k_compact runs only when some exist)
    {  // the bucket's zero count: warp sums, one shared atomic per warp that has any
        const unsigned wz = __reduce_add_sync(0xffffffffu, unsigned(zeros));
        if ((tid & 31) == 0 && wz) atomicAdd(&s_zeros, wz);
    }
    __syncthreads();
    const unsigned bz = s_zeros;
    if (tid == 0) {
        A.bsym[b] = base;
        A.blen[b] = unsigned(total);
        A.bdrop[b] = EARLY ? bz : 0u;  // !EARLY: already dropped in place
        A.read_done[b] = 0;
        if (bz) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->dropped), (unsigned long long)bz);
            if (EARLY) atomicAdd(reinterpret_cast<unsigned long long*>(&A.res->reserved[0]), (unsigned long long)bz);
        }
    }
}

// Removes the exactly-zero sums (sparse.py:177-179) in place; exits at once when there are
// none.  Block 0 first scans the per-bucket zero counts (bshift[b] = zeros of all earlier
// buckets) and fixes nnz; bucket segments then move left by their shift; a bucket writes only
// after every earlier bucket whose source range overlaps its destination has read its source
// (ticket order guarantees those are resident or finished).  Persistent grid, all resident.
constexpr int CMP_THREADS = 256;
constexpr int CMP_CAP = 4096;  // entries held per bucket (dynamic shared memory)
__global__ void __launch_bounds__(CMP_THREADS) k_compact(const unsigned long long* __restrict__ bsym,
                                                          const unsigned* __restrict__ blen,
                                                          const unsigned* __restrict__ bdrop,
                                                          const unsigned long long* bshift,
                                                          unsigned* read_done, unsigned long long* ticket, int64_t nb,
                                                          int64_t rows_per_bucket, int64_t nrows,
                                                          int64_t* __restrict__ rowptr, int32_t* col, double* val,
                                                          fa_result* res, unsigned* scan_ready) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char cmp_raw[];
    double* s_v = reinterpret_cast<double*>(cmp_raw);            // [CMP_CAP]
    int32_t* s_c = reinterpret_cast<int32_t*>(s_v + CMP_CAP);     // [CMP_CAP]
    __shared__ unsigned s_warp[CMP_THREADS / 32];
    __shared__ unsigned s_total;
    __shared__ int64_t s_tile;
    const unsigned long long dropped = res->reserved[0];  // exact zeros left in place by k_rows
    if (dropped == 0) return;
    const int tid = threadIdx.x;
    if (blockIdx.x == 0) {
        __shared__ unsigned long long s_w64[CMP_THREADS / 32];
        __shared__ unsigned long long s_t64;
        const int64_t per = (nb + CMP_THREADS - 1) / CMP_THREADS;
        const int64_t b0 = tid * per, b1 = min(nb, b0 + per);
        unsigned long long run = 0;
        for (int64_t i = b0; i < b1; ++i) run += bdrop[i];
        unsigned long long ex = block_exclusive_scan<CMP_THREADS>(run, s_w64, &s_t64);
        for (int64_t i = b0; i < b1; ++i) {
            const_cast<unsigned long long*>(bshift)[i] = ex;
            ex += bdrop[i];
        }
        __syncthreads();
        if (tid == 0) {
            const int64_t nnz = rowptr[nrows] - int64_t(dropped);
            rowptr[nrows] = nnz;
            res->nnz = nnz;
            __threadfence();
            atomicExch(scan_ready, 1u);
        }
    }
    if (tid == 0)
        for (unsigned spins = 0; atomicAdd(scan_ready, 0u) == 0u; __nanosleep(256))
            FA_DCHECK(++spins < FA_SPIN_LIMIT, "compaction scan wait");
    __syncthreads();
    __threadfence();
    while (true) {  // persistent: buckets in ticket order
    const int64_t b = next_tile(ticket, &s_tile);
    if (b >= nb) return;
    const unsigned long long S = bsym[b], len = blen[b], shift = bshift[b];
    const unsigned drops = bdrop[b];
    if (shift == 0 && drops == 0) {
        if (tid == 0) atomicExch(&read_done[b], 1u);
        continue;
    }
    const unsigned long long D = S - shift;
    // rows of the bucket: symbolic starts -> compacted starts
    const int64_t r0 = b * rows_per_bucket, r1 = min(nrows, r0 + rows_per_bucket);
    // (1) read the segment (whole when it fits) and the symbolic row starts
    const bool fits = len <= (unsigned long long)CMP_CAP;
    if (fits) {
        for (unsigned e = tid; e < len; e += CMP_THREADS) {
            s_c[e] = col[S + e];
            s_v[e] = val[S + e];
        }
    }
    int64_t rs = 0, re = 0;
    const int64_t r = r0 + tid;
    if (r < r1) {
        rs = rowptr[r];
        re = (r + 1 < r1) ? rowptr[r + 1] : int64_t(S + len);
    }
    __syncthreads();
    if (fits && tid == 0) {
        __threadfence();
        atomicExch(&read_done[b], 1u);
    }
    // (2) wait for earlier buckets whose source overlaps the destination
    if (tid == 0) {
        for (int64_t bp = b - 1; bp >= 0; --bp) {
            if (bsym[bp] + blen[bp] <= D) break;
            for (unsigned spins = 0; atomicAdd(&read_done[bp], 0u) == 0u; __nanosleep(64))
                FA_DCHECK(++spins < FA_SPIN_LIMIT, "compaction overlap wait");
        }
        __threadfence();
    }
    __syncthreads();
    // (3) compacted row starts
    unsigned kept = 0;
    if (r < r1) {
        for (int64_t e = rs; e < re; ++e) {
            const double x = fits ? s_v[e - int64_t(S)] : val[e];
            kept += x != 0.0 ? 1u : 0u;
        }
    }
    const unsigned kex = block_exclusive_scan<CMP_THREADS>(kept, s_warp, &s_total);
    if (r < r1) rowptr[r] = int64_t(D) + kex;
    // (4) entries
    if (fits) {
        unsigned base = 0;
        for (unsigned c0 = 0; c0 < len; c0 += CMP_THREADS) {
            const unsigned e = c0 + tid;
            const bool keep = e < len && s_v[e] != 0.0;
            const unsigned rank = block_exclusive_scan<CMP_THREADS>(keep ? 1u : 0u, s_warp, &s_total);
            if (keep) {
                col[D + base + rank] = s_c[e];
                val[D + base + rank] = s_v[e];
            }
            base += s_total;
            __syncthreads();
        }
    } else {
        // large segment: chunk by chunk (each chunk read before it is written; destinations
        // never reach past the chunk's own source)
        unsigned long long base = 0;
        for (unsigned long long c0 = 0; c0 < len; c0 += CMP_CAP) {
            const unsigned cl = unsigned(min((unsigned long long)CMP_CAP, len - c0));
            for (unsigned e = tid; e < cl; e += CMP_THREADS) {
                s_c[e] = col[S + c0 + e];
                s_v[e] = val[S + c0 + e];
            }
            __syncthreads();
            for (unsigned cc = 0; cc < cl; cc += CMP_THREADS) {
                const unsigned e = cc + tid;
                const bool keep = e < cl && s_v[e] != 0.0;
                const unsigned rank = block_exclusive_scan<CMP_THREADS>(keep ? 1u : 0u, s_warp, &s_total);
                if (keep) {
                    col[D + base + rank] = s_c[e];
                    val[D + base + rank] = s_v[e];
                }
                base += s_total;
                __syncthreads();
            }
        }
        if (tid == 0) {
            __threadfence();
            atomicExch(&read_done[b], 1u);
        }
    }
    __syncthreads();
    }
}


// Weighted mass: W_c = (w[me[k,c]] * area_k) / 30 for the three corners, once per triangle
// (assembly.py:232-234), coalesced; the row kernel gathers one 32-byte record per incidence.
// W_c = (w[me[k, c]] * area_k) / 30 for the three corners (assembly.py:232-234), stored as one
// 32-byte record with an L2 evict-last priority (the row kernel gathers it per incidence)
__device__ __forceinline__ void tri_wt_store(double4* Wt, int64_t k, double ar, const double (&wc)[3], uint64_t keep) {
    double4 r;
    r.x = ddiv_rcp(FMUL(wc[0], ar), 30.0, FA_RCP30);
    r.y = ddiv_rcp(FMUL(wc[1], ar), 30.0, FA_RCP30);
    r.z = ddiv_rcp(FMUL(wc[2], ar), 30.0, FA_RCP30);
    r.w = 0.0;
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(Wt + k), "d"(r.x), "d"(r.y),
                 "d"(r.z), "d"(r.w), "l"(keep)
                 : "memory");
}

constexpr int TRI_WT_U = 4;  // triangles in flight per thread
__global__ void __launch_bounds__(256) k_tri_wt(const int32_t* __restrict__ me, int64_t nme, int64_t nq,
                                                 const double* __restrict__ areas, const double* __restrict__ w,
                                                 double4* __restrict__ Wt, int64_t v0, int64_t v1) {
    const uint64_t pol = l2_evict_first_policy();
    const uint64_t keep = l2_evict_last_policy();
    const int64_t k0 = int64_t(blockIdx.x) * (256 * TRI_WT_U) + threadIdx.x;
    int c[TRI_WT_U][3];
    double ar[TRI_WT_U], wc[TRI_WT_U][3];
#pragma unroll
    for (int u = 0; u < TRI_WT_U; ++u) {
        const int64_t k = k0 + u * 256;
        c[u][0] = c[u][1] = c[u][2] = -1;
        if (k < nme) {
            c[u][0] = ld_stream_i32(me + 3 * k, pol);
            c[u][1] = ld_stream_i32(me + 3 * k + 1, pol);
            c[u][2] = ld_stream_i32(me + 3 * k + 2, pol);
            ar[u] = ld_stream_f64(areas + k, pol);
        }
    }
    bool own[TRI_WT_U];  // row blocks: only triangles with a corner in [v0, v1) are gathered
#pragma unroll
    for (int u = 0; u < TRI_WT_U; ++u) {
        bool any = false;
#pragma unroll
        for (int a = 0; a < 3; ++a) any |= c[u][a] >= v0 && c[u][a] < v1;
        own[u] = k0 + u * 256 < nme && any;
    }
#pragma unroll
    for (int u = 0; u < TRI_WT_U; ++u)
        if (own[u])
#pragma unroll
            for (int a = 0; a < 3; ++a)  // out-of-range ids (reported by the plan build) read nothing
                wc[u][a] = unsigned(c[u][a]) < nq ? ld_keep_f64(w + c[u][a], keep) : 0.0;
#pragma unroll
    for (int u = 0; u < TRI_WT_U; ++u)
        if (own[u]) tri_wt_store(Wt, k0 + u * 256, ar[u], wc[u], keep);
}

// Optional CUDA events recorded around the row kernel (bench.py's per-kernel roofline).  Inside
// a stream capture they become external event-record nodes, so a replayed graph times too.
static thread_local cudaEvent_t g_timer_begin = nullptr, g_timer_end = nullptr;

static int record_timer(cudaEvent_t ev, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    FA_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) FA_CUDA(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
    else FA_CUDA(cudaEventRecord(ev, st));
    return FA_OK;
}

template <int KIND>
static int launch_rows(const RowsArgs& A, int64_t nbuckets, cudaStream_t st) {
    const size_t smem = rows_smem_bytes<KIND>();
    FA_CUDA(cudaFuncSetAttribute(k_rows<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (g_timer_begin && record_timer(g_timer_begin, st) != FA_OK) return FA_ERR_CUDA;
    RowsArgs B = A;
    B.pf_dist = KIND == FA_KIND_ELASTIC ? KindTraits<KIND>::MIN_BLOCKS * num_sms() : 0;
    FA_CUDA(launch_pdl(7, k_rows<KIND>, dim3(unsigned(nbuckets)), dim3(KindTraits<KIND>::THREADS), smem, st, B));
    if (g_timer_end && record_timer(g_timer_end, st) != FA_OK) return FA_ERR_CUDA;
    return FA_OK;
}

}  // namespace fa

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
struct fa_plan {
    int device;
    int64_t nme, nq, v0, v1;
    int64_t nb;               // row buckets of BV vertices
    int plog, nparts;         // fine parts (sorted in shared memory)
    int plog_c, nparts_c;     // placement parts (== fine unless two_level)
    bool two_level;           // coarse placement + k_part_split (SPLIT_MIN fine parts or SPLIT_BYTES of records)
    int64_t chunk_place;
    int nblk_place;
    unsigned* part_off;       // nparts + 1 (fine)
    unsigned* part_off_c;     // nparts_c + 1 (== part_off unless two_level)
    unsigned* part_fill;      // nparts_c
    bool fine_hist;           // == two_level: k_part_hist counts the fine parts (k_part_split cursors)
    unsigned* fine_fill;      // nparts (two_level): split cursors
    bool fine_global;         // fine counts by global atomics (more than FINE_HIST_MAX fine parts)
    uint4* tri;               // row blocks: triangles with an owned corner, compacted per K1 block
    unsigned* tri_cnt;
    unsigned* M;              // [nblk_place][nparts_c]
    uint4* rec;               // 3 * nme (owned incidences, grouped by placement part)
    uint4* rec2;              // two_level: regrouped by fine part
    const int32_t* me;        // connectivity of the last build (caller keeps it: weighted mass)
    double4* Wt;              // weighted mass: per-triangle W records (allocated on first use)
    unsigned* skey;           // 3 * nme
    unsigned* sn1;
    unsigned* sn2;
    unsigned* ivptr;          // nv + 1
    uint64_t* status;         // look-back tile status (nb), then tickets and the compaction flag
    unsigned long long* bsym; // nb: symbolic CSR segment start per bucket
    unsigned* blen;           // nb
    unsigned* bdrop;          // nb: exact-zero sums per bucket
    unsigned long long* bshift;  // nb
    unsigned* read_done;      // nb (k_compact)
    int64_t ninc;             // -1 until read back
    cudaStream_t build_stream;  // stream of the last build (fa_plan_capacity reads its counts there)
    bool built;
    // fa_assemble_cold: W records written by the plan's histogram pass, consumed once
    const void* wt_key[3];    // (me, areas, w) the prepared W records belong to; consumed once
    bool wt_ready;
};

using namespace fa;

static void plan_free(fa_plan* p) {
    cudaFree(p->part_off); cudaFree(p->part_fill); cudaFree(p->fine_fill); cudaFree(p->tri); cudaFree(p->tri_cnt); cudaFree(p->M); cudaFree(p->rec); cudaFree(p->skey); cudaFree(p->sn1);
    cudaFree(p->sn2); cudaFree(p->ivptr); cudaFree(p->status);
    cudaFree(p->bsym); cudaFree(p->blen); cudaFree(p->bdrop); cudaFree(p->bshift); cudaFree(p->read_done);
    if (p->part_off_c != p->part_off) cudaFree(p->part_off_c);
    cudaFree(p->rec2);
    cudaFree(p->Wt);
}

static size_t place_smem_bytes(int nparts) {
    return size_t(3 * PLACE_TRI) * sizeof(uint4) + size_t(3) * sizeof(unsigned) * nparts;
}
static size_t sort_smem_bytes(int plog) {
    const size_t pv = size_t(1) << plog;
    return sizeof(unsigned) * pv +
           (pv == (size_t(1) << PLOG0) ? (sizeof(unsigned) * 3 + sizeof(unsigned short) * 2) * SORT_CAP : 0);  // k_part_sort
}

extern "C" int fa_plan_create(fa_plan** out, int64_t nme, int64_t nq, int64_t row_begin, int64_t row_end) {
    if (!out) { set_error("fa_plan_create: out is NULL"); return FA_ERR_ARGUMENT; }
    *out = nullptr;
    if (nme < 1 || nq < 1) { set_error("mesh needs at least one vertex and one triangle"); return FA_ERR_ARGUMENT; }
    if (row_begin < 0 || row_end > nq || row_begin > row_end) {
        set_error("row block [%lld, %lld) outside [0, %lld)", (long long)row_begin, (long long)row_end, (long long)nq);
        return FA_ERR_ARGUMENT;
    }
    if (nme >= (int64_t(1) << 30) || nq >= (int64_t(1) << 28)) {
        set_error("mesh too large: nme=%lld nq=%lld (limits 2^30 triangles, 2^28 vertices)", (long long)nme,
                  (long long)nq);
        return FA_ERR_TOO_LARGE;
    }
    fa_plan* p = new (std::nothrow) fa_plan();
    if (!p) { set_error("out of host memory"); return FA_ERR_ARGUMENT; }
    FA_CUDA(cudaGetDevice(&p->device));
    p->nme = nme; p->nq = nq; p->v0 = row_begin; p->v1 = row_end;
    const int64_t nv = row_end - row_begin;
    p->nb = (nv + BV - 1) / BV;
    // fine parts of 1024 vertices; test hook FEMASM_B200_PART_LOG2 forces larger ones (the
    // sort's general global-memory path)
    p->plog = PLOG0;
    if (const char* env = getenv("FEMASM_B200_PART_LOG2")) {
        const int forced = atoi(env);
        if (forced > p->plog && forced <= 20) p->plog = forced;
    }
    p->nparts = int((nv + (int64_t(1) << p->plog) - 1) >> p->plog);
    if (p->nparts < 1) p->nparts = 1;
    // placement coalesces runs of ~3 * PLACE_TRI / parts records: above SPLIT_MIN fine parts it
    // works on coarse parts (<= SPLIT_COARSE of them) that k_part_split regroups
    p->plog_c = p->plog;
    // two levels when the fine parts are too many for the placement's shared memory, or when
    // the records (16 bytes per owned incidence) do not stay in L2 until the sort reads them
    const int64_t rec_bytes_est = int64_t(48) * nme / (nq > 0 ? nq : 1) * nv;
    p->two_level = p->nparts > SPLIT_MIN || (rec_bytes_est > SPLIT_BYTES && p->nparts > SPLIT_COARSE);
    if (p->two_level)
        while (((nv + (int64_t(1) << p->plog_c) - 1) >> p->plog_c) > SPLIT_COARSE) ++p->plog_c;
    if (const char* env = getenv("FEMASM_B200_COARSE_LOG2")) {  // test hook: force a two-level plan
        const int forced = atoi(env);
        if (forced > p->plog && forced <= p->plog + 8) {
            p->two_level = true;
            p->plog_c = forced;
        }
    }
    p->nparts_c = int((nv + (int64_t(1) << p->plog_c) - 1) >> p->plog_c);
    if (p->nparts_c < 1) p->nparts_c = 1;
    p->fine_hist = p->two_level;
    p->fine_global = p->two_level && (p->nparts > FINE_HIST_MAX || p->nparts_c > SPLIT_COARSE);
    if (const char* env = getenv("FEMASM_B200_FINE_GLOBAL"))  // test hook: global fine counts
        if (atoi(env) == 1 && p->two_level) p->fine_global = true;
    int place_blocks = PLACE_BLOCKS_PER_SM * num_sms();
    if (const char* env = getenv("FEMASM_B200_PLACE_BLOCKS"))  // test hook: fewer histogram/placement blocks
        if (atoi(env) >= 1) place_blocks = atoi(env);
    p->chunk_place = (nme + place_blocks - 1) / place_blocks;
    p->nblk_place = int((nme + p->chunk_place - 1) / p->chunk_place);
    p->ninc = -1;
    const size_t ninc_max = size_t(3) * size_t(nme);
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&p->part_off, sizeof(unsigned) * (p->nparts + 1));
    p->part_off_c = p->part_off;
    if (e == cudaSuccess && p->two_level) e = cudaMalloc(&p->part_off_c, sizeof(unsigned) * (p->nparts_c + 1));
    if (e == cudaSuccess && p->two_level) e = cudaMalloc(&p->rec2, sizeof(uint4) * ninc_max);
    if (e == cudaSuccess) e = cudaMalloc(&p->part_fill, sizeof(unsigned) * p->nparts_c);
    if (e == cudaSuccess && p->fine_hist) e = cudaMalloc(&p->fine_fill, sizeof(unsigned) * p->nparts);
    if (row_begin > 0 || row_end < nq) {  // row block: the placement visits only owning triangles
        if (e == cudaSuccess) e = cudaMalloc(&p->tri, sizeof(uint4) * size_t(nme));
        if (e == cudaSuccess) e = cudaMalloc(&p->tri_cnt, sizeof(unsigned) * size_t(p->nblk_place));
    }
    if (e == cudaSuccess) e = cudaMalloc(&p->M, sizeof(unsigned) * size_t(p->nblk_place) * p->nparts_c);
    if (e == cudaSuccess) e = cudaMalloc(&p->rec, sizeof(uint4) * ninc_max);
    if (e == cudaSuccess) e = cudaMalloc(&p->skey, sizeof(unsigned) * ninc_max);
    if (e == cudaSuccess) e = cudaMalloc(&p->sn1, sizeof(unsigned) * ninc_max);
    if (e == cudaSuccess) e = cudaMalloc(&p->sn2, sizeof(unsigned) * ninc_max);
    if (e == cudaSuccess) e = cudaMalloc(&p->ivptr, sizeof(unsigned) * (nv + 1));
    // look-back status (nb) + the row-kernel ticket, the compaction ticket and scan flag
    if (e == cudaSuccess) e = cudaMalloc(&p->status, sizeof(uint64_t) * ((p->nb > 0 ? p->nb : 1) + 4));
    const size_t nbk = size_t(p->nb > 0 ? p->nb : 1);
    if (e == cudaSuccess) e = cudaMalloc(&p->bsym, sizeof(unsigned long long) * nbk);
    if (e == cudaSuccess) e = cudaMalloc(&p->blen, sizeof(unsigned) * nbk);
    if (e == cudaSuccess) e = cudaMalloc(&p->bdrop, sizeof(unsigned) * nbk);
    if (e == cudaSuccess) e = cudaMalloc(&p->bshift, sizeof(unsigned long long) * nbk);
    if (e == cudaSuccess) e = cudaMalloc(&p->read_done, sizeof(unsigned) * nbk);

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

// pdl: the plan kernels are launched as programmatic dependents of each other (launch_pdl).
// wt_areas, wt_w (weighted mass, fa_assemble_cold): K1 also writes the W records.
static int plan_build(fa_plan* p, const int32_t* d_me, fa_result* d_res, void* stream, bool pdl,
                      const double* wt_areas = nullptr, const double* wt_w = nullptr);

extern "C" int fa_plan_build(fa_plan* p, const int32_t* d_me, fa_result* d_res, void* stream) {
    NvtxRange nv("fa_plan_build");
    return plan_build(p, d_me, d_res, stream, true);
}

static int plan_build(fa_plan* p, const int32_t* d_me, fa_result* d_res, void* stream, bool pdl,
                      const double* wt_areas, const double* wt_w) {
    if (!p || !d_me || !d_res) { set_error("fa_plan_build: NULL argument"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    p->ninc = -1;
    p->built = true;
    p->build_stream = st;
    if (p->nb == 0) {
        k_result_reset<<<1, 32, 0, st>>>(d_res);
        return FA_OK;
    }
    p->me = d_me;
    // result + the part counts K1 accumulates (fine ones when it counts fine parts)
    if (p->fine_hist)
        FA_CUDA(launch_pdl(pdl ? 0 : -1, k_reset, dim3(8), dim3(256), 0, st, d_res, p->part_off, int64_t(p->nparts + 1),
                           (uint64_t*)nullptr, int64_t(0)));
    else
        FA_CUDA(launch_pdl(pdl ? 0 : -1, k_reset, dim3(4), dim3(256), 0, st, d_res, p->part_off_c, int64_t(p->nparts_c + 1),
                           (uint64_t*)nullptr, int64_t(0)));
    PlanArgs P;  // placement level (coarse parts when two_level)
    P.me = d_me; P.nme = p->nme; P.nq = p->nq; P.v0 = p->v0; P.v1 = p->v1;
    P.plog = p->plog_c; P.nparts = p->nparts_c; P.chunk = p->chunk_place;
    P.part_off = p->part_off_c; P.part_fill = p->part_fill; P.M = p->M; P.rec = p->rec;
    P.skey = p->skey; P.sn1 = p->sn1; P.sn2 = p->sn2; P.ivptr = p->ivptr; P.res = d_res;
    P.plog_f = p->plog; P.nparts_f = p->nparts; P.fine_hist = p->fine_hist;
    P.fine_global = p->fine_global;
    P.tri = p->tri; P.tri_cnt = p->tri_cnt;
    P.part_off_f = p->part_off; P.fine_fill = p->fine_fill;
    P.wt_areas = wt_areas; P.wt_w = wt_w; P.Wt = nullptr; P.sort_pf = 0;
    if (wt_areas && wt_w) {
        if (!p->Wt) FA_CUDA(cudaMalloc(&p->Wt, sizeof(double4) * size_t(p->nme)));
        P.Wt = p->Wt;
    }
    const size_t hist_smem = sizeof(unsigned) * (P.fine_hist && !P.fine_global ? (p->nparts + 1) / 2 : p->nparts_c);
    {
        const int mode = !P.fine_hist ? 0 : (P.fine_global ? 2 : 1);
        const bool rb = P.tri != nullptr;
        void (*hist)(PlanArgs) = mode == 0 ? (rb ? k_part_hist<0, true> : k_part_hist<0, false>)
                                 : mode == 1 ? (rb ? k_part_hist<1, true> : k_part_hist<1, false>)
                                             : (rb ? k_part_hist<2, true> : k_part_hist<2, false>);
        FA_CUDA(cudaFuncSetAttribute(hist, cudaFuncAttributeMaxDynamicSharedMemorySize, int(hist_smem)));
        FA_CUDA(launch_pdl(pdl ? 1 : -1, hist, dim3(p->nblk_place), dim3(PLACE_THREADS), hist_smem, st, P));
    }
    const int sper = scan_per(P.fine_hist ? p->nparts : p->nparts_c);
    FA_CUDA(cudaFuncSetAttribute(k_part_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, int(scan_smem_bytes(SCAN_PER))));
    FA_CUDA(launch_pdl(pdl ? 2 : -1, k_part_scan, dim3(1), dim3(PLAN_THREADS), scan_smem_bytes(sper), st, P, sper));
    const size_t place_smem = place_smem_bytes(p->nparts_c);
    {
        void (*place)(PlanArgs) = P.tri ? k_part_place<true> : k_part_place<false>;
        FA_CUDA(cudaFuncSetAttribute(place, cudaFuncAttributeMaxDynamicSharedMemorySize, int(place_smem)));
        FA_CUDA(launch_pdl(pdl ? 3 : -1, place, dim3(p->nblk_place), dim3(PLACE_THREADS), place_smem, st, P));
    }
    if (p->fine_hist) {
        constexpr int RI = SPLIT_RI;
        const size_t split_smem = size_t(RI) * sizeof(uint4) + sizeof(unsigned) * 3 * SPLIT2_LOCAL;
        FA_CUDA(cudaFuncSetAttribute(k_part_split, cudaFuncAttributeMaxDynamicSharedMemorySize, int(split_smem)));
        int nsm = 0, dev = 0;
        FA_CUDA(cudaGetDevice(&dev));
        FA_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int64_t rounds = (3 * p->nme + RI - 1) / RI;  // upper bound on the owned incidences
        const unsigned grid = unsigned(rounds < int64_t(nsm) * SPLIT_MINB ? rounds : int64_t(nsm) * SPLIT_MINB);
        FA_CUDA(launch_pdl(pdl ? 4 : -1, k_part_split, dim3(grid), dim3(SPLIT_THREADS), split_smem, st, p->rec,
                           p->part_off + p->nparts, p->plog, p->fine_fill, p->rec2));
    }
    P.plog = p->plog; P.nparts = p->nparts; P.part_off = p->part_off;  // sort level: fine parts
    P.rec = p->two_level ? p->rec2 : p->rec;
    const size_t sort_smem = sort_smem_bytes(p->plog);
    P.sort_pf = SORT_PF_SMS * num_sms();
    FA_CUDA(cudaFuncSetAttribute(k_part_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sort_smem)));
    FA_CUDA(launch_pdl(pdl ? 5 : -1, k_part_sort, dim3(p->nparts), dim3(SORT_THREADS), sort_smem, st, P));
    return FA_OK;
}


extern "C" int fa_set_kernel_timer(void* ev_begin, void* ev_end) {
    g_timer_begin = reinterpret_cast<cudaEvent_t>(ev_begin);
    g_timer_end = reinterpret_cast<cudaEvent_t>(ev_end);
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
            unsigned total = 0;
            // ordered after the build on its own stream (a non-blocking stream does not
            // synchronise with the legacy default stream)
            FA_CUDA(cudaMemcpyAsync(&total, p->part_off + p->nparts, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                    p->build_stream));
            FA_CUDA(cudaStreamSynchronize(p->build_stream));
            p->ninc = int64_t(total);
        }
    }
    // per vertex: at most 2*deg neighbours + itself; ELASTIC: 2 rows x 2 columns per vertex
    const int64_t per = (kind == FA_KIND_ELASTIC) ? 4 : 1;
    *capacity = per * (2 * p->ninc + nv);
    return FA_OK;
}

// Weighted mass: the per-triangle W records of the plan's connectivity (k_tri_wt).
static int launch_tri_wt(fa_plan* p, const double* d_areas, const double* d_w, cudaStream_t st) {
    if (!p->Wt) FA_CUDA(cudaMalloc(&p->Wt, sizeof(double4) * size_t(p->nme)));
    k_tri_wt<<<unsigned((p->nme + 256 * TRI_WT_U - 1) / (256 * TRI_WT_U)), 256, 0, st>>>(p->me, p->nme, p->nq, d_areas,
                                                                                       d_w, p->Wt, p->v0, p->v1);
    FA_LAUNCH_CHECK("k_tri_wt");
    return FA_OK;
}

extern "C" int fa_assemble(fa_plan* p, int kind, const double* d_q, const double* d_areas, const double* d_w,
                           double lam, double mu, int64_t* d_rowptr, int32_t* d_col, double* d_val, int64_t capacity,
                           fa_result* d_res, void* stream) {
    static const char* const kNames[4] = {"fa_assemble mass", "fa_assemble massw", "fa_assemble stiff",
                                          "fa_assemble elastic"};
    NvtxRange nv(kind >= 0 && kind < 4 ? kNames[kind] : "fa_assemble");
    if (!p || !p->built) { set_error("fa_assemble: plan not built"); return FA_ERR_ARGUMENT; }
    if (!d_rowptr || !d_col || !d_val || !d_res) { set_error("fa_assemble: NULL output"); return FA_ERR_ARGUMENT; }
    if (kind < 0 || kind > 3) { set_error("unknown matrix kind %d", kind); return FA_ERR_ARGUMENT; }
    if ((kind == FA_KIND_STIFF || kind == FA_KIND_ELASTIC || !d_areas) && !d_q) {
        set_error("fa_assemble: vertex coordinates required"); return FA_ERR_ARGUMENT;
    }
    if (kind == FA_KIND_MASSW && !d_w) { set_error("WEIGHTED_MASS requires a WeightField"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    const int64_t nrows = fa_plan_rows(p, kind);
    if (nrows == 0 || p->nb == 0) {
        k_result_reset<<<1, 32, 0, st>>>(d_res);
        FA_CUDA(cudaMemsetAsync(d_rowptr, 0, sizeof(int64_t), st));
        return FA_OK;
    }
    // result block, look-back status (nb), the row-kernel and compaction tickets and the
    // compaction's scan flag (p->status has nb + 4 words)
    FA_CUDA(launch_pdl(6, k_reset, dim3(unsigned((p->nb + 4 + 255) / 256 < 64 ? (p->nb + 4 + 255) / 256 : 64)), dim3(256),
                       0, st, d_res, (unsigned*)nullptr, int64_t(0), p->status, int64_t(p->nb + 4)));
    RowsArgs A;
    A.skey = p->skey; A.sn1 = p->sn1; A.sn2 = p->sn2; A.ivptr = p->ivptr;
    A.q = reinterpret_cast<const double2*>(d_q); A.w = d_w; A.areas = d_areas;
    A.lam = lam; A.mu = mu;
    A.v0 = p->v0; A.v1 = p->v1; A.nrows = nrows;
    A.rowptr = d_rowptr; A.col = d_col; A.val = d_val; A.capacity = capacity;
    A.status = p->status; A.ticket = reinterpret_cast<unsigned long long*>(p->status + p->nb); A.res = d_res;
    A.read_done = p->read_done;
    A.bsym = p->bsym; A.blen = p->blen; A.bdrop = p->bdrop;
    A.Wt = nullptr;
    if (kind == FA_KIND_MASSW) {  // the triangles' W once (k_tri_wt), gathered per incidence
        if (!d_areas) { set_error("WEIGHTED_MASS requires areas"); return FA_ERR_ARGUMENT; }
        const bool prepared = p->wt_ready && p->wt_key[0] == p->me && p->wt_key[1] == d_areas && p->wt_key[2] == d_w;
        p->wt_ready = false;
        if (!prepared) {
            const int rc = launch_tri_wt(p, d_areas, d_w, st);
            if (rc != FA_OK) return rc;
        }
        A.Wt = p->Wt;
    }
    int rc;
    switch (kind) {
        case FA_KIND_MASS: rc = launch_rows<FA_KIND_MASS>(A, p->nb, st); break;
        case FA_KIND_MASSW: rc = launch_rows<FA_KIND_MASSW>(A, p->nb, st); break;
        case FA_KIND_STIFF: rc = launch_rows<FA_KIND_STIFF>(A, p->nb, st); break;
        default: rc = launch_rows<FA_KIND_ELASTIC>(A, p->nb, st); break;
    }
    if (rc != FA_OK) return rc;
    // exact-zero sums (if any) removed in place; exits at once when there are none
    const int64_t rpb = int64_t(BV) * (kind == FA_KIND_ELASTIC ? 2 : 1);
    const size_t cmp_smem = size_t(CMP_CAP) * (sizeof(double) + sizeof(int32_t));
    FA_CUDA(cudaFuncSetAttribute(k_compact, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cmp_smem)));
    const int64_t cmax = 2 * int64_t(num_sms());
    const unsigned cgrid = unsigned(p->nb < cmax ? p->nb : cmax);
    FA_CUDA(launch_pdl(8, k_compact, dim3(cgrid), dim3(CMP_THREADS), cmp_smem, st, p->bsym, p->blen, p->bdrop, p->bshift,
                       p->read_done, reinterpret_cast<unsigned long long*>(p->status + p->nb + 1), int64_t(p->nb), rpb,
                       nrows, d_rowptr, d_col, d_val, d_res, reinterpret_cast<unsigned*>(p->status + p->nb + 2)));
    return FA_OK;
}

// Plan build + numeric assembly in one call (the cold OptV2 of the reference API).  For the
// weighted mass the plan's histogram pass (which reads the connectivity anyway) also writes
// the per-triangle W records, so no separate k_tri_wt pass runs.
extern "C" int fa_assemble_cold(fa_plan* p, const int32_t* d_me, int kind, const double* d_q, const double* d_areas,
                                const double* d_w, double lam, double mu, int64_t* d_rowptr, int32_t* d_col,
                                double* d_val, int64_t capacity, fa_result* d_build_result, fa_result* d_result,
                                void* stream) {
    NvtxRange nv("fa_assemble_cold");
    if (!p || !d_me || !d_build_result) { set_error("fa_assemble_cold: NULL argument"); return FA_ERR_ARGUMENT; }
    // weighted mass: the plan's histogram pass also writes the W records (k_tri_wt's work)
    const bool wt = kind == FA_KIND_MASSW && d_areas && d_w && p->nb > 0;
    int rc = plan_build(p, d_me, d_build_result, stream, true, wt ? d_areas : nullptr, wt ? d_w : nullptr);
    if (rc != FA_OK) return rc;
    if (wt) {
        p->wt_key[0] = d_me; p->wt_key[1] = d_areas; p->wt_key[2] = d_w;
        p->wt_ready = true;
    }
    return fa_assemble(p, kind, d_q, d_areas, d_w, lam, mu, d_rowptr, d_col, d_val, capacity, d_result, stream);
}

// Development diagnostics (not part of include/femasm_b200.h): copies a plan array to the host
// after synchronising the device.  what: 0 fine part offsets (nparts + 1), 1 placement part
// offsets (nparts_c + 1), 2 count matrix (nblk_place x nparts_c).
extern "C" int fa_plan_debug(fa_plan* p, int what, void* host_out, int64_t n) {
    if (!p || !host_out) return FA_ERR_ARGUMENT;
    FA_CUDA(cudaDeviceSynchronize());
    const unsigned* src = what == 0 ? p->part_off : what == 1 ? p->part_off_c : p->M;
    const int64_t avail = what == 0 ? p->nparts + 1 : what == 1 ? p->nparts_c + 1 : int64_t(p->nblk_place) * p->nparts_c;
    FA_CUDA(cudaMemcpy(host_out, src, sizeof(unsigned) * size_t(n < avail ? n : avail), cudaMemcpyDeviceToHost));
    return FA_OK;
}
