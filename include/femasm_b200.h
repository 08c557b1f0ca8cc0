/*
 * femasm_b200 — C ABI of the B200-native OptV2 P1 assembly library.
 *
 * This is the drop-in boundary for the one hot path of the reference package
 * `femasm` (/root/reference/pkg/src/femasm): `assemble(mesh, kind, Strategy.OPTV2)`
 * and the batch kernels it is built from.  The reference is pure Python/numpy and
 * has no FFI of its own; the Python package `paper_1305_3122_b200` binds these
 * symbols with ctypes (paper_1305_3122_b200/_lib.py) and keeps the reference's
 * Python API on top (INTEGRATION.md shows the binding a femasm maintainer would add).
 *
 * Conventions
 *  - Every pointer named d_* is a CUDA device pointer on the current device.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - All calls are stream-ordered and asynchronous unless stated otherwise; the
 *    library never frees caller memory.  A plan owns its workspace.
 *  - Return value: FA_OK or an FA_ERR_* launch/argument status.  Errors found
 *    *on the device* (degenerate triangle, out-of-range index) are written to the
 *    caller's fa_result block and become visible after the stream is synchronised;
 *    fa_result_status() maps a host copy of that block to a status code.
 *  - Value arithmetic is IEEE fp64 without FMA contraction, in the reference's
 *    operation order, so element values are bitwise those of numpy.
 */
#ifndef FEMASM_B200_H
#define FEMASM_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Matrix kinds: femasm MatrixKind (assembly.py:48-62). */
enum fa_kind {
    FA_KIND_MASS = 0,      /* MatrixKind.MASS            batch_kg_mass          assembly.py:214 */
    FA_KIND_MASSW = 1,     /* MatrixKind.WEIGHTED_MASS   batch_kg_mass_weighted assembly.py:227 */
    FA_KIND_STIFF = 2,     /* MatrixKind.STIFFNESS       batch_kg_stiff         assembly.py:246 */
    FA_KIND_ELASTIC = 3    /* MatrixKind.ELASTIC         batch_kg_elastic       assembly.py:267 */
};

enum fa_status {
    FA_OK = 0,
    FA_ERR_ARGUMENT = 1,    /* bad argument (ValueError in the reference)                        */
    FA_ERR_DEGENERATE = 2,  /* area <= 1e-300: DegenerateTriangleError (mesh.py:33, assembly.py:152) */
    FA_ERR_INDEX = 3,       /* index out of range (sparse.py:131-137, mesh.py:95-96)               */
    FA_ERR_CUDA = 4,        /* CUDA runtime error                                                 */
    FA_ERR_TOO_LARGE = 5,   /* size beyond the library's index widths                             */
    FA_ERR_LENGTH = 6       /* triplet arrays disagree in length (sparse.py:151-154)               */
};

/* Device-side result / error block (caller allocates sizeof(fa_result) bytes of device
 * memory; fa_* entry points reset and fill it).  Index fields are INT64_MAX when unset and hold
 * the SMALLEST offending index otherwise (np.flatnonzero(...)[0] semantics). */
typedef struct fa_result {
    int64_t nnz;               /* stored entries after Matlab-sparse zero drops          */
    int64_t degenerate_index;  /* first triangle with area <= 1e-300                       */
    int64_t index_error_pos;   /* first out-of-range connectivity / row index position     */
    int64_t col_error_pos;     /* first out-of-range column index position (triplets)      */
    int64_t dropped;           /* positions dropped because their sum was exactly 0.0     */
    int64_t heavy_rows;        /* rows that took the general (degree > 8) path             */
    int64_t reserved[1];       /* internal: exact zeros left for the in-place compaction    */
    int64_t repeat_error_pos;  /* first connectivity position repeating a vertex id of its
                                  triangle (femasm Mesh rejects those, mesh.py:98-103)       */
} fa_result;

/* Map a HOST copy of an fa_result block to a status code (FA_OK when clean). */
int fa_result_status(const fa_result* host_result);

/* Human-readable description of the last error raised on the calling host thread. */
const char* fa_last_error(void);
const char* fa_version(void);

/* ------------------------------------------------------------------------------------
 * Assembly plan: the symbolic part of OptV2 for one mesh connectivity and one block of
 * vertex rows [row_begin, row_end) (the whole mesh: 0, nq).  Replaces the index builders
 * build_ig_jg_p1 / build_ig_jg_p1_vector (assembly.py:162-192) and the sort of
 * csc_from_triplets (sparse.py:164-168): it records, per owned vertex, the incident
 * (triangle, local corner) pairs.  Multi-GPU: one plan per rank with its row block.
 * ---------------------------------------------------------------------------------- */
typedef struct fa_plan fa_plan;

/* Allocate a plan's workspace (device memory on the current device).  Synchronous. */
int fa_plan_create(fa_plan** out, int64_t nme, int64_t nq, int64_t row_begin, int64_t row_end);

/* (Re)build the incidence structure from connectivity d_me (nme x 3 int32, row-major,
 * 0-based): every owned vertex's (triangle, corner, neighbours) list, sorted by triangle.
 * Asynchronous on `stream`; d_me must stay valid and unchanged until the next
 * fa_plan_build or fa_plan_destroy (the weighted-mass numeric pass reads it once per
 * triangle).  Out-of-range vertex ids are reported in d_result. */
int fa_plan_build(fa_plan* plan, const int32_t* d_me, fa_result* d_result, void* stream);

/* Upper bound on stored entries for `kind` over the plan's rows (capacity of d_col/d_val):
 * sum over owned vertices of nv * (2*deg+1) * (rows per vertex).  Synchronous only the
 * first time it is called after a build (reads the incidence count). */
int fa_plan_capacity(fa_plan* plan, int kind, int64_t* capacity);

/* Number of matrix rows the plan produces for `kind` (row block size times 1 or 2). */
int64_t fa_plan_rows(const fa_plan* plan, int kind);

int fa_plan_destroy(fa_plan* plan);

/* ------------------------------------------------------------------------------------
 * Numeric OptV2 assembly over the plan's rows, fused element values + Matlab sparse():
 * replaces batch_kg_* (assembly.py:214-307) + TripletBatch.to_csc (sparse.py:318-329) +
 * csc_from_triplets (sparse.py:140-189).  Output is CSR over the plan's rows with LOCAL
 * row pointers (d_rowptr[0] = 0, d_rowptr[rows] = nnz) and GLOBAL column ids.  Because
 * every element matrix is exactly symmetric and every position is summed in ascending
 * triangle order, these arrays equal the reference CscMatrix col_ptr/row_idx/values
 * bit for bit.
 *   d_q      (nq x 2) f64 vertex coordinates (STIFF, ELASTIC; may be NULL for MASS, MASSW)
 *   d_areas  (nme) f64 triangle areas, or NULL to recompute them bitwise from d_q with
 *            compute_areas' formula (mesh.py:62-65) - only valid for areas produced by it;
 *            required for MASSW
 *   d_w      (nq) f64 vertex weights (MASSW only; WeightField.sample, assembly.py:114)
 *   lam, mu  Lame parameters (ELASTIC only; ElasticParams, elements.py:81-103)
 * Exact-zero sums are dropped (sparse.py:177-179) and counted in d_result->dropped.
 * Capacity must be >= fa_plan_capacity(kind).  Asynchronous. */
int fa_assemble(fa_plan* plan, int kind, const double* d_q, const double* d_areas,
                const double* d_w, double lam, double mu, int64_t* d_rowptr, int32_t* d_col,
                double* d_val, int64_t capacity, fa_result* d_result, void* stream);

/* Cold OptV2 in one call: fa_plan_build(d_me) followed by fa_assemble, i.e. the whole
 * reference assemble(mesh, kind, OPTV2) (assembly.py:419-452) on device buffers.  Plan
 * build errors land in d_build_result, numeric ones in d_result.  For MASSW the plan's
 * connectivity pass also computes the per-triangle weight records (no separate pass).
 * capacity: >= fa_plan_capacity after the build; 3 * (2 * 3 * nme + rows) (x4 for ELASTIC's
 * 2x2 blocks: use fa_plan_capacity's formula with 3 * nme incidences) is always enough. */
int fa_assemble_cold(fa_plan* plan, const int32_t* d_me, int kind, const double* d_q,
                     const double* d_areas, const double* d_w, double lam, double mu,
                     int64_t* d_rowptr, int32_t* d_col, double* d_val, int64_t capacity,
                     fa_result* d_build_result, fa_result* d_result, void* stream);

/* ------------------------------------------------------------------------------------
 * Batch (OptV2 building-block) kernels of the reference API, SoA layout (r x nme, row il
 * contiguous, i.e. the reference's C-ordered Kg).
 * ---------------------------------------------------------------------------------- */

/* batch_kg_mass / _mass_weighted / _stiff / _elastic (assembly.py:214-307): d_kg has
 * r*nme doubles, r = 9 (scalar) or 36 (ELASTIC).  MASS reads only d_areas; MASSW reads
 * d_me, d_areas, d_w; STIFF/ELASTIC read d_me, d_q, d_areas. */
int fa_element_kg(int kind, const int32_t* d_me, int64_t nme, const double* d_q,
                  const double* d_areas, const double* d_w, double lam, double mu,
                  double* d_kg, fa_result* d_result, void* stream);

/* build_ig_jg_p1 (vector=0, r=9) / build_ig_jg_p1_vector (vector=1, r=36)
 * (assembly.py:162-192): d_ig, d_jg each r*nme int32, SoA. */
int fa_build_ig_jg(int vector, const int32_t* d_me, int64_t nme, int32_t* d_ig, int32_t* d_jg,
                   void* stream);

/* batch_gradients (assembly.py:195-211): d_g is 6*nme doubles laid out as
 * [g1x, g1y, g2x, g2y, g3x, g3y] rows of nme. */
int fa_batch_gradients(const int32_t* d_me, int64_t nme, const double* d_q, const double* d_areas,
                       double* d_g, fa_result* d_result, void* stream);

/* Mesh construction on the device (femasm Mesh.__init__, mesh.py:84-119 + compute_areas,
 * mesh.py:51-69) in one pass over the caller's int64 connectivity d_me64 (nme x 3): the first
 * out-of-range flattened position -> d_result->index_error_pos, the first triangle repeating a
 * vertex id -> repeat_error_pos, the int32 copy the plans use -> d_me32, areas (bitwise
 * compute_areas; 0 for a triangle with a bad id) -> d_areas, the first area <= 1e-300 ->
 * degenerate_index.  The caller raises them in the reference's order (range, repeat, area). */
int fa_mesh_ingest(const int64_t* d_me64, int64_t nme, int64_t nq, const double* d_q,
                   int32_t* d_me32, double* d_areas, fa_result* d_result, void* stream);

/* compute_areas (mesh.py:51-69): 0.5*|cross|, first area <= 1e-300 reported. */
int fa_compute_areas(const int32_t* d_me, int64_t nme, const double* d_q, double* d_areas,
                     fa_result* d_result, void* stream);

/* ------------------------------------------------------------------------------------
 * General Matlab sparse(): csc_from_triplets (sparse.py:140-189) for arbitrary triplet
 * streams (rectangular, any order, long duplicate runs): range checks with the first
 * offending position, input zeros skipped, stable sort by (col, row), left-to-right sums,
 * exact-zero sums dropped.  Outputs CSC: d_colptr (n_cols+1), d_rowidx/d_vals (capacity
 * len).  Workspace: fa_triplets_workspace(len) bytes of device memory.
 * ---------------------------------------------------------------------------------- */
size_t fa_triplets_workspace(int64_t len, int64_t n_rows, int64_t n_cols);
int fa_triplets_to_csc(const int64_t* d_rows, const int64_t* d_cols, const double* d_vals,
                       int64_t len, int64_t n_rows, int64_t n_cols, int64_t* d_colptr,
                       int64_t* d_rowidx, double* d_vals_out, void* d_workspace,
                       size_t workspace_bytes, fa_result* d_result, void* stream);

/* fa_triplets_to_csc with flags.  FA_TRIPLETS_KEEP_ZEROS gives the reference CscBuilder's
 * semantics (sparse.py:208-290, used by the CLASSICAL / OPTV0 element loops,
 * assembly.py:359-375): every position a triplet names is stored - input zeros and zero sums
 * included - and each position's sum starts from its first value (`aa[pos] += v`). */
#define FA_TRIPLETS_KEEP_ZEROS 1
int fa_triplets_to_csc_ex(const int64_t* d_rows, const int64_t* d_cols, const double* d_vals,
                          int64_t len, int64_t n_rows, int64_t n_cols, int flags, int64_t* d_colptr,
                          int64_t* d_rowidx, double* d_vals_out, void* d_workspace,
                          size_t workspace_bytes, fa_result* d_result, void* stream);

/* Element-loop strategies CLASSICAL / OPTV0 / OPTV1 (assembly.py:359-397): the triplets of
 * every triangle's element matrix computed with the per-element formulas of elements.py:34-154
 * (elem_mass, elem_mass_weighted, elem_stiff, elem_stiff_elastic - rounded differently from the
 * batch kernels), in triangle-major order: position k*r + a + order*b holds entry (a, b) of
 * triangle k, order 3 (r = 9) or 6 (ELASTIC, r = 36, interleaved dofs).  d_rows/d_cols int64,
 * d_vals f64, r*nme each.  A triangle with area <= 1e-300 is reported in d_result. */
int fa_element_triplets(int kind, const int32_t* d_me, int64_t nme, const double* d_q,
                        const double* d_areas, const double* d_w, double lam, double mu,
                        int64_t* d_rows, int64_t* d_cols, double* d_vals, fa_result* d_result,
                        void* stream);

/* CSC (col_ptr, row_idx int64; values f64; host arrays) -> coordinate MatrixMarket file, byte
 * identical to femasm's write_matrix_market (pkg/src/femasm/sparse.py:332-339): 1-based "i j v"
 * lines in CSC order, values "%.17g".  threads <= 0: all hardware threads.  Host only. */
int fa_write_matrix_market(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* col_ptr,
                           const int64_t* row_idx, const double* values, int threads);

/* femasm read_mesh (mesh.py:225-286) for well-formed files: header "nq nme", nq lines "x y",
 * nme lines of 1-based ids.  Host only, multithreaded (threads <= 0: all).  Call with
 * vertices == connectivity == NULL to read the header into *nq / *nme, then with (nq x 2) f64
 * and (nme x 3) int64 (0-based ids written) buffers.  FA_ERR_ARGUMENT (no message) when the
 * file is not in the strict layout write_mesh produces - the caller then parses it with the
 * reference's rules, which produce the reference's MeshFormatError. */
int fa_read_mesh_text(const char* path, int64_t* nq, int64_t* nme, double* vertices,
                      int64_t* connectivity, int threads);

/* ------------------------------------------------------------------------------------
 * Diagnostics.  fa_selftest_division compares the library's call-free correctly rounded
 * fp64 division (used by every element value) bitwise with CUDA's __ddiv_rn on n generated
 * operand pairs; *d_bad receives the mismatch count, d_first[0..3] = x, y, mine, ref of one.
 * ---------------------------------------------------------------------------------- */
int fa_selftest_division(int64_t n, uint64_t seed, unsigned long long* d_bad, double* d_first,
                         void* stream);

/* Record two caller-created CUDA events (cudaEvent_t as void*) around every subsequent row
 * kernel launch of fa_assemble on the calling host thread (NULL, NULL disables).  Used by
 * bench.py to time the dominant kernel for its roofline figure. */
int fa_set_kernel_timer(void* ev_begin, void* ev_end);

#ifdef __cplusplus
}
#endif
#endif /* FEMASM_B200_H */
