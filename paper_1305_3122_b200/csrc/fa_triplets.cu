// General Matlab sparse(I, J, K, m, n) on the GPU: csc_from_triplets (sparse.py:140-189)
// for arbitrary triplet streams, used by the public csc_from_triplets / TripletBatch.to_csc
// API.  (assemble() never materialises triplets; it uses the fused row kernel.)
//
// Semantics kept from the reference:
//   - range checks with the first offending position, rows before columns (:157-158)
//   - input zeros ignored (:160-162): adding +-0.0 never changes a partial sum here and an
//     all-zero position sums to 0.0 and is dropped, so zeros are carried, not filtered
//   - code = col * n_rows + row (:164-165), STABLE sort (:166): LSD radix sort of (code, value)
//     pairs, 8-bit digits; each pass ranks a 4096-pair tile stably by digit in shared memory
//     (warp match + ordered per-warp counters), stages it in digit order and writes every
//     digit's run coalesced at its global offset (digit-major scan of the tile histograms)
//   - per position, left-to-right sum in input order (:176): the sort is stable, so each run's
//     values arrive in input order; one thread per run sums them sequentially (a tree or
//     shuffle reduction would round differently)
//   - exact-zero sums dropped (:177-179), row = code % n_rows, col = code / n_rows (:180-181)
//   - col_ptr = cumulative column counts (:187-188)
#include <climits>

#include "fa_common.cuh"

namespace fa {

constexpr int TS_BLOCK = 256;
constexpr int TS_ROUNDS = 16;
constexpr int TS_TILE = TS_BLOCK * TS_ROUNDS;
constexpr int TS_RADIX = 256;
constexpr size_t TS_STAGE_BYTES = size_t(TS_TILE) * (sizeof(uint64_t) + sizeof(double));  // k_trip_scatter staging

struct TripletWs {
    uint64_t *key0, *key1;
    double *val0, *val1;
    int64_t* hist;      // TS_RADIX * ntiles (+1)
    int* flag;          // len
    int64_t* pos;       // len + 1
    uint64_t* status;   // look-back
    unsigned long long* ticket;
    int64_t ntiles, scan_tiles;
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static size_t carve(TripletWs* w, void* base, int64_t len) {
    const int64_t n = len > 0 ? len : 1;
    const int64_t ntiles = (n + TS_TILE - 1) / TS_TILE;
    const int64_t hist_n = TS_RADIX * ntiles;
    const int64_t scan_n = hist_n > n ? hist_n : n;
    const int64_t scan_tiles = (scan_n + 2047) / 2048 + 1;
    size_t off = 0;
    char* b = static_cast<char*>(base);
    auto take = [&](size_t bytes) { char* p = b ? b + off : nullptr; off += align_up(bytes); return p; };
    TripletWs t;
    t.key0 = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * n));
    t.key1 = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * n));
    t.val0 = reinterpret_cast<double*>(take(sizeof(double) * n));
    t.val1 = reinterpret_cast<double*>(take(sizeof(double) * n));
    t.hist = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (hist_n + 1)));
    t.flag = reinterpret_cast<int*>(take(sizeof(int) * (scan_n + 1)));
    t.pos = reinterpret_cast<int64_t*>(take(sizeof(int64_t) * (scan_n + 1)));
    t.status = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * scan_tiles));
    t.ticket = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long)));
    t.ntiles = ntiles;
    t.scan_tiles = scan_tiles;
    if (w) *w = t;
    return off;
}

__global__ void k_trip_keys(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                            const double* __restrict__ vals, int64_t len, int64_t n_rows, int64_t n_cols,
                            uint64_t* __restrict__ key, double* __restrict__ val, fa_result* res) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = rows[i], c = cols[i];
        const bool rbad = r < 0 || r >= n_rows, cbad = c < 0 || c >= n_cols;
        if (rbad) atomic_min_i64(&res->index_error_pos, i);
        if (cbad) atomic_min_i64(&res->col_error_pos, i);
        key[i] = (rbad || cbad) ? 0 : uint64_t(c) * uint64_t(n_rows) + uint64_t(r);
        val[i] = vals[i];
    }
}

__global__ void __launch_bounds__(TS_BLOCK) k_trip_hist(const uint64_t* __restrict__ key, int64_t len, int shift,
                                                         int64_t ntiles, int64_t* __restrict__ hist) {
    __shared__ int s_h[TS_RADIX];
    s_h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * TS_TILE;
    for (int r = 0; r < TS_ROUNDS; ++r) {
        const int64_t i = base + r * TS_BLOCK + threadIdx.x;
        if (i < len) atomicAdd(&s_h[(key[i] >> shift) & 0xff], 1);
    }
    __syncthreads();
    hist[int64_t(threadIdx.x) * ntiles + blockIdx.x] = s_h[threadIdx.x];  // digit-major for the scan
}

// Exclusive scan of int64 values in place (n entries) with decoupled look-back.
__global__ void __launch_bounds__(256) k_scan_i64_inplace(int64_t* __restrict__ a, int64_t n, uint64_t* status,
                                                          unsigned long long* ticket) {
    __shared__ int64_t s_tile;
    __shared__ uint64_t s_prefix;
    __shared__ int64_t s_warp[8];
    __shared__ int64_t s_total;
    const int64_t tile = next_tile(ticket, &s_tile);
    const int64_t base = tile * 2048 + int64_t(threadIdx.x) * 8;
    int64_t x[8], local = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = base + i < n ? a[base + i] : 0;
        local += x[i];
    }
    const int64_t excl = block_exclusive_scan<256>(local, s_warp, &s_total);
    const uint64_t prefix = lookback_prefix(status, tile, uint64_t(s_total), &s_prefix);
    int64_t run = int64_t(prefix) + excl;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (base + i < n) a[base + i] = run;
        run += x[i];
    }
    if (base <= n - 1 && n - 1 < base + 8) a[n] = run;
}

// One stable counting-sort pass over a tile of TS_TILE (code, value) pairs: the tile's digit
// histogram and its exclusive scan, then rounds of TS_BLOCK pairs in input order ranked by
// digit (warp match for the rank among equal digits of a warp, per-warp counters ordered
// across warps), each pair staged at its tile-local sorted position; finally the staged tile
// goes out in digit order, every digit's run to its global offset (coalesced).
__global__ void __launch_bounds__(TS_BLOCK) k_trip_scatter(const uint64_t* __restrict__ kin, const double* __restrict__ vin,
                                                            uint64_t* __restrict__ kout, double* __restrict__ vout,
                                                            int64_t len, int shift, int64_t ntiles,
                                                            const int64_t* __restrict__ hist) {
    extern __shared__ __align__(16) unsigned char ts_dyn[];
    uint64_t* s_key = reinterpret_cast<uint64_t*>(ts_dyn);      // [TS_TILE]
    double* s_val = reinterpret_cast<double*>(s_key + TS_TILE);  // [TS_TILE]
    __shared__ int64_t s_gbase[TS_RADIX];  // global start of the tile's run of each digit
    __shared__ int s_start[TS_RADIX];      // tile-local start of each digit
    __shared__ int s_run[TS_RADIX];        // pairs of each digit staged so far
    __shared__ int s_w[TS_BLOCK / 32][TS_RADIX];
    __shared__ int s_warp[TS_BLOCK / 32];
    __shared__ int s_total;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t base = int64_t(blockIdx.x) * TS_TILE;
    const int tn = int(len - base < TS_TILE ? len - base : TS_TILE);
    s_gbase[tid] = hist[int64_t(tid) * ntiles + blockIdx.x];
    s_run[tid] = 0;
    s_start[tid] = 0;
    __syncthreads();
    uint64_t k[TS_ROUNDS];
    double v[TS_ROUNDS];
#pragma unroll
    for (int r = 0; r < TS_ROUNDS; ++r) {
        const int i = r * TS_BLOCK + tid;
        k[r] = i < tn ? kin[base + i] : 0;
        v[r] = i < tn ? vin[base + i] : 0.0;
        if (i < tn) atomicAdd(&s_start[int((k[r] >> shift) & 0xff)], 1);
    }
    __syncthreads();
    {  // tile-local digit starts
        const int c = s_start[tid];
        const int ex = block_exclusive_scan<TS_BLOCK>(c, s_warp, &s_total);
        __syncthreads();
        s_start[tid] = ex;
    }
    const unsigned lt = (1u << lane) - 1u;
    for (int r = 0; r < TS_ROUNDS; ++r) {
#pragma unroll
        for (int w = 0; w < TS_BLOCK / 32; ++w) s_w[w][tid] = 0;
        __syncthreads();
        const bool valid = r * TS_BLOCK + tid < tn;
        const int d = valid ? int((k[r] >> shift) & 0xff) : 0;
        const unsigned peers = __match_any_sync(0xffffffffu, valid ? d : TS_RADIX + lane);
        const int rank = __popc(peers & lt);
        if (valid && rank == 0) s_w[warp][d] = __popc(peers);
        __syncthreads();
        {  // thread `tid` owns digit tid: ordered offsets of the warps' groups in this round
            int run = s_run[tid];
#pragma unroll
            for (int w = 0; w < TS_BLOCK / 32; ++w) {
                const int c = s_w[w][tid];
                s_w[w][tid] = run;
                run += c;
            }
            s_run[tid] = run;
        }
        __syncthreads();
        if (valid) {
            const int lp = s_start[d] + s_w[warp][d] + rank;
            s_key[lp] = k[r];
            s_val[lp] = v[r];
        }
        __syncthreads();  // s_w is read above before the next round clears it
    }
    for (int p = tid; p < tn; p += TS_BLOCK) {
        const uint64_t key = s_key[p];
        const int d = int((key >> shift) & 0xff);
        const int64_t dest = s_gbase[d] + (p - s_start[d]);
        kout[dest] = key;
        vout[dest] = s_val[p];
    }
}

__global__ void k_trip_heads(const uint64_t* __restrict__ key, int64_t len, int* __restrict__ head) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x)
        head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// One thread per run of equal keys: left-to-right sum in input order (the stable sort kept
// ties in input order), then flag the position when the sum is nonzero.
// keep_zeros (CscBuilder semantics, sparse.py:208-290): the sum starts from the run's first
// value (`aa[pos] += v` after the first insertion stores v) and every position is stored.
__global__ void k_trip_sums(const uint64_t* __restrict__ key, const double* __restrict__ vals, int64_t len,
                            int* __restrict__ keep,
                            double* __restrict__ sums, fa_result* res, int keep_zeros) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x) {
        const bool head = i == 0 || key[i] != key[i - 1];
        if (!head) { keep[i] = 0; continue; }
        double s = keep_zeros ? vals[i] : 0.0;
        int64_t j = keep_zeros ? i + 1 : i;
        while (j < len && key[j] == key[i]) {
            s = __dadd_rn(s, vals[j]);
            ++j;
        }
        sums[i] = s;
        keep[i] = (s != 0.0 || keep_zeros) ? 1 : 0;
        if (keep_zeros) continue;
        if (s == 0.0) {
            // count only positions with at least one nonzero input (the reference never sees
            // all-zero positions); diagnostic only
            bool any = false;
            for (int64_t t = i; t < j; ++t) any |= vals[t] != 0.0;
            if (any) atomicAdd(reinterpret_cast<unsigned long long*>(&res->dropped), 1ull);
        }
    }
}

__global__ void k_trip_emit(const uint64_t* __restrict__ key, const double* __restrict__ sums,
                            const int* __restrict__ keep, const int64_t* __restrict__ pos, int64_t len,
                            int64_t n_rows, int64_t* __restrict__ rowidx, double* __restrict__ vout,
                            int64_t* __restrict__ colbuf) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x) {
        if (!keep[i]) continue;
        const int64_t p = pos[i];
        rowidx[p] = int64_t(key[i] % uint64_t(n_rows));
        vout[p] = sums[i];
        colbuf[p] = int64_t(key[i] / uint64_t(n_rows));
    }
}

// col_ptr[j] = number of stored entries with column < j (binary search in sorted columns).
__global__ void k_trip_colptr(const int64_t* __restrict__ colbuf, const int64_t* __restrict__ nnz_ptr, int64_t n_cols,
                              int64_t* __restrict__ colptr) {
    const int64_t nnz = *nnz_ptr;
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j <= n_cols; j += int64_t(gridDim.x) * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (colbuf[mid] < j) lo = mid + 1; else hi = mid;
        }
        colptr[j] = lo;
    }
}

__global__ void k_trip_finish(const int64_t* __restrict__ pos, int64_t len, fa_result* res) {
    if (threadIdx.x == 0 && blockIdx.x == 0) res->nnz = pos[len];
}

}  // namespace fa

using namespace fa;

extern "C" size_t fa_triplets_workspace(int64_t len, int64_t n_rows, int64_t n_cols) {
    (void)n_rows;
    (void)n_cols;
    return carve(nullptr, nullptr, len) + 256;
}

static int scan_i32_flags(const int* flag, int64_t* pos, int64_t n, TripletWs& w, cudaStream_t st);

extern "C" int fa_triplets_to_csc_ex(const int64_t* d_rows, const int64_t* d_cols, const double* d_vals, int64_t len,
                                     int64_t n_rows, int64_t n_cols, int flags, int64_t* d_colptr, int64_t* d_rowidx,
                                     double* d_vals_out, void* d_ws, size_t ws_bytes, fa_result* d_res, void* stream);

extern "C" int fa_triplets_to_csc(const int64_t* d_rows, const int64_t* d_cols, const double* d_vals, int64_t len,
                                  int64_t n_rows, int64_t n_cols, int64_t* d_colptr, int64_t* d_rowidx,
                                  double* d_vals_out, void* d_ws, size_t ws_bytes, fa_result* d_res, void* stream) {
    return fa_triplets_to_csc_ex(d_rows, d_cols, d_vals, len, n_rows, n_cols, 0, d_colptr, d_rowidx, d_vals_out, d_ws,
                                 ws_bytes, d_res, stream);
}

extern "C" int fa_triplets_to_csc_ex(const int64_t* d_rows, const int64_t* d_cols, const double* d_vals, int64_t len,
                                     int64_t n_rows, int64_t n_cols, int flags, int64_t* d_colptr, int64_t* d_rowidx,
                                     double* d_vals_out, void* d_ws, size_t ws_bytes, fa_result* d_res, void* stream) {
    NvtxRange nv("fa_triplets_to_csc");
    if (len < 0 || n_rows < 1 || n_cols < 1) { set_error("matrix dimensions must be positive"); return FA_ERR_ARGUMENT; }
    if (!d_colptr || !d_res || !d_ws || (len > 0 && (!d_rows || !d_cols || !d_vals || !d_rowidx || !d_vals_out))) {
        set_error("fa_triplets_to_csc: NULL argument"); return FA_ERR_ARGUMENT;
    }
    if (ws_bytes < fa_triplets_workspace(len, n_rows, n_cols)) { set_error("fa_triplets_to_csc: workspace too small"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = as_stream(stream);
    TripletWs w;
    void* base = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(d_ws) + 255) & ~uintptr_t(255));
    carve(&w, base, len);
    k_result_reset<<<1, 32, 0, st>>>(d_res);
    if (len == 0) {
        FA_CUDA(cudaMemsetAsync(d_colptr, 0, sizeof(int64_t) * (n_cols + 1), st));
        return FA_OK;
    }
    const int tb = 256;
    k_trip_keys<<<grid_for(len, tb), tb, 0, st>>>(d_rows, d_cols, d_vals, len, n_rows, n_cols, w.key0, w.val0, d_res);
    FA_LAUNCH_CHECK("k_trip_keys");
    // bits needed for codes in [0, n_rows*n_cols)
    const unsigned __int128 span = (unsigned __int128)n_rows * (unsigned __int128)n_cols;
    int bits = 0;
    while (bits < 64 && ((unsigned __int128)1 << bits) < span) ++bits;
    uint64_t *kin = w.key0, *kout = w.key1;
    double *vin = w.val0, *vout = w.val1;
    FA_CUDA(cudaFuncSetAttribute(k_trip_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(TS_STAGE_BYTES)));
    for (int shift = 0; shift < bits; shift += 8) {
        k_trip_hist<<<dim3(unsigned(w.ntiles)), TS_BLOCK, 0, st>>>(kin, len, shift, w.ntiles, w.hist);
        FA_LAUNCH_CHECK("k_trip_hist");
        const int64_t hn = TS_RADIX * w.ntiles;
        const int64_t stiles = (hn + 2047) / 2048;
        FA_CUDA(cudaMemsetAsync(w.status, 0, sizeof(uint64_t) * stiles, st));
        FA_CUDA(cudaMemsetAsync(w.ticket, 0, sizeof(unsigned long long), st));
        k_scan_i64_inplace<<<dim3(unsigned(stiles)), 256, 0, st>>>(w.hist, hn, w.status, w.ticket);
        FA_LAUNCH_CHECK("k_scan_i64_inplace");
        k_trip_scatter<<<dim3(unsigned(w.ntiles)), TS_BLOCK, TS_STAGE_BYTES, st>>>(kin, vin, kout, vout, len, shift,
                                                                                   w.ntiles, w.hist);
        FA_LAUNCH_CHECK("k_trip_scatter");
        uint64_t* tk = kin; kin = kout; kout = tk;
        double* tv = vin; vin = vout; vout = tv;
    }
    // sums per run (the values travelled with their codes); kout is free f64 storage
    double* sums = reinterpret_cast<double*>(kout);
    k_trip_sums<<<grid_for(len, tb), tb, 0, st>>>(kin, vin, len, w.flag, sums, d_res,
                                                   (flags & FA_TRIPLETS_KEEP_ZEROS) ? 1 : 0);
    FA_LAUNCH_CHECK("k_trip_sums");
    int rc = scan_i32_flags(w.flag, w.pos, len, w, st);
    if (rc != FA_OK) return rc;
    int64_t* colbuf = reinterpret_cast<int64_t*>(vout);
    k_trip_emit<<<grid_for(len, tb), tb, 0, st>>>(kin, sums, w.flag, w.pos, len, n_rows, d_rowidx, d_vals_out, colbuf);
    FA_LAUNCH_CHECK("k_trip_emit");
    k_trip_colptr<<<grid_for(n_cols + 1, tb), tb, 0, st>>>(colbuf, w.pos + len, n_cols, d_colptr);
    FA_LAUNCH_CHECK("k_trip_colptr");
    k_trip_finish<<<1, 32, 0, st>>>(w.pos, len, d_res);
    FA_LAUNCH_CHECK("k_trip_finish");
    return FA_OK;
}

// int32 flags -> int64 exclusive offsets (n+1 entries) via the in-place int64 scan
__global__ void k_widen(const int* __restrict__ f, int64_t* __restrict__ o, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) o[i] = f[i];
}

static int scan_i32_flags(const int* flag, int64_t* pos, int64_t n, TripletWs& w, cudaStream_t st) {
    const int tb = 256;
    k_widen<<<grid_for(n, tb), tb, 0, st>>>(flag, pos, n);
    FA_LAUNCH_CHECK("k_widen");
    const int64_t stiles = (n + 2047) / 2048;
    FA_CUDA(cudaMemsetAsync(w.status, 0, sizeof(uint64_t) * stiles, st));
    FA_CUDA(cudaMemsetAsync(w.ticket, 0, sizeof(unsigned long long), st));
    k_scan_i64_inplace<<<dim3(unsigned(stiles)), 256, 0, st>>>(pos, n, w.status, w.ticket);
    FA_LAUNCH_CHECK("k_scan_i64_inplace");
    return FA_OK;
}
