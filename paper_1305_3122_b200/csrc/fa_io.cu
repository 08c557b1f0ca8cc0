// Host-side CSC -> coordinate MatrixMarket writer.
//
// Replaces femasm's write_matrix_market (pkg/src/femasm/sparse.py:332-339), a per-entry Python
// loop, with the byte-identical output: header "%%MatrixMarket matrix coordinate real
// general", "n_rows n_cols nnz", then one "i j v" line per stored entry in CSC order (column by
// column, rows ascending), 1-based indices, values as C printf "%.17g" (== Python '%.17g' %
// v: both correctly rounded, two-digit minimum exponent, "inf"/"nan"/"-0").  Entries are
// formatted in parallel in bounded chunks and written in order.
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fa_common.cuh"

namespace {

inline char* put_u64(char* p, uint64_t x) {
    char tmp[24];
    int n = 0;
    do {
        tmp[n++] = char('0' + x % 10);
        x /= 10;
    } while (x);
    while (n) *p++ = tmp[--n];
    return p;
}

// entries [e0, e1) of the CSC arrays, column of e0 given
void format_range(const int64_t* col_ptr, const int64_t* row_idx, const double* values, int64_t e0, int64_t e1,
                  int64_t col, std::string& out) {
    out.resize(size_t(e1 - e0) * 64);
    char* p = &out[0];
    for (int64_t e = e0; e < e1; ++e) {
        while (col_ptr[col + 1] <= e) ++col;
        p = put_u64(p, uint64_t(row_idx[e] + 1));
        *p++ = ' ';
        p = put_u64(p, uint64_t(col + 1));
        *p++ = ' ';
        p += snprintf(p, 40, "%.17g", values[e]);
        *p++ = '\n';
    }
    out.resize(size_t(p - &out[0]));
}

int64_t column_of(const int64_t* col_ptr, int64_t n_cols, int64_t e) {
    int64_t lo = 0, hi = n_cols;  // last column with col_ptr[c] <= e
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (col_ptr[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

}  // namespace

extern "C" int fa_write_matrix_market(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* col_ptr,
                                      const int64_t* row_idx, const double* values, int threads) {
    using namespace fa;
    if (!path || n_rows < 0 || n_cols < 0 || (n_cols > 0 && !col_ptr)) {
        set_error("fa_write_matrix_market: bad arguments");
        return FA_ERR_ARGUMENT;
    }
    const int64_t nnz = n_cols > 0 ? col_ptr[n_cols] : 0;
    if (nnz > 0 && (!row_idx || !values)) {
        set_error("fa_write_matrix_market: NULL entry arrays");
        return FA_ERR_ARGUMENT;
    }
    FILE* f = fopen(path, "wb");
    if (!f) {
        set_error("fa_write_matrix_market: cannot open %s", path);
        return FA_ERR_ARGUMENT;
    }
    fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%" PRId64 " %" PRId64 " %" PRId64 "\n", n_rows, n_cols,
            nnz);
    if (threads <= 0) threads = int(std::thread::hardware_concurrency());
    if (threads <= 0) threads = 1;
    const int64_t chunk = int64_t(1) << 22;  // entries formatted per round (bounded memory)
    std::vector<std::string> bufs(static_cast<size_t>(threads));
    bool ok = true;
    for (int64_t c0 = 0; c0 < nnz && ok; c0 += chunk) {
        const int64_t c1 = c0 + chunk < nnz ? c0 + chunk : nnz;
        const int64_t per = (c1 - c0 + threads - 1) / threads;
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            const int64_t e0 = c0 + t * per, e1 = e0 + per < c1 ? e0 + per : c1;
            if (e0 >= e1) {
                bufs[size_t(t)].clear();
                continue;
            }
            pool.emplace_back([=, &bufs] {
                format_range(col_ptr, row_idx, values, e0, e1, column_of(col_ptr, n_cols, e0), bufs[size_t(t)]);
            });
        }
        for (auto& th : pool) th.join();
        for (int t = 0; t < threads && ok; ++t)
            if (!bufs[size_t(t)].empty()) ok = fwrite(bufs[size_t(t)].data(), 1, bufs[size_t(t)].size(), f) == bufs[size_t(t)].size();
    }
    if (fclose(f) != 0) ok = false;
    if (!ok) {
        set_error("fa_write_matrix_market: write to %s failed", path);
        return FA_ERR_ARGUMENT;
    }
    return FA_OK;
}
