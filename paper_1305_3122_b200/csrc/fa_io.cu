// Host-side CSC -> coordinate MatrixMarket writer.
//
// Replaces femasm's write_matrix_market (pkg/src/femasm/sparse.py:332-339), a per-entry Python
// loop, with the byte-identical output: header "%%MatrixMarket matrix coordinate real
// general", "n_rows n_cols nnz", then one "i j v" line per stored entry in CSC order (column by
// column, rows ascending), 1-based indices, values as C printf "%.17g" (== Python '%.17g' %
// v: both correctly rounded, two-digit minimum exponent, "inf"/"nan"/"-0").  Entries are
// formatted in parallel in bounded chunks and written in order.
#include <cinttypes>
#include <cstdlib>
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

// ------------------------------------------------------------------------------------------
// Mesh text reader (femasm read_mesh, pkg/src/femasm/mesh.py:225-286), multithreaded.
//
// Fast path for the well-formed files write_mesh produces: ASCII, lines ending in "\n" or
// "\r\n", fields separated by blanks/tabs, header "nq nme" (unsigned decimal), nq lines of two
// decimal coordinates, nme lines of three unsigned decimal 1-based vertex ids in 1..nq, then
// only blank lines.  Coordinates are parsed with strtod after a decimal-grammar check (both
// strtod and Python's float() round correctly, so the values are identical).  Anything else -
// a malformed line, a sign, an underscore, inf/nan, a hex literal, another line terminator -
// returns FA_ERR_ARGUMENT without a message and the caller runs the reference-equivalent parser,
// which accepts what Python accepts and raises the reference's MeshFormatError (line number
// and text) for the rest.  Call with vertices == connectivity == NULL to read the header.
// ------------------------------------------------------------------------------------------
namespace {

struct LineSpan {
    const char* b;
    const char* e;
};

inline bool is_blank(char c) { return c == ' ' || c == '\t'; }

// next field in [p, e): skips blanks; returns false at the end of the line
inline bool next_field(const char*& p, const char* e, const char*& fb, const char*& fe) {
    while (p < e && is_blank(*p)) ++p;
    if (p >= e) return false;
    fb = p;
    while (p < e && !is_blank(*p)) ++p;
    fe = p;
    return true;
}

inline bool parse_uint(const char* b, const char* e, int64_t& out) {
    if (b >= e || e - b > 18) return false;
    int64_t v = 0;
    for (const char* p = b; p < e; ++p) {
        if (*p < '0' || *p > '9') return false;
        v = v * 10 + (*p - '0');
    }
    out = v;
    return true;
}

// [+-]? (digits [. digits?] | . digits) ([eE] [+-]? digits)?
inline bool parse_decimal(const char* b, const char* e, double& out) {
    const char* p = b;
    if (p < e && (*p == '+' || *p == '-')) ++p;
    int digits = 0;
    while (p < e && *p >= '0' && *p <= '9') { ++p; ++digits; }
    if (p < e && *p == '.') {
        ++p;
        while (p < e && *p >= '0' && *p <= '9') { ++p; ++digits; }
    }
    if (digits == 0) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        ++p;
        if (p < e && (*p == '+' || *p == '-')) ++p;
        int ed = 0;
        while (p < e && *p >= '0' && *p <= '9') { ++p; ++ed; }
        if (ed == 0) return false;
    }
    if (p != e || e - b > 400) return false;
    char buf[408];
    memcpy(buf, b, size_t(e - b));
    buf[e - b] = '\0';
    out = strtod(buf, nullptr);
    return true;
}

}  // namespace

extern "C" int fa_read_mesh_text(const char* path, int64_t* nq_out, int64_t* nme_out, double* vertices,
                                 int64_t* connectivity, int threads) {
    using namespace fa;
    if (!path || !nq_out || !nme_out) { set_error("fa_read_mesh_text: bad arguments"); return FA_ERR_ARGUMENT; }
    FILE* f = fopen(path, "rb");
    if (!f) return FA_ERR_ARGUMENT;  // the reference parser reports it (OSError)
    std::string data;
    {
        char chunk[1 << 16];
        size_t n;
        while ((n = fread(chunk, 1, sizeof(chunk), f)) > 0) data.append(chunk, n);
        fclose(f);
    }
    const char* s = data.data();
    const char* end = s + data.size();
    // lines: "\n" or "\r\n" terminated; any other control byte or non-ASCII -> fallback
    std::vector<LineSpan> lines;
    lines.reserve(data.size() / 16 + 2);
    const char* lb = s;
    for (const char* p = s; p < end; ++p) {
        const unsigned char c = static_cast<unsigned char>(*p);
        if (c == '\n') {
            const char* le = (p > lb && p[-1] == '\r') ? p - 1 : p;
            lines.push_back({lb, le});
            lb = p + 1;
        } else if (c >= 0x80 || (c < 0x20 && c != '\t' && c != '\r')) {
            return FA_ERR_ARGUMENT;
        } else if (c == '\r' && !(p + 1 < end && p[1] == '\n')) {
            return FA_ERR_ARGUMENT;
        }
    }
    if (lb < end) lines.push_back({lb, end});
    if (lines.empty()) return FA_ERR_ARGUMENT;
    int64_t nq = 0, nme = 0;
    {
        const char* p = lines[0].b;
        const char *fb, *fe;
        if (!next_field(p, lines[0].e, fb, fe) || !parse_uint(fb, fe, nq)) return FA_ERR_ARGUMENT;
        if (!next_field(p, lines[0].e, fb, fe) || !parse_uint(fb, fe, nme)) return FA_ERR_ARGUMENT;
        if (next_field(p, lines[0].e, fb, fe)) return FA_ERR_ARGUMENT;
    }
    if (nq < 1 || nme < 1 || int64_t(lines.size()) < 1 + nq + nme) return FA_ERR_ARGUMENT;
    *nq_out = nq;
    *nme_out = nme;
    if (!vertices && !connectivity) return FA_OK;
    if (!vertices || !connectivity) { set_error("fa_read_mesh_text: bad arguments"); return FA_ERR_ARGUMENT; }
    for (size_t i = size_t(1 + nq + nme); i < lines.size(); ++i) {  // trailing lines: blank only
        const char* p = lines[i].b;
        const char *fb, *fe;
        if (next_field(p, lines[i].e, fb, fe)) return FA_ERR_ARGUMENT;
    }
    if (threads <= 0) threads = int(std::thread::hardware_concurrency());
    if (threads <= 0) threads = 1;
    const int64_t total = nq + nme;
    std::vector<int> ok(size_t(threads), 1);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        const int64_t a = total * t / threads, b = total * (t + 1) / threads;
        pool.emplace_back([=, &lines, &ok] {
            for (int64_t i = a; i < b; ++i) {
                const LineSpan& L = lines[size_t(1 + i)];
                const char* p = L.b;
                const char *fb, *fe;
                if (i < nq) {
                    double x, y;
                    if (!next_field(p, L.e, fb, fe) || !parse_decimal(fb, fe, x) || !next_field(p, L.e, fb, fe) ||
                        !parse_decimal(fb, fe, y) || next_field(p, L.e, fb, fe)) {
                        ok[size_t(t)] = 0;
                        return;
                    }
                    vertices[2 * i] = x;
                    vertices[2 * i + 1] = y;
                } else {
                    const int64_t k = i - nq;
                    for (int c = 0; c < 3; ++c) {
                        int64_t id;
                        if (!next_field(p, L.e, fb, fe) || !parse_uint(fb, fe, id) || id < 1 || id > nq) {
                            ok[size_t(t)] = 0;
                            return;
                        }
                        connectivity[3 * k + c] = id - 1;
                    }
                    if (next_field(p, L.e, fb, fe)) {
                        ok[size_t(t)] = 0;
                        return;
                    }
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    for (int t = 0; t < threads; ++t)
        if (!ok[size_t(t)]) return FA_ERR_ARGUMENT;
    return FA_OK;
}
