/*
 * femasm_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the reference OptV2
 * path (femasm, /root/reference/pkg/src/femasm) used to check the GPU library at the
 * BASELINE sizes, where the numpy oracle needs tens of GB and minutes.  Never linked into
 * or called by the product package.
 *
 * What it restates
 *   element values  assembly.py:214-307 (same operation order; build with
 *                   -ffp-contract=off so no FMA changes a bit; SSE2 doubles are IEEE)
 *   sparse()        sparse.py:140-189: input zeros skipped, entries of one position summed
 *                   left to right in input (= ascending triangle) order starting at 0.0,
 *                   exact-zero sums dropped, CSC output.
 * How: instead of sorting 9*nme keys, a counting sort by column (filled in ascending
 * triangle order, hence stable) followed by a stable insertion sort of each column's few
 * entries by row — the same order the reference's stable argsort produces.
 * Columns [col_begin, col_end) only: the row-block subset oracle of SURVEY.md §8(c).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define AREA_EPS 1e-300

enum { K_MASS = 0, K_MASSW = 1, K_STIFF = 2, K_ELASTIC = 3 };

/* mesh.py:62-65 */
static double area_of(const double* q, const int64_t* t) {
    const double x1 = q[2 * t[0]], y1 = q[2 * t[0] + 1];
    const double x2 = q[2 * t[1]], y2 = q[2 * t[1] + 1];
    const double x3 = q[2 * t[2]], y3 = q[2 * t[2] + 1];
    const double cross = (x2 - x1) * (y3 - y1) - (x3 - x1) * (y2 - y1);
    return 0.5 * fabs(cross);
}

void fo_areas(int64_t nme, const double* q, const int64_t* me, double* out) {
    for (int64_t k = 0; k < nme; ++k) out[k] = area_of(q, me + 3 * k);
}

/* Full element matrix E (rd x rd, E[a*rd + b] = entry (a, b)) of triangle k. */
static void element(int kind, const double* q, const int64_t* t, double area, const double* w, double lam,
                    double mu, double* E) {
    if (kind == K_MASS) { /* assembly.py:219-224 */
        const double d = area / 6.0, o = area / 12.0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) E[a * 3 + b] = a == b ? d : o;
        return;
    }
    if (kind == K_MASSW) { /* assembly.py:232-242 */
        const double W1 = w[t[0]] * area / 30.0, W2 = w[t[1]] * area / 30.0, W3 = w[t[2]] * area / 30.0;
        double low[3][3];
        low[0][0] = 3.0 * W1 + W2 + W3;
        low[1][0] = W1 + W2 + W3 / 2.0;
        low[2][0] = W1 + W2 / 2.0 + W3;
        low[1][1] = W1 + 3.0 * W2 + W3;
        low[2][1] = W1 / 2.0 + W2 + W3;
        low[2][2] = W1 + W2 + 3.0 * W3;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) E[a * 3 + b] = a >= b ? low[a][b] : low[b][a];
        return;
    }
    /* edges u = q2 - q3, v = q3 - q1, w = q1 - q2 (assembly.py:251-254) */
    double p[3][2], e[3][2];
    for (int c = 0; c < 3; ++c) { p[c][0] = q[2 * t[c]]; p[c][1] = q[2 * t[c] + 1]; }
    for (int d = 0; d < 2; ++d) {
        e[0][d] = p[1][d] - p[2][d];
        e[1][d] = p[2][d] - p[0][d];
        e[2][d] = p[0][d] - p[1][d];
    }
    if (kind == K_STIFF) { /* assembly.py:256-263 */
        const double a4 = 4.0 * area;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b <= a; ++b) {
                /* numpy's (x*y).sum(axis=1) starts from the additive identity: 0.0 + p0 + p1 */
                const double v = (0.0 + e[a][0] * e[b][0] + e[a][1] * e[b][1]) / a4;
                E[a * 3 + b] = v;
                E[b * 3 + a] = v;
            }
        return;
    }
    /* elastic: gradients assembly.py:203-210, rows :283-306 */
    const double inv2a = 0.5 / area;
    double g[3][2];
    for (int c = 0; c < 3; ++c) { g[c][0] = e[c][1] * inv2a; g[c][1] = (-e[c][0]) * inv2a; }
    const double L = lam, M = mu, P = lam + 2.0 * mu;
    for (int j = 0; j < 6; ++j)
        for (int i = j; i < 6; ++i) {
            const int A = i / 2, s = i % 2, B = j / 2, tt = j % 2;
            const double *gA = g[A], *gB = g[B];
            double v;
            if (s == 0 && tt == 0) v = (P * gB[0] * gA[0] + M * gB[1] * gA[1]) * area;
            else if (s == 1 && tt == 1) v = (P * gB[1] * gA[1] + M * gB[0] * gA[0]) * area;
            else if (s == 1 && A == B) v = (L * gB[0] * gA[1] + M * gB[0] * gA[1]) * area;
            else if (s == 1) v = (L * gB[0] * gA[1] + M * gB[1] * gA[0]) * area;
            else v = (L * gB[1] * gA[0] + M * gB[0] * gA[1]) * area;
            E[i * 6 + j] = v;
            E[j * 6 + i] = v;
        }
}

void fo_element_values(int kind, int64_t nme, const double* q, const int64_t* me, const double* areas,
                       const double* w, double lam, double mu, double* kg /* r x nme */) {
    const int rd = kind == K_ELASTIC ? 6 : 3, r = rd * rd;
    double E[36];
    for (int64_t k = 0; k < nme; ++k) {
        element(kind, q, me + 3 * k, areas[k], w, lam, mu, E);
        for (int il = 0; il < r; ++il) kg[il * nme + k] = E[(il % rd) * rd + il / rd];
    }
}

typedef struct { int64_t row; double val; } entry_t;

static int64_t dof(int kind, const int64_t* t, int local) {
    return kind == K_ELASTIC ? 2 * t[local / 2] + (local & 1) : t[local];
}

/* Returns nnz (>= 0), or -1 on allocation failure, -(2 + k) for the first degenerate k,
 * -3 - cap if capacity is too small is not possible: call with cap = fo_capacity first. */
int64_t fo_capacity(int kind, int64_t nme, const int64_t* me, int64_t col_begin, int64_t col_end) {
    const int rd = kind == K_ELASTIC ? 6 : 3;
    int64_t n = 0;
    for (int64_t k = 0; k < nme; ++k)
        for (int b = 0; b < rd; ++b) {
            const int64_t c = dof(kind, me + 3 * k, b);
            if (c >= col_begin && c < col_end) n += rd;
        }
    return n;
}

int64_t fo_assemble(int kind, int64_t nme, const double* q, const int64_t* me, const double* areas,
                    const double* w, double lam, double mu, int64_t col_begin, int64_t col_end,
                    int64_t* colptr, int64_t* rowidx, double* vals, int64_t* first_degenerate) {
    const int rd = kind == K_ELASTIC ? 6 : 3;
    const int64_t ncols = col_end - col_begin;
    *first_degenerate = -1;
    if (kind != K_MASSW)
        for (int64_t k = 0; k < nme; ++k)
            if (areas[k] <= AREA_EPS) { *first_degenerate = k; return 0; }
    int64_t* start = (int64_t*)calloc((size_t)ncols + 1, sizeof(int64_t));
    if (!start) return -1;
    for (int64_t k = 0; k < nme; ++k)
        for (int b = 0; b < rd; ++b) {
            const int64_t c = dof(kind, me + 3 * k, b);
            if (c >= col_begin && c < col_end) start[c - col_begin + 1] += rd;
        }
    for (int64_t c = 0; c < ncols; ++c) start[c + 1] += start[c];
    const int64_t total = start[ncols];
    entry_t* ent = (entry_t*)malloc(sizeof(entry_t) * (size_t)(total > 0 ? total : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncols > 0 ? ncols : 1));
    if (!ent || !fill) { free(start); free(ent); free(fill); return -1; }
    memcpy(fill, start, sizeof(int64_t) * (size_t)ncols);
    double E[36];
    for (int64_t k = 0; k < nme; ++k) { /* ascending triangle order */
        const int64_t* t = me + 3 * k;
        int touched = 0;
        for (int b = 0; b < rd; ++b) {
            const int64_t c = dof(kind, t, b);
            if (c >= col_begin && c < col_end) touched = 1;
        }
        if (!touched) continue;
        element(kind, q, t, areas[k], w, lam, mu, E);
        for (int b = 0; b < rd; ++b) { /* slot il = a + rd*b: column b, rows a */
            const int64_t c = dof(kind, t, b);
            if (c < col_begin || c >= col_end) continue;
            for (int a = 0; a < rd; ++a) {
                entry_t* e = &ent[fill[c - col_begin]++];
                e->row = dof(kind, t, a);
                e->val = E[a * rd + b];
            }
        }
    }
    int64_t nnz = 0;
    colptr[0] = 0;
    for (int64_t c = 0; c < ncols; ++c) {
        entry_t* seg = ent + start[c];
        const int64_t m = start[c + 1] - start[c];
        for (int64_t i = 1; i < m; ++i) { /* stable insertion sort by row */
            entry_t x = seg[i];
            int64_t j = i - 1;
            while (j >= 0 && seg[j].row > x.row) { seg[j + 1] = seg[j]; --j; }
            seg[j + 1] = x;
        }
        for (int64_t i = 0; i < m;) {
            int64_t j = i;
            double s = 0.0;
            int any = 0;
            while (j < m && seg[j].row == seg[i].row) {
                if (seg[j].val != 0.0) { s += seg[j].val; any = 1; }
                ++j;
            }
            if (any && s != 0.0) {
                rowidx[nnz] = seg[i].row;
                vals[nnz] = s;
                ++nnz;
            }
            i = j;
        }
        colptr[c + 1] = nnz;
    }
    free(start); free(ent); free(fill);
    return nnz;
}
