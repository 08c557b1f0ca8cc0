// Bit-exact P1 element values of the reference OptV2 batch kernels.
//
// numpy evaluates every expression left to right and rounds after each operation; the
// functions below repeat the reference's operation order with explicit round-to-nearest
// intrinsics (__dmul_rn/__dadd_rn/__dsub_rn and the correctly rounded fa::ddiv), so no FMA
// contraction can change a bit whatever the compiler flags, and divisions stay true
// divisions (never a reciprocal multiply).  Sources:
//   areas     mesh.py:62-65          0.5*|(x2-x1)(y3-y1) - (x3-x1)(y2-y1)|
//   mass      assembly.py:219-224    diag area/6.0, off-diagonal area/12.0
//   massw     assembly.py:232-242    W_b = (tw_b*area)/30.0 and the six row formulas
//   stiff     assembly.py:251-263    dot(e_a, e_b)/(4.0*area), edges u=q2-q3, v=q3-q1, w=q1-q2
//   gradients assembly.py:203-210    g_b = (e_b.y*inv2a, (-e_b.x)*inv2a), inv2a = 0.5/area
//   elastic   assembly.py:278-306    21 lower-triangle rows, upper = copies
// Entry (a, b) of an element matrix with a < b is the stored copy of (b, a) (the reference
// computes the lower triangle and copies it, assembly.py:242, :263, :304-306).
#pragma once

#include <cuda_runtime.h>

#include "fa_common.cuh"
#include "fa_div.cuh"

namespace fa {

#define FMUL __dmul_rn
#define FADD __dadd_rn
#define FSUB __dsub_rn
#define FDIV ::fa::ddiv  // call-free correctly rounded division (fa_div.cuh)

template <typename T>
__device__ __forceinline__ T sel3(int i, T x0, T x1, T x2) {
    return i == 0 ? x0 : (i == 1 ? x1 : x2);
}

// compute_areas (mesh.py:62-65) with corners in triangle order.
__device__ __forceinline__ double tri_area(double2 p1, double2 p2, double2 p3) {
    double cross = FSUB(FMUL(FSUB(p2.x, p1.x), FSUB(p3.y, p1.y)), FMUL(FSUB(p3.x, p1.x), FSUB(p2.y, p1.y)));
    return FMUL(0.5, fabs(cross));
}

__device__ __forceinline__ double2 dsub2(double2 a, double2 b) { return make_double2(FSUB(a.x, b.x), FSUB(a.y, b.y)); }

// compute_areas from the local edges of the corner at position a (eo = n1 - n2, e1 = n2 - own,
// e2 = own - n1): the corner differences of the triangle-order formula are +-(e2, e1) (a = 0),
// (e1, eo) (a = 1), (eo, e2) (a = 2); RN(-x) = -RN(x) makes the cross product the exact negation
// of tri_area's and fabs removes the sign, so the result is bitwise tri_area(c0, c1, c2).
__device__ __forceinline__ double tri_area_edges(int a, double2 eo, double2 e1, double2 e2) {
    const double2 u = sel3(a, e2, e1, eo), v = sel3(a, e1, eo, e2);
    return FMUL(0.5, fabs(FSUB(FMUL(u.x, v.y), FMUL(v.x, u.y))));
}

// ---- per-kind prepared triangle data ---------------------------------------------------

struct MassTri {
    double d, o;  // area/6.0, area/12.0
};
// RN(1/6), RN(1/12), RN(1/30) for the constant-divisor division (exact check in ddiv_rcp)
#define FA_RCP6 0.16666666666666666
#define FA_RCP12 0.083333333333333329
#define FA_RCP30 0.033333333333333333
__device__ __forceinline__ MassTri mass_prepare(double area) {
    return {ddiv_rcp(area, 6.0, FA_RCP6), ddiv_rcp(area, 12.0, FA_RCP12)};
}
__device__ __forceinline__ double mass_entry(const MassTri& t, int a, int b) { return a == b ? t.d : t.o; }

struct MasswTri {
    double e00, e10, e20, e11, e21, e22;  // lower-triangle entries (row il = a + 3b)
};
__device__ __forceinline__ MasswTri massw_prepare(double area, double tw0, double tw1, double tw2) {
    const double W1 = ddiv_rcp(FMUL(tw0, area), 30.0, FA_RCP30);
    const double W2 = ddiv_rcp(FMUL(tw1, area), 30.0, FA_RCP30);
    const double W3 = ddiv_rcp(FMUL(tw2, area), 30.0, FA_RCP30);
    MasswTri t;
    t.e00 = FADD(FADD(FMUL(3.0, W1), W2), W3);     // kg[0] = 3*w1 + w2 + w3
    // x / 2.0 == x * 0.5 exactly (division by a power of two is an exact rescale in both)
    t.e10 = FADD(FADD(W1, W2), FMUL(W3, 0.5));     // kg[1] = w1 + w2 + w3/2
    t.e20 = FADD(FADD(W1, FMUL(W2, 0.5)), W3);     // kg[2] = w1 + w2/2 + w3
    t.e11 = FADD(FADD(W1, FMUL(3.0, W2)), W3);     // kg[4] = w1 + 3*w2 + w3
    t.e21 = FADD(FADD(FMUL(W1, 0.5), W2), W3);     // kg[5] = w1/2 + w2 + w3
    t.e22 = FADD(FADD(W1, W2), FMUL(3.0, W3));     // kg[8] = w1 + w2 + 3*w3
    return t;
}
// the six formulas of assembly.py:236-241 from W1..W3
__device__ __forceinline__ void massw_from_w(double W1, double W2, double W3, MasswTri& t) {
    t.e00 = FADD(FADD(FMUL(3.0, W1), W2), W3);
    t.e10 = FADD(FADD(W1, W2), FMUL(W3, 0.5));
    t.e20 = FADD(FADD(W1, FMUL(W2, 0.5)), W3);
    t.e11 = FADD(FADD(W1, FMUL(3.0, W2)), W3);
    t.e21 = FADD(FADD(FMUL(W1, 0.5), W2), W3);
    t.e22 = FADD(FADD(W1, W2), FMUL(3.0, W3));
}
__device__ __forceinline__ double massw_entry(const MasswTri& t, int a, int b) {
    const int hi = a > b ? a : b, lo = a > b ? b : a;
    // (hi, lo) in {(0,0),(1,0),(2,0),(1,1),(2,1),(2,2)}
    if (lo == 0) return sel3(hi, t.e00, t.e10, t.e20);
    if (lo == 1) return hi == 1 ? t.e11 : t.e21;
    return t.e22;
}

struct StiffTri {
    double2 e0, e1, e2;  // u = q2 - q3, v = q3 - q1, w = q1 - q2
    double a4;           // 4.0 * area
    DivBy d4;            // division by a4 (reciprocal shared by the entries)
};
__device__ __forceinline__ StiffTri stiff_prepare(double2 p1, double2 p2, double2 p3, double area) {
    const double a4 = FMUL(4.0, area);
    return {dsub2(p2, p3), dsub2(p3, p1), dsub2(p1, p2), a4, div_prepare(a4)};
}
__device__ __forceinline__ double stiff_entry(const StiffTri& t, int a, int b) {
    // kg row for (a, b) is (e_a * e_b).sum(axis=1) / a4.  numpy's sum over the length-2 axis
    // starts from the additive identity, ((0.0 + x*x') + y*y'), which only matters for the
    // sign of an exact zero.  IEEE products commute, so the stored lower entry equals the
    // same formula evaluated for (a, b).
    const double2 ea = sel3(a, t.e0, t.e1, t.e2);
    const double2 eb = sel3(b, t.e0, t.e1, t.e2);
    return div_by(t.d4, FADD(FADD(0.0, FMUL(ea.x, eb.x)), FMUL(ea.y, eb.y)));
}

struct ElasticTri {
    double2 g0, g1, g2;  // true basis gradients (g1, g2, g3 of the reference)
    double area;
};
__device__ __forceinline__ ElasticTri elastic_prepare(double2 p1, double2 p2, double2 p3, double area) {
    const double inv2a = FDIV(0.5, area);
    const double2 u = dsub2(p2, p3), v = dsub2(p3, p1), w = dsub2(p1, p2);
    ElasticTri t;
    t.g0 = make_double2(FMUL(u.y, inv2a), FMUL(-u.x, inv2a));
    t.g1 = make_double2(FMUL(v.y, inv2a), FMUL(-v.x, inv2a));
    t.g2 = make_double2(FMUL(w.y, inv2a), FMUL(-w.x, inv2a));
    t.area = area;
    return t;
}

// Lower-triangle entry (i, j), i >= j, of the 6x6 element matrix in the interleaved order
// (x1, y1, x2, y2, x3, y3).  With i = 2A+s, j = 2B+t (B <= A) every reference row
// (assembly.py:283-303) has the form ((c1*gB.p)*gA.q + (c2*gB.r)*gA.s) * area where the
// column vertex B's gradient always comes first:
//   s=0,t=0: (P*gBx)*gAx + (M*gBy)*gAy          s=1,t=1: (P*gBy)*gAy + (M*gBx)*gAx
//   s=1,t=0: (L*gBx)*gAy + (M*gBy)*gAx  (A>B)    (L*gBx)*gAy + (M*gBx)*gAy  (A==B)
//   s=0,t=1: (L*gBy)*gAx + (M*gBx)*gAy  (A>B only)
__device__ __forceinline__ double elastic_lower(const ElasticTri& T, int i, int j, double L, double M, double P) {
    const int A = i >> 1, s = i & 1, B = j >> 1, t = j & 1;
    const double2 gA = sel3(A, T.g0, T.g1, T.g2);
    const double2 gB = sel3(B, T.g0, T.g1, T.g2);
    double r;
    if (s == 0 && t == 0) {
        r = FADD(FMUL(FMUL(P, gB.x), gA.x), FMUL(FMUL(M, gB.y), gA.y));
    } else if (s == 1 && t == 1) {
        r = FADD(FMUL(FMUL(P, gB.y), gA.y), FMUL(FMUL(M, gB.x), gA.x));
    } else if (s == 1) {  // t == 0
        r = A == B ? FADD(FMUL(FMUL(L, gB.x), gA.y), FMUL(FMUL(M, gB.x), gA.y))
                   : FADD(FMUL(FMUL(L, gB.x), gA.y), FMUL(FMUL(M, gB.y), gA.x));
    } else {  // s == 0, t == 1, A > B
        r = FADD(FMUL(FMUL(L, gB.y), gA.x), FMUL(FMUL(M, gB.x), gA.y));
    }
    return FMUL(r, T.area);
}
__device__ __forceinline__ double elastic_entry(const ElasticTri& T, int i, int j, double L, double M, double P) {
    return i >= j ? elastic_lower(T, i, j, L, M, P) : elastic_lower(T, j, i, L, M, P);
}
// ---- per-element formulas of elements.py (the element-loop strategies and elem_*) --------
// These differ in rounding from the batch kernels above, so they are transcribed separately:
//   elem_mass            elements.py:34-39    d = area/6.0, o = area/12.0 (same as the batch)
//   elem_mass_weighted   elements.py:42-57    s = area/30.0; e_aa = s*((3wa + wb) + wc) ...
//   elem_stiff           elements.py:60-78    c = 1.0/(4.0*area); entry = c * (e_a @ e_b)
//   elem_stiff_elastic   elements.py:111-154  upper triangle computed, lower mirrored
// numpy's `x @ y` of two length-2 float64 vectors runs OpenBLAS ddot, whose kernel on this
// image evaluates fma(x1, y1, x0*y0) (checked on 20,000 random pairs against both plain
// orders: 0 mismatches, 25-33 % mismatches respectively).
__device__ __forceinline__ double dot2_blas(double2 x, double2 y) { return __fma_rn(x.y, y.y, FMUL(x.x, y.x)); }

// Element matrix entry (i, j) of the element-loop formulas, 3x3 (scalar kinds) or 6x6.
struct ElemLoopTri {
    double e[6][6];
};
template <int KIND>
__device__ __forceinline__ void elem_loop_matrix(double2 p1, double2 p2, double2 p3, double area, double w1, double w2,
                                                 double w3, double lam, double mu, ElemLoopTri& m) {
    if constexpr (KIND == FA_KIND_MASS) {
        const MassTri t = mass_prepare(area);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) m.e[a][b] = a == b ? t.d : t.o;
    } else if constexpr (KIND == FA_KIND_MASSW) {
        const double s = ddiv_rcp(area, 30.0, FA_RCP30);
        const double e11 = FMUL(s, FADD(FADD(FMUL(3.0, w1), w2), w3));
        const double e22 = FMUL(s, FADD(FADD(w1, FMUL(3.0, w2)), w3));
        const double e33 = FMUL(s, FADD(FADD(w1, w2), FMUL(3.0, w3)));
        const double e12 = FMUL(s, FADD(FADD(w1, w2), FMUL(w3, 0.5)));  // w3 / 2.0 (exact)
        const double e13 = FMUL(s, FADD(FADD(w1, FMUL(w2, 0.5)), w3));
        const double e23 = FMUL(s, FADD(FADD(FMUL(w1, 0.5), w2), w3));
        m.e[0][0] = e11; m.e[0][1] = e12; m.e[0][2] = e13;
        m.e[1][0] = e12; m.e[1][1] = e22; m.e[1][2] = e23;
        m.e[2][0] = e13; m.e[2][1] = e23; m.e[2][2] = e33;
    } else if constexpr (KIND == FA_KIND_STIFF) {
        const double2 u = dsub2(p2, p3), v = dsub2(p3, p1), w = dsub2(p1, p2);
        const double c = FDIV(1.0, FMUL(4.0, area));
        const double2 ed[3] = {u, v, w};
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = a; b < 3; ++b) {
                // uu, uv, uw, vv, vw, ww as computed (elements.py:71-76); the matrix is mirrored
                const double x = FMUL(c, dot2_blas(ed[a], ed[b]));
                m.e[a][b] = x;
                m.e[b][a] = x;
            }
    } else {
        const double inv2a = FDIV(0.5, area);
        const double2 u = dsub2(p2, p3), v = dsub2(p3, p1), w = dsub2(p1, p2);
        const double2 g[3] = {make_double2(FMUL(u.y, inv2a), FMUL(-u.x, inv2a)),
                              make_double2(FMUL(v.y, inv2a), FMUL(-v.x, inv2a)),
                              make_double2(FMUL(w.y, inv2a), FMUL(-w.x, inv2a))};
        const double lpm2 = FADD(lam, FMUL(2.0, mu));
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = a; b < 3; ++b) {
                const double2 ga = g[a], gb = g[b];
                const double xx = FMUL(FADD(FMUL(FMUL(lpm2, ga.x), gb.x), FMUL(FMUL(mu, ga.y), gb.y)), area);
                const double xy = FMUL(FADD(FMUL(FMUL(lam, ga.x), gb.y), FMUL(FMUL(mu, ga.y), gb.x)), area);
                const double yx = FMUL(FADD(FMUL(FMUL(lam, ga.y), gb.x), FMUL(FMUL(mu, ga.x), gb.y)), area);
                const double yy = FMUL(FADD(FMUL(FMUL(lpm2, ga.y), gb.y), FMUL(FMUL(mu, ga.x), gb.x)), area);
                m.e[2 * a][2 * b] = xx;
                m.e[2 * a][2 * b + 1] = xy;
                m.e[2 * a + 1][2 * b + 1] = yy;
                if (a < b) m.e[2 * a + 1][2 * b] = yx;  // (a == b: the lower entry is the mirror)
            }
#pragma unroll
        for (int i = 0; i < 6; ++i)  // ke[iu[1], iu[0]] = ke[iu]: strictly upper mirrored down
#pragma unroll
            for (int j = i + 1; j < 6; ++j) m.e[j][i] = m.e[i][j];
    }
}

}  // namespace fa
