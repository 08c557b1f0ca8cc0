// Correctly rounded (IEEE round-to-nearest-even) fp64 division without a subroutine call.
//
// CUDA's __ddiv_rn / '/' expand to a fast path plus an out-of-line slow-path CALL; inside
// the row kernel's loops that call forces ABI register saves and local-memory spills.  This
// version is branch-light and call-free:
//   fast path (operands and quotient comfortably inside the normal range):
//     r = rcp.approx(y), two Newton steps, q = x*r, one residual correction, then an exact
//     check of the residual rem = fma(-q, y, x) against half an ulp of q times y (exact:
//     half an ulp is a power of two) that moves q to its neighbour when the neighbour is
//     nearer (ties to even).  q is within one ulp before the check, so one step suffices.
//   slow path (zeros, infinities, NaN, subnormals, extreme exponents): integer restoring
//     division of the 53-bit significands with guard/sticky bits and explicit rounding,
//     including subnormal results.
// Verified bitwise against __ddiv_rn by fa_selftest_division (tests/test_gpu_division.py).
#pragma once

#include <cstdint>

namespace fa {

__device__ __forceinline__ double ddiv_slow(double x, double y) {
    const uint64_t bx = __double_as_longlong(x), by = __double_as_longlong(y);
    const uint64_t sign = (bx ^ by) & 0x8000000000000000ull;
    int ex = int((bx >> 52) & 0x7ff), ey = int((by >> 52) & 0x7ff);
    uint64_t mx = bx & 0xfffffffffffffull, my = by & 0xfffffffffffffull;
    const bool xnan = ex == 0x7ff && mx, ynan = ey == 0x7ff && my;
    if (xnan || ynan) return __longlong_as_double(0x7fffffffffffffffll);
    const bool xinf = ex == 0x7ff, yinf = ey == 0x7ff;
    const bool xzero = ex == 0 && mx == 0, yzero = ey == 0 && my == 0;
    if ((xinf && yinf) || (xzero && yzero)) return __longlong_as_double(0x7fffffffffffffffll);
    if (xinf || yzero) return __longlong_as_double(sign | 0x7ff0000000000000ull);
    if (xzero || yinf) return __longlong_as_double(sign);
    // normalise significands to [2^52, 2^53)
    if (ex == 0) {
        const int sh = __clzll(mx) - 11;
        mx <<= sh;
        ex = 1 - sh;
    } else {
        mx |= 1ull << 52;
    }
    if (ey == 0) {
        const int sh = __clzll(my) - 11;
        my <<= sh;
        ey = 1 - sh;
    } else {
        my |= 1ull << 52;
    }
    int e = ex - ey + 1023;  // biased exponent of the quotient in [1, 2)
    if (mx < my) {
        mx <<= 1;
        e -= 1;
    }
    // 55 quotient bits: q in [2^54, 2^55), value q / 2^54
    uint64_t q = 0, rem = mx;
    for (int i = 0; i < 55; ++i) {
        q <<= 1;
        if (rem >= my) {
            rem -= my;
            q |= 1;
        }
        rem <<= 1;
    }
    const bool sticky_rem = rem != 0;
    int shift = 2;                 // drop guard + round position for a normal result
    if (e <= 0) shift += 1 - e;    // subnormal result: denormalise first
    uint64_t m, g, st;
    if (shift >= 57) {
        m = 0; g = 0; st = 1;
    } else {
        m = q >> shift;
        g = (q >> (shift - 1)) & 1;
        st = ((q & ((1ull << (shift - 1)) - 1)) != 0) || sticky_rem;
    }
    uint64_t bits;
    if (e <= 0) {
        bits = m;  // exponent field 0
    } else {
        if (e >= 2047) return __longlong_as_double(sign | 0x7ff0000000000000ull);
        bits = (uint64_t(e - 1) << 52) + m;  // m carries the hidden bit into the exponent
    }
    if (g && (st || (m & 1))) bits += 1;      // round to nearest even; carries propagate
    if (bits >= 0x7ff0000000000000ull) bits = 0x7ff0000000000000ull;
    return __longlong_as_double(sign | bits);
}

// x / y for a divisor known in advance with r = RN(1/y) (the constants 6, 12, 30 of the mass
// formulas).  q0 = RN(x r) is within 1.5 ulp of x/y; one correction q1 = RN(q0 + RN(x - y q0) r)
// (the residual is exact with an fma) makes it faithful; Markstein's theorem (a faithful q and
// an approximation of 1/y with relative error < 2^-53, which RN(1/y) is, give
// RN(q + (x - y q) r) = RN(x/y) in the normal range) makes the second correction correctly
// rounded.  Operands outside the safe exponent range take the exact integer path.
__device__ __forceinline__ double ddiv_rcp(double x, double y, double r) {
    const uint64_t bx = __double_as_longlong(x);
    const int ex = int((bx >> 52) & 0x7ff) - 1023;
    if (!(ex >= -960 && ex <= 960)) return ddiv_slow(x, y);
    double q = __dmul_rn(x, r);
    q = __fma_rn(__fma_rn(-q, y, x), r, q);
    return __fma_rn(__fma_rn(-q, y, x), r, q);
}

__device__ __forceinline__ double ddiv(double x, double y) {
    const uint64_t bx = __double_as_longlong(x), by = __double_as_longlong(y);
    const int ex = int((bx >> 52) & 0x7ff) - 1023, ey = int((by >> 52) & 0x7ff) - 1023;
    const bool fast = ex >= -960 && ex <= 960 && ey >= -960 && ey <= 960 && (ex - ey) >= -960 && (ex - ey) <= 960;
    if (!fast) return ddiv_slow(x, y);
    const uint64_t sign = (bx ^ by) & 0x8000000000000000ull;
    const double ax = fabs(x), ay = fabs(y);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(ay));
    double e = __fma_rn(-ay, r, 1.0);
    r = __fma_rn(e, r, r);
    e = __fma_rn(-ay, r, 1.0);
    r = __fma_rn(e, r, r);
    double q = __dmul_rn(ax, r);
    double rem = __fma_rn(-q, ay, ax);
    q = __fma_rn(rem, r, q);
    // exact correction: compare |rem| with half the gap to the neighbour in rem's direction
    rem = __fma_rn(-q, ay, ax);
    const uint64_t bq = __double_as_longlong(q);
    const uint64_t qexp = bq & 0x7ff0000000000000ull;
    const double half_up = __longlong_as_double(qexp - (53ull << 52));        // ulp(q)/2
    const bool pow2 = (bq & 0xfffffffffffffull) == 0;
    const double half_dn = pow2 ? __longlong_as_double(qexp - (54ull << 52)) : half_up;
    if (rem > 0.0) {
        const double lim = __dmul_rn(half_up, ay);
        if (rem > lim || (rem == lim && (bq & 1))) q = __longlong_as_double(bq + 1);
    } else if (rem < 0.0) {
        const double lim = __dmul_rn(half_dn, ay);
        if (-rem > lim || (-rem == lim && (bq & 1))) q = __longlong_as_double(bq - 1);
    }
    return __longlong_as_double(__double_as_longlong(q) | sign);
}

// Several quotients x_i / y with one divisor (the stiffness row's three entries share 4*area):
// r = RN(1/y) once, then each quotient by ddiv_rcp's two residual corrections (Markstein:
// faithful q + RN(1/y) give RN(x/y)).  Operands, 1/y or the quotient outside the safe exponent
// range take ddiv for that quotient.
//
// RN(1/y) for a positive y inside the safe exponent range: two Newton steps from rcp.approx
// leave r within an ulp of 1/y, and one more step r + r * (1 - y r) with the exact fma residual
// is then the correctly rounded reciprocal unless y's significand is all ones (Markstein's
// reciprocal theorem) - that divisor, like zero, negative or extreme ones, takes ddiv.
struct DivBy {
    double y, r;
    int ey;
    bool ok;
};
__device__ __forceinline__ DivBy div_prepare(double y) {
    DivBy d;
    const uint64_t by = __double_as_longlong(y);
    d.y = y;
    d.ey = int((by >> 52) & 0x7ff) - 1023;
    const bool plain = unsigned(d.ey + 960) <= 1920u && int64_t(by) > 0 &&
                       (by & 0xfffffffffffffull) != 0xfffffffffffffull;
    d.ok = unsigned(d.ey + 960) <= 1920u;
    if (plain) {
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
        double e = __fma_rn(-y, r, 1.0);
        r = __fma_rn(e, r, r);
        e = __fma_rn(-y, r, 1.0);
        r = __fma_rn(e, r, r);
        e = __fma_rn(-y, r, 1.0);
        d.r = __fma_rn(e, r, r);
    } else {
        d.r = d.ok ? ddiv(1.0, y) : 0.0;
    }
    return d;
}
__device__ __forceinline__ double div_by(const DivBy& d, double x) {
    const int ex = int((__double_as_longlong(x) >> 52) & 0x7ff) - 1023;
    if (!(d.ok && ex >= -960 && ex <= 960 && ex - d.ey >= -960 && ex - d.ey <= 960)) return ddiv(x, d.y);
    double q = __dmul_rn(x, d.r);
    q = __fma_rn(__fma_rn(-q, d.y, x), d.r, q);
    return __fma_rn(__fma_rn(-q, d.y, x), d.r, q);
}
// Three quotients by the same divisor with one range check for all (the largest and the
// smallest numerator exponent bound the others); any operand outside takes div_by's path.
__device__ __forceinline__ void div_by3(const DivBy& d, double x0, double x1, double x2, double& q0, double& q1,
                                        double& q2) {
    const int e0 = int((__double_as_longlong(x0) >> 52) & 0x7ff), e1 = int((__double_as_longlong(x1) >> 52) & 0x7ff),
              e2 = int((__double_as_longlong(x2) >> 52) & 0x7ff);
    const int lo = min(e0, min(e1, e2)) - 1023, hi = max(e0, max(e1, e2)) - 1023;
    if (d.ok && lo >= -960 && hi <= 960 && lo - d.ey >= -960 && hi - d.ey <= 960) {
        double a = __dmul_rn(x0, d.r), b = __dmul_rn(x1, d.r), c = __dmul_rn(x2, d.r);
        a = __fma_rn(__fma_rn(-a, d.y, x0), d.r, a);
        b = __fma_rn(__fma_rn(-b, d.y, x1), d.r, b);
        c = __fma_rn(__fma_rn(-c, d.y, x2), d.r, c);
        q0 = __fma_rn(__fma_rn(-a, d.y, x0), d.r, a);
        q1 = __fma_rn(__fma_rn(-b, d.y, x1), d.r, b);
        q2 = __fma_rn(__fma_rn(-c, d.y, x2), d.r, c);
    } else {
        q0 = div_by(d, x0);
        q1 = div_by(d, x1);
        q2 = div_by(d, x2);
    }
}

}  // namespace fa
