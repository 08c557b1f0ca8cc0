// Device self-tests exported through the C ABI (diagnostics, not on the assembly path).
#include "fa_common.cuh"
#include "fa_div.cuh"

#define FA_RCP6_ 0.16666666666666666
#define FA_RCP12_ 0.083333333333333329
#define FA_RCP30_ 0.033333333333333333

namespace fa {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Operand generator mixing raw bit patterns (every exponent, subnormals, inf, nan, zeros),
// values near 1 and the magnitudes the assembly divides (areas, weights, dot products).
__device__ __forceinline__ double gen_operand(uint64_t h) {
    const int mode = int(h & 7);
    const uint64_t r = splitmix64(h);
    switch (mode) {
        case 0: return __longlong_as_double(r);                                   // any bits
        case 1: return __longlong_as_double(r & 0x800fffffffffffffull);           // subnormal / zero
        case 2: return 1.0 + double(r >> 11) * 0x1.0p-53;                         // [1, 2)
        case 3: return __longlong_as_double((r & 0x800fffffffffffffull) | (uint64_t(1023 + int(r >> 52) % 40 - 20) << 52));
        case 4: return double(int64_t(r % 2000001) - 1000000);                      // integers
        case 5: return __longlong_as_double((r & 0x800fffffffffffffull) | (uint64_t(1 + (r >> 40) % 2046) << 52));
        case 6: return double(r >> 11) * 0x1.0p-53 * 1e-6;                         // small areas
        default: return __longlong_as_double(r & 0xfff0000000000000ull);          // powers of two / inf
    }
}

__global__ void k_selftest_div(int64_t n, uint64_t seed, unsigned long long* bad, double* first) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t h = splitmix64(seed ^ uint64_t(i) * 0x2545f4914f6cdd1dull);
        const double x = gen_operand(h), y = gen_operand(splitmix64(h + 17));
        const double mine = ddiv(x, y), ref = __ddiv_rn(x, y);
        const bool both_nan = mine != mine && ref != ref;
        if (!both_nan && __double_as_longlong(mine) != __double_as_longlong(ref)) {
            if (atomicAdd(bad, 1ull) == 0) {
                first[0] = x; first[1] = y; first[2] = mine; first[3] = ref;
            }
        }
        // shared divisor (RN(1/y) once, then residual corrections): the stiffness entries
        {
            const DivBy d = div_prepare(y);
            const double x2 = gen_operand(splitmix64(h + 29));
            const double xs[2] = {x, x2};
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const double m3 = div_by(d, xs[j]), r3 = __ddiv_rn(xs[j], y);
                if (!(m3 != m3 && r3 != r3) && __double_as_longlong(m3) != __double_as_longlong(r3)) {
                    if (atomicAdd(bad, 1ull) == 0) {
                        first[0] = xs[j]; first[1] = y; first[2] = m3; first[3] = r3;
                    }
                }
            }
        }
        // the same three at a time (div_by3), also for divisors whose significand is all ones or
        // just below (the reciprocal's exceptional case) and for plain positive divisors
        {
            const uint64_t hs = splitmix64(h + 41);
            const double ya = __longlong_as_double((uint64_t(1 + (hs >> 40) % 2046) << 52) |
                                                   (0xfffffffffffffull - ((hs >> 8) & 3ull)));
            const double yb = __longlong_as_double((uint64_t(1023 - 40 + (hs >> 30) % 80) << 52) | (splitmix64(hs) >> 12));
            const double ys3[3] = {y, ya, yb};
            const double xs[3] = {x, gen_operand(splitmix64(h + 29)), 1.0 + double(hs >> 11) * 0x1.0p-53};
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const DivBy d = div_prepare(ys3[t]);
                double m[3];
                div_by3(d, xs[0], xs[1], xs[2], m[0], m[1], m[2]);
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const double r3 = __ddiv_rn(xs[j], ys3[t]);
                    if (!(m[j] != m[j] && r3 != r3) && __double_as_longlong(m[j]) != __double_as_longlong(r3)) {
                        if (atomicAdd(bad, 1ull) == 0) {
                            first[0] = xs[j]; first[1] = ys3[t]; first[2] = m[j]; first[3] = r3;
                        }
                    }
                }
                // the reciprocal itself
                if (d.ok) {
                    const double rr = __ddiv_rn(1.0, ys3[t]);
                    if (!(d.r != d.r && rr != rr) && __double_as_longlong(d.r) != __double_as_longlong(rr)) {
                        if (atomicAdd(bad, 1ull) == 0) {
                            first[0] = 1.0; first[1] = ys3[t]; first[2] = d.r; first[3] = rr;
                        }
                    }
                }
            }
        }
        // constant divisors of the mass formulas (x only: y fixed)
        const double ys[3] = {6.0, 12.0, 30.0}, rs[3] = {FA_RCP6_, FA_RCP12_, FA_RCP30_};
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double m2 = ddiv_rcp(x, ys[j], rs[j]), r2 = __ddiv_rn(x, ys[j]);
            if (!(m2 != m2 && r2 != r2) && __double_as_longlong(m2) != __double_as_longlong(r2)) {
                if (atomicAdd(bad, 1ull) == 0) {
                    first[0] = x; first[1] = ys[j]; first[2] = m2; first[3] = r2;
                }
            }
        }
    }
}

}  // namespace fa

extern "C" int fa_selftest_division(int64_t n, uint64_t seed, unsigned long long* d_bad, double* d_first,
                                    void* stream) {
    if (n < 0 || !d_bad || !d_first) { fa::set_error("fa_selftest_division: bad argument"); return FA_ERR_ARGUMENT; }
    cudaStream_t st = fa::as_stream(stream);
    FA_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), st));
    fa::k_selftest_div<<<fa::grid_for(n, 256), 256, 0, st>>>(n, seed, d_bad, d_first);
    FA_LAUNCH_CHECK("k_selftest_div");
    return FA_OK;
}
