// fastnorm_math.cuh -- per-row arithmetic of the normalization kernels (device side).
//
// Every function here restates one reference routine of pkg/src/fastnorm/_kernels.pyx
// (cited per function) with the SAME operation order and one IEEE rounding per
// written operation: products and sums go through the __{d,f}{mul,add}_rn intrinsics,
// which nvcc never contracts into FMA (the reference is built -ffp-contract=off,
// setup.py:9), square roots through __{d,f}sqrt_rn, reciprocals through __{d,f}rcp_rn
// (correctly rounded 1/x == the reference's IEEE `1.0 / rt`), and the quotient /
// naive families through __{d,f}div_rn (true IEEE division; x/0 follows IEEE like
// Cython's cdivision=True, _kernels.pyx:5).  f32 computes entirely in binary32 with
// subnormals kept (built with -ftz=false), like the reference's `float` instantiation.
//
// The scaling families (normalize / norm) classify each row by integer operations on
// the IEEE bit patterns (exponent extraction): the largest |x_k| is the unsigned max of
// the sign-cleared bit patterns, and the band test against tau_min / tau_max is an
// unsigned compare.  DESIGN.md §3 proves this selects exactly the reference cascade's
// (inv, sigma) for every NaN-free row and produces the reference's all-NaN output for
// every row holding a NaN; the zero branch is taken iff every component is +-0.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace fnb {

// ---------------------------------------------------------------------------------
// Precision traits: the correctly rounded primitive operations, per binary format.
// ---------------------------------------------------------------------------------
template <typename T> struct Fp;

template <> struct Fp<double> {
    using Bits = unsigned long long;
    static constexpr Bits kAbsMask = 0x7fffffffffffffffull;
    __device__ __forceinline__ static Bits bits(double x) { return (Bits)__double_as_longlong(x); }
    __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
    __device__ __forceinline__ static double rcp(double a) { return __drcp_rn(a); }
    __device__ __forceinline__ static double sqrt(double a) { return __dsqrt_rn(a); }
    __device__ __forceinline__ static double abs(double a) { return fabs(a); }
    __device__ __forceinline__ static double sign1(double a) { return copysign(1.0, a); }
    __device__ __forceinline__ static bool isnan_(double a) { return isnan(a); }
    __device__ __forceinline__ static double ldexp_(double a, int e) { return ldexp(a, e); }
    __device__ __forceinline__ static int exponent_of_pow2(double p) {
        // p = 2^k (normal): k from the biased exponent field.
        return (int)((bits(p) >> 52) & 0x7ff) - 1023;
    }
    static constexpr int kShift = 52, kExpMax = 2046;
    __device__ __forceinline__ static double from_bits(Bits b) { return __longlong_as_double((long long)b); }
    __device__ __forceinline__ static int biased_exponent(double x) {
        return (int)(((unsigned)__double2hiint(x) >> 20) & 0x7ffu);
    }
};

template <> struct Fp<float> {
    using Bits = unsigned int;
    static constexpr Bits kAbsMask = 0x7fffffffu;
    __device__ __forceinline__ static Bits bits(float x) { return (Bits)__float_as_uint(x); }
    __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
    __device__ __forceinline__ static float div(float a, float b) { return __fdiv_rn(a, b); }
    __device__ __forceinline__ static float rcp(float a) { return __frcp_rn(a); }
    __device__ __forceinline__ static float sqrt(float a) { return __fsqrt_rn(a); }
    __device__ __forceinline__ static float abs(float a) { return fabsf(a); }
    __device__ __forceinline__ static float sign1(float a) { return copysignf(1.0f, a); }
    __device__ __forceinline__ static bool isnan_(float a) { return isnan(a); }
    __device__ __forceinline__ static float ldexp_(float a, int e) { return ldexpf(a, e); }
    __device__ __forceinline__ static int exponent_of_pow2(float p) {
        return (int)((bits(p) >> 23) & 0xff) - 127;
    }
    static constexpr int kShift = 23, kExpMax = 254;
    __device__ __forceinline__ static float from_bits(Bits b) { return __uint_as_float(b); }
    __device__ __forceinline__ static int biased_exponent(float x) {
        return (int)((__float_as_uint(x) >> 23) & 0xffu);
    }
};

// Power-of-two scaling by exponent insertion: x * 2^k computed as an integer add on the
// exponent field when both x and the result are normal -- exactly the bits of the IEEE
// product there -- and by the IEEE multiply otherwise (zero, subnormal input or result,
// overflow, inf, NaN), which rounds exactly as the reference's `sigma * x`.
//
// FNB_EXPONENT_INSERTION = 1 builds the scaling kernels with it (bit-identical: the
// full GPU parity suite passes, profiles/r01u_insertion.txt); the default 0 multiplies
// by the exact power of two instead, because the integer path measured 7 % slower on
// the bench workload (9.93 vs 9.21 ms per 2^30 rows: the per-row instruction count,
// not the FP64 pipe at 19 %, paces the tile loop).
#ifndef FNB_EXPONENT_INSERTION
#define FNB_EXPONENT_INSERTION 0
#endif
template <typename T>
__device__ __forceinline__ bool pow2_insertable(T x, int k) {
    const int e = Fp<T>::biased_exponent(x);
    return e >= 1 && e <= Fp<T>::kExpMax && e + k >= 1 && e + k <= Fp<T>::kExpMax;
}
template <typename T>
__device__ __forceinline__ T pow2_insert(T x, int k) {
    using B = typename Fp<T>::Bits;
    return Fp<T>::from_bits(Fp<T>::bits(x) + (B)((long long)k << Fp<T>::kShift));
}
template <typename T>
__device__ __forceinline__ T pow2_scale(T x, int k, T factor, bool insert_ok) {
#if FNB_EXPONENT_INSERTION
    return (insert_ok && pow2_insertable(x, k)) ? pow2_insert(x, k) : Fp<T>::mul(factor, x);
#else
    (void)k;
    (void)insert_ok;
    return Fp<T>::mul(factor, x);  // factor = 2^k exactly: same bits as the insertion
#endif
}

// The six kernel arguments (scale.py:26-30), already rounded to T, plus the bit
// patterns of the two band thresholds for the integer band test.
template <typename T> struct KArgs {
    T tau_min, tau_max, sigma_min, sigma_max, inv_min, inv_max;
    typename Fp<T>::Bits tau_min_bits, tau_max_bits;
    int k_min, k_max;   // log2(sigma_min), log2(sigma_max) when pow2 (validated sets)
    bool pow2;          // sigma_min, sigma_max and their inverses are powers of two
    unsigned long long* invalid;  // rows rejected by the rotations (may be NULL)
    unsigned* sched;              // tma_stream_kernel's dynamic tile counter (NULL: the
                                  // static round-robin schedule)
    unsigned* sched_next;         // the counter of the next launch on the stream (zeroed here;
                                  // NULL for captured launches)
    unsigned* sched_done;         // captured launches: CTAs finished; the last one re-zeroes
                                  // sched and this word for the next replay (NULL otherwise)
    int sched_batch;              // tiles per claim of the dynamic schedule
    T rot[9];           // FN_OP_ROT_APPLY: the matrix, row-major
};

// ---------------------------------------------------------------------------------
// Scaling: integer classification + power-of-two scale (Algs 3/4, Alg 7 lines 4-23).
// Returns false for the all-zero row.  s_k = fl(sigma * x_k) exactly as the reference
// (_kernels.pyx:97-112): exact unless the sigma_max product drops below nu.
// ---------------------------------------------------------------------------------
template <typename T, int N>
__device__ __forceinline__ bool scale_classified(const T (&x)[N], const KArgs<T>& ka, T& inv,
                                                 T (&s)[N]) {
    using F = Fp<T>;
    typename F::Bits m = F::bits(x[0]) & F::kAbsMask;
#pragma unroll
    for (int k = 1; k < N; ++k) {
        typename F::Bits a = F::bits(x[k]) & F::kAbsMask;
        m = a > m ? a : m;
    }
    // m is the bit pattern of max |x_k| (NaN > inf > finite in this order).
    const bool big = m > ka.tau_max_bits;     // includes inf and NaN rows
    const bool small = m < ka.tau_min_bits;
    const T sigma = big ? ka.sigma_max : (small ? ka.sigma_min : T(1));
    inv = big ? ka.inv_max : (small ? ka.inv_min : T(1));
    // s_k = sigma * x_k by exponent insertion (k = log2 sigma) where exact, else IEEE mul
    const int k = big ? ka.k_max : (small ? ka.k_min : 0);
#pragma unroll
    for (int c = 0; c < N; ++c) s[c] = pow2_scale(x[c], k, sigma, ka.pow2);
    return m != 0;
}

template <typename T>
__device__ __forceinline__ int inv_exponent(const KArgs<T>& ka, T inv) {
    // inv = 2^-k of the selected branch (1, 1/sigma_max, 1/sigma_min)
    return inv == ka.inv_max ? -ka.k_max : (inv == ka.inv_min ? -ka.k_min : 0);
}

// ---------------------------------------------------------------------------------
// Correctly rounded division by a shared divisor (the quotient / naive families divide
// n numerators by the same m, h or r; _kernels.pyx:262-362).
//
// Fast path (binary64): y = RN(1/b) once per divisor (__drcp_rn), then per numerator
//   q0 = RN(a*y); r0 = fma(-b, q0, a); q1 = fma(r0, y, q0)     -> q1 faithful
//   r1 = fma(-b, q1, a)  (exact: remainder of a faithful quotient, Boldo-Daumas)
//   q2 = fma(r1, y, q1)  == RN(a/b)  (Markstein: y = RN(1/b), q1 faithful, r1 exact)
// valid while a >= 2^-967, 2^-1020 <= |b| < 2^1022 and the quotient exponent is in
// [-967, 1021] (no subnormal intermediate or result).  Outside that range: an exactly
// zero numerator gives the signed zero; a quotient provably below 2^-1075 rounds to the
// signed zero (|a/b| < 2^(ea - eb + 1)); everything else (subnormal results, zero /
// inf / NaN divisors) takes the IEEE __ddiv_rn.  This keeps the very common "tiny
// component over huge max" case of wide-range rows off the slow path.
//
// binary32: the numerator and divisor are widened to binary64 (exactly), divided with
// the binary64 fast path above (always in range for float operands) and rounded once to
// binary32.  Double rounding is innocuous for division since 53 >= 2*24 + 2 (the same
// argument the reference's pure-Python twin relies on, _pykernels.py:7-11), including
// subnormal float results (a midpoint of the subnormal grid has <= 24 significant bits,
// so a binary64 quotient can only land on it when it is exact).  Every case is checked
// bit for bit against __ddiv_rn / __fdiv_rn by fn_selftest_div (tests/test_gpu_parity.py).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double div_markstein(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double r0 = __fma_rn(-b, q0, a);
    const double q1 = __fma_rn(r0, y, q0);
    const double r1 = __fma_rn(-b, q1, a);
    return __fma_rn(r1, y, q1);
}

__device__ __forceinline__ int biased_exp(double v) {
    return (int)(((unsigned)__double2hiint(v) >> 20) & 0x7ffu);
}

__device__ __forceinline__ double signed_zero_of_quotient(double a, double b) {
    const long long s = (__double_as_longlong(a) ^ __double_as_longlong(b)) & (long long)0x8000000000000000ull;
    return __longlong_as_double(s);
}

template <typename T> struct Divider;

// Binary64 shared-divisor division with the Markstein fast path described above.
struct MarksteinDivider {
    double b, y;
    int eb;
    bool bfast;
    __device__ __forceinline__ explicit MarksteinDivider(double b_) : b(b_) {
        eb = biased_exp(b_);
        bfast = eb >= 3 && eb <= 2044;
        y = __drcp_rn(bfast ? b_ : 1.0);
    }
    __device__ __forceinline__ double operator()(double a) const {
        const int ea = biased_exp(a);
        const int d = ea - eb;
        const double fast = div_markstein(a, b, y);
        if (bfast && ea >= 56 && ea <= 2046 && d >= -967 && d <= 1021) return fast;
        const bool b_finite_nonzero = eb <= 2046 && b != 0.0;
        // exact zero numerator, or a quotient provably below half the least subnormal
        if (b_finite_nonzero && ea <= 2046 &&
            (a == 0.0 || (ea >= 1 && eb >= 1 && d <= -1076) || (ea == 0 && eb >= 1076)))
            return signed_zero_of_quotient(a, b);
        return __ddiv_rn(a, b);
    }
};

// FNB_F64_DIV_MARKSTEIN = 1 selects MarksteinDivider for the binary64 quotient / naive
// families; 0 divides with __ddiv_rn per numerator.  Both are correctly rounded; on
// wide-range rows (config 5) the subnormal-result slow path dominates and plain
// __ddiv_rn measured faster (profiles/r01d_div_*.csv); for rotation_general (9 entries
// over one ss) it also measured slower (5338 vs 5552 GB/s, profiles/r01f_tune_rot.csv).
// So 0 is the default; the variant stays selectable and is checked by fn_selftest_div.
#ifndef FNB_F64_DIV_MARKSTEIN
#define FNB_F64_DIV_MARKSTEIN 0
#endif

// Quotients that land on the subnormal grid (or flush to zero), computed exactly without
// the library division's generic slow path.  Preconditions: a finite, b finite normal
// (biased exponent 1..2046), and the normalised exponent gap ea - eb <= -1023, so
// |a/b| < 2^-1022 and RN(a/b) = n 2^-1074 with n = RN_int(X), X = (fa / fb) 2^s,
// fa, fb in [1, 2), s = ea - eb + 1074 <= 51 (for s = 51, X < 2^52, RN(A/fb) is within
// 2^-2 of X and |r| <= 1.5 stays exact; n = 2^52 is the bit pattern of 2^-1022, the
// correct result when X rounds up onto the normal range):
//   s <= -2 : X < 1/2, n = 0;
//   s == -1 : X in (1/4, 1), n = [fa > fb] (X == 1/2 only if fa == fb: tie -> 0, even);
//   s >=  0 : n0 = rint(RN(A / fb)), A = fa 2^s; |RN(A/fb) - X| <= 2^-3, so n0 is off by
//             at most one; r = A - n0 fb is exact (a multiple of 2^-52 below 2 in
//             magnitude) and decides: 2|r| > fb moves n0 one step towards X.  A tie
//             (2|r| == fb) means X = n0 +- 1/2 is representable, hence RN(A/fb) = X and
//             rint already chose the even neighbour.
// The result bits are n itself (n <= 2^51) with the xor sign.
__device__ __forceinline__ double tiny_quotient(double a, double b, int ea, unsigned long long ma, int eb) {
    const unsigned long long kMant = 0x000FFFFFFFFFFFFFull, kOne = 1023ull << 52;
    const unsigned long long sign = (__double_as_longlong(a) ^ __double_as_longlong(b)) & 0x8000000000000000ull;
    const int s = ea - eb + 1074;
    const double fa = __longlong_as_double((long long)(ma | kOne));
    const double fb = __longlong_as_double((long long)((__double_as_longlong(b) & kMant) | kOne));
    long long n = 0;
    if (s == -1) {
        n = fa > fb ? 1 : 0;
    } else if (s >= 0) {
        const double A = __longlong_as_double((long long)(ma | ((unsigned long long)(1023 + s) << 52)));
        double n0 = rint(__ddiv_rn(A, fb));
        const double r = __fma_rn(-n0, fb, A);
        if (fabs(__dadd_rn(r, r)) > fb) n0 = __dadd_rn(n0, r > 0.0 ? 1.0 : -1.0);
        n = __double2ll_rn(n0);
    }
    return __longlong_as_double((long long)((unsigned long long)n | sign));
}

// IEEE quotient when an operand is zero, infinite or NaN (the cases a library division
// sends to its slow path): NaN for 0/0, inf/inf and any NaN; a signed infinity for
// x/0 and inf/x; a signed zero for 0/x and x/inf.  Signs combine by xor.
__device__ __forceinline__ float special_quotient(float a, float b) {
    const unsigned sign = (__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u;
    const bool nan = isnan(a) || isnan(b) || (a == 0.0f && b == 0.0f) || (isinf(a) && isinf(b));
    const bool inf = isinf(a) || b == 0.0f;
    return nan ? __uint_as_float(0x7fc00000u) : __uint_as_float(sign | (inf ? 0x7f800000u : 0u));
}

__device__ __forceinline__ double special_quotient(double a, double b) {
    const unsigned long long sign =
        ((unsigned long long)__double_as_longlong(a) ^ (unsigned long long)__double_as_longlong(b)) &
        0x8000000000000000ull;
    const bool nan = isnan(a) || isnan(b) || (a == 0.0 && b == 0.0) || (isinf(a) && isinf(b));
    const bool inf = isinf(a) || b == 0.0;
    return nan ? __longlong_as_double(0x7ff8000000000000ll)
               : __longlong_as_double((long long)(sign | (inf ? 0x7ff0000000000000ull : 0ull)));
}

#if !FNB_F64_DIV_MARKSTEIN
// Plain IEEE division per numerator (__ddiv_rn).  Measured alternatives, all exact and
// checked by fn_selftest_div, all slower on unit-range rows (configs 1, 3):
//   * Markstein shared reciprocal (MarksteinDivider below): profiles/r01d_div_*.csv;
//   * skipping provably-zero quotients in a branch: profiles/r01l_div_zero_shortcut.csv;
//   * branch-free tiny-result path (numerator scaled by 2^600, one rounding onto the
//     subnormal grid, midpoint fix from the exact remainder): +20 % on config 2 and +6 %
//     on config 5 quotient rows, but -40 % on configs 1 and 3 (profiles/r01s_div.csv).
// FNB_F64_TINY_QUOTIENT = 1 routes subnormal-grid quotients to tiny_quotient instead of
// the library slow path.  Exact (fn_selftest_div, golden, full-size parity), but the
// division-bound kernels are issue-bound and the per-division range test costs more
// than it saves: quotient2 cfg 2 55.2 -> 50.9, quotient3 cfg 5 36.6 -> 30.1 and cfg 1
// 101 -> 79 Gvec/s (profiles/r01bq_ab.txt).  Also measured: the same out of line
// (__noinline__), and a form that keeps every lane on __ddiv_rn's fast path (tiny lanes
// divide 1 by b) and patches afterwards -- both as slow on the unit-range configs
// (quotient3 cfg 1: 80 / 76 Gvec/s; profiles/r01cg_ab.txt, r01ch_ab.txt).  Off.
#ifndef FNB_F64_TINY_QUOTIENT
#define FNB_F64_TINY_QUOTIENT 0
#endif
// FNB_F64_DIV_SPECIAL: 1 = a zero, infinite or NaN divisor (tested once per divisor)
// gives special_quotient instead of the library division's slow path; 2 = also a zero
// numerator inline; 0 = plain __ddiv_rn.  Measured mixed (profiles/r01s29_ab_f64special.txt,
// alternated processes): 1 = naive3 cfg 5 +3.9 %, quotient4 cfg 3 +4.7 %, quotient3
// cfg 1 +3.4 %, but quotient2 cfg 2 -6.7 %, quotient3 cfg 5 -4.5 %; 2 = quotient2 +5.4 %,
// naive3 +4.7 %, quotient3 +4.2 %, but quotient3_fast -4.2 %, quotient4 -3.0 %.  The
// binary32 version pays because binary32 quotients are emulated in binary64; here the
// special divisors are not where the time goes, so the plain division stays.
#ifndef FNB_F64_DIV_SPECIAL
#define FNB_F64_DIV_SPECIAL 0
#endif
template <> struct Divider<double> {
    double b;
    bool bok;
#if FNB_F64_TINY_QUOTIENT
    int eb;
    __device__ __forceinline__ explicit Divider(double b_) : b(b_) {
        eb = biased_exp(b_);
        bok = isfinite(b_) && b_ != 0.0;
    }
#else
    __device__ __forceinline__ explicit Divider(double b_) : b(b_) { bok = isfinite(b_) && b_ != 0.0; }
#endif
    __device__ __forceinline__ double operator()(double a) const {
#if FNB_F64_DIV_SPECIAL >= 1
        if (!bok) return special_quotient(a, b);
#endif
#if FNB_F64_DIV_SPECIAL >= 2
        if (a == 0.0)
            return __longlong_as_double(
                (long long)(((unsigned long long)__double_as_longlong(a) ^ (unsigned long long)__double_as_longlong(b)) &
                            0x8000000000000000ull));
#endif
#if FNB_F64_TINY_QUOTIENT
        // Wide-range rows divide small components by large ones: results on the subnormal
        // grid take tiny_quotient (normal or subnormal numerator, normal divisor).
        const unsigned long long ba = (unsigned long long)__double_as_longlong(a) & 0x7FFFFFFFFFFFFFFFull;
        int ea = (int)(ba >> 52);
        unsigned long long ma = ba & 0x000FFFFFFFFFFFFFull;
        if (ea == 0 && ma != 0) {  // subnormal numerator: normalise the significand
            const int lz = __clzll((long long)ma) - 11;
            ma = (ma << lz) & 0x000FFFFFFFFFFFFFull;
            ea = 1 - lz;
        }
        if (ba != 0 && ea <= 2046 && eb >= 1 && eb <= 2046 && ea - eb <= -1024)
            return tiny_quotient(a, b, ea, ma, eb);
#endif
        return __ddiv_rn(a, b);
    }
};
#else
template <> struct Divider<double> : MarksteinDivider {
    __device__ __forceinline__ explicit Divider(double b_) : MarksteinDivider(b_) {}
};
#endif

// Binary32 Markstein division in binary32 arithmetic (same argument as div_markstein
// above, p = 24): y = RN(1/b) (__frcp_rn), q1 faithful, r1 exact, q2 = RN(a/b).
__device__ __forceinline__ float div_markstein32(float a, float b, float y) {
    const float q0 = __fmul_rn(a, y);
    const float r0 = __fmaf_rn(-b, q0, a);
    const float q1 = __fmaf_rn(r0, y, q0);
    const float r1 = __fmaf_rn(-b, q1, a);
    return __fmaf_rn(r1, y, q1);
}

__device__ __forceinline__ int biased_exp32(float v) { return (int)((__float_as_uint(v) >> 23) & 0xffu); }

// FNB_F32_DIV_NATIVE = 1 divides in-range binary32 operands natively (div_markstein32)
// and keeps the binary64 path for the rest.  Exact (fn_selftest_div), but measured
// slower everywhere (__frcp_rn plus the range test cost more than the binary64 Markstein
// with its shared reciprocal): quotient3 f32 3780 -> 2440 GB/s on config 4 and
// 3818 -> 3204 in band; quotient3_fast 5461 -> 3961 (profiles/r01bn_ab.txt).  Off.
#ifndef FNB_F32_DIV_NATIVE
#define FNB_F32_DIV_NATIVE 0
#endif

#ifndef FNB_F32_DIV_RECIP
#define FNB_F32_DIV_RECIP 1
#endif
template <> struct Divider<float> {
    double b, y;
    float bf;
    bool bok;
#if FNB_F32_DIV_NATIVE
    float yf;
    bool bfast;
    int eb;
#endif
    __device__ __forceinline__ explicit Divider(float b_) : b((double)b_), bf(b_) {
        bok = isfinite(b_) && b_ != 0.0f;
        y = __drcp_rn(bok ? b : 1.0);
#if FNB_F32_DIV_NATIVE
        eb = biased_exp32(b_);
        bfast = eb >= 3 && eb <= 252;
        yf = __frcp_rn(bfast ? b_ : 1.0f);
#endif
    }
    __device__ __forceinline__ float operator()(float a) const {
#if FNB_F32_DIV_NATIVE
        // |a| >= 2^-100, 2^-124 <= |b| < 2^126, quotient exponent in [-100, 125] (the
        // binary32 image of the binary64 bounds above): no intermediate under/overflow,
        // r0 and r1 exact, so the Markstein result is RN(a/b).
        const int ea = biased_exp32(a);
        const int d = ea - eb;
        if (bfast && ea >= 27 && ea <= 254 && d >= -100 && d <= 125) return div_markstein32(a, bf, yf);
#endif
        // Finite operands: the binary64 quotient of two binary32 values rounded once to
        // binary32 (innocuous double rounding); a zero numerator gives the xor-signed zero.
        // The rest goes to special_quotient instead of the library division's slow path:
        // naive3 f32 63 -> 125 Gvec/s, quotient3_fast f32 165 -> 179, quotient3 f32
        // 113 -> 117 (config 4, profiles/r01ad_ab.txt; "old" is the library fallback).
#if FNB_F32_DIV_RECIP
        // One binary64 product with the shared reciprocal y = RN64(1/b), rounded once to
        // binary32.  q = (a/b)(1 + e), |e| <= 2^-52 + 2^-106.  For 24-bit a and b, a
        // quotient that is not itself a binary32 midpoint lies at least 2^-49 (relative)
        // from every midpoint of the result grid: a/b - mu = (A 2^s - M B) 2^em / B with
        // integers A, B < 2^24, M < 2^25 and s >= -1.  The same holds on the subnormal
        // grid (absolute gap >= 2^-175, error <= M 2^-202).  So q and a/b round to the
        // same binary32 value.  Exact midpoints need b a power of two, where y and q are
        // exact.  A zero numerator gives the xor-signed zero by itself.  Checked bit for
        // bit against __fdiv_rn by fn_selftest_div.
#ifdef FNB_DIV_NEGATIVE_CONTROL
        // test-only: a reciprocal truncated to 45 bits must be caught by the selftest's
        // near-midpoint category (tools/selftest_big.py)
        if (bok && isfinite(a))
            return __double2float_rn(__dmul_rn((double)a, __longlong_as_double(__double_as_longlong(y) & ~0xFFll)));
#endif
        if (bok && isfinite(a)) return __double2float_rn(__dmul_rn((double)a, y));
#else
        if (bok && isfinite(a)) {
            const float q = __double2float_rn(div_markstein((double)a, b, y));
            const float z = __uint_as_float((__float_as_uint(a) ^ __float_as_uint(bf)) & 0x80000000u);
            return a != 0.0f ? q : z;
        }
#endif
        return special_quotient(a, bf);
    }
};

// Left-to-right sum of squares without contraction: ((s1^2 + s2^2) + s3^2) + s4^2.
template <typename T, int N>
__device__ __forceinline__ T sum_squares(const T (&s)[N]) {
    using F = Fp<T>;
    T acc = F::mul(s[0], s[0]);
#pragma unroll
    for (int k = 1; k < N; ++k) acc = F::add(acc, F::mul(s[k], s[k]));
    return acc;
}

// normalize{2,3,4}: _kernels.pyx:167-225.  Zero row -> r = 0, unit = 0 (n = 4: the
// identity quaternion (0,0,0,1), :211-218).  Optional squared length (config 3):
// sq = ldexp(ss, 2*log2(inv)), correctly rounded.
template <typename T, int N, bool kSq>
__device__ __forceinline__ void normalize_row(const T (&x)[N], const KArgs<T>& ka, T& r,
                                              T (&u)[N], T& sq) {
    using F = Fp<T>;
    T inv, s[N];
    const bool nonzero = scale_classified<T, N>(x, ka, inv, s);
    const T ss = sum_squares<T, N>(s);
    const T rt = F::sqrt(ss);
    const T h = F::rcp(rt);
    const int ki = inv_exponent(ka, inv);
    // r = inv * rt: exponent insertion while the length stays normal, IEEE mul otherwise
    // (warranted overflow to inf, rounding into subnormals)
    r = nonzero ? pow2_scale(rt, ki, inv, ka.pow2) : T(0);
#pragma unroll
    for (int k = 0; k < N; ++k) u[k] = nonzero ? F::mul(h, s[k]) : T(0);
    if (N == 4) u[N - 1] = nonzero ? u[N - 1] : T(1);
    if (kSq) {
        // sq = ss * inv^2 = ldexp(ss, 2 ki), one correct rounding
        const int ks = ka.pow2 ? ki : F::exponent_of_pow2(inv);
        const bool ins = FNB_EXPONENT_INSERTION && ka.pow2 && pow2_insertable(ss, 2 * ks);
        sq = nonzero ? (ins ? pow2_insert(ss, 2 * ks) : F::ldexp_(ss, 2 * ks)) : T(0);
    }
}

// norm{2,3,4}: _kernels.pyx:228-255; bit-identical to normalize's r.
template <typename T, int N>
__device__ __forceinline__ T norm_row(const T (&x)[N], const KArgs<T>& ka) {
    using F = Fp<T>;
    T inv, s[N];
    const bool nonzero = scale_classified<T, N>(x, ka, inv, s);
    const T r = pow2_scale(F::sqrt(sum_squares<T, N>(s)), inv_exponent(ka, inv), inv, ka.pow2);
    return nonzero ? r : T(0);
}

// scale{2,3,4}: the exported preprocessor keeps the reference's exact comparison
// cascade, because with a NaN present its (inv, s) outcome depends on the order of
// the comparisons.  Verbatim branch structure of _kernels.pyx:51-160.
// Band test of the cascade (_kernels.pyx:63-75 and siblings).  Returns true for the
// in-band row, whose components are passed through unscaled.
template <typename T>
__device__ __forceinline__ bool scale_tail(T m, const KArgs<T>& ka, T& inv, T& sigma) {
    if (m >= ka.tau_min) {
        if (m <= ka.tau_max) { inv = T(1); sigma = T(1); return true; }
        inv = ka.inv_max; sigma = ka.sigma_max; return false;
    }
    inv = ka.inv_min; sigma = ka.sigma_min; return false;
}

template <typename T>
__device__ __forceinline__ void scale_row(const T (&x)[2], const KArgs<T>& ka, T& inv, T (&s)[2]) {
    using F = Fp<T>;
    T m = F::abs(x[0]);  // _kernels.pyx:54-62
    if (m >= F::abs(x[1])) {
        if (m == T(0)) { inv = T(0); s[0] = T(0); s[1] = T(0); return; }
    } else {
        m = F::abs(x[1]);
    }
    T sigma;
    if (scale_tail(m, ka, inv, sigma)) { s[0] = x[0]; s[1] = x[1]; return; }
    s[0] = F::mul(sigma, x[0]); s[1] = F::mul(sigma, x[1]);
}

template <typename T>
__device__ __forceinline__ void scale_row(const T (&x)[3], const KArgs<T>& ka, T& inv, T (&s)[3]) {
    using F = Fp<T>;
    T m = F::abs(x[0]);  // _kernels.pyx:81-96
    if (m < F::abs(x[1])) {
        m = F::abs(x[1]);
        if (m < F::abs(x[2])) m = F::abs(x[2]);
    } else {
        if (m >= F::abs(x[2])) {
            if (m == T(0) && !F::isnan_(x[1])) {
                inv = T(0); s[0] = T(0); s[1] = T(0); s[2] = T(0); return;
            }
        } else {
            m = F::abs(x[2]);
        }
    }
    T sigma;
    if (scale_tail(m, ka, inv, sigma)) { s[0] = x[0]; s[1] = x[1]; s[2] = x[2]; return; }
    s[0] = F::mul(sigma, x[0]); s[1] = F::mul(sigma, x[1]); s[2] = F::mul(sigma, x[2]);
}

template <typename T>
__device__ __forceinline__ void scale_row(const T (&x)[4], const KArgs<T>& ka, T& inv, T (&s)[4]) {
    using F = Fp<T>;
    T m = F::abs(x[0]);  // _kernels.pyx:119-141
    if (m < F::abs(x[1])) {
        m = F::abs(x[1]);
        if (m < F::abs(x[2])) m = F::abs(x[2]);
        if (m < F::abs(x[3])) m = F::abs(x[3]);
    } else {
        if (m < F::abs(x[2])) {
            m = F::abs(x[2]);
            if (m < F::abs(x[3])) m = F::abs(x[3]);
        } else {
            if (m >= F::abs(x[3])) {
                if (m == T(0) && !(F::isnan_(x[1]) || F::isnan_(x[2]))) {
                    inv = T(0); s[0] = T(0); s[1] = T(0); s[2] = T(0); s[3] = T(0); return;
                }
            } else {
                m = F::abs(x[3]);
            }
        }
    }
    T sigma;
    if (scale_tail(m, ka, inv, sigma)) {
        s[0] = x[0]; s[1] = x[1]; s[2] = x[2]; s[3] = x[3]; return;
    }
    s[0] = F::mul(sigma, x[0]); s[1] = F::mul(sigma, x[1]);
    s[2] = F::mul(sigma, x[2]); s[3] = F::mul(sigma, x[3]);
}

// naive{2,3,4}: _kernels.pyx:262-285.  r = sqrt(sum x^2), u = x / r (true divisions).
template <typename T, int N>
__device__ __forceinline__ void naive_row(const T (&x)[N], T& r, T (&u)[N]) {
    using F = Fp<T>;
    const T rr = F::sqrt(sum_squares<T, N>(x));
    r = rr;
    const Divider<T> by_r(rr);
#pragma unroll
    for (int k = 0; k < N; ++k) u[k] = by_r(x[k]);
}

// quotient{2,3,4}: _kernels.pyx:288-362 (Alg 1 generalised).  m = max via strict '>',
// zero row (no NaN) -> all +0 (n = 4: five zeros, no identity quaternion).
//
// FNB_QUOTIENT_PIVOT = 1 (default) computes the same IEEE results with n - 1 divisions
// per stage instead of n.  For a row with finite m > 0, a component with |x_j| == m has
// x_j / m = +-1 exactly and x_j / m / h = +-RN(1/h) (rounding is sign-symmetric), so only
// the other n - 1 components are divided, the reciprocal of h is one correctly rounded
// __drcp_rn / __frcp_rn, and the sum of squares is still formed in the reference's left-
// to-right order over all n quotients.  Like quotient3_fast_row, the row's operands are
// selected first (the other components in their original order) so every lane of a warp
// runs the same n - 1 division sites whichever component is largest: on wide-range rows,
// where quotients land on the subnormal grid, each site with such a lane costs the warp
// one pass of the library division's slow path.  Rows with a NaN or an infinity give NaN
// everywhere (NaN / m, inf / inf), as the reference's arithmetic does; the zero row gives
// zeros.  FNB_QUOTIENT_PIVOT = 0 is the literal transcription kept for A/B timing.
// Measured (tools/ab_quotient.sh, profiles/r02e_ab_quotient.txt, r02f_ab_quotient.txt):
// quotient2 config 2 2226 -> 3260 GB/s, quotient3 config 5 2134 -> 2624, quotient4
// config 3 5812 -> 6042, quotient3 config 1 5761 -> 5885.  Binary32 keeps the literal
// form (pivot: 4655 -> 4424 GB/s on config 4).  Also measured and dropped: the Markstein
// division by h with the shared reciprocal (-4 % on configs 2 and 5), and routing the
// quotients below 2^-1022 to tiny_quotient by exponent gap (-11 % on config 2, -13 % on
// config 5: the extra path is longer than the library's slow path it replaces).
#ifndef FNB_QUOTIENT_PIVOT
#define FNB_QUOTIENT_PIVOT 1
#endif

template <typename T, int N>
__device__ __forceinline__ void quotient_row(const T (&x)[N], T& r, T (&u)[N]) {
    using F = Fp<T>;
    T m = F::abs(x[0]);
#pragma unroll
    for (int k = 1; k < N; ++k) {
        const T a = F::abs(x[k]);
        if (a > m) m = a;
    }
    bool anynan = false;
#pragma unroll
    for (int k = 0; k < N; ++k) anynan = anynan || F::isnan_(x[k]);
#if FNB_QUOTIENT_PIVOT
  if constexpr (std::is_same<T, double>::value) {  // binary32 quotients are one binary64
    // product each (Divider<float>): the pivot's selects cost more than they save there
    // finite m > 0 and no NaN: every component finite (an infinity would be m)
    const bool regular = !anynan && m > T(0) && isfinite(m);
    int j = N - 1;  // first component of magnitude m
#pragma unroll
    for (int k = N - 2; k >= 0; --k)
        if (F::abs(x[k]) == m) j = k;
    T o[N - 1];  // the other components, original order
#pragma unroll
    for (int i = 0; i < N - 1; ++i) o[i] = (i < j) ? x[i] : x[i + 1];
    T qo[N - 1];
    const Divider<T> by_m(regular ? m : T(1));
#pragma unroll
    for (int i = 0; i < N - 1; ++i) qo[i] = by_m(regular ? o[i] : T(0));
    T sj = x[0];
#pragma unroll
    for (int k = 1; k < N; ++k) sj = (k == j) ? x[k] : sj;
    sj = F::sign1(sj);
    T q[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        T v = sj;
        if (k < N - 1) v = (k < j) ? qo[k < N - 1 ? k : 0] : v;
        if (k > 0) v = (k > j) ? qo[k > 0 ? k - 1 : 0] : v;
        q[k] = v;
    }
    const T h = F::sqrt(sum_squares<T, N>(q));
    r = F::mul(m, h);
    const T y = F::rcp(h);
    T uo[N - 1];
    const Divider<T> by_h(h);
#pragma unroll
    for (int i = 0; i < N - 1; ++i) uo[i] = by_h(qo[i]);
    const T uj = F::mul(sj, y);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        T v = uj;
        if (k < N - 1) v = (k < j) ? uo[k < N - 1 ? k : 0] : v;
        if (k > 0) v = (k > j) ? uo[k > 0 ? k - 1 : 0] : v;
        u[k] = v;
    }
    if (!regular) {
        const T fill = anynan || m > T(0) ? T(NAN) : T(0);  // NaN / infinity rows, zero row
        r = fill;
#pragma unroll
        for (int k = 0; k < N; ++k) u[k] = fill;
    }
    return;
  }
#endif
    {  // the literal transcription: binary32, or FNB_QUOTIENT_PIVOT = 0
    if (m == T(0) && !anynan) {
        r = T(0);
#pragma unroll
        for (int k = 0; k < N; ++k) u[k] = T(0);
        return;
    }
    T q[N];
    const Divider<T> by_m(m);
#pragma unroll
    for (int k = 0; k < N; ++k) q[k] = by_m(x[k]);
    const T h = F::sqrt(sum_squares<T, N>(q));
    r = F::mul(m, h);
    const Divider<T> by_h(h);
#pragma unroll
    for (int k = 0; k < N; ++k) u[k] = by_h(q[k]);
    }
}

// Shared body of the pivoted fast quotient (_kernels.pyx:370-377 and siblings):
// p dominates, a and b ride along.  h = sqrt((1 + qa^2) + qb^2), t = sign(p)/h.
template <typename T>
__device__ __forceinline__ void qf_pivot(T p, T a, T b, T& r, T& t, T& ua, T& ub) {
    using F = Fp<T>;
    const Divider<T> by_p(p);
    const T qa = by_p(a);
    const T qb = by_p(b);
    const T h = F::sqrt(F::add(F::add(T(1), F::mul(qa, qa)), F::mul(qb, qb)));
    t = F::div(F::sign1(p), h);
    r = F::mul(F::abs(p), h);
    ua = F::mul(qa, t);
    ub = F::mul(qb, t);
}

// quotient3_fast: _kernels.pyx:365-412 (Alg 2).  The reference's pivot decision tree
// (verbatim comparisons, ties and zero test) is evaluated with selects instead of
// branches, then ONE pivot body runs for every lane: each branch of the reference
// computes the same formula (qf_pivot) on a permutation of (x1, x2, x3), so selecting
// the operands first and permuting the results after gives identical values while a
// warp with mixed pivots no longer executes three division sequences in turn.
//   |x1| > |x2|:  |x3| > |x1| ? pivot x3 (a=x1, b=x2; u=(ua,ub,t))
//                              : pivot x1 (a=x3, b=x2; u=(t,ub,ua))
//   otherwise:    |x3| >= |x2| ? [x3 == 0 && !isnan(x1) -> zero] pivot x3 (u=(ua,ub,t))
//                              : pivot x2 (a=x1, b=x3; u=(ua,t,ub))
template <typename T>
__device__ __forceinline__ void quotient3_fast_row(const T (&x)[3], T& r, T (&u)[3]) {
    using F = Fp<T>;
    const T a1 = F::abs(x[0]), a2 = F::abs(x[1]), a3 = F::abs(x[2]);
    const bool c1 = a1 > a2;
    const bool piv3 = c1 ? (a3 > a1) : (a3 >= a2);
    const bool piv1 = c1 && !piv3;
    const bool piv2 = !c1 && !piv3;
    const bool zero = !c1 && piv3 && x[2] == T(0) && !F::isnan_(x[0]);
    const T p = piv3 ? x[2] : (piv1 ? x[0] : x[1]);
    const T a = piv1 ? x[2] : x[0];
    const T b = piv2 ? x[2] : x[1];
    T t, ua, ub;
    qf_pivot(p, a, b, r, t, ua, ub);
    u[0] = piv1 ? t : ua;
    u[1] = piv2 ? t : ub;
    u[2] = piv3 ? t : (piv1 ? ua : ub);
    if (zero) {
        r = T(0); u[0] = T(0); u[1] = T(0); u[2] = T(0);
    }
}

// ---------------------------------------------------------------------------------
// Rotation matrices of quaternions (rotation.py:53-111), q = (q1, q2, q3, q4) with q4 the
// scalar part, R row-major.  Python evaluation order, one rounding per operation.  The
// reference raises ValueError for a non-finite quaternion (both forms, :44-50) and for
// the zero quaternion (general form, :63-64); the batched form writes NaN for such a row
// and reports it (return false) so the caller can raise.
// ---------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ bool rotation_unit_row(const T (&q)[4], T* R) {
    using F = Fp<T>;
    const bool ok = isfinite(q[0]) && isfinite(q[1]) && isfinite(q[2]) && isfinite(q[3]);
    const T q1 = q[0], q2 = q[1], q3 = q[2], q4 = q[3];
    const T two = T(2);
    auto sub = [](T a, T b) { return F::add(a, -b); };
    R[0] = sub(T(1), F::mul(two, F::add(F::mul(q2, q2), F::mul(q3, q3))));
    R[1] = F::mul(two, sub(F::mul(q1, q2), F::mul(q3, q4)));
    R[2] = F::mul(two, F::add(F::mul(q1, q3), F::mul(q2, q4)));
    R[3] = F::mul(two, F::add(F::mul(q1, q2), F::mul(q3, q4)));
    R[4] = sub(T(1), F::mul(two, F::add(F::mul(q1, q1), F::mul(q3, q3))));
    R[5] = F::mul(two, sub(F::mul(q2, q3), F::mul(q1, q4)));
    R[6] = F::mul(two, sub(F::mul(q1, q3), F::mul(q2, q4)));
    R[7] = F::mul(two, F::add(F::mul(q2, q3), F::mul(q1, q4)));
    R[8] = sub(T(1), F::mul(two, F::add(F::mul(q1, q1), F::mul(q2, q2))));
    if (!ok) {
#pragma unroll
        for (int k = 0; k < 9; ++k) R[k] = T(NAN);
    }
    return ok;
}

// RotationMatrix.apply (rotation.py:39-41): out_i = ((R_i0 v_0 + R_i1 v_1) + R_i2 v_2)
// with every product and sum rounded separately, as the reference's Python floats.
template <typename T>
__device__ __forceinline__ void rotation_apply_row(const T (&v)[3], const T (&R)[9], T* out) {
    using F = Fp<T>;
#pragma unroll
    for (int i = 0; i < 3; ++i)
        out[i] = F::add(F::add(F::mul(R[3 * i], v[0]), F::mul(R[3 * i + 1], v[1])), F::mul(R[3 * i + 2], v[2]));
}

// rotation_general: scale4 (exact cascade, :61-62), ss = ((q1^2+q2^2)+q3^2)+q4^2 on the
// scaled components, every entry divided by ss (:66-84).
template <typename T>
__device__ __forceinline__ bool rotation_general_row(const T (&x)[4], const KArgs<T>& ka, T* R) {
    using F = Fp<T>;
    bool ok = isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]) && isfinite(x[3]);
    // Rows that reach R are finite and nonzero; there the integer classification gives
    // the cascade's (inv, s) exactly, without its divergent branches.
    // Rejected rows (non-finite or zero) get NaN matrices below either way.
    T inv, q[4];
    ok = scale_classified<T, 4>(x, ka, inv, q) && ok;
    const T q1 = q[0], q2 = q[1], q3 = q[2], q4 = q[3];
    const T a11 = F::mul(q1, q1), a22 = F::mul(q2, q2), a33 = F::mul(q3, q3), a44 = F::mul(q4, q4);
    const T ss = F::add(F::add(F::add(a11, a22), a33), a44);
    const T two = T(2);
    auto sub = [](T a, T b) { return F::add(a, -b); };
    const Divider<T> by_ss(ss);
    R[0] = by_ss(sub(sub(F::add(a11, a44), a22), a33));
    R[1] = by_ss(F::mul(two, sub(F::mul(q1, q2), F::mul(q3, q4))));
    R[2] = by_ss(F::mul(two, F::add(F::mul(q1, q3), F::mul(q2, q4))));
    R[3] = by_ss(F::mul(two, F::add(F::mul(q1, q2), F::mul(q3, q4))));
    R[4] = by_ss(sub(sub(F::add(a22, a44), a11), a33));
    R[5] = by_ss(F::mul(two, sub(F::mul(q2, q3), F::mul(q1, q4))));
    R[6] = by_ss(F::mul(two, sub(F::mul(q1, q3), F::mul(q2, q4))));
    R[7] = by_ss(F::mul(two, F::add(F::mul(q2, q3), F::mul(q1, q4))));
    R[8] = by_ss(sub(sub(F::add(a33, a44), a11), a22));
    if (!ok) {
#pragma unroll
        for (int k = 0; k < 9; ++k) R[k] = T(NAN);
    }
    return ok;
}

}  // namespace fnb
