// bounds.cu -- error-bound sweep of normalize outputs on the GPU.
//
// Restates the acceptance checks of the reference's high-precision oracle
// (pkg/src/fastnorm/oracle.py:151-250, `_measure`) for batched outputs: for every
// finite nonzero input row x with computed (r_hat, unit) it evaluates, in double-double
// arithmetic (~106 significant bits; the reference uses 256-bit mpfr with exact
// rational sums), the true length r = ||x||, the relative / absolute length error, the
// direction error ||unit - x/r||, sin(phi) between unit and x (n = 2, 3) and the ten
// quaternion product bounds (n = 4), and counts the rows that break the paper's bounds:
//   sin-phi          |sin phi| <= 1.001 u
//   direction        ||unit - x/r|| <= (3.001 + n/2) u
//   length           |r_hat - r| <= c u r (+ alpha/2 when r < 3 nu / 2), c = 1 + n/2
//                    (3 for n = 4), applicable when (1 + c u) r <= omega; otherwise an
//                    infinite r_hat is warranted
//   quaternion       |q_i q_j - x_i x_j / r^2| <= (1.001 + 8.001 |x_i x_j| / r^2) u
//   plus nan-output, nonzero-length, finite-unit as in oracle.py:176-191.
// A check can only be misjudged when the true error lies within ~2^-100 relative of the
// bound -- far below anything a binary32/binary64 kernel produces.  Inputs are scaled by
// a power of two (exact) so the double-double sums neither overflow nor underflow.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/fastnorm_b200.h"

namespace fnb {
int set_error(int code, const char* msg);
}

namespace {

struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dadd_rn(s, -a);
    const double err = __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb));
    return {s, err};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return {s, __dadd_rn(b, -__dadd_rn(s, -a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
    dd s = two_sum(x.hi, y.hi);
    const double e = __dadd_rn(s.lo, __dadd_rn(x.lo, y.lo));
    return quick_two_sum(s.hi, e);
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
    dd p = two_prod(x.hi, y.hi);
    const double e = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(x.hi, y.lo), __dmul_rn(x.lo, y.hi)));
    return quick_two_sum(p.hi, e);
}
__device__ __forceinline__ dd dd_from(double a) { return {a, 0.0}; }
__device__ __forceinline__ dd dd_div(dd x, dd y) {
    const double q1 = __ddiv_rn(x.hi, y.hi);
    dd r = dd_sub(x, dd_mul(dd_from(q1), y));
    const double q2 = __ddiv_rn(r.hi, y.hi);
    r = dd_sub(r, dd_mul(dd_from(q2), y));
    const double q3 = __ddiv_rn(r.hi, y.hi);
    return dd_add(quick_two_sum(q1, q2), dd_from(q3));
}
__device__ __forceinline__ dd dd_sqrt(dd x) {
    if (x.hi <= 0.0) return {0.0, 0.0};
    const double q = __dsqrt_rn(x.hi);
    dd r = dd_sub(x, two_prod(q, q));
    return dd_add(dd_from(q), dd_from(__ddiv_rn(r.hi, __dmul_rn(2.0, q))));
}
__device__ __forceinline__ dd dd_abs(dd x) { return x.hi < 0.0 ? dd_neg(x) : x; }
__device__ __forceinline__ bool dd_gt(dd a, dd b) { return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo); }
__device__ __forceinline__ double dd_to(dd x) { return __dadd_rn(x.hi, x.lo); }

struct Limits {
    double u, alpha, nu, omega;
};

// counters: see fn_measure_bounds in the header
enum { V_NAN = 0, V_ZERO_R, V_FIN_UNIT, V_SIN, V_DIR, V_FIN_LEN, V_LEN_IN, V_LEN_UNDER, V_QPROD,
       C_MEASURED, C_SKIPPED, C_VIOLATING_ROWS, NCOUNT };
enum { M_REL = 0, M_ABS, M_DIR, M_SIN, NMAX };

template <typename T, int N>
__global__ void bounds_kernel(const T* __restrict__ x, const T* __restrict__ rh,
                              const T* __restrict__ uh, int64_t n, Limits lim,
                              unsigned long long* counts, unsigned long long* maxbits,
                              unsigned long long* argmax) {
    unsigned long long c[NCOUNT];
#pragma unroll
    for (int k = 0; k < NCOUNT; ++k) c[k] = 0;
    double mx[NMAX] = {0, 0, 0, 0};
    long long am[NMAX] = {-1, -1, -1, -1};
    unsigned long long first_bad = ~0ull;
    const double cn = (N == 4) ? 3.0 : 1.0 + N / 2.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double xs[N], u[N];
        bool finite = true, allzero = true;
        double m = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            xs[k] = (double)x[i * N + k];
            u[k] = (double)uh[i * N + k];
            finite = finite && isfinite(xs[k]);
            allzero = allzero && xs[k] == 0.0;
            m = fmax(m, fabs(xs[k]));
        }
        if (!finite || allzero) {
            ++c[C_SKIPPED];
            continue;
        }
        ++c[C_MEASURED];
        const double r_hat = (double)rh[i];
        bool nan_out = isnan(r_hat);
#pragma unroll
        for (int k = 0; k < N; ++k) nan_out = nan_out || isnan(u[k]);
        unsigned viol = 0;
        if (nan_out) {
            viol |= 1u << V_NAN;
        } else {
            // scale by 2^-e so that max |x_k| lies in [1, 2): exact for every component
            // that stays normal; smaller ones are negligible at double-double precision.
            int e;
            frexp(m, &e);
            e -= 1;
            dd s = {0.0, 0.0};
            double xsc[N];
#pragma unroll
            for (int k = 0; k < N; ++k) {
                xsc[k] = ldexp(xs[k], -e);
                s = dd_add(s, two_prod(xsc[k], xsc[k]));
            }
            const dd rs = dd_sqrt(s);  // true length / 2^e
            if (r_hat == 0.0) viol |= 1u << V_ZERO_R;
            bool unit_finite = true;
#pragma unroll
            for (int k = 0; k < N; ++k) unit_finite = unit_finite && isfinite(u[k]);
            if (!unit_finite) {
                viol |= 1u << V_FIN_UNIT;
            } else {
                dd d2 = {0.0, 0.0}, us = {0.0, 0.0};
                dd xbar[N];
#pragma unroll
                for (int k = 0; k < N; ++k) {
                    xbar[k] = dd_div(dd_from(xsc[k]), rs);
                    const dd diff = dd_sub(dd_from(u[k]), xbar[k]);
                    d2 = dd_add(d2, dd_mul(diff, diff));
                    us = dd_add(us, two_prod(u[k], u[k]));
                }
                const double dir_err = dd_to(dd_sqrt(d2));
                if (dir_err > (3.001 + N / 2.0) * lim.u) viol |= 1u << V_DIR;
                if (dir_err > mx[M_DIR]) { mx[M_DIR] = dir_err; am[M_DIR] = i; }
                if (N == 2 || N == 3) {
                    dd cr2;
                    if (N == 2) {
                        const dd c3 = dd_sub(two_prod(xsc[0], u[1 % N]), two_prod(xsc[1 % N], u[0]));
                        cr2 = dd_mul(c3, c3);
                    } else {
                        const dd c1 = dd_sub(two_prod(xsc[1], u[2 % N]), two_prod(xsc[2 % N], u[1]));
                        const dd c2 = dd_sub(two_prod(xsc[2 % N], u[0]), two_prod(xsc[0], u[2 % N]));
                        const dd c3 = dd_sub(two_prod(xsc[0], u[1]), two_prod(xsc[1], u[0]));
                        cr2 = dd_add(dd_add(dd_mul(c1, c1), dd_mul(c2, c2)), dd_mul(c3, c3));
                    }
                    const dd un = dd_sqrt(us);
                    double sinp;
                    if (un.hi == 0.0) {
                        sinp = INFINITY;
                    } else {
                        sinp = dd_to(dd_div(dd_sqrt(cr2), dd_mul(rs, un)));
                    }
                    if (sinp > 1.001 * lim.u) viol |= 1u << V_SIN;
                    if (sinp > mx[M_SIN]) { mx[M_SIN] = sinp; am[M_SIN] = i; }
                }
                if (N == 4) {
                    // |u_i u_j - xbar_i xbar_j| <= (1.001 + 8.001 |xbar_i xbar_j|) u
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = a; b < 4; ++b) {
                            const dd xx = dd_mul(xbar[a], xbar[b]);
                            const dd lhs = dd_abs(dd_sub(two_prod(u[a], u[b]), xx));
                            const double rhs = (1.001 + 8.001 * fabs(dd_to(xx))) * lim.u;
                            if (dd_gt(lhs, dd_from(rhs))) viol |= 1u << V_QPROD;
                        }
                }
            }
            // length, relative to the scaled true length rs = r / 2^e
            const dd cap = dd_div(dd_from(ldexp(lim.omega, -e)), dd_from(1.0 + cn * lim.u));
            const bool premise = !dd_gt(rs, cap);
            if (isinf(r_hat)) {
                if (premise) viol |= 1u << V_FIN_LEN;  // otherwise the overflow is warranted
            } else {
                // r_hat * 2^-e exactly: split the exponent so no intermediate rounds
                const dd rhs_scaled = dd_from(ldexp(ldexp(r_hat, -(e / 2)), -(e - e / 2)));
                const double abs_err_s = dd_to(dd_abs(dd_sub(rhs_scaled, rs)));  // / 2^e
                const double rel = abs_err_s / dd_to(rs);
                const double abs_err = ldexp(abs_err_s, e);
                if (rel > mx[M_REL]) { mx[M_REL] = rel; am[M_REL] = i; }
                if (abs_err > mx[M_ABS]) { mx[M_ABS] = abs_err; am[M_ABS] = i; }
                if (premise) {
                    const bool in_range = !dd_gt(dd_from(ldexp(1.5 * lim.nu, -e)), rs);
                    const double tol_s = cn * lim.u * dd_to(rs);
                    if (in_range) {
                        if (abs_err_s > tol_s) viol |= 1u << V_LEN_IN;
                    } else {
                        if (abs_err_s > tol_s + ldexp(lim.alpha, -e - 1)) viol |= 1u << V_LEN_UNDER;  // alpha/2 at scale
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k <= V_QPROD; ++k) c[k] += (viol >> k) & 1u;
        c[C_VIOLATING_ROWS] += viol != 0;
        if (viol && (unsigned long long)i < first_bad) first_bad = (unsigned long long)i;
    }
    if (first_bad != ~0ull) atomicMin(argmax + NMAX, first_bad);
    // warp-aggregate, one atomic per warp and counter
#pragma unroll
    for (int k = 0; k < NCOUNT; ++k) {
        unsigned long long v = c[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(counts + k, v);
    }
#pragma unroll
    for (int k = 0; k < NMAX; ++k) {
        if (am[k] >= 0) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(mx[k]);
            const unsigned long long old = atomicMax(maxbits + k, bits);
            if (old < bits) argmax[k] = (unsigned long long)am[k];  // best effort under races
        }
    }
}

int grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + 255) / 256;
    const int64_t cap = (int64_t)sms * 16;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" int fn_measure_bounds(int dim, int dtype, const void* x, const void* r, const void* unit,
                                 int64_t n, const double* limits, uint64_t* counts, uint64_t* maxbits,
                                 uint64_t* argmax, void* stream) {
    if (dim < 2 || dim > 4) return fnb::set_error(FN_EINVAL, "dim must be 2, 3 or 4");
    if (dtype != FN_F32 && dtype != FN_F64) return fnb::set_error(FN_EINVAL, "bad dtype");
    if (n < 0 || !limits || !counts || !maxbits || !argmax)
        return fnb::set_error(FN_EINVAL, "bad arguments");
    if (n == 0) return FN_OK;
    if (!x || !r || !unit) return fnb::set_error(FN_EINVAL, "NULL array");
    Limits lim{limits[0], limits[1], limits[2], limits[3]};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* c = reinterpret_cast<unsigned long long*>(counts);
    auto* m = reinterpret_cast<unsigned long long*>(maxbits);
    auto* a = reinterpret_cast<unsigned long long*>(argmax);
    const int g = grid_for(n);
#define FNB_B(T, D)                                                                               \
    bounds_kernel<T, D><<<g, 256, 0, s>>>(static_cast<const T*>(x), static_cast<const T*>(r),     \
                                          static_cast<const T*>(unit), n, lim, c, m, a)
    if (dtype == FN_F64) {
        if (dim == 2) FNB_B(double, 2);
        if (dim == 3) FNB_B(double, 3);
        if (dim == 4) FNB_B(double, 4);
    } else {
        if (dim == 2) FNB_B(float, 2);
        if (dim == 3) FNB_B(float, 3);
        if (dim == 4) FNB_B(float, 4);
    }
#undef FNB_B
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fnb::set_error(FN_ECUDA, cudaGetErrorString(e));
    return FN_OK;
}
