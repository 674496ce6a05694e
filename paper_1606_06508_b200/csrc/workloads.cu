// workloads.cu -- seeded synthetic workloads (BASELINE.json configs 1-5) and per-row
// validation counters, generated / counted directly in HBM.
//
// The generator is counter based: every 64-bit word is splitmix64 of
// key + (row*16 + j) * GOLDEN, with key = splitmix64(seed ^ cfg * K).  A row is a pure
// function of (cfg, seed, global row index), so a shard [row0, row0+n) generated on any
// GPU equals the same rows generated anywhere else -- including by the host-side numpy
// restatement in paper_1606_06508_b200/workloads.py (bit-identical for configs 1, 2, 4,
// 5, which use only integer ops and exact ldexp; config 3 draws normals with
// Box-Muller through libm-class log/sin/cos and matches in distribution only).
// The distributions follow BASELINE.json `configs` and SURVEY.md §8(d); DESIGN.md §6
// lists the exact recipe.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/fastnorm_b200.h"

namespace fnb {
int set_error(int code, const char* msg);
}

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += kGolden;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t word(uint64_t key, int64_t row, int j) {
    return mix64(key + ((uint64_t)row * 16u + (uint64_t)j) * kGolden);
}

// Thresholds on the top 53 bits of a word: floor(p * 2^53).
constexpr uint64_t kP1pct = 90071992547409ull;     // 0.01
constexpr uint64_t kP01pct = 9007199254740ull;     // 0.001
constexpr uint64_t kP001pct = 900719925474ull;     // 0.0001
constexpr uint64_t kP05pct = 45035996273704ull;    // 0.005

__device__ __forceinline__ double sign_of(uint64_t w) { return (w >> 63) ? -1.0 : 1.0; }
__device__ __forceinline__ double mant52(uint64_t w) {  // uniform in [1, 2)
    return 1.0 + (double)(w >> 12) * 0x1p-52;
}
__device__ __forceinline__ int uexp(uint64_t w, int lo, int span) {
    return lo + (int)((w & 0xffffffffull) % (uint64_t)span);
}

__global__ void gen_cfg1(double* x, int64_t row0, int64_t n, uint64_t key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = row0 + i;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            x[i * 3 + k] = (double)(word(key, row, k) >> 11) * 0x1p-52 - 1.0;
    }
}

__global__ void gen_cfg2(double* x, int64_t row0, int64_t n, uint64_t key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = row0 + i;
        const bool zero = (word(key, row, 15) >> 11) < kP1pct;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint64_t w = word(key, row, k);
            const double v = zero ? 0.0 : ldexp(mant52(word(key, row, 4 + k)), uexp(w, -1000, 2001));
            x[i * 2 + k] = sign_of(w) * v;
        }
    }
}

__global__ void gen_cfg3(double* x, int64_t row0, int64_t n, uint64_t key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = row0 + i;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const double u1 = (double)((word(key, row, 2 * p) >> 11) + 1) * 0x1p-53;  // (0, 1]
            const double u2 = (double)(word(key, row, 2 * p + 1) >> 11) * 0x1p-53;    // [0, 1)
            const double rad = sqrt(-2.0 * log(u1));
            double sn, cs;
            sincospi(2.0 * u2, &sn, &cs);
            x[i * 4 + 2 * p] = rad * cs;
            x[i * 4 + 2 * p + 1] = rad * sn;
        }
    }
}

__global__ void gen_cfg4(float* x, int64_t row0, int64_t n, uint64_t key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = row0 + i;
        const uint64_t v = word(key, row, 15) >> 11;
        const bool zero = v < kP01pct;
        const bool special = !zero && v < kP01pct + kP001pct;
        const int which = (int)(word(key, row, 14) % 3u);
        const int kind = (int)(word(key, row, 13) % 3u);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint64_t w = word(key, row, k);
            float out;
            if (zero) {
                out = (float)(sign_of(w) * 0.0);
            } else if (special && k == which) {
                out = kind == 0 ? __int_as_float(0x7fc00000) : (kind == 1 ? INFINITY : -INFINITY);
            } else {
                const double m = 1.0 + (double)(word(key, row, 4 + k) >> 41) * 0x1p-23;
                out = __double2float_rn(sign_of(w) * ldexp(m, uexp(w, -149, 277)));
            }
            x[i * 3 + k] = out;
        }
    }
}

__global__ void gen_cfg5(double* x, int64_t row0, int64_t n, uint64_t key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = row0 + i;
        const uint64_t v = word(key, row, 15) >> 11;
        const bool nearmax = v < kP05pct;
        const bool subn = !nearmax && v < 2 * kP05pct;
        const int which = (int)(word(key, row, 14) % 3u);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint64_t w = word(key, row, k);
            const uint64_t wm = word(key, row, 4 + k);
            double out;
            if (subn) {
                const uint64_t mant = ((wm >> 12) | (1ull << 51)) >> ((word(key, row, 8 + k) & 0xffffffffull) % 52u);
                out = __longlong_as_double((long long)((w & 0x8000000000000000ull) | mant));
            } else if (nearmax && k == which) {
                out = sign_of(w) * ldexp(mant52(wm), 1023);
            } else {
                out = sign_of(w) * ldexp(mant52(wm), uexp(w, -1020, 2041));
            }
            x[i * 3 + k] = out;
        }
    }
}

// ---- the reference's input regimes (bench.py:146-207), counter-based ----------------
// regime 0 normal    |x_k| in [tau_min, tau_max)        (1+m) 2^e, e ~ U[tmin, tmax)
//        1 subnormal |x_k| in [alpha, nu)               e ~ U[sub_min, norm_min), capped
//        2 huge      |x_k| > tau_max, sums finite        e ~ U[tmax+1, emax-1)
//        3 mixed     full range incl. subnormals         e ~ U[sub_min, emax)
//        4 unit-ish  norms within 2^-10 of one           normalised normals x (1 +- 2^-10 U)
// computed in binary64 and rounded once to the row type (single: then capped like the
// reference's clip of the subnormal regime).
template <typename T, int DIM>
__global__ void gen_regime(T* x, int64_t row0, int64_t n, uint64_t key, int regime, int tmin, int tmax,
                           int sub_min, int norm_min, int emax, double nu_minus_alpha) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = row0 + i;
        double v[DIM];
        if (regime == 4) {
            double g[4];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const double u1 = (double)((word(key, row, 2 * p) >> 11) + 1) * 0x1p-53;
                const double u2 = (double)(word(key, row, 2 * p + 1) >> 11) * 0x1p-53;
                const double rad = sqrt(-2.0 * log(u1));
                double sn, cs;
                sincospi(2.0 * u2, &sn, &cs);
                g[2 * p] = rad * cs;
                g[2 * p + 1] = rad * sn;
            }
            double ss = 0.0;
#pragma unroll
            for (int k = 0; k < DIM; ++k) ss = __dadd_rn(ss, __dmul_rn(g[k], g[k]));
            double nrm = sqrt(ss);
            if (nrm == 0.0) g[0] = 1.0;
            nrm = fmax(nrm, 2.2250738585072014e-308);
            const double u = (double)(word(key, row, 12) >> 11) * 0x1p-53;
            const double stretch = 1.0 + (u * 2.0 - 1.0) * 0x1p-10;
#pragma unroll
            for (int k = 0; k < DIM; ++k) v[k] = (g[k] / nrm) * stretch;
        } else {
            int lo, span;
            if (regime == 0) { lo = tmin; span = tmax - tmin; }
            else if (regime == 1) { lo = sub_min; span = norm_min - sub_min; }
            else if (regime == 2) { lo = tmax + 1; span = emax - 1 - (tmax + 1); }
            else { lo = sub_min; span = emax - sub_min; }
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                const uint64_t w = word(key, row, k);
                double mag = ldexp(mant52(word(key, row, 4 + k)), uexp(w, lo, span));
                if (regime == 1) mag = fmin(mag, nu_minus_alpha);
                v[k] = sign_of(w) * mag;
            }
        }
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            T out = (T)v[k];
            if (sizeof(T) == 4 && regime == 1) {
                const T cap = (T)nu_minus_alpha;
                out = out > cap ? cap : (out < -cap ? -cap : out);
            }
            x[i * DIM + k] = out;
        }
    }
}

// ---- validation counters ------------------------------------------------------------
template <typename T> struct Bits;
template <> struct Bits<double> {
    using U = unsigned long long;
    static constexpr U kAbs = 0x7fffffffffffffffull, kInf = 0x7ff0000000000000ull;
    __device__ static U of(double v) { return (U)__double_as_longlong(v); }
};
template <> struct Bits<float> {
    using U = unsigned int;
    static constexpr U kAbs = 0x7fffffffu, kInf = 0x7f800000u;
    __device__ static U of(float v) { return __float_as_uint(v); }
};

template <typename T, int N>
__global__ void row_stats_kernel(const T* __restrict__ x, int64_t n, unsigned long long* counts,
                                 typename Bits<T>::U tmin, typename Bits<T>::U tmax) {
    using B = Bits<T>;
    unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        typename B::U m = 0;
        bool nan = false, inf = false;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const typename B::U a = B::of(x[i * N + k]) & B::kAbs;
            nan |= a > B::kInf;
            inf |= a == B::kInf;
            m = a > m ? a : m;
        }
        const int cls = nan ? 0 : inf ? 1 : m == 0 ? 2 : m < tmin ? 3 : m > tmax ? 4 : 5;
#pragma unroll
        for (int k = 0; k < 6; ++k) c[k] += (cls == k);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        unsigned long long v = c[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(counts + k, v);
    }
}

int grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (n + 255) / 256;
    int64_t cap = (int64_t)sms * 16;
    return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" int fn_generate(int cfg, uint64_t seed, int64_t row0, int64_t n, void* x, void* stream) {
    if (n < 0 || row0 < 0) return fnb::set_error(FN_EINVAL, "n and row0 must be >= 0");
    if (n == 0) return FN_OK;
    if (!x) return fnb::set_error(FN_EINVAL, "x is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t key = mix64(seed ^ ((uint64_t)cfg * 0xD6E8FEB86659FD93ull));
    const int g = grid_for(n);
    switch (cfg) {
        case 1: gen_cfg1<<<g, 256, 0, s>>>(static_cast<double*>(x), row0, n, key); break;
        case 2: gen_cfg2<<<g, 256, 0, s>>>(static_cast<double*>(x), row0, n, key); break;
        case 3: gen_cfg3<<<g, 256, 0, s>>>(static_cast<double*>(x), row0, n, key); break;
        case 4: gen_cfg4<<<g, 256, 0, s>>>(static_cast<float*>(x), row0, n, key); break;
        case 5: gen_cfg5<<<g, 256, 0, s>>>(static_cast<double*>(x), row0, n, key); break;
        default: return fnb::set_error(FN_EINVAL, "cfg must be 1..5");
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fnb::set_error(FN_ECUDA, cudaGetErrorString(e));
    return FN_OK;
}

extern "C" int fn_generate_regime(int regime, int dim, int dtype, uint64_t seed, int64_t row0,
                                  int64_t n, void* x, void* stream) {
    if (regime < 0 || regime > 4) return fnb::set_error(FN_EINVAL, "regime must be 0..4");
    if (dim < 2 || dim > 4) return fnb::set_error(FN_EINVAL, "dim must be 2, 3 or 4");
    if (dtype != FN_F32 && dtype != FN_F64) return fnb::set_error(FN_EINVAL, "bad dtype");
    if (n < 0 || row0 < 0) return fnb::set_error(FN_EINVAL, "n and row0 must be >= 0");
    if (n == 0) return FN_OK;
    if (!x) return fnb::set_error(FN_EINVAL, "x is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t cfg_id = 100 + (uint64_t)regime * 16 + (uint64_t)dim * 2 + (uint64_t)dtype;
    const uint64_t key = mix64(seed ^ (cfg_id * 0xD6E8FEB86659FD93ull));
    const int g = grid_for(n);
    const bool f64 = dtype == FN_F64;
    const int tmin = f64 ? -482 : -49, tmax = f64 ? 510 : 62;
    const int sub_min = f64 ? -1074 : -149, norm_min = f64 ? -1022 : -126, emax = f64 ? 1023 : 127;
    const double cap = f64 ? (0x1p-1022 - 0x1p-1074) : (0x1p-126 - 0x1p-149);
#define FNB_GEN(T, D)                                                                             \
    gen_regime<T, D><<<g, 256, 0, s>>>(static_cast<T*>(x), row0, n, key, regime, tmin, tmax, sub_min, \
                                       norm_min, emax, cap)
    if (f64) {
        if (dim == 2) FNB_GEN(double, 2);
        if (dim == 3) FNB_GEN(double, 3);
        if (dim == 4) FNB_GEN(double, 4);
    } else {
        if (dim == 2) FNB_GEN(float, 2);
        if (dim == 3) FNB_GEN(float, 3);
        if (dim == 4) FNB_GEN(float, 4);
    }
#undef FNB_GEN
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fnb::set_error(FN_ECUDA, cudaGetErrorString(e));
    return FN_OK;
}

extern "C" int fn_row_stats(int dim, int dtype, const void* x, int64_t n, uint64_t* counts,
                            const double* ka, void* stream) {
    if (dim < 2 || dim > 4) return fnb::set_error(FN_EINVAL, "dim must be 2, 3 or 4");
    if (n < 0 || !counts || !ka) return fnb::set_error(FN_EINVAL, "bad arguments");
    if (n == 0) return FN_OK;
    if (!x) return fnb::set_error(FN_EINVAL, "x is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long* c = reinterpret_cast<unsigned long long*>(counts);
    const int g = grid_for(n);
    if (dtype == FN_F64) {
        const double a = ka[0], b = ka[1];
        const unsigned long long tmin = *reinterpret_cast<const unsigned long long*>(&a);
        const unsigned long long tmax = *reinterpret_cast<const unsigned long long*>(&b);
        const double* xd = static_cast<const double*>(x);
        if (dim == 2) row_stats_kernel<double, 2><<<g, 256, 0, s>>>(xd, n, c, tmin, tmax);
        if (dim == 3) row_stats_kernel<double, 3><<<g, 256, 0, s>>>(xd, n, c, tmin, tmax);
        if (dim == 4) row_stats_kernel<double, 4><<<g, 256, 0, s>>>(xd, n, c, tmin, tmax);
    } else if (dtype == FN_F32) {
        const float a = (float)ka[0], b = (float)ka[1];
        const unsigned int tmin = *reinterpret_cast<const unsigned int*>(&a);
        const unsigned int tmax = *reinterpret_cast<const unsigned int*>(&b);
        const float* xf = static_cast<const float*>(x);
        if (dim == 2) row_stats_kernel<float, 2><<<g, 256, 0, s>>>(xf, n, c, tmin, tmax);
        if (dim == 3) row_stats_kernel<float, 3><<<g, 256, 0, s>>>(xf, n, c, tmin, tmax);
        if (dim == 4) row_stats_kernel<float, 4><<<g, 256, 0, s>>>(xf, n, c, tmin, tmax);
    } else {
        return fnb::set_error(FN_EINVAL, "dtype must be FN_F32/FN_F64");
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fnb::set_error(FN_ECUDA, cudaGetErrorString(e));
    return FN_OK;
}
