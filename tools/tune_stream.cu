// tune_stream.cu -- tile-geometry sweep for the streaming kernel (developer tool).
//
// Times tma_stream_kernel<T, N, OP, TR, S, NT, HINTS> for several tile geometries and
// CTAs-per-SM caps on BASELINE workload rows, for the kernel families the configs use,
// plus speed-of-light references with the same traffic (cudaMemcpy D2D and a naive
// 16-byte-vector read/write kernel).
//
// Build: make -C tools tune    Run: tools/tune_stream [log2_rows=28] [reps=10] [which=all]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ws_kernel.cuh"

extern "C" int fn_generate(int cfg, uint64_t seed, int64_t row0, int64_t n, void* x, void* stream);

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

// Speed-of-light stand-ins with the record shapes of real ops but almost no arithmetic
// (op codes 90+ are tool-only): they bound what the pipeline and DRAM can do for that
// traffic mix.
namespace fnb {
template <typename T, int N> struct RowOp<T, N, 90> {  // normalize4_rotation shape: 32 B in, 112 B out
    static constexpr int W0 = 1, W1 = 4, W2 = 9;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>&, T* o0, T* o1, T* o2) {
        o0[0] = x[0];
#pragma unroll
        for (int c = 0; c < 4; ++c) o1[c] = x[c];
#pragma unroll
        for (int c = 0; c < 9; ++c) o2[c] = x[c & 3];
        return true;
    }
};
template <typename T, int N> struct RowOp<T, N, 91> {  // normalize3 shape: 24 B in, 32 B out
    static constexpr int W0 = 1, W1 = 3, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>&, T* o0, T* o1, T*) {
        o0[0] = x[0];
#pragma unroll
        for (int c = 0; c < 3; ++c) o1[c] = x[c];
        return true;
    }
};
}  // namespace fnb

using namespace fnb;

__global__ void sol_kernel(const double2* __restrict__ x, int64_t npairs, double2* __restrict__ r,
                           double2* __restrict__ u) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npairs;
         i += (int64_t)gridDim.x * blockDim.x) {
        double2 a = __ldcs(x + 3 * i), b = __ldcs(x + 3 * i + 1), c = __ldcs(x + 3 * i + 2);
        __stcs(r + i, make_double2(a.x, b.y));
        __stcs(u + 3 * i, a);
        __stcs(u + 3 * i + 1, b);
        __stcs(u + 3 * i + 2, c);
    }
}

struct Bufs {
    void *x, *h, *b, *q;
    int64_t n;
};

template <typename T>
KArgs<T> make_ka() {
    KArgs<T> ka;
    memset(&ka, 0, sizeof(ka));
    const bool f = sizeof(T) == 4;
    ka.tau_min = (T)(f ? 0x1p-49 : 0x1p-482);
    ka.tau_max = (T)(f ? 0x1p62 : 0x1p510);
    ka.sigma_min = (T)(f ? 0x1p100 : 0x1p592);
    ka.sigma_max = (T)(f ? 0x1p-66 : 0x1p-514);
    ka.inv_min = (T)(f ? 0x1p-100 : 0x1p-592);
    ka.inv_max = (T)(f ? 0x1p66 : 0x1p514);
    memcpy(&ka.tau_min_bits, &ka.tau_min, sizeof(T));
    memcpy(&ka.tau_max_bits, &ka.tau_max, sizeof(T));
    const double rot[9] = {0.36, 0.48, -0.8, -0.8, 0.6, 0.0, 0.48, 0.64, 0.6};
    for (int k = 0; k < 9; ++k) ka.rot[k] = (T)rot[k];
    return ka;
}

template <typename T, int N, int OP, int TR, int S, int NT, int H, int OB = OutTiles<OP>::value>
float time_variant(const Bufs& b, int cps, int reps, int sms, int* occ_out) {
    using L = TileLayout<T, N, OP, TR, S, OB>;
    auto kern = tma_stream_kernel<T, N, OP, TR, S, NT, H, OB>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemBytes));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, L::kSmemBytes));
    *occ_out = occ;
    const int per = cps > 0 ? std::min(cps, occ) : occ;
    const int64_t ntiles = b.n / TR;
    const int grid = (int)std::min<int64_t>((int64_t)per * sms, ntiles);
    const KArgs<T> ka = make_ka<T>();
    const T* x = (const T*)b.x;
    T *h = (T*)b.h, *bd = (T*)b.b, *q = (T*)b.q;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 2; ++i) kern<<<grid, NT, L::kSmemBytes>>>(x, (const T*)b.b, b.n, h, bd, q, ka);
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) kern<<<grid, NT, L::kSmemBytes>>>(x, (const T*)b.b, b.n, h, bd, q, ka);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaEventDestroy(e0));
    CK(cudaEventDestroy(e1));
    return ms / reps;
}

// The warp-specialised kernel (NT compute threads + a producer warp); H is unused.
template <typename T, int N, int OP, int TR, int S, int NT, int H>
float time_variant_ws(const Bufs& b, int cps, int reps, int sms, int* occ_out) {
    using L = TileLayout<T, N, OP, TR, S>;
    auto kern = tma_ws_kernel<T, N, OP, TR, S, NT>;
    const int smem = L::kSmemBytes + (S + 2 * L::OB) * 8;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT + 32, smem));
    *occ_out = occ;
    const int per = cps > 0 ? std::min(cps, occ) : occ;
    const int64_t ntiles = b.n / TR;
    const int grid = (int)std::min<int64_t>((int64_t)per * sms, ntiles);
    const KArgs<T> ka = make_ka<T>();
    const T* x = (const T*)b.x;
    T *h = (T*)b.h, *bd = (T*)b.b, *q = (T*)b.q;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 2; ++i) kern<<<grid, NT + 32, smem>>>(x, (const T*)b.b, b.n, h, bd, q, ka);
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) kern<<<grid, NT + 32, smem>>>(x, (const T*)b.b, b.n, h, bd, q, ka);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaEventDestroy(e0));
    CK(cudaEventDestroy(e1));
    return ms / reps;
}

struct Variant {
    std::string fam;
    int cfg, tr, s, nt, h, cps, bytes_per_row;
    float (*fn)(const Bufs&, int, int, int, int*);
    std::vector<float> ms;
    int occ = 0;
};

template <typename T, int N, int OP>
constexpr int row_bytes() {
    using Op = RowOp<T, N, OP>;
    return (int)sizeof(T) * (N + Op::W0 + Op::W1 + Op::W2);
}

#define V(FAM, CFG, T, N, OP, TR, S, NT, H, CPS)                                         \
    Variant{FAM, CFG, TR, S, NT, H, CPS, row_bytes<T, N, OP>(),                          \
            &time_variant<T, N, OP, TR, S, NT, H>, {}, 0}
// warp-specialised kernel (family name gets a _ws suffix)
#define VW(FAM, CFG, T, N, OP, TR, S, NT, CPS)                                           \
    Variant{FAM "_ws", CFG, TR, S, NT, 0, CPS, row_bytes<T, N, OP>(),                    \
            &time_variant_ws<T, N, OP, TR, S, NT, 0>, {}, 0}
// same with OB output staging tiles (reported in the HINTS column as 10*OB + HINTS)
#define VO(FAM, CFG, T, N, OP, TR, S, NT, H, CPS, OB)                                    \
    Variant{FAM, CFG, TR, S, NT, 10 * OB + H, CPS, row_bytes<T, N, OP>(),                \
            &time_variant<T, N, OP, TR, S, NT, H, OB>, {}, 0}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 28;
    const int reps = argc > 2 ? atoi(argv[2]) : 10;
    const std::string which = argc > 3 ? argv[3] : "all";
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int64_t n = (int64_t)1 << lg;
    Bufs b;
    b.n = n;
    // sized for the largest records (4 x f64 in; head / extra up to a 3x3 f64 matrix)
    CK(cudaMalloc(&b.x, n * 32));
    CK(cudaMalloc(&b.h, n * 72));
    CK(cudaMalloc(&b.b, n * 32));
    CK(cudaMalloc(&b.q, n * 72));
    printf("rows=%lld sms=%d\n", (long long)n, sms);

    if (which == "all" || which == "sol") {
        CK(fn_generate(5, 5, 0, n, b.x, nullptr) == 0 ? cudaSuccess : cudaErrorUnknown);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        for (int g : {sms * 8, sms * 32}) {
            for (int i = 0; i < 2; ++i)
                sol_kernel<<<g, 256>>>((const double2*)b.x, n / 2, (double2*)b.h, (double2*)b.b);
            CK(cudaEventRecord(e0));
            for (int i = 0; i < reps; ++i)
                sol_kernel<<<g, 256>>>((const double2*)b.x, n / 2, (double2*)b.h, (double2*)b.b);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            ms /= reps;
            printf("sol_vec16_f64x3,grid=%d,ms=%.4f,GBps=%.1f\n", g, ms, n * 56.0 / (ms * 1e-3) / 1e9);
        }
        for (int i = 0; i < 2; ++i) CK(cudaMemcpy(b.b, b.x, n * 24, cudaMemcpyDeviceToDevice));
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) CK(cudaMemcpy(b.b, b.x, n * 24, cudaMemcpyDeviceToDevice));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= reps;
        printf("memcpy_d2d,bytes=%lld,ms=%.4f,GBps(r+w)=%.1f\n", (long long)(n * 24), ms,
               n * 48.0 / (ms * 1e-3) / 1e9);
        fflush(stdout);
    }

    std::vector<Variant> vs;
    if (which == "all" || which == "f64x3") {
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 0, 2));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 3, 256, 0, 2));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 5, 256, 0, 2));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 128, 4, 128, 0, 4));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 512, 2, 256, 0, 2));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 512, 3, 512, 0, 1));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 1024, 3, 256, 3, 1));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 128, 0, 2));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 512, 0, 2));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 4, 256, 0, 2));
        vs.push_back(V("scale3_f64", 5, double, 3, FN_OP_SCALE, 256, 4, 256, 0, 2));
        vs.push_back(V("quotient3_f64", 5, double, 3, FN_OP_QUOTIENT, 256, 4, 256, 0, 2));
        vs.push_back(V("quotient3_f64", 5, double, 3, FN_OP_QUOTIENT, 256, 4, 256, 0, 4));
        vs.push_back(V("quotient3_fast_f64", 5, double, 3, FN_OP_QUOTIENT3_FAST, 256, 4, 256, 0, 2));
        vs.push_back(V("quotient3_fast_f64", 5, double, 3, FN_OP_QUOTIENT3_FAST, 256, 4, 256, 0, 4));
        vs.push_back(V("naive3_f64", 5, double, 3, FN_OP_NAIVE, 256, 4, 256, 0, 2));
    }
    if (which == "all" || which == "div") {
        vs.push_back(V("quotient3_f64", 1, double, 3, FN_OP_QUOTIENT, 256, 4, 256, 0, 4));
        vs.push_back(V("quotient3_fast_f64", 1, double, 3, FN_OP_QUOTIENT3_FAST, 256, 4, 256, 0, 4));
        vs.push_back(V("naive3_f64", 1, double, 3, FN_OP_NAIVE, 256, 4, 256, 0, 4));
        vs.push_back(V("quotient3_f64", 5, double, 3, FN_OP_QUOTIENT, 256, 4, 256, 0, 4));
        vs.push_back(V("quotient3_fast_f64", 5, double, 3, FN_OP_QUOTIENT3_FAST, 256, 4, 256, 0, 4));
        vs.push_back(V("naive3_f64", 5, double, 3, FN_OP_NAIVE, 256, 4, 256, 0, 4));
        vs.push_back(V("quotient2_f64", 2, double, 2, FN_OP_QUOTIENT, 256, 4, 256, 0, 4));
        vs.push_back(V("quotient4_f64", 3, double, 4, FN_OP_QUOTIENT, 256, 4, 256, 0, 4));
        vs.push_back(V("quotient3_f32", 4, float, 3, FN_OP_QUOTIENT, 512, 4, 256, 0, 4));
        vs.push_back(V("quotient3_fast_f32", 4, float, 3, FN_OP_QUOTIENT3_FAST, 512, 4, 256, 0, 4));
        vs.push_back(V("naive3_f32", 4, float, 3, FN_OP_NAIVE, 512, 4, 256, 0, 4));
    }
    if (which == "all" || which == "norm") {
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 4, 256, 0, 2));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 4, 256, 0, 3));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 4, 256, 0, 4));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 6, 256, 0, 2));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 512, 4, 256, 0, 2));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 512, 3, 512, 0, 2));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 8, 256, 0, 2));
        vs.push_back(V("norm2_f64", 2, double, 2, FN_OP_NORM, 512, 4, 256, 0, 2));
        vs.push_back(V("norm2_f64", 2, double, 2, FN_OP_NORM, 512, 4, 256, 0, 3));
        vs.push_back(V("norm4_f64", 3, double, 4, FN_OP_NORM, 256, 3, 256, 0, 2));
        vs.push_back(V("norm4_f64", 3, double, 4, FN_OP_NORM, 256, 4, 256, 0, 3));
        vs.push_back(V("normalize4_f64", 3, double, 4, FN_OP_NORMALIZE, 256, 3, 256, 0, 2));
        vs.push_back(V("normalize4_f64", 3, double, 4, FN_OP_NORMALIZE, 128, 4, 128, 0, 4));
        vs.push_back(V("normalize4_f64", 3, double, 4, FN_OP_NORMALIZE, 256, 2, 256, 0, 3));
        vs.push_back(V("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 512, 4, 256, 0, 2));
        vs.push_back(V("normalize2_f32", 4, float, 2, FN_OP_NORMALIZE, 512, 4, 256, 0, 2));
        vs.push_back(V("normalize2_f32", 4, float, 2, FN_OP_NORMALIZE, 1024, 4, 256, 0, 2));
        vs.push_back(V("normalize4_f32", 4, float, 4, FN_OP_NORMALIZE, 512, 3, 256, 0, 2));
        vs.push_back(V("normalize4_f32", 4, float, 4, FN_OP_NORMALIZE, 256, 4, 256, 0, 2));
    }
    if (which == "all" || which == "copy") {
        vs.push_back(V("copy_nrot_shape", 3, double, 4, 90, 128, 3, 256, 0, 2));
        vs.push_back(V("copy_nrot_shape", 3, double, 4, 90, 256, 2, 256, 0, 2));
        vs.push_back(V("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 3, 256, 0, 2));
        vs.push_back(V("copy_n3_shape", 5, double, 3, 91, 256, 4, 256, 0, 2));
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 0, 2));
    }
    if (which == "all" || which == "rot") {
        vs.push_back(V("rotation_unit_f64", 3, double, 4, FN_OP_ROT_UNIT, 256, 3, 256, 0, 2));
        vs.push_back(V("rotation_general_f64", 3, double, 4, FN_OP_ROT_GENERAL, 256, 3, 256, 0, 2));
        vs.push_back(V("rotation_general_f64", 3, double, 4, FN_OP_ROT_GENERAL, 256, 3, 256, 0, 4));
        vs.push_back(V("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 3, 256, 0, 2));
        vs.push_back(V("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 4, 128, 0, 3));
        vs.push_back(VO("rotation_unit_f64", 3, double, 4, FN_OP_ROT_UNIT, 256, 3, 256, 0, 2, 4));
        vs.push_back(VO("rotation_unit_f64", 3, double, 4, FN_OP_ROT_UNIT, 256, 3, 256, 0, 2, 5));
        vs.push_back(VO("rotation_unit_f64", 3, double, 4, FN_OP_ROT_UNIT, 128, 3, 128, 0, 3, 4));
        vs.push_back(VO("rotation_unit_f64", 3, double, 4, FN_OP_ROT_UNIT, 128, 3, 128, 0, 3, 6));
        vs.push_back(VO("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 256, 3, 256, 0, 2, 3));
        vs.push_back(VO("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 256, 2, 256, 0, 2, 3));
        vs.push_back(VO("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 4, 256, 0, 2, 3));
        vs.push_back(VO("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 3, 256, 0, 3, 3));
        vs.push_back(VO("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 3, 256, 0, 2, 4));
        vs.push_back(VO("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 3, 256, 0, 2, 5));
        vs.push_back(VO("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 0, 2, 3));
        vs.push_back(VO("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 0, 2, 4));
        vs.push_back(VO("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 0, 2, 5));
        vs.push_back(V("rot_apply_f64", 5, double, 3, FN_OP_ROT_APPLY, 256, 4, 256, 0, 2));
        vs.push_back(V("rot_apply_f64", 5, double, 3, FN_OP_ROT_APPLY, 256, 4, 256, 0, 3));
        vs.push_back(V("rot_apply_f64", 5, double, 3, FN_OP_ROT_APPLY, 256, 4, 256, 0, 4));
    }
    if (which == "all" || which == "f64x2") {
        vs.push_back(V("normalize2_f64", 2, double, 2, FN_OP_NORMALIZE, 512, 4, 256, 0, 2));
        vs.push_back(V("normalize2_f64", 2, double, 2, FN_OP_NORMALIZE, 256, 4, 256, 0, 2));
        vs.push_back(V("normalize2_f64", 2, double, 2, FN_OP_NORMALIZE, 512, 2, 256, 0, 3));
        vs.push_back(V("normalize2_f64", 2, double, 2, FN_OP_NORMALIZE, 256, 4, 256, 0, 3));
        vs.push_back(V("quotient2_f64", 2, double, 2, FN_OP_QUOTIENT, 512, 4, 256, 0, 2));
        vs.push_back(V("quotient2_f64", 2, double, 2, FN_OP_QUOTIENT, 256, 4, 256, 0, 4));
    }
    if (which == "all" || which == "f64x4") {
        vs.push_back(V("normalize4_sq_f64", 3, double, 4, FN_OP_NORMALIZE_SQ, 256, 4, 256, 0, 2));
        vs.push_back(V("normalize4_sq_f64", 3, double, 4, FN_OP_NORMALIZE_SQ, 128, 4, 128, 0, 4));
        vs.push_back(V("normalize4_sq_f64", 3, double, 4, FN_OP_NORMALIZE_SQ, 256, 3, 256, 0, 2));
        vs.push_back(V("normalize4_sq_f64", 3, double, 4, FN_OP_NORMALIZE_SQ, 128, 4, 256, 0, 2));
        vs.push_back(V("normalize4_f64", 3, double, 4, FN_OP_NORMALIZE, 256, 4, 256, 0, 2));
        vs.push_back(V("quotient4_f64", 3, double, 4, FN_OP_QUOTIENT, 256, 4, 256, 0, 2));
    }
    if (which == "all" || which == "f32x3") {
        vs.push_back(V("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 512, 4, 256, 0, 2));
        vs.push_back(V("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 256, 4, 256, 0, 2));
        vs.push_back(V("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 512, 4, 256, 0, 3));
        vs.push_back(V("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 1024, 4, 256, 0, 2));
        vs.push_back(V("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 1024, 2, 256, 0, 2));
        vs.push_back(V("quotient3_f32", 4, float, 3, FN_OP_QUOTIENT, 512, 4, 256, 0, 2));
    }
    if (which == "all" || which == "ws") {
        vs.push_back(V("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 0, 2));
        vs.push_back(VW("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 2));
        vs.push_back(VW("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 3, 256, 2));
        vs.push_back(VW("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 128, 2));
        vs.push_back(VW("normalize3_f64", 5, double, 3, FN_OP_NORMALIZE, 256, 4, 256, 3));
        vs.push_back(V("normalize2_f64", 2, double, 2, FN_OP_NORMALIZE, 512, 4, 256, 0, 2));
        vs.push_back(VW("normalize2_f64", 2, double, 2, FN_OP_NORMALIZE, 512, 4, 256, 2));
        vs.push_back(V("normalize4_sq_f64", 3, double, 4, FN_OP_NORMALIZE_SQ, 256, 3, 256, 0, 2));
        vs.push_back(VW("normalize4_sq_f64", 3, double, 4, FN_OP_NORMALIZE_SQ, 256, 3, 256, 2));
        vs.push_back(V("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 512, 4, 256, 0, 2));
        vs.push_back(VW("normalize3_f32", 4, float, 3, FN_OP_NORMALIZE, 512, 4, 256, 2));
        vs.push_back(V("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 4, 256, 0, 4));
        vs.push_back(VW("norm3_f64", 5, double, 3, FN_OP_NORM, 256, 4, 256, 4));
        vs.push_back(V("quotient3_f64", 5, double, 3, FN_OP_QUOTIENT, 256, 4, 256, 0, 8));
        vs.push_back(VW("quotient3_f64", 5, double, 3, FN_OP_QUOTIENT, 256, 4, 256, 8));
        vs.push_back(V("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 3, 256, 0, 2));
        vs.push_back(VW("normalize4_rot_f64", 3, double, 4, FN_OP_NORMALIZE_ROT, 128, 3, 256, 2));
    }
    // generate the input each variant family needs (configs 2..5) once per group
    int cur_cfg = -1;
    const int rounds = 3;
    for (int rd = 0; rd < rounds; ++rd) {
        for (auto& v : vs) {
            if (v.cfg != cur_cfg) {
                CK(fn_generate(v.cfg, v.cfg, 0, n, b.x, nullptr) == 0 ? cudaSuccess : cudaErrorUnknown);
                CK(cudaDeviceSynchronize());
                cur_cfg = v.cfg;
            }
            v.ms.push_back(v.fn(b, v.cps, reps, sms, &v.occ));
        }
    }
    for (auto& v : vs) {
        std::vector<float> m = v.ms;
        std::sort(m.begin(), m.end());
        const float med = m[m.size() / 2];
        printf("%s,cfg=%d,TR=%d,S=%d,NT=%d,HINTS=%d,occ=%d,ctas_per_sm=%d,B/row=%d,ms_med=%.4f,"
               "GBps_med=%.1f,GBps_best=%.1f,Gvecps_med=%.2f\n",
               v.fam.c_str(), v.cfg, v.tr, v.s, v.nt, v.h, v.occ, v.cps == 0 ? v.occ : std::min(v.cps, v.occ),
               v.bytes_per_row, med, n * (double)v.bytes_per_row / (med * 1e-3) / 1e9,
               n * (double)v.bytes_per_row / (m[0] * 1e-3) / 1e9, n / (med * 1e-3) / 1e9);
    }
    return 0;
}
