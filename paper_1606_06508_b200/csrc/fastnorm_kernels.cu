// fastnorm_kernels.cu -- sm_100a kernels and the C ABI (include/fastnorm_b200.h).
//
// Memory path.  Rows are AoS records of n = 2/3/4 elements (16/24/32 B
// for f64, 8/12/16 B for f32); a stride-3 record cannot be loaded coalesced by a
// thread-per-row mapping.  The streaming kernel therefore moves whole tiles of TR
// rows with the Blackwell bulk-copy engine (TMA, `cp.async.bulk`):
//   * persistent CTAs (grid = resident CTAs per SM x 148), tiles dealt round-robin;
//   * an S-stage ring of input tiles in shared memory, each completed on an mbarrier
//     with expect_tx (one elected thread issues, every thread waits);
//   * per-row arithmetic in registers (fastnorm_math.cuh), results written to one of
//     three output staging tiles in shared memory;
//   * one elected thread issues bulk stores (shared -> global) of the r / unit / sq
//     tiles in one bulk group; `wait_group.read 1` right after the commit guarantees
//     that the staging tile written two iterations later has been drained.
// Every HBM byte is touched exactly once, in 16-byte-aligned bulk transactions.
// Rows past the last full tile (and arrays that are not 16-byte aligned) use a plain
// thread-per-row kernel with the same row arithmetic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fastnorm_math.cuh"
#include "../../include/fastnorm_b200.h"

#ifndef FNB_BUILD_FLAGS
#define FNB_BUILD_FLAGS "nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -ftz=false -prec-div=true -prec-sqrt=true"
#endif

namespace fnb {

// ---------------------------------------------------------------------------------
// Error slot (per host thread).
// ---------------------------------------------------------------------------------
static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int set_error(int code, const char* msg) { return fail(code, msg); }

static int cuda_fail(cudaError_t e, const char* where) {
    return fail(FN_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------------
// Row operations: one functor per kernel family.
// ---------------------------------------------------------------------------------
template <typename T, int N, int OP> struct RowOp;

template <typename T, int N> struct RowOp<T, N, FN_OP_NORMALIZE> {
    static constexpr bool kBody = true, kSq = false;
    __device__ __forceinline__ static void apply(const T (&x)[N], const KArgs<T>& ka, T& head,
                                                 T (&body)[N], T& sq) {
        normalize_row<T, N, false>(x, ka, head, body, sq);
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_NORMALIZE_SQ> {
    static constexpr bool kBody = true, kSq = true;
    __device__ __forceinline__ static void apply(const T (&x)[N], const KArgs<T>& ka, T& head,
                                                 T (&body)[N], T& sq) {
        normalize_row<T, N, true>(x, ka, head, body, sq);
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_NORM> {
    static constexpr bool kBody = false, kSq = false;
    __device__ __forceinline__ static void apply(const T (&x)[N], const KArgs<T>& ka, T& head,
                                                 T (&)[N], T&) {
        head = norm_row<T, N>(x, ka);
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_SCALE> {
    static constexpr bool kBody = true, kSq = false;
    __device__ __forceinline__ static void apply(const T (&x)[N], const KArgs<T>& ka, T& head,
                                                 T (&body)[N], T&) {
        scale_row(x, ka, head, body);
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_NAIVE> {
    static constexpr bool kBody = true, kSq = false;
    __device__ __forceinline__ static void apply(const T (&x)[N], const KArgs<T>&, T& head,
                                                 T (&body)[N], T&) {
        naive_row<T, N>(x, head, body);
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_QUOTIENT> {
    static constexpr bool kBody = true, kSq = false;
    __device__ __forceinline__ static void apply(const T (&x)[N], const KArgs<T>&, T& head,
                                                 T (&body)[N], T&) {
        quotient_row<T, N>(x, head, body);
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_QUOTIENT3_FAST> {
    static_assert(N == 3, "quotient3_fast is 3-D only (_backend.py:96-98)");
    static constexpr bool kBody = true, kSq = false;
    __device__ __forceinline__ static void apply(const T (&x)[N], const KArgs<T>&, T& head,
                                                 T (&body)[N], T&) {
        quotient3_fast_row<T>(x, head, body);
    }
};

// One row through global memory (tails, unaligned arrays, tiny batches).
template <typename T, int N, int OP>
__device__ __forceinline__ void row_global(const T* __restrict__ x, int64_t i, T* __restrict__ head,
                                           T* __restrict__ body, T* __restrict__ sq,
                                           const KArgs<T>& ka) {
    using Op = RowOp<T, N, OP>;
    T xr[N], b[N], h, q;
#pragma unroll
    for (int c = 0; c < N; ++c) xr[c] = __ldg(x + i * N + c);
    Op::apply(xr, ka, h, b, q);
    head[i] = h;
    if (Op::kBody) {
#pragma unroll
        for (int c = 0; c < N; ++c) body[i * N + c] = b[c];
    }
    if (Op::kSq) sq[i] = q;
}

template <typename T, int N, int OP>
__global__ void __launch_bounds__(256) direct_kernel(const T* __restrict__ x, int64_t nrows,
                                                     T* __restrict__ head, T* __restrict__ body,
                                                     T* __restrict__ sq, KArgs<T> ka) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += stride)
        row_global<T, N, OP>(x, i, head, body, sq, ka);
}

// ---------------------------------------------------------------------------------
// Bulk-copy (TMA) primitives.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// global -> shared bulk copy, completion counted on the mbarrier; streaming input is
// read exactly once, so it is marked evict-first in L2.
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                          uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_addr(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int kPending>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kPending) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Tile geometry per (T, N): ~6-8 KiB of input per stage, a multiple of 16 rows.
template <typename T, int N> struct Tile {
    static constexpr int kRows = (N * (int)sizeof(T) <= 16) ? 512 : 256;
    static constexpr int kStages = 4;
    static constexpr int kOutBufs = 3;
    static constexpr int kThreads = 256;
};

template <typename T, int N, int OP> struct TileLayout {
    using Op = RowOp<T, N, OP>;
    static constexpr int TR = Tile<T, N>::kRows;
    static constexpr int S = Tile<T, N>::kStages;
    static constexpr int OB = Tile<T, N>::kOutBufs;
    static constexpr int kInBytes = TR * N * (int)sizeof(T);
    static constexpr int kHeadBytes = TR * (int)sizeof(T);
    static constexpr int kBodyBytes = Op::kBody ? TR * N * (int)sizeof(T) : 0;
    static constexpr int kSqBytes = Op::kSq ? TR * (int)sizeof(T) : 0;
    static constexpr int kOutBytes = kHeadBytes + kBodyBytes + kSqBytes;
    static constexpr int kSmemBytes = S * kInBytes + OB * kOutBytes + S * 8;
    static_assert(kInBytes % 16 == 0 && kHeadBytes % 16 == 0, "bulk copies need 16 B multiples");
};

template <typename T, int N, int OP>
__global__ void __launch_bounds__(256) tma_stream_kernel(const T* __restrict__ x, int64_t nrows,
                                                         T* __restrict__ head, T* __restrict__ body,
                                                         T* __restrict__ sq, KArgs<T> ka) {
    using L = TileLayout<T, N, OP>;
    using Op = typename L::Op;
    constexpr int TR = L::TR, S = L::S, OB = L::OB;
    constexpr int NT = Tile<T, N>::kThreads;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* s_in = smem;
    unsigned char* s_out = smem + S * L::kInBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(s_out + OB * L::kOutBytes);

    const int64_t ntiles = nrows / TR;
    const int64_t my_tiles =
        ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
    const bool leader = threadIdx.x == 0;
    uint64_t policy = 0;

    if (leader) {
        policy = policy_evict_first();
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (leader) {
        for (int64_t k = 0; k < my_tiles && k < S; ++k) {
            const int64_t tile = (int64_t)blockIdx.x + k * gridDim.x;
            mbar_arrive_expect_tx(&full[k], L::kInBytes);
            bulk_load(s_in + k * L::kInBytes, x + tile * TR * N, L::kInBytes, &full[k], policy);
        }
    }

    for (int64_t k = 0; k < my_tiles; ++k) {
        const int s = (int)(k % S);
        const uint32_t parity = (uint32_t)((k / S) & 1);
        const int ob = (int)(k % OB);
        const int64_t tile = (int64_t)blockIdx.x + k * gridDim.x;
        mbar_wait(&full[s], parity);

        const T* tin = reinterpret_cast<const T*>(s_in + s * L::kInBytes);
        T* th = reinterpret_cast<T*>(s_out + ob * L::kOutBytes);
        T* tb = th + TR;
        T* tq = tb + (Op::kBody ? TR * N : 0);
#pragma unroll
        for (int j = threadIdx.x; j < TR; j += NT) {
            T xr[N], b[N], h, q;
#pragma unroll
            for (int c = 0; c < N; ++c) xr[c] = tin[j * N + c];
            Op::apply(xr, ka, h, b, q);
            th[j] = h;
            if (Op::kBody) {
#pragma unroll
                for (int c = 0; c < N; ++c) tb[j * N + c] = b[c];
            }
            if (Op::kSq) tq[j] = q;
        }
        fence_proxy_async_smem();  // generic-proxy smem traffic -> visible to bulk copies
        __syncthreads();
        if (leader) {
            const int64_t row0 = tile * TR;
            bulk_store(head + row0, th, L::kHeadBytes);
            if (Op::kBody) bulk_store(body + row0 * N, tb, L::kBodyBytes);
            if (Op::kSq) bulk_store(sq + row0, tq, L::kSqBytes);
            bulk_commit();
            if (k + S < my_tiles) {
                const int64_t nt = tile + (int64_t)S * gridDim.x;
                mbar_arrive_expect_tx(&full[s], L::kInBytes);
                bulk_load(s_in + s * L::kInBytes, x + nt * TR * N, L::kInBytes, &full[s], policy);
            }
            // The staging tile written at iteration k+1 was last drained by group k-2.
            bulk_wait_read<1>();
        }
    }

    // Rows after the last full tile: plain per-thread path in the last CTA.
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t i = ntiles * TR + threadIdx.x; i < nrows; i += NT)
            row_global<T, N, OP>(x, i, head, body, sq, ka);
    }
    if (leader) bulk_wait_all();
}

// ---------------------------------------------------------------------------------
// Launch plumbing.
// ---------------------------------------------------------------------------------
struct DeviceInfo {
    int sms = 0;
    bool ok = false;
};
static std::mutex g_dev_mu;
static std::vector<DeviceInfo> g_dev;

static int device_sms(int dev) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
    if (!g_dev[dev].ok) {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 148;
        g_dev[dev].sms = sms;
        g_dev[dev].ok = true;
    }
    return g_dev[dev].sms;
}

// Per-instantiation occupancy (computed once per process and device).
template <typename T, int N, int OP> struct TmaLaunch {
    static int blocks_per_sm(int dev) {
        static std::mutex mu;
        static int cache[64] = {0};
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 0 || dev >= 64) return 1;
        if (cache[dev] == 0) {
            using L = TileLayout<T, N, OP>;
            auto kern = tma_stream_kernel<T, N, OP>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemBytes);
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Tile<T, N>::kThreads,
                                                              L::kSmemBytes) != cudaSuccess ||
                nb < 1)
                nb = 1;
            cache[dev] = nb;
        }
        return cache[dev];
    }
};

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static int g_force_direct = -1;  // FASTNORM_B200_PATH=direct forces the per-row kernel

static bool force_direct() {
    if (g_force_direct < 0) {
        const char* e = getenv("FASTNORM_B200_PATH");
        g_force_direct = (e && strcmp(e, "direct") == 0) ? 1 : 0;
    }
    return g_force_direct == 1;
}

template <typename T, int N, int OP>
static int launch(const void* xv, int64_t n, void* hv, void* bv, void* qv, const KArgs<T>& ka,
                  cudaStream_t stream) {
    using L = TileLayout<T, N, OP>;
    const T* x = static_cast<const T*>(xv);
    T* head = static_cast<T*>(hv);
    T* body = static_cast<T*>(bv);
    T* sq = static_cast<T*>(qv);
    if (n == 0) return FN_OK;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const int sms = device_sms(dev);
    const bool aligned = aligned16(x) && aligned16(head) && (!L::Op::kBody || aligned16(body)) &&
                         (!L::Op::kSq || aligned16(sq));
    if (aligned && !force_direct() && n >= (int64_t)L::TR) {
        const int64_t ntiles = n / L::TR;
        const int64_t resident = (int64_t)TmaLaunch<T, N, OP>::blocks_per_sm(dev) * sms;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, resident));
        tma_stream_kernel<T, N, OP>
            <<<grid, Tile<T, N>::kThreads, L::kSmemBytes, stream>>>(x, n, head, body, sq, ka);
    } else {
        const int64_t want = (n + 255) / 256;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
        direct_kernel<T, N, OP><<<grid, 256, 0, stream>>>(x, n, head, body, sq, ka);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return FN_OK;
}

template <typename T>
static int make_kargs(const double* ka, bool needed, KArgs<T>& out) {
    memset(&out, 0, sizeof(out));
    if (!needed) return FN_OK;
    if (!ka) return fail(FN_EINVAL, "ka is NULL for a scaling kernel");
    // The reference casts each double to the kernel's precision (_kernels.pyx:526-527).
    out.tau_min = (T)ka[0];
    out.tau_max = (T)ka[1];
    out.sigma_min = (T)ka[2];
    out.sigma_max = (T)ka[3];
    out.inv_min = (T)ka[4];
    out.inv_max = (T)ka[5];
    // Integer band test == IEEE compare only for +0 <= tau (not NaN); see DESIGN.md §3.
    if (!(out.tau_min >= (T)0) || !(out.tau_max >= (T)0) || std::signbit(out.tau_min) ||
        std::signbit(out.tau_max))
        return fail(FN_EINVAL, "tau_min/tau_max must be non-negative and not NaN");
    memcpy(&out.tau_min_bits, &out.tau_min, sizeof(T));
    memcpy(&out.tau_max_bits, &out.tau_max, sizeof(T));
    return FN_OK;
}

template <typename T, int OP>
static int dispatch_dim(int dim, const void* x, int64_t n, void* h, void* b, void* q,
                        const KArgs<T>& ka, cudaStream_t s) {
    switch (dim) {
        case 2: return launch<T, 2, OP>(x, n, h, b, q, ka, s);
        case 3: return launch<T, 3, OP>(x, n, h, b, q, ka, s);
        case 4: return launch<T, 4, OP>(x, n, h, b, q, ka, s);
        default: return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    }
}

template <typename T>
static int dispatch(int op, int dim, const void* x, int64_t n, void* h, void* b, void* q,
                    const double* kad, cudaStream_t s) {
    const bool scaling = op == FN_OP_SCALE || op == FN_OP_NORMALIZE || op == FN_OP_NORM ||
                         op == FN_OP_NORMALIZE_SQ;
    KArgs<T> ka;
    int rc = make_kargs<T>(kad, scaling, ka);
    if (rc != FN_OK) return rc;
    switch (op) {
        case FN_OP_SCALE: return dispatch_dim<T, FN_OP_SCALE>(dim, x, n, h, b, q, ka, s);
        case FN_OP_NORMALIZE: return dispatch_dim<T, FN_OP_NORMALIZE>(dim, x, n, h, b, q, ka, s);
        case FN_OP_NORMALIZE_SQ:
            return dispatch_dim<T, FN_OP_NORMALIZE_SQ>(dim, x, n, h, b, q, ka, s);
        case FN_OP_NORM: return dispatch_dim<T, FN_OP_NORM>(dim, x, n, h, b, q, ka, s);
        case FN_OP_NAIVE: return dispatch_dim<T, FN_OP_NAIVE>(dim, x, n, h, b, q, ka, s);
        case FN_OP_QUOTIENT: return dispatch_dim<T, FN_OP_QUOTIENT>(dim, x, n, h, b, q, ka, s);
        case FN_OP_QUOTIENT3_FAST:
            if (dim != 3) return fail(FN_EINVAL, "quotient3_fast is defined for dim 3 only");
            return launch<T, 3, FN_OP_QUOTIENT3_FAST>(x, n, h, b, q, ka, s);
        default: return fail(FN_EINVAL, "unknown op");
    }
}

int check_args(int op, int dim, int dtype, const void* x, int64_t n, const void* head,
               const void* body, const void* sq) {
    if (op < FN_OP_SCALE || op > FN_OP_NORMALIZE_SQ) return fail(FN_EINVAL, "unknown op");
    if (dim < 2 || dim > 4) return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    if (dtype != FN_F32 && dtype != FN_F64) return fail(FN_EINVAL, "dtype must be FN_F32/FN_F64");
    if (n < 0) return fail(FN_EINVAL, "n must be >= 0");
    if (n == 0) return FN_OK;
    if (!x || !head) return fail(FN_EINVAL, "x and head must not be NULL");
    if (op == FN_OP_NORM) {
        if (body) return fail(FN_EINVAL, "norm has no body output; pass NULL");
    } else if (!body) {
        return fail(FN_EINVAL, "body output must not be NULL");
    }
    if (op == FN_OP_NORMALIZE_SQ && !sq) return fail(FN_EINVAL, "sq must not be NULL");
    return FN_OK;
}

int run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body, void* sq,
        const double* ka, void* stream) {
    int rc = check_args(op, dim, dtype, x, n, head, body, sq);
    if (rc != FN_OK || n == 0) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == FN_F64) return dispatch<double>(op, dim, x, n, head, body, sq, ka, s);
    return dispatch<float>(op, dim, x, n, head, body, sq, ka, s);
}

// ---------------------------------------------------------------------------------
// Host-buffer path: chunked H2D -> kernel -> D2H pipeline over three streams, with
// per-device staging buffers that persist across calls (no allocation on the data
// path after the first call).  H2D and D2H of different chunks proceed concurrently
// on the two copy engines while the kernel of a third chunk runs.
// ---------------------------------------------------------------------------------
struct Staging {
    static constexpr int kPipes = 3;
    cudaStream_t streams[kPipes] = {};
    void* buf[kPipes] = {};
    size_t bytes = 0;
    bool init = false;
};
static std::mutex g_stage_mu;
static std::vector<Staging> g_stage;

static int staging_get(int dev, size_t bytes_per_pipe, Staging** out) {
    if ((int)g_stage.size() <= dev) g_stage.resize(dev + 1);
    Staging& st = g_stage[dev];
    cudaError_t e;
    if (!st.init) {
        for (int p = 0; p < Staging::kPipes; ++p) {
            e = cudaStreamCreateWithFlags(&st.streams[p], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        }
        st.init = true;
    }
    if (st.bytes < bytes_per_pipe) {
        for (int p = 0; p < Staging::kPipes; ++p) {
            if (st.buf[p]) cudaFree(st.buf[p]);
            st.buf[p] = nullptr;
        }
        st.bytes = 0;
        for (int p = 0; p < Staging::kPipes; ++p) {
            e = cudaMalloc(&st.buf[p], bytes_per_pipe);
            if (e != cudaSuccess) return fail(FN_ENOMEM, "cudaMalloc staging buffer failed");
        }
        st.bytes = bytes_per_pipe;
    }
    *out = &st;
    return FN_OK;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int host_run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
             void* sq, const double* ka) {
    int rc = check_args(op, dim, dtype, x, n, head, body, sq);
    if (rc != FN_OK || n == 0) return rc;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const size_t w = dtype == FN_F64 ? 8 : 4;
    const bool has_body = op != FN_OP_NORM;
    const bool has_sq = op == FN_OP_NORMALIZE_SQ;
    // ~48 MiB of input per chunk keeps three chunks in flight well inside L2-independent
    // streaming while amortising the per-copy latency.
    const int64_t chunk_rows = std::max<int64_t>(4096, ((int64_t)48 << 20) / (int64_t)(dim * w));
    const int64_t rows = std::min<int64_t>(n, chunk_rows);
    const size_t bx = align256(rows * dim * w), bh = align256(rows * w),
                 bb = has_body ? align256(rows * dim * w) : 0, bq = has_sq ? align256(rows * w) : 0;
    std::lock_guard<std::mutex> lk(g_stage_mu);
    Staging* st = nullptr;
    rc = staging_get(dev, bx + bh + bb + bq, &st);
    if (rc != FN_OK) return rc;
    int64_t chunk = 0;
    for (int64_t r0 = 0; r0 < n; r0 += rows, ++chunk) {
        const int p = (int)(chunk % Staging::kPipes);
        const int64_t m = std::min<int64_t>(rows, n - r0);
        cudaStream_t s = st->streams[p];
        char* base = static_cast<char*>(st->buf[p]);
        void* dx = base;
        void* dh = base + bx;
        void* db = has_body ? base + bx + bh : nullptr;
        void* dq = has_sq ? base + bx + bh + bb : nullptr;
        e = cudaMemcpyAsync(dx, static_cast<const char*>(x) + r0 * dim * w, m * dim * w,
                            cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
        rc = run(op, dim, dtype, dx, m, dh, db, dq, ka, s);
        if (rc != FN_OK) return rc;
        e = cudaMemcpyAsync(static_cast<char*>(head) + r0 * w, dh, m * w, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && has_body)
            e = cudaMemcpyAsync(static_cast<char*>(body) + r0 * dim * w, db, m * dim * w,
                                cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && has_sq)
            e = cudaMemcpyAsync(static_cast<char*>(sq) + r0 * w, dq, m * w, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync D2H");
    }
    for (int p = 0; p < Staging::kPipes; ++p) {
        e = cudaStreamSynchronize(st->streams[p]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    }
    return FN_OK;
}

}  // namespace fnb

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

const char* fn_version(void) { return "fastnorm-b200 0.1.0 sm_100a"; }
const char* fn_build_flags(void) { return FNB_BUILD_FLAGS; }
const char* fn_backend_name(void) { return "cuda"; }
const char* fn_last_error(void) { return fnb::g_last_error.c_str(); }

int fn_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

int fn_run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body, void* sq,
           const double* ka, void* stream) {
    return fnb::run(op, dim, dtype, x, n, head, body, sq, ka, stream);
}

int fn_host_run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
                void* sq, const double* ka) {
    return fnb::host_run(op, dim, dtype, x, n, head, body, sq, ka);
}

#define FNB_DEF_SCALING(base, OP)                                                              \
    int fn_##base##2_f64(const double* x, int64_t n, double* h, double* b, const double ka[6], \
                         void* s) { return fnb::run(OP, 2, FN_F64, x, n, h, b, nullptr, ka, s); } \
    int fn_##base##3_f64(const double* x, int64_t n, double* h, double* b, const double ka[6], \
                         void* s) { return fnb::run(OP, 3, FN_F64, x, n, h, b, nullptr, ka, s); } \
    int fn_##base##4_f64(const double* x, int64_t n, double* h, double* b, const double ka[6], \
                         void* s) { return fnb::run(OP, 4, FN_F64, x, n, h, b, nullptr, ka, s); } \
    int fn_##base##2_f32(const float* x, int64_t n, float* h, float* b, const double ka[6],    \
                         void* s) { return fnb::run(OP, 2, FN_F32, x, n, h, b, nullptr, ka, s); } \
    int fn_##base##3_f32(const float* x, int64_t n, float* h, float* b, const double ka[6],    \
                         void* s) { return fnb::run(OP, 3, FN_F32, x, n, h, b, nullptr, ka, s); } \
    int fn_##base##4_f32(const float* x, int64_t n, float* h, float* b, const double ka[6],    \
                         void* s) { return fnb::run(OP, 4, FN_F32, x, n, h, b, nullptr, ka, s); }

FNB_DEF_SCALING(scale, FN_OP_SCALE)
FNB_DEF_SCALING(normalize, FN_OP_NORMALIZE)

#define FNB_DEF_SQ(D)                                                                          \
    int fn_normalize##D##_sq_f64(const double* x, int64_t n, double* q, double* h, double* b,  \
                                 const double ka[6], void* s) {                                \
        return fnb::run(FN_OP_NORMALIZE_SQ, D, FN_F64, x, n, h, b, q, ka, s);                  \
    }                                                                                          \
    int fn_normalize##D##_sq_f32(const float* x, int64_t n, float* q, float* h, float* b,      \
                                 const double ka[6], void* s) {                                \
        return fnb::run(FN_OP_NORMALIZE_SQ, D, FN_F32, x, n, h, b, q, ka, s);                  \
    }
FNB_DEF_SQ(2)
FNB_DEF_SQ(3)
FNB_DEF_SQ(4)

#define FNB_DEF_NORM(D)                                                                        \
    int fn_norm##D##_f64(const double* x, int64_t n, double* h, const double ka[6], void* s) { \
        return fnb::run(FN_OP_NORM, D, FN_F64, x, n, h, nullptr, nullptr, ka, s);              \
    }                                                                                          \
    int fn_norm##D##_f32(const float* x, int64_t n, float* h, const double ka[6], void* s) {   \
        return fnb::run(FN_OP_NORM, D, FN_F32, x, n, h, nullptr, nullptr, ka, s);              \
    }
FNB_DEF_NORM(2)
FNB_DEF_NORM(3)
FNB_DEF_NORM(4)

#define FNB_DEF_PLAIN(base, OP, D)                                                             \
    int fn_##base##D##_f64(const double* x, int64_t n, double* h, double* b, void* s) {        \
        return fnb::run(OP, D, FN_F64, x, n, h, b, nullptr, nullptr, s);                       \
    }                                                                                          \
    int fn_##base##D##_f32(const float* x, int64_t n, float* h, float* b, void* s) {           \
        return fnb::run(OP, D, FN_F32, x, n, h, b, nullptr, nullptr, s);                       \
    }
FNB_DEF_PLAIN(naive, FN_OP_NAIVE, 2)
FNB_DEF_PLAIN(naive, FN_OP_NAIVE, 3)
FNB_DEF_PLAIN(naive, FN_OP_NAIVE, 4)
FNB_DEF_PLAIN(quotient, FN_OP_QUOTIENT, 2)
FNB_DEF_PLAIN(quotient, FN_OP_QUOTIENT, 3)
FNB_DEF_PLAIN(quotient, FN_OP_QUOTIENT, 4)

int fn_quotient3_fast_f64(const double* x, int64_t n, double* h, double* b, void* s) {
    return fnb::run(FN_OP_QUOTIENT3_FAST, 3, FN_F64, x, n, h, b, nullptr, nullptr, s);
}
int fn_quotient3_fast_f32(const float* x, int64_t n, float* h, float* b, void* s) {
    return fnb::run(FN_OP_QUOTIENT3_FAST, 3, FN_F32, x, n, h, b, nullptr, nullptr, s);
}

}  // extern "C"
