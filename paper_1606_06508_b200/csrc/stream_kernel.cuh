// stream_kernel.cuh -- the streaming kernels shared by the library and the tuner.
//
// Memory path.  Rows are AoS records of n = 2/3/4 elements (16/24/32 B
// for f64, 8/12/16 B for f32); a stride-3 record cannot be loaded coalesced by a
// thread-per-row mapping.  tma_stream_kernel therefore moves whole tiles of TR rows
// with the Blackwell bulk-copy engine (TMA, `cp.async.bulk`):
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
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "fastnorm_math.cuh"
#include "../../include/fastnorm_b200.h"

namespace fnb {

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
__device__ __forceinline__ void bulk_load_plain(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                                uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* dst_gmem, const void* src_smem, uint32_t bytes,
                                                uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                     dst_gmem),
                 "r"(smem_addr(src_smem)), "r"(bytes), "l"(policy)
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

// Default tile geometry per (T, N): ~6-8 KiB of input per stage (a multiple of 16 rows)
// and ~48 KiB of loads in flight per SM (stages x stage bytes x CTAs per SM).  Measured
// on B200 (tools/tune_stream.cu; profiles/r01_tune2.csv, r01_tune3.csv): more bytes in
// flight per SM (4 CTAs, or 8 stages) LOSES 6-8 % of DRAM throughput, while
// 2 CTAs x 4 stages x 6 KiB reaches the cudaMemcpy bandwidth.  L2 policy hints measured
// neutral (within noise) -> off.  The division-bound comparison variants (naive,
// quotient) are FP64-issue bound instead and prefer full occupancy (kCtasPerSm below).
template <typename T, int N> struct Tile {
    static constexpr int kRows = (N * (int)sizeof(T) <= 16) ? 512 : 256;
    static constexpr int kStageBytes = kRows * N * (int)sizeof(T);
    static constexpr int kStages = kStageBytes <= 6144 ? 4 : 3;
    static constexpr int kThreads = 256;
    static constexpr int kHints = 0;
};

template <int OP> struct CtasPerSm {
    static constexpr int value =
        (OP == FN_OP_NAIVE || OP == FN_OP_QUOTIENT || OP == FN_OP_QUOTIENT3_FAST) ? 8 : 2;
};

template <typename T, int N, int OP, int TR_, int S_> struct TileLayout {
    using Op = RowOp<T, N, OP>;
    static constexpr int TR = TR_;
    static constexpr int S = S_;
    static constexpr int OB = 3;
    static constexpr int kInBytes = TR * N * (int)sizeof(T);
    static constexpr int kHeadBytes = TR * (int)sizeof(T);
    static constexpr int kBodyBytes = Op::kBody ? TR * N * (int)sizeof(T) : 0;
    static constexpr int kSqBytes = Op::kSq ? TR * (int)sizeof(T) : 0;
    static constexpr int kOutBytes = kHeadBytes + kBodyBytes + kSqBytes;
    static constexpr int kSmemBytes = S * kInBytes + OB * kOutBytes + S * 8;
    static_assert(kInBytes % 16 == 0 && kHeadBytes % 16 == 0, "bulk copies need 16 B multiples");
};

// HINTS: bit 0 -> input loads carry an L2 evict-first policy (read once);
//        bit 1 -> output bulk stores carry an L2 evict-first policy.
template <typename T, int N, int OP, int TR_ = Tile<T, N>::kRows, int S_ = Tile<T, N>::kStages,
          int NT = Tile<T, N>::kThreads, int HINTS = Tile<T, N>::kHints>
__global__ void __launch_bounds__(NT) tma_stream_kernel(const T* __restrict__ x, int64_t nrows,
                                                        T* __restrict__ head, T* __restrict__ body,
                                                        T* __restrict__ sq, KArgs<T> ka) {
    using L = TileLayout<T, N, OP, TR_, S_>;
    using Op = typename L::Op;
    constexpr int TR = L::TR, S = L::S, OB = L::OB;
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
            if (HINTS & 1)
                bulk_load(s_in + k * L::kInBytes, x + tile * TR * N, L::kInBytes, &full[k], policy);
            else
                bulk_load_plain(s_in + k * L::kInBytes, x + tile * TR * N, L::kInBytes, &full[k]);
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
            if (HINTS & 2) {
                bulk_store_hint(head + row0, th, L::kHeadBytes, policy);
                if (Op::kBody) bulk_store_hint(body + row0 * N, tb, L::kBodyBytes, policy);
                if (Op::kSq) bulk_store_hint(sq + row0, tq, L::kSqBytes, policy);
            } else {
                bulk_store(head + row0, th, L::kHeadBytes);
                if (Op::kBody) bulk_store(body + row0 * N, tb, L::kBodyBytes);
                if (Op::kSq) bulk_store(sq + row0, tq, L::kSqBytes);
            }
            bulk_commit();
            if (k + S < my_tiles) {
                const int64_t nt = tile + (int64_t)S * gridDim.x;
                mbar_arrive_expect_tx(&full[s], L::kInBytes);
                if (HINTS & 1)
                    bulk_load(s_in + s * L::kInBytes, x + nt * TR * N, L::kInBytes, &full[s], policy);
                else
                    bulk_load_plain(s_in + s * L::kInBytes, x + nt * TR * N, L::kInBytes, &full[s]);
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

}  // namespace fnb
