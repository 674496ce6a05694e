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
// Rows past the last full tile, outputs that are not 16-byte aligned and irregular row
// strides use a plain thread-per-row kernel with the same row arithmetic; inputs off the
// 16-byte grid take the MIS instantiation (each tile loaded from the boundary below it).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "fastnorm_math.cuh"
#include "../../include/fastnorm_b200.h"

namespace fnb {

// ---------------------------------------------------------------------------------
// Row operations: one functor per kernel family.  Each row of N inputs produces up to
// three output records of W0 / W1 / W2 elements (written to three arrays: "head",
// "body", "extra"); apply() returns false for a row the reference would reject with
// an exception (rotations only), which the kernel counts.
// ---------------------------------------------------------------------------------
template <typename T, int N, int OP> struct RowOp;

template <typename T, int N> struct RowOp<T, N, FN_OP_NORMALIZE> {
    static constexpr int W0 = 1, W1 = N, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>& ka, T* o0, T* o1, T*) {
        T sq;
        normalize_row<T, N, false>(x, ka, o0[0], *reinterpret_cast<T(*)[N]>(o1), sq);
        return true;
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_NORMALIZE_SQ> {
    static constexpr int W0 = 1, W1 = N, W2 = 1;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>& ka, T* o0, T* o1, T* o2) {
        normalize_row<T, N, true>(x, ka, o0[0], *reinterpret_cast<T(*)[N]>(o1), o2[0]);
        return true;
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_NORM> {
    static constexpr int W0 = 1, W1 = 0, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>& ka, T* o0, T*, T*) {
        o0[0] = norm_row<T, N>(x, ka);
        return true;
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_SCALE> {
    static constexpr int W0 = 1, W1 = N, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>& ka, T* o0, T* o1, T*) {
        scale_row(x, ka, o0[0], *reinterpret_cast<T(*)[N]>(o1));
        return true;
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_NAIVE> {
    static constexpr int W0 = 1, W1 = N, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>&, T* o0, T* o1, T*) {
        naive_row<T, N>(x, o0[0], *reinterpret_cast<T(*)[N]>(o1));
        return true;
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_QUOTIENT> {
    static constexpr int W0 = 1, W1 = N, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>&, T* o0, T* o1, T*) {
        quotient_row<T, N>(x, o0[0], *reinterpret_cast<T(*)[N]>(o1));
        return true;
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_QUOTIENT3_FAST> {
    static_assert(N == 3, "quotient3_fast is 3-D only (_backend.py:96-98)");
    static constexpr int W0 = 1, W1 = N, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>&, T* o0, T* o1, T*) {
        quotient3_fast_row<T>(x, o0[0], *reinterpret_cast<T(*)[N]>(o1));
        return true;
    }
};
// Rotations (rotation.py:53-111; binary64 quaternions only): R is a row-major 3x3.
template <typename T, int N> struct RowOp<T, N, FN_OP_ROT_UNIT> {
    static_assert(N == 4, "rotations take quaternions");
    static constexpr int W0 = 9, W1 = 0, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>&, T* o0, T*, T*) {
        return rotation_unit_row(x, o0);
    }
};
template <typename T, int N> struct RowOp<T, N, FN_OP_ROT_GENERAL> {
    static_assert(N == 4, "rotations take quaternions");
    static constexpr int W0 = 9, W1 = 0, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>& ka, T* o0, T*, T*) {
        return rotation_general_row(x, ka, o0);
    }
};
// normalize4 fused with rotation_unit of its unit output: r, unit, R in one pass.
template <typename T, int N> struct RowOp<T, N, FN_OP_NORMALIZE_ROT> {
    static_assert(N == 4, "rotations take quaternions");
    static constexpr int W0 = 1, W1 = 4, W2 = 9;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>& ka, T* o0, T* o1, T* o2) {
        T sq;
        T(&u)[4] = *reinterpret_cast<T(*)[4]>(o1);
        normalize_row<T, 4, false>(x, ka, o0[0], u, sq);
        return rotation_unit_row(u, o2);
    }
};

// R v for a batch of vectors with one matrix (in the kernel arguments).
template <typename T, int N> struct RowOp<T, N, FN_OP_ROT_APPLY> {
    static_assert(N == 3, "the rotation is applied to 3-vectors");
    static constexpr int W0 = 3, W1 = 0, W2 = 0;
    __device__ __forceinline__ static bool apply(const T (&x)[N], const KArgs<T>& ka, T* o0, T*, T*) {
        rotation_apply_row(x, ka.rot, o0);
        return true;
    }
};

// Two-input ops (a second AoS record per row, N2 wide): per-row rotation of vectors.
// normalize4 -> rotation_unit of its unit output -> apply to v: the reference
// composition rotation_unit(normalize4(p, *q).unit).apply(v) (rotation.py:39-41, 87-111).
template <typename T, int N> struct RowOp<T, N, FN_OP_QUAT_ROTATE> {
    static_assert(N == 4, "quaternions");
    static constexpr int W0 = 3, W1 = 0, W2 = 0, N2 = 3;
    __device__ __forceinline__ static bool apply2(const T (&q)[N], const T (&v)[3], const KArgs<T>& ka,
                                                  T* o0, T*, T*) {
        T r, u[4], sq, R[9];
        normalize_row<T, 4, false>(q, ka, r, u, sq);
        const bool ok = rotation_unit_row(u, R);
        rotation_apply_row(v, R, o0);
        return ok;
    }
};
// Per-row RotationMatrix.apply: R[N,9] (row-major) times v[N,3].
template <typename T, int N> struct RowOp<T, N, FN_OP_MAT_APPLY> {
    static_assert(N == 9, "row-major 3x3 matrices");
    static constexpr int W0 = 3, W1 = 0, W2 = 0, N2 = 3;
    __device__ __forceinline__ static bool apply2(const T (&R)[N], const T (&v)[3], const KArgs<T>&, T* o0,
                                                  T*, T*) {
        rotation_apply_row(v, R, o0);
        return true;
    }
};

// Width of an op's second input record (0: single-input op).
template <typename Op, typename = void> struct InWidth2 {
    static constexpr int value = 0;
};
template <typename Op> struct InWidth2<Op, std::void_t<decltype(Op::N2)>> {
    static constexpr int value = Op::N2;
};

template <int W> struct Slot { static constexpr int value = W > 0 ? W : 1; };

template <typename Op, typename T, int N, int N2S>
__device__ __forceinline__ bool apply_op(const T (&x)[N], const T (&x2)[N2S], const KArgs<T>& ka, T* o0, T* o1,
                                         T* o2) {
    if constexpr (InWidth2<Op>::value > 0)
        return Op::apply2(x, x2, ka, o0, o1, o2);
    else
        return Op::apply(x, ka, o0, o1, o2);
}

// One row through global memory (tails, unaligned arrays, tiny batches).  Row i of x
// starts at element i * ldx (ldx = N for dense records; larger for padded records such
// as xyz in xyzw, whose extra elements are not read).
template <typename T, int N, int OP>
__device__ __forceinline__ bool row_global(const T* __restrict__ x, const T* __restrict__ x2, int64_t i,
                                           T* __restrict__ head, T* __restrict__ body,
                                           T* __restrict__ extra, const KArgs<T>& ka, int64_t ldx = N) {
    using Op = RowOp<T, N, OP>;
    constexpr int N2 = InWidth2<Op>::value;
    T xr[N], x2r[Slot<N2>::value], o0[Slot<Op::W0>::value], o1[Slot<Op::W1>::value], o2[Slot<Op::W2>::value];
#pragma unroll
    for (int c = 0; c < N; ++c) xr[c] = __ldg(x + i * ldx + c);
#pragma unroll
    for (int c = 0; c < N2; ++c) x2r[c] = __ldg(x2 + i * N2 + c);
    const bool ok = apply_op<Op>(xr, x2r, ka, o0, o1, o2);
#pragma unroll
    for (int c = 0; c < Op::W0; ++c) head[i * Op::W0 + c] = o0[c];
#pragma unroll
    for (int c = 0; c < Op::W1; ++c) body[i * Op::W1 + c] = o1[c];
#pragma unroll
    for (int c = 0; c < Op::W2; ++c) extra[i * Op::W2 + c] = o2[c];
    return ok;
}

// Captured launches (CUDA graphs) own their counter instead of alternating a per-stream
// pair: every CTA's leader reports in after its last claim, and the last one to do so
// zeroes the counter and the report word, so the node's next replay starts from zero.
// (A graph's launches are ordered by the graph; griddepcontrol.wait in the successor
// covers these stores like any other write of the predecessor.)
template <typename T>
__device__ __forceinline__ void sched_report_done(const KArgs<T>& ka) {
    if (ka.sched != nullptr && ka.sched_done != nullptr) {
        __threadfence();
        if (atomicAdd(ka.sched_done, 1u) == gridDim.x - 1) {
            *ka.sched = 0u;
            *ka.sched_done = 0u;
            __threadfence();
        }
    }
}

// Per-thread count of rejected rows -> one atomic per warp (rotations only).
__device__ __forceinline__ void count_invalid(unsigned long long* counter, unsigned long long bad) {
    if (counter == nullptr) return;
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(counter, bad);
}

// Programmatic dependent launch (PDL).  The host launches the streaming kernels with
// programmatic stream serialization allowed, so a kernel may become resident while its
// predecessor on the stream drains.  griddepcontrol.wait (a no-op for a normal launch)
// blocks until every predecessor grid has completed and its memory is visible, so it
// runs before the first global load or store; launch_dependents then lets the next
// PDL launch on the stream start its own prologue early.
__device__ __forceinline__ void grid_dependency_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void grid_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename T, int N, int OP>
__global__ void __launch_bounds__(256) direct_kernel(const T* __restrict__ x, const T* __restrict__ x2,
                                                     int64_t nrows, T* __restrict__ head,
                                                     T* __restrict__ body, T* __restrict__ extra,
                                                     KArgs<T> ka, int64_t ldx) {
    grid_dependency_wait();
    grid_launch_dependents();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long bad = 0;
    const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t trips = nrows > start ? (nrows - 1 - start) / stride + 1 : 0;
    // uniform trip count per warp so the shuffle-reduce below sees every lane
    for (int64_t t = 0, i = start; t < trips; ++t, i += stride)
        bad += row_global<T, N, OP>(x, x2, i, head, body, extra, ka, ldx) ? 0 : 1;
    count_invalid(ka.invalid, bad);
}

// ---------------------------------------------------------------------------------
// Structure-of-arrays rows: component k of row i is xs[k][i]; outputs likewise (head[i],
// body[c][i], extra[i]).  Every warp access is a contiguous 256 B run per array, so plain
// loads and stores coalesce; the arithmetic is the same RowOp as the AoS kernels.
// ---------------------------------------------------------------------------------
template <typename T, int N> struct SoaPtrs {
    const T* x[N];
    T* head;
    T* body[N];
    T* extra;
};

template <typename T, int N, int OP>
__global__ void __launch_bounds__(256) soa_kernel(SoaPtrs<T, N> p, int64_t nrows, KArgs<T> ka) {
    using Op = RowOp<T, N, OP>;
    static_assert(Op::W0 == 1 && (Op::W1 == 0 || Op::W1 == N) && Op::W2 <= 1, "per-component outputs");
    grid_dependency_wait();
    grid_launch_dependents();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += stride) {
        T xr[N], o0[1], o1[Slot<Op::W1>::value], o2[1];
#pragma unroll
        for (int c = 0; c < N; ++c) xr[c] = __ldcs(p.x[c] + i);
        (void)Op::apply(xr, ka, o0, o1, o2);
        __stcs(p.head + i, o0[0]);
#pragma unroll
        for (int c = 0; c < Op::W1; ++c) __stcs(p.body[c] + i, o1[c]);
        if constexpr (Op::W2 == 1) __stcs(p.extra + i, o2[0]);
    }
}

// Vectorised form: each thread moves 16 B per array per step (2 f64 or 4 f32 rows), so
// every warp request is a contiguous 512 B run.  All arrays must be 16 B aligned; rows
// past the last whole vector go through the scalar form.
template <typename T> struct Vec16;
template <> struct Vec16<double> {
    using type = double2;
    static constexpr int kRows = 2;
    __device__ __forceinline__ static double get(const double2& v, int j) { return j ? v.y : v.x; }
    __device__ __forceinline__ static double2 make(const double (&a)[2]) { return make_double2(a[0], a[1]); }
};
template <> struct Vec16<float> {
    using type = float4;
    static constexpr int kRows = 4;
    __device__ __forceinline__ static float get(const float4& v, int j) {
        return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
    }
    __device__ __forceinline__ static float4 make(const float (&a)[4]) { return make_float4(a[0], a[1], a[2], a[3]); }
};

template <typename T, int N, int OP>
__global__ void __launch_bounds__(256) soa_vec_kernel(SoaPtrs<T, N> p, int64_t nvec, KArgs<T> ka) {
    using Op = RowOp<T, N, OP>;
    using VT = typename Vec16<T>::type;
    constexpr int V = Vec16<T>::kRows;
    grid_dependency_wait();
    grid_launch_dependents();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nvec; g += stride) {
        VT xv[N];
#pragma unroll
        for (int c = 0; c < N; ++c) xv[c] = __ldcs(reinterpret_cast<const VT*>(p.x[c]) + g);
        T h[V], b[Slot<Op::W1>::value][V], q[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            T xr[N], o0[1], o1[Slot<Op::W1>::value], o2[1];
#pragma unroll
            for (int c = 0; c < N; ++c) xr[c] = Vec16<T>::get(xv[c], j);
            (void)Op::apply(xr, ka, o0, o1, o2);
            h[j] = o0[0];
#pragma unroll
            for (int c = 0; c < Op::W1; ++c) b[c][j] = o1[c];
            q[j] = o2[0];
        }
        __stcs(reinterpret_cast<VT*>(p.head) + g, Vec16<T>::make(h));
#pragma unroll
        for (int c = 0; c < Op::W1; ++c) __stcs(reinterpret_cast<VT*>(p.body[c]) + g, Vec16<T>::make(b[c]));
        if constexpr (Op::W2 == 1) __stcs(reinterpret_cast<VT*>(p.extra) + g, Vec16<T>::make(q));
    }
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
// Plain arrive (release at CTA scope): one count of the barrier's current phase.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
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
// The binary64 division-bound kernels (quotient, quotient3_fast, naive) are latency
// bound at 3-4 CTAs per SM (24-32 warps): ncu on quotient2 / config 2 shows "wait" and
// barrier stalls on top, 1.6 eligible warps per scheduler, shared memory limiting the CTA
// count to 3 (profiles/r02o_quotient2_stalls.txt).  FNB_DIV_ROWS_SHIFT halves their tile
// (rows per stage) that many times and FNB_DIV_STAGES sets their ring depth, so more
// CTAs fit per SM; FNB_DIV_MIN_BLOCKS is the launch-bounds minimum (register cap).
#ifndef FNB_DIV_ROWS_SHIFT
#define FNB_DIV_ROWS_SHIFT 0
#endif
#ifndef FNB_DIV_STAGES
#define FNB_DIV_STAGES 0
#endif
#ifndef FNB_DIV_MIN_BLOCKS
#define FNB_DIV_MIN_BLOCKS 1
#endif
template <typename T, int OP> struct DivBound {
    static constexpr bool value = std::is_same<T, double>::value &&
                                  (OP == FN_OP_QUOTIENT || OP == FN_OP_QUOTIENT3_FAST || OP == FN_OP_NAIVE);
};
template <typename T, int OP> struct MinBlocks {
    static constexpr int value = DivBound<T, OP>::value ? FNB_DIV_MIN_BLOCKS : 1;
};

#ifndef FNB_STREAM_STAGES
#define FNB_STREAM_STAGES 0  // experiments: ring depth of every (T, N) default tile
#endif
#ifndef FNB_STREAM_TILE_BYTES
#define FNB_STREAM_TILE_BYTES 8192  // experiments: input bytes per stage (upper bound)
#endif
constexpr int pow2_floor(int v) { return v >= 2 ? 2 * pow2_floor(v / 2) : 1; }

template <typename T, int N> struct Tile {
    // largest power of two with at most 8 KiB of input per stage
    static constexpr int kRows = pow2_floor(FNB_STREAM_TILE_BYTES / (N * (int)sizeof(T)));
    static constexpr int kStageBytes = kRows * N * (int)sizeof(T);
    // measured (profiles/r01j_tune_all.csv): 4 stages for n = 2, 3; 3 for quaternions,
    // whose wider output staging already keeps more bytes in flight per CTA.
    static constexpr int kStages = FNB_STREAM_STAGES > 0 ? FNB_STREAM_STAGES : (N == 4 ? 3 : 4);
    static constexpr int kThreads = 256;
    static constexpr int kHints = 0;
};

// CTAs per SM of the streaming kernel.
// * norm writes 8 B per row against 16-32 B read: read-dominated traffic wants more loads
//   in flight (4 CTAs: 7090 vs 5963 GB/s at 2, profiles/r01i_tune_norm.csv).
// * The other families: 2 CTAs under round 1's static schedule (profiles/r01_tune*.csv);
//   with the dynamic schedule 3 CTAs measure better (profiles/r02w_ab_ctas_table.txt,
//   2 -> 3: normalize2 f64 +8.8 %, normalize4_sq +4.1 %, normalize4 +2.4 %, scale3
//   +2.6 %, normalize4_rotation +1.3 %, normalize3 f64 at 2^30 rows -0.7 to +2.8 %
//   over three rounds, normalize2 f32 +7.9 %, normalize4 f32 +2.3 %).  3-D binary32
//   rows lose 8 % at 3 CTAs under the STATIC schedule, which normalize3 f32 kept until
//   the two were measured together: dynamic at 3 CTAs gives normalize3 f32 6912 against
//   6591 GB/s on config 4, scale3 f32 6889 against 5460, normalize3_sq f32 6889 against
//   5919 (profiles/r02ao_sweep_table.txt, r02ap_tables.txt).  scale3 f32 and normalize3_sq
//   f32 take 4 (in one process over both regimes and two sizes: normalize3_sq 6152-6827 at
//   3 -> 6768-6886 at 4, scale3 6102-6913 -> 6761-6881; normalize3 f32 unchanged within
//   0.3 %, so it stays at 3; profiles/r02as_f32_dim3.txt).
// * The division-bound comparison kernels want full occupancy (FNB_DIV_CTAS).
#ifndef FNB_DIV_CTAS
#define FNB_DIV_CTAS 8
#endif
#ifndef FNB_STREAM_CTAS
#define FNB_STREAM_CTAS 3
#endif
template <typename T, int N, int OP> struct CtasPerSm {
    static constexpr int value =
        (OP == FN_OP_NAIVE || OP == FN_OP_QUOTIENT || OP == FN_OP_QUOTIENT3_FAST) ? FNB_DIV_CTAS
        : OP == FN_OP_NORM                            ? 4
        : (std::is_same<T, float>::value && N == 3 && (OP == FN_OP_SCALE || OP == FN_OP_NORMALIZE_SQ)) ? 4
                                                      : FNB_STREAM_CTAS;
};

// Output staging tiles: 3 (one bulk-store group reading behind the current one).  A
// fourth tile for the write-heavy rotations measured +2 % in tools/tune_stream
// (profiles/r01ax_rot.csv) but -5 % through the library (normalize4_rotation 6265 vs
// 5950 GB/s, A/B of the two builds alternated on one box, profiles/r01az_ab.txt), so
// FNB_ROT_OUT_TILES stays 3.
#ifndef FNB_ROT_OUT_TILES
#define FNB_ROT_OUT_TILES 3
#endif
template <int OP> struct OutTiles {
    static constexpr int value =
        (OP == FN_OP_ROT_UNIT || OP == FN_OP_ROT_GENERAL || OP == FN_OP_NORMALIZE_ROT) ? FNB_ROT_OUT_TILES : 3;
};

// LDX_: elements per input record (0 = N, dense rows; N = 3 with LDX_ = 4 reads xyz out of
// xyzw records: the bulk copy moves whole records, the row op reads the first N).
// MIS_: the instantiation for inputs off the 16-byte grid (see tma_stream_kernel); the
// aligned instantiation keeps the plain layout and code.
template <typename T, int N, int OP, int TR_, int S_, int OB_ = OutTiles<OP>::value, int LDX_ = 0,
          bool MIS_ = false>
struct TileLayout {
    using Op = RowOp<T, N, OP>;
    static constexpr int TR = TR_;
    static constexpr int S = S_;
    static constexpr int OB = OB_;  // output staging tiles (bulk-store groups in flight)
    static constexpr int LDX = LDX_ > 0 ? LDX_ : N;
    static_assert(OB >= 3, "the store pipeline keeps OB - 2 groups reading behind the current one");
    static_assert(LDX >= N, "an input record holds at least the N components");
    static constexpr int kInBytes = TR * LDX * (int)sizeof(T);
    // MIS_: a stage holds one tile of records plus room for 16 more bytes (rows whose
    // storage is not 16-byte aligned are loaded from the aligned address below them);
    // 128 bytes of room keep every stage and staging tile 128-byte aligned
    static constexpr int kRoom = MIS_ ? 128 : 0;
    static constexpr int kStageBytes = kInBytes + kRoom;
    static constexpr int kIn2Bytes = TR * InWidth2<Op>::value * (int)sizeof(T);  // second input
    static constexpr int kB0 = TR * Op::W0 * (int)sizeof(T);
    static constexpr int kB1 = TR * Op::W1 * (int)sizeof(T);
    static constexpr int kB2 = TR * Op::W2 * (int)sizeof(T);
    static constexpr int kOutBytes = kB0 + kB1 + kB2;
    static constexpr int kIn2StageBytes = kIn2Bytes > 0 ? kIn2Bytes + kRoom : 0;  // same room for x2
    static constexpr int kSmemBytes = S * (kStageBytes + kIn2StageBytes) + OB * kOutBytes + S * 8;
    static_assert(kInBytes % 16 == 0 && kIn2Bytes % 16 == 0 && kB0 % 16 == 0 && kB1 % 16 == 0 &&
                      kB2 % 16 == 0,
                  "bulk copies need 16 B multiples");
};

// Rows per tile for an op: the default, halved while the three output staging tiles
// would exceed 64 KiB (rotations write 72-112 B per row).
// 3-D rows of the scaling families under the dynamic schedule (round 2): binary64 takes
// 512-row stages (12 KiB) in a 3-deep ring, 2 CTAs per SM by shared memory (72 KiB of
// loads in flight per SM, as before): at 2^30 rows the 256-row tiles ran 6500 GB/s and
// these 6978, stable over three rounds, with 2^28 rows unchanged (6935 vs 6949;
// profiles/r02z_ab_tiles.txt).  binary32 keeps 512-row stages in a 5-deep ring (+2.8 %
// on config 4, profiles/r02y_ab_stages_table.txt).
#ifndef FNB_BIG_TILES
#define FNB_BIG_TILES 1
#endif
// BIG = false selects the default geometry for the same kernel: batches below
// kBigTileRows rows and the many-batch kernel keep it (1e6-row batches: 0.84 vs 0.80 of
// the copy peak as a graph-replayed stream, profiles/r02aa_many.txt).
template <typename T, int N, int OP, bool BIG = true> struct Rows3 {
    static constexpr bool scaling = OP == FN_OP_NORMALIZE || OP == FN_OP_NORMALIZE_SQ || OP == FN_OP_SCALE;
    static constexpr bool f64 = BIG && FNB_BIG_TILES && N == 3 && scaling && std::is_same<T, double>::value;
    static constexpr bool f32 = BIG && FNB_BIG_TILES && N == 3 && OP == FN_OP_NORMALIZE && std::is_same<T, float>::value;
    static constexpr bool any = f64 || f32;
};
constexpr int64_t kBigTileRows = int64_t(1) << 24;

// The binary32 division-bound kernels ask for 8 CTAs per SM like the binary64 ones, but their
// default tiles (512-1024 rows, 48-68 KiB per CTA) let only 3-4 fit.  Halving the tile
// (FNB_DIV32_ROWS_SHIFT = 1) pays for 2-D rows only (1024 -> 512 rows: quotient2 f32
// 4732 -> 5223 GB/s, naive2 f32 on full-range rows 3294 -> 4134; 3-D and 4-D rows lose
// 2-37 %, a quarter tile loses everywhere; profiles/r02ay_div32_table.txt), so it applies
// to N = 2.
#ifndef FNB_DIV32_ROWS_SHIFT
#define FNB_DIV32_ROWS_SHIFT 1
#endif
template <typename T, int OP> struct DivBound32 {
    static constexpr bool value = std::is_same<T, float>::value &&
                                  (OP == FN_OP_QUOTIENT || OP == FN_OP_QUOTIENT3_FAST || OP == FN_OP_NAIVE);
};
template <typename T, int N, int OP, bool BIG = true> struct OpRows {
    static constexpr int kOutRow = (RowOp<T, N, OP>::W0 + RowOp<T, N, OP>::W1 + RowOp<T, N, OP>::W2) * (int)sizeof(T);
    static constexpr int kTile = Rows3<T, N, OP, BIG>::f64 ? 512 : Tile<T, N>::kRows;
    static constexpr int kBase = (3 * kOutRow * kTile > 65536) ? kTile / 2 : kTile;
    static constexpr int value = DivBound<T, OP>::value     ? kBase >> FNB_DIV_ROWS_SHIFT
                                 : (DivBound32<T, OP>::value && N == 2) ? kBase >> FNB_DIV32_ROWS_SHIFT
                                                            : kBase;
};

// Per-row matrices are 72 B records: the default 8 KiB stage would hold only 64 of them
// (5840 GB/s).  256 rows x 3 stages (18 KiB of matrices + 6 KiB of vectors per stage)
// reach 6900 GB/s, 1.05 of the measured copy peak (read-dominated traffic,
// profiles/r01bw_mat.txt).
#ifndef FNB_MAT_APPLY_ROWS
#define FNB_MAT_APPLY_ROWS 256
#endif
#ifndef FNB_MAT_APPLY_STAGES
#define FNB_MAT_APPLY_STAGES 3
#endif
template <typename T, bool BIG> struct OpRows<T, 9, FN_OP_MAT_APPLY, BIG> {
    static constexpr int value = FNB_MAT_APPLY_ROWS;
};
template <typename T> struct Tile<T, 9> {
    static constexpr int kRows = FNB_MAT_APPLY_ROWS;
    static constexpr int kStages = FNB_MAT_APPLY_STAGES;
    static constexpr int kThreads = 256;
    static constexpr int kHints = 0;
};

// Stages per op: the (T, N) default; the fused normalize4 -> rotation (144 B per row,
// 112 B of it written) is tunable through FNB_NROT_ROWS / FNB_NROT_STAGES.  Through the
// library (profiles/r01ca_nrot.txt): 128 x 3 (default) 6267 GB/s, 256 x 2 6308,
// 128 x 4 5994, 256 x 3 5880 -- the tuner's ranking (r01bz_rot.csv) does not carry over.
// normalize2_sq stages 16 B (f32) / 32 B (f64) of results per row, the most per input byte:
// with the default 4-deep ring a CTA takes 80 KiB and only two fit per SM.  A 3-deep ring
// (72 KiB, three CTAs): f32 5877 -> 6792 GB/s on in-band rows and 4859 -> 6594 on
// full-range rows, f64 6871 -> 6825 and 6684 -> 6824 (profiles/r02ap_tables.txt).
#ifndef FNB_SQ2_STAGES
#define FNB_SQ2_STAGES 3
#endif
template <typename T, int N, int OP, bool BIG = true> struct OpStages {
    static constexpr int value = (DivBound<T, OP>::value && FNB_DIV_STAGES > 0) ? FNB_DIV_STAGES
                                 : Rows3<T, N, OP, BIG>::f64                   ? 3
                                 : Rows3<T, N, OP, BIG>::f32                   ? 5
                                 : (N == 2 && OP == FN_OP_NORMALIZE_SQ)         ? FNB_SQ2_STAGES
                                                                               : Tile<T, N>::kStages;
};
// quotient2 f64 with two 512-row stages (4 CTAs per SM instead of 3) gained 9 % on
// config 2 but ran bimodal on unit-range 2-D rows (0.388 or 0.493 ms per 2^26 rows from
// one process to the next: a two-stage ring is too shallow for HBM-bound rows), so every
// division-bound kernel keeps the default ring (profiles/r02q_ab_quotient2_stages_table.txt).

// Threads per CTA: one row per thread at least (a division-bound tile shrunk below 256
// rows gets as many threads as rows).
template <typename T, int N, int OP, bool BIG = true> struct OpThreads {
    static constexpr int value =
        OpRows<T, N, OP, BIG>::value < Tile<T, N>::kThreads ? OpRows<T, N, OP, BIG>::value : Tile<T, N>::kThreads;
};
#ifdef FNB_NROT_STAGES
template <typename T, int N, bool BIG> struct OpStages<T, N, FN_OP_NORMALIZE_ROT, BIG> {
    static constexpr int value = FNB_NROT_STAGES;
};
#endif
#ifdef FNB_NROT_ROWS
template <typename T, int N, bool BIG> struct OpRows<T, N, FN_OP_NORMALIZE_ROT, BIG> {
    static constexpr int value = FNB_NROT_ROWS;
};
#endif

// HINTS: bit 0 -> input loads carry an L2 evict-first policy (read once);
//        bit 1 -> output bulk stores carry an L2 evict-first policy.
// Per-CTA timeline (developer probe tools/probe/cfg1_timeline.cu only; compiled out of
// the library): thread 0 of each CTA stores %globaltimer into
// fnb_timeline[blockIdx.x * kTimelineSlots + slot]: slots 0-4 at five points of the
// kernel, and for its first kTimelineTiles tiles three per tile (data landed, tile
// computed and staged, previous store group read out).
#ifdef FNB_TIMELINE
constexpr int kTimelineSlots = 64, kTimelineTiles = 19;
__device__ unsigned long long* fnb_timeline;
__device__ int fnb_timeline_tiles;  // per-tile marks on (they perturb the timing)
__device__ __forceinline__ void timeline_mark(int slot) {
    if (threadIdx.x == 0 && fnb_timeline != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        fnb_timeline[blockIdx.x * kTimelineSlots + slot] = t;
    }
}
__device__ __forceinline__ void timeline_tile(int64_t k, int phase, bool me = true) {
    if (me && k < kTimelineTiles && fnb_timeline != nullptr && fnb_timeline_tiles) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        fnb_timeline[blockIdx.x * kTimelineSlots + 5 + 3 * (int)k + phase] = t;
    }
}
#else
__device__ __forceinline__ void timeline_mark(int) {}
__device__ __forceinline__ void timeline_tile(int64_t, int, bool = true) {}
#endif

template <typename T, int N, int OP, int TR_ = OpRows<T, N, OP>::value, int S_ = OpStages<T, N, OP>::value,
          int NT = Tile<T, N>::kThreads, int HINTS = Tile<T, N>::kHints, int OB_ = OutTiles<OP>::value,
          int LDX_ = 0, bool MIS = false>
__global__ void __launch_bounds__(NT, MinBlocks<T, OP>::value) tma_stream_kernel(const T* __restrict__ x, const T* __restrict__ x2,
                                                        int64_t nrows, T* __restrict__ head,
                                                        T* __restrict__ body, T* __restrict__ extra,
                                                        KArgs<T> ka) {
    using L = TileLayout<T, N, OP, TR_, S_, OB_, LDX_, MIS>;
    using Op = typename L::Op;
    constexpr int TR = L::TR, S = L::S, OB = L::OB, LDX = L::LDX;
    constexpr int W0 = Op::W0, W1 = Op::W1, W2 = Op::W2;
    constexpr int N2 = InWidth2<Op>::value;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* s_in = smem;
    unsigned char* s_in2 = smem + S * L::kStageBytes;  // second input ring (two-input ops)
    unsigned char* s_out = s_in2 + S * L::kIn2StageBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(s_out + OB * L::kOutBytes);
    timeline_mark(0);

    // MIS: inputs whose storage is not 16-byte aligned (x[1:] of a dense array; outputs
    // must be aligned, the host checks).  Every stage is loaded from the 16-byte boundary
    // `mis` bytes below its first row, 16 bytes longer, and read at offset `mis`.  Bulk
    // tiles only cover bytes between that boundary and the last row's end; the reach
    // below x stays inside x's 16-byte block, hence inside its allocation.  The second
    // input of the two-input ops gets its own offset under the same rule.  (A separate
    // instantiation: folding this into the aligned kernel cost 1-2.6 % on aligned rows,
    // profiles/r01s23_ab_mis.txt.)
    // Padded records: the last row may end at its N-th element (a strided view of a
    // shorter allocation), so it never rides in a bulk tile that would read its padding.
    const int mis = MIS ? (int)(reinterpret_cast<uintptr_t>(x) & 15) : 0;
    const int mis2 = MIS && N2 > 0 ? (int)(reinterpret_cast<uintptr_t>(x2) & 15) : 0;
    int64_t ntiles = (LDX == N ? nrows : nrows - 1) / TR;
    if constexpr (MIS) {
        const int64_t avail = ((nrows - 1) * LDX + N) * (int64_t)sizeof(T);  // x to the last row's end
        const int64_t reach = mis ? 16 - mis : 0;                               // bytes read past a tile
        ntiles = avail >= reach ? (avail - reach) / L::kInBytes : 0;
        if constexpr (N2 > 0) {
            const int64_t avail2 = nrows * N2 * (int64_t)sizeof(T), reach2 = mis2 ? 16 - mis2 : 0;
            const int64_t ntiles2 = avail2 >= reach2 ? (avail2 - reach2) / L::kIn2Bytes : 0;
            if (ntiles2 < ntiles) ntiles = ntiles2;
        }
    }
    const unsigned char* xa = reinterpret_cast<const unsigned char*>(x) - mis;
    const unsigned char* x2a = reinterpret_cast<const unsigned char*>(x2) - mis2;
    const uint32_t load_bytes = L::kInBytes + (MIS && mis ? 16 : 0);
    const uint32_t load2_bytes = L::kIn2Bytes + (MIS && mis2 ? 16 : 0);
    // Schedule.  Static: CTA b owns tiles b, b + grid, b + 2 grid, ...
    // Dynamic (ka.sched != NULL): every CTA's first S tiles are the static ones (no atomic
    // on the critical start), then its leader claims further tiles from a counter in
    // global memory, ka.sched_batch consecutive tiles per claim and one claim ahead of
    // use, so the atomic's round trip overlaps tiles of work; CTAs that run ahead take
    // more tiles and all finish within a batch of each other.  The tile id of
    // each stage travels to the CTA's threads through s_tile[], written before the stage's
    // mbarrier arrive (release) and read after its wait (acquire); -1 = no more tiles.
    // Counters: the host gives every (device, stream) a pair and alternates launches
    // between them; each launch zeroes the other one (the next launch's) once its
    // griddepcontrol.wait has returned, so no launch ends with atomics and a successor
    // (stream order, PDL included) always starts from zero.
    unsigned* const sched = ka.sched;
    const bool dyn = sched != nullptr;
    __shared__ int64_t s_tile[S];
    const int64_t my_tiles = dyn ? INT64_MAX
        : (ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0);
    const bool leader = threadIdx.x == 0;
    uint64_t policy = 0;
    unsigned long long bad = 0;
    bool claiming = true;  // leader: no -1 claimed yet
    unsigned ahead = 0;    // leader: the next batch of the dynamic schedule, claimed one
                           // batch early so the atomic's round trip overlaps tiles of work
    int64_t cur = 0, end = 0;  // leader: the batch being handed out, [cur, end)
    const int batch = dyn ? ka.sched_batch : 1;  // tiles per claim (fewer atomics on big runs)
    auto claim = [&](int64_t k) -> int64_t {  // tile of the CTA's k-th stage fill (leader)
        int64_t t;
        if (k < S) {
            t = (int64_t)blockIdx.x + k * gridDim.x;
        } else {
            if (cur == end) {
                cur = (int64_t)S * gridDim.x + (int64_t)ahead * batch;
                end = cur + batch;
                if (cur < ntiles) ahead = atomicAdd(&sched[0], 1u);
            }
            t = cur++;
        }
        return t < ntiles ? t : -1;
    };

    if (leader) {
        policy = policy_evict_first();
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    grid_dependency_wait();
    grid_launch_dependents();
    if (dyn && blockIdx.x == 0 && threadIdx.x == 0 && ka.sched_next != nullptr) *ka.sched_next = 0u;
    timeline_mark(1);
    // One stage = the tile's input records (and its second-input records), one mbarrier.
    auto load_stage = [&](int st, int64_t tile) {
        if constexpr (MIS) {
            mbar_arrive_expect_tx(&full[st], load_bytes + (N2 > 0 ? load2_bytes : 0));
            bulk_load_plain(s_in + st * L::kStageBytes, xa + tile * L::kInBytes, load_bytes, &full[st]);
            if constexpr (N2 > 0)
                bulk_load_plain(s_in2 + st * L::kIn2StageBytes, x2a + tile * L::kIn2Bytes, load2_bytes, &full[st]);
        } else {
            mbar_arrive_expect_tx(&full[st], L::kInBytes + L::kIn2Bytes);
            if (HINTS & 1)
                bulk_load(s_in + st * L::kInBytes, x + tile * TR * LDX, L::kInBytes, &full[st], policy);
            else
                bulk_load_plain(s_in + st * L::kInBytes, x + tile * TR * LDX, L::kInBytes, &full[st]);
            if constexpr (N2 > 0)
                bulk_load_plain(s_in2 + st * L::kIn2Bytes, x2 + tile * TR * N2, L::kIn2Bytes, &full[st]);
        }
    };
    // Dynamic schedule: fill stage st with the CTA's k-th tile, or mark it empty.
    auto fill_dyn = [&](int st, int64_t k) {
        if (!claiming) return;
        const int64_t t = claim(k);
        s_tile[st] = t;
        if (t >= 0) {
            load_stage(st, t);
        } else {
            claiming = false;
            mbar_arrive(&full[st]);  // completes the phase with no bytes: "no tile"
        }
    };
    if (leader) {
        if (dyn) {
            for (int k = 0; k < S; ++k) fill_dyn(k, k);
            if (claiming) ahead = atomicAdd(&sched[0], 1u);
        } else {
            for (int64_t k = 0; k < my_tiles && k < S; ++k) load_stage((int)k, (int64_t)blockIdx.x + k * gridDim.x);
        }
    }

    for (int64_t k = 0; k < my_tiles; ++k) {
        const int s = (int)(k % S);
        const uint32_t parity = (uint32_t)((k / S) & 1);
        const int ob = (int)(k % OB);
        mbar_wait(&full[s], parity);
        const int64_t tile = dyn ? s_tile[s] : (int64_t)blockIdx.x + k * gridDim.x;
        if (tile < 0) break;  // dynamic schedule exhausted (uniform across the CTA)
        if (k == 0) timeline_mark(2);
        timeline_tile(k, 0, threadIdx.x == 0);

        const T* tin = reinterpret_cast<const T*>(s_in + s * L::kStageBytes + (MIS ? mis : 0));
        const T* tin2 = reinterpret_cast<const T*>(s_in2 + s * L::kIn2StageBytes + (MIS ? mis2 : 0));
        T* t0 = reinterpret_cast<T*>(s_out + ob * L::kOutBytes);
        T* t1 = t0 + TR * W0;
        T* t2 = t1 + TR * W1;
        auto row = [&](int j) {
            T xr[N], x2r[Slot<N2>::value], o0[Slot<W0>::value], o1[Slot<W1>::value], o2[Slot<W2>::value];
#pragma unroll
            for (int c = 0; c < N; ++c) xr[c] = tin[j * LDX + c];
#pragma unroll
            for (int c = 0; c < N2; ++c) x2r[c] = tin2[j * N2 + c];
            bad += apply_op<Op>(xr, x2r, ka, o0, o1, o2) ? 0 : 1;
#pragma unroll
            for (int c = 0; c < W0; ++c) t0[j * W0 + c] = o0[c];
#pragma unroll
            for (int c = 0; c < W1; ++c) t1[j * W1 + c] = o1[c];
#pragma unroll
            for (int c = 0; c < W2; ++c) t2[j * W2 + c] = o2[c];
        };
        if constexpr (TR >= NT) {
            static_assert(TR % NT == 0, "a tile is a whole number of rows per thread");
#pragma unroll
            for (int it = 0; it < TR / NT; ++it) row((int)threadIdx.x + it * NT);  // no guard
        } else {
            if ((int)threadIdx.x < TR) row((int)threadIdx.x);
        }
        fence_proxy_async_smem();  // generic-proxy smem traffic -> visible to bulk copies
        __syncthreads();
        timeline_tile(k, 1, threadIdx.x == 0);
        if (leader) {
            const int64_t row0 = tile * TR;
            if (HINTS & 2) {
                bulk_store_hint(head + row0 * W0, t0, L::kB0, policy);
                if (W1) bulk_store_hint(body + row0 * W1, t1, L::kB1, policy);
                if (W2) bulk_store_hint(extra + row0 * W2, t2, L::kB2, policy);
            } else {
                bulk_store(head + row0 * W0, t0, L::kB0);
                if (W1) bulk_store(body + row0 * W1, t1, L::kB1);
                if (W2) bulk_store(extra + row0 * W2, t2, L::kB2);
            }
            bulk_commit();
            if (dyn)
                fill_dyn(s, k + S);
            else if (k + S < my_tiles)
                load_stage(s, tile + (int64_t)S * gridDim.x);
            // Threads write staging tile (k+2) % OB after the next __syncthreads, so group
            // k+2-OB must have been read out by then: at most OB-2 groups stay pending.
            bulk_wait_read<OB - 2>();
            timeline_tile(k, 2, true);
        }
    }

    // Rows after the last full tile: plain per-thread path in the last CTA (the loop
    // runs the same trip count on every lane of a warp so count_invalid can shuffle).
    if (blockIdx.x == gridDim.x - 1) {
        const int64_t tail = nrows - ntiles * TR;
        for (int64_t j = threadIdx.x & ~31; j < tail; j += NT) {
            const int64_t i = ntiles * TR + j + (threadIdx.x & 31);
            if (i < nrows) bad += row_global<T, N, OP>(x, x2, i, head, body, extra, ka, LDX) ? 0 : 1;
        }
    }
    timeline_mark(3);
    count_invalid(ka.invalid, bad);
    if (leader) {
        sched_report_done(ka);
        bulk_wait_all();
    }
    timeline_mark(4);
}

// ---------------------------------------------------------------------------------
// Many independent batches in one launch (fn_run_many): a table of segments, each a
// dense 16-byte aligned [rows, N] array with its own outputs.  Global tile g belongs to
// the segment whose tile range holds it (tile0 prefix sums, searched per tile); the
// same ring / mbarrier / store-group pipeline as tma_stream_kernel streams the tiles of
// all segments back to back, so a stream of small batches pays one launch ramp and one
// tail instead of one per batch.  Rows after a segment's last whole tile go through
// the per-row path, one segment per CTA, after the streaming loop.
// ---------------------------------------------------------------------------------
constexpr int kMaxSegments = 48;
template <typename T> struct Segment {
    const T* x;
    T *head, *body, *extra;
    int64_t rows;
    int64_t tile0;  // first global tile of the segment
};
template <typename T> struct SegmentTable {
    Segment<T> seg[kMaxSegments];
    int nseg;
    int64_t ntiles;  // whole tiles of all segments
};

// A CTA visits its tiles in increasing order, so the segment of each tile is found by
// moving a cursor forward, with the current segment held in registers: the leader's
// per-tile work stays a compare (a binary search over the table per tile, on the
// leader's critical path, cost 40 % on a stream of 1e6-row batches).
template <typename T> struct SegmentCursor {
    int cur = -1;
    int64_t next = 0;  // first tile of the segment after cur
    Segment<T> s;
    __device__ __forceinline__ void advance(const SegmentTable<T>& t, int64_t g) {
        while (g >= next) {
            ++cur;
            s = t.seg[cur];
            next = cur + 1 < t.nseg ? t.seg[cur + 1].tile0 : INT64_MAX;
        }
    }
};

template <typename T, int N, int OP, int TR_ = OpRows<T, N, OP, false>::value,
          int S_ = OpStages<T, N, OP, false>::value, int NT = Tile<T, N>::kThreads>
__global__ void __launch_bounds__(NT) tma_segments_kernel(const __grid_constant__ SegmentTable<T> tab,
                                                          KArgs<T> ka) {
    using L = TileLayout<T, N, OP, TR_, S_>;
    using Op = typename L::Op;
    static_assert(InWidth2<Op>::value == 0, "single-input ops");
    constexpr int TR = L::TR, S = L::S, OB = L::OB;
    constexpr int W0 = Op::W0, W1 = Op::W1, W2 = Op::W2;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* s_in = smem;
    unsigned char* s_out = smem + S * L::kInBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(s_out + OB * L::kOutBytes);
    const int64_t ntiles = tab.ntiles;
    // Tile schedule: static round-robin, or (ka.sched != NULL) tma_stream_kernel's dynamic
    // one.  Either way a CTA's tiles come in increasing order, which the cursors need.
    unsigned* const sched = ka.sched;
    const bool dyn = sched != nullptr;
    __shared__ int64_t s_tile[S];
    const int64_t my_tiles = dyn ? INT64_MAX
        : (ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0);
    const bool leader = threadIdx.x == 0;
    unsigned long long bad = 0;
    bool claiming = true;
    unsigned ahead = 0;
    int64_t cur = 0, end = 0;
    const int batch = dyn ? ka.sched_batch : 1;
    auto claim = [&](int64_t k) -> int64_t {
        int64_t t;
        if (k < S) {
            t = (int64_t)blockIdx.x + k * gridDim.x;
        } else {
            if (cur == end) {
                cur = (int64_t)S * gridDim.x + (int64_t)ahead * batch;
                end = cur + batch;
                if (cur < ntiles) ahead = atomicAdd(&sched[0], 1u);
            }
            t = cur++;
        }
        return t < ntiles ? t : -1;
    };
    if (leader) {
#pragma unroll
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        fence_barrier_init();
    }
    __syncthreads();
    grid_dependency_wait();
    grid_launch_dependents();
    if (dyn && blockIdx.x == 0 && threadIdx.x == 0 && ka.sched_next != nullptr) *ka.sched_next = 0u;
    SegmentCursor<T> lc, sc;  // segment cursors of the loads (S tiles ahead) and the stores
    auto load_stage = [&](int st, int64_t g) {
        lc.advance(tab, g);
        const Segment<T>& sg = lc.s;
        mbar_arrive_expect_tx(&full[st], L::kInBytes);
        bulk_load_plain(s_in + st * L::kInBytes, sg.x + (g - sg.tile0) * TR * N, L::kInBytes, &full[st]);
    };
    auto fill_dyn = [&](int st, int64_t k) {
        if (!claiming) return;
        const int64_t t = claim(k);
        s_tile[st] = t;
        if (t >= 0) {
            load_stage(st, t);
        } else {
            claiming = false;
            mbar_arrive(&full[st]);  // completes the phase with no bytes: "no tile"
        }
    };
    if (leader) {
        if (dyn) {
            for (int k = 0; k < S; ++k) fill_dyn(k, k);
            if (claiming) ahead = atomicAdd(&sched[0], 1u);
        } else {
            for (int64_t k = 0; k < my_tiles && k < S; ++k) load_stage((int)k, (int64_t)blockIdx.x + k * gridDim.x);
        }
    }
    for (int64_t k = 0; k < my_tiles; ++k) {
        const int st = (int)(k % S), ob = (int)(k % OB);
        mbar_wait(&full[st], (uint32_t)((k / S) & 1));
        const int64_t g = dyn ? s_tile[st] : (int64_t)blockIdx.x + k * gridDim.x;
        if (g < 0) break;  // dynamic schedule exhausted (uniform across the CTA)
        const T* tin = reinterpret_cast<const T*>(s_in + st * L::kInBytes);
        T* t0 = reinterpret_cast<T*>(s_out + ob * L::kOutBytes);
        T* t1 = t0 + TR * W0;
        T* t2 = t1 + TR * W1;
        auto row = [&](int j) {
            T xr[N], o0[Slot<W0>::value], o1[Slot<W1>::value], o2[Slot<W2>::value];
#pragma unroll
            for (int c = 0; c < N; ++c) xr[c] = tin[j * N + c];
            bad += Op::apply(xr, ka, o0, o1, o2) ? 0 : 1;
#pragma unroll
            for (int c = 0; c < W0; ++c) t0[j * W0 + c] = o0[c];
#pragma unroll
            for (int c = 0; c < W1; ++c) t1[j * W1 + c] = o1[c];
#pragma unroll
            for (int c = 0; c < W2; ++c) t2[j * W2 + c] = o2[c];
        };
        if constexpr (TR >= NT) {
#pragma unroll
            for (int it = 0; it < TR / NT; ++it) row((int)threadIdx.x + it * NT);
        } else {
            if ((int)threadIdx.x < TR) row((int)threadIdx.x);
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (leader) {
            sc.advance(tab, g);
            const Segment<T>& sg = sc.s;
            const int64_t row0 = (g - sg.tile0) * TR;
            bulk_store(sg.head + row0 * W0, t0, L::kB0);
            if (W1) bulk_store(sg.body + row0 * W1, t1, L::kB1);
            if (W2) bulk_store(sg.extra + row0 * W2, t2, L::kB2);
            bulk_commit();
            if (dyn)
                fill_dyn(st, k + S);
            else if (k + S < my_tiles)
                load_stage(st, g + (int64_t)S * gridDim.x);
            bulk_wait_read<OB - 2>();
        }
    }
    if (leader) sched_report_done(ka);
    // rows after each segment's last whole tile: segment j in CTA j % gridDim.x
    for (int j = (int)blockIdx.x; j < tab.nseg; j += (int)gridDim.x) {
        const Segment<T>& sg = tab.seg[j];
        const int64_t r0 = sg.rows / TR * TR;
        for (int64_t i = r0 + (int64_t)threadIdx.x; i < sg.rows; i += NT)
            bad += row_global<T, N, OP>(sg.x, nullptr, i, sg.head, sg.body, sg.extra, ka) ? 0 : 1;
    }
    (void)bad;  // single-input scaling / baseline ops never reject a row
    if (leader) bulk_wait_all();
}

// ---------------------------------------------------------------------------------
// Structure-of-arrays rows through the bulk-copy pipeline: a tile is TR rows of every
// component array (one bulk load per array into a per-array smem run), outputs are
// staged per array and written with one bulk store each.  Same ring / mbarrier /
// store-group protocol as tma_stream_kernel.
// ---------------------------------------------------------------------------------
// 4 KiB runs x 3 stages: 0.96 of the copy peak for normalize2/3 f64 and normalize3 f32
// under round 1's static schedule at 2 CTAs per SM (2 KiB runs: 0.84-0.94; 8 KiB:
// 0.90-1.02; profiles/r01da_soa.txt).  With the dynamic schedule (round 2) the same
// geometry reaches 6870-6910 GB/s (1.06-1.07; profiles/r02ae_soa_ab.txt) with up to 3
// CTAs per SM where the shared memory holds them (the host clamps to what fits).
#ifndef FNB_SOA_RUN_BYTES
#define FNB_SOA_RUN_BYTES 4096
#endif
#ifndef FNB_SOA_STAGES
#define FNB_SOA_STAGES 3
#endif
#ifndef FNB_SOA_CTAS_PER_SM
#define FNB_SOA_CTAS_PER_SM 3
#endif
template <typename T, int N, int OP, bool MIS = false> struct SoaTile {
    using Op = RowOp<T, N, OP>;
    static constexpr int TR = FNB_SOA_RUN_BYTES / (int)sizeof(T);  // one run of every array per tile
    static constexpr int S = FNB_SOA_STAGES, OB = 3, NT = 256;
    static constexpr int kCtasPerSm = FNB_SOA_CTAS_PER_SM;
    static constexpr int kOutArrays = 1 + Op::W1 + Op::W2;
    static constexpr int kArr = TR * (int)sizeof(T);           // bytes of one array's run
    static constexpr int kArrStage = kArr + (MIS ? 128 : 0);    // + room for a misaligned array
    static constexpr int kInBytes = N * kArrStage, kOutBytes = kOutArrays * kArr;
    static constexpr int kSmemBytes = S * kInBytes + OB * kOutBytes + S * 8;
};

// A component array whose storage is off the 16-byte grid (a[1:] of an array) is
// loaded like tma_stream_kernel's misaligned rows: from the boundary below the run,
// 16 bytes longer, read at the offset.  The host keeps every tile's reach inside the
// arrays (ntiles is computed with it) and requires 16-byte aligned outputs.
template <typename T, int N, int OP, bool MIS = false>
__global__ void __launch_bounds__(256) tma_soa_kernel(SoaPtrs<T, N> p, int64_t ntiles, KArgs<T> ka) {
    using L = SoaTile<T, N, OP, MIS>;
    using Op = typename L::Op;
    constexpr int TR = L::TR, S = L::S, OB = L::OB, NT = L::NT;
    constexpr int W1 = Op::W1, W2 = Op::W2;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* s_in = smem;
    unsigned char* s_out = smem + S * L::kInBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(s_out + OB * L::kOutBytes);
    // Tile schedule: static round-robin, or (ka.sched != NULL) tma_stream_kernel's dynamic
    // one -- the CTA's first S tiles static, then ka.sched_batch tiles per atomic claim,
    // one claim ahead of use, tile ids handed to the threads through s_tile[].
    unsigned* const sched = ka.sched;
    const bool dyn = sched != nullptr;
    __shared__ int64_t s_tile[S];
    const int64_t my_tiles = dyn ? INT64_MAX
        : (ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0);
    const bool leader = threadIdx.x == 0;
    bool claiming = true;
    unsigned ahead = 0;
    int64_t cur = 0, end = 0;
    const int batch = dyn ? ka.sched_batch : 1;
    auto claim = [&](int64_t k) -> int64_t {
        int64_t t;
        if (k < S) {
            t = (int64_t)blockIdx.x + k * gridDim.x;
        } else {
            if (cur == end) {
                cur = (int64_t)S * gridDim.x + (int64_t)ahead * batch;
                end = cur + batch;
                if (cur < ntiles) ahead = atomicAdd(&sched[0], 1u);
            }
            t = cur++;
        }
        return t < ntiles ? t : -1;
    };
    int mis[N];
    uint32_t tx = 0;
#pragma unroll
    for (int c = 0; c < N; ++c) {
        mis[c] = MIS ? (int)(reinterpret_cast<uintptr_t>(p.x[c]) & 15) : 0;
        tx += L::kArr + (mis[c] ? 16 : 0);
    }
    if (leader) {
#pragma unroll
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        fence_barrier_init();
    }
    __syncthreads();
    grid_dependency_wait();
    grid_launch_dependents();
    if (dyn && blockIdx.x == 0 && threadIdx.x == 0 && ka.sched_next != nullptr) *ka.sched_next = 0u;
    auto load_stage = [&](int st, int64_t tile) {
        mbar_arrive_expect_tx(&full[st], tx);
#pragma unroll
        for (int c = 0; c < N; ++c)
            bulk_load_plain(s_in + st * L::kInBytes + c * L::kArrStage,
                            reinterpret_cast<const unsigned char*>(p.x[c]) - mis[c] + tile * L::kArr,
                            L::kArr + (mis[c] ? 16 : 0), &full[st]);
    };
    auto fill_dyn = [&](int st, int64_t k) {
        if (!claiming) return;
        const int64_t t = claim(k);
        s_tile[st] = t;
        if (t >= 0) {
            load_stage(st, t);
        } else {
            claiming = false;
            mbar_arrive(&full[st]);  // completes the phase with no bytes: "no tile"
        }
    };
    if (leader) {
        if (dyn) {
            for (int k = 0; k < S; ++k) fill_dyn(k, k);
            if (claiming) ahead = atomicAdd(&sched[0], 1u);
        } else {
            for (int64_t k = 0; k < my_tiles && k < S; ++k) load_stage((int)k, (int64_t)blockIdx.x + k * gridDim.x);
        }
    }
    for (int64_t k = 0; k < my_tiles; ++k) {
        const int st = (int)(k % S);
        const int ob = (int)(k % OB);
        mbar_wait(&full[st], (uint32_t)((k / S) & 1));
        const int64_t tile = dyn ? s_tile[st] : (int64_t)blockIdx.x + k * gridDim.x;
        if (tile < 0) break;  // dynamic schedule exhausted (uniform across the CTA)
        const unsigned char* tin = s_in + st * L::kInBytes;
        T* tout = reinterpret_cast<T*>(s_out + ob * L::kOutBytes);
#pragma unroll
        for (int it = 0; it < TR / NT; ++it) {
            const int j = (int)threadIdx.x + it * NT;
            T xr[N], o0[1], o1[Slot<W1>::value], o2[1];
#pragma unroll
            for (int c = 0; c < N; ++c)
                xr[c] = *reinterpret_cast<const T*>(tin + c * L::kArrStage + mis[c] + j * (int)sizeof(T));
            (void)Op::apply(xr, ka, o0, o1, o2);
            tout[j] = o0[0];
#pragma unroll
            for (int c = 0; c < W1; ++c) tout[(1 + c) * TR + j] = o1[c];
            if constexpr (W2 == 1) tout[(1 + W1) * TR + j] = o2[0];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (leader) {
            const int64_t row0 = tile * TR;
            bulk_store(p.head + row0, tout, L::kArr);
#pragma unroll
            for (int c = 0; c < W1; ++c) bulk_store(p.body[c] + row0, tout + (1 + c) * TR, L::kArr);
            if constexpr (W2 == 1) bulk_store(p.extra + row0, tout + (1 + W1) * TR, L::kArr);
            bulk_commit();
            if (dyn)
                fill_dyn(st, k + S);
            else if (k + S < my_tiles)
                load_stage(st, tile + (int64_t)S * gridDim.x);
            bulk_wait_read<OB - 2>();
        }
    }
    if (leader) {
        sched_report_done(ka);
        bulk_wait_all();
    }
}

}  // namespace fnb
