// ws_kernel.cuh -- developer experiment, not part of the library: a warp-specialised
// form of fnb::tma_stream_kernel (one producer warp for the bulk copies, compute warps
// synchronised only through mbarriers).  Measured against the library kernel in
// profiles/r01s14_ws_tune.csv (steady state, 2^28 rows) and r01s15_lone.txt (config-1
// lone launches): no better in either, so the library keeps tma_stream_kernel.
#pragma once
#include "../paper_1606_06508_b200/csrc/stream_kernel.cuh"

namespace fnb {

// ---------------------------------------------------------------------------------
// Warp-specialised form of tma_stream_kernel (same tiles, same RowOp, same outputs):
// NT compute threads plus one producer warp, synchronised only through mbarriers.
//   full[s]    input stage s landed (expect_tx, arrived by the producer);
//   empty[s]   every compute warp has read stage s (NT/32 arrivals);
//   staged[o]  every compute warp has written output staging tile o and fenced it
//              for the async proxy (NT/32 arrivals);
//   ofree[o]   the bulk stores of staging tile o have read it out (1 arrival).
// A compute warp moves to its next tile as soon as that tile's input has landed and its
// staging tile is free; there is no CTA-wide barrier per tile, so one warp's arithmetic
// overlaps another's wait and the producer's store read-out.  Lane 0 of the producer
// warp issues every bulk copy: stores of tile k once staged[k] completes, then the
// refill of tile k's input stage once empty[k] completes.
// ---------------------------------------------------------------------------------
template <typename T, int N, int OP, int TR_ = OpRows<T, N, OP>::value, int S_ = OpStages<T, N, OP>::value,
          int NT = Tile<T, N>::kThreads, int OB_ = OutTiles<OP>::value, int LDX_ = 0>
__global__ void __launch_bounds__(NT + 32) tma_ws_kernel(const T* __restrict__ x, const T* __restrict__ x2,
                                                         int64_t nrows, T* __restrict__ head,
                                                         T* __restrict__ body, T* __restrict__ extra,
                                                         KArgs<T> ka) {
    using L = TileLayout<T, N, OP, TR_, S_, OB_, LDX_>;
    using Op = typename L::Op;
    constexpr int TR = L::TR, S = L::S, OB = L::OB, LDX = L::LDX;
    constexpr int W0 = Op::W0, W1 = Op::W1, W2 = Op::W2;
    constexpr int N2 = InWidth2<Op>::value;
    constexpr int kWarps = NT / 32;
    static_assert(NT % 32 == 0 && (TR % NT == 0 || TR < NT), "whole rows per thread");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* s_in = smem;
    unsigned char* s_in2 = smem + S * L::kInBytes;
    unsigned char* s_out = s_in2 + S * L::kIn2Bytes;
    // kSmemBytes reserves S * 8 bytes of barriers; this kernel needs 2S + 2*OB words,
    // placed after them (the launch adds (S + 2 * OB) * 8 bytes).
    uint64_t* full = reinterpret_cast<uint64_t*>(s_out + OB * L::kOutBytes);
    uint64_t* empty = full + S;
    uint64_t* staged = empty + S;
    uint64_t* ofree = staged + OB;

    const int64_t ntiles = (LDX == N ? nrows : nrows - 1) / TR;
    const int64_t my_tiles =
        ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
    const int warp = (int)threadIdx.x >> 5, lane = (int)threadIdx.x & 31;
    const bool producer = warp == kWarps;

    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kWarps);
        }
#pragma unroll
        for (int i = 0; i < OB; ++i) {
            mbar_init(&staged[i], kWarps);
            mbar_init(&ofree[i], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    timeline_mark(0);
    grid_dependency_wait();
    grid_launch_dependents();
    timeline_mark(1);

    if (producer) {
        if (lane == 0) {
            auto load = [&](int st, int64_t tile) {
                mbar_arrive_expect_tx(&full[st], L::kInBytes + L::kIn2Bytes);
                bulk_load_plain(s_in + st * L::kInBytes, x + tile * TR * LDX, L::kInBytes, &full[st]);
                if constexpr (N2 > 0)
                    bulk_load_plain(s_in2 + st * L::kIn2Bytes, x2 + tile * TR * N2, L::kIn2Bytes, &full[st]);
            };
            for (int64_t k = 0; k < my_tiles && k < S; ++k) load((int)k, (int64_t)blockIdx.x + k * gridDim.x);
            for (int64_t k = 0; k < my_tiles; ++k) {
                const int st = (int)(k % S), ob = (int)(k % OB);
                const int64_t tile = (int64_t)blockIdx.x + k * gridDim.x;
                // refill tile k's input stage as soon as every warp has read it ...
                if (k + S < my_tiles) {
                    mbar_wait(&empty[st], (uint32_t)((k / S) & 1));
                    load(st, tile + (int64_t)S * gridDim.x);
                }
                // ... then store tile k once every warp has staged its rows
                mbar_wait(&staged[ob], (uint32_t)((k / OB) & 1));
                const int64_t row0 = tile * TR;
                T* t0 = reinterpret_cast<T*>(s_out + ob * L::kOutBytes);
                bulk_store(head + row0 * W0, t0, L::kB0);
                if (W1) bulk_store(body + row0 * W1, t0 + TR * W0, L::kB1);
                if (W2) bulk_store(extra + row0 * W2, t0 + TR * (W0 + W1), L::kB2);
                bulk_commit();
                // the group before this one has been read out: its staging tile is free
                bulk_wait_read<1>();
                if (k >= 1) mbar_arrive(&ofree[(int)((k - 1) % OB)]);
                timeline_tile(k, 2);
            }
            bulk_wait_all();
        }
    } else {
        unsigned long long bad = 0;
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int st = (int)(k % S), ob = (int)(k % OB);
            constexpr int kRows = TR >= NT ? TR / NT : 1;  // rows per thread per tile
            const bool active = TR >= NT || (int)threadIdx.x < TR;
            mbar_wait(&full[st], (uint32_t)((k / S) & 1));
            timeline_tile(k, 0, threadIdx.x == 0);
            // inputs into registers, then the stage goes back to the producer
            const T* tin = reinterpret_cast<const T*>(s_in + st * L::kInBytes);
            const T* tin2 = reinterpret_cast<const T*>(s_in2 + st * L::kIn2Bytes);
            T xr[kRows][N], x2r[kRows][Slot<N2>::value];
#pragma unroll
            for (int it = 0; it < kRows; ++it) {
                const int j = (int)threadIdx.x + it * NT;
                if (active) {
#pragma unroll
                    for (int c = 0; c < N; ++c) xr[it][c] = tin[j * LDX + c];
#pragma unroll
                    for (int c = 0; c < N2; ++c) x2r[it][c] = tin2[j * N2 + c];
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (k >= OB) mbar_wait(&ofree[ob], (uint32_t)(((k / OB) - 1) & 1));
            T* t0 = reinterpret_cast<T*>(s_out + ob * L::kOutBytes);
            T* t1 = t0 + TR * W0;
            T* t2 = t1 + TR * W1;
#pragma unroll
            for (int it = 0; it < kRows; ++it) {
                const int j = (int)threadIdx.x + it * NT;
                if (active) {
                    T o0[Slot<W0>::value], o1[Slot<W1>::value], o2[Slot<W2>::value];
                    bad += apply_op<Op>(xr[it], x2r[it], ka, o0, o1, o2) ? 0 : 1;
#pragma unroll
                    for (int c = 0; c < W0; ++c) t0[j * W0 + c] = o0[c];
#pragma unroll
                    for (int c = 0; c < W1; ++c) t1[j * W1 + c] = o1[c];
#pragma unroll
                    for (int c = 0; c < W2; ++c) t2[j * W2 + c] = o2[c];
                }
            }
            fence_proxy_async_smem();  // this thread's staging writes -> async proxy
            __syncwarp();
            if (lane == 0) mbar_arrive(&staged[ob]);
            timeline_tile(k, 1, threadIdx.x == 0);
        }
        // Rows after the last full tile: per-thread path in the last CTA's compute warps.
        if (blockIdx.x == gridDim.x - 1) {
            const int64_t tail = nrows - ntiles * TR;
            for (int64_t j = threadIdx.x & ~31; j < tail; j += NT) {
                const int64_t i = ntiles * TR + j + lane;
                if (i < nrows) bad += row_global<T, N, OP>(x, x2, i, head, body, extra, ka, LDX) ? 0 : 1;
            }
        }
        count_invalid(ka.invalid, bad);
    }
    timeline_mark(3);
    timeline_mark(4);
}

}  // namespace fnb
