// fastnorm_kernels.cu -- launch plumbing and the C ABI (include/fastnorm_b200.h).
// The kernels themselves live in stream_kernel.cuh (memory path) and fastnorm_math.cuh
// (per-row arithmetic).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <string>
#include <type_traits>
#include <vector>

#include "stream_kernel.cuh"
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

// Output record widths (elements per row) of the three output arrays of an op.
struct Widths {
    int w0, w1, w2;
};
static Widths op_widths(int op, int dim) {
    switch (op) {
        case FN_OP_NORM: return {1, 0, 0};
        case FN_OP_NORMALIZE_SQ: return {1, dim, 1};
        case FN_OP_ROT_UNIT:
        case FN_OP_ROT_GENERAL: return {9, 0, 0};
        case FN_OP_NORMALIZE_ROT: return {1, 4, 9};
        case FN_OP_ROT_APPLY:
        case FN_OP_QUAT_ROTATE:
        case FN_OP_MAT_APPLY: return {3, 0, 0};
        default: return {1, dim, 0};
    }
}
static bool is_rotation(int op) {
    return op == FN_OP_ROT_UNIT || op == FN_OP_ROT_GENERAL || op == FN_OP_NORMALIZE_ROT ||
           op == FN_OP_ROT_APPLY;
}

// Per-instantiation occupancy (computed once per process and device).
template <typename T, int N, int OP, int LDX = 0, bool MIS = false, bool BIG = true> struct TmaLaunch {
    static constexpr int kThreads = OpThreads<T, N, OP, BIG>::value;
    using L = TileLayout<T, N, OP, OpRows<T, N, OP, BIG>::value, OpStages<T, N, OP, BIG>::value, OutTiles<OP>::value,
                         LDX, MIS>;
    static constexpr auto kernel() {
        return tma_stream_kernel<T, N, OP, OpRows<T, N, OP, BIG>::value, OpStages<T, N, OP, BIG>::value, kThreads,
                                 Tile<T, N>::kHints, OutTiles<OP>::value, LDX, MIS>;
    }
    static int blocks_per_sm(int dev) {
        static std::mutex mu;
        static int cache[64] = {0};
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 0 || dev >= 64) return 1;
        if (cache[dev] == 0) {
            auto kern = kernel();
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemBytes);
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads,
                                                              L::kSmemBytes) != cudaSuccess ||
                nb < 1)
                nb = 1;
            cache[dev] = nb;
        }
        return cache[dev];
    }
};

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// Launch-shape overrides read once from the environment (function-local statics:
// thread-safe initialisation):
//   FASTNORM_B200_PATH=direct       force the per-row kernel (diagnostics)
//   FASTNORM_B200_CTAS_PER_SM=<k>   CTAs per SM for the streaming kernel (experiments)
// The zero-copy small-batch host path (rows in mapped page-locked memory) asks for the
// per-row kernel on its own thread.
static thread_local bool tl_direct = false;

static bool force_direct() {
    static const bool v = [] {
        const char* e = getenv("FASTNORM_B200_PATH");
        return e && strcmp(e, "direct") == 0;
    }();
    return v || tl_direct;
}

static int cps_override() {
    static const int v = [] {
        const char* e = getenv("FASTNORM_B200_CTAS_PER_SM");
        return e ? atoi(e) : -1;
    }();
    return v;
}

// FASTNORM_B200_SCHED_BATCH=<k>: tiles per claim of the dynamic schedule (experiments).
static int sched_batch_override() {
    static const int v = [] {
        const char* e = getenv("FASTNORM_B200_SCHED_BATCH");
        return e ? atoi(e) : -1;
    }();
    return v;
}

// Kernels this library has launched, process-wide (fn_launch_count): the bench counts
// its launches inside a timed region from the library itself.
static std::atomic<int64_t> g_launches{0};

// Programmatic dependent launch for the streaming kernels (FASTNORM_B200_PDL=0 turns it
// off).  Back-to-back launches on a stream overlap one kernel's drain with the next one's
// launch and prologue; each kernel still waits (griddepcontrol.wait) for its
// predecessor before touching global memory, so stream order semantics are unchanged.
static bool pdl_enabled() {
    static const bool v = [] {
        const char* e = getenv("FASTNORM_B200_PDL");
        return !(e && strcmp(e, "0") == 0);
    }();
    return v;
}

template <typename... Params, typename... Args>
static cudaError_t launch_pdl(void (*kern)(Params...), int grid, int block, size_t smem,
                              cudaStream_t stream, Args... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

// CTAs per SM: the measured streaming optimum (CtasPerSm); small batches (few tiles per
// CTA) fill the machine with the occupancy maximum instead, to shorten the pipeline
// fill / drain.
template <typename T, int N, int OP>
static int ctas_per_sm_for(int64_t ntiles, int sms) {
    if (cps_override() > 0) return cps_override();
    const int64_t tiles_per_cta = ntiles / ((int64_t)CtasPerSm<T, N, OP>::value * sms);
    return tiles_per_cta < 32 ? 64 : CtasPerSm<T, N, OP>::value;
}

// Input records of LDX elements, N of them read per row (LDX > N only for N = 3, LDX = 4,
// the xyz-in-xyzw layout; other strides take the per-row kernel).
template <int N> struct PaddedLdx {
    static constexpr int value = N == 3 ? 4 : 0;
};

// Dynamic tile schedule (tma_stream_kernel): two tile counters per (device, stream),
// zeroed in stream order when the stream first uses them.  Launch i on the stream claims
// from counter i % 2 and zeroes counter (i + 1) % 2 for launch i + 1 after its
// griddepcontrol.wait, i.e. after launch i - 1 (the last user of that counter) is
// complete.  The host takes i and launches under one lock, so the counter order matches
// the stream order even when several threads launch on the same stream.  Launches on
// different streams never share counters.  Batches with at most S tiles per CTA (nothing
// to balance) take the static schedule; launches under stream capture take a counter of
// their own (capture_pair below).  The streaming, SoA and many-batch kernels share this
// code (sched_lease).  FASTNORM_B200_DYN=0 forces the static schedule everywhere.
static bool dyn_enabled() {
    static const bool v = [] {
        const char* e = getenv("FASTNORM_B200_DYN");
        return !(e && strcmp(e, "0") == 0);
    }();
    return v;
}

// Kernels that keep the static schedule: none by default.  Dynamic vs static, back-to-back
// launches, three boxes (profiles/r02h_ab_dyn.txt, r02j_ab_dyn.txt, r02k_steady.jsonl):
// +5 to +23 % on the quotient, norm, normalize2 and normalize4_sq kernels, +0.3 to +2 % on
// normalize3 f64 at 2^30 rows.  normalize3 f32 (config 4) lost 1.7 % at 2 CTAs per SM and
// kept the static schedule until it was measured at 3 CTAs per SM, where the dynamic
// schedule wins (6912 vs 6591 GB/s, profiles/r02ap_tables.txt); FNB_DYN_F32_NORMALIZE3=0
// builds the old choice.
#ifndef FNB_DYN_F32_NORMALIZE3
#define FNB_DYN_F32_NORMALIZE3 1
#endif
template <typename T, int N, int OP> struct DynamicSchedule {
    static constexpr bool value =
        FNB_DYN_F32_NORMALIZE3 || !(std::is_same<T, float>::value && N == 3 && OP == FN_OP_NORMALIZE);
};

struct SchedSlots {
    int dev;
    cudaStream_t stream;
    unsigned* ctr;       // two counters
    uint64_t launches;   // dynamic launches so far on this stream
    std::mutex mu;       // held from taking a launch index to the launch itself
};
static std::mutex g_sched_mu;
static std::vector<std::unique_ptr<SchedSlots>>* g_sched = new std::vector<std::unique_ptr<SchedSlots>>();

// Captured launches (CUDA graphs): a graph may be replayed on any stream, so a captured
// kernel node cannot share a stream's alternating pair.  It gets a {counter, done} pair of
// its own from a per-device pool, and its last CTA re-zeroes the pair for the node's next
// replay (sched_report_done).  The pool is allocated and zeroed by the device's first
// eager dynamic launch (cudaMalloc is not allowed while a stream captures); a capture
// before that, or after the pool's kCapturePairs pairs are handed out, takes the static
// schedule.  Two instances of one captured node running at the same time would share the
// pair -- and already race on their output buffers.  FASTNORM_B200_DYN_CAPTURE=0 keeps
// captured launches static.
constexpr int kCapturePairs = 16384;
struct CapturePool {
    unsigned* base = nullptr;
    int next = 0;
};
static std::vector<CapturePool>* g_capture = new std::vector<CapturePool>();  // by device, under g_sched_mu

static bool dyn_capture_enabled() {
    static const bool v = [] {
        const char* e = getenv("FASTNORM_B200_DYN_CAPTURE");
        return !(e && strcmp(e, "0") == 0);
    }();
    return v;
}

// Called without a capture in progress on `stream`, g_sched_mu held.
static void capture_pool_init(int dev, cudaStream_t stream) {
    if ((int)g_capture->size() <= dev) g_capture->resize(dev + 1);
    CapturePool& cp = (*g_capture)[dev];
    if (cp.base || cp.next < 0) return;
    unsigned* p = nullptr;
    const size_t bytes = (size_t)kCapturePairs * 2 * sizeof(unsigned);
    if (cudaMalloc(&p, bytes) != cudaSuccess || cudaMemsetAsync(p, 0, bytes, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess) {
        cudaGetLastError();
        if (p) cudaFree(p);
        cp.next = -1;  // do not try again
        return;
    }
    cp.base = p;
}

static unsigned* capture_pair(int dev) {
    std::lock_guard<std::mutex> lk(g_sched_mu);
    if (!dyn_capture_enabled() || (int)g_capture->size() <= dev) return nullptr;
    CapturePool& cp = (*g_capture)[dev];
    if (!cp.base || cp.next >= kCapturePairs) return nullptr;
    return cp.base + 2 * (cp.next++);
}

static bool stream_capturing(cudaStream_t stream, bool* known) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess) {
        cudaGetLastError();
        *known = false;
        return false;
    }
    *known = true;
    return cap != cudaStreamCaptureStatusNone;
}

// The per-stream pair of an eager launch (not capturing).
static SchedSlots* sched_slots(int dev, cudaStream_t stream) {
    std::lock_guard<std::mutex> lk(g_sched_mu);
    capture_pool_init(dev, stream);
    for (auto& e : *g_sched)
        if (e->dev == dev && e->stream == stream) return e.get();
    unsigned* p = nullptr;
    if (cudaMalloc(&p, 2 * sizeof(unsigned)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;  // static schedule instead
    }
    if (cudaMemsetAsync(p, 0, 2 * sizeof(unsigned), stream) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p);
        return nullptr;
    }
    std::unique_ptr<SchedSlots> e(new SchedSlots());
    e->dev = dev;
    e->stream = stream;
    e->ctr = p;
    e->launches = 0;
    g_sched->push_back(std::move(e));
    return g_sched->back().get();
}

// The tile schedule of one launch.  Fills kd.sched* (all NULL: static schedule) and, for an
// eager dynamic launch, holds the stream's lock until the launch is made; commit() after a
// successful launch advances the stream's alternation.
struct SchedLease {
    SchedSlots* slots = nullptr;
    std::unique_lock<std::mutex> lk;
    uint64_t i = 0;
    void commit() {
        if (slots) slots->launches = i + 1;
    }
};
// Tiles per atomic claim.  2 everywhere (measured against 1, 4, 8 and 16 on nine kernel /
// config pairs, profiles/r02t_sched_batch_table.txt: one tile per claim loses up to 25 %
// where many CTAs claim short tiles -- the counter's round trip is on every tile's path --
// and larger batches lose balance: normalize3 config 5 +3.7 % at 2, +2.3 % at 8 over the
// static schedule) except the norm kernels, which take 4: their tiles are the shortest
// (24 B in, 8 B out per row) and at 2 tiles per claim they fall into a slow mode on some
// boxes and builds (norm3 f64, 2^28 rows: 4900-5070 GB/s at 2, 7200 at 4, 7150 at 8, static
// 6460-6670; profiles/r02ak_norm3_batch.txt), while 4 costs 0.3 % where 2 runs well.
template <int OP> struct SchedBatch {
    static constexpr int value = OP == FN_OP_NORM ? 4 : 2;
};

// `tiles_per_cta`: whole tiles over resident CTAs.  Captured launches with fewer than 32
// (config-1-sized batches, where the schedule gains nothing in eager mode either) stay
// static: the report at the end of a self-resetting launch costs them ~1.4 us per launch
// (7.5 -> 8.9 us, profiles/r02ah_graph_dyn.jsonl).
template <typename T>
static SchedLease sched_lease(bool want, int batch, int64_t tiles_per_cta, int dev, cudaStream_t stream,
                              KArgs<T>& kd) {
    SchedLease l;
    kd.sched = kd.sched_next = kd.sched_done = nullptr;
    if (!want || !dyn_enabled()) return l;
    kd.sched_batch = sched_batch_override() > 0 ? sched_batch_override() : batch;
    bool known = false;
    if (stream_capturing(stream, &known)) {
        unsigned* pair = tiles_per_cta >= 32 ? capture_pair(dev) : nullptr;
        if (pair) {
            kd.sched = pair;
            kd.sched_done = pair + 1;
        }
        return l;
    }
    if (!known) return l;
    SchedSlots* slots = sched_slots(dev, stream);
    if (!slots) return l;
    l.slots = slots;
    l.lk = std::unique_lock<std::mutex>(slots->mu);
    l.i = slots->launches;
    kd.sched = slots->ctr + (l.i & 1);
    kd.sched_next = slots->ctr + ((l.i + 1) & 1);
    return l;
}

template <typename T, int N, int OP, int LDX, bool MIS, bool BIG>
static cudaError_t launch_tma_as(const T* x, const T* x2, int64_t n, T* head, T* body, T* extra,
                                 const KArgs<T>& ka, int dev, int sms, cudaStream_t stream) {
    using TL = TmaLaunch<T, N, OP, LDX, MIS, BIG>;
    using L = typename TL::L;
    const int64_t ntiles = n / L::TR;
    const int64_t per_sm = std::min<int64_t>(TL::blocks_per_sm(dev), ctas_per_sm_for<T, N, OP>(ntiles, sms));
    const int64_t resident = per_sm * sms;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, resident));
    KArgs<T> kd = ka;
    SchedLease lease = sched_lease(DynamicSchedule<T, N, OP>::value && ntiles > (int64_t)L::S * grid,
                                   SchedBatch<OP>::value, ntiles / grid, dev, stream, kd);
    const cudaError_t e = launch_pdl(TL::kernel(), grid, TL::kThreads, L::kSmemBytes, stream, x, x2, n,
                                     head, body, extra, kd);
    if (e == cudaSuccess) lease.commit();
    return e;
}

// MIS: the instantiation for inputs off the 16-byte grid (tma_stream_kernel).
// BIG: the large-batch geometry (Rows3); smaller batches take the default one when it
// differs (one more instantiation only for the kernels Rows3 changes).
template <typename T, int N, int OP, int LDX = 0>
static cudaError_t launch_tma(const T* x, const T* x2, int64_t n, T* head, T* body, T* extra, const KArgs<T>& ka,
                              int dev, int sms, cudaStream_t stream) {
    const bool mis = !aligned16(x) || (x2 && !aligned16(x2));
    if constexpr (Rows3<T, N, OP>::any) {
        if (n < kBigTileRows)
            return mis ? launch_tma_as<T, N, OP, LDX, true, false>(x, x2, n, head, body, extra, ka, dev, sms, stream)
                       : launch_tma_as<T, N, OP, LDX, false, false>(x, x2, n, head, body, extra, ka, dev, sms, stream);
    }
    return mis ? launch_tma_as<T, N, OP, LDX, true, true>(x, x2, n, head, body, extra, ka, dev, sms, stream)
               : launch_tma_as<T, N, OP, LDX, false, true>(x, x2, n, head, body, extra, ka, dev, sms, stream);
}

template <typename T, int N, int OP>
static int launch(const void* xv, const void* x2v, int64_t n, void* hv, void* bv, void* qv,
                  const KArgs<T>& ka, cudaStream_t stream, int64_t ldx = N) {
    using TL = TmaLaunch<T, N, OP, 0, false, false>;  // the geometry of the smallest batches it takes
    using L = typename TL::L;
    using Op = typename L::Op;
    const T* x = static_cast<const T*>(xv);
    T* head = static_cast<T*>(hv);
    T* body = static_cast<T*>(bv);
    T* extra = static_cast<T*>(qv);
    const T* x2 = static_cast<const T*>(x2v);
    constexpr int N2 = InWidth2<Op>::value;
    if (n == 0) return FN_OK;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const int sms = device_sms(dev);
    // The bulk-copy kernel needs 16-byte aligned outputs; inputs only need element
    // alignment: a misaligned input is loaded from the 16-byte boundary below each tile
    // (tma_stream_kernel).
    const bool x_ok = ((uintptr_t)x % sizeof(T)) == 0 && (N2 == 0 || ((uintptr_t)x2 % sizeof(T)) == 0);
    const bool aligned = x_ok && aligned16(head) && (Op::W1 == 0 || aligned16(body)) &&
                         (Op::W2 == 0 || aligned16(extra));
    constexpr int kPad = PaddedLdx<N>::value;
    if (aligned && !force_direct() && ldx == N && n >= (int64_t)L::TR) {
        e = launch_tma<T, N, OP>(x, x2, n, head, body, extra, ka, dev, sms, stream);
    } else if (kPad > 0 && N2 == 0 && aligned && !force_direct() && ldx == kPad && n > (int64_t)L::TR) {
        // (the branch is only reachable when the instantiation below exists)
        if constexpr (kPad > 0 && N2 == 0) e = launch_tma<T, N, OP, kPad>(x, x2, n, head, body, extra, ka, dev, sms, stream);
    } else {
        const int64_t want = (n + 255) / 256;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
        e = launch_pdl(direct_kernel<T, N, OP>, grid, 256, 0, stream, x, x2, n, head, body, extra, ka, ldx);
    }
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
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
    // Exponent insertion needs sigma = 2^k and inv = 2^-k exactly (validate_conditions
    // requires powers of two, and kernel_args passes exact inverses); otherwise the
    // kernels multiply, as the reference does for any parameter set.
    auto log2_exact = [](T v, int* k) {
        if (!(v > (T)0) || !std::isfinite(v)) return false;
        int e = 0;
        const T f = std::frexp(v, &e);
        *k = e - 1;
        return f == (T)0.5;
    };
    int kmin = 0, kmax = 0, kimin = 0, kimax = 0;
    out.pow2 = log2_exact(out.sigma_min, &kmin) && log2_exact(out.sigma_max, &kmax) &&
               log2_exact(out.inv_min, &kimin) && log2_exact(out.inv_max, &kimax) &&
               kimin == -kmin && kimax == -kmax && out.inv_min != out.inv_max &&
               out.inv_min != (T)1 && out.inv_max != (T)1;
    out.k_min = out.pow2 ? kmin : 0;
    out.k_max = out.pow2 ? kmax : 0;
    return FN_OK;
}

// Kernel arguments of an op: the six scaling constants, or for FN_OP_ROT_APPLY the nine
// matrix entries (the ka pointer of the ABI carries R there).
template <typename T>
static int make_kargs_op(int op, const double* ka, bool needed, KArgs<T>& out) {
    if (op != FN_OP_ROT_APPLY) return make_kargs<T>(ka, needed, out);
    memset(&out, 0, sizeof(out));
    if (!ka) return fail(FN_EINVAL, "FN_OP_ROT_APPLY needs the 9 matrix entries in ka");
    for (int k = 0; k < 9; ++k) out.rot[k] = (T)ka[k];
    return FN_OK;
}

template <typename T, int OP>
static int dispatch_dim(int dim, const void* x, int64_t n, void* h, void* b, void* q,
                        const KArgs<T>& ka, cudaStream_t s, int64_t ldx) {
    switch (dim) {
        case 2: return launch<T, 2, OP>(x, nullptr, n, h, b, q, ka, s, ldx);
        case 3: return launch<T, 3, OP>(x, nullptr, n, h, b, q, ka, s, ldx);
        case 4: return launch<T, 4, OP>(x, nullptr, n, h, b, q, ka, s, ldx);
        default: return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    }
}

static bool needs_ka(int op) {
    return op == FN_OP_SCALE || op == FN_OP_NORMALIZE || op == FN_OP_NORM ||
           op == FN_OP_NORMALIZE_SQ || op == FN_OP_ROT_GENERAL || op == FN_OP_NORMALIZE_ROT;
}

template <typename T>
static int dispatch(int op, int dim, const void* x, int64_t n, void* h, void* b, void* q,
                    const double* kad, unsigned long long* invalid, cudaStream_t s, int64_t ldx) {
    KArgs<T> ka;
    int rc = make_kargs<T>(kad, needs_ka(op), ka);
    if (rc != FN_OK) return rc;
    ka.invalid = invalid;
    switch (op) {
        case FN_OP_SCALE: return dispatch_dim<T, FN_OP_SCALE>(dim, x, n, h, b, q, ka, s, ldx);
        case FN_OP_NORMALIZE: return dispatch_dim<T, FN_OP_NORMALIZE>(dim, x, n, h, b, q, ka, s, ldx);
        case FN_OP_NORMALIZE_SQ:
            return dispatch_dim<T, FN_OP_NORMALIZE_SQ>(dim, x, n, h, b, q, ka, s, ldx);
        case FN_OP_NORM: return dispatch_dim<T, FN_OP_NORM>(dim, x, n, h, b, q, ka, s, ldx);
        case FN_OP_NAIVE: return dispatch_dim<T, FN_OP_NAIVE>(dim, x, n, h, b, q, ka, s, ldx);
        case FN_OP_QUOTIENT: return dispatch_dim<T, FN_OP_QUOTIENT>(dim, x, n, h, b, q, ka, s, ldx);
        case FN_OP_QUOTIENT3_FAST:
            if (dim != 3) return fail(FN_EINVAL, "quotient3_fast is defined for dim 3 only");
            return launch<T, 3, FN_OP_QUOTIENT3_FAST>(x, nullptr, n, h, b, q, ka, s, ldx);
        default: return fail(FN_EINVAL, "unknown op");
    }
}

// Rotations: quaternions in binary64 only (the reference computes them in Python floats).
static int dispatch_rot(int op, const void* x, int64_t n, void* h, void* b, void* q,
                        const double* kad, unsigned long long* invalid, cudaStream_t s, int64_t ldx) {
    KArgs<double> ka;
    int rc = make_kargs_op<double>(op, kad, needs_ka(op), ka);
    if (rc != FN_OK) return rc;
    ka.invalid = invalid;
    switch (op) {
        case FN_OP_ROT_UNIT: return launch<double, 4, FN_OP_ROT_UNIT>(x, nullptr, n, h, b, q, ka, s, ldx);
        case FN_OP_ROT_GENERAL: return launch<double, 4, FN_OP_ROT_GENERAL>(x, nullptr, n, h, b, q, ka, s, ldx);
        case FN_OP_NORMALIZE_ROT: return launch<double, 4, FN_OP_NORMALIZE_ROT>(x, nullptr, n, h, b, q, ka, s, ldx);
        case FN_OP_ROT_APPLY: return launch<double, 3, FN_OP_ROT_APPLY>(x, nullptr, n, h, b, q, ka, s, ldx);
        default: return fail(FN_EINVAL, "unknown rotation op");
    }
}

int check_args(int op, int dim, int dtype, const void* x, int64_t n, const void* head,
               const void* body, const void* sq) {
    if (op < FN_OP_SCALE || op > FN_OP_ROT_APPLY) return fail(FN_EINVAL, "unknown op");
    if (dim < 2 || dim > 4) return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    if (dtype != FN_F32 && dtype != FN_F64) return fail(FN_EINVAL, "dtype must be FN_F32/FN_F64");
    if (op == FN_OP_ROT_APPLY && (dim != 3 || dtype != FN_F64))
        return fail(FN_EINVAL, "FN_OP_ROT_APPLY takes float64 3-vectors (dim 3, FN_F64)");
    if (is_rotation(op) && op != FN_OP_ROT_APPLY && (dim != 4 || dtype != FN_F64))
        return fail(FN_EINVAL, "rotations take float64 quaternions (dim 4, FN_F64)");
    if (n < 0) return fail(FN_EINVAL, "n must be >= 0");
    if (n == 0) return FN_OK;
    const Widths w = op_widths(op, dim);
    if (!x || !head) return fail(FN_EINVAL, "x and head must not be NULL");
    if (w.w1 == 0) {
        if (body) return fail(FN_EINVAL, "this op has no body output; pass NULL");
    } else if (!body) {
        return fail(FN_EINVAL, "body output must not be NULL");
    }
    if (w.w2 > 0 && !sq) return fail(FN_EINVAL, "sq/extra output must not be NULL");
    return FN_OK;
}

// ldx: elements from one input row to the next (0 = dim, dense rows).
int run_ex(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body, void* sq,
           const double* ka, unsigned long long* invalid, void* stream, int64_t ldx = 0) {
    int rc = check_args(op, dim, dtype, x, n, head, body, sq);
    if (rc != FN_OK || n == 0) return rc;
    if (ldx == 0) ldx = dim;
    if (ldx < dim) return fail(FN_EINVAL, "ldx (elements per input row) must be >= dim");
    if (ldx > (INT64_MAX - dim) / n) return fail(FN_EINVAL, "n * ldx overflows");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (is_rotation(op)) return dispatch_rot(op, x, n, head, body, sq, ka, invalid, s, ldx);
    if (dtype == FN_F64) return dispatch<double>(op, dim, x, n, head, body, sq, ka, invalid, s, ldx);
    return dispatch<float>(op, dim, x, n, head, body, sq, ka, invalid, s, ldx);
}

// ---------------------------------------------------------------------------------
// Many independent batches (segments) per launch: fn_run_many.
// ---------------------------------------------------------------------------------
// FASTNORM_B200_MANY_DYN=0: the many-batch kernel keeps the static tile schedule (A/B).
static bool many_dyn_enabled() {
    static const bool v = [] {
        const char* e = getenv("FASTNORM_B200_MANY_DYN");
        return !(e && strcmp(e, "0") == 0);
    }();
    return v;
}

template <typename T, int N, int OP> struct SegLaunch {
    using L = TileLayout<T, N, OP, OpRows<T, N, OP, false>::value, OpStages<T, N, OP, false>::value>;
    static int blocks_per_sm(int dev) {
        static std::mutex mu;
        static int cache[64] = {0};
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 0 || dev >= 64) return 1;
        if (cache[dev] == 0) {
            auto kern = tma_segments_kernel<T, N, OP>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemBytes);
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, Tile<T, N>::kThreads, L::kSmemBytes) !=
                    cudaSuccess ||
                nb < 1)
                nb = 1;
            cache[dev] = nb;
        }
        return cache[dev];
    }
};

template <typename T, int N, int OP>
static int launch_many(int nseg, const void* const* xs, const int64_t* ns, void* const* heads, void* const* bodies,
                       void* const* extras, const KArgs<T>& ka, cudaStream_t stream) {
    using SL = SegLaunch<T, N, OP>;
    using L = typename SL::L;
    using Op = typename L::Op;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const int sms = device_sms(dev);
    SegmentTable<T> tab;
    tab.nseg = 0;
    tab.ntiles = 0;
    auto flush = [&]() -> int {
        if (tab.nseg == 0) return FN_OK;
        const int64_t work = std::max<int64_t>(tab.ntiles, 1);
        const int64_t per_sm = std::min<int64_t>(SL::blocks_per_sm(dev), ctas_per_sm_for<T, N, OP>(tab.ntiles, sms));
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(work, tab.nseg), per_sm * sms));
        KArgs<T> kd = ka;
        SchedLease lease = sched_lease(many_dyn_enabled() && tab.ntiles > (int64_t)L::S * grid, SchedBatch<OP>::value,
                                       tab.ntiles / grid, dev, stream, kd);
        const cudaError_t le = launch_pdl(tma_segments_kernel<T, N, OP>, grid, Tile<T, N>::kThreads, L::kSmemBytes,
                                          stream, tab, kd);
        if (le != cudaSuccess) return cuda_fail(le, "kernel launch");
        lease.commit();
        tab.nseg = 0;
        tab.ntiles = 0;
        return FN_OK;
    };
    for (int j = 0; j < nseg; ++j) {
        const int64_t n = ns[j];
        if (n == 0) continue;
        const bool aligned = aligned16(xs[j]) && aligned16(heads[j]) && (Op::W1 == 0 || aligned16(bodies[j])) &&
                             (Op::W2 == 0 || aligned16(extras[j]));
        if (!aligned || force_direct()) {  // this segment on its own (per-row or misaligned kernels)
            const int rc = launch<T, N, OP>(xs[j], nullptr, n, heads[j], Op::W1 ? bodies[j] : nullptr,
                                            Op::W2 ? extras[j] : nullptr, ka, stream);
            if (rc != FN_OK) return rc;
            continue;
        }
        Segment<T>& sg = tab.seg[tab.nseg++];
        sg.x = static_cast<const T*>(xs[j]);
        sg.head = static_cast<T*>(heads[j]);
        sg.body = Op::W1 ? static_cast<T*>(bodies[j]) : nullptr;
        sg.extra = Op::W2 ? static_cast<T*>(extras[j]) : nullptr;
        sg.rows = n;
        sg.tile0 = tab.ntiles;
        tab.ntiles += n / L::TR;
        if (tab.nseg == kMaxSegments) {
            const int rc = flush();
            if (rc != FN_OK) return rc;
        }
    }
    return flush();
}

template <typename T, int OP>
static int many_dim(int dim, int nseg, const void* const* xs, const int64_t* ns, void* const* h, void* const* b,
                    void* const* q, const KArgs<T>& ka, cudaStream_t s) {
    switch (dim) {
        case 2: return launch_many<T, 2, OP>(nseg, xs, ns, h, b, q, ka, s);
        case 3: return launch_many<T, 3, OP>(nseg, xs, ns, h, b, q, ka, s);
        case 4: return launch_many<T, 4, OP>(nseg, xs, ns, h, b, q, ka, s);
        default: return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    }
}

template <typename T>
static int dispatch_many(int op, int dim, int nseg, const void* const* xs, const int64_t* ns, void* const* h,
                         void* const* b, void* const* q, const double* kad, cudaStream_t s) {
    KArgs<T> ka;
    int rc = make_kargs<T>(kad, needs_ka(op), ka);
    if (rc != FN_OK) return rc;
    switch (op) {
        case FN_OP_SCALE: return many_dim<T, FN_OP_SCALE>(dim, nseg, xs, ns, h, b, q, ka, s);
        case FN_OP_NORMALIZE: return many_dim<T, FN_OP_NORMALIZE>(dim, nseg, xs, ns, h, b, q, ka, s);
        case FN_OP_NORMALIZE_SQ: return many_dim<T, FN_OP_NORMALIZE_SQ>(dim, nseg, xs, ns, h, b, q, ka, s);
        case FN_OP_NORM: return many_dim<T, FN_OP_NORM>(dim, nseg, xs, ns, h, b, q, ka, s);
        case FN_OP_NAIVE: return many_dim<T, FN_OP_NAIVE>(dim, nseg, xs, ns, h, b, q, ka, s);
        case FN_OP_QUOTIENT: return many_dim<T, FN_OP_QUOTIENT>(dim, nseg, xs, ns, h, b, q, ka, s);
        case FN_OP_QUOTIENT3_FAST:
            if (dim != 3) return fail(FN_EINVAL, "quotient3_fast is defined for dim 3 only");
            return launch_many<T, 3, FN_OP_QUOTIENT3_FAST>(nseg, xs, ns, h, b, q, ka, s);
        default: return fail(FN_EINVAL, "fn_run_many takes the scaling and baseline families");
    }
}

int run_many(int op, int dim, int dtype, int nseg, const void* const* xs, const int64_t* ns, void* const* heads,
             void* const* bodies, void* const* extras, const double* ka, void* stream) {
    if (nseg < 0 || (nseg > 0 && (!xs || !ns || !heads))) return fail(FN_EINVAL, "bad segment arrays");
    if (op < FN_OP_SCALE || op > FN_OP_NORMALIZE_SQ) return fail(FN_EINVAL, "fn_run_many takes the scaling and baseline families");
    const Widths w = op_widths(op, dim);
    if (w.w1 && !bodies) return fail(FN_EINVAL, "bodies must not be NULL for this op");
    if (w.w2 && !extras) return fail(FN_EINVAL, "extras must not be NULL for this op");
    for (int j = 0; j < nseg; ++j) {
        const int rc = check_args(op, dim, dtype, xs[j], ns[j], heads[j], w.w1 ? bodies[j] : nullptr,
                                  w.w2 ? extras[j] : nullptr);
        if (rc != FN_OK) return rc;
    }
    if (nseg == 0) return FN_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == FN_F64) return dispatch_many<double>(op, dim, nseg, xs, ns, heads, bodies, extras, ka, s);
    return dispatch_many<float>(op, dim, nseg, xs, ns, heads, bodies, extras, ka, s);
}

int run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body, void* sq,
        const double* ka, void* stream) {
    return run_ex(op, dim, dtype, x, n, head, body, sq, ka, nullptr, stream);
}

// ---------------------------------------------------------------------------------
// Structure-of-arrays entry: the reference's scalar signatures vectorised over arrays
// (normalize3(p, x1[], x2[], x3[]) -> r[], (u1[], u2[], u3[])).
// ---------------------------------------------------------------------------------
// FASTNORM_B200_SOA=vec selects the register-vector SoA kernel over the bulk-copy one.
static int soa_path() {
    static const int v = [] {
        const char* e = getenv("FASTNORM_B200_SOA");
        return e && strcmp(e, "vec") == 0 ? 1 : 0;
    }();
    return v;
}

// FASTNORM_B200_SOA_DYN=0: the SoA bulk-copy kernel keeps the static tile schedule (A/B).
static bool soa_dyn_enabled() {
    static const bool v = [] {
        const char* e = getenv("FASTNORM_B200_SOA_DYN");
        return !(e && strcmp(e, "0") == 0);
    }();
    return v;
}

template <typename T, int N, int OP>
static int launch_soa(const void* const* xs, int64_t n, void* head, void* const* body, void* sq,
                      const KArgs<T>& ka, cudaStream_t stream) {
    using Op = RowOp<T, N, OP>;
    SoaPtrs<T, N> p;
    for (int c = 0; c < N; ++c) {
        p.x[c] = static_cast<const T*>(xs[c]);
        p.body[c] = Op::W1 ? static_cast<T*>(body[c]) : nullptr;
    }
    p.head = static_cast<T*>(head);
    p.extra = static_cast<T*>(sq);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    bool outs_aligned = aligned16(p.head) && (Op::W2 == 0 || aligned16(p.extra));
    bool ins_aligned = true, ins_elem = true;
    int64_t reach = 0;  // bytes the bulk loads of a misaligned array read past a run
    for (int c = 0; c < N; ++c) {
        outs_aligned = outs_aligned && (Op::W1 == 0 || aligned16(p.body[c]));
        ins_aligned = ins_aligned && aligned16(p.x[c]);
        ins_elem = ins_elem && ((uintptr_t)p.x[c] % sizeof(T)) == 0;
        const int mis = (int)((uintptr_t)p.x[c] & 15);
        if (mis) reach = std::max<int64_t>(reach, 16 - mis);
    }
    const bool aligned = outs_aligned && ins_aligned;
    constexpr int V = Vec16<T>::kRows;
    const int sms = device_sms(dev);
    using ST = SoaTile<T, N, OP>;
    if (outs_aligned && ins_elem && !force_direct() && soa_path() == 0 && n >= ST::TR) {
        // bulk-copy pipeline over whole runs (the instantiation for arrays off the 16-byte
        // grid when any is), the rest through the kernels below
        const bool mis = !ins_aligned;
        auto kern = mis ? tma_soa_kernel<T, N, OP, true> : tma_soa_kernel<T, N, OP, false>;
        const int smem = mis ? SoaTile<T, N, OP, true>::kSmemBytes : ST::kSmemBytes;
        {  // the shared-memory opt-in is a per-device function attribute
            static std::mutex mu;
            static bool attr_set[64] = {false};
            std::lock_guard<std::mutex> lk(mu);
            if (dev >= 0 && dev < 64 && !attr_set[dev]) {
                cudaFuncSetAttribute(tma_soa_kernel<T, N, OP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     ST::kSmemBytes);
                cudaFuncSetAttribute(tma_soa_kernel<T, N, OP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SoaTile<T, N, OP, true>::kSmemBytes);
                attr_set[dev] = true;
            }
        }
        // whole runs whose loads (and their reach past a misaligned run) stay inside the arrays
        const int64_t ntiles = (n * (int64_t)sizeof(T) - reach) / ST::kArr;
        // CTAs per SM: 3 where the shared memory holds them (2-D rows: 6433-6553 -> 6873 GB/s,
        // profiles/r02af_soa_ctas.txt), else what fits (3-D and 4-D rows: 2)
        const int fit = std::max(1, (int)(227 * 1024 / (smem + 1024)));
        const int per_sm = std::min(cps_override() > 0 ? cps_override() : ST::kCtasPerSm, fit);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sms * per_sm));
        if (ntiles > 0) {
            // the dynamic tile schedule of launch_tma_as (same counters, same rules)
            KArgs<T> kd = ka;
            SchedLease lease = sched_lease(soa_dyn_enabled() && ntiles > (int64_t)ST::S * grid, SchedBatch<OP>::value,
                                           ntiles / grid, dev, stream, kd);
            e = launch_pdl(kern, grid, ST::NT, (size_t)smem, stream, p, ntiles, kd);
            if (e == cudaSuccess) lease.commit();
        }
        if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
        const int64_t done = ntiles * ST::TR;
        if (done == n) return FN_OK;
        for (int c = 0; c < N; ++c) {
            p.x[c] += done;
            if (Op::W1) p.body[c] += done;
        }
        p.head += done;
        if (Op::W2) p.extra += done;
        n -= done;
    }
    const int64_t nvec = aligned && !force_direct() ? n / V : 0;
    if (nvec > 0) {
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nvec + 255) / 256, (int64_t)sms * 8));
        e = launch_pdl(soa_vec_kernel<T, N, OP>, grid, 256, 0, stream, p, nvec, ka);
        if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    }
    const int64_t done = nvec * V;
    if (done < n) {  // rows after the last whole vector (or everything, unaligned)
        SoaPtrs<T, N> t = p;
        for (int c = 0; c < N; ++c) {
            t.x[c] += done;
            if (Op::W1) t.body[c] += done;
        }
        t.head += done;
        if (Op::W2) t.extra += done;
        const int64_t rest = n - done;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rest + 255) / 256, (int64_t)sms * 8));
        e = launch_pdl(soa_kernel<T, N, OP>, grid, 256, 0, stream, t, rest, ka);
        if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    }
    return FN_OK;
}

template <typename T, int OP>
static int soa_dim(int dim, const void* const* xs, int64_t n, void* h, void* const* b, void* q,
                   const KArgs<T>& ka, cudaStream_t s) {
    switch (dim) {
        case 2: return launch_soa<T, 2, OP>(xs, n, h, b, q, ka, s);
        case 3: return launch_soa<T, 3, OP>(xs, n, h, b, q, ka, s);
        default: return launch_soa<T, 4, OP>(xs, n, h, b, q, ka, s);
    }
}

template <typename T>
static int dispatch_soa(int op, int dim, const void* const* xs, int64_t n, void* h, void* const* b, void* q,
                        const double* kad, cudaStream_t s) {
    KArgs<T> ka;
    int rc = make_kargs<T>(kad, needs_ka(op), ka);
    if (rc != FN_OK) return rc;
    switch (op) {
        case FN_OP_SCALE: return soa_dim<T, FN_OP_SCALE>(dim, xs, n, h, b, q, ka, s);
        case FN_OP_NORMALIZE: return soa_dim<T, FN_OP_NORMALIZE>(dim, xs, n, h, b, q, ka, s);
        case FN_OP_NORMALIZE_SQ: return soa_dim<T, FN_OP_NORMALIZE_SQ>(dim, xs, n, h, b, q, ka, s);
        case FN_OP_NORM: return soa_dim<T, FN_OP_NORM>(dim, xs, n, h, b, q, ka, s);
        case FN_OP_NAIVE: return soa_dim<T, FN_OP_NAIVE>(dim, xs, n, h, b, q, ka, s);
        case FN_OP_QUOTIENT: return soa_dim<T, FN_OP_QUOTIENT>(dim, xs, n, h, b, q, ka, s);
        case FN_OP_QUOTIENT3_FAST:
            if (dim != 3) return fail(FN_EINVAL, "quotient3_fast is defined for dim 3 only");
            return launch_soa<T, 3, FN_OP_QUOTIENT3_FAST>(xs, n, h, b, q, ka, s);
        default: return fail(FN_EINVAL, "the SoA entry takes the scale / normalize / norm / naive / quotient families");
    }
}

int run_soa(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head, void* const* body,
            void* sq, const double* ka, void* stream) {
    if (op < FN_OP_SCALE || op > FN_OP_NORMALIZE_SQ) return fail(FN_EINVAL, "unknown op for the SoA entry");
    if (dim < 2 || dim > 4) return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    if (dtype != FN_F32 && dtype != FN_F64) return fail(FN_EINVAL, "dtype must be FN_F32/FN_F64");
    if (n < 0) return fail(FN_EINVAL, "n must be >= 0");
    if (n == 0) return FN_OK;
    const Widths w = op_widths(op, dim);
    if (!xs || !head) return fail(FN_EINVAL, "xs and head must not be NULL");
    for (int c = 0; c < dim; ++c)
        if (!xs[c]) return fail(FN_EINVAL, "component array is NULL");
    if (w.w1) {
        if (!body) return fail(FN_EINVAL, "body arrays must not be NULL");
        for (int c = 0; c < dim; ++c)
            if (!body[c]) return fail(FN_EINVAL, "body array is NULL");
    } else if (body) {
        return fail(FN_EINVAL, "this op has no body output; pass NULL");
    }
    if (w.w2 && !sq) return fail(FN_EINVAL, "sq output must not be NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype == FN_F64) return dispatch_soa<double>(op, dim, xs, n, head, body, sq, ka, s);
    return dispatch_soa<float>(op, dim, xs, n, head, body, sq, ka, s);
}

// Two-input ops: record width of the first input (q: 4, R: 9); the second is v[N,3].
static int rows2_dim(int op) { return op == FN_OP_QUAT_ROTATE ? 4 : (op == FN_OP_MAT_APPLY ? 9 : 0); }

static int check_rows2(int op, const void* a, const void* v, int64_t n, const void* out) {
    if (!rows2_dim(op)) return fail(FN_EINVAL, "op must be FN_OP_QUAT_ROTATE or FN_OP_MAT_APPLY");
    if (n < 0) return fail(FN_EINVAL, "n must be >= 0");
    if (n > 0 && (!a || !v || !out)) return fail(FN_EINVAL, "a, v and out must not be NULL");
    return FN_OK;
}

int run_rows2(int op, const void* a, const void* v, int64_t n, void* out, const double* kad,
              unsigned long long* invalid, cudaStream_t s) {
    int rc = check_rows2(op, a, v, n, out);
    if (rc != FN_OK || n == 0) return rc;
    KArgs<double> ka;
    rc = make_kargs<double>(kad, op == FN_OP_QUAT_ROTATE, ka);
    if (rc != FN_OK) return rc;
    ka.invalid = invalid;
    if (op == FN_OP_QUAT_ROTATE)
        return launch<double, 4, FN_OP_QUAT_ROTATE>(a, v, n, out, nullptr, nullptr, ka, s);
    return launch<double, 9, FN_OP_MAT_APPLY>(a, v, n, out, nullptr, nullptr, ka, s);
}

// ---------------------------------------------------------------------------------
// Host-buffer path: chunked H2D -> kernel -> D2H pipeline over three streams, with
// per-device staging buffers that persist across calls (no allocation on the data
// path after the first call).  H2D and D2H of different chunks proceed concurrently
// on the two copy engines while the kernel of a third chunk runs.
// ---------------------------------------------------------------------------------
struct Staging {
    static constexpr int kMaxPipes = 8;
    int pipes = 3;
    cudaStream_t streams[kMaxPipes] = {};
    cudaEvent_t done[kMaxPipes] = {};
    void* buf[kMaxPipes] = {};   // device staging
    void* hbuf[kMaxPipes] = {};  // page-locked host staging (pageable callers only)
    size_t bytes = 0, hbytes = 0;
    bool init = false;
};

// ---------------------------------------------------------------------------------
// Parallel host memcpy for pageable callers: a small persistent worker pool copies the
// slices of one job; jobs are serialised (host memory bandwidth is shared anyway).
// The pool has FASTNORM_B200_COPY_THREADS workers (default min(16, cores)); a job may
// use fewer.  On the 16-core B200 host (2^28 3-D f64 rows, profiles/r02h_host_sweep.txt):
// with the outputs staged too, all 16 threads do best (0.80 G rows/s, 0.73 with 12);
// when only the input is staged (page-locked outputs, e.g. the library's own result
// pool), half of them do best (1.50 G rows/s with 8 of 16, 1.40 with 6 of 12, 1.22
// with 4 of 8, 0.97 with all 12) -- more copy threads compete with the concurrent DMA
// traffic and the driver's threads.
// ---------------------------------------------------------------------------------
class CopyPool {
  public:
    CopyPool() {
        const int hw = (int)std::thread::hardware_concurrency();
        const char* e = getenv("FASTNORM_B200_COPY_THREADS");
        nthreads_ = e ? std::max(1, atoi(e)) : std::max(1, std::min(16, hw));
        for (int k = 1; k < nthreads_; ++k) workers_.emplace_back([this, k] { work(k); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int threads() const { return nthreads_; }
    // Copies with at most max_threads threads (the caller's included).
    void copy(void* dst, const void* src, size_t bytes, int max_threads = 1 << 30) {
        const int use = std::max(1, std::min(nthreads_, max_threads));
        if (bytes < ((size_t)4 << 20) || use == 1) {
            memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            active_ = use;
            pending_ = use - 1;
            ++gen_;
        }
        cv_.notify_all();
        slice(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void slice(int k) {
        const size_t per = (bytes_ / active_ + 63) & ~(size_t)63;
        const size_t lo = std::min(bytes_, per * k), hi = std::min(bytes_, per * (k + 1));
        if (hi > lo) memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
    void work(int k) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                if (k >= active_) continue;  // not part of this job
            }
            slice(k);
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    int nthreads_ = 1;
    std::vector<std::thread> workers_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_, done_cv_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    int active_ = 1;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

static int copy_pool_threads();

// Threads for one staging copy: every worker when the call stages its outputs too,
// about half of them (6 of 12) when only the input is staged.
static int copy_threads(bool stage_out) {
    return stage_out ? 1 << 30 : std::max(1, (copy_pool_threads() + 1) / 2);
}

static CopyPool& copy_pool() {
    static CopyPool pool;
    return pool;
}

static int copy_pool_threads() { return copy_pool().threads(); }

static bool is_page_locked(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Host-path pipeline shape: FASTNORM_B200_HOST_PIPES (2..8, default 3) streams and
// FASTNORM_B200_HOST_CHUNK_MB (default 48) MiB of input per chunk.
static int env_int(const char* name, int dflt, int lo, int hi) {
    const char* e = getenv(name);
    if (!e) return dflt;
    const int v = atoi(e);
    return v < lo ? lo : (v > hi ? hi : v);
}
// One staging set and one mutex per device; the table itself is guarded by g_stage_mu.
static std::mutex g_stage_mu;
static std::vector<std::unique_ptr<Staging>> g_stage;
static std::vector<std::unique_ptr<std::mutex>> g_stage_dev_mu;

static std::mutex& device_mutex(int dev) {
    std::lock_guard<std::mutex> lk(g_stage_mu);
    while ((int)g_stage.size() <= dev) {
        g_stage.emplace_back(new Staging());
        g_stage_dev_mu.emplace_back(new std::mutex());
    }
    return *g_stage_dev_mu[dev];
}

// Caller holds device_mutex(dev).
static int staging_get(int dev, size_t bytes_per_pipe, Staging** out) {
    Staging* stp;
    {
        std::lock_guard<std::mutex> lk(g_stage_mu);
        stp = g_stage[dev].get();
    }
    Staging& st = *stp;
    cudaError_t e;
    if (!st.init) {
        st.pipes = env_int("FASTNORM_B200_HOST_PIPES", 3, 2, Staging::kMaxPipes);
        for (int p = 0; p < st.pipes; ++p) {
            e = cudaStreamCreateWithFlags(&st.streams[p], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
            e = cudaEventCreateWithFlags(&st.done[p], cudaEventDisableTiming);
            if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
        }
        st.init = true;
    }
    if (st.bytes < bytes_per_pipe) {
        for (int p = 0; p < st.pipes; ++p) {
            if (st.buf[p]) cudaFree(st.buf[p]);
            st.buf[p] = nullptr;
        }
        st.bytes = 0;
        for (int p = 0; p < st.pipes; ++p) {
            e = cudaMalloc(&st.buf[p], bytes_per_pipe);
            if (e != cudaSuccess) return fail(FN_ENOMEM, "cudaMalloc staging buffer failed");
        }
        st.bytes = bytes_per_pipe;
    }
    *out = &st;
    return FN_OK;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Armed once the first chunk is enqueued: an error return would otherwise leave H2D / D2H
// copies of earlier chunks in flight on the pipe streams, reading or writing caller
// buffers the caller may free as soon as the call has returned.  Declared after the
// device lock, so it runs before the lock is released.
struct PipeDrainGuard {
    Staging* st = nullptr;
    ~PipeDrainGuard() {
        if (!st) return;
        for (int p = 0; p < st->pipes; ++p) cudaStreamSynchronize(st->streams[p]);
    }
};

// Page-locked host staging of bytes_per_pipe per pipe (caller holds device_mutex(dev)).
static int host_staging_get(Staging* st, size_t bytes_per_pipe) {
    if (st->hbytes >= bytes_per_pipe) return FN_OK;
    for (int p = 0; p < st->pipes; ++p) {
        if (st->hbuf[p]) cudaFreeHost(st->hbuf[p]);
        st->hbuf[p] = nullptr;
    }
    st->hbytes = 0;
    for (int p = 0; p < st->pipes; ++p) {
        if (cudaHostAlloc(&st->hbuf[p], bytes_per_pipe, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            return fail(FN_ENOMEM, "cudaHostAlloc staging buffer failed");
        }
    }
    st->hbytes = bytes_per_pipe;
    return FN_OK;
}

// ---------------------------------------------------------------------------------
// Small host batches (up to kSmallHostBytes of rows in and results out): copy the rows
// into a per-thread page-locked buffer mapped into the device, run the per-row kernel
// on it in place (the kernel reads and writes host memory over PCIe), synchronise, copy
// the results out.  One launch and one synchronisation instead of the staged pipeline's
// transfers and events: ~48 -> ~15 us for a few hundred rows (profiles/r01cr_*).
// ---------------------------------------------------------------------------------
constexpr size_t kSmallHostBytes = 256 << 10;

struct SmallCtx {
    int dev = -1;
    cudaStream_t stream = nullptr;
    char* host = nullptr;
    char* dptr = nullptr;
};

// Contexts live in a per-device free list, not in thread_local storage: fn_host_run_multi
// runs each shard on a fresh std::thread, and a thread_local context (a mapped
// page-locked buffer and a stream) would leak with every such thread.  The pool holds
// at most as many contexts per device as there were concurrent small calls on it.
constexpr size_t kSmallCtxBytes = kSmallHostBytes + 16 * 256;

class SmallPool {
  public:
    // Takes a context of device `dev` (the caller's current device), creating one if none is free.
    int acquire(int dev, SmallCtx** out) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            if ((int)free_.size() <= dev) free_.resize(dev + 1);
            if (!free_[dev].empty()) {
                *out = free_[dev].back();
                free_[dev].pop_back();
                return FN_OK;
            }
        }
        std::unique_ptr<SmallCtx> c(new SmallCtx());
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        e = cudaHostAlloc(reinterpret_cast<void**>(&c->host), kSmallCtxBytes, cudaHostAllocMapped);
        if (e != cudaSuccess) {
            cudaStreamDestroy(c->stream);
            return cuda_fail(e, "cudaHostAlloc");
        }
        e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->dptr), c->host, 0);
        if (e != cudaSuccess) {
            cudaFreeHost(c->host);
            cudaStreamDestroy(c->stream);
            return cuda_fail(e, "cudaHostGetDevicePointer");
        }
        c->dev = dev;
        std::lock_guard<std::mutex> lk(mu_);
        ++created_;
        *out = c.release();
        return FN_OK;
    }
    void release(SmallCtx* c) {
        std::lock_guard<std::mutex> lk(mu_);
        free_[c->dev].push_back(c);
    }
    int64_t created() {
        std::lock_guard<std::mutex> lk(mu_);
        return created_;
    }

  private:
    std::mutex mu_;
    std::vector<std::vector<SmallCtx*>> free_;
    int64_t created_ = 0;
};

static SmallPool& small_pool() {
    static SmallPool* pool = new SmallPool();  // never destroyed: contexts outlive static teardown
    return *pool;
}

struct SmallLease {
    SmallCtx* c = nullptr;
    ~SmallLease() {
        if (c) small_pool().release(c);
    }
};

static int host_run_small(int op, int dim, int dtype, const void* x, const void* x2, int dim2, int64_t n,
                          void* head, void* body, void* sq, const double* ka, int dev, int64_t ldx) {
    SmallLease lease;
    int rc0 = small_pool().acquire(dev, &lease.c);
    if (rc0 != FN_OK) return rc0;
    SmallCtx& c = *lease.c;
    cudaError_t e;
    const size_t w = dtype == FN_F64 ? 8 : 4;
    const Widths wd = op_widths(op, dim);
    const size_t bx = align256(n * ldx * w), bx2 = align256(n * dim2 * w), b0 = align256(n * wd.w0 * w),
                 b1 = align256(n * wd.w1 * w);
    const size_t off[5] = {0, bx, bx + bx2, bx + bx2 + b0, bx + bx2 + b0 + b1};
    memcpy(c.host + off[0], x, ((n - 1) * ldx + dim) * w);
    if (x2) memcpy(c.host + off[1], x2, n * dim2 * w);
    void* d0 = c.dptr + off[2];
    void* d1 = wd.w1 ? c.dptr + off[3] : nullptr;
    void* d2 = wd.w2 ? c.dptr + off[4] : nullptr;
    tl_direct = true;
    const int rc = x2 ? run_rows2(op, c.dptr + off[0], c.dptr + off[1], n, d0, ka, nullptr, c.stream)
                      : run_ex(op, dim, dtype, c.dptr + off[0], n, d0, d1, d2, ka, nullptr, c.stream, ldx);
    tl_direct = false;
    if (rc != FN_OK) return rc;
    e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    memcpy(head, c.host + off[2], n * wd.w0 * w);
    if (wd.w1) memcpy(body, c.host + off[3], n * wd.w1 * w);
    if (wd.w2) memcpy(sq, c.host + off[4], n * wd.w2 * w);
    return FN_OK;
}

// x2 / dim2: the second input of the two-input ops (NULL / 0 otherwise).  ldx: elements
// from one row of x to the next (0 = dim); each chunk moves its rows' records as they are
// ((m - 1) * ldx + dim elements, the last row's padding excluded) and the kernel reads
// them with the same stride.
static int host_run_impl(int op, int dim, int dtype, const void* x, const void* x2, int dim2, int64_t n,
                         void* head, void* body, void* sq, const double* ka, int64_t ldx = 0) {
    int rc = x2 ? check_rows2(op, x, x2, n, head) : check_args(op, dim, dtype, x, n, head, body, sq);
    if (rc != FN_OK || n == 0) return rc;
    if (ldx == 0) ldx = dim;
    if (ldx < dim || (x2 && ldx != dim)) return fail(FN_EINVAL, "ldx (elements per input row) must be >= dim");
    if (ldx > (INT64_MAX / 16 - dim) / n) return fail(FN_EINVAL, "n * ldx overflows");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const size_t w = dtype == FN_F64 ? 8 : 4;
    const Widths wd = op_widths(op, dim);
    if ((size_t)n * (ldx + dim2 + wd.w0 + wd.w1 + wd.w2) * w + 8 * 256 <= kSmallHostBytes &&
        env_int("FASTNORM_B200_HOST_SMALL", 1, 0, 1))  // FASTNORM_B200_HOST_SMALL=0: always stage
        return host_run_small(op, dim, dtype, x, x2, dim2, n, head, body, sq, ka, dev, ldx);
    // Pageable caller memory cannot be DMA'd asynchronously: such sides go through
    // page-locked staging filled / drained by the parallel host copier, overlapped with
    // the transfers and kernels of the other pipes.
    const bool stage_in = !is_page_locked(x);
    const bool stage_in2 = x2 && !is_page_locked(x2);
    const bool stage_out = !is_page_locked(head) || (wd.w1 && !is_page_locked(body)) ||
                           (wd.w2 && !is_page_locked(sq));
    const bool staged = stage_in || stage_in2 || stage_out;
    // Input bytes per chunk (profiles/r01cs_chunks.txt, 3-D f64 rows):
    //  * page-locked callers: 48 MiB for large arrays, and at least 8 chunks of >= 4 MiB
    //    for mid-size ones so transfers and kernels of different chunks overlap;
    //  * pageable callers: 8-32 MiB (32 MiB from 192 MiB of input up: 1.18 against 0.88
    //    G rows/s at 16 MiB with page-locked outputs, profiles/r02e_host_sweep.txt).
    // FASTNORM_B200_HOST_CHUNK_MB fixes the chunk size instead.
    const int64_t row_in = (int64_t)((ldx + dim2) * w), in_total = n * row_in;
    int64_t chunk_bytes;
    if (getenv("FASTNORM_B200_HOST_CHUNK_MB")) {
        chunk_bytes = (int64_t)env_int("FASTNORM_B200_HOST_CHUNK_MB", 48, 1, 1024) << 20;
    } else if (staged) {
        chunk_bytes = std::max<int64_t>((int64_t)8 << 20, std::min<int64_t>((int64_t)32 << 20, in_total / 6));
    } else {
        chunk_bytes = std::max<int64_t>((int64_t)4 << 20, std::min<int64_t>((int64_t)48 << 20, in_total / 8));
    }
    const int64_t chunk_rows = std::max<int64_t>(4096, chunk_bytes / row_in);
    const int64_t rows = std::min<int64_t>(n, chunk_rows);
    const size_t bx = align256(rows * ldx * w), bx2 = align256(rows * dim2 * w),
                 b0 = align256(rows * wd.w0 * w), b1 = align256(rows * wd.w1 * w),
                 b2 = align256(rows * wd.w2 * w);
    const size_t per_pipe = bx + bx2 + b0 + b1 + b2;
    std::lock_guard<std::mutex> lk(device_mutex(dev));
    Staging* st = nullptr;
    rc = staging_get(dev, per_pipe, &st);
    if (rc != FN_OK) return rc;
    if (staged) {
        rc = host_staging_get(st, per_pipe);
        if (rc != FN_OK) return rc;
    }
    struct Pending {
        bool live = false;
        int64_t r0 = 0, m = 0;
    } pending[Staging::kMaxPipes];
    char* const outs[3] = {static_cast<char*>(head), static_cast<char*>(body), static_cast<char*>(sq)};
    const int ws[3] = {wd.w0, wd.w1, wd.w2};
    const size_t offs[3] = {bx + bx2, bx + bx2 + b0, bx + bx2 + b0 + b1};
    auto drain = [&](int p) -> int {
        if (!pending[p].live) return FN_OK;
        cudaError_t ee = cudaEventSynchronize(st->done[p]);
        if (ee != cudaSuccess) return cuda_fail(ee, "cudaEventSynchronize");
        if (stage_out) {
            const char* hb = static_cast<const char*>(st->hbuf[p]);
            for (int k = 0; k < 3; ++k)
                if (ws[k])
                    copy_pool().copy(outs[k] + pending[p].r0 * ws[k] * w, hb + offs[k],
                                     pending[p].m * ws[k] * w);
        }
        pending[p].live = false;
        return FN_OK;
    };
    PipeDrainGuard in_flight;
    in_flight.st = st;
    int64_t chunk = 0;
    for (int64_t r0 = 0; r0 < n; r0 += rows, ++chunk) {
        const int p = (int)(chunk % st->pipes);
        const int64_t m = std::min<int64_t>(rows, n - r0);
        cudaStream_t s = st->streams[p];
        rc = drain(p);  // staging of pipe p is free again (its previous chunk completed)
        if (rc != FN_OK) return rc;
        char* base = static_cast<char*>(st->buf[p]);
        char* hbase = static_cast<char*>(st->hbuf[p]);
        void* dx = base;
        void* dptr[3] = {base + offs[0], wd.w1 ? base + offs[1] : nullptr, wd.w2 ? base + offs[2] : nullptr};
        const char* src = static_cast<const char*>(x) + r0 * ldx * w;
        const size_t in_bytes = ((m - 1) * ldx + dim) * w;
        if (stage_in) {
            copy_pool().copy(hbase, src, in_bytes, copy_threads(stage_out));
            src = hbase;
        }
        e = cudaMemcpyAsync(dx, src, in_bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
        if (x2) {
            void* dx2 = base + bx;
            const char* src2 = static_cast<const char*>(x2) + r0 * dim2 * w;
            if (stage_in2) {
                copy_pool().copy(hbase + bx, src2, m * dim2 * w, copy_threads(stage_out));
                src2 = hbase + bx;
            }
            e = cudaMemcpyAsync(dx2, src2, m * dim2 * w, cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
            rc = run_rows2(op, dx, dx2, m, dptr[0], ka, nullptr, s);
        } else {
            rc = run_ex(op, dim, dtype, dx, m, dptr[0], dptr[1], dptr[2], ka, nullptr, s, ldx);
        }
        if (rc != FN_OK) return rc;
        for (int k = 0; k < 3 && e == cudaSuccess; ++k) {
            if (!ws[k]) continue;
            char* dst = stage_out ? hbase + offs[k] : outs[k] + r0 * ws[k] * w;
            e = cudaMemcpyAsync(dst, dptr[k], m * ws[k] * w, cudaMemcpyDeviceToHost, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync D2H");
        e = cudaEventRecord(st->done[p], s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
        pending[p] = {true, r0, m};
    }
    for (int64_t c = std::max<int64_t>(0, chunk - st->pipes); c < chunk; ++c) {
        rc = drain((int)(c % st->pipes));
        if (rc != FN_OK) return rc;
    }
    for (int p = 0; p < st->pipes; ++p) {
        e = cudaStreamSynchronize(st->streams[p]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    }
    in_flight.st = nullptr;
    return FN_OK;
}

int host_run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
             void* sq, const double* ka, int64_t ldx = 0) {
    return host_run_impl(op, dim, dtype, x, nullptr, 0, n, head, body, sq, ka, ldx);
}

// ---------------------------------------------------------------------------------
// Host structure-of-arrays rows (fn_host_run_soa): the reference's scalar signatures
// called with host component arrays.  The same chunked pipeline as host_run_impl --
// per chunk, every component array goes H2D (through page-locked staging filled by the
// parallel copier when the caller's memory is pageable), the SoA kernels run, every
// output array comes back -- over `pipes` streams, so transfers and kernels of
// different chunks overlap.
// ---------------------------------------------------------------------------------
// Small host SoA batches: the zero-copy route of host_run_small (components copied into
// a per-thread page-locked buffer mapped into the device, the per-row SoA kernel run on
// it in place, one synchronisation, results copied out).
static int host_run_soa_small(int op, int dim, int dtype, const void* const* xs, int64_t n, char* const* outs,
                              int nout, bool has_body, bool has_sq, const double* ka, int dev) {
    SmallLease lease;
    int rc0 = small_pool().acquire(dev, &lease.c);
    if (rc0 != FN_OK) return rc0;
    SmallCtx& c = *lease.c;
    cudaError_t e;
    const size_t w = dtype == FN_F64 ? 8 : 4;
    const size_t arr = align256(n * w);
    const void* dx[4];
    for (int k = 0; k < dim; ++k) {
        memcpy(c.host + k * arr, xs[k], n * w);
        dx[k] = c.dptr + k * arr;
    }
    void* dout[6];
    for (int k = 0; k < nout; ++k) dout[k] = c.dptr + (dim + k) * arr;
    tl_direct = true;
    const int rc = run_soa(op, dim, dtype, dx, n, dout[0], has_body ? &dout[1] : nullptr,
                           has_sq ? dout[nout - 1] : nullptr, ka, c.stream);
    tl_direct = false;
    if (rc != FN_OK) return rc;
    e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    for (int k = 0; k < nout; ++k) memcpy(outs[k], c.host + (dim + k) * arr, n * w);
    return FN_OK;
}

int host_run_soa(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head, void* const* body,
                 void* sq, const double* ka) {
    if (op < FN_OP_SCALE || op > FN_OP_NORMALIZE_SQ) return fail(FN_EINVAL, "unknown op for the SoA entry");
    if (dim < 2 || dim > 4) return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    if (dtype != FN_F32 && dtype != FN_F64) return fail(FN_EINVAL, "dtype must be FN_F32/FN_F64");
    if (n < 0) return fail(FN_EINVAL, "n must be >= 0");
    if (n == 0) return FN_OK;
    const Widths wd = op_widths(op, dim);
    if (!xs || !head) return fail(FN_EINVAL, "xs and head must not be NULL");
    for (int c = 0; c < dim; ++c)
        if (!xs[c]) return fail(FN_EINVAL, "component array is NULL");
    if (wd.w1) {
        if (!body) return fail(FN_EINVAL, "body arrays must not be NULL");
        for (int c = 0; c < dim; ++c)
            if (!body[c]) return fail(FN_EINVAL, "body array is NULL");
    }
    if (wd.w2 && !sq) return fail(FN_EINVAL, "sq output must not be NULL");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const size_t w = dtype == FN_F64 ? 8 : 4;
    // output arrays: head, body[0..dim), sq -- each one element per row
    const int nout = 1 + (wd.w1 ? dim : 0) + (wd.w2 ? 1 : 0);
    char* outs[6];
    outs[0] = static_cast<char*>(head);
    for (int c = 0; c < (wd.w1 ? dim : 0); ++c) outs[1 + c] = static_cast<char*>(body[c]);
    if (wd.w2) outs[nout - 1] = static_cast<char*>(sq);
    if ((size_t)(dim + nout) * align256(n * w) <= kSmallHostBytes && env_int("FASTNORM_B200_HOST_SMALL", 1, 0, 1))
        return host_run_soa_small(op, dim, dtype, xs, n, outs, nout, wd.w1 != 0, wd.w2 != 0, ka, dev);
    bool stage_in = false, stage_out = false;
    for (int c = 0; c < dim; ++c) stage_in = stage_in || !is_page_locked(xs[c]);
    for (int k = 0; k < nout; ++k) stage_out = stage_out || !is_page_locked(outs[k]);
    const bool staged = stage_in || stage_out;
    const int64_t row_in = (int64_t)(dim * w), in_total = n * row_in;
    int64_t chunk_bytes;
    if (getenv("FASTNORM_B200_HOST_CHUNK_MB")) {
        chunk_bytes = (int64_t)env_int("FASTNORM_B200_HOST_CHUNK_MB", 48, 1, 1024) << 20;
    } else if (staged) {
        chunk_bytes = std::max<int64_t>((int64_t)8 << 20, std::min<int64_t>((int64_t)32 << 20, in_total / 6));
    } else {
        chunk_bytes = std::max<int64_t>((int64_t)4 << 20, std::min<int64_t>((int64_t)48 << 20, in_total / 8));
    }
    const int64_t rows = std::min<int64_t>(n, std::max<int64_t>(4096, chunk_bytes / row_in));
    const size_t arr = align256(rows * w);  // one array's chunk
    const size_t per_pipe = arr * (size_t)(dim + nout);
    std::lock_guard<std::mutex> lk(device_mutex(dev));
    Staging* st = nullptr;
    int rc = staging_get(dev, per_pipe, &st);
    if (rc != FN_OK) return rc;
    if (staged) {
        rc = host_staging_get(st, per_pipe);
        if (rc != FN_OK) return rc;
    }
    struct Pending {
        bool live = false;
        int64_t r0 = 0, m = 0;
    } pending[Staging::kMaxPipes];
    auto drain = [&](int p) -> int {
        if (!pending[p].live) return FN_OK;
        cudaError_t ee = cudaEventSynchronize(st->done[p]);
        if (ee != cudaSuccess) return cuda_fail(ee, "cudaEventSynchronize");
        if (stage_out) {
            const char* hb = static_cast<const char*>(st->hbuf[p]);
            for (int k = 0; k < nout; ++k)
                copy_pool().copy(outs[k] + pending[p].r0 * w, hb + (size_t)(dim + k) * arr, pending[p].m * w);
        }
        pending[p].live = false;
        return FN_OK;
    };
    PipeDrainGuard in_flight;
    in_flight.st = st;
    int64_t chunk = 0;
    for (int64_t r0 = 0; r0 < n; r0 += rows, ++chunk) {
        const int p = (int)(chunk % st->pipes);
        const int64_t m = std::min<int64_t>(rows, n - r0);
        cudaStream_t s = st->streams[p];
        rc = drain(p);
        if (rc != FN_OK) return rc;
        char* base = static_cast<char*>(st->buf[p]);
        char* hbase = static_cast<char*>(st->hbuf[p]);
        const void* dx[4];
        for (int c = 0; c < dim; ++c) {
            const char* src = static_cast<const char*>(xs[c]) + r0 * w;
            if (stage_in) {
                copy_pool().copy(hbase + (size_t)c * arr, src, m * w, copy_threads(stage_out));
                src = hbase + (size_t)c * arr;
            }
            e = cudaMemcpyAsync(base + (size_t)c * arr, src, m * w, cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
            dx[c] = base + (size_t)c * arr;
        }
        void* dout[6];
        for (int k = 0; k < nout; ++k) dout[k] = base + (size_t)(dim + k) * arr;
        rc = run_soa(op, dim, dtype, dx, m, dout[0], wd.w1 ? &dout[1] : nullptr, wd.w2 ? dout[nout - 1] : nullptr, ka,
                     s);
        if (rc != FN_OK) return rc;
        for (int k = 0; k < nout && e == cudaSuccess; ++k) {
            char* dst = stage_out ? hbase + (size_t)(dim + k) * arr : outs[k] + r0 * w;
            e = cudaMemcpyAsync(dst, dout[k], m * w, cudaMemcpyDeviceToHost, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync D2H");
        e = cudaEventRecord(st->done[p], s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
        pending[p] = {true, r0, m};
    }
    for (int64_t c = std::max<int64_t>(0, chunk - st->pipes); c < chunk; ++c) {
        rc = drain((int)(c % st->pipes));
        if (rc != FN_OK) return rc;
    }
    for (int p = 0; p < st->pipes; ++p) {
        e = cudaStreamSynchronize(st->streams[p]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    }
    in_flight.st = nullptr;
    return FN_OK;
}

// ---------------------------------------------------------------------------------
// One row, low latency (the reference's scalar signatures).  The row travels inside the
// kernel's parameter block (no device read of host memory); one thread computes it with
// the same RowOp as the batched kernels, stores the results into a per-thread,
// per-device page-locked buffer mapped into the device address space, fences at system
// scope and publishes a sequence number there.  The host spins on that word instead
// of synchronising the stream (cudaStreamQuery every few thousand spins catches a
// failed launch).  No staging copies, no allocation after the first call.
// ---------------------------------------------------------------------------------
template <typename T, int N> struct RowArg {
    T v[N];
};

constexpr int kScalarFlagOffset = 128;  // bytes; outputs (at most 14 values) sit below

template <typename T, int N, int OP>
__global__ void __launch_bounds__(32) scalar_kernel(RowArg<T, N> x, KArgs<T> ka, T* out,
                                                    unsigned* flag, unsigned seq) {
    using Op = RowOp<T, N, OP>;
    if (threadIdx.x != 0) return;
    T xr[N], o0[Slot<Op::W0>::value], o1[Slot<Op::W1>::value], o2[Slot<Op::W2>::value];
#pragma unroll
    for (int c = 0; c < N; ++c) xr[c] = x.v[c];
    (void)Op::apply(xr, ka, o0, o1, o2);
    int k = 0;
#pragma unroll
    for (int c = 0; c < Op::W0; ++c) out[k++] = o0[c];
#pragma unroll
    for (int c = 0; c < Op::W1; ++c) out[k++] = o1[c];
#pragma unroll
    for (int c = 0; c < Op::W2; ++c) out[k++] = o2[c];
    __threadfence_system();
    *reinterpret_cast<volatile unsigned*>(flag) = seq;
}

struct ScalarCtx {
    int dev = -1;
    cudaStream_t stream = nullptr;
    char* host = nullptr;   // 256 B page-locked, mapped
    char* dptr = nullptr;   // its device alias
    unsigned seq = 0;
};

template <typename T, int N, int OP>
static cudaError_t scalar_launch(const double* xin, const KArgs<T>& ka, const ScalarCtx& c) {
    RowArg<T, N> x;
    for (int k = 0; k < N; ++k) x.v[k] = (T)xin[k];  // f32: the reference's <float> cast
    scalar_kernel<T, N, OP><<<1, 32, 0, c.stream>>>(
        x, ka, reinterpret_cast<T*>(c.dptr), reinterpret_cast<unsigned*>(c.dptr + kScalarFlagOffset), c.seq);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
}

template <typename T, int OP>
static cudaError_t scalar_dim(int dim, const double* xin, const KArgs<T>& ka, const ScalarCtx& c) {
    switch (dim) {
        case 2: return scalar_launch<T, 2, OP>(xin, ka, c);
        case 3: return scalar_launch<T, 3, OP>(xin, ka, c);
        default: return scalar_launch<T, 4, OP>(xin, ka, c);
    }
}

template <typename T>
static int scalar_dispatch(int op, int dim, const double* xin, const double* kad, const ScalarCtx& c) {
    KArgs<T> ka;
    int rc = make_kargs_op<T>(op, kad, needs_ka(op), ka);
    if (rc != FN_OK) return rc;
    cudaError_t e;
    switch (op) {
        case FN_OP_SCALE: e = scalar_dim<T, FN_OP_SCALE>(dim, xin, ka, c); break;
        case FN_OP_NORMALIZE: e = scalar_dim<T, FN_OP_NORMALIZE>(dim, xin, ka, c); break;
        case FN_OP_NORMALIZE_SQ: e = scalar_dim<T, FN_OP_NORMALIZE_SQ>(dim, xin, ka, c); break;
        case FN_OP_NORM: e = scalar_dim<T, FN_OP_NORM>(dim, xin, ka, c); break;
        case FN_OP_NAIVE: e = scalar_dim<T, FN_OP_NAIVE>(dim, xin, ka, c); break;
        case FN_OP_QUOTIENT: e = scalar_dim<T, FN_OP_QUOTIENT>(dim, xin, ka, c); break;
        case FN_OP_QUOTIENT3_FAST:
            if (dim != 3) return fail(FN_EINVAL, "quotient3_fast is defined for dim 3 only");
            e = scalar_launch<T, 3, FN_OP_QUOTIENT3_FAST>(xin, ka, c);
            break;
        default:
            if constexpr (std::is_same<T, double>::value) {
                if (op == FN_OP_ROT_UNIT) { e = scalar_launch<double, 4, FN_OP_ROT_UNIT>(xin, ka, c); break; }
                if (op == FN_OP_ROT_GENERAL) { e = scalar_launch<double, 4, FN_OP_ROT_GENERAL>(xin, ka, c); break; }
                if (op == FN_OP_NORMALIZE_ROT) { e = scalar_launch<double, 4, FN_OP_NORMALIZE_ROT>(xin, ka, c); break; }
                if (op == FN_OP_ROT_APPLY) { e = scalar_launch<double, 3, FN_OP_ROT_APPLY>(xin, ka, c); break; }
            }
            return fail(FN_EINVAL, "unknown op");
    }
    return e == cudaSuccess ? FN_OK : cuda_fail(e, "scalar kernel launch");
}

static inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
}

// Scalar contexts are cached per thread (no lock on the ~10 us path) and handed back to
// a process-wide free list when the thread exits, so short-lived caller threads reuse
// them instead of each leaking a stream and a mapped page-locked buffer.
static std::mutex g_scalar_free_mu;
static std::vector<ScalarCtx>* g_scalar_free = new std::vector<ScalarCtx>();  // never destroyed

struct ScalarCtxCache {
    std::vector<ScalarCtx> ctxs;  // indexed by device
    ~ScalarCtxCache() {
        std::lock_guard<std::mutex> lk(g_scalar_free_mu);
        for (auto& c : ctxs)
            if (c.dev >= 0) g_scalar_free->push_back(c);
    }
    ScalarCtx& get(int dev) {
        if ((int)ctxs.size() <= dev) ctxs.resize(dev + 1);
        ScalarCtx& c = ctxs[dev];
        if (c.dev < 0) {
            std::lock_guard<std::mutex> lk(g_scalar_free_mu);
            for (size_t k = 0; k < g_scalar_free->size(); ++k)
                if ((*g_scalar_free)[k].dev == dev) {
                    c = (*g_scalar_free)[k];
                    g_scalar_free->erase(g_scalar_free->begin() + k);
                    break;
                }
        }
        return c;
    }
};

int scalar_run(int op, int dim, int dtype, const double* xin, double* out, const double* ka) {
    static thread_local ScalarCtxCache cache;
    if (!xin || !out) return fail(FN_EINVAL, "xin and out must not be NULL");
    if (op < FN_OP_SCALE || op > FN_OP_ROT_APPLY || dim < 2 || dim > 4)
        return fail(FN_EINVAL, "unknown op or dim");
    {
        const Widths v = op_widths(op, dim);
        const int rc0 = check_args(op, dim, dtype, xin, 1, out, v.w1 ? out : nullptr, v.w2 ? out : nullptr);
        if (rc0 != FN_OK) return rc0;
    }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    ScalarCtx& c = cache.get(dev);
    if (c.dev < 0) {
        e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        e = cudaHostAlloc(reinterpret_cast<void**>(&c.host), 256, cudaHostAllocMapped);
        if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc");
        memset(c.host, 0, 256);
        e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.dptr), c.host, 0);
        if (e != cudaSuccess) return cuda_fail(e, "cudaHostGetDevicePointer");
        c.dev = dev;
    }
    if (++c.seq == 0) c.seq = 1;  // 0 is the initial flag value
    const int rc = dtype == FN_F64 ? scalar_dispatch<double>(op, dim, xin, ka, c)
                                   : scalar_dispatch<float>(op, dim, xin, ka, c);
    if (rc != FN_OK) return rc;
    unsigned* flag = reinterpret_cast<unsigned*>(c.host + kScalarFlagOffset);
    for (unsigned spin = 1;; ++spin) {
        if (__atomic_load_n(flag, __ATOMIC_ACQUIRE) == c.seq) break;
        if ((spin & 4095u) == 0) {
            e = cudaStreamQuery(c.stream);
            if (e == cudaSuccess) {
                if (__atomic_load_n(flag, __ATOMIC_ACQUIRE) == c.seq) break;
                return fail(FN_ECUDA, "scalar kernel finished without publishing its result");
            }
            if (e != cudaErrorNotReady) return cuda_fail(e, "scalar kernel");
        }
        cpu_relax();
    }
    const Widths wd = op_widths(op, dim);
    const int total = wd.w0 + wd.w1 + wd.w2;
    for (int o = 0; o < total; ++o)
        out[o] = dtype == FN_F64 ? reinterpret_cast<const double*>(c.host)[o]
                                 : (double)reinterpret_cast<const float*>(c.host)[o];
    return FN_OK;
}

// Row shards over several devices, one host thread per device, each running the
// chunked host pipeline above on its own streams and staging buffers.  No data moves
// between devices (rows are independent, _kernels.pyx:167-412).
template <typename ShardFn>
static int over_devices(int64_t n, const int* devices, int ndev, ShardFn shard) {
    if (ndev < 1 || !devices) return fail(FN_EINVAL, "need at least one device");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    for (int k = 0; k < ndev; ++k)
        if (devices[k] < 0 || devices[k] >= count) return fail(FN_EINVAL, "device index out of range");
    std::vector<int> rcs(ndev, FN_OK);
    std::vector<std::string> errs(ndev);
    std::vector<std::thread> pool;
    const int64_t base = n / ndev, extra = n % ndev;
    int64_t lo = 0;
    for (int k = 0; k < ndev; ++k) {
        const int64_t m = base + (k < extra ? 1 : 0);
        const int64_t r0 = lo;
        lo += m;
        pool.emplace_back([&, k, r0, m]() {
            cudaError_t ee = cudaSetDevice(devices[k]);
            if (ee != cudaSuccess) {
                rcs[k] = cuda_fail(ee, "cudaSetDevice");
            } else if (m > 0) {
                rcs[k] = shard(r0, m);
            }
            if (rcs[k] != FN_OK) errs[k] = g_last_error;
        });
    }
    for (auto& t : pool) t.join();
    for (int k = 0; k < ndev; ++k)
        if (rcs[k] != FN_OK) return fail(rcs[k], "device " + std::to_string(devices[k]) + ": " + errs[k]);
    return FN_OK;
}

int host_run_multi(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
                   void* sq, const double* ka, const int* devices, int ndev, int64_t ldx = 0) {
    int rc = check_args(op, dim, dtype, x, n, head, body, sq);
    if (rc != FN_OK) return rc;
    if (ndev < 1 || !devices) return fail(FN_EINVAL, "need at least one device");
    if (n == 0) return FN_OK;
    if (ldx == 0) ldx = dim;
    if (ldx < dim) return fail(FN_EINVAL, "ldx (elements per input row) must be >= dim");
    const size_t w = dtype == FN_F64 ? 8 : 4;
    const Widths wd = op_widths(op, dim);
    return over_devices(n, devices, ndev, [&](int64_t r0, int64_t m) {
        return host_run(op, dim, dtype, static_cast<const char*>(x) + r0 * ldx * w, m,
                        static_cast<char*>(head) + r0 * wd.w0 * w,
                        wd.w1 ? static_cast<char*>(body) + r0 * wd.w1 * w : nullptr,
                        wd.w2 ? static_cast<char*>(sq) + r0 * wd.w2 * w : nullptr, ka, ldx);
    });
}

// The structure-of-arrays host call sharded the same way (each component and output
// array split at the same row boundaries).
int host_run_soa_multi(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head,
                       void* const* body, void* sq, const double* ka, const int* devices, int ndev) {
    if (op < FN_OP_SCALE || op > FN_OP_NORMALIZE_SQ) return fail(FN_EINVAL, "unknown op for the SoA entry");
    if (dim < 2 || dim > 4) return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    if (dtype != FN_F32 && dtype != FN_F64) return fail(FN_EINVAL, "dtype must be FN_F32/FN_F64");
    if (n < 0) return fail(FN_EINVAL, "n must be >= 0");
    if (ndev < 1 || !devices) return fail(FN_EINVAL, "need at least one device");
    if (n == 0) return FN_OK;
    const Widths wd = op_widths(op, dim);
    if (!xs || !head || (wd.w1 && !body)) return fail(FN_EINVAL, "xs, head and body must not be NULL");
    const size_t w = dtype == FN_F64 ? 8 : 4;
    return over_devices(n, devices, ndev, [&](int64_t r0, int64_t m) {
        const void* xk[4] = {};
        void* bk[4] = {};
        for (int c = 0; c < dim; ++c) {
            xk[c] = xs[c] ? static_cast<const char*>(xs[c]) + r0 * w : nullptr;
            if (wd.w1) bk[c] = body[c] ? static_cast<char*>(body[c]) + r0 * w : nullptr;
        }
        return host_run_soa(op, dim, dtype, xk, m, static_cast<char*>(head) + r0 * w, wd.w1 ? bk : nullptr,
                            wd.w2 ? static_cast<char*>(sq) + r0 * w : nullptr, ka);
    });
}

// ---------------------------------------------------------------------------------
// Device-resident shards on several GPUs, driven by one host thread (the north star's
// single-process multi-GPU driver): shard k of the batch lives on device devices[k]
// and runs on a stream of its own, so the devices work concurrently; no data moves
// between devices (rows are independent, _kernels.pyx:167-412) and there is no
// collective.  A device named more than once gets one stream per shard.
// ---------------------------------------------------------------------------------
struct ShardSlot {
    cudaStream_t stream = nullptr;
    cudaEvent_t after = nullptr, t0 = nullptr, t1 = nullptr;
};
static std::mutex g_shard_mu;
// g_shard_slots[dev][j]: the j-th shard stream of device dev; never destroyed
static std::vector<std::vector<ShardSlot>>* g_shard_slots = new std::vector<std::vector<ShardSlot>>();

// Called with the slot's device current.
static int shard_slot(int dev, int j, ShardSlot* out) {
    std::lock_guard<std::mutex> lk(g_shard_mu);
    if ((int)g_shard_slots->size() <= dev) g_shard_slots->resize(dev + 1);
    auto& v = (*g_shard_slots)[dev];
    while ((int)v.size() <= j) {
        ShardSlot s;
        cudaError_t e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.after, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreate(&s.t0);
        if (e == cudaSuccess) e = cudaEventCreate(&s.t1);
        if (e != cudaSuccess) return cuda_fail(e, "shard stream setup");
        v.push_back(s);
    }
    *out = v[j];
    return FN_OK;
}

int run_sharded(int op, int dim, int dtype, int nshard, const int* devices, const void* const* xs,
                const int64_t* ns, void* const* heads, void* const* bodies, void* const* extras,
                const double* ka, void* const* after, float* elapsed_ms) {
    if (nshard < 1) return fail(FN_EINVAL, "need at least one shard");
    if (!devices || !xs || !ns || !heads) return fail(FN_EINVAL, "devices, xs, ns and heads must not be NULL");
    if (op < FN_OP_SCALE || op > FN_OP_NORMALIZE_SQ)
        return fail(FN_EINVAL, "the sharded entry takes the scale / normalize / norm / naive / quotient families");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (dim < 2 || dim > 4) return fail(FN_EINVAL, "dim must be 2, 3 or 4");
    const Widths w = op_widths(op, dim);
    if (w.w1 && !bodies) return fail(FN_EINVAL, "bodies must not be NULL for this op");
    if (w.w2 && !extras) return fail(FN_EINVAL, "extras must not be NULL for this op");
    for (int k = 0; k < nshard; ++k) {
        if (devices[k] < 0 || devices[k] >= count) return fail(FN_EINVAL, "device index out of range");
        const int rc = check_args(op, dim, dtype, xs[k], ns[k], heads[k], w.w1 ? bodies[k] : nullptr,
                                  w.w2 ? extras[k] : nullptr);
        if (rc != FN_OK) return fail(rc, "shard " + std::to_string(k) + ": " + g_last_error);
    }
    // One sharded call at a time: the shard streams and their events are shared by every
    // caller (the call is synchronous, so concurrent callers would only interleave).
    static std::mutex call_mu;
    std::lock_guard<std::mutex> call_lock(call_mu);
    int home = 0;
    e = cudaGetDevice(&home);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::vector<ShardSlot> slot(nshard);
    std::vector<int> nth(nshard, 0);
    int rc = FN_OK, enq = 0;
    std::string err;
    // pass 1: enqueue every shard on its device's stream without waiting for any of them
    for (int k = 0; k < nshard && rc == FN_OK; ++k) {
        for (int j = 0; j < k; ++j) nth[k] += devices[j] == devices[k];
        e = cudaSetDevice(devices[k]);
        if (e != cudaSuccess) { rc = cuda_fail(e, "cudaSetDevice"); break; }
        rc = shard_slot(devices[k], nth[k], &slot[k]);
        if (rc != FN_OK) break;
        enq = k + 1;
        const ShardSlot& s = slot[k];
        if (after && after[k]) {  // the producer of xs[k] on this device
            e = cudaEventRecord(s.after, static_cast<cudaStream_t>(after[k]));
            if (e == cudaSuccess) e = cudaStreamWaitEvent(s.stream, s.after, 0);
            if (e != cudaSuccess) { rc = cuda_fail(e, "wait for the shard's producer stream"); break; }
        }
        if (elapsed_ms) cudaEventRecord(s.t0, s.stream);
        if (ns[k] > 0)
            rc = run(op, dim, dtype, xs[k], ns[k], heads[k], w.w1 ? bodies[k] : nullptr,
                     w.w2 ? extras[k] : nullptr, ka, s.stream);
        if (elapsed_ms) cudaEventRecord(s.t1, s.stream);
        if (rc != FN_OK) err = "shard " + std::to_string(k) + " (device " + std::to_string(devices[k]) + "): " + g_last_error;
    }
    if (rc != FN_OK && err.empty()) err = g_last_error;
    // pass 2: wait for every enqueued shard (also after an error: nothing stays in flight)
    for (int k = 0; k < enq; ++k) {
        if (cudaSetDevice(devices[k]) != cudaSuccess) continue;
        e = cudaStreamSynchronize(slot[k].stream);
        if (e != cudaSuccess && rc == FN_OK) {
            rc = cuda_fail(e, "shard synchronise");
            err = "shard " + std::to_string(k) + " (device " + std::to_string(devices[k]) + "): " + g_last_error;
        }
        if (elapsed_ms) {
            elapsed_ms[k] = 0.f;
            if (e == cudaSuccess) cudaEventElapsedTime(&elapsed_ms[k], slot[k].t0, slot[k].t1);
        }
    }
    cudaSetDevice(home);
    return rc == FN_OK ? FN_OK : fail(rc, err);
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

int fn_run_many(int op, int dim, int dtype, int nseg, const void* const* xs, const int64_t* ns, void* const* heads,
                void* const* bodies, void* const* extras, const double* ka, void* stream) {
    return fnb::run_many(op, dim, dtype, nseg, xs, ns, heads, bodies, extras, ka, stream);
}

int fn_run_sharded(int op, int dim, int dtype, int nshard, const int* devices, const void* const* xs,
                   const int64_t* ns, void* const* heads, void* const* bodies, void* const* extras,
                   const double* ka, void* const* after, float* elapsed_ms) {
    return fnb::run_sharded(op, dim, dtype, nshard, devices, xs, ns, heads, bodies, extras, ka, after, elapsed_ms);
}

int fn_run_ld(int op, int dim, int dtype, const void* x, int64_t n, int64_t ldx, void* head, void* body,
              void* sq, const double* ka, void* stream) {
    if (ldx < 1) return fnb::set_error(FN_EINVAL, "ldx must be >= dim");
    return fnb::run_ex(op, dim, dtype, x, n, head, body, sq, ka, nullptr, stream, ldx);
}

int fn_host_alloc(size_t bytes, void** ptr) {
    if (!ptr) return fnb::set_error(FN_EINVAL, "ptr must not be NULL");
    *ptr = nullptr;
    if (bytes == 0) return FN_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fnb::set_error(FN_ENODEV, "no CUDA device");
    }
    const cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        *ptr = nullptr;
        return fnb::set_error(e == cudaErrorMemoryAllocation ? FN_ENOMEM : FN_ECUDA, cudaGetErrorString(e));
    }
    return FN_OK;
}

int fn_host_is_page_locked(const void* ptr) { return ptr && fnb::is_page_locked(ptr) ? 1 : 0; }

int fn_host_free(void* ptr) {
    if (!ptr) return FN_OK;
    const cudaError_t e = cudaFreeHost(ptr);
    if (e != cudaSuccess) return fnb::set_error(FN_ECUDA, cudaGetErrorString(e));
    return FN_OK;
}

int fn_host_run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
                void* sq, const double* ka) {
    return fnb::host_run(op, dim, dtype, x, n, head, body, sq, ka);
}

int fn_scalar(int op, int dim, int dtype, const double* x, double* out, const double* ka) {
    return fnb::scalar_run(op, dim, dtype, x, out, ka);
}

int fn_host_run_multi(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
                      void* sq, const double* ka, const int* devices, int ndev) {
    return fnb::host_run_multi(op, dim, dtype, x, n, head, body, sq, ka, devices, ndev);
}

int fn_host_run_ld(int op, int dim, int dtype, const void* x, int64_t n, int64_t ldx, void* head, void* body,
                   void* sq, const double* ka) {
    if (ldx < 1) return fnb::set_error(FN_EINVAL, "ldx must be >= dim");
    return fnb::host_run(op, dim, dtype, x, n, head, body, sq, ka, ldx);
}

int fn_host_run_multi_ld(int op, int dim, int dtype, const void* x, int64_t n, int64_t ldx, void* head,
                         void* body, void* sq, const double* ka, const int* devices, int ndev) {
    if (ldx < 1) return fnb::set_error(FN_EINVAL, "ldx must be >= dim");
    return fnb::host_run_multi(op, dim, dtype, x, n, head, body, sq, ka, devices, ndev, ldx);
}

int fn_host_run_soa(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head, void* const* body,
                    void* sq, const double* ka) {
    return fnb::host_run_soa(op, dim, dtype, xs, n, head, body, sq, ka);
}

int fn_host_run_soa_multi(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head,
                          void* const* body, void* sq, const double* ka, const int* devices, int ndev) {
    return fnb::host_run_soa_multi(op, dim, dtype, xs, n, head, body, sq, ka, devices, ndev);
}

int64_t fn_launch_count(void) { return fnb::g_launches.load(std::memory_order_relaxed); }

int64_t fn_small_contexts(void) { return fnb::small_pool().created(); }

int fn_run_soa(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head,
               void* const* body, void* sq, const double* ka, void* stream) {
    return fnb::run_soa(op, dim, dtype, xs, n, head, body, sq, ka, stream);
}

int fn_rotate_rows_f64(int op, const double* a, const double* v, int64_t n, double* out,
                       const double* ka, uint64_t* invalid, void* stream) {
    return fnb::run_rows2(op, a, v, n, out, ka, reinterpret_cast<unsigned long long*>(invalid),
                          static_cast<cudaStream_t>(stream));
}

int fn_host_rotate_rows_f64(int op, const double* a, const double* v, int64_t n, double* out,
                            const double* ka) {
    const int rc = fnb::check_rows2(op, a, v, n, out);
    if (rc != FN_OK || n == 0) return rc;
    return fnb::host_run_impl(op, fnb::rows2_dim(op), FN_F64, a, v, 3, n, out, nullptr, nullptr, ka);
}

int fn_rotate_apply_f64(const double R[9], const double* v, int64_t n, double* out, void* stream) {
    return fnb::run(FN_OP_ROT_APPLY, 3, FN_F64, v, n, out, nullptr, nullptr, R, stream);
}

int fn_run_rot(int op, const double* q, int64_t n, double* head, double* body, double* extra,
               const double* ka, uint64_t* invalid, void* stream) {
    if (!fnb::is_rotation(op)) return fnb::set_error(FN_EINVAL, "fn_run_rot takes a rotation op");
    return fnb::run_ex(op, op == FN_OP_ROT_APPLY ? 3 : 4, FN_F64, q, n, head, body, extra, ka,
                       reinterpret_cast<unsigned long long*>(invalid), stream);
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
