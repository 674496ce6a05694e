// cfg1_timeline.cu -- per-CTA timeline of one lone config-1 launch (developer probe).
//
// Builds tma_stream_kernel<double, 3, normalize> with FNB_TIMELINE, so thread 0 of every
// CTA stores %globaltimer at: entry, after griddepcontrol.wait, first tile landed, last
// tile's stores issued, bulk stores drained.  Each launch follows a 512 MB read (L2
// flush).  Printed per launch shape (tile rows TR, stages S, CTAs per SM): the event
// time and, relative to the first CTA's entry, percentiles of those five marks.
//
// Build/run (B200): make -C tools/probe timeline && tools/probe/cfg1_timeline [rows=1000000]
#define FNB_TIMELINE 1
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../ws_kernel.cuh"

extern "C" int fn_generate(int cfg, uint64_t seed, int64_t row0, int64_t n, void* x, void* stream);

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

using namespace fnb;

__global__ void read_flush(const int4* __restrict__ p, int64_t n, int* sink) {
    int acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc ^= __ldcs(p + i).x;
    if (acc == 0x7fffffff) *sink = acc;
}

// One CTA stamps %globaltimer: brackets the streaming launch on the same stream.  Its
// dynamic shared memory selects the SM's shared-memory carveout before the launch.
__global__ void marker(unsigned long long* t) {
    if (threadIdx.x == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        t[0] = g;
    }
}

static KArgs<double> make_ka() {
    KArgs<double> ka;
    memset(&ka, 0, sizeof(ka));
    ka.tau_min = 0x1p-482;
    ka.tau_max = 0x1p510;
    ka.sigma_min = 0x1p592;
    ka.sigma_max = 0x1p-514;
    ka.inv_min = 0x1p-592;
    ka.inv_max = 0x1p514;
    memcpy(&ka.tau_min_bits, &ka.tau_min, 8);
    memcpy(&ka.tau_max_bits, &ka.tau_max, 8);
    return ka;
}

static double pct(std::vector<double> v, double p) {
    std::sort(v.begin(), v.end());
    return v[std::min(v.size() - 1, (size_t)(p * (v.size() - 1) + 0.5))];
}

static unsigned long long* g_marks = nullptr;  // [2]: before, after (device)
static int g_marker_smem = -1;                   // -1: no markers

// WS = true: the warp-specialised kernel (256 compute threads + 1 producer warp).
template <int TR, int S, bool WS = false>
static void run_shape(int cps, int64_t n, const double* x, double* r, double* u, const int4* flush,
                      int64_t flush_n, int* sink, unsigned long long* tl, int sms, int reps) {
    using L = TileLayout<double, 3, FN_OP_NORMALIZE, TR, S>;
    auto kern = WS ? tma_ws_kernel<double, 3, FN_OP_NORMALIZE, TR, S> : tma_stream_kernel<double, 3, FN_OP_NORMALIZE, TR, S>;
    const int smem = L::kSmemBytes + (WS ? (S + 2 * L::OB) * 8 : 0);
    const int block = WS ? 256 + 32 : 256;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem));
    const int per = std::min(cps, occ);
    const int64_t ntiles = n / TR;
    const int grid = (int)std::min<int64_t>((int64_t)per * sms, ntiles);
    const KArgs<double> ka = make_ka();
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::vector<double> ev, m[5], gap_in, gap_out;
    // per tile index k (first kTimelineTiles): data wait, compute+stage, store/read-out
    std::vector<double> tw[kTimelineTiles], tc[kTimelineTiles], ts[kTimelineTiles];
    if (g_marker_smem >= 0)
        CK(cudaFuncSetAttribute(marker, cudaFuncAttributeMaxDynamicSharedMemorySize, g_marker_smem));
    std::vector<unsigned long long> h((size_t)grid * kTimelineSlots);
    // reps timed launches without per-tile marks, then reps with them (tile breakdown)
    for (int it = 0; it < 2 * reps + 2; ++it) {
        const int tiles_on = it >= reps + 2;
        CK(cudaMemcpyToSymbol(fnb_timeline_tiles, &tiles_on, sizeof(int)));
        read_flush<<<sms * 8, 256>>>(flush, flush_n, sink);
        if (g_marker_smem >= 0) marker<<<1, 32, g_marker_smem>>>(g_marks);
        CK(cudaEventRecord(e0));
        kern<<<grid, block, smem>>>(x, nullptr, n, r, u, nullptr, ka);
        CK(cudaEventRecord(e1));
        if (g_marker_smem >= 0) marker<<<1, 32, g_marker_smem>>>(g_marks + 1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        if (it < 2) continue;
        CK(cudaMemcpy(h.data(), tl, h.size() * 8, cudaMemcpyDeviceToHost));
        if (tiles_on) {
            for (int b = 0; b < grid; ++b) {
                const unsigned long long* hb = &h[(size_t)b * kTimelineSlots];
                for (int k = 0; k < kTimelineTiles && (int64_t)b + (int64_t)k * grid < ntiles; ++k) {
                    const double prev = k == 0 ? (double)hb[1] : (double)hb[5 + 3 * (k - 1) + 1];
                    tw[k].push_back(((double)hb[5 + 3 * k] - prev) / 1e3);
                    tc[k].push_back(((double)hb[6 + 3 * k] - (double)hb[5 + 3 * k]) / 1e3);
                    ts[k].push_back(((double)hb[7 + 3 * k] - (double)hb[6 + 3 * k]) / 1e3);
                }
            }
            continue;
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ev.push_back(ms * 1e3);
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[(size_t)b * kTimelineSlots]);
        unsigned long long t4 = 0;
        for (int b = 0; b < grid; ++b) t4 = std::max(t4, h[(size_t)b * kTimelineSlots + 4]);
        for (int s = 0; s < 5; ++s)
            for (int b = 0; b < grid; ++b) m[s].push_back((double)(h[(size_t)b * kTimelineSlots + s] - t0) / 1e3);
        if (g_marker_smem >= 0) {
            unsigned long long mk[2];
            CK(cudaMemcpy(mk, g_marks, 16, cudaMemcpyDeviceToHost));
            gap_in.push_back(((double)t0 - (double)mk[0]) / 1e3);
            gap_out.push_back(((double)mk[1] - (double)t4) / 1e3);
        }
    }
    // timer granularity: smallest nonzero gap between sorted entry marks of one launch
    std::vector<unsigned long long> st;
    for (int b = 0; b < grid; ++b) st.push_back(h[(size_t)b * kTimelineSlots]);
    std::sort(st.begin(), st.end());
    unsigned long long gmin = ~0ull;
    for (size_t i = 1; i < st.size(); ++i)
        if (st[i] != st[i - 1]) gmin = std::min(gmin, st[i] - st[i - 1]);
    printf("%sTR=%d S=%d cps=%d grid=%d tiles=%lld tiles/cta=%.2f smem=%d  event_us med=%.2f  timer_step_ns=%llu\n",
           WS ? "WS " : "", TR, S, per, grid, (long long)ntiles, (double)ntiles / grid, smem, pct(ev, 0.5), gmin);
    if (g_marker_smem >= 0)
        printf("  marker(smem=%d) -> first CTA entry us: med=%.2f   last drained -> marker us: med=%.2f\n",
               g_marker_smem, pct(gap_in, 0.5), pct(gap_out, 0.5));
    const char* names[5] = {"entry", "after_wait", "first_tile", "loop_done", "drained"};
    for (int s = 0; s < 5; ++s)
        printf("  %-10s us: p0=%.2f p10=%.2f p50=%.2f p90=%.2f p100=%.2f\n", names[s], pct(m[s], 0), pct(m[s], 0.1),
               pct(m[s], 0.5), pct(m[s], 0.9), pct(m[s], 1.0));
    printf("  per tile (median over CTAs, us; thread 0's view; the globaltimer moves in ~0.26 us steps): "
           "k: wait since prev tile staged / compute+stage / to store read-out\n   ");
    for (int k = 0; k < kTimelineTiles && !tw[k].empty(); ++k)
        printf(" %d: %.2f/%.2f/%.2f", k, pct(tw[k], 0.5), pct(tc[k], 0.5), pct(ts[k], 0.5));
    printf("\n");
    CK(cudaEventDestroy(e0));
    CK(cudaEventDestroy(e1));
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1000000;
    const int reps = 20;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double *x, *r, *u;
    CK(cudaMalloc(&x, n * 24));
    CK(cudaMalloc(&r, n * 8));
    CK(cudaMalloc(&u, n * 24));
    if (fn_generate(1, 0, 0, n, x, nullptr) != 0) return 1;
    const int64_t flush_bytes = 512ll << 20;
    int4* flush;
    int* sink;
    CK(cudaMalloc(&flush, flush_bytes));
    CK(cudaMemset(flush, 1, flush_bytes));
    CK(cudaMalloc(&sink, 4));
    unsigned long long* tl;
    CK(cudaMalloc(&tl, (size_t)sms * 64 * kTimelineSlots * 8));
    CK(cudaMemcpyToSymbol(fnb_timeline, &tl, sizeof(tl)));
    const int64_t fn16 = flush_bytes / 16;
    printf("rows=%lld sms=%d ideal_us_at_6544GBps=%.2f\n", (long long)n, sms, n * 56 / 6544e9 * 1e6);
    for (int cps : {2, 4}) run_shape<256, 4>(cps, n, x, r, u, flush, fn16, sink, tl, sms, reps);
    for (int cps : {2, 3, 4}) run_shape<256, 4, true>(cps, n, x, r, u, flush, fn16, sink, tl, sms, reps);
    for (int cps : {4, 6}) run_shape<128, 4, true>(cps, n, x, r, u, flush, fn16, sink, tl, sms, reps);
    for (int cps : {4, 8}) run_shape<128, 4>(cps, n, x, r, u, flush, fn16, sink, tl, sms, reps);
    run_shape<64, 6>(8, n, x, r, u, flush, fn16, sink, tl, sms, reps);
    run_shape<512, 2>(2, n, x, r, u, flush, fn16, sink, tl, sms, reps);
    // launch gaps around the default shape, with a marker kernel before and after; the
    // marker's dynamic shared memory (0 / the streaming kernel's) sets the carveout
    CK(cudaMalloc(&g_marks, 16));
    for (int ms : {0, 49184, 2 * 49184}) {
        g_marker_smem = ms;
        run_shape<256, 4>(4, n, x, r, u, flush, fn16, sink, tl, sms, reps);
    }
    return 0;
}
