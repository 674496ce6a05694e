// cfg1_lone.cu -- lone-launch time of one config-1 batch (1e6 x 3 f64 normalize3), no
// instrumentation: each launch follows a 512 MB read (L2 flush) and is timed with CUDA
// events; median of 50.  Compares tma_stream_kernel with the warp-specialised
// tma_ws_kernel over launch shapes, and a back-to-back stream of 64 launches per shape.
//
// Build/run (B200): make -C tools lone && tools/probe/cfg1_lone [rows=1000000]
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

struct Ctx {
    int64_t n;
    const double* x;
    double *r, *u;
    const int4* flush;
    int64_t flush_n;
    int* sink;
    int sms;
};

template <int TR, int S, bool WS, int NT = 256>
static void shape(const Ctx& c, int cps) {
    using L = TileLayout<double, 3, FN_OP_NORMALIZE, TR, S>;
    auto kern = WS ? tma_ws_kernel<double, 3, FN_OP_NORMALIZE, TR, S, NT>
                   : tma_stream_kernel<double, 3, FN_OP_NORMALIZE, TR, S, NT>;
    const int smem = L::kSmemBytes + (WS ? (S + 2 * L::OB) * 8 : 0);
    const int block = WS ? NT + 32 : NT;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem));
    const int per = std::min(cps, occ);
    const int grid = (int)std::min<int64_t>((int64_t)per * c.sms, c.n / TR);
    const KArgs<double> ka = make_ka();
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::vector<float> t;
    for (int it = 0; it < 53; ++it) {
        read_flush<<<c.sms * 8, 256>>>(c.flush, c.flush_n, c.sink);
        CK(cudaEventRecord(e0));
        kern<<<grid, block, smem>>>(c.x, nullptr, c.n, c.r, c.u, nullptr, ka);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (it >= 3) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    // back-to-back stream: 64 launches over the same buffers (outputs stay partly in L2)
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 64; ++i) kern<<<grid, block, smem>>>(c.x, nullptr, c.n, c.r, c.u, nullptr, ka);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("%s TR=%d S=%d NT=%d cps=%d grid=%d  lone_us med=%.2f p10=%.2f  stream_us_per_launch=%.2f\n",
           WS ? "ws    " : "stream", TR, S, NT, per, grid, t[t.size() / 2], t[t.size() / 10], ms * 1e3 / 64);
    CK(cudaEventDestroy(e0));
    CK(cudaEventDestroy(e1));
}

int main(int argc, char** argv) {
    Ctx c;
    c.n = argc > 1 ? atoll(argv[1]) : 1000000;
    CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, 0));
    double *x, *r, *u;
    CK(cudaMalloc(&x, c.n * 24));
    CK(cudaMalloc(&r, c.n * 8));
    CK(cudaMalloc(&u, c.n * 24));
    if (fn_generate(1, 0, 0, c.n, x, nullptr) != 0) return 1;
    const int64_t flush_bytes = 512ll << 20;
    int4* flush;
    CK(cudaMalloc(&flush, flush_bytes));
    CK(cudaMemset(flush, 1, flush_bytes));
    CK(cudaMalloc(&c.sink, 4));
    c.x = x;
    c.r = r;
    c.u = u;
    c.flush = flush;
    c.flush_n = flush_bytes / 16;
    printf("rows=%lld ideal_us_at_6544GBps=%.2f\n", (long long)c.n, c.n * 56 / 6544e9 * 1e6);
    for (int rep = 0; rep < 2; ++rep) {
        for (int cps : {2, 4}) shape<256, 4, false>(c, cps);
        for (int cps : {2, 3, 4}) shape<256, 4, true>(c, cps);
        for (int cps : {2, 4}) shape<256, 4, true, 128>(c, cps);
        for (int cps : {4, 6}) shape<128, 4, true, 128>(c, cps);
        shape<128, 4, false, 128>(c, 4);
    }
    return 0;
}
