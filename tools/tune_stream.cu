// tune_stream.cu -- tile-geometry sweep for the streaming kernel (developer tool).
//
// Times tma_stream_kernel<double, 3, NORMALIZE> (the bench kernel) for several
// (rows per tile, stages, threads, CTAs per SM) choices on BASELINE config-5 rows, and
// two speed-of-light references with the same traffic mix (24 B read + 32 B written
// per row): a 16-byte-vector read/write kernel and cudaMemcpy of the same byte count.
//
// Build: make -C tools tune    Run: tools/tune_stream [log2_rows=28] [reps=20]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>

#include "../paper_1606_06508_b200/csrc/stream_kernel.cuh"

extern "C" int fn_generate(int cfg, uint64_t seed, int64_t row0, int64_t n, void* x, void* stream);

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

using namespace fnb;

// 24 B read + 32 B written per row, 16-byte vectors, grid-stride over row pairs.
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
    double *x, *r, *u;
    int64_t n;
};

template <int TR, int S, int NT, int H>
float time_variant(const Bufs& b, const KArgs<double>& ka, int ctas_per_sm, int reps, int sms,
                   int* occ_out) {
    using L = TileLayout<double, 3, FN_OP_NORMALIZE, TR, S>;
    auto kern = tma_stream_kernel<double, 3, FN_OP_NORMALIZE, TR, S, NT, H>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemBytes));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, L::kSmemBytes));
    *occ_out = occ;
    int per = ctas_per_sm > 0 ? (ctas_per_sm < occ ? ctas_per_sm : occ) : occ;
    int64_t ntiles = b.n / TR;
    int grid = (int)((int64_t)per * sms < ntiles ? (int64_t)per * sms : ntiles);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 2; ++i) kern<<<grid, NT, L::kSmemBytes>>>(b.x, b.n, b.r, b.u, nullptr, ka);
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) kern<<<grid, NT, L::kSmemBytes>>>(b.x, b.n, b.r, b.u, nullptr, ka);
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
    const char* name;
    int tr, s, nt, h, cps;
    float (*fn)(const Bufs&, const KArgs<double>&, int, int, int, int*);
    std::vector<float> ms;
    int occ = 0;
};

#define V(TR, S, NT, H, CPS) \
    Variant{"tma", TR, S, NT, H, CPS, &time_variant<TR, S, NT, H>, {}, 0}

int main(int argc, char** argv) {
    int lg = argc > 1 ? atoi(argv[1]) : 28;
    int reps = argc > 2 ? atoi(argv[2]) : 20;
    Bufs b;
    b.n = (int64_t)1 << lg;
    CK(cudaMalloc(&b.x, b.n * 24));
    CK(cudaMalloc(&b.r, b.n * 8));
    CK(cudaMalloc(&b.u, b.n * 24));
    if (fn_generate(5, 5, 0, b.n, b.x, nullptr) != 0) return 1;
    CK(cudaDeviceSynchronize());
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    KArgs<double> ka;
    ka.tau_min = 0x1p-482; ka.tau_max = 0x1p510; ka.sigma_min = 0x1p592; ka.sigma_max = 0x1p-514;
    ka.inv_min = 0x1p-592; ka.inv_max = 0x1p514;
    memcpy(&ka.tau_min_bits, &ka.tau_min, 8);
    memcpy(&ka.tau_max_bits, &ka.tau_max, 8);
    printf("rows=%lld sms=%d\n", (long long)b.n, sms);

    // speed-of-light references
    {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        int64_t np = b.n / 2;
        for (int g : {sms * 4, sms * 8, sms * 16, sms * 32}) {
            for (int i = 0; i < 3; ++i)
                sol_kernel<<<g, 256>>>((const double2*)b.x, np, (double2*)b.r, (double2*)b.u);
            CK(cudaEventRecord(e0));
            for (int i = 0; i < reps; ++i)
                sol_kernel<<<g, 256>>>((const double2*)b.x, np, (double2*)b.r, (double2*)b.u);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            ms /= reps;
            printf("sol_vec16,grid=%d,ms=%.4f,GBps=%.1f\n", g, ms, b.n * 56.0 / (ms * 1e-3) / 1e9);
        }
        // plain device copy of 28 B/row each way (same 56 B/row total traffic)
        for (int i = 0; i < 3; ++i) CK(cudaMemcpy(b.u, b.x, b.n * 24, cudaMemcpyDeviceToDevice));
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) CK(cudaMemcpy(b.u, b.x, b.n * 24, cudaMemcpyDeviceToDevice));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= reps;
        printf("memcpy_d2d,bytes=%lld,ms=%.4f,GBps(r+w)=%.1f\n", (long long)(b.n * 24), ms,
               b.n * 48.0 / (ms * 1e-3) / 1e9);
        fflush(stdout);
    }
    std::vector<Variant> vs = {
        V(256, 4, 256, 1, 0), V(256, 4, 256, 1, 2), V(256, 4, 256, 1, 3), V(256, 4, 256, 0, 2),
        V(256, 4, 256, 3, 2), V(256, 4, 256, 2, 2), V(256, 4, 256, 0, 4), V(256, 4, 256, 3, 4),
        V(256, 8, 256, 1, 2), V(256, 6, 256, 1, 2), V(512, 4, 256, 1, 2), V(512, 4, 256, 3, 2),
        V(512, 3, 512, 1, 2), V(512, 6, 512, 1, 1), V(1024, 3, 256, 1, 1), V(1024, 3, 256, 3, 1),
        V(1024, 4, 512, 1, 1), V(128, 4, 128, 1, 4), V(128, 4, 128, 1, 3), V(128, 8, 128, 1, 3),
        V(256, 2, 256, 1, 4), V(512, 2, 256, 1, 2),
    };
    const int rounds = 3;
    for (int rd = 0; rd < rounds; ++rd)
        for (auto& v : vs) v.ms.push_back(v.fn(b, ka, v.cps, reps, sms, &v.occ));
    for (auto& v : vs) {
        std::vector<float> m = v.ms;
        std::sort(m.begin(), m.end());
        float med = m[m.size() / 2];
        printf("tma,TR=%d,S=%d,NT=%d,HINTS=%d,occ=%d,ctas_per_sm=%d,ms_med=%.4f,ms_min=%.4f,GBps_med=%.1f,GBps_best=%.1f\n",
               v.tr, v.s, v.nt, v.h, v.occ, v.cps == 0 ? v.occ : std::min(v.cps, v.occ), med, m[0],
               b.n * 56.0 / (med * 1e-3) / 1e9, b.n * 56.0 / (m[0] * 1e-3) / 1e9);
    }
    return 0;
}
