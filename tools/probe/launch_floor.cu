// Round-trip floors on this box: empty kernel + stream sync, and a kernel that writes a
// mapped host flag which the host spins on.
#include <cuda_runtime.h>
#include <cstdio>
#include <chrono>

__global__ void empty_k() {}
__global__ void flag_k(volatile unsigned* f, unsigned s) { __threadfence_system(); *f = s; }

int main() {
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    unsigned* h; cudaHostAlloc((void**)&h, 4096, cudaHostAllocMapped); *h = 0;
    unsigned* d; cudaHostGetDevicePointer((void**)&d, h, 0);
    auto now = [] { return std::chrono::steady_clock::now(); };
    for (int rep = 0; rep < 3; ++rep) {
        const int n = 5000;
        for (int i = 0; i < 100; ++i) { empty_k<<<1, 32, 0, st>>>(); cudaStreamSynchronize(st); }
        auto t0 = now();
        for (int i = 0; i < n; ++i) { empty_k<<<1, 32, 0, st>>>(); cudaStreamSynchronize(st); }
        auto t1 = now();
        unsigned seq = 0;
        auto t2 = now();
        for (int i = 0; i < n; ++i) {
            ++seq; flag_k<<<1, 32, 0, st>>>(d, seq);
            while (__atomic_load_n(h, __ATOMIC_ACQUIRE) != seq) __builtin_ia32_pause();
        }
        auto t3 = now();
        auto t4 = now();
        for (int i = 0; i < n; ++i) empty_k<<<1, 32, 0, st>>>();
        auto t5 = now();
        cudaStreamSynchronize(st);
        printf("empty+sync %.2f us | flag spin %.2f us | launch only (cpu) %.2f us\n",
               std::chrono::duration<double, std::micro>(t1 - t0).count() / n,
               std::chrono::duration<double, std::micro>(t3 - t2).count() / n,
               std::chrono::duration<double, std::micro>(t5 - t4).count() / n);
    }
    return 0;
}
