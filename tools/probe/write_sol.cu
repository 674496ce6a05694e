// Write-heavy speed-of-light probes: cudaMemset (pure write), cudaMemcpy D2D (1:1), and a
// plain vectorised kernel with the rotation_unit record shape (32 B read, 72 B written).
#include <cuda_runtime.h>
#include <cstdio>

__global__ void rot_shape(const double2* __restrict__ q, long long npairs, double2* __restrict__ R) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npairs;
         i += (long long)gridDim.x * blockDim.x) {
        double2 a = __ldcs(q + 4 * i), b = __ldcs(q + 4 * i + 1), c = __ldcs(q + 4 * i + 2), d = __ldcs(q + 4 * i + 3);
        double2* o = R + 9 * i;
        __stcs(o + 0, a); __stcs(o + 1, b); __stcs(o + 2, c); __stcs(o + 3, d);
        __stcs(o + 4, make_double2(a.x + b.y, c.x)); __stcs(o + 5, a); __stcs(o + 6, b);
        __stcs(o + 7, c); __stcs(o + 8, d);
    }
}

int main() {
    const long long rows = 1ll << 28;
    double *q, *R;
    cudaMalloc(&q, rows * 32);
    cudaMalloc(&R, rows * 72);
    cudaMemset(q, 0, rows * 32);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) cudaMemsetAsync(R, 1, rows * 72);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("memset write-only: %.1f GB/s\n", 5.0 * rows * 72 / (ms * 1e6));
        cudaEventRecord(e0);
        for (int i = 0; i < 5; ++i) cudaMemcpyAsync(R, q, rows * 32, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("memcpy D2D: %.1f GB/s (read+write)\n", 5.0 * rows * 64 / (ms * 1e6));
        for (int cps = 4; cps <= 16; cps *= 2) {
            cudaEventRecord(e0);
            for (int i = 0; i < 5; ++i) rot_shape<<<148 * cps, 256>>>((const double2*)q, rows / 2, (double2*)R);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            printf("rot-shape plain kernel (%d CTAs/SM): %.1f GB/s (32 B read + 72 B write per row)\n", cps,
                   5.0 * rows * 104 / (ms * 1e6));
        }
    }
    return 0;
}
