/* fn_scalar latency from C (no Python): us per call, median of 5 x 2000 calls. */
#include <stdio.h>
#include <time.h>
#include "../../include/fastnorm_b200.h"

static double now(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}

int main(void) {
    const double ka[6] = {0x1p-482, 0x1p510, 0x1p592, 0x1p-514, 0x1p-592, 0x1p514};
    const double x[3] = {3.0, 4.0, 12.0};
    double out[4];
    for (int i = 0; i < 200; ++i)
        if (fn_scalar(FN_OP_NORMALIZE, 3, FN_F64, x, out, ka)) { printf("err %s\n", fn_last_error()); return 1; }
    for (int rep = 0; rep < 5; ++rep) {
        const int n = 2000;
        double t0 = now();
        for (int i = 0; i < n; ++i) fn_scalar(FN_OP_NORMALIZE, 3, FN_F64, x, out, ka);
        double t1 = now();
        printf("fn_scalar normalize3 f64: %.2f us/call  (r=%g u=%g,%g,%g)\n", (t1 - t0) / n * 1e6, out[0], out[1], out[2], out[3]);
    }
    return 0;
}
