/*
 * normalize_host.c -- calling the library from plain C through include/fastnorm_b200.h.
 *
 * Normalizes N host-resident 3-D float64 vectors with the scaling algorithm
 * (fn_host_run: chunked H2D -> kernel -> D2H) and prints a few results, then checks
 * the error path.  Build and run (needs a GPU to run):
 *   make -C examples && ./examples/normalize_host 1000000
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "fastnorm_b200.h"

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 1000;
    /* kernel_args(preset("double")): tau_min, tau_max, sigma_min, sigma_max, 1/sigma_min, 1/sigma_max */
    const double ka[6] = {0x1p-482, 0x1p510, 0x1p592, 0x1p-514, 0x1p-592, 0x1p514};
    double* x = malloc(sizeof(double) * 3 * n);
    double* r = malloc(sizeof(double) * n);
    double* u = malloc(sizeof(double) * 3 * n);
    if (!x || !r || !u) return 1;
    for (int64_t i = 0; i < n; ++i) {
        x[3 * i] = 3.0 * ldexp(1.0, (int)(i % 2000) - 1000);
        x[3 * i + 1] = 4.0 * ldexp(1.0, (int)(i % 2000) - 1000);
        x[3 * i + 2] = 12.0 * ldexp(1.0, (int)(i % 2000) - 1000);
    }
    printf("%s, %d device(s)\n", fn_version(), fn_device_count());
    int rc = fn_host_run(FN_OP_NORMALIZE, 3, FN_F64, x, n, r, u, NULL, ka);
    if (rc != FN_OK) {
        fprintf(stderr, "fn_host_run failed (%d): %s\n", rc, fn_last_error());
        return 2;
    }
    for (int64_t i = 0; i < n && i < 3; ++i)
        printf("row %lld: r = %.17g  unit = (%.17g, %.17g, %.17g)\n", (long long)i, r[i], u[3 * i],
               u[3 * i + 1], u[3 * i + 2]);
    /* (3, 4, 12) * 2^k has length 13 * 2^k exactly, at every scale */
    for (int64_t i = 0; i < n; ++i)
        if (r[i] != 13.0 * ldexp(1.0, (int)(i % 2000) - 1000)) {
            fprintf(stderr, "row %lld: unexpected length %.17g\n", (long long)i, r[i]);
            return 3;
        }
    /* the same rows as xyz of xyzw records (padding never read): fn_host_run_ld, ldx 4 */
    double* x4 = malloc(sizeof(double) * 4 * n);
    double* r4 = malloc(sizeof(double) * n);
    double* u4 = malloc(sizeof(double) * 3 * n);
    if (!x4 || !r4 || !u4) return 1;
    for (int64_t i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c) x4[4 * i + c] = x[3 * i + c];
        x4[4 * i + 3] = NAN;
    }
    rc = fn_host_run_ld(FN_OP_NORMALIZE, 3, FN_F64, x4, n, 4, r4, u4, NULL, ka);
    if (rc != FN_OK) {
        fprintf(stderr, "fn_host_run_ld failed (%d): %s\n", rc, fn_last_error());
        return 2;
    }
    for (int64_t i = 0; i < n; ++i)
        if (r4[i] != r[i] || u4[3 * i] != u[3 * i] || u4[3 * i + 1] != u[3 * i + 1] || u4[3 * i + 2] != u[3 * i + 2]) {
            fprintf(stderr, "row %lld: padded records differ from dense rows\n", (long long)i);
            return 5;
        }
    printf("xyz of xyzw records: %lld rows identical to the dense call\n", (long long)n);
    free(x4);
    free(r4);
    free(u4);
    /* argument errors come back as FN_EINVAL with a message */
    rc = fn_host_run(FN_OP_QUOTIENT3_FAST, 2, FN_F64, x, n, r, u, NULL, NULL);
    printf("quotient3_fast with dim 2 -> %d (%s)\n", rc, fn_last_error());
    free(x);
    free(r);
    free(u);
    return rc == FN_EINVAL ? 0 : 4;
}
