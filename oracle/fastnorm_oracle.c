/*
 * fastnorm_oracle.c -- CPU restatement of the reference kernels, batched.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA library:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It is never linked into, called by, or substituted for the
 * product path (paper_1606_06508_b200/), which fails loudly without its CUDA library.
 *
 * Each routine restates the Cython kernel it cites in pkg/src/fastnorm/_kernels.pyx,
 * in plain C with the reference's own build contract (gcc -O3 -ffp-contract=off,
 * pkg/setup.py:9): one rounding per written operation, left-to-right sums, IEEE
 * division and sqrt from libm, no FMA.  The restatement is pinned bit-for-bit against
 * the reference itself (golden vectors produced by the reference's compiled module and
 * its pure-Python twin, tests/golden/make_golden.py; and, when oracle/_ref is built,
 * live comparison in tests/test_oracle_vs_reference.py).
 *
 * Batched entry points (AoS rows, like the CUDA C ABI):
 *   orc_run(op, dim, dtype, x, n, head, body, sq, ka)   -- op codes of fastnorm_b200.h
 *   orc_loop(algo, dim, dtype, buf, iters, mask, ka)     -- the reference timing loops
 *                                                           (_kernels.pyx:646-789)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

enum { OP_SCALE = 0, OP_NORMALIZE = 1, OP_NORM = 2, OP_NAIVE = 3, OP_QUOTIENT = 4,
       OP_QUOTIENT3_FAST = 5, OP_NORMALIZE_SQ = 6 };
enum { DT_F32 = 0, DT_F64 = 1 };
enum { ALGO_SCALING = 0, ALGO_QUOTIENT = 1, ALGO_QUOTIENT_FAST = 2, ALGO_NAIVE = 3,
       ALGO_EMPTY = 4 };

/*
 * The kernels are written once as a macro over the element type R with its libm
 * functions; instantiated for double (suffix d) and float (suffix f).
 */
#define ORACLE_KERNELS(R, SFX, FABS, SQRT, COPYSIGN, LDEXP)                                     \
                                                                                                \
/* _scale2: _kernels.pyx:51-75 */                                                               \
static void scale2_##SFX(const R* ka, R x1, R x2, R* inv, R* s) {                               \
    R m = FABS(x1);                                                                             \
    if (m >= FABS(x2)) {                                                                        \
        if (m == (R)0) { *inv = 0; s[0] = 0; s[1] = 0; return; }                                \
    } else {                                                                                    \
        m = FABS(x2);                                                                           \
    }                                                                                           \
    if (m >= ka[0]) {                                                                           \
        if (m <= ka[1]) { *inv = 1; s[0] = x1; s[1] = x2; return; }                             \
        *inv = ka[5]; s[0] = ka[3] * x1; s[1] = ka[3] * x2; return;                             \
    }                                                                                           \
    *inv = ka[4]; s[0] = ka[2] * x1; s[1] = ka[2] * x2;                                         \
}                                                                                               \
                                                                                                \
/* _scale3: _kernels.pyx:78-112 */                                                              \
static void scale3_##SFX(const R* ka, R x1, R x2, R x3, R* inv, R* s) {                         \
    R m = FABS(x1);                                                                             \
    if (m < FABS(x2)) {                                                                         \
        m = FABS(x2);                                                                           \
        if (m < FABS(x3)) m = FABS(x3);                                                         \
    } else if (m >= FABS(x3)) {                                                                 \
        if (m == (R)0 && !isnan(x2)) { *inv = 0; s[0] = s[1] = s[2] = 0; return; }              \
    } else {                                                                                    \
        m = FABS(x3);                                                                           \
    }                                                                                           \
    if (m >= ka[0]) {                                                                           \
        if (m <= ka[1]) { *inv = 1; s[0] = x1; s[1] = x2; s[2] = x3; return; }                  \
        *inv = ka[5]; s[0] = ka[3] * x1; s[1] = ka[3] * x2; s[2] = ka[3] * x3; return;          \
    }                                                                                           \
    *inv = ka[4]; s[0] = ka[2] * x1; s[1] = ka[2] * x2; s[2] = ka[2] * x3;                      \
}                                                                                               \
                                                                                                \
/* _scale4: _kernels.pyx:115-160 */                                                             \
static void scale4_##SFX(const R* ka, R x1, R x2, R x3, R x4, R* inv, R* s) {                   \
    R m = FABS(x1);                                                                             \
    if (m < FABS(x2)) {                                                                         \
        m = FABS(x2);                                                                           \
        if (m < FABS(x3)) m = FABS(x3);                                                         \
        if (m < FABS(x4)) m = FABS(x4);                                                         \
    } else if (m < FABS(x3)) {                                                                  \
        m = FABS(x3);                                                                           \
        if (m < FABS(x4)) m = FABS(x4);                                                         \
    } else if (m >= FABS(x4)) {                                                                 \
        if (m == (R)0 && !(isnan(x2) || isnan(x3))) {                                           \
            *inv = 0; s[0] = s[1] = s[2] = s[3] = 0; return;                                    \
        }                                                                                       \
    } else {                                                                                    \
        m = FABS(x4);                                                                           \
    }                                                                                           \
    if (m >= ka[0]) {                                                                           \
        if (m <= ka[1]) { *inv = 1; s[0] = x1; s[1] = x2; s[2] = x3; s[3] = x4; return; }       \
        *inv = ka[5];                                                                           \
        s[0] = ka[3] * x1; s[1] = ka[3] * x2; s[2] = ka[3] * x3; s[3] = ka[3] * x4; return;     \
    }                                                                                           \
    *inv = ka[4];                                                                               \
    s[0] = ka[2] * x1; s[1] = ka[2] * x2; s[2] = ka[2] * x3; s[3] = ka[2] * x4;                 \
}                                                                                               \
                                                                                                \
static void scale_##SFX(int dim, const R* ka, const R* x, R* inv, R* s) {                       \
    if (dim == 2) scale2_##SFX(ka, x[0], x[1], inv, s);                                         \
    else if (dim == 3) scale3_##SFX(ka, x[0], x[1], x[2], inv, s);                              \
    else scale4_##SFX(ka, x[0], x[1], x[2], x[3], inv, s);                                      \
}                                                                                               \
                                                                                                \
/* left-to-right sum of squares, one rounding per operation */                                  \
static R sumsq_##SFX(int dim, const R* s) {                                                     \
    R acc = s[0] * s[0];                                                                        \
    for (int k = 1; k < dim; ++k) acc = acc + s[k] * s[k];                                      \
    return acc;                                                                                 \
}                                                                                               \
                                                                                                \
/* _normalize{2,3,4}: _kernels.pyx:167-225 (+ squared length) */                    \
static void normalize_##SFX(int dim, const R* ka, const R* x, R* r, R* u, R* sq) {              \
    R inv, s[4];                                                                                \
    scale_##SFX(dim, ka, x, &inv, s);                                                           \
    if (inv == (R)0) {                                                                          \
        *r = 0;                                                                                 \
        for (int k = 0; k < dim; ++k) u[k] = 0;                                                 \
        if (dim == 4) u[3] = 1; /* zero quaternion -> identity, :211-218 */                     \
        if (sq) *sq = 0;                                                                        \
        return;                                                                                 \
    }                                                                                           \
    R ss = sumsq_##SFX(dim, s);                                                                 \
    R rt = SQRT(ss);                                                                            \
    R h = (R)1 / rt;                                                                            \
    *r = inv * rt;                                                                              \
    for (int k = 0; k < dim; ++k) u[k] = h * s[k];                                              \
    if (sq) {                                                                                   \
        int e;                                                                                  \
        (void)frexp((double)inv, &e); /* inv = 2^(e-1) */                                       \
        *sq = LDEXP(ss, 2 * (e - 1));                                                           \
    }                                                                                           \
}                                                                                               \
                                                                                                \
/* _norm{2,3,4}: _kernels.pyx:228-255 */                                                        \
static R norm_##SFX(int dim, const R* ka, const R* x) {                                         \
    R inv, s[4];                                                                                \
    scale_##SFX(dim, ka, x, &inv, s);                                                           \
    if (inv == (R)0) return 0;                                                                  \
    return inv * SQRT(sumsq_##SFX(dim, s));                                                     \
}                                                                                               \
                                                                                                \
/* _naive{2,3,4}: _kernels.pyx:262-285 */                                                       \
static void naive_##SFX(int dim, const R* x, R* r, R* u) {                                      \
    R rr = SQRT(sumsq_##SFX(dim, x));                                                           \
    *r = rr;                                                                                    \
    for (int k = 0; k < dim; ++k) u[k] = x[k] / rr;                                             \
}                                                                                               \
                                                                                                \
/* _quotient{2,3,4}: _kernels.pyx:288-362 */                                                    \
static void quotient_##SFX(int dim, const R* x, R* r, R* u) {                                   \
    R m = FABS(x[0]);                                                                           \
    int anynan = isnan(x[0]);                                                                   \
    for (int k = 1; k < dim; ++k) {                                                             \
        R a = FABS(x[k]);                                                                       \
        if (a > m) m = a;                                                                       \
        anynan = anynan || isnan(x[k]);                                                         \
    }                                                                                           \
    if (m == (R)0 && !anynan) {                                                                 \
        *r = 0;                                                                                 \
        for (int k = 0; k < dim; ++k) u[k] = 0;                                                 \
        return;                                                                                 \
    }                                                                                           \
    R q[4];                                                                                     \
    for (int k = 0; k < dim; ++k) q[k] = x[k] / m;                                              \
    R h = SQRT(sumsq_##SFX(dim, q));                                                            \
    *r = m * h;                                                                                 \
    for (int k = 0; k < dim; ++k) u[k] = q[k] / h;                                              \
}                                                                                               \
                                                                                                \
/* pivot body of _quotient3_fast: _kernels.pyx:370-377 */                                      \
static void qf_pivot_##SFX(R p, R a, R b, R* r, R* t, R* ua, R* ub) {                           \
    R qa = a / p;                                                                               \
    R qb = b / p;                                                                               \
    R h = SQRT((R)1 + qa * qa + qb * qb);                                                       \
    *t = COPYSIGN((R)1, p) / h;                                                                 \
    *r = FABS(p) * h;                                                                           \
    *ua = qa * *t;                                                                              \
    *ub = qb * *t;                                                                              \
}                                                                                               \
                                                                                                \
/* _quotient3_fast: _kernels.pyx:365-412 */                                                     \
static void quotient3_fast_##SFX(const R* x, R* r, R* u) {                                      \
    R t, ua, ub;                                                                                \
    if (FABS(x[0]) > FABS(x[1])) {                                                              \
        if (FABS(x[2]) > FABS(x[0])) {                                                          \
            qf_pivot_##SFX(x[2], x[0], x[1], r, &t, &ua, &ub);                                  \
            u[0] = ua; u[1] = ub; u[2] = t;                                                     \
        } else {                                                                                \
            qf_pivot_##SFX(x[0], x[2], x[1], r, &t, &ua, &ub);                                  \
            u[0] = t; u[1] = ub; u[2] = ua;                                                     \
        }                                                                                       \
    } else if (FABS(x[2]) >= FABS(x[1])) {                                                      \
        if (x[2] == (R)0 && !isnan(x[0])) {                                                     \
            *r = 0; u[0] = u[1] = u[2] = 0; return;                                             \
        }                                                                                       \
        qf_pivot_##SFX(x[2], x[0], x[1], r, &t, &ua, &ub);                                      \
        u[0] = ua; u[1] = ub; u[2] = t;                                                         \
    } else {                                                                                    \
        qf_pivot_##SFX(x[1], x[0], x[2], r, &t, &ua, &ub);                                      \
        u[0] = ua; u[1] = t; u[2] = ub;                                                         \
    }                                                                                           \
}                                                                                               \
                                                                                                \
static void row_##SFX(int op, int dim, const R* ka, const R* x, R* head, R* body, R* sq) {      \
    switch (op) {                                                                               \
        case OP_SCALE: scale_##SFX(dim, ka, x, head, body); break;                              \
        case OP_NORMALIZE: normalize_##SFX(dim, ka, x, head, body, 0); break;                   \
        case OP_NORMALIZE_SQ: normalize_##SFX(dim, ka, x, head, body, sq); break;               \
        case OP_NORM: *head = norm_##SFX(dim, ka, x); break;                                    \
        case OP_NAIVE: naive_##SFX(dim, x, head, body); break;                                  \
        case OP_QUOTIENT: quotient_##SFX(dim, x, head, body); break;                            \
        case OP_QUOTIENT3_FAST: quotient3_fast_##SFX(x, head, body); break;                     \
        default: break;                                                                         \
    }                                                                                           \
}                                                                                               \
                                                                                                \
static void run_##SFX(int op, int dim, const R* x, int64_t n, R* head, R* body, R* sq,          \
                      const double* kad) {                                                      \
    R ka[6] = {0, 0, 0, 0, 0, 0};                                                               \
    if (kad)                                                                                    \
        for (int k = 0; k < 6; ++k) ka[k] = (R)kad[k]; /* <float> casts, :526-527 */            \
    for (int64_t i = 0; i < n; ++i) {                                                           \
        R b[4], q = 0;                                                                          \
        row_##SFX(op, dim, ka, x + i * dim, head + i, b, &q);                                   \
        if (body)                                                                               \
            for (int k = 0; k < dim; ++k) body[i * dim + k] = b[k];                             \
        if (sq) sq[i] = q;                                                                      \
    }                                                                                           \
}                                                                                               \
                                                                                                \
/* timing-loop bodies: _kernels.pyx:646-789 -- acc += <double>r + <double>u1 + ... */           \
static double loop_##SFX(int algo, int dim, const R* buf, int64_t iters, int64_t mask,          \
                         const double* kad) {                                                   \
    R ka[6] = {0, 0, 0, 0, 0, 0};                                                               \
    if (kad)                                                                                    \
        for (int k = 0; k < 6; ++k) ka[k] = (R)kad[k];                                          \
    double acc = 0.0;                                                                           \
    for (int64_t i = 0; i < iters; ++i) {                                                       \
        const R* x = buf + (i & mask) * dim;                                                    \
        R r, u[4];                                                                              \
        double term;                                                                            \
        if (algo == ALGO_EMPTY) {                                                               \
            term = (double)x[0];                                                                \
            for (int k = 1; k < dim; ++k) term = term + (double)x[k];                           \
            acc += term;                                                                        \
            continue;                                                                           \
        }                                                                                       \
        if (algo == ALGO_SCALING) normalize_##SFX(dim, ka, x, &r, u, 0);                        \
        else if (algo == ALGO_QUOTIENT) quotient_##SFX(dim, x, &r, u);                          \
        else if (algo == ALGO_QUOTIENT_FAST) quotient3_fast_##SFX(x, &r, u);                    \
        else naive_##SFX(dim, x, &r, u);                                                        \
        term = (double)r;                                                                       \
        for (int k = 0; k < dim; ++k) term = term + (double)u[k];                               \
        acc += term;                                                                            \
    }                                                                                           \
    return acc;                                                                                 \
}

ORACLE_KERNELS(double, d, fabs, sqrt, copysign, ldexp)
ORACLE_KERNELS(float, f, fabsf, sqrtf, copysignf, ldexpf)

int orc_run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
            void* sq, const double* ka) {
    if (dim < 2 || dim > 4 || n < 0) return -1;
    if (op == OP_QUOTIENT3_FAST && dim != 3) return -1;
    if (dtype == DT_F64)
        run_d(op, dim, (const double*)x, n, (double*)head, (double*)body, (double*)sq, ka);
    else
        run_f(op, dim, (const float*)x, n, (float*)head, (float*)body, (float*)sq, ka);
    return 0;
}

double orc_loop(int algo, int dim, int dtype, const void* buf, int64_t iters, int64_t mask,
                const double* ka) {
    if (dtype == DT_F64) return loop_d(algo, dim, (const double*)buf, iters, mask, ka);
    return loop_f(algo, dim, (const float*)buf, iters, mask, ka);
}

/*
 * Rotations of quaternions (rotation.py:53-111), binary64, Python evaluation order.
 * op 7 = rotation_unit (:87-111), 8 = rotation_general (:53-84, via _scale4 on the
 * double kernel args), 9 = normalize4 then rotation_unit of the unit output.
 * Returns the number of rows the reference would reject (ValueError); those rows get
 * NaN matrices.  head = R[N*9] for 7/8; for 9: head = r[N], body = unit[N*4], R = sq.
 */
static int rot_unit(const double* q, double* R) {
    int ok = isfinite(q[0]) && isfinite(q[1]) && isfinite(q[2]) && isfinite(q[3]);
    double q1 = q[0], q2 = q[1], q3 = q[2], q4 = q[3];
    R[0] = 1.0 - 2.0 * (q2 * q2 + q3 * q3);
    R[1] = 2.0 * (q1 * q2 - q3 * q4);
    R[2] = 2.0 * (q1 * q3 + q2 * q4);
    R[3] = 2.0 * (q1 * q2 + q3 * q4);
    R[4] = 1.0 - 2.0 * (q1 * q1 + q3 * q3);
    R[5] = 2.0 * (q2 * q3 - q1 * q4);
    R[6] = 2.0 * (q1 * q3 - q2 * q4);
    R[7] = 2.0 * (q2 * q3 + q1 * q4);
    R[8] = 1.0 - 2.0 * (q1 * q1 + q2 * q2);
    if (!ok)
        for (int k = 0; k < 9; ++k) R[k] = NAN;
    return ok;
}

static int rot_general(const double* ka, const double* x, double* R) {
    int ok = isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]) && isfinite(x[3]);
    double inv, q[4];
    scale4_d(ka, x[0], x[1], x[2], x[3], &inv, q);
    ok = ok && inv != 0.0;
    double q1 = q[0], q2 = q[1], q3 = q[2], q4 = q[3];
    double ss = q1 * q1 + q2 * q2 + q3 * q3 + q4 * q4;
    R[0] = (q1 * q1 + q4 * q4 - q2 * q2 - q3 * q3) / ss;
    R[1] = 2.0 * (q1 * q2 - q3 * q4) / ss;
    R[2] = 2.0 * (q1 * q3 + q2 * q4) / ss;
    R[3] = 2.0 * (q1 * q2 + q3 * q4) / ss;
    R[4] = (q2 * q2 + q4 * q4 - q1 * q1 - q3 * q3) / ss;
    R[5] = 2.0 * (q2 * q3 - q1 * q4) / ss;
    R[6] = 2.0 * (q1 * q3 - q2 * q4) / ss;
    R[7] = 2.0 * (q2 * q3 + q1 * q4) / ss;
    R[8] = (q3 * q3 + q4 * q4 - q1 * q1 - q2 * q2) / ss;
    if (!ok)
        for (int k = 0; k < 9; ++k) R[k] = NAN;
    return ok;
}

int64_t orc_rotation(int op, const double* q, int64_t n, double* head, double* body, double* rot,
                     const double* ka) {
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (op == 7) {
            bad += !rot_unit(q + 4 * i, head + 9 * i);
        } else if (op == 8) {
            bad += !rot_general(ka, q + 4 * i, head + 9 * i);
        } else {
            double r, u[4];
            normalize_d(4, ka, q + 4 * i, &r, u, 0);
            head[i] = r;
            for (int k = 0; k < 4; ++k) body[4 * i + k] = u[k];
            bad += !rot_unit(u, rot + 9 * i);
        }
    }
    return bad;
}

/* RotationMatrix.apply (rotation.py:39-41) with one matrix over v[N,3]:
 * out_i = r[0]*v[0] + r[1]*v[1] + r[2]*v[2], evaluated left to right (Python floats). */
void orc_rotate_apply(const double* R, const double* v, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) {
        const double* x = v + 3 * i;
        for (int k = 0; k < 3; ++k)
            out[3 * i + k] = R[3 * k] * x[0] + R[3 * k + 1] * x[1] + R[3 * k + 2] * x[2];
    }
}

/* Per-row rotation of vectors (two inputs):
 * op 11: out_i = rotation_unit(normalize4(q_i).unit).apply(v_i)  (normalize.py:65,
 *        rotation.py:87-111, :39-41); returns the rows whose unit quaternion is
 *        non-finite (the reference's rotation_unit raises ValueError there; NaN here);
 * op 12: out_i = R_i.apply(v_i) with R_i the row-major 3x3 a[9 i .. 9 i + 8]. */
int64_t orc_rotate_rows(int op, const double* a, const double* v, int64_t n, double* out,
                        const double* ka) {
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        double R[9];
        const double* M = R;
        if (op == 11) {
            double r, u[4];
            normalize_d(4, ka, a + 4 * i, &r, u, 0);
            bad += !rot_unit(u, R);
        } else {
            M = a + 9 * i;
        }
        orc_rotate_apply(M, v + 3 * i, 1, out + 3 * i);
    }
    return bad;
}

const char* orc_build_flags(void) { return "gcc -O3 -ffp-contract=off"; }
