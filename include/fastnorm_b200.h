/*
 * fastnorm_b200.h -- C ABI of the B200 (sm_100a) batched normalization library.
 *
 * This is the drop-in boundary for the reference package's kernel registry.
 * The reference resolves every kernel by name through
 *     getattr(module, f"{base}_{suffix}")                 (_backend.py:86-93)
 * over the flat scalar exports of its Cython module
 *     {base}_{f32,f64}(tau_min, tau_max, sigma_min, sigma_max, inv_min, inv_max, x1..xn)
 *                                                         (_kernels.pyx:419-634)
 * This library exports the same 16 kernel families x 2 precisions, batched over an
 * AoS array of N rows, as  fn_{base}_{f32,f64}.  The six scaling constants keep the
 * reference's meaning and order (scale.py:26-30 kernel_args) and are always passed as
 * doubles; the f32 entry points round them to binary32 exactly like the reference's
 * `<float>` casts (_kernels.pyx:526-527).
 *
 * Layout (all arrays caller-owned, contiguous, C order):
 *   x     [N, n]  input rows (AoS: x1..xn of row i at x[i*n .. i*n+n-1])
 *   r     [N]     length           (normalize / norm / naive / quotient families)
 *   inv   [N]     inverse scale    (scale family; 0 marks an all-zero row)
 *   unit  [N, n]  unit vector      (normalize / naive / quotient families)
 *   scaled[N, n]  scaled row       (scale family)
 *   sq    [N]     squared length, ldexp(ss, 2*log2(inv)) (the *_sq entry points; no
 *                 reference function exists -- see DESIGN.md "squared norm")
 *
 * Device entry points (fn_*): every pointer is device memory (or managed); the call
 * enqueues work on `stream` (a cudaStream_t, NULL = legacy default stream) and returns
 * without synchronising.  Host entry points (fn_host_*): every pointer is host memory
 * (pinned is fastest); the call copies in, computes on the current device, copies out
 * and returns when the results are in the caller's buffers.
 *
 * Errors: kernels never fail on values -- IEEE results for every input, exactly as the
 * reference (`cdivision=True`, _kernels.pyx:5).  Argument problems return a negative
 * fn_status; the message is available from fn_last_error() (per thread).  ka must
 * satisfy the reference's validate_conditions (params.py:134-197), which kernel_args
 * enforces upstream (scale.py:26-30); the library itself rejects only tau values that
 * are negative or NaN (they would break the bit-pattern band test).
 *
 * Thread safety: stateless apart from the per-thread last-error slot and a per-device
 * cache of staging buffers used by the fn_host_* entry points (mutex protected).
 */
#ifndef FASTNORM_B200_H
#define FASTNORM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FN_OK = 0,
    FN_EINVAL = -1,   /* bad N, NULL pointer, bad ka, unknown op/dim/dtype */
    FN_ECUDA = -2,    /* a CUDA runtime error; see fn_last_error() */
    FN_ENODEV = -3,   /* no CUDA device visible */
    FN_ENOMEM = -4    /* staging allocation failed (host entry points) */
} fn_status;

/* Kernel families (reference names, tests/test_backends.py:20-27). */
typedef enum {
    FN_OP_SCALE = 0,          /* scale{2,3,4}        _kernels.pyx:51-160  */
    FN_OP_NORMALIZE = 1,      /* normalize{2,3,4}    _kernels.pyx:167-225 */
    FN_OP_NORM = 2,           /* norm{2,3,4}         _kernels.pyx:228-255 */
    FN_OP_NAIVE = 3,          /* naive{2,3,4}        _kernels.pyx:262-285 */
    FN_OP_QUOTIENT = 4,       /* quotient{2,3,4}     _kernels.pyx:288-362 */
    FN_OP_QUOTIENT3_FAST = 5, /* quotient3_fast      _kernels.pyx:365-412 */
    FN_OP_NORMALIZE_SQ = 6,   /* normalize{2,3,4} + squared length (BASELINE config 3) */
    /* Rotations of quaternions (rotation.py:53-111; dim 4, FN_F64 only).  head = R[N,3,3]
     * row-major.  Rows the reference rejects with ValueError (non-finite; zero for the
     * general form) get NaN matrices and are counted into *invalid (fn_run_rot). */
    FN_OP_ROT_UNIT = 7,       /* rotation_unit(q)                      rotation.py:87-111 */
    FN_OP_ROT_GENERAL = 8,    /* rotation_general(q) via scale4        rotation.py:53-84  */
    FN_OP_NORMALIZE_ROT = 9,  /* normalize4 fused with rotation_unit of its unit output:
                                 head = r[N], body = unit[N,4], sq slot = R[N,3,3]       */
    /* RotationMatrix.apply (rotation.py:39-41) over a batch of vectors: x = v[N,3]
     * (dim 3, FN_F64), head = R v [N,3]; the ka argument points to the 9 entries of R,
     * row-major.  out_i = ((R_i0 v_0 + R_i1 v_1) + R_i2 v_2), each operation rounded. */
    FN_OP_ROT_APPLY = 10,
    /* Two-input ops (fn_rotate_rows_f64 / fn_host_rotate_rows_f64 only), float64, one
     * output record out[N,3] per row:
     *  QUAT_ROTATE: a = q[N,4]; out_i = rotation_unit(normalize4(p, q_i).unit).apply(v_i)
     *               (normalize.py:65 -> rotation.py:87-111 -> rotation.py:39-41); rows
     *               with a non-finite quaternion give NaN and are counted (*invalid).
     *  MAT_APPLY:   a = R[N,9] row-major; out_i = R_i.apply(v_i) (rotation.py:39-41). */
    FN_OP_QUAT_ROTATE = 11,
    FN_OP_MAT_APPLY = 12
} fn_op;

typedef enum { FN_F32 = 0, FN_F64 = 1 } fn_dtype;

/* ---- library metadata ------------------------------------------------------------- */
const char* fn_version(void);         /* e.g. "fastnorm-b200 0.1.0 sm_100a"             */
const char* fn_build_flags(void);     /* nvcc flags (reference analogue: BUILD_FLAGS)   */
const char* fn_backend_name(void);    /* "cuda"  (reference analogue: BACKEND_NAME)     */
const char* fn_last_error(void);      /* message of the last failing call on this thread */
int fn_device_count(void);

/* ---- generic entry points --------------------------------------------------------- */
/* head = r (or inv for FN_OP_SCALE); body = unit (or scaled); sq only for
 * FN_OP_NORMALIZE_SQ.  body must be NULL for FN_OP_NORM.  ka is ignored (may be NULL)
 * for the naive / quotient families, which take no constants (_kernels.pyx:481-520). */
int fn_run(int op, int dim, int dtype, const void* x, int64_t n, void* head, void* body,
           void* sq, const double* ka, void* stream);
/* Many independent batches in one launch: segment j is xs[j] [ns[j], dim] with its own
 * outputs heads[j] / bodies[j] / extras[j] (bodies / extras may be NULL when the op has
 * no such output).  16-byte aligned segments stream through one bulk-copy kernel (up to
 * 48 per launch), so a stream of small batches pays one launch ramp and tail instead of
 * one per batch; other segments are launched on their own.  Ops SCALE..NORMALIZE_SQ.
 * Async on stream.  No reference interface (the reference takes one row per call). */
int fn_run_many(int op, int dim, int dtype, int nseg, const void* const* xs, const int64_t* ns,
                void* const* heads, void* const* bodies, void* const* extras, const double* ka,
                void* stream);
/* One batch as device-resident row shards on several GPUs of this process, driven by one
 * host thread (north star (c): one stream per device, no collective on the data path):
 * shard k is xs[k] [ns[k], dim] on device devices[k] with outputs heads[k] / bodies[k] /
 * extras[k] on the same device (bodies / extras may be NULL when the op has no such
 * output).  Every shard's kernel is enqueued on a library-owned stream of its device
 * before any is waited for, then all are synchronised: the call returns with every output
 * complete.  after[k] (after may be NULL, and so may any entry) is a stream of device
 * devices[k] whose already-enqueued work (the producer of xs[k]) the shard waits for.
 * elapsed_ms[k] (may be NULL) receives shard k's device time by CUDA events on its stream.
 * A device may be named more than once (one stream per shard).  Calls from several host
 * threads are serialised.  Ops SCALE..NORMALIZE_SQ.
 * No reference interface: the reference is CPU only and takes one row per call. */
int fn_run_sharded(int op, int dim, int dtype, int nshard, const int* devices, const void* const* xs,
                   const int64_t* ns, void* const* heads, void* const* bodies, void* const* extras,
                   const double* ka, void* const* after, float* elapsed_ms);
/* fn_run over rows that are ldx elements apart (ldx >= dim): row i is x[i*ldx .. i*ldx+dim),
 * the other ldx - dim elements of each record are not used.  Padded records such as xyz
 * in xyzw (dim 3, ldx 4; float4-style 16 B / 32 B records) and views like X[:, :3] of a
 * wider array run without a gather copy.  dim 3 with ldx 4 and 16 B aligned buffers uses
 * the bulk-copy kernel (whole records staged, the first three elements read); other
 * strides use the per-row kernel.  Outputs are dense, as for fn_run.  ldx == dim is
 * fn_run.  No reference interface: the reference takes one row per call. */
int fn_run_ld(int op, int dim, int dtype, const void* x, int64_t n, int64_t ldx, void* head,
              void* body, void* sq, const double* ka, void* stream);
int fn_host_run(int op, int dim, int dtype, const void* x, int64_t n, void* head,
                void* body, void* sq, const double* ka);
/* Structure-of-arrays rows on the device: the reference's scalar signatures vectorised
 * over arrays (normalize.py:51-89 / scale.py:33-51 / baselines.py:30-76 with x1..xn
 * arrays).  xs[k] = component k of every row, head[N], body[k] = output component k
 * (unit or scaled; NULL for FN_OP_NORM), sq[N] for FN_OP_NORMALIZE_SQ.  Same arithmetic
 * as the AoS kernels, bit for bit.  Ops SCALE..NORMALIZE_SQ, both dtypes. */
int fn_run_soa(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head,
               void* const* body, void* sq, const double* ka, void* stream);
/* fn_run_soa for host component arrays: the host pipeline of fn_host_run (page-locked
 * arrays DMA'd directly, pageable ones staged by the parallel copier), synchronous. */
int fn_host_run_soa(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head,
                    void* const* body, void* sq, const double* ka);
/* Page-locked (portable) host memory for fn_host_run / fn_host_run_multi callers: buffers
 * from here are DMA'd directly instead of through the library's staging copies
 * (1.56 vs 0.64 Gvec/s for 3-D f64 rows).  No reference analogue (the reference is CPU
 * only).  fn_host_free(NULL) is a no-op. */
int fn_host_alloc(size_t bytes, void** ptr);
int fn_host_free(void* ptr);
/* 1 if ptr is page-locked host memory known to CUDA (fn_host_alloc, cudaHostAlloc,
 * cudaHostRegister, or the outputs the Python API allocates from its pool), else 0. */
int fn_host_is_page_locked(const void* ptr);
/* One row with the reference's scalar semantics, low latency: x[dim] as doubles (the f32
 * families round them to binary32 like the reference's <float> casts), results written
 * to out as doubles in the order head, body..., extra... (e.g. r, u1..un; inv, s1..sn;
 * r, u1..un, sq).  Uses a per-thread page-locked buffer mapped into the device; one
 * kernel launch and one stream synchronisation per call. */
int fn_scalar(int op, int dim, int dtype, const double* x, double* out, const double* ka);

/* fn_host_run over several devices of one process: rows are split into ndev contiguous
 * balanced shards, one host thread per device runs the pipelined host path on its
 * shard (no inter-device traffic; each device brings its own PCIe link). */
int fn_host_run_multi(int op, int dim, int dtype, const void* x, int64_t n, void* head,
                      void* body, void* sq, const double* ka, const int* devices, int ndev);
/* fn_host_run / fn_host_run_multi over host rows ldx elements apart (see fn_run_ld):
 * each chunk's records cross PCIe as they are (no host-side gather) and the device
 * kernel reads them with the same stride.  Outputs are dense host arrays. */
int fn_host_run_ld(int op, int dim, int dtype, const void* x, int64_t n, int64_t ldx, void* head,
                   void* body, void* sq, const double* ka);
int fn_host_run_multi_ld(int op, int dim, int dtype, const void* x, int64_t n, int64_t ldx,
                         void* head, void* body, void* sq, const double* ka, const int* devices,
                         int ndev);
/* fn_host_run_soa over several devices of one process, sharded like fn_host_run_multi
 * (every component and output array split at the same row boundaries). */
int fn_host_run_soa_multi(int op, int dim, int dtype, const void* const* xs, int64_t n, void* head,
                          void* const* body, void* sq, const double* ka, const int* devices, int ndev);
/* Kernels this library has launched so far, process-wide (all threads and devices; the
 * scalar path included).  Callers difference it around a region to count its launches. */
int64_t fn_launch_count(void);
/* Diagnostics: zero-copy contexts created so far for small host batches (each holds a
 * mapped page-locked buffer and a stream; they are pooled per device and reused). */
int64_t fn_small_contexts(void);
/* fn_run for the rotation ops, with a device counter (uint64, accumulated; may be NULL)
 * of rows the reference would reject. */
int fn_run_rot(int op, const double* q, int64_t n, double* head, double* body, double* extra,
               const double* ka, uint64_t* invalid, void* stream);

/* RotationMatrix.apply (rotation.py:39-41) for a batch: out[N,3] = R v[N,3], R[9]
 * row-major (same as fn_run(FN_OP_ROT_APPLY, 3, FN_F64, v, n, out, NULL, NULL, R, s)). */
int fn_rotate_apply_f64(const double R[9], const double* v, int64_t n, double* out, void* stream);

/* Per-row rotation of vectors (two input arrays, see FN_OP_QUAT_ROTATE / FN_OP_MAT_APPLY):
 * a, v, out on the device (async on stream), ka = the six double constants for
 * QUAT_ROTATE (ignored, may be NULL, for MAT_APPLY), invalid = device uint64 counter or
 * NULL.  The host variant takes host arrays and pipelines them like fn_host_run. */
int fn_rotate_rows_f64(int op, const double* a, const double* v, int64_t n, double* out,
                       const double* ka, uint64_t* invalid, void* stream);
int fn_host_rotate_rows_f64(int op, const double* a, const double* v, int64_t n, double* out,
                            const double* ka);

/* ---- named entry points: one per reference export --------------------------------- */
/* scale{n}_{f64,f32}      replaces _kernels.pyx:419-439 / :523-546 */
int fn_scale2_f64(const double* x, int64_t n, double* inv, double* scaled, const double ka[6], void* stream);
int fn_scale3_f64(const double* x, int64_t n, double* inv, double* scaled, const double ka[6], void* stream);
int fn_scale4_f64(const double* x, int64_t n, double* inv, double* scaled, const double ka[6], void* stream);
int fn_scale2_f32(const float* x, int64_t n, float* inv, float* scaled, const double ka[6], void* stream);
int fn_scale3_f32(const float* x, int64_t n, float* inv, float* scaled, const double ka[6], void* stream);
int fn_scale4_f32(const float* x, int64_t n, float* inv, float* scaled, const double ka[6], void* stream);

/* normalize{n}_{f64,f32}  replaces _kernels.pyx:442-463 / :549-573 */
int fn_normalize2_f64(const double* x, int64_t n, double* r, double* unit, const double ka[6], void* stream);
int fn_normalize3_f64(const double* x, int64_t n, double* r, double* unit, const double ka[6], void* stream);
int fn_normalize4_f64(const double* x, int64_t n, double* r, double* unit, const double ka[6], void* stream);
int fn_normalize2_f32(const float* x, int64_t n, float* r, float* unit, const double ka[6], void* stream);
int fn_normalize3_f32(const float* x, int64_t n, float* r, float* unit, const double ka[6], void* stream);
int fn_normalize4_f32(const float* x, int64_t n, float* r, float* unit, const double ka[6], void* stream);

/* normalize{n}_sq_{f64,f32}: normalize{n} plus the squared length (config 3). */
int fn_normalize2_sq_f64(const double* x, int64_t n, double* sq, double* r, double* unit, const double ka[6], void* stream);
int fn_normalize3_sq_f64(const double* x, int64_t n, double* sq, double* r, double* unit, const double ka[6], void* stream);
int fn_normalize4_sq_f64(const double* x, int64_t n, double* sq, double* r, double* unit, const double ka[6], void* stream);
int fn_normalize2_sq_f32(const float* x, int64_t n, float* sq, float* r, float* unit, const double ka[6], void* stream);
int fn_normalize3_sq_f32(const float* x, int64_t n, float* sq, float* r, float* unit, const double ka[6], void* stream);
int fn_normalize4_sq_f32(const float* x, int64_t n, float* sq, float* r, float* unit, const double ka[6], void* stream);

/* norm{n}_{f64,f32}       replaces _kernels.pyx:466-478 / :576-592 */
int fn_norm2_f64(const double* x, int64_t n, double* r, const double ka[6], void* stream);
int fn_norm3_f64(const double* x, int64_t n, double* r, const double ka[6], void* stream);
int fn_norm4_f64(const double* x, int64_t n, double* r, const double ka[6], void* stream);
int fn_norm2_f32(const float* x, int64_t n, float* r, const double ka[6], void* stream);
int fn_norm3_f32(const float* x, int64_t n, float* r, const double ka[6], void* stream);
int fn_norm4_f32(const float* x, int64_t n, float* r, const double ka[6], void* stream);

/* naive{n}_{f64,f32}      replaces _kernels.pyx:481-496 / :595-610 */
int fn_naive2_f64(const double* x, int64_t n, double* r, double* unit, void* stream);
int fn_naive3_f64(const double* x, int64_t n, double* r, double* unit, void* stream);
int fn_naive4_f64(const double* x, int64_t n, double* r, double* unit, void* stream);
int fn_naive2_f32(const float* x, int64_t n, float* r, float* unit, void* stream);
int fn_naive3_f32(const float* x, int64_t n, float* r, float* unit, void* stream);
int fn_naive4_f32(const float* x, int64_t n, float* r, float* unit, void* stream);

/* quotient{n}_{f64,f32}   replaces _kernels.pyx:499-514 / :613-628 */
int fn_quotient2_f64(const double* x, int64_t n, double* r, double* unit, void* stream);
int fn_quotient3_f64(const double* x, int64_t n, double* r, double* unit, void* stream);
int fn_quotient4_f64(const double* x, int64_t n, double* r, double* unit, void* stream);
int fn_quotient2_f32(const float* x, int64_t n, float* r, float* unit, void* stream);
int fn_quotient3_f32(const float* x, int64_t n, float* r, float* unit, void* stream);
int fn_quotient4_f32(const float* x, int64_t n, float* r, float* unit, void* stream);

/* quotient3_fast_{f64,f32} replaces _kernels.pyx:517-520 / :631-634 */
int fn_quotient3_fast_f64(const double* x, int64_t n, double* r, double* unit, void* stream);
int fn_quotient3_fast_f32(const float* x, int64_t n, float* r, float* unit, void* stream);

/* ---- row statistics (validation counters for the multi-GPU driver) ---------------- */
/* Counts, over rows [0, n): [0] rows with a NaN component, [1] rows with an infinite
 * component and no NaN, [2] all-zero rows, [3] rows whose max |x_k| is below tau_min,
 * [4] rows whose max |x_k| is above tau_max (finite), [5] rows inside the band.
 * `counts` is a device array of 6 uint64 that is ACCUMULATED into (zero it first). */
int fn_row_stats(int dim, int dtype, const void* x, int64_t n, uint64_t* counts,
                 const double* ka, void* stream);

/* ---- seeded synthetic workloads (BASELINE.json configs) ------------- */
/* Writes rows [row0, row0+n) of workload `cfg` (1..5) into device array x.  Rows are a
 * pure function of (cfg, seed, global row index), so any sharding produces identical
 * data.  dim/dtype must match the config (1: 3/f64, 2: 2/f64, 3: 4/f64, 4: 3/f32,
 * 5: 3/f64). */
int fn_generate(int cfg, uint64_t seed, int64_t row0, int64_t n, void* x, void* stream);

/* The reference harness's input regimes (pkg/src/fastnorm/bench.py:146-207):
 * 0 normal, 1 subnormal, 2 huge, 3 mixed, 4 unit-ish; rows [row0, row0+n) of an
 * [*, dim] array of dtype, a pure function of (regime, dim, dtype, seed, row). */
int fn_generate_regime(int regime, int dim, int dtype, uint64_t seed, int64_t row0, int64_t n,
                       void* x, void* stream);

/* ---- error-bound sweep (reference oracle.py:151-250, in double-double) ----------- */
/* For rows x[N,dim] with computed r[N], unit[N,dim] (device arrays of dtype), checks the
 * paper's bounds for the scaling algorithm.  limits = {u, alpha, nu, omega} of the format.
 * counts[12] (accumulated): nan-output, nonzero-length, finite-unit, sin-phi, direction,
 *   finite-length, length-in-range, length-near-underflow, quaternion-product,
 *   rows measured (finite nonzero input), rows skipped, rows with any violation.
 * maxbits[4] (atomicMax on the bit patterns; zero them first): max relative length
 *   error, max absolute length error, max direction error, max sin(phi).
 * argmax[5]: row index of each maximum (best effort), argmax[4] = first violating row
 *   (atomicMin; initialise to UINT64_MAX). */
int fn_measure_bounds(int dim, int dtype, const void* x, const void* r, const void* unit, int64_t n,
                      const double* limits, uint64_t* counts, uint64_t* maxbits, uint64_t* argmax,
                      void* stream);

/* ---- device self-test of the shared-divisor division (fastnorm_math.cuh) ----------- */
/* Compares the kernels' correctly-rounded division against the CUDA math library's
 * IEEE division on n generated operand pairs (full range, mantissa / exponent edge
 * cases, specials).  out: device array of 3 uint64 (zero it first) -> [0] mismatches,
 * [1], [2] bit patterns of the first mismatching numerator / divisor. */
int fn_selftest_div(int dtype, uint64_t seed, int64_t n, uint64_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FASTNORM_B200_H */
