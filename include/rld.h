/*
 * rld.h -- C ABI of the B200-native rational log-determinant estimator.
 *
 * This is the drop-in boundary for the reference package `ratlogdet`'s r* path
 * (arXiv 2405.03474, Algorithm 1).  Every entry point below names the
 * reference interface it replaces (paths relative to
 * /root/reference/pkg/src/ratlogdet/).  Plain C types only: pointers, sizes,
 * enums, POD structs.  No torch or numpy types cross this line.
 *
 * Conventions
 *  - "rows" layout everywhere, as in the reference: a block of m vectors of
 *    length n is an m x n row-major array (probes s x n, src/probes.py:26;
 *    sketch w x n, src/precond.py:183).
 *  - Every call is synchronous with respect to the host: it returns after its
 *    device work finished and its outputs are visible at the given pointers.
 *  - A handle is not thread-safe; distinct handles are independent.
 *  - Results are deterministic for a fixed device count: every reduction has
 *    a fixed order (no floating-point atomics).
 *  - Status codes map one-to-one onto the reference's exception types
 *    (src/linalg.py:24-33, ValueError for argument errors); the message of the
 *    last failure on a handle is available from rld_last_error().
 */
#ifndef RLD_H
#define RLD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLD_ABI_VERSION 4

typedef enum rld_status {
  RLD_OK = 0,
  RLD_ERR_INVALID_ARGUMENT = 1,        /* ValueError (src/estimators.py:41-45, src/precond.py:241-242) */
  RLD_ERR_NOT_POSITIVE_DEFINITE = 2,   /* NotPositiveDefinite (src/linalg.py:24-25, 113-116) */
  RLD_ERR_SINGULAR_SHIFTED_SYSTEM = 3, /* SingularShiftedSystem (src/linalg.py:140-148) */
  RLD_ERR_RANK_DEFICIENT = 4,          /* RankDeficient after the retry (src/precond.py:181-197) */
  RLD_ERR_CUDA = 5,
  RLD_ERR_NCCL = 6,
  RLD_ERR_OUT_OF_MEMORY = 7,
  RLD_ERR_NOT_SUPPORTED = 8
} rld_status;

typedef enum rld_dtype { RLD_FP64 = 0, RLD_FP32 = 1 } rld_dtype;
typedef enum rld_family { RLD_RBF = 0, RLD_MATERN52 = 1 } rld_family; /* src/kernels.py:17-30 */
typedef enum rld_source { RLD_SOURCE_DENSE = 0, RLD_SOURCE_POINTS = 1 } rld_source;
typedef enum rld_path { RLD_PATH_STORED = 0, RLD_PATH_ON_THE_FLY = 1 } rld_path;
typedef enum rld_memory { RLD_HOST = 0, RLD_DEVICE = 1 } rld_memory;
typedef enum rld_probe_kind {   /* src/probes.py:12 */
  RLD_RADEMACHER = 0,
  RLD_GAUSSIAN = 1,
  RLD_NORMAL_ORTHOGONAL = 2   /* orthonormalised Gaussian blocks scaled by chi(n) radii, src/probes.py:15-22 */
} rld_probe_kind;
#define RLD_MAX_PROBE_BLOCKS 4  /* normal-orthogonal: s <= 4 n */
typedef enum rld_precond_kind {  /* the nine kinds of src/precond.py:25-35 */
  RLD_PRECOND_RAND_SVD = 0,                /* randomized truncated SVD, src/precond.py:262-267 (the r* default) */
  RLD_PRECOND_IDENTITY = 1,                /* src/precond.py:245-246 */
  RLD_PRECOND_DIAGONAL = 2,                /* src/precond.py:247-248 */
  RLD_PRECOND_RAND_SVD_SCALED = 3,         /* rand-svd low rank, base = scale, src/precond.py:265-266 */
  RLD_PRECOND_PARTIAL_CHOLESKY = 4,        /* pivoted partial Cholesky, src/precond.py:215-228, 253-258 */
  RLD_PRECOND_PARTIAL_CHOLESKY_SCALED = 5, /* src/precond.py:259 */
  RLD_PRECOND_TRUNC_SVD = 6,               /* dense eigh of K (one GPU), src/precond.py:260-263 */
  RLD_PRECOND_TRUNC_SVD_SCALED = 7,
  RLD_PRECOND_RANK_ONE = 8                 /* power iteration, src/precond.py:201-213, 249-251 */
} rld_precond_kind;

/* The stochastic estimators of src/estimators.py behind rld_logdet. */
typedef enum rld_estimator {
  RLD_ESTIMATOR_RSTAR = 0, /* rstar_logdet r1/r3/r5 (src/estimators.py:77-96) */
  RLD_ESTIMATOR_SLQ = 1    /* slq_logdet: Lanczos on K itself with full reorthogonalisation, no
                              preconditioner, Gauss quadrature of log (src/estimators.py:99-122) */
} rld_estimator;

typedef struct rld_handle rld_handle;
typedef struct rld_vgroup rld_vgroup;   /* "virtual shards": G ranks of one process (rld_vgroup_create) */

typedef enum rld_comm_kind {
  RLD_COMM_NCCL = 0,     /* one process (or thread) per GPU, NCCL over NVLink / NVSwitch */
  RLD_COMM_THREADS = 1   /* G handles of one process, one host thread each, host-barrier exchange
                            through device staging slots: runs the row-sharded path on one GPU */
} rld_comm_kind;

/* `world_size` ranks row-shard K; world_size 1 = single GPU, no collectives. */
typedef struct rld_device_set {
  int32_t device;       /* CUDA ordinal */
  int32_t rank;         /* row-shard index, 0 <= rank < world_size */
  int32_t world_size;   /* 1 = single GPU (no NCCL) */
  int32_t comm_kind;    /* rld_comm_kind (was `reserved`, 0 = NCCL) */
  const void* nccl_id;  /* RLD_COMM_NCCL: 128-byte ncclUniqueId shared by all ranks (NULL if world_size == 1) */
  rld_vgroup* group;    /* RLD_COMM_THREADS: the group every rank's handle joins */
} rld_device_set;

/* The matrix: a dense K (the reference's only input, src/estimators.py:77) or the
 * points + kernel it is built from (src/kernels.py:59, src/bench.py:105-109). */
typedef struct rld_problem {
  int32_t source;        /* rld_source */
  int32_t path;          /* rld_path (points source): build K in HBM or generate tiles per product */
  int32_t dtype;         /* rld_dtype: storage and product arithmetic of K */
  int32_t family;        /* rld_family */
  int64_t n;             /* order of K */
  int32_t d;             /* point dimension */
  int32_t data_memory;   /* rld_memory of `data` */
  double amplitude;      /* K = amplitude^2 k(r) + jitter I  (src/kernels.py:41, 72) */
  double length_scale;
  double jitter;
  const void* data;      /* dense: K rows (n x ld, data_dtype); points: n x d float64 row-major */
  int32_t data_dtype;    /* rld_dtype of a dense `data` */
  int32_t reserved;
  int64_t ld;            /* row stride of dense K in elements (0 -> n) */
} rld_problem;

/* EstimatorConfig + PreconditionerConfig (src/estimators.py:32-45, src/precond.py:40-55). */
typedef struct rld_config {
  int32_t order;          /* 1, 3 or 5 (algorithm r1/r3/r5) */
  int32_t num_probes;     /* s */
  int32_t lanczos_iters;  /* t, clamped to n as in src/estimators.py:62 */
  int32_t probe_kind;     /* rld_probe_kind */
  int32_t precond_kind;   /* rld_precond_kind */
  int32_t precond_rank;   /* l (k) */
  int32_t precond_iters;  /* q */
  int32_t oversample;     /* 10 (src/precond.py:165) */
  double diag_floor;      /* 1e-12 (src/precond.py:37) */
  double keep_rtol;       /* 1e-14 (src/precond.py:97) */
  double breakdown_rtol;  /* 1e-12 (src/lanczos.py:20) */
  double orth_rtol;       /* 1e-12 (src/linalg.py:177) */
  uint64_t probe_key[2];  /* Philox4x64 key of numpy stream (seed, (2,))      -- src/estimators.py:64 */
  uint64_t omega_key[4];  /* keys of streams (seed,(1,0)) and (seed,(1,1))    -- src/precond.py:183 */
  int32_t estimator;      /* rld_estimator: r* (order above) or SLQ (src/estimators.py:99-122) */
  int32_t reserved2;
  double precond_scale;   /* base scalar a of the "-scaled" kinds (PreconditionerConfig.scale, src/precond.py:45) */
  uint64_t precond_key[2];/* Philox key of stream (seed, (1,)): the rank-one power-iteration start (src/precond.py:202) */
  uint64_t probe_block_keys[2 * RLD_MAX_PROBE_BLOCKS]; /* normal-orthogonal: keys of streams (seed, (2, i)) */
} rld_config;

/* Optional injected random inputs.  NULL -> generated on the device from the
 * Philox keys in rld_config, reproducing numpy's streams: Rademacher probes
 * bit-identically, Gaussian rows (sketch, Gaussian probes) with numpy's
 * ziggurat (rld_normal). */
typedef struct rld_inputs {
  const double* probes;   /* s x n */
  const double* omega0;   /* w x n, attempt 0 */
  const double* omega1;   /* w x n, attempt 1 (only read after a RankDeficient retry) */
  int32_t memory;         /* rld_memory of the three pointers */
  int32_t reserved;
} rld_inputs;

/* LogDetEstimate (src/estimators.py:48-55) plus device-side diagnostics. */
typedef struct rld_result {
  double value;
  double logdet_P;
  double trace_term;
  double* per_probe;      /* caller-allocated host array of num_probes doubles */
  double wall_time;       /* seconds, CUDA events around the estimate */
  int32_t attempts;       /* sketch attempts used (1 or 2) */
  int32_t rank_kept;      /* columns of U kept by the 1e-14 filter (src/precond.py:97) */
  int32_t kv_products;    /* K x block products issued */
  int32_t kernel_launches;/* own kernels launched by the estimate */
  double phase_ms[8];     /* [0] K build [1] sketch+QR [2] projected eig [3] precond factors
                             [4] Lanczos [5] shifted solves + Hutchinson [6] collectives [7] total */
  int32_t clamped_eigs;   /* SLQ: Ritz values <= 0 floored before the log (src/estimators.py:113-115) */
  int32_t qr_fallback;    /* rand-svd: 1 when an ill-conditioned sketch sent the QR to Householder / TSQR */
} rld_result;

int rld_abi_version(void);

/* Fill `out` (128 bytes) with a fresh ncclUniqueId; rank 0 calls it and
 * broadcasts the bytes to the other ranks before rld_create. */
int rld_nccl_unique_id(void* out);

/* Bind a handle to one GPU (and, for world_size > 1, to an NCCL communicator). */
int rld_create(const rld_device_set* devices, rld_handle** out);
/* Virtual-shard group for RLD_COMM_THREADS: create once, pass to every rank's rld_create, destroy
 * after every handle of the group is destroyed.  No reference counterpart (the reference has no
 * parallel path); test / single-GPU plumbing of the row-sharded estimate. */
int rld_vgroup_create(int32_t world_size, rld_vgroup** out);
void rld_vgroup_destroy(rld_vgroup* group);
void rld_destroy(rld_handle* h);
const char* rld_last_error(const rld_handle* h);

/* The cudaStream_t (as void*) the handle orders all its work on, so callers can
 * record timing events or chain their own work on the same stream. */
void* rld_stream(rld_handle* h);

/* rstar_logdet(M, cfg) -- src/estimators.py:77-96 -- or, with
 * cfg->estimator == RLD_ESTIMATOR_SLQ, slq_logdet(M, cfg) -- src/estimators.py:99-122
 * (estimate_logdet for r1/r3/r5/slq, src/estimators.py:132-138).  Uploads / builds K, runs the
 * preconditioner build, s-probe Lanczos, multishift solves and the Hutchinson
 * mean on the device, and fills `result`. */
int rld_logdet(rld_handle* h, const rld_problem* problem, const rld_config* cfg,
               const rld_inputs* inputs, rld_result* result);

/* Make `problem` resident in the handle (upload points / build or copy K into
 * HBM) so rld_logdet_resident can be called repeatedly without host traffic. */
int rld_prepare(rld_handle* h, const rld_problem* problem);
int rld_logdet_resident(rld_handle* h, const rld_config* cfg, const rld_inputs* inputs,
                        rld_result* result);

/* build_covariance(spec, points) -- src/kernels.py:59-73: write the dense K
 * (n x n, dtype = problem->dtype) to `out` (host or device per out_memory). */
int rld_build_covariance(rld_handle* h, const rld_problem* problem, void* out, int32_t out_memory);

/* The operator seam `M @ x` of src/estimators.py:72 for a block: Y = V K for the
 * m x n rows V (device, float64), using the resident problem and its product
 * arithmetic.  Y (device, float64) is m x n on one GPU; with world_size > 1 it
 * is this rank's row shard, m x rows (rows of K this rank holds, see
 * rld_prepare).  Stream-ordered: enqueued on rld_stream(h), not synchronised. */
int rld_kv_apply(rld_handle* h, int64_t m, const double* V, double* Y);

/* build_preconditioner(M, cfg, rng) on its own (src/precond.py:236-267) for the resident problem:
 * the preconditioner fields of `cfg` (kind, rank, num_iters, scale, diag_floor, keep_rtol,
 * omega_key / precond_key streams; the estimator fields are ignored).  The factors stay in the
 * handle (until the next prepare or estimate) for rld_precond_apply.  Errors as rld_logdet. */
typedef struct rld_precond_info {
  double log_det;          /* log det P (src/precond.py:69-80) */
  int32_t rank;            /* columns of the low-rank factor A (k; < rank when partial Cholesky runs out) */
  int32_t rank_kept;       /* columns of U kept by the 1e-14 filter (src/precond.py:97) */
  int32_t attempts;        /* sketch attempts (rand-svd: 2 after a RankDeficient retry) */
  int32_t qr_fallback;     /* 1 when the sketch QR fell back to Householder / TSQR */
  int32_t kernel_launches;
  int32_t reserved;
} rld_precond_info;
int rld_precond_build(rld_handle* h, const rld_config* cfg, const rld_inputs* inputs, rld_precond_info* info);

typedef enum rld_precond_op {
  RLD_SOLVE_SQRT = 0,    /* N^-1 z   (Preconditioner.solve_sqrt,   src/precond.py:102-108) */
  RLD_SOLVE_SQRT_T = 1,  /* N^-T x   (Preconditioner.solve_sqrt_t, src/precond.py:110-115) */
  RLD_SOLVE = 2          /* P^-1 u = N^-T N^-1 u */
} rld_precond_op;
/* Y = op(V) for m rows V (m x n float64, device) with the last preconditioner build; one GPU.
 * Stream-ordered on rld_stream(h) and synchronised before returning. */
int rld_precond_apply(rld_handle* h, int32_t op, int64_t m, const double* V, double* Y);

/* Rng(seed).child(...).rademacher((rows, n)) -- src/linalg.py:84-85, on the
 * device from the stream's Philox key; `out` is device float64, rows x n. */
int rld_rademacher(rld_handle* h, const uint64_t key[2], int64_t rows, int64_t n, double* out);

/* Rng(...).normal((rows, n)) -- src/linalg.py:81-82: numpy's Generator.standard_normal
 * (256-layer ziggurat over Philox4x64) reproduced on the device from the stream's key;
 * `out` is device float64, rows x n. */
int rld_normal(rld_handle* h, const uint64_t key[2], int64_t rows, int64_t n, double* out);

/* Rng.chi(df, count) -- src/linalg.py:87-88 (sqrt of numpy's Generator.chisquare) -- drawn on the
 * host from the numpy Philox stream `key` starting at 64-bit word `word0`: the continuation of the
 * stream after Gaussian rows the device generated (normal-orthogonal probes, src/probes.py:15-22).
 * Host only; needs no GPU. */
int rld_chi_radii(const uint64_t key[2], uint64_t word0, int64_t df, int64_t count, double* out);

/* The dense Cholesky the preconditioner build uses (CholQR's w x w Gram, src/linalg.py:159-180
 * restated; the k x k inner factor, src/precond.py:75-80): G = R^T R in place on the n x n
 * column-major float64 device matrix G (upper triangle read and overwritten with R).  *info
 * (host) = 0, or the 1-based index of the first non-positive pivot as LAPACK's potrf.
 * Synchronous. */
int rld_dense_cholesky(rld_handle* h, int32_t n, double* G, int32_t* info);

/* The symmetric eigensolver of the preconditioner build (eigh of B, src/precond.py:189-190, and of
 * At^T At, src/precond.py:96) on the n x n column-major float64 device matrix A (positive
 * semi-definite): eigenvalues ascending into w (device, n), eigenvectors over A (column j <-> w[j],
 * signs arbitrary as LAPACK's).  Synchronous. */
int rld_dense_eigh(rld_handle* h, int32_t n, double* A, double* w);

/* exact_logdet(M) -- src/estimators.py:125-129: Cholesky log det of the
 * resident problem's K in float64 on the device. */
int rld_exact_logdet(rld_handle* h, double* value);

/* Work of the int8-slice product on the resident K (no reference counterpart: the measurement
 * hook of bench.py's roofline).  stats[0..3] = the 128 x 32 blocks of the slice image, the K slices
 * a product reads over them (of 7 per block for a float64 K, 3 for a float32 K from Morton-ordered
 * points; leading all-zero slices are skipped), the slice pairs it multiplies (s + t <= 6 of 7 x 7,
 * or s + t <= 3 of 3 x 4), and 1 if the wide (sketch) products run on the CRT residue image
 * instead.  All 0 when the resident K has no slice image. */
int rld_slice_stats(rld_handle* h, int64_t* stats);

#ifdef __cplusplus
}
#endif

#endif /* RLD_H */
