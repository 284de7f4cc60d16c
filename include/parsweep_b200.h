/*
 * parsweep_b200 — C ABI of the B200-native batched dichotomy tridiagonal
 * solver (Terekhov, arXiv:0901.2859). Drop-in for the hot path of the
 * reference `parsweep` library: one-time setup on the matrix, then the
 * batched solve of A X_k = F_k for many right-hand sides.
 *
 * Plain pointers and sizes only; no CUDA, torch or C++ types cross this
 * boundary (streams are passed as `void*` = cudaStream_t). Reference paths
 * below are relative to parsweep/ in the reference tree
 * (proj/include/parsweep/). Every call is thread-safe; a plan is immutable
 * after creation and may be used concurrently from several streams.
 *
 * Storage layouts of the right-hand-side / solution series (N systems of
 * order n, element (row i, rhs k), 0-based):
 *   PSW_LAYOUT_R  "RHS-contiguous":    F[i * ld + k], ld >= N
 *   PSW_LAYOUT_S  "system-contiguous": F[k * ld + i], ld >= n   (the reference's
 *                 own layout: each std::vector<double> is one system,
 *                 dichotomy/batch.hpp:57-60)
 */
#ifndef PARSWEEP_B200_H
#define PARSWEEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSW_ABI_VERSION 4

/* Status codes. The C++ wrapper (parsweep_b200.hpp) maps them back onto the
 * reference exception types of core/errors.hpp:9-62. */
typedef enum psw_status {
    PSW_OK = 0,
    PSW_INVALID_ARGUMENT = 1, /* std::invalid_argument: tridiag.hpp:57-66, partition.hpp:31-42 */
    PSW_PIVOT_BREAKDOWN = 2,  /* PivotBreakdown(row): thomas.hpp:14,32,38; row in last_error_index */
    PSW_TOO_MANY_PES = 3,     /* TooManyPEs: decompose.hpp:34-35 */
    PSW_NOT_SUPPORTED = 4,    /* e.g. non-symmetric A (Symmetrize route, preliminary.hpp:111-132) */
    PSW_CUDA_ERROR = 5,
    PSW_NCCL_ERROR = 6,
    PSW_OUT_OF_MEMORY = 7,
    PSW_NOT_SYMMETRIZABLE = 8,       /* NotSymmetrizable(k): errors.hpp:29-38; k in last_error_index */
    PSW_ORACLE_FALLBACK_REQUIRED = 9 /* OracleFallbackRequired: errors.hpp:40-43 */
} psw_status;

/* GRowStrategy (dichotomy/preliminary.hpp:18-24): how the inverse-matrix
 * rows of the setup are obtained. AUTO picks DIRECT_SYMMETRIC for
 * sub == super, otherwise SYMMETRIZE with the reference's automatic
 * fallbacks to EXPLICIT_INVERSE and TRANSPOSE_SOLVE (preliminary.hpp:111-132). */
typedef enum psw_grow_strategy {
    PSW_GROW_AUTO = 0,
    PSW_GROW_DIRECT_SYMMETRIC = 1,
    PSW_GROW_SYMMETRIZE = 2,
    PSW_GROW_EXPLICIT_INVERSE = 3,
    PSW_GROW_TRANSPOSE_SOLVE = 4
} psw_grow_strategy;

typedef enum psw_dtype { PSW_F64 = 0, PSW_F32 = 1 } psw_dtype;
typedef enum psw_layout { PSW_LAYOUT_R = 0, PSW_LAYOUT_S = 1 } psw_layout;

/* Solve-path selection (psw_solve_ex). AUTO picks the fastest path that
 * supports the plan/shape: CLUSTER and FUSED keep every RHS tile resident on
 * chip and read F once (layout R, uniform partitions whose blocks fit a
 * cluster; CLUSTER: one CTA per SM holding G blocks, FUSED: 16-CTA clusters);
 * RESWEEP reads F twice from HBM and writes X once, with a few aggregates per
 * 256 rows in between (either layout, e.g. the 2^20-row config); STAGED is
 * the general three-kernel path (and the only one returning betas/boundary
 * values). */
typedef enum psw_path {
    PSW_PATH_AUTO = 0,
    PSW_PATH_STAGED = 1,
    PSW_PATH_FUSED = 2,
    /* 3, 4, 5, 8: retired paths (PSW_NOT_SUPPORTED) */
    PSW_PATH_CHUNKED = 5,
    PSW_PATH_RESWEEP = 6,
    PSW_PATH_CLUSTER = 7,
    PSW_PATH_HOLD = 8
} psw_path;

typedef struct psw_plan psw_plan;

/* Description of a created plan (psw_plan_info). */
typedef struct psw_plan_info_t {
    int64_t n;              /* order */
    int64_t p;              /* interior boundaries (partition.hpp:20), P = p + 1 blocks */
    int32_t dtype;          /* psw_dtype */
    int32_t device;         /* CUDA ordinal */
    int32_t uniform;        /* 1 if the partition is decompose(n, p+1).induced_partition() */
    int32_t fused_ok;       /* 1 if the fused on-chip path supports this plan (layout R) */
    int64_t device_bytes;   /* resident preliminary bytes in HBM */
    int64_t combine_terms;  /* WorkCounters::combine_terms of one RHS (boundary_solve.hpp:18-34) */
    int64_t comm_rounds;    /* RunStats::comm_rounds (run.hpp:93-94) */
    double setup_seconds;   /* host time of the preliminary phase */
    double max_z_norm;      /* PreliminaryData::max_z_norm (preliminary.hpp:75-83) */
    int32_t strategy_used;  /* psw_grow_strategy: PreliminaryData::strategy_used (:65) */
    int32_t device_setup;   /* 1 if the preliminary's boundary sweeps ran on the GPU (psw_prelim.cu) */
} psw_plan_info_t;

/* ---- errors ------------------------------------------------------------ */
/* Message and index (row for PIVOT_BREAKDOWN) of the last failing call on
 * the calling thread. */
const char* psw_last_error_message(void);
int64_t psw_last_error_index(void);
int psw_abi_version(void);

/* ---- partition helpers ------------------------------------------------ */
/* Replaces runtime/decompose.hpp:33-47 + Decomposition::induced_partition
 * (:23-29): writes the P-1 one-based interior boundaries of the near-equal
 * split of n rows into P ranges. PSW_TOO_MANY_PES if n < 2P. */
int psw_decompose(int64_t n, int64_t P, int64_t* boundaries_out);

/* Replaces Partition::validate (dichotomy/partition.hpp:31-42). */
int psw_partition_validate(int64_t n, int64_t p, const int64_t* boundaries);

/* ---- setup ------------------------------------------------------------ */
/* Replaces compute_preliminary(A, part, GRowStrategy::Auto, exec)
 * (dichotomy/preliminary.hpp:171-199). `sub`/`sup` hold n-1
 * entries (a_2..a_n / c_1..c_{n-1}), `diag` n entries, all host fp64 (the
 * reference's TridiagMatrix, tridiag.hpp:31-34). `boundaries` are the p
 * one-based interior rows of the reference `Partition` (partition.hpp:16-18).
 * The preliminary is computed in fp64 on the host, reduced to what the
 * per-RHS kernels read, and uploaded to `device` (dtype = PSW_F64 or
 * PSW_F32 for the solve arithmetic). Fails with PSW_PIVOT_BREAKDOWN exactly
 * where the reference's preliminary would throw. */
int psw_plan_create(psw_plan** out, int64_t n, const double* sub, const double* diag,
                    const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                    int device);
/* compute_preliminary(A, part, strategy) (preliminary.hpp:171-173) with an
 * explicit psw_grow_strategy. An explicit strategy that cannot be applied
 * fails like the reference: PSW_NOT_SYMMETRIZABLE (index k) for SYMMETRIZE,
 * PSW_ORACLE_FALLBACK_REQUIRED for EXPLICIT_INVERSE (core/inverse_rows.hpp:46-80). */
int psw_plan_create_ex(psw_plan** out, int64_t n, const double* sub, const double* diag,
                       const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                       int device, int strategy);
/* psw_plan_create_ex with flags: PSW_PLAN_STAGED_ONLY builds only what the
 * STAGED path and the multi-matrix solve read (no segment tables): plan setup
 * for many small systems, e.g. one plan per Fourier harmonic. */
#define PSW_PLAN_STAGED_ONLY 1
int psw_plan_create_flags(psw_plan** out, int64_t n, const double* sub, const double* diag,
                          const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                          int device, int strategy, int flags);
int psw_plan_destroy(psw_plan* plan);
int psw_plan_info(const psw_plan* plan, psw_plan_info_t* info);

/* ---- multi-matrix batched solve ---------------------------------------- */
/* Replaces the per-harmonic loop of fourier_solve (poisson/fourier.hpp:157-164)
 * over FourierWorkspace::solve_harmonic (:75-86): column k of the layout-R
 * series F (device, k < nplans, row pitch ldf) is solved with plans[k] into
 * column k of X, all columns in one pass (the STAGED kernels with per-column
 * plan tables; betas and boundary values bitwise the reference's). The plans
 * must share the order, the partition, the dtype and the device. */
int psw_solve_multi(const psw_plan* const* plans, int64_t nplans, const void* F, int64_t ldf,
                    void* X, int64_t ldx, void* stream);
/* The same solve for repeated use (one FourierWorkspace, many right-hand
 * sides): psw_multi_create gathers the plans' sweep tables once into
 * RHS-interleaved device arrays (coalesced loads) and keeps the Z-sample
 * table on the device; psw_multi_solve is then asynchronous on `stream`
 * (no host copies). The plans must outlive the bundle. */
typedef struct psw_multi psw_multi;
int psw_multi_create(psw_multi** out, const psw_plan* const* plans, int64_t nplans);
/* The same bundle for nsys symmetric systems (sub == super) sharing one
 * partition, set up on the device in one pass (every system's preliminary,
 * dichotomy/preliminary.hpp:171-199, and block sweep coefficients) instead of
 * one plan per system: FourierWorkspace's per-harmonic plan list
 * (poisson/fourier.hpp:41-105). Host arrays sub[nsys][n-1], diag[nsys][n],
 * super[nsys][n-1]. Tables bitwise those of psw_multi_create over per-system
 * plans. PSW_NOT_SUPPORTED for non-symmetric input or batches beyond 32 GB of
 * device scratch (create plans one by one then). */
int psw_multi_create_systems(psw_multi** out, int64_t n, int64_t nsys, const double* sub,
                             const double* diag, const double* super, int64_t p,
                             const int64_t* boundaries, int dtype, int device);
void psw_multi_destroy(psw_multi* multi);
int psw_multi_solve(const psw_multi* multi, const void* F, int64_t ldf, void* X, int64_t ldx,
                    void* stream);

/* ---- batched solve ---------------------------------------------------- */
/* Replaces the per-RHS loop of solve_batch (dichotomy/batch.hpp:67-73) over
 * solve_with_preliminary_into (batch.hpp:20-51): solves all `nrhs` systems
 * whose right-hand sides are in F (device memory, plan dtype) and writes the
 * solutions to X (device). Asynchronous on `stream` (cudaStream_t, NULL =
 * legacy default stream). F == X with ldf == ldx is allowed (in place). */
int psw_solve(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
              int64_t nrhs, int layout, void* stream);

/* Extended solve: explicit path, and optional device outputs of the
 * per-RHS intermediates for parity checks — betas_left/right ((p+1) x nrhs,
 * fp64, [t * nrhs + k], as BetaSet betas.hpp:20-23) and boundary values
 * (p x nrhs, fp64, [j * nrhs + k], as solve_boundaries boundary_solve.hpp:96).
 * Intermediates are only produced by the STAGED path. */
typedef struct psw_solve_opts {
    int32_t path;            /* psw_path */
    int32_t nevents;         /* entries in `events` (0 = none) */
    double* betas_left;      /* device, optional */
    double* betas_right;     /* device, optional */
    double* boundary_values; /* device, optional */
    void** events;           /* optional cudaEvent_t[nevents]: events[i] is recorded on the
                                stream before kernel i of the path and events[L] after the
                                last of its L kernels (per-kernel timing, bench.py) */
} psw_solve_opts;
int psw_solve_ex(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                 int64_t nrhs, int layout, void* stream, const psw_solve_opts* opts);

/* End-to-end variant of solve_batch (batch.hpp:57-75) on HOST buffers: the
 * series is copied to the device in RHS chunks, solved and copied back, with
 * copies of chunk c+1 / c-1 overlapping the solve of chunk c. Blocking.
 * Pinned host memory gives full PCIe/C2C bandwidth. */
int psw_solve_host(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                   int64_t nrhs, int layout);

/* Device kernels launched by the last successful psw_solve* on this thread
 * (launch accounting for the benchmark). */
int64_t psw_last_launch_count(void);
/* ---- ADI consumer (poisson/adi.hpp) ----------------
 * Peaceman-Rachford half-step right-hand sides on the reference's Grid2D
 * layout ((n1+1) x (n2+1) fp64 nodes, row-major, j contiguous, zero
 * boundary), device pointers, stream-ordered:
 *   dir 1: rhs[(i-1)*ldr + (j-1)] = -h1^2 (u/tau + L2 u + f)   (adi.hpp:143-158)
 *          -> the direction-1 systems (along i) in layout R;
 *   dir 2: rhs[(i-1)*ldr + (j-1)] = -h2^2 (u/tau + L1 u + f)   (adi.hpp:160-175)
 *          -> the direction-2 systems (along j) in layout S.
 * Same operation order as the reference. The driver (AdiWorkspace /
 * AdiIteration / adi_solve) is paper_0901_2859_b200/adi.py. */
int psw_adi_rhs(int dir, const double* u, int64_t ldu, const double* f, int64_t ldf, double* rhs,
                int64_t ldr, int64_t n1, int64_t n2, double h1, double h2, double tau,
                void* stream);
/* out2[0] = max |a - b|, out2[1] = max |b| over rows x cols doubles with row
 * pitches lda / ldb (device pointers; max_abs_diff / max_abs of
 * poisson/grid2d.hpp:43-53). */
int psw_grid_max_abs_diff(const double* a, int64_t lda, const double* b, int64_t ldb,
                          int64_t rows, int64_t cols, double* out2, void* stream);

/* psw_path taken by the last psw_solve/psw_solve_ex on this thread (0 before any). */
int psw_last_path(void);

/* ---- multi-GPU row sharding (dichotomy across devices) ---------------- */
/* The reference simulates message passing (runtime/run.hpp:30-35,93-94) with
 * logical PEs; here the PEs are GPUs, one process (or thread) per GPU. Rank r
 * of `world` owns the blocks [r*P/world, (r+1)*P/world) of ONE global
 * partition (P = p+1 must be divisible by world) and the rows of those
 * blocks (the paper's data decomposition); F/X hold only
 * the owned rows, layout R (row offset psw_shard_row_offset, psw_shard_rows
 * rows). The dichotomy combination (dichotomy/boundary_solve.hpp:96-121) is
 * linear in the betas, so each rank forms its share of every boundary value
 * and the solve's only exchange is one all-reduce(sum) of p x nrhs fp64.
 *
 *   psw_shard_solve     forward sweep + betas + the rank's share of the p
 *                       boundary values, ncclAllReduce over `comm`, back
 *                       substitution: all on `stream`, CUDA-graph capturable.
 *   psw_shard_forward / psw_shard_backward   the two halves around a caller-
 *                       run reduction of `partials` (p x nrhs fp64, [j*nrhs+k]);
 *                       `workspace` (psw_shard_workspace_bytes) carries the
 *                       per-run aggregates from one to the other.
 * A shard plan is created by psw_shard_plan_create; psw_solve refuses it. */
int psw_shard_plan_create(psw_plan** out, int64_t n, const double* sub, const double* diag,
                          const double* sup, int64_t p, const int64_t* boundaries, int dtype,
                          int device, int rank, int world);
int64_t psw_shard_partials_count(const psw_plan* plan);
int64_t psw_shard_row_offset(const psw_plan* plan);
int64_t psw_shard_rows(const psw_plan* plan);
int64_t psw_shard_workspace_bytes(const psw_plan* plan, int64_t nrhs);
int psw_shard_forward(const psw_plan* plan, const void* F, int64_t ldf, int64_t nrhs,
                      void* workspace, double* partials, void* stream);
int psw_shard_backward(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                       int64_t nrhs, void* workspace, const double* partials, void* stream);

/* NCCL communicator of the row-sharded solve (NCCL is loaded at run time,
 * libnccl.so.2; PSW_NCCL_ERROR when it is absent or a call fails). Rank 0
 * creates the 128-byte unique id, every rank passes it to psw_comm_create
 * (collective over the `nranks` ranks, like ncclCommInitRank). */
typedef struct psw_comm psw_comm;
int psw_comm_unique_id(void* id_out /* 128 bytes */);
int psw_comm_create(psw_comm** out, int nranks, int rank, const void* id, int device);
int psw_comm_destroy(psw_comm* comm);
int psw_shard_solve(const psw_plan* plan, const void* F, int64_t ldf, void* X, int64_t ldx,
                    int64_t nrhs, psw_comm* comm, void* stream);

/* Host-only (no GPU needed): the p x 2P combination matrix of the partition
 * (row j = [MR[j][0..P) | ML[j][0..P)]), i.e. the action of solve_boundaries
 * (dichotomy/boundary_solve.hpp:96-121) on unit betas: boundary value
 * v_j = sum_t MR[j][t] right[t] + ML[j][t] left[t]. Used by the FUSED kernel
 * and the row-sharded exchange. */
int psw_combine_matrix(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* boundaries, double* out);

/* ---- utilities (benchmark / test data) -------------------------------- */
/* Fill a device buffer with the seeded counter-based uniform generator
 * u_i = (splitmix64(seed ^ (offset + i)) >> 11) * 2^-53, v = lo + (hi-lo) u
 * (SURVEY.md §8(d)); bitwise identical to the host generator for fp64. */
int psw_fill_uniform(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset,
                     double lo, double hi, void* stream);
/* Standard normal via Box-Muller on pairs of the same uniform stream. */
int psw_fill_normal(void* dst, int dtype, int64_t count, uint64_t seed, uint64_t offset,
                    void* stream);
/* Profiling aid: when `device_buffer` is non-NULL the FUSED kernel writes,
 * per CTA, 16 uint64 slots: clock64() at its phase boundaries (0..8) and
 * %globaltimer at start/end (14, 15). NULL disables tracing (default). */
int psw_debug_trace(void* device_buffer);

/* DST-I of `rows` rows (Fourier consumer; replaces poisson/dst.hpp:85-164
 * DstPlan::apply_raw / apply_raw_pair): out[r][l-1] = scale * sum_{j=1}^{N-1}
 * in[r][j-1] sin(pi j l / N), l = 1..N-1, fp64 device rows of pitch ldin /
 * ldout. Power-of-two N <= 4096: the reference's paired radix-2 FFT of the
 * odd extension (one CTA per pair of rows, shared memory); other N: the
 * direct sine sum (dst.hpp:120-128). Asynchronous on `stream`. */
int psw_dst_rows(const double* in, int64_t ldin, double* out, int64_t ldout, int64_t rows,
                 int64_t N, double scale, void* stream);

/* Write `bytes` of zeros+index pattern over a scratch buffer (L2 flush). */
int psw_l2_flush(void* scratch, int64_t bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PARSWEEP_B200_H */
