/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the parsweep hot path.
 *
 * This is the oracle the GPU product is checked against. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * The product library (paper_0901_2859_b200/csrc) never links or calls it.
 *
 * Every function restates one reference function (file:line relative to
 * /root/reference/proj/include/parsweep/). Rows are 0-based in storage;
 * partition boundaries are 1-based row indices exactly like the reference
 * `Partition` (dichotomy/partition.hpp:16-18).
 *
 * Parity pin: tests/test_oracle.py checks this restatement against the
 * reference's own known-answer tests (tests/test_core.cpp,
 * tests/test_dichotomy.cpp, tests/test_runtime.cpp) and bitwise against the
 * reference compiled from its sources (oracle/_ref, see oracle/Makefile),
 * through the committed fixtures in tests/golden/.
 */
#ifndef PSW_ORACLE_H
#define PSW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_INVALID_ARGUMENT = 1,
    ORC_PIVOT_BREAKDOWN = 2,
    ORC_TOO_MANY_PES = 3,
    ORC_NOT_SUPPORTED = 4,
    ORC_NO_MEMORY = 7,
    ORC_NOT_SYMMETRIZABLE = 8,  /* NotSymmetrizable(k), core/errors.hpp:29-38; k in *bad */
    ORC_ORACLE_FALLBACK = 9     /* OracleFallbackRequired, core/errors.hpp:40-43 */
};

/* GRowStrategy (dichotomy/preliminary.hpp:18-24) */
enum {
    ORC_GROW_AUTO = 0,
    ORC_GROW_DIRECT_SYMMETRIC = 1,
    ORC_GROW_SYMMETRIZE = 2,
    ORC_GROW_EXPLICIT_INVERSE = 3,
    ORC_GROW_TRANSPOSE_SOLVE = 4
};

/* core/thomas.hpp:14 */
#define ORC_PIVOT_FLOOR 1e-300

/* core/thomas.hpp:22-45. Returns ORC_OK or ORC_PIVOT_BREAKDOWN (row in *bad). */
int orc_thomas(int64_t n, const double* sub, const double* diag, const double* sup,
               const double* f, double* x, int64_t* bad);

/* runtime/decompose.hpp:33-47 followed by induced_partition() :23-29.
 * Writes P-1 1-based boundaries. */
int orc_decompose(int64_t n, int64_t P, int64_t* boundaries);

/* dichotomy/partition.hpp:31-42 */
int orc_partition_validate(int64_t n, int64_t p, const int64_t* boundaries);

/* dichotomy/level_sets.hpp:18-37. order[p] receives the 1-based positions in
 * level order; level_off[0..depth] the level offsets. Returns depth. */
int64_t orc_level_sets(int64_t p, int64_t* order, int64_t* level_off);

/* dichotomy/preliminary.hpp:171-199 with GRowStrategy Auto (:111-132).
 * g: p*n full inverse rows; zr_s/zl_s: p*p samples (:85-96);
 * max_z (optional): PreliminaryData::max_z_norm (:75-83). */
int orc_preliminary(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, double* g, double* zr_s, double* zl_s,
                    double* max_z, int64_t* bad);

/* Same with an explicit strategy (preliminary.hpp:108-164: Auto picks
 * DirectSymmetric for sub == super, else Symmetrize -> ExplicitInverse ->
 * TransposeSolve fallbacks; an explicit strategy that fails reports
 * ORC_NOT_SYMMETRIZABLE / ORC_ORACLE_FALLBACK). *used receives the
 * strategy actually used (PreliminaryData::strategy_used). */
int orc_preliminary_ex(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, int strategy, int* used, double* g,
                       double* zr_s, double* zl_s, double* max_z, int64_t* bad);

/* dichotomy/betas.hpp:34-59. left/right have p+1 entries. */
void orc_betas(int64_t n, int64_t p, const int64_t* bnd, const double* g, const double* f,
               double* left, double* right);

/* dichotomy/boundary_solve.hpp:96-121 (terms: WorkCounters::combine_terms). */
void orc_solve_boundaries(int64_t p, const double* zr_s, const double* zl_s,
                          const double* left, const double* right, double* value,
                          uint64_t* terms);

/* dichotomy/boundary_solve.hpp:126-136 (Theorem 2, O(p^2)). */
void orc_solve_boundaries_two_sided(int64_t p, const double* zr_s, const double* zl_s,
                                    const double* left, const double* right, double* value,
                                    uint64_t* terms);

/* dichotomy/local_solve.hpp:25-50. out has hi-lo+1 entries (closed block). */
int orc_solve_local(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, int64_t t, const double* f, int has_first,
                    double first_val, int has_last, double last_val, double* out, int64_t* bad);

/* dichotomy/batch.hpp:20-51. */
int orc_solve_with_preliminary(int64_t n, const double* sub, const double* diag,
                               const double* sup, int64_t p, const int64_t* bnd,
                               const double* g, const double* zr_s, const double* zl_s,
                               const double* f, double* out, uint64_t* terms, int64_t* bad);

/* dichotomy/batch.hpp:57-75, system-contiguous (layout S) series:
 * F[k*ldf + i], X[k*ldx + i]. Runs the preliminary once. */
int orc_solve_batch(int64_t n, const double* sub, const double* diag, const double* sup,
                    int64_t p, const int64_t* bnd, int64_t nrhs, const double* F, int64_t ldf,
                    double* X, int64_t ldx, int64_t* bad);

/* orc_solve_batch with an explicit GRowStrategy (batch.hpp:57-61). */
int orc_solve_batch_ex(int64_t n, const double* sub, const double* diag, const double* sup,
                       int64_t p, const int64_t* bnd, int strategy, int64_t nrhs,
                       const double* F, int64_t ldf, double* X, int64_t ldx, int64_t* bad);

/* Same as orc_solve_batch but uses `nthreads` POSIX threads over disjoint RHS
 * slices with one shared preliminary (the labelled harness-level RHS-parallel
 * CPU baseline). Returns setup/solve seconds. */
int orc_solve_batch_threads(int64_t n, const double* sub, const double* diag, const double* sup,
                            int64_t p, const int64_t* bnd, int64_t nrhs, const double* F,
                            int64_t ldf, double* X, int64_t ldx, int nthreads,
                            double* setup_s, double* solve_s, int64_t* bad);

/* runtime/run.hpp:93-94: comm_rounds = levels + 2 (0 when p == 0). */
uint64_t orc_comm_rounds(int64_t p);

/* Seeded counter-based generator shared with bench/tests:
 * u_i = (splitmix64(seed ^ i) >> 11) * 2^-53, value = lo + (hi - lo) * u_i. */
void orc_fill_uniform(double* out, int64_t count, uint64_t seed, uint64_t offset, double lo,
                      double hi);

#ifdef __cplusplus
}
#endif

#endif
