/*
 * sa_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference `parsa` algorithm
 * (/root/reference/proj) used as the CPU checker for the B200 engine.  Every
 * function cites the reference file:line it restates.  It calls the system
 * glibc libm (sin/cos/exp/sqrt and the float variants) exactly as the
 * reference does, so on the same host it reproduces the reference bit for
 * bit; tests/test_oracle.py pins that against oracle/_ref (the reference's
 * own sources compiled unchanged) and against tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker: the product engine
 * (paper_2408_00018_b200) never links or calls it.
 */
#ifndef SA_ORACLE_H
#define SA_ORACLE_H

#include <stdint.h>

#include "parsa_b200.h" /* shared plain-C struct layouts (psa_objective, ...) */

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:39-52 */
void orc_philox4x32_10(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]);
/* rng.hpp:66-75 — draws first..first+count-1 of stream (seed, chain, level) */
void orc_uniforms(uint64_t seed, uint32_t chain, uint32_t level, uint64_t first, int32_t count,
                  double* out);
/* rng.hpp:78-81 */
int32_t orc_coordinate_index(double u, int32_t n);

/* sa_core.cpp:8-35 */
int32_t orc_schedule_validate(const psa_schedule* s); /* 0 ok, else error code 1..3 */
int32_t orc_ladder(const psa_schedule* s, double* temps, int32_t capacity);
uint64_t orc_expected_evaluations(const psa_schedule* s, int32_t n_chains);

/* objectives.cpp:23-284 — f64 / f32 (widened) evaluation of one point */
double orc_evaluate(int32_t family, int32_t n, const double* x);
double orc_evaluate_single(int32_t family, int32_t n, const double* x);

/* engines.cpp:55-64 */
int32_t orc_reduce_min(const double* f, const int32_t* chain, int32_t count);

/* Per-level detail captured by the synchronous restatement (not part of the
 * reference API; used to localise parity failures). Arrays have `levels`
 * entries; pass NULL to skip. */
typedef struct orc_level_detail {
    int32_t* winner;       /* level winner chain (engines.cpp:187-190)   */
    double* winner_f;      /* its end energy                             */
    uint32_t* accept_mask; /* optional: levels*ceil(N/32) words, winner's accept bits */
} orc_level_detail;

/* engines.cpp:131-207.  Returns 0 or an error code (psa_status values). */
int32_t orc_run_synchronous(const psa_objective* f, const psa_engine_config* cfg,
                            psa_run_result* out, orc_level_detail* detail);
/* engines.cpp:66-123 */
int32_t orc_run_asynchronous(const psa_objective* f, const psa_engine_config* cfg,
                             psa_run_result* out);
/* nelder_mead.cpp:37-115 */
int32_t orc_nelder_mead_minimize(const psa_objective* f, const double* x_start,
                                 const psa_nm_config* nm, psa_nm_result* out);
/* nelder_mead.cpp:117-136 */
int32_t orc_hybrid_run(const psa_objective* f, const psa_engine_config* cfg,
                       const psa_schedule* truncated, const psa_nm_config* nm,
                       psa_run_result* out);

#ifdef __cplusplus
}
#endif
#endif
