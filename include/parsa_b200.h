/*
 * parsa_b200.h — C-ABI of the B200-native synchronous parallel simulated
 * annealing engine (arXiv 2408.00018).
 *
 * This is the drop-in boundary for the reference `parsa` C++ library
 * (/root/reference/proj).  Every entry point below replaces one reference
 * C++ function; the citation after each declaration names it.  Signatures use
 * plain pointers and sizes only (no C++ or torch types) so that any host
 * language can bind them (the C++ shim in include/parsa/, ctypes in Python;
 * see INTEGRATION.md).
 *
 * Error model: every function returns a psa_status.  Non-zero statuses map
 * 1:1 onto the reference's exception classes and psa_last_error() returns the
 * reference's exact message text (thread-local, valid until the next call on
 * the same thread).  There is no CPU fallback: on a host without a usable
 * B200 every engine entry point fails with PSA_ERR_NO_DEVICE.
 */
#ifndef PARSA_B200_H
#define PARSA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSA_ABI_VERSION 2

typedef enum psa_status {
    PSA_OK = 0,
    PSA_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                 */
    PSA_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range (unknown ids)       */
    PSA_ERR_LOGIC = 3,            /* std::logic_error (accounting)         */
    PSA_ERR_CUDA = 4,             /* device runtime failure                */
    PSA_ERR_NO_DEVICE = 5         /* no sm_100 device / kernel image       */
} psa_status;

/* sa_core.hpp:11 `enum class Precision { f64, f32 }` */
typedef enum psa_precision { PSA_F64 = 0, PSA_F32 = 1 } psa_precision;

/* engines.hpp:12 `enum class StartMode { shared_point, random_per_chain }` */
typedef enum psa_start_mode { PSA_SHARED_POINT = 0, PSA_RANDOM_PER_CHAIN = 1 } psa_start_mode;

/* Cost-function families: the device twin of each formula template in
 * objectives.cpp (numbering follows the registry ids F0..F19).  The reference
 * plug-in is a pair of host function pointers (objectives.hpp:31-39); on the
 * device a family id selects the compiled cost kernel instead.            */
typedef enum psa_family {
    PSA_FN_SCHWEFEL = 0,         /* objectives.cpp:23-29   F0  */
    PSA_FN_ACKLEY = 1,           /* objectives.cpp:31-41   F1  */
    PSA_FN_BRANIN = 2,           /* objectives.cpp:43-49   F2  */
    PSA_FN_COSINE_MIXTURE = 3,   /* objectives.cpp:54-62   F3  */
    PSA_FN_DEKKERS_AARTS = 4,    /* objectives.cpp:64-69   F4  */
    PSA_FN_EASOM = 5,            /* objectives.cpp:71-75   F5  */
    PSA_FN_EXPONENTIAL = 6,      /* objectives.cpp:77-83   F6  */
    PSA_FN_GOLDSTEIN_PRICE = 7,  /* objectives.cpp:85-94   F7  */
    PSA_FN_GRIEWANK = 8,         /* objectives.cpp:99-107  F8  */
    PSA_FN_HIMMELBLAU = 9,       /* objectives.cpp:109-114 F9  */
    PSA_FN_LEVY_MONTALVO = 10,   /* objectives.cpp:116-131 F10 */
    PSA_FN_MOD_LANGERMAN = 11,   /* objectives.cpp:172-185 F11 */
    PSA_FN_MICHALEWICZ = 12,     /* objectives.cpp:187-198 F12 */
    PSA_FN_RASTRIGIN = 13,       /* objectives.cpp:200-206 F13 */
    PSA_FN_ROSENBROCK = 14,      /* objectives.cpp:212-221 F14 */
    PSA_FN_SALOMON = 15,         /* objectives.cpp:223-230 F15 */
    PSA_FN_SIX_HUMP_CAMEL = 16,  /* objectives.cpp:232-237 F16 */
    PSA_FN_SHUBERT = 17,         /* objectives.cpp:239-248 F17 */
    PSA_FN_SHEKEL5 = 18,         /* objectives.cpp:258-270 F18_a (m=5)  */
    PSA_FN_SHEKEL7 = 19,         /*                        F18_b (m=7)  */
    PSA_FN_SHEKEL10 = 20,        /*                        F18_c (m=10) */
    PSA_FN_SHEKEL_FOXHOLES = 21, /* objectives.cpp:272-284 F19 */
    PSA_FN_SPHERE = 22,          /* sum x_k^2: the "bowl" fixture of test_nelder_mead.cpp:17-38 */
    PSA_FN_CONSTANT = 23,        /* f = param: the constant fixtures of test_engines.cpp:91-99,
                                    test_sa_core.cpp:140-160 */
    PSA_FN_COUNT = 24
} psa_family;

/* ObjectiveFunction (objectives.hpp:31-39) reduced to what the device needs.
 * `id` is only used in error messages ("infeasible start point for <id>"). */
typedef struct psa_objective {
    const char* id;
    int32_t family; /* psa_family */
    int32_t dim;    /* n */
    const double* lower; /* BoxDomain::lower, dim entries */
    const double* upper; /* BoxDomain::upper, dim entries */
    double param;        /* family parameter: PSA_FN_CONSTANT's value (else unused) */
} psa_objective;

/* AnnealSchedule (sa_core.hpp:15-22) */
typedef struct psa_schedule {
    double t0;
    double t_min;
    double rho;
    int32_t sweep_length;
    int32_t reserved;
} psa_schedule;

/* EngineConfig (engines.hpp:14-24) */
typedef struct psa_engine_config {
    int32_t n_chains;
    int32_t start_mode;          /* psa_start_mode */
    const double* start_point;   /* NULL (or len 0) => box centre */
    int32_t start_point_len;
    int32_t precision;           /* psa_precision */
    uint64_t seed;
    int32_t workers;             /* accepted for API parity; results never depend on it */
    int32_t reserved;
    psa_schedule schedule;
} psa_engine_config;

/* TracePoint (engines.hpp:26-30) */
typedef struct psa_trace_point {
    int32_t level;
    int32_t reserved;
    uint64_t cumulative_evals;
    double best_f;
} psa_trace_point;

/* RunResult (engines.hpp:38-47) + PhaseBreakdown (:32-36).  All buffers are
 * caller-owned: best_x holds dim doubles, trace holds trace_capacity rows
 * (levels for v0/v1/v2, levels+1 for hybrid; psa_ladder gives `levels`). */
typedef struct psa_run_result {
    double* best_x;
    psa_trace_point* trace;
    int32_t trace_capacity;
    int32_t trace_len;
    double best_f;
    uint64_t evaluations;
    double wall_time_s;
    int32_t winning_chain;
    int32_t has_phases;
    uint64_t rng_draws;
    uint64_t sa_evaluations;     /* PhaseBreakdown, hybrid only */
    uint64_t refine_evaluations;
    double sa_best_f;
} psa_run_result;

/* NelderMeadConfig (nelder_mead.hpp:11-22) */
typedef struct psa_nm_config {
    double reflect, expand, contract, shrink;
    double f_tol, x_tol;
    int32_t max_iters; /* 0 => 50000 * n */
    int32_t reserved;
} psa_nm_config;

/* NelderMeadResult (nelder_mead.hpp:24-29) */
typedef struct psa_nm_result {
    double* x_best; /* caller-owned, dim entries */
    double f_best;
    int32_t iterations;
    int32_t reserved;
    uint64_t evaluations;
} psa_nm_result;

/* ---- library / errors ------------------------------------------------- */
int32_t psa_abi_version(void);
const char* psa_last_error(void);
/* Number of visible sm_100 devices (0 on a CPU-only host). */
int32_t psa_device_count(void);

/* ---- host-side schedule helpers (byte-identical behaviour) ------------- */
/* AnnealSchedule::validate, sa_core.cpp:8-15 */
psa_status psa_schedule_validate(const psa_schedule* s);
/* ladder, sa_core.cpp:17-27.  temps may be NULL to query *levels only. */
psa_status psa_ladder(const psa_schedule* s, double* temps, int32_t capacity, int32_t* levels);
/* expected_evaluations, sa_core.cpp:29-35 */
psa_status psa_expected_evaluations(const psa_schedule* s, int32_t n_chains, uint64_t* out);
/* reduce_min, engines.cpp:55-64: index (into the arrays) of the winner. */
psa_status psa_reduce_min(const double* f_values, const int32_t* chain_index, int32_t count,
                          int32_t* winner_pos);

/* ---- engines (device) -------------------------------------------------- */
/* run_sequential, engines.cpp:125-129 */
psa_status psa_run_sequential(const psa_objective* f, const psa_engine_config* cfg,
                              psa_run_result* out);
/* run_asynchronous, engines.cpp:66-123 */
psa_status psa_run_asynchronous(const psa_objective* f, const psa_engine_config* cfg,
                                psa_run_result* out);
/* run_synchronous, engines.cpp:131-207 */
psa_status psa_run_synchronous(const psa_objective* f, const psa_engine_config* cfg,
                               psa_run_result* out);
/* nelder_mead_minimize, nelder_mead.cpp:37-115 */
psa_status psa_nelder_mead_minimize(const psa_objective* f, const double* x_start,
                                    const psa_nm_config* nm, psa_nm_result* out);
/* Batched nelder_mead_minimize (nelder_mead.cpp:37-115): `count`
 * independent instances from x_starts (count x dim, row-major), one device
 * thread each, every instance bit-identical to the reference's run from its
 * start.  Outputs are caller-owned arrays of count (x_best: count x dim).
 * For small dim (the simplex lives in per-thread global scratch). */
psa_status psa_nelder_mead_batch(const psa_objective* f, const double* x_starts, int32_t count,
                                 const psa_nm_config* nm, double* x_best, double* f_best,
                                 int32_t* iterations, uint64_t* evaluations);
/* hybrid_run, nelder_mead.cpp:117-136 */
psa_status psa_hybrid_run(const psa_objective* f, const psa_engine_config* cfg,
                          const psa_schedule* truncated, const psa_nm_config* nm,
                          psa_run_result* out);

/* metropolis_sweep, sa_core.cpp:61-79: n_steps Metropolis trials of ONE
 * caller-held chain on the device.  x (dim doubles) and *energy are the
 * ChainState (updated in place); (seed, chain, level, *counter) is its
 * UniformStream (StreamKey + draw counter, advanced by 3*n_steps);
 * *eval_count is incremented by n_steps (may be NULL).  Precision follows
 * chain_energy (sa_core.cpp:57-59). */
psa_status psa_metropolis_sweep(const psa_objective* f, int32_t precision, double* x, double* energy,
                                uint64_t seed, uint32_t chain, uint32_t level, uint64_t* counter,
                                double temperature, int32_t n_steps, uint64_t* eval_count);

/* ---- device-resident plans (benchmarks, multi-GPU shards) --------------
 * A plan uploads the problem once, owns the device buffers and launches the
 * persistent engine kernel on a caller-supplied cudaStream_t (as void*), so
 * a caller can time the device region with its own CUDA events.  A plan may
 * cover a shard [chain_begin, chain_end) of the global chain range; streams
 * are keyed by the global chain index so results do not depend on sharding.
 * engine: 1 = asynchronous (V1), 2 = synchronous (V2). */
typedef struct psa_plan psa_plan;
psa_status psa_plan_create(const psa_objective* f, const psa_engine_config* cfg, int32_t engine,
                           int32_t chain_begin, int32_t chain_end, psa_plan** out);
psa_status psa_plan_launch(psa_plan* p, void* cuda_stream);
psa_status psa_plan_fetch(psa_plan* p, void* cuda_stream, psa_run_result* out);
/* number of levels, chains and device kernel launches per psa_plan_launch */
psa_status psa_plan_info(const psa_plan* p, int32_t* levels, int32_t* chains,
                         int32_t* launches_per_run);
/* human-readable launch description of the plan's engine kernel (layout,
 * block, grid, shared memory), NUL-terminated into buf[capacity] */
psa_status psa_plan_describe(const psa_plan* p, char* buf, int32_t capacity);
psa_status psa_plan_destroy(psa_plan* p);
/* Multi-GPU: a plan may be one rank of a `world`-GPU synchronous run.  Each
 * rank owns a mailbox in its device memory; every rank maps every peer's
 * mailbox (CUDA IPC across processes, or plain pointers within one process)
 * and the persistent kernel exchanges the per-level minloc record through
 * them (engine.cu: exchange_level).  max_blocks > 0 caps the grid (lets
 * several cooperative plans share one GPU). */
typedef struct psa_plan_options {
    int32_t max_blocks;
    int32_t rank;
    int32_t world;
    int32_t reserved;
} psa_plan_options;
psa_status psa_plan_create_ex(const psa_objective* f, const psa_engine_config* cfg, int32_t engine,
                              int32_t chain_begin, int32_t chain_end, const psa_plan_options* opt,
                              psa_plan** out);
psa_status psa_plan_mailbox(const psa_plan* p, void** dev_ptr, uint64_t* bytes);
/* 64-byte cudaIpcMemHandle_t of the plan's mailbox */
psa_status psa_plan_mailbox_ipc_handle(const psa_plan* p, void* handle);
psa_status psa_ipc_open(const void* handle, void** dev_ptr);
psa_status psa_ipc_close(void* dev_ptr);
/* mailboxes[r] = rank r's mailbox as addressable from this device; must be
 * called before the first launch of a world > 1 plan */
psa_status psa_plan_set_peers(psa_plan* p, void* const* mailboxes, int32_t world);
/* synchronous plans: per-level winner chain and its end energy (diagnostic,
 * engines.cpp:187-192), copied to caller buffers of `capacity` entries */
psa_status psa_plan_level_detail(const psa_plan* p, int32_t* winners, double* winner_f,
                                 int32_t capacity);
/* deferred-fold plans (v2_lazy_kernel): how many trials of the last fetched
 * run needed an exact fold to settle their Metropolis decision (0 for the
 * other kernels, which fold every trial) */
psa_status psa_plan_stats(const psa_plan* p, uint64_t* exact_settles);

/* ---- device probes for parity tests ------------------------------------
 * Run the device implementations of the RNG and the cost functions on
 * caller-supplied inputs so tests can compare them bit-for-bit with the
 * oracle.  All buffers are host buffers. */
/* draws first..first+count-1 of stream (seed, chain, level): uniforms */
psa_status psa_device_uniforms(uint64_t seed, uint32_t chain, uint32_t level, uint64_t first,
                               int32_t count, double* out);
/* raw Philox4x32-10 blocks: ctr[4*count] and key[2] -> out[4*count] */
psa_status psa_device_philox(const uint32_t* ctr, const uint32_t* key, int32_t count,
                             uint32_t* out);
/* f(x_i) for count points x[count*dim] (row-major), computed by the device
 * cost kernel in the given precision (f32 results widened to double) */
psa_status psa_device_evaluate(const psa_objective* f, int32_t precision, const double* x,
                               int32_t count, double* out);

/* device copies of the glibc restatements (fn: 0 sinf, 1 cosf, 2 expf,
 * 3/4/5 the branch-free hot-loop sqrtf/sinf/cosf with their validity flag in
 * ok[i], 6 the compiler's sqrt.rn.f32) and of sin/cos/exp (fn 0/1/2) */
psa_status psa_device_libm_f32(int32_t fn, const float* x, int32_t count, float* out, int32_t* ok);
/* the Metropolis pre-test (engine.cuh metropolis_fast) on `count` draws
 * placed at the decision boundary: out = {certain, certain but different
 * from the exact test, undecided} */
psa_status psa_device_metropolis_check(int32_t precision, uint64_t seed, uint64_t count, uint64_t* out);
psa_status psa_device_libm_f64(int32_t fn, const double* x, int32_t count, double* out);

/* ---- host restatements of glibc libm used by the device code ------------
 * The same __host__ __device__ source the kernels use, compiled for the host
 * so CPU tests can pin it against the system libm. */
float psa_libm_sinf(float x);
float psa_libm_cosf(float x);
float psa_libm_expf(float x);
double psa_libm_sin(double x);
double psa_libm_cos(double x);
double psa_libm_exp(double x);

#ifdef __cplusplus
}
#endif

#endif /* PARSA_B200_H */
