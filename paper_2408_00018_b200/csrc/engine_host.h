// engine_host.h — plain structs shared by the kernels (engine.cu) and the
// host driver (capi.cu).
#pragma once

#include <stddef.h>
#include <stdint.h>

#include "parsa_b200.h"
#include "philox.cuh"

namespace psa {

// candidate for the argmin reductions (see engine.cuh: better())
struct Cand {
    double e;
    int32_t c;   // global chain index, INT32_MAX = empty
    int32_t aux; // asynchronous engine: owning thread
};

struct OutScalars {
    double best_f;
    int32_t best_chain;
    int32_t pad;
    unsigned long long evaluations;
    unsigned long long rng_draws;
    unsigned long long exact_settles; // deferred fold: trials decided by exact folds
};

// Kernel arguments (passed by value; all pointers are device pointers).
struct EngineArgs {
    int n;
    int family;
    int N;      // sweep_length
    int levels;
    int uniform_box;
    int random_start;
    double lo0, w0;
    const double* lower;
    const double* width;
    const double* start;
    const double* temps;
    PhiloxKeys keys;
    size_t chains_local;   // chains in this shard
    uint32_t chain_begin;  // global index of the shard's first chain
    uint32_t chains_total;
    void* rows;            // HBM layout only: [n*A][threads] chain state (R elements)
    double* xrows;         // V1: [n][threads] point of each thread's chain ([2][n][threads] for pairs)
    size_t threads;        // grid * block (the SoA stride of rows/xrows)
    uint32_t* masks;       // V2: [2][ceil(N/32)][mask_stride] accept bits
    size_t mask_stride;    // chains_local, rounded up to even (chain pairs)
    Cand* cand;            // V2: [2][grid]; V1: [grid]
    Cand* cand_start;      // V2 random start: [grid]
    Cand* trace_cand;      // V1: [levels][grid]
    double* trace_best;    // [levels]
    double* best_x;        // [n]
    double* xbest;         // V1: [grid*B][n]
    int32_t* level_winner; // V2: [levels] (diagnostic)
    double* level_winner_f;
    OutScalars* out_scalars;
    // multi-GPU level exchange (world > 1): peer-mapped mailboxes
    int world;
    int rank;
    unsigned epoch;         // launch counter, tags mailbox records
    size_t rec_stride;      // bytes per mailbox record
    char* mail_self;        // this GPU's mailbox [2][world] records
    char* const* mail_peers; // device array: every GPU's mailbox as seen from here
    long long spin_limit;   // clock64 cycles before a missing peer is reported
    int* error_flag;
    // deferred fold (v2_lazy_kernel): half-width of the interval of the
    // energy difference, and the finish slope
    double lazy_r;
    double lazy_alpha;
    unsigned long long* work; // [2] per-level chain counters (dynamic assignment)
    double fparam;            // family parameter (PSA_FN_CONSTANT's value)
    int lazy_adapt;           // switch a block to fold-every-trial when settles pass 2%
};

struct NMOut {
    double f_best;
    int32_t iterations;
    int32_t pad;
    unsigned long long evaluations;
};

struct NMArgsHost {
    int n;
    int family;
    int max_iters;
    int q_smem; // 1: each CTA keeps its columns of Q and P in shared memory
    double reflect, expand, contract, shrink, f_tol, x_tol;
    const double* lower;
    const double* upper;
    const double* x_start;
    double* X;      // (n+1) x n simplex storage (vertex-major)
    double* Q;      // (n+1) x n: Q[v][k] = X[v][k] / n, refreshed when vertex v changes
    double* P;      // (n+1) x n: P[p][k] = centroid prefix over the first p sorted vertices
    double* T;      // (n+1) x ldt: cost terms of many vertices evaluated at once (start, shrink)
    int ldt;        // even, >= n * (cached values per coordinate)
    double* x_best; // n
    NMOut* out;
    double fparam;  // family parameter (PSA_FN_CONSTANT's value)
};

// batched NM: one instance per thread (nm_batch_kernel)
struct NMBatchArgs {
    int n;
    int family;
    int max_iters;
    int count;
    double reflect, expand, contract, shrink, f_tol, x_tol;
    const double* lower;
    const double* upper;
    const double* x_starts; // count x n
    double* scratch;        // count x ((n+1)(n+1) + (4+A) n) doubles
    int* order;             // count x (n+1)
    double* x_best;         // count x n
    double* f_best;         // count
    int* iterations;        // count
    unsigned long long* evaluations; // count
    double fparam;                   // family parameter (PSA_FN_CONSTANT's value)
};
const void* nm_batch_kernel_for(int family);
// scratch doubles per batched instance: vertices, values, centroid and three
// trial points, cost terms (A <= 2)
PSA_HD size_t nm_batch_doubles(int n) {
    const size_t d = static_cast<size_t>(n + 1) * n + static_cast<size_t>(n + 1) + 6 * static_cast<size_t>(n);
    return (d + 1) & ~size_t(1); // even: every instance's terms stay 16-byte aligned
}

struct EngineKernels {
    const void* v2;
    const void* v1;
    const void* v2p; // chain pairs (binary32 separable families), or nullptr
    const void* v1p; // V1 with chain pairs, or nullptr
    const void* v2pc; // producer/consumer blocks (small chain counts)
    const void* v1pc; // V1 producer/consumer blocks
    size_t (*smem_v1pc)(int n, int B, bool box);
    size_t (*smem_v2pc)(int n, int B, bool box);
    size_t (*smem_v2p)(int n, int B, bool box); // pair rows (the same for V1 pairs)
    const void* v2g; // HBM chain-state layout (large n)
    const void* v1g;
    size_t (*smem_g)(int n, int B, bool box);
    size_t state_bytes; // sizeof(R) * A: bytes per coordinate of a chain row
    const void* eval;
    const void* sweep; // sweep_one: single caller-held chain (parsa::metropolis_sweep)
    size_t (*smem_v2)(int n, int B, bool box);
    size_t (*smem_v1)(int n, int B, bool box);
    size_t (*smem_eval)(int n, int B);
    // deferred fold (LazyOf families), else nullptr
    const void* v2z;  // shared-memory rows
    const void* v2zu; // shared-memory rows, uniform box
    const void* v2gz; // HBM rows
    const void* v2gzu; // HBM rows, uniform box
    const void* v2pz; // chain pairs (binary32), shared-memory pair rows
    const void* v2pcz; // producer/consumer blocks with the deferred-fold consumer
    const void* v1pcz; // V1 producer/consumer blocks with the deferred-fold consumer
    const void* v0z;   // V0 latency path (one chain in one warp's registers, n <= 32)
    double (*lazy_radius)(int n, const double* lower, const double* upper);
    double (*lazy_alpha_of)(int n);
};

EngineKernels engine_kernels(int precision, int family, int n);
const void* probe_uniforms_kernel();
const void* probe_philox_kernel();
const void* v1_finalize_kernel();
const void* probe_libm_f32_kernel();
const void* nm_kernel_for(int family);
size_t nm_smem_bytes(int n, int cluster_ctas, bool q_smem);
const void* probe_libm_f64_kernel();
const void* probe_metropolis_kernel(int precision);

} // namespace psa
