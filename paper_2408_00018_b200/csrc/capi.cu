// capi.cu — the extern "C" boundary (include/parsa_b200.h) and the host
// driver of the device engines.
//
// Host-side semantics restate the reference exactly where they are host
// logic: schedule validation and the do-while ladder (sa_core.cpp:8-35),
// start resolution (engines.cpp:36-41), the reduce_min tie-break
// (engines.cpp:55-64), trace bookkeeping (engines.cpp:48-51,198) and the
// reference's exception messages, mapped to psa_status codes.  Everything
// that touches chains runs on the device; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "engine_host.h"
#include "libm_glibc64.cuh"
#include "parsa_b200.h"

using psa::Cand;
using psa::EngineArgs;
using psa::EngineKernels;
using psa::OutScalars;

namespace {

thread_local std::string g_err;

struct Failure {
    psa_status code;
    std::string msg;
};

[[noreturn]] void fail(psa_status code, const std::string& msg) { throw Failure{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        std::ostringstream m;
        m << "parsa_b200: " << what << ": " << cudaGetErrorString(e);
        fail(PSA_ERR_CUDA, m.str());
    }
}

template <class Fn>
psa_status guarded(Fn&& fn) {
    try {
        fn();
        return PSA_OK;
    } catch (const Failure& f) {
        g_err = f.msg;
        return f.code;
    } catch (const std::bad_alloc&) {
        g_err = "parsa_b200: host allocation failed";
        return PSA_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PSA_ERR_CUDA;
    }
}

// sa_core.cpp:8-15
void validate_schedule(const psa_schedule& s) {
    if (!(s.t0 > 0) || !(s.t_min > 0) || !(s.t_min < s.t0))
        fail(PSA_ERR_INVALID_ARGUMENT, "schedule: need 0 < t_min < t0");
    if (!(s.rho > 0) || !(s.rho < 1)) fail(PSA_ERR_INVALID_ARGUMENT, "schedule: need rho in (0,1)");
    if (s.sweep_length < 1) fail(PSA_ERR_INVALID_ARGUMENT, "schedule: need sweep_length >= 1");
}

// sa_core.cpp:17-27: repeated multiplication, not pow
std::vector<double> ladder_of(const psa_schedule& s) {
    validate_schedule(s);
    std::vector<double> t;
    double v = s.t0;
    do {
        t.push_back(v);
        v *= s.rho;
    } while (v > s.t_min);
    return t;
}

uint64_t expected_evals(const psa_schedule& s, int n_chains, const char* who) {
    if (n_chains < 1) fail(PSA_ERR_INVALID_ARGUMENT, std::string(who) + ": need n_chains >= 1");
    const uint64_t levels = ladder_of(s).size();
    return static_cast<uint64_t>(n_chains) * (1 + static_cast<uint64_t>(s.sweep_length) * levels);
}

void require_dim(int expected, int got, const char* what) {
    if (expected != got) {
        std::ostringstream m;
        m << what << ": expected dimension " << expected << ", got " << got;
        fail(PSA_ERR_INVALID_ARGUMENT, m.str());
    }
}

void check_objective(const psa_objective* f) {
    if (!f) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null objective");
    if (f->family < 0 || f->family >= PSA_FN_COUNT) {
        std::ostringstream m;
        m << "parsa_b200: no device implementation for objective '" << (f->id ? f->id : "?")
          << "' (family " << f->family << ")";
        fail(PSA_ERR_INVALID_ARGUMENT, m.str());
    }
    if (f->dim < 1 || !f->lower || !f->upper)
        fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: objective needs dim >= 1 and a box");
    const int fam = f->family;
    // formulas that read a fixed coordinate count (objectives.cpp:43-114,232-284)
    int need = 0;
    if (fam == PSA_FN_BRANIN || fam == PSA_FN_DEKKERS_AARTS || fam == PSA_FN_EASOM ||
        fam == PSA_FN_GOLDSTEIN_PRICE || fam == PSA_FN_HIMMELBLAU || fam == PSA_FN_SIX_HUMP_CAMEL)
        need = 2;
    if (fam == PSA_FN_SHEKEL5 || fam == PSA_FN_SHEKEL7 || fam == PSA_FN_SHEKEL10) need = 4;
    if (need && f->dim < need) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: dimension too small for family");
    if ((fam == PSA_FN_MOD_LANGERMAN || fam == PSA_FN_SHEKEL_FOXHOLES) && f->dim > 10)
        fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: Langerman/Foxholes data has 10 columns");
}

// engines.cpp:36-41 + BoxDomain::center (objectives.cpp:484-488) + contains (:490-496)
std::vector<double> resolve_start(const psa_objective* f, const psa_engine_config* cfg) {
    const int n = f->dim;
    std::vector<double> s(n);
    if (cfg->start_point && cfg->start_point_len > 0) {
        require_dim(n, cfg->start_point_len, "contains");
        s.assign(cfg->start_point, cfg->start_point + cfg->start_point_len);
    } else {
        for (int k = 0; k < n; ++k) s[k] = 0.5 * (f->lower[k] + f->upper[k]);
    }
    for (int k = 0; k < n; ++k)
        if (s[k] < f->lower[k] || s[k] > f->upper[k])
            fail(PSA_ERR_INVALID_ARGUMENT, std::string("infeasible start point for ") + (f->id ? f->id : ""));
    return s;
}

// sm_100 devices visible to this process; queried once (cudaGetDeviceProperties
// costs milliseconds per device and every engine call checks for a device)
int device_count_sm100() {
    static const int count = [] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        int ok = 0;
        for (int d = 0; d < n; ++d) {
            int major = 0;
            if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10) ++ok;
        }
        return ok;
    }();
    return count;
}

// per-device launch limits, cached (the same device query on every plan)
struct DeviceLimits {
    int sms = 0;
    size_t smem_optin = 0;
};
const DeviceLimits& device_limits(int dev) {
    static DeviceLimits cache[64];
    static std::once_flag once[64];
    const int d = dev < 0 || dev >= 64 ? 0 : dev;
    std::call_once(once[d], [&] {
        int v = 0;
        cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d), "cudaDeviceGetAttribute");
        cache[d].sms = v;
        cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d), "cudaDeviceGetAttribute");
        cache[d].smem_optin = static_cast<size_t>(v);
    });
    return cache[d];
}

void require_device() {
    if (device_count_sm100() == 0)
        fail(PSA_ERR_NO_DEVICE, "parsa_b200: no sm_100 CUDA device available (there is no CPU fallback)");
}

// Device buffers come from the device's stream-ordered memory pool, which
// keeps freed memory for reuse (release threshold: unlimited), so repeated
// engine calls do not pay cudaMalloc/cudaFree (and cudaFree's implicit device
// synchronisation).  Allocation and release are ordered on the legacy
// stream; every user of a buffer has completed before it is released (the
// engine entry points synchronise their stream, psa_plan_destroy the device).
void retain_pool_memory() {
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    });
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        free();
        n = count;
        if (count) {
            retain_pool_memory();
            cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, 0), "cudaMallocAsync");
            cuda_check(cudaStreamSynchronize(0), "cudaMallocAsync");
        }
    }
    void free() {
        if (p) cudaFreeAsync(p, 0);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { free(); }
};

// A buffer another process maps through CUDA IPC: cudaIpcGetMemHandle is
// specified for cudaMalloc allocations only (stream-ordered pool memory is
// not exportable, and a pool sub-allocation is not an allocation base), so
// the multi-GPU mailbox gets its own cudaMalloc.
struct IpcBuf {
    char* p = nullptr;
    size_t n = 0;
    void alloc(size_t bytes) {
        free();
        n = bytes;
        if (bytes) cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), bytes), "cudaMalloc(mailbox)");
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~IpcBuf() { free(); }
};

} // namespace

struct psa_plan {
    int engine = 2; // 1 async, 2 sync
    int n = 0, levels = 0, N = 0, precision = 0, family = 0;
    int32_t chains_local = 0;
    uint32_t chain_begin = 0, chains_total = 0;
    int random_start = 0;
    std::vector<double> temps;
    EngineKernels ks{};
    int block = 128, grid = 0;
    size_t smem = 0;
    EngineArgs args{};
    bool hbm_rows = false;        // chain rows in HBM (large n) instead of shared memory
    bool pair = false;            // two chains per thread (v2_pair_kernel)
    bool pc = false;              // producer/consumer blocks (v2_pc_kernel)
    bool lazy = false;            // deferred fold (v2_lazy_kernel)
    bool lazy_pc = false;         // producer/consumer with the deferred-fold consumer
    bool v0 = false;              // the V0 latency kernel (v0_kernel)
    uint64_t last_settles = 0;    // exact-fold decisions of the last fetched run
    size_t mask_stride = 0;
    const void* kernel = nullptr; // the engine kernel this plan launches
    DevBuf<double> d_lower, d_width, d_start, d_temps, d_trace, d_bestx, d_xbest, d_winner_f, d_xrows;
    DevBuf<unsigned char> d_rows;
    DevBuf<int32_t> d_winner;
    DevBuf<uint32_t> d_masks;
    DevBuf<Cand> d_cand, d_cand_start, d_trace_cand;
    DevBuf<OutScalars> d_out;
    DevBuf<unsigned long long> d_work; // per-level chain counters (v2_lazy_kernel)
    uint64_t expected_evals = 0, expected_draws = 0;
    // multi-GPU exchange
    int world = 1, rank = 0, max_blocks = 0;
    unsigned epoch = 0;
    bool peers_set = false;
    IpcBuf d_mail;                // cudaMalloc'd: exported to peer processes
    DevBuf<char*> d_peers;
    DevBuf<int> d_error;
    size_t rec_stride = 0;
};

namespace {

void plan_build(psa_plan* p, const psa_objective* f, const psa_engine_config* cfg, int engine,
                int32_t chain_begin, int32_t chain_end, const psa_plan_options* opt = nullptr) {
    if (opt) {
        p->world = opt->world > 0 ? opt->world : 1;
        p->rank = opt->rank;
        p->max_blocks = opt->max_blocks;
        if (p->rank < 0 || p->rank >= p->world) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: rank out of range");
        if (p->world > 1 && engine != 2)
            fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: multi-GPU exchange needs the synchronous engine");
    }
    const char* who = engine == 1 ? "run_asynchronous" : "run_synchronous";
    validate_schedule(cfg->schedule); // engines.cpp:133
    if (cfg->n_chains < 1) fail(PSA_ERR_INVALID_ARGUMENT, std::string(who) + ": need n_chains >= 1");
    check_objective(f);
    p->temps = ladder_of(cfg->schedule);
    const std::vector<double> start = resolve_start(f, cfg);
    require_device();
    if (chain_begin < 0 || chain_end > cfg->n_chains || chain_begin >= chain_end)
        fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: invalid chain shard");

    p->engine = engine;
    p->n = f->dim;
    p->levels = static_cast<int>(p->temps.size());
    p->N = cfg->schedule.sweep_length;
    p->precision = cfg->precision == PSA_F32 ? PSA_F32 : PSA_F64;
    p->family = f->family;
    p->chain_begin = static_cast<uint32_t>(chain_begin);
    p->chains_local = chain_end - chain_begin;
    p->chains_total = static_cast<uint32_t>(cfg->n_chains);
    p->random_start = cfg->start_mode == PSA_RANDOM_PER_CHAIN;
    p->ks = psa::engine_kernels(p->precision, p->family, f->dim);

    const int n = p->n;
    std::vector<double> width(n);
    for (int k = 0; k < n; ++k) width[k] = f->upper[k] - f->lower[k]; // BoxDomain::width
    bool uniform = true;
    for (int k = 1; k < n; ++k)
        if (f->lower[k] != f->lower[0] || width[k] != width[0]) uniform = false;

    // block size: the largest of 128/64/32 whose state fits in shared memory
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const DeviceLimits& lim = device_limits(dev);
    const size_t smem_cap = lim.smem_optin;
    auto smem_of = [&](int B) { return engine == 1 ? p->ks.smem_v1(n, B, !uniform) : p->ks.smem_v2(n, B, !uniform); };
    // Kernel choice (all variants are bit-identical; PSA_V2_MODE = single |
    // pair | pc | lazy | lazy1 | lazypair forces one for A/B measurements and
    // tests, PSA_LAZY=0 turns the deferred fold off).
    const char* mode_env = std::getenv("PSA_V2_MODE");
    const std::string mode = mode_env ? mode_env : "";
    const char* lazy_env = std::getenv("PSA_LAZY");
    // Affine families (LazyOf): the deferred-fold sweep settles decisions
    // from an energy interval and folds only when the interval straddles the
    // Metropolis threshold (engine.cuh) — no n-term fold per trial.
    // With few chains (fewer than 8 warps per SM of one chain per thread) the
    // producer/consumer kernel's overlap wins (measured: C1, C3), so the
    // deferred fold is the default only at larger chain counts.
    const bool few_chains = static_cast<long long>(p->chains_local) < 256ll * lim.sms;
    const bool lazy_allowed = p->ks.v2z && !(lazy_env && lazy_env[0] == '0');
    p->lazy = engine == 2 && lazy_allowed &&
              ((mode.empty() && !few_chains) || mode == "lazy" || mode == "lazy1" || mode == "lazypair");
    // block size: of 128/96/64/32 threads, the one that keeps the most
    // chain rows resident per SM (large rows: three 32-thread blocks hold
    // more rows than one 64-thread block); ties go to the larger block
    auto kern_of = [&](bool g) {
        if (p->lazy) return g ? (uniform ? p->ks.v2gzu : p->ks.v2gz) : uniform ? p->ks.v2zu : p->ks.v2z;
        return engine == 1 ? (g ? p->ks.v1g : p->ks.v1) : (g ? p->ks.v2g : p->ks.v2);
    };
    int B = 32;
    int best = -1; // chain rows resident per SM with shared-memory rows
    {
        for (int cand : {128, 96, 64, 32}) {
            const size_t sm_b = smem_of(cand);
            if (sm_b > smem_cap) continue;
            cuda_check(cudaFuncSetAttribute(kern_of(false), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(sm_b)),
                       "cudaFuncSetAttribute");
            int per = 0;
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern_of(false), cand, sm_b), "occupancy");
            if (per * cand > best) {
                best = per * cand;
                B = cand;
            }
        }
    }
    // chain rows that do not fit in shared memory even at 32 threads per
    // block go to the HBM structure-of-arrays layout (large n)
    // (PSA_FORCE_HBM_ROWS=1 selects it at any n: the parity tests compare the
    // two layouts bit for bit)
    const char* force = std::getenv("PSA_FORCE_HBM_ROWS");
    // The deferred fold touches a row once per trial (one term read, a write
    // on acceptance) plus rare folds, so when shared-memory rows leave fewer
    // than 8 warps per SM (large n: C4's n = 500 keeps 3) its rows go to HBM
    // and the SM keeps its full complement of warps (PSA_FORCE_HBM_ROWS=0
    // keeps them in shared memory).
    // In binary32 at large n the interval is wide enough that low
    // temperatures settle often (n = 500: 1.3% of trials at T = 1, each
    // settle two n-term folds from HBM), so there HBM rows are used only
    // when the ladder stays above rr * n (measured: settles <= 0.2% at
    // n = 500 down to T ~ rr n / 1); binary64 intervals are ~1e-12 wide.
    double lazy_rr = 0;
    if (lazy_allowed) {
        std::vector<double> upper(n);
        for (int k = 0; k < n; ++k) upper[k] = f->lower[k] + width[k];
        lazy_rr = p->ks.lazy_radius(n, f->lower, upper.data());
    }
    const bool warm = p->precision == PSA_F64 || p->temps.back() >= lazy_rr * n;
    const bool lazy_hbm = p->lazy && best < 256 && warm && !(force && force[0] == '0');
    p->hbm_rows = smem_of(B) > smem_cap || (force && force[0] == '1') || lazy_hbm;
    if (p->hbm_rows) {
        B = 128;
        if (p->ks.smem_g(n, B, !uniform) > smem_cap)
            fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: dimension too large for the block-shared level state");
    }
    p->block = B;
    p->smem = p->hbm_rows ? p->ks.smem_g(n, B, !uniform) : smem_of(B);
    const void* kern = kern_of(p->hbm_rows);
    // Few chains (fewer than 8 warps per SM of one chain per thread): each
    // chain's level is a latency-bound dependency chain, so producer warps
    // take the proposals off its critical path (v2_pc_kernel).
    // (Not for the families whose finish() runs transcendentals every trial —
    // Ackley, exponential, Salomon: alone on the consumer's critical path
    // they cost more than the producers save; measured on C3.)
    const bool heavy_finish = p->family == PSA_FN_ACKLEY || p->family == PSA_FN_EXPONENTIAL ||
                              p->family == PSA_FN_SALOMON;
    const bool few = static_cast<long long>(p->chains_local) < 256ll * lim.sms && !heavy_finish;
    // (affine families: the consumer warp uses the deferred fold, v2_lazy_pc_kernel)
    const bool lazy_pc = lazy_allowed && (engine == 2 ? p->ks.v2pcz : p->ks.v1pcz) &&
                         (mode.empty() || mode == "lazypc");
    const void* pc_kern = engine == 2 ? (lazy_pc ? p->ks.v2pcz : p->ks.v2pc) : (lazy_pc ? p->ks.v1pcz : p->ks.v1pc);
    const size_t smem_pc = engine == 2 ? p->ks.smem_v2pc(n, 128, !uniform) : p->ks.smem_v1pc(n, 128, !uniform);
    if (!p->lazy && !p->hbm_rows && pc_kern && (mode == "pc" || mode == "lazypc" || (mode.empty() && few)) &&
        smem_pc <= smem_cap) {
        p->pc = true;
        p->lazy_pc = lazy_pc;
        // one chain group (32 chains) per block; when the groups do not fill
        // the SMs (C1: 32 groups), seven producer warps per block instead of
        // three (the producers bound the deferred-fold consumer)
        const long long groups = (static_cast<long long>(p->chains_local) + 31) / 32;
        p->block = B = groups <= lim.sms ? 256 : 128;
        p->smem = smem_pc;
        kern = pc_kern;
    }
    // Binary32 separable families: two chains per thread (FADD2 fold).
    // Pairs halve the threads for the same chains, so they pay off only when
    // the pair kernel still keeps >= 8 warps per SM resident and there are
    // enough pairs to fill them (small chain counts or large n keep one chain
    // per thread; PSA_V2_MODE=pair forces pairs whenever the rows fit).
    // (the deferred fold has a pair form too: v2_lazy_pair_kernel; "lazy1"
    // forces its one-chain form)
    // (measured: the pair form is no faster than one chain per thread, so
    // it runs only when forced)
    const void* pair_kern = p->lazy ? (mode == "lazypair" ? p->ks.v2pz : nullptr) : engine == 2 ? p->ks.v2p : p->ks.v1p;
    if (!p->pc && !p->hbm_rows && pair_kern && mode != "single" && mode != "pc" && mode != "lazy1") {
        int Bp = 128;
        while (Bp > 32 && p->ks.smem_v2p(n, Bp, !uniform) > smem_cap) Bp /= 2;
        const size_t smem_p = p->ks.smem_v2p(n, Bp, !uniform);
        if (smem_p <= smem_cap) {
            cuda_check(cudaFuncSetAttribute(pair_kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem_p)),
                       "cudaFuncSetAttribute");
            int per_sm_p = 0;
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_p, pair_kern, Bp, smem_p), "occupancy");
            const long long pair_threads = static_cast<long long>(per_sm_p) * Bp * lim.sms;
            const long long pairs = (static_cast<long long>(p->chains_local) + 1) / 2;
            const bool worth = per_sm_p * Bp >= 256 && pairs >= pair_threads;
            if (worth || mode == "pair" || mode == "lazypair") {
                p->pair = true;
                p->block = B = Bp;
                p->smem = smem_p;
                kern = pair_kern;
            }
        }
    }
    // V0 (one chain of V1, run_sequential): the latency path when the family
    // has the deferred fold and the chain fits one warp's registers
    if (engine == 1 && p->chains_local == 1 && p->world == 1 && lazy_allowed && p->ks.v0z && n <= 32 &&
        (mode.empty() || mode == "v0")) {
        p->v0 = true;
        p->pc = false;
        p->pair = false;
        p->hbm_rows = false;
        p->block = B = 128;
        p->smem = 0;
        kern = p->ks.v0z;
    }
    p->kernel = kern;
    cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(p->smem)),
               "cudaFuncSetAttribute");
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, B, p->smem), "occupancy");
    if (per_sm < 1) fail(PSA_ERR_CUDA, "parsa_b200: engine kernel cannot be resident");
    const long long units = p->pc     ? (static_cast<long long>(p->chains_local) + 31) / 32 * B
                            : p->pair ? (static_cast<long long>(p->chains_local) + 1) / 2
                                      : p->chains_local;
    const long long need = (units + B - 1) / B;
    p->grid = static_cast<int>(std::min<long long>(need, static_cast<long long>(per_sm) * lim.sms));
    if (p->max_blocks > 0) p->grid = std::min(p->grid, p->max_blocks);

    // device buffers
    p->d_lower.alloc(n);
    p->d_width.alloc(n);
    p->d_start.alloc(n);
    p->d_temps.alloc(p->levels);
    p->d_trace.alloc(p->levels);
    p->d_bestx.alloc(n);
    p->d_out.alloc(1);
    cuda_check(cudaMemcpy(p->d_lower.p, f->lower, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(p->d_width.p, width.data(), sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(p->d_start.p, start.data(), sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(p->d_temps.p, p->temps.data(), sizeof(double) * p->levels, cudaMemcpyHostToDevice), "H2D");
    const size_t W = (p->N + 31) / 32;
    p->mask_stride = (static_cast<size_t>(p->chains_local) + 1) & ~size_t(1);
    if (engine == 2) {
        p->d_masks.alloc(2 * W * static_cast<size_t>(p->mask_stride));
        p->d_cand.alloc(2 * static_cast<size_t>(p->grid));
        p->d_cand_start.alloc(p->grid);
        p->d_winner.alloc(p->levels);
        p->d_winner_f.alloc(p->levels);
    } else {
        p->d_cand.alloc(p->grid);
        p->d_trace_cand.alloc(static_cast<size_t>(p->levels) * p->grid);
        p->d_xbest.alloc(static_cast<size_t>(p->grid) * B * n);
        p->d_xrows.alloc((p->pair ? 2 : 1) * static_cast<size_t>(p->grid) * B * n);
    }
    const size_t threads = static_cast<size_t>(p->grid) * B;
    // HBM rows: n*A values per thread, padded to whole 16-byte vectors
    if (p->hbm_rows) p->d_rows.alloc(threads * ((static_cast<size_t>(n) * p->ks.state_bytes + 15) & ~size_t(15)));

    EngineArgs& a = p->args;
    a.n = n;
    a.family = p->family;
    a.fparam = f->param;
    a.N = p->N;
    a.levels = p->levels;
    a.uniform_box = uniform;
    a.random_start = p->random_start;
    a.lo0 = f->lower[0];
    a.w0 = width[0];
    a.lower = p->d_lower.p;
    a.width = p->d_width.p;
    a.start = p->d_start.p;
    a.temps = p->d_temps.p;
    a.keys = psa::make_keys(cfg->seed);
    a.chains_local = static_cast<size_t>(p->chains_local);
    a.chain_begin = p->chain_begin;
    a.chains_total = p->chains_total;
    a.rows = p->d_rows.p;
    a.xrows = p->d_xrows.p;
    a.threads = threads;
    a.masks = p->d_masks.p;
    a.mask_stride = p->mask_stride;
    a.cand = p->d_cand.p;
    a.cand_start = p->d_cand_start.p;
    a.trace_cand = p->d_trace_cand.p;
    a.trace_best = p->d_trace.p;
    a.best_x = p->d_bestx.p;
    a.xbest = p->d_xbest.p;
    a.level_winner = p->d_winner.p;
    a.level_winner_f = p->d_winner_f.p;
    a.out_scalars = p->d_out.p;
    p->d_work.alloc(2);
    a.work = p->d_work.p;
    p->d_error.alloc(1);
    cuda_check(cudaMemset(p->d_error.p, 0, sizeof(int)), "memset");
    a.error_flag = p->d_error.p;
    a.world = p->world;
    a.rank = p->rank;
    a.spin_limit = 60ll * 2000000000ll; // ~60 s at 2 GHz
    if (p->lazy || p->lazy_pc || p->v0) {
        a.lazy_r = lazy_rr;
        const char* adapt = std::getenv("PSA_LAZY_ADAPT"); // 0: never fall back (tests)
        a.lazy_adapt = !(adapt && adapt[0] == '0');
        a.lazy_alpha = p->ks.lazy_alpha_of(n);
    }
    if (p->world > 1) {
        p->rec_stride = (48 + sizeof(double) * static_cast<size_t>(n) + 127) & ~size_t(127);
        p->d_mail.alloc(2 * static_cast<size_t>(p->world) * p->rec_stride);
        cuda_check(cudaMemset(p->d_mail.p, 0, 2 * static_cast<size_t>(p->world) * p->rec_stride), "memset");
        p->d_peers.alloc(p->world);
        a.rec_stride = p->rec_stride;
        a.mail_self = p->d_mail.p;
        a.mail_peers = p->d_peers.p;
    }

    // the device keeps per-stream draw counters in 32 bits (philox.cuh)
    const uint64_t max_draw = static_cast<uint64_t>(n) + 3ull * p->N * (engine == 1 ? p->levels : 1) + 8;
    if (max_draw >= (1ull << 32))
        fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: more than 2^32 draws per stream is not supported");

    // engines.cpp:48-51 / sa_core.cpp:29-35
    p->expected_evals = static_cast<uint64_t>(p->chains_local) *
                        (1 + static_cast<uint64_t>(p->N) * static_cast<uint64_t>(p->levels));
    p->expected_draws = 3ull * static_cast<uint64_t>(p->N) * p->levels * p->chains_local +
                        (p->random_start ? static_cast<uint64_t>(n) * p->chains_local : 0);
}

void plan_launch(psa_plan* p, cudaStream_t s) {
    if (p->world > 1 && !p->peers_set)
        fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: multi-GPU plan launched before psa_plan_set_peers");
    cuda_check(cudaMemsetAsync(p->d_out.p, 0, sizeof(OutScalars), s), "memset");
    cuda_check(cudaMemsetAsync(p->d_work.p, 0, 2 * sizeof(unsigned long long), s), "memset");
    p->args.epoch = ++p->epoch; // mailbox records of this launch carry the epoch
    void* params[] = {&p->args};
    if (p->engine == 2) {
        cuda_check(cudaLaunchCooperativeKernel(p->kernel, dim3(p->grid), dim3(p->block), params, p->smem, s),
                   "launch v2_kernel");
    } else {
        cuda_check(cudaLaunchKernel(p->kernel, dim3(p->grid), dim3(p->block), params, p->smem, s),
                   "launch v1_kernel");
        int blocks = p->grid;
        void* fparams[] = {&p->args, &blocks};
        cuda_check(cudaLaunchKernel(psa::v1_finalize_kernel(), dim3(1), dim3(256), fparams, 0, s),
                   "launch v1_finalize");
    }
}

void plan_fetch(psa_plan* p, cudaStream_t s, psa_run_result* out) {
    OutScalars o;
    std::vector<double> trace(p->levels);
    cuda_check(cudaMemcpyAsync(&o, p->d_out.p, sizeof(o), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaMemcpyAsync(trace.data(), p->d_trace.p, sizeof(double) * p->levels, cudaMemcpyDeviceToHost, s), "D2H");
    if (out->best_x)
        cuda_check(cudaMemcpyAsync(out->best_x, p->d_bestx.p, sizeof(double) * p->n, cudaMemcpyDeviceToHost, s), "D2H");
    int err_flag = 0;
    cuda_check(cudaMemcpyAsync(&err_flag, p->d_error.p, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "engine run");
    if (err_flag) fail(PSA_ERR_CUDA, "parsa_b200: multi-GPU level exchange timed out (a peer never published)");
    // accounting cross-check (harness.cpp:148-155): the device counted every trial
    if (o.evaluations != p->expected_evals) {
        std::ostringstream m;
        m << "evaluation count mismatch: engine reported " << o.evaluations << ", expected "
          << p->expected_evals;
        fail(PSA_ERR_LOGIC, m.str());
    }
    if (o.rng_draws != p->expected_draws) {
        std::ostringstream m;
        m << "rng draw count mismatch: engine reported " << o.rng_draws << ", expected " << p->expected_draws;
        fail(PSA_ERR_LOGIC, m.str());
    }
    p->last_settles = o.exact_settles;
    out->best_f = o.best_f;
    out->winning_chain = o.best_chain;
    out->evaluations = o.evaluations;
    out->rng_draws = o.rng_draws;
    out->has_phases = 0;
    out->trace_len = p->levels;
    for (int l = 0; l < p->levels && l < out->trace_capacity; ++l) {
        out->trace[l].level = l;
        out->trace[l].reserved = 0;
        // engines.cpp:48-51, over the global chain count (a shard reports the
        // global trace; evaluations/rng_draws above are the shard's own)
        out->trace[l].cumulative_evals =
            static_cast<uint64_t>(p->chains_total) * (1 + static_cast<uint64_t>(p->N) * (l + 1));
        out->trace[l].best_f = trace[l];
    }
}

psa_status run_engine(const psa_objective* f, const psa_engine_config* cfg, int engine,
                      psa_run_result* out) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!out) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null result");
        psa_plan p;
        plan_build(&p, f, cfg, engine, 0, cfg ? cfg->n_chains : 0);
        cudaStream_t s;
        cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
        try {
            plan_launch(&p, s);
            plan_fetch(&p, s, out);
        } catch (...) {
            cudaStreamDestroy(s);
            throw;
        }
        cudaStreamDestroy(s);
        out->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// NelderMeadConfig::validate (nelder_mead.cpp:30-35)
void validate_nm(const psa_nm_config& c) {
    if (!(c.reflect > 0) || !(c.expand > 1) || !(c.contract > 0) || !(c.contract < 1) || !(c.shrink > 0) ||
        !(c.shrink < 1))
        fail(PSA_ERR_INVALID_ARGUMENT, "nelder-mead: coefficient out of range");
}

// nelder_mead_minimize (nelder_mead.cpp:37-115) on the device
void nm_run(const psa_objective* f, const double* x_start, const psa_nm_config* nm, psa_nm_result* out,
            cudaStream_t stream) {
    if (!nm || !out || !x_start) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null argument");
    validate_nm(*nm);
    check_objective(f);
    const int n = f->dim;
    for (int k = 0; k < n; ++k)
        if (x_start[k] < f->lower[k] || x_start[k] > f->upper[k])
            fail(PSA_ERR_INVALID_ARGUMENT, "nelder_mead_minimize: infeasible start");
    require_device();
    const int max_iters = nm->max_iters > 0 ? nm->max_iters : 50000 * n;
    DevBuf<double> d_lo, d_hi, d_x0, d_X, d_Q, d_P, d_T, d_xb;
    DevBuf<psa::NMOut> d_out;
    const int ldt = 2 * n; // >= n * cached values per coordinate (<= 2), even: 16-byte aligned rows
    d_lo.alloc(n);
    d_hi.alloc(n);
    d_x0.alloc(n);
    d_xb.alloc(n);
    d_X.alloc(static_cast<size_t>(n + 1) * n);
    d_Q.alloc(static_cast<size_t>(n + 1) * n);
    d_P.alloc(static_cast<size_t>(n + 1) * n);
    d_T.alloc(static_cast<size_t>(n + 1) * ldt);
    d_out.alloc(1);
    cuda_check(cudaMemcpy(d_lo.p, f->lower, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d_hi.p, f->upper, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d_x0.p, x_start, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
    psa::NMArgsHost a{};
    a.n = n;
    a.family = f->family;
    a.fparam = f->param;
    a.max_iters = max_iters;
    a.reflect = nm->reflect;
    a.expand = nm->expand;
    a.contract = nm->contract;
    a.shrink = nm->shrink;
    a.f_tol = nm->f_tol;
    a.x_tol = nm->x_tol;
    a.lower = d_lo.p;
    a.upper = d_hi.p;
    a.x_start = d_x0.p;
    a.X = d_X.p;
    a.Q = d_Q.p;
    a.P = d_P.p;
    a.T = d_T.p;
    a.ldt = ldt;
    a.x_best = d_xb.p;
    a.out = d_out.p;
    const void* k = psa::nm_kernel_for(f->family);
    // one thread-block cluster: CTA r owns ~32 coordinate columns (up to 16
    // CTAs, the non-portable cluster size of sm_100)
    int cl_max = 16;
    if (const char* e = std::getenv("PSA_NM_CLUSTER")) cl_max = std::max(1, std::min(16, std::atoi(e)));
    const int cl = std::max(1, std::min(cl_max, (n + 31) / 32));
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    int smem_cap = 0;
    cuda_check(cudaDeviceGetAttribute(&smem_cap, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attribute");
    a.q_smem = psa::nm_smem_bytes(n, cl, true) <= static_cast<size_t>(smem_cap) ? 1 : 0;
    const size_t smem = psa::nm_smem_bytes(n, cl, a.q_smem != 0);
    cuda_check(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "cudaFuncSetAttribute");
    if (cl > 8)
        cuda_check(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                   "cudaFuncSetAttribute(non-portable cluster)");
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cl);
    int nm_block = 512;
    if (const char* e = std::getenv("PSA_NM_BLOCK")) nm_block = std::max(32, std::min(512, std::atoi(e) / 32 * 32));
    lc.blockDim = dim3(nm_block);
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    void* params[] = {&a};
    cuda_check(cudaLaunchKernelExC(&lc, k, params), "launch nm_kernel");
    psa::NMOut o;
    cuda_check(cudaMemcpyAsync(&o, d_out.p, sizeof(o), cudaMemcpyDeviceToHost, stream), "D2H");
    if (out->x_best)
        cuda_check(cudaMemcpyAsync(out->x_best, d_xb.p, sizeof(double) * n, cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_check(cudaStreamSynchronize(stream), "nm_kernel");
    out->f_best = o.f_best;
    out->iterations = o.iterations;
    out->evaluations = o.evaluations;
}

} // namespace

extern "C" {

int32_t psa_abi_version(void) { return PSA_ABI_VERSION; }
const char* psa_last_error(void) { return g_err.c_str(); }
int32_t psa_device_count(void) { return device_count_sm100(); }

psa_status psa_schedule_validate(const psa_schedule* s) {
    return guarded([&] { validate_schedule(*s); });
}

psa_status psa_ladder(const psa_schedule* s, double* temps, int32_t capacity, int32_t* levels) {
    return guarded([&] {
        const auto t = ladder_of(*s);
        if (levels) *levels = static_cast<int32_t>(t.size());
        if (temps)
            for (size_t i = 0; i < t.size() && static_cast<int32_t>(i) < capacity; ++i) temps[i] = t[i];
    });
}

psa_status psa_expected_evaluations(const psa_schedule* s, int32_t n_chains, uint64_t* out) {
    return guarded([&] { *out = expected_evals(*s, n_chains, "expected_evaluations"); });
}

psa_status psa_reduce_min(const double* f, const int32_t* chain, int32_t count, int32_t* pos) {
    return guarded([&] {
        if (count < 1) fail(PSA_ERR_INVALID_ARGUMENT, "reduce_min: empty candidate list");
        int32_t best = 0;
        for (int32_t i = 0; i < count; ++i)
            if (f[i] < f[best] || (f[i] == f[best] && chain[i] < chain[best])) best = i;
        *pos = best;
    });
}

psa_status psa_run_synchronous(const psa_objective* f, const psa_engine_config* cfg, psa_run_result* out) {
    return run_engine(f, cfg, 2, out);
}

psa_status psa_run_asynchronous(const psa_objective* f, const psa_engine_config* cfg, psa_run_result* out) {
    return run_engine(f, cfg, 1, out);
}

psa_status psa_run_sequential(const psa_objective* f, const psa_engine_config* cfg, psa_run_result* out) {
    if (cfg && cfg->n_chains != 1) {
        g_err = "run_sequential: requires n_chains == 1";
        return PSA_ERR_INVALID_ARGUMENT;
    }
    return run_engine(f, cfg, 1, out);
}

psa_status psa_nelder_mead_minimize(const psa_objective* f, const double* x_start, const psa_nm_config* nm,
                                    psa_nm_result* out) {
    return guarded([&] { nm_run(f, x_start, nm, out, nullptr); });
}

psa_status psa_nelder_mead_batch(const psa_objective* f, const double* x_starts, int32_t count,
                                 const psa_nm_config* nm, double* x_best, double* f_best, int32_t* iterations,
                                 uint64_t* evaluations) {
    return guarded([&] {
        if (!nm || (count > 0 && (!x_starts || !x_best || !f_best || !iterations || !evaluations)))
            fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null argument");
        if (count < 0) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: negative instance count");
        validate_nm(*nm);
        check_objective(f);
        const int n = f->dim;
        for (int32_t i = 0; i < count; ++i)
            for (int k = 0; k < n; ++k) {
                const double v = x_starts[static_cast<size_t>(i) * n + k];
                if (v < f->lower[k] || v > f->upper[k])
                    fail(PSA_ERR_INVALID_ARGUMENT, "nelder_mead_minimize: infeasible start");
            }
        if (count == 0) return;
        require_device();
        DevBuf<double> d_lo, d_hi, d_x0, d_scr, d_xb, d_fb;
        DevBuf<int> d_ord, d_it;
        DevBuf<unsigned long long> d_ev;
        d_lo.alloc(n);
        d_hi.alloc(n);
        d_x0.alloc(static_cast<size_t>(count) * n);
        d_scr.alloc(static_cast<size_t>(count) * psa::nm_batch_doubles(n));
        d_ord.alloc(static_cast<size_t>(count) * (n + 1));
        d_xb.alloc(static_cast<size_t>(count) * n);
        d_fb.alloc(count);
        d_it.alloc(count);
        d_ev.alloc(count);
        cuda_check(cudaMemcpy(d_lo.p, f->lower, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(d_hi.p, f->upper, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(d_x0.p, x_starts, sizeof(double) * count * n, cudaMemcpyHostToDevice), "H2D");
        psa::NMBatchArgs a{};
        a.n = n;
        a.family = f->family;
        a.fparam = f->param;
        a.max_iters = nm->max_iters > 0 ? nm->max_iters : 50000 * n;
        a.count = count;
        a.reflect = nm->reflect;
        a.expand = nm->expand;
        a.contract = nm->contract;
        a.shrink = nm->shrink;
        a.f_tol = nm->f_tol;
        a.x_tol = nm->x_tol;
        a.lower = d_lo.p;
        a.upper = d_hi.p;
        a.x_starts = d_x0.p;
        a.scratch = d_scr.p;
        a.order = d_ord.p;
        a.x_best = d_xb.p;
        a.f_best = d_fb.p;
        a.iterations = d_it.p;
        a.evaluations = d_ev.p;
        void* params[] = {&a};
        cuda_check(cudaLaunchKernel(psa::nm_batch_kernel_for(f->family), dim3((count + 127) / 128), dim3(128), params,
                                    0, 0),
                   "launch nm_batch_kernel");
        cuda_check(cudaMemcpy(x_best, d_xb.p, sizeof(double) * count * n, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(f_best, d_fb.p, sizeof(double) * count, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(iterations, d_it.p, sizeof(int) * count, cudaMemcpyDeviceToHost), "D2H");
        static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "u64");
        cuda_check(cudaMemcpy(evaluations, d_ev.p, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost), "D2H");
    });
}

psa_status psa_hybrid_run(const psa_objective* f, const psa_engine_config* cfg, const psa_schedule* truncated,
                          const psa_nm_config* nm, psa_run_result* out) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!out || !cfg || !truncated || !nm) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null argument");
        psa_engine_config sa = *cfg; // nelder_mead.cpp:119-121
        sa.schedule = *truncated;
        {
            psa_plan p;
            plan_build(&p, f, &sa, 2, 0, sa.n_chains);
            cudaStream_t s;
            cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
            try {
                plan_launch(&p, s);
                plan_fetch(&p, s, out);
            } catch (...) {
                cudaStreamDestroy(s);
                throw;
            }
            cudaStreamDestroy(s);
        }
        out->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const double sa_best = out->best_f;
        // nelder_mead.cpp:124-135
        const auto t1 = std::chrono::steady_clock::now();
        std::vector<double> xb(f->dim);
        psa_nm_result r{xb.data(), 0, 0, 0, 0};
        nm_run(f, out->best_x, nm, &r, nullptr);
        out->wall_time_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
        if (r.f_best <= out->best_f) {
            out->best_f = r.f_best;
            std::memcpy(out->best_x, xb.data(), sizeof(double) * f->dim);
        }
        out->has_phases = 1;
        out->sa_evaluations = out->evaluations;
        out->refine_evaluations = r.evaluations;
        out->sa_best_f = sa_best;
        out->evaluations += r.evaluations;
        const int row = out->trace_len;
        if (row < out->trace_capacity) {
            out->trace[row].level = row;
            out->trace[row].reserved = 0;
            out->trace[row].cumulative_evals = out->evaluations;
            out->trace[row].best_f = out->best_f;
        }
        out->trace_len = row + 1;
    });
}

psa_status psa_plan_create(const psa_objective* f, const psa_engine_config* cfg, int32_t engine,
                           int32_t chain_begin, int32_t chain_end, psa_plan** out) {
    return guarded([&] {
        if (engine != 1 && engine != 2) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: engine must be 1 or 2");
        auto* p = new psa_plan;
        try {
            plan_build(p, f, cfg, engine, chain_begin, chain_end);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

psa_status psa_plan_create_ex(const psa_objective* f, const psa_engine_config* cfg, int32_t engine,
                              int32_t chain_begin, int32_t chain_end, const psa_plan_options* opt,
                              psa_plan** out) {
    return guarded([&] {
        if (engine != 1 && engine != 2) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: engine must be 1 or 2");
        auto* p = new psa_plan;
        try {
            plan_build(p, f, cfg, engine, chain_begin, chain_end, opt);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

psa_status psa_plan_mailbox(const psa_plan* p, void** dev_ptr, uint64_t* bytes) {
    return guarded([&] {
        if (p->world < 2) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: plan has no mailbox (world == 1)");
        *dev_ptr = p->d_mail.p;
        if (bytes) *bytes = p->d_mail.n;
    });
}

psa_status psa_plan_mailbox_ipc_handle(const psa_plan* p, void* handle) {
    return guarded([&] {
        if (p->world < 2) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: plan has no mailbox (world == 1)");
        cudaIpcMemHandle_t h;
        cuda_check(cudaIpcGetMemHandle(&h, p->d_mail.p), "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, sizeof(h));
    });
}

psa_status psa_ipc_open(const void* handle, void** dev_ptr) {
    return guarded([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        cuda_check(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

psa_status psa_ipc_close(void* dev_ptr) {
    return guarded([&] { cuda_check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle"); });
}

psa_status psa_plan_set_peers(psa_plan* p, void* const* mailboxes, int32_t world) {
    return guarded([&] {
        if (world != p->world) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: peer count does not match the plan");
        std::vector<char*> v(world);
        for (int i = 0; i < world; ++i) v[i] = static_cast<char*>(mailboxes[i]);
        if (v[p->rank] != p->d_mail.p)
            fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: peers[rank] must be the plan's own mailbox");
        cuda_check(cudaMemcpy(p->d_peers.p, v.data(), sizeof(char*) * world, cudaMemcpyHostToDevice), "H2D");
        p->peers_set = true;
    });
}

psa_status psa_plan_launch(psa_plan* p, void* stream) {
    return guarded([&] { plan_launch(p, static_cast<cudaStream_t>(stream)); });
}

psa_status psa_plan_fetch(psa_plan* p, void* stream, psa_run_result* out) {
    return guarded([&] { plan_fetch(p, static_cast<cudaStream_t>(stream), out); });
}

psa_status psa_plan_info(const psa_plan* p, int32_t* levels, int32_t* chains, int32_t* launches) {
    return guarded([&] {
        if (levels) *levels = p->levels;
        if (chains) *chains = p->chains_local;
        if (launches) *launches = p->engine == 2 ? 1 : 2;
    });
}

psa_status psa_plan_describe(const psa_plan* p, char* buf, int32_t capacity) {
    return guarded([&] {
        if (!p || !buf || capacity < 1) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null argument");
        std::ostringstream d;
        const char* layout = p->engine == 1 ? (p->v0 ? "v0_kernel (one chain in one warp's registers, deferred fold, producer warps)"
                                               : p->pc && p->lazy_pc ? "v1_lazy_pc_kernel (deferred-fold consumer, producer/consumer warps, 32 chains per block)"
                                               : p->pc         ? "v1_pc_kernel (producer/consumer warps, 32 chains per block)"
                                               : p->pair       ? "v1_pair_kernel (two chains per thread, shared-memory pair rows)"
                                               : p->hbm_rows ? "v1_kernel (HBM SoA rows)"
                                                             : "v1_kernel (shared-memory rows)")
                             : p->lazy && p->pair ? "v2_lazy_pair_kernel (deferred fold, two chains per thread, shared-memory pair rows)"
                             : p->pair     ? "v2_pair_kernel (two chains per thread, shared-memory pair rows)"
                             : p->pc && p->lazy_pc ? "v2_lazy_pc_kernel (deferred-fold consumer, producer/consumer warps, 32 chains per block)"
                             : p->pc       ? "v2_pc_kernel (producer/consumer warps, 32 chains per block)"
                             : p->lazy     ? (p->hbm_rows ? "v2_lazy_kernel (deferred fold, HBM SoA rows)"
                                                              : "v2_lazy_kernel (deferred fold, one chain per thread, shared-memory rows)")
                             : p->hbm_rows ? "v2_kernel (HBM SoA rows)"
                                           : "v2_kernel (one chain per thread, shared-memory rows)";
        d << layout << " precision=" << (p->precision == PSA_F32 ? "f32" : "f64") << " family=" << p->family
          << " n=" << p->n << " block=" << p->block << " grid=" << p->grid << " smem=" << p->smem;
        const std::string t = d.str();
        const size_t len = std::min(t.size(), static_cast<size_t>(capacity - 1));
        std::memcpy(buf, t.data(), len);
        buf[len] = 0;
    });
}

psa_status psa_plan_level_detail(const psa_plan* p, int32_t* winners, double* winner_f, int32_t capacity) {
    return guarded([&] {
        if (p->engine != 2) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: level detail needs the synchronous engine");
        const int m = std::min(capacity, p->levels);
        if (winners) cuda_check(cudaMemcpy(winners, p->d_winner.p, sizeof(int32_t) * m, cudaMemcpyDeviceToHost), "D2H");
        if (winner_f) cuda_check(cudaMemcpy(winner_f, p->d_winner_f.p, sizeof(double) * m, cudaMemcpyDeviceToHost), "D2H");
    });
}

psa_status psa_plan_stats(const psa_plan* p, uint64_t* exact_settles) {
    return guarded([&] {
        if (!p || !exact_settles) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null argument");
        *exact_settles = p->last_settles;
    });
}

psa_status psa_plan_destroy(psa_plan* p) {
    cudaDeviceSynchronize(); // its buffers return to the pool only after every use
    delete p;
    return PSA_OK;
}

psa_status psa_device_uniforms(uint64_t seed, uint32_t chain, uint32_t level, uint64_t first, int32_t count,
                               double* out) {
    return guarded([&] {
        require_device();
        DevBuf<double> d;
        d.alloc(count);
        int c = count;
        void* params[] = {&seed, &chain, &level, &first, &c, &d.p};
        cuda_check(cudaLaunchKernel(psa::probe_uniforms_kernel(), dim3((count + 255) / 256), dim3(256), params, 0, 0),
                   "probe_uniforms");
        cuda_check(cudaMemcpy(out, d.p, sizeof(double) * count, cudaMemcpyDeviceToHost), "D2H");
    });
}

psa_status psa_device_philox(const uint32_t* ctr, const uint32_t* key, int32_t count, uint32_t* out) {
    return guarded([&] {
        require_device();
        DevBuf<uint32_t> dc, dout;
        dc.alloc(4 * static_cast<size_t>(count));
        dout.alloc(4 * static_cast<size_t>(count));
        cuda_check(cudaMemcpy(dc.p, ctr, sizeof(uint32_t) * 4 * count, cudaMemcpyHostToDevice), "H2D");
        uint32_t k0 = key[0], k1 = key[1];
        int c = count;
        const uint32_t* cp = dc.p;
        void* params[] = {&cp, &k0, &k1, &c, &dout.p};
        cuda_check(cudaLaunchKernel(psa::probe_philox_kernel(), dim3((count + 255) / 256), dim3(256), params, 0, 0),
                   "probe_philox");
        cuda_check(cudaMemcpy(out, dout.p, sizeof(uint32_t) * 4 * count, cudaMemcpyDeviceToHost), "D2H");
    });
}

psa_status psa_device_evaluate(const psa_objective* f, int32_t precision, const double* x, int32_t count,
                               double* out) {
    return guarded([&] {
        check_objective(f);
        require_device();
        const int n = f->dim;
        const EngineKernels ks = psa::engine_kernels(precision == PSA_F32 ? PSA_F32 : PSA_F64, f->family, 0);
        int B = 64;
        while (B > 1 && ks.smem_eval(n, B) > 160 * 1024) B /= 2;
        const size_t smem = ks.smem_eval(n, B);
        cuda_check(cudaFuncSetAttribute(ks.eval, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                   "cudaFuncSetAttribute");
        DevBuf<double> dx, dout;
        dx.alloc(static_cast<size_t>(count) * n);
        dout.alloc(count);
        cuda_check(cudaMemcpy(dx.p, x, sizeof(double) * count * n, cudaMemcpyHostToDevice), "H2D");
        EngineArgs a{};
        a.n = n;
        a.family = f->family;
        a.fparam = f->param;
        int c = count;
        const double* xp = dx.p;
        void* params[] = {&a, &xp, &c, &dout.p};
        cuda_check(cudaLaunchKernel(ks.eval, dim3((count + B - 1) / B), dim3(B), params, smem, 0), "probe_evaluate");
        cuda_check(cudaMemcpy(out, dout.p, sizeof(double) * count, cudaMemcpyDeviceToHost), "D2H");
    });
}

psa_status psa_metropolis_sweep(const psa_objective* f, int32_t precision, double* x, double* energy,
                                uint64_t seed, uint32_t chain, uint32_t level, uint64_t* counter,
                                double temperature, int32_t n_steps, uint64_t* eval_count) {
    return guarded([&] {
        check_objective(f);
        if (!x || !energy || !counter) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null argument");
        if (n_steps <= 0) return; // the reference loop runs zero times
        require_device();
        const int n = f->dim;
        const int prec = precision == PSA_F32 ? PSA_F32 : PSA_F64;
        const EngineKernels ks = psa::engine_kernels(prec, f->family, 0);
        std::vector<double> width(n);
        for (int k = 0; k < n; ++k) width[k] = f->upper[k] - f->lower[k]; // BoxDomain::width
        const size_t row_bytes = (prec == PSA_F32 ? 4 : 8) * static_cast<size_t>(n) * 2 + 16;
        DevBuf<double> d_lo, d_w, d_x, d_e;
        DevBuf<unsigned long long> d_ctr;
        DevBuf<unsigned char> d_row;
        d_lo.alloc(n);
        d_w.alloc(n);
        d_x.alloc(n);
        d_e.alloc(1);
        d_ctr.alloc(1);
        d_row.alloc(row_bytes);
        cuda_check(cudaMemcpy(d_lo.p, f->lower, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(d_w.p, width.data(), sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(d_x.p, x, sizeof(double) * n, cudaMemcpyHostToDevice), "H2D");
        cuda_check(cudaMemcpy(d_e.p, energy, sizeof(double), cudaMemcpyHostToDevice), "H2D");
        const unsigned long long c0 = *counter;
        cuda_check(cudaMemcpy(d_ctr.p, &c0, sizeof(c0), cudaMemcpyHostToDevice), "H2D");
        EngineArgs a{};
        a.n = n;
        a.family = f->family;
        a.fparam = f->param;
        a.lower = d_lo.p;
        a.width = d_w.p;
        a.keys = psa::make_keys(seed);
        void* row = d_row.p;
        double* xp = d_x.p;
        double* ep = d_e.p;
        unsigned long long* cp = d_ctr.p;
        uint32_t ch = chain, lv = level;
        double T = temperature;
        int steps = n_steps;
        void* params[] = {&a, &xp, &row, &ep, &cp, &ch, &lv, &T, &steps};
        cuda_check(cudaLaunchKernel(ks.sweep, dim3(1), dim3(32), params, 0, 0), "sweep_one");
        unsigned long long c1 = 0;
        cuda_check(cudaMemcpy(x, d_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(energy, d_e.p, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        cuda_check(cudaMemcpy(&c1, d_ctr.p, sizeof(c1), cudaMemcpyDeviceToHost), "D2H");
        *counter = c1;
        if (eval_count) *eval_count += static_cast<uint64_t>(n_steps);
    });
}

psa_status psa_device_libm_f32(int32_t fn, const float* x, int32_t count, float* out, int32_t* ok) {
    return guarded([&] {
        require_device();
        DevBuf<float> dx, dout;
        DevBuf<int32_t> dok;
        dx.alloc(count);
        dout.alloc(count);
        dok.alloc(count);
        cuda_check(cudaMemcpy(dx.p, x, sizeof(float) * count, cudaMemcpyHostToDevice), "H2D");
        int f = fn, c = count;
        const float* xp = dx.p;
        void* params[] = {&f, &xp, &c, &dout.p, &dok.p};
        cuda_check(cudaLaunchKernel(psa::probe_libm_f32_kernel(), dim3(std::min(4096, (count + 255) / 256)), dim3(256),
                                    params, 0, 0), "probe_libm_f32");
        cuda_check(cudaMemcpy(out, dout.p, sizeof(float) * count, cudaMemcpyDeviceToHost), "D2H");
        if (ok) cuda_check(cudaMemcpy(ok, dok.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost), "D2H");
    });
}

psa_status psa_device_metropolis_check(int32_t precision, uint64_t seed, uint64_t count, uint64_t* out) {
    return guarded([&] {
        if (!out) fail(PSA_ERR_INVALID_ARGUMENT, "parsa_b200: null argument");
        require_device();
        DevBuf<unsigned long long> d;
        d.alloc(3);
        cuda_check(cudaMemset(d.p, 0, 3 * sizeof(unsigned long long)), "memset");
        unsigned long long c = count;
        void* params[] = {&seed, &c, &d.p};
        cuda_check(cudaLaunchKernel(psa::probe_metropolis_kernel(precision == PSA_F32 ? PSA_F32 : PSA_F64),
                                    dim3(148 * 8), dim3(256), params, 0, 0),
                   "probe_metropolis");
        unsigned long long h[3];
        cuda_check(cudaMemcpy(h, d.p, sizeof(h), cudaMemcpyDeviceToHost), "D2H");
        for (int i = 0; i < 3; ++i) out[i] = h[i];
    });
}

psa_status psa_device_libm_f64(int32_t fn, const double* x, int32_t count, double* out) {
    return guarded([&] {
        require_device();
        DevBuf<double> dx, dout;
        dx.alloc(count);
        dout.alloc(count);
        cuda_check(cudaMemcpy(dx.p, x, sizeof(double) * count, cudaMemcpyHostToDevice), "H2D");
        int f = fn, c = count;
        const double* xp = dx.p;
        void* params[] = {&f, &xp, &c, &dout.p};
        cuda_check(cudaLaunchKernel(psa::probe_libm_f64_kernel(), dim3(std::min(4096, (count + 255) / 256)), dim3(256),
                                    params, 0, 0), "probe_libm_f64");
        cuda_check(cudaMemcpy(out, dout.p, sizeof(double) * count, cudaMemcpyDeviceToHost), "D2H");
    });
}

float psa_libm_sinf(float x) { return psa::libm::sinf(x); }
float psa_libm_cosf(float x) { return psa::libm::cosf(x); }
float psa_libm_expf(float x) { return psa::libm::expf(x); }
double psa_libm_sin(double x) { return psa::libm::sin(x); }
double psa_libm_cos(double x) { return psa::libm::cos(x); }
double psa_libm_exp(double x) { return psa::libm::exp(x); }

} // extern "C"
