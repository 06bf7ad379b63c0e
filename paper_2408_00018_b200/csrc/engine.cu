// engine.cu — host-side dispatch of the engine kernel sets over (precision,
// family), the non-template kernels (V1 finalize) and the device probes
// used by the parity tests.  The kernel templates are in engine_kernels.cuh
// and are instantiated per family group in engine_fam_*.cu.
#include "engine_kernels.cuh"

namespace psa {

extern template EngineKernels sep_set<float, Schwefel>(int);
extern template EngineKernels sep_set<float, Ackley>(int);
extern template EngineKernels sep_set_generic<float, CosineMixture>(int);
extern template EngineKernels sep_set_generic<float, Exponential>(int);
extern template EngineKernels sep_set<float, Griewank>(int);
extern template EngineKernels sep_set_generic<float, Michalewicz>(int);
extern template EngineKernels sep_set<float, Rastrigin>(int);
extern template EngineKernels sep_set_generic<float, Salomon>(int);
extern template EngineKernels sep_set_generic<float, Shubert>(int);
extern template EngineKernels sep_set_generic<float, Sphere>(int);
extern template EngineKernels full_set<float>(int);
extern template EngineKernels sep_set<double, Schwefel>(int);
extern template EngineKernels sep_set<double, Ackley>(int);
extern template EngineKernels sep_set_generic<double, CosineMixture>(int);
extern template EngineKernels sep_set_generic<double, Exponential>(int);
extern template EngineKernels sep_set<double, Griewank>(int);
extern template EngineKernels sep_set_generic<double, Michalewicz>(int);
extern template EngineKernels sep_set<double, Rastrigin>(int);
extern template EngineKernels sep_set_generic<double, Salomon>(int);
extern template EngineKernels sep_set_generic<double, Shubert>(int);
extern template EngineKernels sep_set_generic<double, Sphere>(int);
extern template EngineKernels full_set<double>(int);

__global__ void v1_finalize(const EngineArgs a, int blocks) {
    __shared__ Cand scratch[34];
    const int tid = threadIdx.x;
    Cand w = empty_cand();
    for (int i = tid; i < blocks; i += blockDim.x)
        if (better(a.cand[i], w)) w = a.cand[i];
    w = block_argmin(w, scratch);
    for (int k = tid; k < a.n; k += blockDim.x)
        a.best_x[k] = a.xbest[static_cast<size_t>(w.aux) * a.n + k];
    if (tid == 0) {
        a.out_scalars->best_f = w.e;
        a.out_scalars->best_chain = w.c;
    }
    for (int l = 0; l < a.levels; ++l) {
        Cand t = empty_cand();
        for (int i = tid; i < blocks; i += blockDim.x) {
            const Cand c = a.trace_cand[static_cast<size_t>(l) * blocks + i];
            if (better(c, t)) t = c;
        }
        t = block_argmin(t, scratch);
        if (tid == 0) a.trace_best[l] = t.c == INT32_MAX ? __longlong_as_double(0x7ff0000000000000ll) : t.e;
    }
}

// ---------------------------------------------------------------------------
// Probes
// ---------------------------------------------------------------------------

__global__ void probe_uniforms(uint64_t seed, uint32_t chain, uint32_t level, uint64_t first,
                               int count, double* out) {
    const PhiloxKeys keys = make_keys(seed);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        out[i] = bits_to_uniform(draw_bits53(first + i, chain, level, keys));
}

__global__ void probe_philox(const uint32_t* ctr, uint32_t k0, uint32_t k1, int count,
                             uint32_t* out) {
    PhiloxKeys keys;
    uint32_t a = k0, b = k1;
    for (int r = 0; r < 10; ++r) {
        keys.k0[r] = a;
        keys.k1[r] = b;
        a += kPhiloxW0;
        b += kPhiloxW1;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        uint32_t v[4] = {ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]};
        philox4x32_10(v, keys);
        for (int q = 0; q < 4; ++q) out[4 * i + q] = v[q];
    }
}

// device libm restatements on caller points: fn 0 sinf, 1 cosf, 2 expf,
// 3 sqrtf_common (ok ? value : NaN-flag), 4 sinf_common, 5 cosf_common,
// 6 sqrt.rn.f32 (compiler intrinsic, reference for 3)
__global__ void probe_libm_f32(int fn, const float* x, int count, float* out, int* ok_out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const float v = x[i];
        bool ok = true;
        float r;
        switch (fn) {
        case 0: r = libm::sinf(v); break;
        case 1: r = libm::cosf(v); break;
        case 2: r = libm::expf(v); break;
        case 3: r = libm::sqrtf_common(v, ok); break;
        case 4: r = libm::sinf_common(v, ok); break;
        case 5: r = libm::cosf_common(v, ok); break;
        default: r = __fsqrt_rn(v); break;
        }
        out[i] = r;
        ok_out[i] = ok;
    }
}

// device double libm restatements: fn 0 sin, 1 cos, 2 exp
__global__ void probe_libm_f64(int fn, const double* x, int count, double* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
        const double v = x[i];
        out[i] = fn == 0 ? libm::sin(v) : fn == 1 ? libm::cos(v) : libm::exp(v);
    }
}

// Metropolis pre-test check: draws placed at (and around) the decision
// boundary dE* = -T ln(u); out = {certain, certain but different from the
// exact test of sa_core.cpp:46-55, undecided}
template <class R>
__global__ void probe_metropolis(uint64_t seed, unsigned long long count, unsigned long long* out) {
    const PhiloxKeys keys = make_keys(seed);
    unsigned long long certain = 0, wrong = 0, undecided = 0;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += stride) {
        const uint32_t c = static_cast<uint32_t>(i >> 20), lv = static_cast<uint32_t>(i & 0xfffff);
        const uint64_t m = draw_bits53(0, c, lv, keys);
        const double ua = bits_to_uniform(draw_bits53(1, c, lv, keys));
        const double ub = bits_to_uniform(draw_bits53(2, c, lv, keys));
        const double uc = bits_to_uniform(draw_bits53(3, c, lv, keys));
        const double T = exp2(-10.0 + 20.0 * ua);             // 2^-10 .. 2^10
        const double dstar = -T * log(bits_to_uniform(m));     // the boundary (inf for m = 0)
        double dd;
        if ((i & 7) == 0) dd = 2.0 * dstar * ub;               // anywhere below 2 dE*
        else dd = dstar * (1.0 + (ub < 0.5 ? -1.0 : 1.0) * exp2(-40.0 + 34.0 * uc)); // within 2^-40..2^-6
        const R E = static_cast<R>(-500.0 + 1000.0 * ub);
        const R trial = static_cast<R>(static_cast<double>(E) + dd);
        const int r = metropolis_fast<R>(trial, E, metropolis_k2(T), metropolis_band(m));
        const double delta = static_cast<double>(trial) - static_cast<double>(E);
        const bool ref = delta <= 0 || Accept<R>::exact(delta, T, m);
        if (r < 0) {
            ++undecided;
        } else {
            ++certain;
            if ((r != 0) != ref) ++wrong;
        }
    }
    atomicAdd(out, certain);
    atomicAdd(out + 1, wrong);
    atomicAdd(out + 2, undecided);
}

template <class R>
EngineKernels kernels_for(int family, int n) {
#ifdef PSA_EXPERIMENT_ONLY
    // experiment builds: only the benchmark kernel (fast compile)
    (void)family;
    return sep_set<R, Schwefel>(n);
#else
    // compile-time n (10, 30, 100: BASELINE.json's dimensions) for Schwefel
    // and the n = 30 suite of configs[2] (Ackley, Rastrigin, Griewank)
    switch (family) {
    case PSA_FN_SCHWEFEL: return sep_set<R, Schwefel>(n);
    case PSA_FN_ACKLEY: return sep_set<R, Ackley>(n);
    case PSA_FN_COSINE_MIXTURE: return sep_set_generic<R, CosineMixture>(n);
    case PSA_FN_EXPONENTIAL: return sep_set_generic<R, Exponential>(n);
    case PSA_FN_GRIEWANK: return sep_set<R, Griewank>(n);
    case PSA_FN_MICHALEWICZ: return sep_set_generic<R, Michalewicz>(n);
    case PSA_FN_RASTRIGIN: return sep_set<R, Rastrigin>(n);
    case PSA_FN_SALOMON: return sep_set_generic<R, Salomon>(n);
    case PSA_FN_SHUBERT: return sep_set_generic<R, Shubert>(n);
    case PSA_FN_SPHERE: return sep_set_generic<R, Sphere>(n);
    default: return full_set<R>(n);
    }
#endif
}

EngineKernels engine_kernels(int precision, int family, int n) {
    return precision == PSA_F32 ? kernels_for<float>(family, n) : kernels_for<double>(family, n);
}

const void* probe_uniforms_kernel() { return reinterpret_cast<const void*>(&probe_uniforms); }
const void* probe_philox_kernel() { return reinterpret_cast<const void*>(&probe_philox); }
const void* v1_finalize_kernel() { return reinterpret_cast<const void*>(&v1_finalize); }
const void* probe_libm_f32_kernel() { return reinterpret_cast<const void*>(&probe_libm_f32); }
const void* probe_libm_f64_kernel() { return reinterpret_cast<const void*>(&probe_libm_f64); }
const void* probe_metropolis_kernel(int precision) {
    return precision == PSA_F32 ? reinterpret_cast<const void*>(&probe_metropolis<float>)
                                : reinterpret_cast<const void*>(&probe_metropolis<double>);
}

} // namespace psa
