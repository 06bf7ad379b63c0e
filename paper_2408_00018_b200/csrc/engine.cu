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

} // namespace psa
