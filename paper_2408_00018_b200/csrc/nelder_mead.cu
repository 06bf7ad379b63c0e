// nelder_mead.cu — device Nelder–Mead polish of the hybrid engine.
//
// Restates nelder_mead.cpp:37-115 (always f64) as ONE thread block that
// runs every iteration on the device: simplex vertices in global memory
// (row-major, (n+1) x n doubles: 2 MB at n = 500, L2-resident), the
// centroid / trial points / cached terms in shared memory, and the simplex
// order as an index permutation.  Each phase parallelises over coordinates
// while keeping the reference's per-coordinate operation order:
//   * centroid[k] += x_i[k] / n over i in sorted order (sequential per k,
//     one IEEE division per element, nelder_mead.cpp:70-73);
//   * each cost evaluation computes per-coordinate terms in parallel and
//     folds them in index order on one thread (objectives.cpp semantics);
//   * std::sort of the simplex becomes an insertion of the replaced vertex
//     (or a full stable rank sort after a shrink) — identical order whenever
//     the vertex values are distinct (and for any ties when n + 1 <= 16,
//     where libstdc++'s std::sort is an insertion sort).
#include <cuda_runtime.h>

#include <stdint.h>

#include "engine.cuh"
#include "engine_host.h"
#include "parsa_stdsort.h"

namespace psa {

using NMArgs = NMArgsHost;

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v); // std::clamp
}

// f64 evaluation of the shared-memory point xs (block-cooperative)
template <class Cost>
__device__ double block_eval(const double* xs, int n, int family, double* terms, double* result) {
    constexpr int A = Cost::A;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        double t[A];
        Cost::cache(xs[k], k, n, t);
#pragma unroll
        for (int a = 0; a < A; ++a) terms[k * A + a] = t[a];
    }
    __syncthreads();
    if (threadIdx.x == 0) *result = Cost::template energy<0>(terms, n, family);
    __syncthreads();
    return *result;
}

template <class Cost>
__global__ void __launch_bounds__(512) nm_kernel(const NMArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n, tid = threadIdx.x, B = blockDim.x;
    double* cen = reinterpret_cast<double*>(smem_raw);
    double* xr = cen + n;
    double* xe = xr + n;
    double* xc = xe + n;
    double* terms = xc + n;                         // n*A (A <= 2)
    double* red = terms + 2 * static_cast<size_t>(n); // block reduction scratch (32)
    double* scal = red + 32;                         // scalars
    int* ord_s = reinterpret_cast<int*>(scal + 8);   // n+1
    double* f_s = reinterpret_cast<double*>(ord_s + ((n + 1 + 1) & ~1)); // n+1
    unsigned long long evals = 0;
    double* X = a.X;

    // initial simplex (nelder_mead.cpp:50-59)
    for (int v = 0; v <= n; ++v) {
        for (int k = tid; k < n; k += B) {
            double xk = a.x_start[k];
            if (v > 0 && k == v - 1) {
                const double step = 0.05 * (a.upper[k] - a.lower[k]);
                xk = (xk + step <= a.upper[k]) ? xk + step : xk - step;
            }
            X[static_cast<size_t>(v) * n + k] = xk;
            xr[k] = xk;
        }
        __syncthreads();
        const double fv = block_eval<Cost>(xr, n, a.family, terms, scal);
        if (tid == 0) {
            f_s[v] = fv;
            ord_s[v] = v;
        }
        ++evals;
        __syncthreads();
    }
    // std::sort of the simplex (nelder_mead.cpp:60,111).  With pairwise
    // distinct values every correct sort yields the same order, so the block
    // sorts in parallel (rank sort, or one insertion after replacing the worst
    // vertex); if any two values are equivalent (equal or NaN) the order of
    // the tied vertices is what libstdc++'s introsort makes of the physical
    // order, so thread 0 runs that exact algorithm (parsa_stdsort.h).
    int* saved = reinterpret_cast<int*>(terms) + 2 * (n + 1); // pre-sort physical order
    auto equiv = [](double a, double b) { return !(a < b) && !(b < a); };
    auto exact_sort = [&]() {
        if (tid == 0) psa_std_sort(ord_s, n + 1, f_s);
        __syncthreads();
    };
    auto full_sort = [&]() {
        for (int p = tid; p <= n; p += B) saved[p] = ord_s[p];
        __syncthreads();
        // rank of the vertex at position p = #{q : f_q < f_p or (f_q == f_p and q < p)}
        for (int p = tid; p <= n; p += B) {
            const double fp = f_s[saved[p]];
            int r = 0;
            for (int q = 0; q <= n; ++q) {
                const double fq = f_s[saved[q]];
                r += (fq < fp) || (fq == fp && q < p);
            }
            reinterpret_cast<int*>(terms)[p] = r;
        }
        __syncthreads();
        for (int p = tid; p <= n; p += B) ord_s[reinterpret_cast<int*>(terms)[p]] = saved[p];
        __syncthreads();
        int tie = 0;
        for (int p = tid; p < n; p += B) tie |= equiv(f_s[ord_s[p]], f_s[ord_s[p + 1]]);
        if (__syncthreads_or(tie)) {
            for (int p = tid; p <= n; p += B) ord_s[p] = saved[p];
            __syncthreads();
            exact_sort();
        }
    };
    full_sort();

    // replace the worst vertex (physical position n) by the point in src
    // (shared) with value fv, then std::sort
    auto replace_worst = [&](const double* src, double fv) {
        const int w = ord_s[n];
        for (int k = tid; k < n; k += B) X[static_cast<size_t>(w) * n + k] = src[k];
        if (tid == 0) f_s[w] = fv;
        __syncthreads();
        int tie = 0;
        for (int p = tid; p < n; p += B) {
            tie |= equiv(f_s[ord_s[p]], fv);
            if (p + 1 < n) tie |= equiv(f_s[ord_s[p]], f_s[ord_s[p + 1]]);
        }
        if (__syncthreads_or(tie)) {
            exact_sort();
            return;
        }
        if (tid == 0) {
            int p = n;
            while (p > 0 && fv < f_s[ord_s[p - 1]]) {
                ord_s[p] = ord_s[p - 1];
                --p;
            }
            ord_s[p] = w;
        }
        __syncthreads();
    };

    int iter = 0;
    for (; iter < a.max_iters; ++iter) {
        // termination (nelder_mead.cpp:67-68; simplex_diameter :21-27)
        const int b0 = ord_s[0];
        double dmax = 0;
        for (int k = tid; k < n; k += B) {
            const double x0 = X[static_cast<size_t>(b0) * n + k];
            for (int i = 1; i <= n; ++i) {
                const double d = fabs(X[static_cast<size_t>(ord_s[i]) * n + k] - x0);
                dmax = dmax < d ? d : dmax;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(0xffffffffu, dmax, o);
            dmax = dmax < w ? w : dmax;
        }
        if ((tid & 31) == 0) red[tid >> 5] = dmax;
        __syncthreads();
        if (tid == 0) {
            double m = 0;
            for (int w = 0; w < (B + 31) / 32; ++w) m = m < red[w] ? red[w] : m;
            scal[1] = m;
        }
        __syncthreads();
        if (f_s[ord_s[n]] - f_s[ord_s[0]] <= a.f_tol || scal[1] <= a.x_tol) break;

        // centroid of the n best (nelder_mead.cpp:70-73)
        for (int k = tid; k < n; k += B) {
            double c = 0.0;
            for (int i = 0; i < n; ++i) c += X[static_cast<size_t>(ord_s[i]) * n + k] / n;
            cen[k] = c;
        }
        const int worst = ord_s[n];
        const double worst_f = f_s[worst];
        for (int k = tid; k < n; k += B) {
            const double wk = X[static_cast<size_t>(worst) * n + k];
            xr[k] = clampd(cen[k] + a.reflect * (cen[k] - wk), a.lower[k], a.upper[k]);
        }
        __syncthreads();
        const double fr = block_eval<Cost>(xr, n, a.family, terms, scal);
        ++evals;
        if (fr < f_s[ord_s[0]]) {
            for (int k = tid; k < n; k += B)
                xe[k] = clampd(cen[k] + a.expand * (xr[k] - cen[k]), a.lower[k], a.upper[k]);
            __syncthreads();
            const double fe = block_eval<Cost>(xe, n, a.family, terms, scal);
            ++evals;
            if (fe < fr) replace_worst(xe, fe);
            else replace_worst(xr, fr);
        } else if (fr < f_s[ord_s[n - 1]]) {
            replace_worst(xr, fr);
        } else {
            const bool outside = fr < worst_f;
            for (int k = tid; k < n; k += B) {
                const double toward = outside ? xr[k] : X[static_cast<size_t>(worst) * n + k];
                xc[k] = clampd(cen[k] + a.contract * (toward - cen[k]), a.lower[k], a.upper[k]);
            }
            __syncthreads();
            const double fc = block_eval<Cost>(xc, n, a.family, terms, scal);
            ++evals;
            if (fc < (outside ? fr : worst_f)) {
                replace_worst(xc, fc);
            } else {
                // shrink towards the best vertex (nelder_mead.cpp:101-108)
                const int best = ord_s[0];
                for (int i = 1; i <= n; ++i) {
                    const int v = ord_s[i];
                    for (int k = tid; k < n; k += B) {
                        const double x0 = X[static_cast<size_t>(best) * n + k];
                        const double xv = X[static_cast<size_t>(v) * n + k];
                        const double nv = clampd(x0 + a.shrink * (xv - x0), a.lower[k], a.upper[k]);
                        X[static_cast<size_t>(v) * n + k] = nv;
                        xr[k] = nv;
                    }
                    __syncthreads();
                    const double fv = block_eval<Cost>(xr, n, a.family, terms, scal);
                    ++evals;
                    if (tid == 0) f_s[v] = fv;
                    __syncthreads();
                }
                full_sort();
            }
        }
        __syncthreads();
    }
    const int b = ord_s[0];
    for (int k = tid; k < n; k += B) a.x_best[k] = X[static_cast<size_t>(b) * n + k];
    if (tid == 0) {
        a.out->f_best = f_s[b];
        a.out->iterations = iter;
        a.out->evaluations = evals;
    }
}

size_t nm_smem_bytes(int n) {
    // cen, xr, xe, xc (4n) + terms (2n, also int scratch for 3(n+1) ids) +
    // reduction/scalars (40) + order (n+1 ints) + values (n+1)
    return sizeof(double) * (6 * static_cast<size_t>(n) + 48) + sizeof(int) * (n + 3) +
           sizeof(double) * (n + 2) + 64;
}

template <class Cost>
const void* nm_kernel_ptr() {
    return reinterpret_cast<const void*>(&nm_kernel<Cost>);
}

const void* nm_kernel_for(int family) {
    switch (family) {
    case PSA_FN_SCHWEFEL: return nm_kernel_ptr<SepCost<double, Schwefel>>();
    case PSA_FN_ACKLEY: return nm_kernel_ptr<SepCost<double, Ackley>>();
    case PSA_FN_COSINE_MIXTURE: return nm_kernel_ptr<SepCost<double, CosineMixture>>();
    case PSA_FN_EXPONENTIAL: return nm_kernel_ptr<SepCost<double, Exponential>>();
    case PSA_FN_GRIEWANK: return nm_kernel_ptr<SepCost<double, Griewank>>();
    case PSA_FN_MICHALEWICZ: return nm_kernel_ptr<SepCost<double, Michalewicz>>();
    case PSA_FN_RASTRIGIN: return nm_kernel_ptr<SepCost<double, Rastrigin>>();
    case PSA_FN_SALOMON: return nm_kernel_ptr<SepCost<double, Salomon>>();
    case PSA_FN_SHUBERT: return nm_kernel_ptr<SepCost<double, Shubert>>();
    case PSA_FN_SPHERE: return nm_kernel_ptr<SepCost<double, Sphere>>();
    default: return nm_kernel_ptr<FullCost<double>>();
    }
}

} // namespace psa
