// nelder_mead.cu — device Nelder–Mead polish of the hybrid engine.
//
// Restates nelder_mead.cpp:37-115 (always f64) as ONE thread block that
// runs every iteration on the device, with the reference's results bit for
// bit.  Simplex vertices live in global memory (vertex-major (n+1) x n
// doubles, 2 MB at n = 500, L2-resident); the simplex order is an index
// permutation in shared memory.
//
// The reference spends O(n^2) per iteration on two scans of the whole
// simplex: the centroid (centroid[k] += x_i[k] / n over the n best vertices
// in sorted order, one division per element, :70-73) and the diameter test
// (:21-27).  Yet an iteration changes ONE vertex (except a shrink), so both
// are kept incrementally, with the same floating-point operations:
//   * Q[v][k] = x_v[k] / n is computed once when vertex v changes;
//   * P[p/16][k] = the centroid's running sum after the first p sorted
//     vertices, for p a multiple of 16.  Replacing the worst vertex and
//     re-sorting leaves the order of positions < q unchanged (q = where the
//     new vertex lands), so the sum is re-added in order from the last
//     checkpoint at or below q (no divisions: Q is cached);
//   * D[v] = max_k |x_v[k] - x_best[k]| per vertex, valid while the best
//     vertex is unchanged; the diameter is the max over D (order-free).
// A shrink, a new best vertex, or a tie-broken exact sort invalidates what
// they touch, which is then rebuilt in full.  Each cost evaluation computes
// the per-coordinate terms in parallel and folds them in index order on one
// thread (objectives.cpp semantics).  std::sort becomes an insertion of the
// replaced vertex at the position found by a parallel count (a full rank
// sort after a shrink) — the unique sorted order when the values are
// distinct; with ties, thread 0 runs libstdc++'s introsort itself
// (parsa_stdsort.h).
#include <cuda_runtime.h>

#include <stdint.h>

#include "engine.cuh"
#include "engine_host.h"
#include "parsa_stdsort.h"

namespace psa {

using NMArgs = NMArgsHost;

// centroid prefix sums are kept at positions 0, C, 2C, ... (P row p/C)
constexpr int kNmCheckpoint = 16;

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
    double* terms = xc + n;                          // n*A (A <= 2); also int scratch
    double* red = terms + 2 * static_cast<size_t>(n) + 8; // block reduction scratch (32)
    double* scal = red + 32;                          // scalars
    double* f_s = scal + 8;                           // n+1 vertex values
    double* D = f_s + (n + 1);                        // n+1 vertex diameters (vs. the best)
    int* ord_s = reinterpret_cast<int*>(D + (n + 1)); // n+1 sorted order
    int* ist = ord_s + (n + 1);                       // int scalars: [0] vp, [1] D owner (best id, -1 = stale)
    unsigned long long evals = 0;
    double* X = a.X;
    double* Q = a.Q;
    double* P = a.P;
    const double dn = static_cast<double>(n);

    // block-wide max (std::max semantics: NaN never replaces the running max)
    auto block_max = [&](double v) {
        for (int o = 16; o > 0; o >>= 1) {
            const double w = __shfl_xor_sync(0xffffffffu, v, o);
            v = v < w ? w : v;
        }
        if ((tid & 31) == 0) red[tid >> 5] = v;
        __syncthreads();
        if (tid == 0) {
            double m = 0;
            for (int w = 0; w < (B + 31) / 32; ++w) m = m < red[w] ? red[w] : m;
            scal[1] = m;
        }
        __syncthreads();
        const double r = scal[1];
        __syncthreads();
        return r;
    };
    // D[v] for one vertex against the current best (vertex id b)
    auto vertex_diameter = [&](int v, int b) {
        double d = 0;
        for (int k = tid; k < n; k += B) {
            const double t = fabs(X[static_cast<size_t>(v) * n + k] - X[static_cast<size_t>(b) * n + k]);
            d = d < t ? t : d;
        }
        const double m = block_max(d);
        if (tid == 0) D[v] = m;
    };
    auto set_vertex = [&](int v, const double* src) { // X[v] = src, Q[v] = src / n
        for (int k = tid; k < n; k += B) {
            X[static_cast<size_t>(v) * n + k] = src[k];
            Q[static_cast<size_t>(v) * n + k] = src[k] / dn;
        }
    };

    // initial simplex (nelder_mead.cpp:50-59)
    for (int v = 0; v <= n; ++v) {
        for (int k = tid; k < n; k += B) {
            double xk = a.x_start[k];
            if (v > 0 && k == v - 1) {
                const double step = 0.05 * (a.upper[k] - a.lower[k]);
                xk = (xk + step <= a.upper[k]) ? xk + step : xk - step;
            }
            xr[k] = xk;
        }
        __syncthreads();
        set_vertex(v, xr);
        const double fv = block_eval<Cost>(xr, n, a.family, terms, scal);
        if (tid == 0) {
            f_s[v] = fv;
            ord_s[v] = v;
        }
        ++evals;
        __syncthreads();
    }
    for (int k = tid; k < n; k += B) P[k] = 0.0; // P[0] = the centroid's 0.0 fill
    if (tid == 0) {
        ist[0] = 0;  // valid centroid prefix length
        ist[1] = -1; // diameters stale
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
        if (tid == 0) {
            psa_std_sort(ord_s, n + 1, f_s);
            ist[0] = 0;
            ist[1] = -1;
        }
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
        if (tid == 0) {
            ist[0] = 0;
            ist[1] = -1;
        }
        __syncthreads();
    };
    full_sort();

    // replace the worst vertex (physical position n) by the point in src
    // (shared) with value fv, then std::sort
    auto replace_worst = [&](const double* src, double fv) {
        const int w = ord_s[n];
        set_vertex(w, src);
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
        // distinct values: the new vertex lands after every smaller value
        int below = 0;
        for (int p = tid; p < n; p += B) below += f_s[ord_s[p]] < fv;
        for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
        if ((tid & 31) == 0) reinterpret_cast<int*>(red)[tid >> 5] = below;
        __syncthreads();
        int pos = 0;
        for (int i = 0; i < (B + 31) / 32; ++i) pos += reinterpret_cast<int*>(red)[i];
        __syncthreads();
        // shift ord[pos..n-1] up by one and insert w at pos
        for (int p = tid; p <= n; p += B) saved[p] = ord_s[p];
        __syncthreads();
        for (int p = pos + 1 + tid; p <= n; p += B) ord_s[p] = saved[p - 1];
        if (tid == 0) {
            ord_s[pos] = w;
            if (pos < ist[0]) ist[0] = pos;  // centroid prefixes before pos stay valid
            if (pos == 0) ist[1] = -1;       // a new best: every diameter is stale
        }
        __syncthreads();
        if (pos > 0 && ist[1] >= 0) vertex_diameter(w, ord_s[0]);
        __syncthreads();
    };

    int iter = 0;
    for (; iter < a.max_iters; ++iter) {
        // termination (nelder_mead.cpp:67-68; simplex_diameter :21-27)
        const int b0 = ord_s[0];
        if (ist[1] != b0) {
            // all diameters against the best: one warp per vertex
            const int lane = tid & 31, warp = tid >> 5, nw = B >> 5;
            for (int v = warp; v <= n; v += nw) {
                double d = 0;
                for (int k = lane; k < n; k += 32) {
                    const double t = fabs(X[static_cast<size_t>(v) * n + k] - X[static_cast<size_t>(b0) * n + k]);
                    d = d < t ? t : d;
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const double w = __shfl_xor_sync(0xffffffffu, d, o);
                    d = d < w ? w : d;
                }
                if (lane == 0) D[v] = d;
            }
            __syncthreads();
            if (tid == 0) ist[1] = b0;
            __syncthreads();
        }
        double dm = 0;
        for (int i = 1 + tid; i <= n; i += B) dm = dm < D[ord_s[i]] ? D[ord_s[i]] : dm;
        const double dmax = block_max(dm);
        if (f_s[ord_s[n]] - f_s[ord_s[0]] <= a.f_tol || dmax <= a.x_tol) break;

        // centroid of the n best (nelder_mead.cpp:70-73): re-add from the
        // first position whose vertex changed
        // (prefixes are stored every kNmCheckpoint positions: re-adding from
        // the checkpoint at or below the first changed position costs a few
        // adds, storing every prefix would cost an O(n^2) write stream)
        const int vp = (ist[0] / kNmCheckpoint) * kNmCheckpoint;
        for (int k = tid; k < n; k += B) {
            double c = P[static_cast<size_t>(vp / kNmCheckpoint) * n + k];
            for (int p = vp; p < n; ++p) {
                c += Q[static_cast<size_t>(ord_s[p]) * n + k];
                if ((p + 1) % kNmCheckpoint == 0) P[static_cast<size_t>((p + 1) / kNmCheckpoint) * n + k] = c;
            }
            cen[k] = c;
        }
        __syncthreads();
        if (tid == 0) ist[0] = n;
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
                        xr[k] = clampd(x0 + a.shrink * (xv - x0), a.lower[k], a.upper[k]);
                    }
                    __syncthreads();
                    set_vertex(v, xr);
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
    // reduction/scalars (40) + values and diameters (2(n+1)) + order (n+1
    // ints) + int scalars
    return sizeof(double) * (6 * static_cast<size_t>(n) + 48 + 2 * (static_cast<size_t>(n) + 1)) +
           sizeof(int) * (n + 1 + 4) + 64;
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
