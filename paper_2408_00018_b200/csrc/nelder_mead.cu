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
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <stdint.h>
#include <stdio.h>

#include "engine.cuh"
#include "engine_host.h"
#include "parsa_stdsort.h"
#include "parsa_stdsort_pairs.hpp"

namespace psa {

namespace cg = cooperative_groups;

using NMArgs = NMArgsHost;

// centroid prefix sums are kept at positions 0, C, 2C, ... (P row p/C)
constexpr int kNmCheckpoint = 16;

// ranges of one introsort level over n+1 values (each larger than the
// insertion threshold, so at most (n+1)/17 of them), with slack
PSA_HD int nm_sort_ranges(int n) { return (n + 1) / 16 + 2; }

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v < lo ? lo : (hi < v ? hi : v); // std::clamp
}

// ---------------------------------------------------------------------------
// One Nelder–Mead instance on a thread-block CLUSTER of CL CTAs (CL = 1 for
// small n).  CTA r owns the coordinate columns [c0, c1): it keeps its slice
// of the simplex (X, Q, P in global memory), of the centroid and of the trial
// points, and computes those columns' cost terms.  The cost fold needs every
// term in index order, so the terms are gathered into CTA 0's shared memory
// (DSMEM stores), CTA 0 folds them on one thread and stores the value into
// every CTA (two cluster barriers per evaluation).  Everything that decides
// the control flow — the values f, the sorted order, ties, insertion points —
// is replicated in every CTA and updated by the same operations on the same
// data, so every CTA takes the same branches.  The simplex diameter is a max
// over columns, so each CTA keeps per-vertex maxima over its own columns and
// the termination test max-reduces CL partials through DSMEM.
// ---------------------------------------------------------------------------

// The centroid re-add of one column (nelder_mead.cpp:70-73 from the
// checkpoint at vp): one dependent DADD chain in the reference's summation
// order, so its cost is latency — whole checkpoint segments load their 16
// quotients, then add unconditionally (no predicated selects in the chain;
// the caller passes shared-memory pointers when Q lives there, so the loads
// are LDS rather than generic loads).  Q element (v, 0) at
// Qc[v * st], P row r at Pc[r * st]; writes the checkpoints it passes.
static __device__ __forceinline__ double centroid_readd(const double* Qc, double* Pc, size_t st, const int* ord_s,
                                                       int vp, int n) {
    double c = Pc[static_cast<size_t>(vp / kNmCheckpoint) * st];
    int p0 = vp;
    for (; p0 + kNmCheckpoint <= n; p0 += kNmCheckpoint) {
        double q[kNmCheckpoint];
#pragma unroll
        for (int i = 0; i < kNmCheckpoint; ++i) q[i] = Qc[static_cast<size_t>(ord_s[p0 + i]) * st];
#pragma unroll
        for (int i = 0; i < kNmCheckpoint; ++i) c += q[i];
        Pc[static_cast<size_t>((p0 + kNmCheckpoint) / kNmCheckpoint) * st] = c;
    }
    for (; p0 < n; ++p0) c += Qc[static_cast<size_t>(ord_s[p0]) * st]; // the last, partial segment
    return c;
}

template <class Cost>
__global__ void __launch_bounds__(512, 1) nm_kernel(const NMArgs a) {
    constexpr int A = Cost::A;
    fn_param_init<Cost>(a.fparam);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int CL = static_cast<int>(cluster.num_blocks());
    const int rank = static_cast<int>(cluster.block_rank());
    const int n = a.n, tid = threadIdx.x, B = blockDim.x;
    const int c0 = static_cast<int>((static_cast<long long>(rank) * n) / CL);
    const int c1 = static_cast<int>((static_cast<long long>(rank + 1) * n) / CL);
    const int nc = c1 - c0; // columns of this CTA
    // every CTA uses the same shared-memory layout (sized for the widest
    // column slice), so DSMEM addresses mapped from local pointers line up
    const int ncmax = (n + CL - 1) / CL;

    double* terms = reinterpret_cast<double*>(smem_raw);  // n*A: the gather target in CTA 0
    double* cen = terms + 2 * static_cast<size_t>(n) + 8;  // own columns
    double* xr = cen + ncmax;
    double* xe = xr + ncmax;
    double* xc = xe + ncmax;
    double* red = xc + ncmax;                               // block reduction scratch (32)
    double* scal = red + 32;                                // scalars: [0] broadcast f, [1] block max
    double* dslot = scal + 8;                               // CL diameter partials (<= 16)
    double* f_s = dslot + 16;                               // n+1 vertex values
    double* D = f_s + (n + 1);                              // n+1 vertex diameters over own columns
    int* ord_s = reinterpret_cast<int*>(D + (n + 1));       // n+1 sorted order
    int* ist = ord_s + (n + 1);                             // int scalars: [0] vp, [1] D owner (-1 = stale)
    unsigned long long evals = 0;
#ifdef PSA_NM_PROFILE
    // measurement builds only (scripts/build_nm_profile.sh): cycles per phase
    // and path counters on CTA 0 thread 0, printed at the end
    unsigned long long pf[6] = {0, 0, 0, 0, 0, 0}, pc[6] = {0, 0, 0, 0, 0, 0}, pt[2] = {0, 0};
    long long tq = clock64();
#define NMP(i)                                   \
    do {                                         \
        if (rank == 0 && tid == 0) {             \
            const long long t_ = clock64();      \
            pf[i] += static_cast<unsigned long long>(t_ - tq); \
            tq = t_;                             \
        }                                        \
    } while (0)
#define NMC(i, v)                                \
    do {                                         \
        if (rank == 0 && tid == 0) pc[i] += (v); \
    } while (0)
#else
#define NMP(i) \
    do {       \
    } while (0)
#define NMC(i, v) \
    do {          \
    } while (0)
#endif
    double* X = a.X;
    // Q (and the centroid checkpoints P) of this CTA's columns: in shared
    // memory when the slice fits (a.q_smem), else in global memory.  Element
    // (v, j) of either lives at base[v * stride + j].
    // (the shared slice starts after the int scratch: ist[4], ranks, saved order)
    const int nranges = nm_sort_ranges(n); // range lists of the warp exact sort
    const uintptr_t qraw =
        (reinterpret_cast<uintptr_t>(ist + 4 + 2 * (n + 1) + 10 * nranges) + 15) & ~uintptr_t(15);
    double* Qb = a.q_smem ? reinterpret_cast<double*>(qraw) : a.Q + c0;
    const size_t qst = a.q_smem ? static_cast<size_t>(ncmax) : static_cast<size_t>(n);
    double* Pb = a.q_smem ? Qb + static_cast<size_t>(n + 1) * ncmax : a.P + c0;
    const double dn = static_cast<double>(n);
    double* terms0 = cluster.map_shared_rank(terms, 0);
    // cluster barrier (a plain block barrier when the cluster is one CTA)
    auto csync = [&]() {
        if (CL == 1) __syncthreads();
        else cluster.sync();
    };

    // f(x) for the point whose own columns are in xs (every CTA calls this)
    auto eval = [&](const double* xs) {
        for (int j = tid; j < nc; j += B) {
            double t[A];
            Cost::cache(xs[j], c0 + j, n, t);
#pragma unroll
            for (int q = 0; q < A; ++q) terms0[static_cast<size_t>(c0 + j) * A + q] = t[q];
        }
        csync();
        if (rank == 0 && tid == 0) {
            const double f = Cost::template energy<0>(terms, n, a.family);
            for (int r = 0; r < CL; ++r) cluster.map_shared_rank(scal, r)[0] = f;
        }
        csync();
        return scal[0];
    };
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
    auto col = [&](int v, int j) -> double& { return X[static_cast<size_t>(v) * n + c0 + j]; };
    // D[v] over own columns against the current best (vertex id b)
    auto vertex_diameter = [&](int v, int b) {
        double d = 0;
        for (int j = tid; j < nc; j += B) {
            const double t = fabs(col(v, j) - col(b, j));
            d = d < t ? t : d;
        }
        const double m = block_max(d);
        if (tid == 0) D[v] = m;
    };
    auto set_vertex = [&](int v, const double* src) { // X[v] = src, Q[v] = src / n (own columns)
        for (int j = tid; j < nc; j += B) {
            col(v, j) = src[j];
            Qb[static_cast<size_t>(v) * qst + j] = src[j] / dn;
        }
    };

    // f of many vertices at once (the initial simplex, a shrink): the caller
    // has stored the terms of vertex list[first + i] (or first + i) into row i
    // of T (global memory, L2-resident); the cluster's threads then fold one
    // row each — the same index-order fold as eval(), for every vertex in
    // parallel instead of one after another — and store each value into every
    // CTA's f_s.
    auto eval_rows = [&](int first, int count, const int* list) {
        __threadfence();
        csync();
        for (int i = rank * B + tid; i < count; i += CL * B) {
            const double f = Cost::template energy<0>(a.T + static_cast<size_t>(i) * a.ldt, n, a.family);
            const int v = list ? list[first + i] : first + i;
            for (int r = 0; r < CL; ++r) cluster.map_shared_rank(f_s, r)[v] = f;
        }
        csync();
    };
    auto put_terms = [&](int row, int j, double x) { // row `row` of T, own column j
        double t[A];
        Cost::cache(x, c0 + j, n, t);
#pragma unroll
        for (int q = 0; q < A; ++q) a.T[static_cast<size_t>(row) * a.ldt + static_cast<size_t>(c0 + j) * A + q] = t[q];
    };

    // initial simplex (nelder_mead.cpp:50-59): n+1 independent evaluations
    for (int idx = tid; idx < (n + 1) * nc; idx += B) {
        const int v = idx / nc, j = idx - v * nc, k = c0 + j;
        double xk = a.x_start[k];
        if (v > 0 && k == v - 1) {
            const double step = 0.05 * (a.upper[k] - a.lower[k]);
            xk = (xk + step <= a.upper[k]) ? xk + step : xk - step;
        }
        col(v, j) = xk;
        Qb[static_cast<size_t>(v) * qst + j] = xk / dn;
        put_terms(v, j, xk);
    }
    for (int v = tid; v <= n; v += B) ord_s[v] = v;
    eval_rows(0, n + 1, nullptr);
    evals += n + 1;
    for (int j = tid; j < nc; j += B) Pb[j] = 0.0; // P[0] = the centroid's 0.0 fill
    if (tid == 0) {
        ist[0] = 0;  // valid centroid prefix length
        ist[1] = -1; // diameters stale
    }
    // std::sort of the simplex (nelder_mead.cpp:60,111).  With pairwise
    // distinct values every correct sort yields the same order, so the block
    // sorts in parallel (rank sort, or one insertion after replacing the worst
    // vertex); if any two values are equivalent (equal or NaN) the order of
    // the tied vertices is what libstdc++'s introsort makes of the physical
    // order, so the block runs that exact algorithm (parsa_stdsort.h).
    int* rk = ist + 4;         // n+1 ints: ranks of the full sort
    int* saved = rk + (n + 1); // n+1 ints: the pre-sort order
    // the warp exact sort: rk / saved hold its stop lists, these its ranges
    const psa_sort::WarpSortLists wsl{saved + (n + 1), saved + (n + 1) + 3 * nranges,
                                      saved + (n + 1) + 6 * nranges};
    auto equiv = [](double a, double b) { return !(a < b) && !(b < a); };
    // (key, id) pairs for the exact sort: one 16-byte load per comparison
    // instead of an id and then its key (the terms area is idle here)
    psa_sort::KeyId* kp = reinterpret_cast<psa_sort::KeyId*>(terms);
    // Without NaN keys warp 0 runs the sort's task form (psa_sort::range_task:
    // the introsort's disjoint ranges one per lane, level by level; the same
    // order as sort(), see parsa_stdsort_pairs.hpp); with NaNs thread 0 runs
    // sort() itself.  Range lists: rk / saved (idle here), 3 ints per range.
    //  w >= 0: the sort follows replace_worst(w), the only vertex that changed:
    //  centroid prefixes before the first reordered position and (if the best
    //  vertex stays) every other diameter stay valid; w < 0: all are stale.
    auto exact_sort = [&](int w) {
#ifdef PSA_NM_PROFILE
        const long long xs0 = clock64();
#endif
        if (tid == 0) ist[3] = n + 1;
        int has_nan = 0;
        for (int p = tid; p <= n; p += B) {
            const double fk = f_s[ord_s[p]];
            kp[p] = psa_sort::KeyId{fk, ord_s[p], 0};
            has_nan |= fk != fk;
        }
#ifdef PSA_NM_SEQ_SORT
        has_nan = 1; // A/B builds: always the one-thread sort
#endif
        const bool any_nan = __syncthreads_or(has_nan);
        // tie_min: the smallest value held by two vertices.  After
        // replace_worst the first n keys are still in sorted order, so ties
        // are adjacent pairs there or the new value against any of them;
        // after a full rank sort (w < 0) it is not computed (-inf: the warp
        // sort's heap phase then pops everything)
        double tie_min = -__builtin_huge_val();
        if (w >= 0 && !any_nan) {
            double t = __builtin_huge_val();
            for (int p = tid; p < n; p += B) {
                const double k = kp[p].key;
                if (p + 1 < n && k == kp[p + 1].key) t = fmin(t, k);
                if (k == kp[n].key) t = fmin(t, k);
            }
            for (int o = 16; o > 0; o >>= 1) t = fmin(t, __shfl_xor_sync(0xffffffffu, t, o));
            if ((tid & 31) == 0) red[tid >> 5] = t;
            __syncthreads();
            t = __builtin_huge_val();
            for (int i = 0; i < (B + 31) / 32; ++i) t = fmin(t, red[i]);
            tie_min = t;
            __syncthreads();
        }
        if (any_nan || n + 1 <= PSA_SORT_THRESHOLD) {
            if (tid == 0) psa_sort::sort(kp, n + 1);
        } else if (tid < 32) {
            psa_sort::warp_sort(kp, n + 1, rk, saved, wsl, tie_min);
        }
        __syncthreads();
        const int old_best = ord_s[0];
        for (int p = tid; p <= n; p += B)
            if (kp[p].id != ord_s[p]) atomicMin(&ist[3], p); // first reordered position
        __syncthreads();
        for (int p = tid; p <= n; p += B) ord_s[p] = kp[p].id;
        __syncthreads();
        const bool keep_d = w >= 0 && ist[1] >= 0 && ord_s[0] == old_best;
        __syncthreads(); // every thread has read ist[1] before thread 0 updates it
        NMC(0, 1);
        NMC(4, keep_d ? 1 : 0);
        if (tid == 0) {
            ist[0] = w >= 0 ? min(ist[0], ist[3]) : 0;
            if (!keep_d) ist[1] = -1;
        }
        __syncthreads();
        if (keep_d) vertex_diameter(w, ord_s[0]);
        __syncthreads();
#ifdef PSA_NM_PROFILE
        if (rank == 0 && tid == 0) pc[5] += static_cast<unsigned long long>(clock64() - xs0);
        // tie groups after the sort: adjacent equal values whose points are
        // bitwise identical over this CTA's columns (pt[0]) or not (pt[1])
        if (rank == 0 && tid == 0) {
            for (int p = 0; p < n; ++p) {
                if (!(f_s[ord_s[p]] == f_s[ord_s[p + 1]])) continue;
                bool same = true;
                for (int j = 0; j < nc && same; ++j)
                    same = __double_as_longlong(col(ord_s[p], j)) == __double_as_longlong(col(ord_s[p + 1], j));
                pt[same ? 0 : 1] += 1;
            }
        }
#endif
    };
    auto full_sort = [&]() {
        // a NaN value breaks the rank count below (it would share rank 0 with
        // the minimum and leave positions unwritten): such keys go straight to
        // the exact introsort, whose one-thread form handles them
        int nan_key = 0;
        for (int v = tid; v <= n; v += B) nan_key |= f_s[v] != f_s[v];
        if (__syncthreads_or(nan_key)) {
            exact_sort(-1);
            return;
        }
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
            rk[p] = r;
        }
        __syncthreads();
        for (int p = tid; p <= n; p += B) ord_s[rk[p]] = saved[p];
        __syncthreads();
        int tie = 0;
        for (int p = tid; p < n; p += B) tie |= equiv(f_s[ord_s[p]], f_s[ord_s[p + 1]]);
        if (__syncthreads_or(tie)) {
            for (int p = tid; p <= n; p += B) ord_s[p] = saved[p];
            __syncthreads();
            exact_sort(-1);
        }
        if (tid == 0) {
            ist[0] = 0;
            ist[1] = -1;
        }
        __syncthreads();
    };
    full_sort();

    // replace the worst vertex (physical position n) by the point in src
    // (own columns) with value fv, then std::sort
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
            exact_sort(w);
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
            NMC(1, 1);
            // all diameters (own columns) against the best: one warp per vertex
            const int lane = tid & 31, warp = tid >> 5, nw = B >> 5;
            for (int v = warp; v <= n; v += nw) {
                double d = 0;
                for (int j = lane; j < nc; j += 32) {
                    const double t = fabs(col(v, j) - col(b0, j));
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
        dm = block_max(dm);
        if (tid == 0)
            for (int r = 0; r < CL; ++r) cluster.map_shared_rank(dslot, r)[rank] = dm;
        csync();
        double dmax = 0;
        for (int r = 0; r < CL; ++r) dmax = dmax < dslot[r] ? dslot[r] : dmax;
        if (f_s[ord_s[n]] - f_s[ord_s[0]] <= a.f_tol || dmax <= a.x_tol) break;
        NMP(0);

        // centroid of the n best (nelder_mead.cpp:70-73), own columns: re-add
        // from the checkpoint at or below the first changed position (prefix
        // sums are stored every kNmCheckpoint positions)
        const int vp = (ist[0] / kNmCheckpoint) * kNmCheckpoint;
        NMC(2, n - vp);
        // The re-add is one dependent DADD chain per column (the reference's
        // summation order), so its cost is latency: whole checkpoint segments
        // add unconditionally (no predicated selects in the chain), the next
        // segment's quotients are loaded while this one adds, and with Q in
        // shared memory the loads are LDS (the branch keeps the pointer's
        // address space visible to the compiler).
        if (a.q_smem) {
            const double* Qs = reinterpret_cast<const double*>(qraw);
            double* Ps = reinterpret_cast<double*>(qraw) + static_cast<size_t>(n + 1) * ncmax;
            for (int j = tid; j < nc; j += B)
                cen[j] = centroid_readd(Qs + j, Ps + j, static_cast<size_t>(ncmax), ord_s, vp, n);
        } else {
            for (int j = tid; j < nc; j += B)
                cen[j] = centroid_readd(a.Q + c0 + j, a.P + c0 + j, static_cast<size_t>(n), ord_s, vp, n);
        }
        __syncthreads();
        if (tid == 0) ist[0] = n;
        const int worst = ord_s[n];
        const double worst_f = f_s[worst];
        for (int j = tid; j < nc; j += B) {
            const int k = c0 + j;
            xr[j] = clampd(cen[j] + a.reflect * (cen[j] - col(worst, j)), a.lower[k], a.upper[k]);
        }
        __syncthreads();
        NMP(1);
        const double fr = eval(xr);
        ++evals;
        NMP(2);
        if (fr < f_s[ord_s[0]]) {
            for (int j = tid; j < nc; j += B)
                xe[j] = clampd(cen[j] + a.expand * (xr[j] - cen[j]), a.lower[c0 + j], a.upper[c0 + j]);
            __syncthreads();
            const double fe = eval(xe);
            ++evals;
            NMP(2);
            if (fe < fr) replace_worst(xe, fe);
            else replace_worst(xr, fr);
        } else if (fr < f_s[ord_s[n - 1]]) {
            replace_worst(xr, fr);
        } else {
            const bool outside = fr < worst_f;
            for (int j = tid; j < nc; j += B) {
                const double toward = outside ? xr[j] : col(worst, j);
                xc[j] = clampd(cen[j] + a.contract * (toward - cen[j]), a.lower[c0 + j], a.upper[c0 + j]);
            }
            __syncthreads();
            const double fc = eval(xc);
            ++evals;
            NMP(2);
            if (fc < (outside ? fr : worst_f)) {
                replace_worst(xc, fc);
            } else {
                // shrink towards the best vertex (nelder_mead.cpp:101-108)
                // (each new vertex depends only on itself and the best one,
                // so all n are built and evaluated at once)
                const int best = ord_s[0];
                for (int idx = tid; idx < n * nc; idx += B) {
                    const int i = idx / nc, j = idx - i * nc;
                    const int v = ord_s[i + 1];
                    const double x0 = col(best, j);
                    const double xv = clampd(x0 + a.shrink * (col(v, j) - x0), a.lower[c0 + j], a.upper[c0 + j]);
                    col(v, j) = xv;
                    Qb[static_cast<size_t>(v) * qst + j] = xv / dn;
                    put_terms(i, j, xv);
                }
                eval_rows(1, n, ord_s);
                evals += n;
                full_sort();
                NMC(3, 1);
                NMP(4);
            }
        }
        NMP(3);
        __syncthreads();
    }
#ifdef PSA_NM_PROFILE
    if (rank == 0 && tid == 0)
        printf("NMPROF iters=%d evals=%llu cyc_term=%llu cyc_centroid=%llu cyc_eval=%llu cyc_replace=%llu "
               "cyc_shrink=%llu tie_sorts=%llu diam_full=%llu readd_len=%llu shrinks=%llu keep_d=%llu "
               "cyc_exact_sort=%llu tie_pairs_same_point=%llu tie_pairs_distinct=%llu\n",
               iter, evals, pf[0], pf[1], pf[2], pf[3], pf[4], pc[0], pc[1], pc[2], pc[3], pc[4], pc[5], pt[0], pt[1]);
#endif
    const int b = ord_s[0];
    for (int j = tid; j < nc; j += B) a.x_best[c0 + j] = col(b, j);
    if (rank == 0 && tid == 0) {
        a.out->f_best = f_s[b];
        a.out->iterations = iter;
        a.out->evaluations = evals;
    }
    cluster.sync(); // no CTA may exit while others can still store into its shared memory
}

// ---------------------------------------------------------------------------
// Batched Nelder–Mead: one independent instance per thread (small n).
//
// nelder_mead_minimize (nelder_mead.cpp:37-115) restated literally for one
// thread — the O(n^2) centroid with a division per element, the clamped
// trial points, std::sort through the libstdc++ introsort restatement
// (parsa_stdsort.h) — so every instance equals the reference's run from its
// start point bit for bit.  Used to polish many points at once (e.g. the
// best chains of a run); scratch is instance-major global memory (L1/L2).
// ---------------------------------------------------------------------------

template <class Cost>
__global__ void __launch_bounds__(128) nm_batch_kernel(const NMBatchArgs a) {
    constexpr int A = Cost::A;
    fn_param_init<Cost>(a.fparam);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.count) return;
    const int n = a.n;
    const size_t per = nm_batch_doubles(n); // (host allocates count * per)
    // terms first: the fold reads them with 16-byte loads (per is even)
    double* terms = a.scratch + static_cast<size_t>(i) * per; // n*A (A <= 2)
    double* X = terms + 2 * static_cast<size_t>(n);            // (n+1) x n vertices
    double* F = X + static_cast<size_t>(n + 1) * n;            // n+1 values
    double* cen = F + (n + 1);
    double* xr = cen + n;
    double* xe = xr + n;
    double* xc = xe + n;
    int* ord = a.order + static_cast<size_t>(i) * (n + 1);
    const double* x0 = a.x_starts + static_cast<size_t>(i) * n;
    unsigned long long evals = 0;
    auto eval = [&](const double* x) {
        for (int k = 0; k < n; ++k) {
            double t[A];
            Cost::cache(x[k], k, n, t);
#pragma unroll
            for (int q = 0; q < A; ++q) terms[k * A + q] = t[q];
        }
        ++evals;
        return static_cast<double>(Cost::template energy<0>(terms, n, a.family));
    };
    auto vx = [&](int v) { return X + static_cast<size_t>(v) * n; };
    // initial simplex (nelder_mead.cpp:50-59)
    for (int v = 0; v <= n; ++v) {
        double* x = vx(v);
        for (int k = 0; k < n; ++k) x[k] = x0[k];
        if (v > 0) {
            const int k = v - 1;
            const double step = 0.05 * (a.upper[k] - a.lower[k]);
            x[k] = (x[k] + step <= a.upper[k]) ? x[k] + step : x[k] - step;
        }
        F[v] = eval(x);
        ord[v] = v;
    }
    psa_std_sort(ord, n + 1, F);
    int iter = 0;
    for (; iter < a.max_iters; ++iter) {
        // termination (:67-68) with simplex_diameter (:21-27)
        double diam = 0;
        const double* b = vx(ord[0]);
        for (int v = 1; v <= n; ++v) {
            const double* x = vx(ord[v]);
            for (int k = 0; k < n; ++k) {
                const double d = fabs(x[k] - b[k]);
                diam = diam < d ? d : diam;
            }
        }
        if (F[ord[n]] - F[ord[0]] <= a.f_tol || diam <= a.x_tol) break;
        for (int k = 0; k < n; ++k) cen[k] = 0.0;
        for (int v = 0; v < n; ++v) {
            const double* x = vx(ord[v]);
            for (int k = 0; k < n; ++k) cen[k] += x[k] / n;
        }
        const int w = ord[n];
        const double* worst = vx(w);
        const double worst_f = F[w];
        for (int k = 0; k < n; ++k) xr[k] = clampd(cen[k] + a.reflect * (cen[k] - worst[k]), a.lower[k], a.upper[k]);
        const double fr = eval(xr);
        const double* src = nullptr;
        double fs = 0;
        if (fr < F[ord[0]]) {
            for (int k = 0; k < n; ++k) xe[k] = clampd(cen[k] + a.expand * (xr[k] - cen[k]), a.lower[k], a.upper[k]);
            const double fe = eval(xe);
            src = fe < fr ? xe : xr;
            fs = fe < fr ? fe : fr;
        } else if (fr < F[ord[n - 1]]) {
            src = xr;
            fs = fr;
        } else {
            const bool outside = fr < worst_f;
            for (int k = 0; k < n; ++k) {
                const double toward = outside ? xr[k] : worst[k];
                xc[k] = clampd(cen[k] + a.contract * (toward - cen[k]), a.lower[k], a.upper[k]);
            }
            const double fc = eval(xc);
            if (fc < (outside ? fr : worst_f)) {
                src = xc;
                fs = fc;
            } else {
                // shrink towards the best vertex (:101-108)
                const double* x0b = vx(ord[0]);
                for (int v = 1; v <= n; ++v) {
                    double* x = vx(ord[v]);
                    for (int k = 0; k < n; ++k) x[k] = clampd(x0b[k] + a.shrink * (x[k] - x0b[k]), a.lower[k], a.upper[k]);
                    F[ord[v]] = eval(x);
                }
            }
        }
        if (src) {
            double* x = vx(w);
            for (int k = 0; k < n; ++k) x[k] = src[k];
            F[w] = fs;
        }
        psa_std_sort(ord, n + 1, F);
    }
    const double* b = vx(ord[0]);
    for (int k = 0; k < n; ++k) a.x_best[static_cast<size_t>(i) * n + k] = b[k];
    a.f_best[i] = F[ord[0]];
    a.iterations[i] = iter;
    a.evaluations[i] = evals;
}

template <class Cost>
const void* nm_batch_ptr() {
    return reinterpret_cast<const void*>(&nm_batch_kernel<Cost>);
}

const void* nm_batch_kernel_for(int family) {
    switch (family) {
    case PSA_FN_SCHWEFEL: return nm_batch_ptr<SepCost<double, Schwefel>>();
    case PSA_FN_ACKLEY: return nm_batch_ptr<SepCost<double, Ackley>>();
    case PSA_FN_COSINE_MIXTURE: return nm_batch_ptr<SepCost<double, CosineMixture>>();
    case PSA_FN_EXPONENTIAL: return nm_batch_ptr<SepCost<double, Exponential>>();
    case PSA_FN_GRIEWANK: return nm_batch_ptr<SepCost<double, Griewank>>();
    case PSA_FN_MICHALEWICZ: return nm_batch_ptr<SepCost<double, Michalewicz>>();
    case PSA_FN_RASTRIGIN: return nm_batch_ptr<SepCost<double, Rastrigin>>();
    case PSA_FN_SALOMON: return nm_batch_ptr<SepCost<double, Salomon>>();
    case PSA_FN_SHUBERT: return nm_batch_ptr<SepCost<double, Shubert>>();
    case PSA_FN_SPHERE: return nm_batch_ptr<SepCost<double, Sphere>>();
    default: return nm_batch_ptr<FullCost<double>>();
    }
}

// shared memory of one CTA of an NM cluster of `cl` CTAs; with q_smem the
// CTA also keeps its columns' quotients Q ((n+1) x ceil(n/cl)) and centroid
// checkpoints (n/16+1 rows) in shared memory
size_t nm_smem_bytes(int n, int cl, bool q_smem) {
    const size_t nc = (static_cast<size_t>(n) + cl - 1) / cl;
    const size_t ranges = static_cast<size_t>(nm_sort_ranges(n));
    // doubles: terms (2n + 8), own-column cen/xr/xe/xc (4 nc), red/scal/dslot
    // (56), f and D (2(n+1)); ints: order, ranks, saved order (3(n+1)) and
    // scalars (4), padding (2)
    size_t b = sizeof(double) * (2 * static_cast<size_t>(n) + 8 + 4 * nc + 56 + 2 * (static_cast<size_t>(n) + 1)) +
               sizeof(int) * (3 * (static_cast<size_t>(n) + 1) + 6 + 10 * ranges);
    b = (b + 15) & ~size_t(15);
    if (q_smem) b += sizeof(double) * nc * (static_cast<size_t>(n) + 1 + static_cast<size_t>(n) / kNmCheckpoint + 1);
    return b + 64;
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
