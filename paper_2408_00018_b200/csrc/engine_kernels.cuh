#pragma once
// engine_kernels.cuh — kernel templates of the persistent synchronous engine
// (V2), the asynchronous engine (V1/V0) and their per-family kernel sets.
// Instantiated per family in engine_fam_*.cu (parallel compilation);
// engine.cu holds the dispatch and the non-template kernels.
//
// Synchronous engine (engines.cpp:131-207) as ONE cooperative kernel:
//
//   for each level l (engines.cpp:171):
//     every thread sweeps its chains c = gtid, gtid + G*B, ... from the
//       level start x*_l: cache V := V*, N Metropolis trials on stream
//       (seed, c, l) with the term-cached energy, accept bits -> masks;
//     warp-shuffle -> block argmin -> cand[l&1][block]          (:187-190)
//     grid.sync()
//     every block: argmin over cand[l&1][*] (identical in all blocks), then
//       rebuilds x*_{l+1} by replaying the winner's accepted moves from its
//       accept mask and stream (no chain state leaves the SM), recomputes
//       V* = cache(x*_{l+1}); block 0 keeps best-so-far and the trace
//       (:191-198).
//
// One grid-wide barrier per level; cand and masks are double-buffered by
// level parity so a block that runs ahead cannot overwrite data a slower
// block is still reading.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <stdint.h>

#include <type_traits>

#include "engine.cuh"
#include "engine_host.h"

namespace cg = cooperative_groups;

// Engine blocks never exceed 128 threads (capi.cu picks 128/64/32), and the
// shared-memory chain state caps residency at about 4 such blocks per SM, so
// the register budget can be 128 per thread without costing occupancy.
#ifndef PSA_V2_MAX_THREADS
#define PSA_V2_MAX_THREADS 128
#endif
#ifndef PSA_V2_MIN_BLOCKS
#define PSA_V2_MIN_BLOCKS 4
#endif

namespace psa {

// ---------------------------------------------------------------------------
// shared-memory carve-up
// ---------------------------------------------------------------------------

struct Smem {
    unsigned char* base;
    size_t off = 0;
    template <class T>
    __device__ T* take(size_t count) {
        off = (off + 15) & ~size_t(15);
        T* p = reinterpret_cast<T*>(base + off);
        off += sizeof(T) * count;
        return p;
    }
};

template <class R, int A>
size_t engine_smem_bytes(int n, int B, bool box, bool rows_in_smem, bool pair = false) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        off = (off + 15) & ~size_t(15);
        off += bytes;
    };
    if (rows_in_smem) take(sizeof(R) * size_t(row_stride<R>(pair ? 2 * n : n, A)) * B); // per-thread state rows
    take(sizeof(double) * n);            // x*
    take(sizeof(R) * size_t(n) * A);     // V*
    if (box) take(sizeof(double) * n);   // lower (only for a non-uniform box)
    if (box) take(sizeof(double) * n);   // width
    take(sizeof(Cand) * 34);             // reduction scratch
    take(64);                            // scalars
    return off;
}

struct SharedScalars {
    double estar;
    double best_f;
    int32_t best_c;
    int32_t fold_mode;               // deferred-fold kernel: fold every trial from now on
    unsigned long long lv_settles;   // deferred-fold kernel: this level's exact settles
    unsigned long long lv_chains;    //   and chains swept by the block
};

template <class R, class Cost>
__device__ void load_box(const EngineArgs& a, double* lower, double* width, Box& box) {
    for (int k = threadIdx.x; k < a.n; k += blockDim.x) {
        if (!a.uniform_box) {
            lower[k] = a.lower[k];
            width[k] = a.width[k];
        }
    }
    box.lower = lower;
    box.width = width;
    box.lo0 = a.lo0;
    box.w0 = a.w0;
    box.uniform = a.uniform_box != 0;
}

// cache values of point xs (shared, n doubles) into vs (shared, n*A)
template <class R, class Cost>
__device__ void cache_point(const double* xs, R* vs, int n, int family) {
    constexpr int A = Cost::A;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        R t[A];
        Cost::cache(static_cast<R>(xs[k]), k, n, t);
#pragma unroll
        for (int q = 0; q < A; ++q) vs[k * A + q] = t[q];
    }
    (void)family;
}

// The thread's chain-state row: shared memory (G = false) or HBM SoA (G = true)
template <class R, bool G>
struct RowSel;
template <class R>
struct RowSel<R, false> {
    using T = R*;
    static __device__ T make(R* V, int S, const EngineArgs&, size_t) { return V + static_cast<size_t>(threadIdx.x) * S; }
};
template <class R>
struct RowSel<R, true> {
    using T = StridedRow<R>;
    // S = n*A values per row; a warp's 32 rows form one contiguous tile of
    // nv = ceil(S/W) vectors x 32 lanes, so a fold walks its tile
    // sequentially (512 B per vector step: coalesced, and page/TLB-local)
    static __device__ T make(R*, int S, const EngineArgs& a, size_t gtid) {
        const size_t nv = (static_cast<size_t>(S) + T::W - 1) / T::W;
        return T{static_cast<R*>(a.rows) + ((gtid / 32) * nv * 32 + (gtid % 32)) * T::W, 32 * T::W};
    }
};

// ---------------------------------------------------------------------------
// Producer/consumer sweep for small chain counts (v2_pc_kernel)
//
// With few chains a level is one long dependency chain per thread: 100
// trials of ~290 instructions each, with one warp per scheduler and nothing
// to overlap.  But the proposals are independent of the chain's state
// (counter-based streams), so other warps can make them: warps 1..3 of the
// block compute every trial's coordinate, new cached term and acceptance
// draw (the three Philox draws and the glibc-exact term — the bulk of a
// trial's instructions) into a double-buffered shared-memory ring, 32
// trials ahead, while warp 0 runs only what depends on the chain: slot
// write, fold, Metropolis decision.  Each chain's draws, terms and decisions
// are exactly those of sweep().
// ---------------------------------------------------------------------------

template <class R, int A>
struct PcEntry {
    uint64_t m; // acceptance draw (53-bit mantissa integer)
    int32_t d;  // coordinate
    R t[A];     // its new cached value(s)
};

// entries for trials [j0, j0 + jn) of the 32 chains of a group:
// buf[trial][lane], filled by threads 32.. of the block
template <class R, class Cost>
__device__ void pc_produce(PcEntry<R, Cost::A>* buf, int j0, int jn, int n, uint32_t chain_base, uint32_t level,
                           uint32_t ctr0, const Box& box, const PhiloxKeys& keys, int lanes = 32) {
    // (lanes: the group's live chains — a short last group, or V0's single
    // chain, gets no entries for lanes that have no chain)
    const int p = static_cast<int>(threadIdx.x) - 32, np = static_cast<int>(blockDim.x) - 32;
    const double idx_scale = static_cast<double>(n) * 0x1.0p-53;
    for (int e = p; e < lanes * jn; e += np) {
        const int jj = e / lanes, lane = e - jj * lanes;
        const PhiloxChain pc = philox_chain(chain_base + lane, level, keys);
        const uint32_t ctr = ctr0 + 3u * static_cast<uint32_t>(j0 + jj);
        const uint64_t m1 = draw_bits53_fast(ctr, pc, keys);
        const uint64_t m2 = draw_bits53_fast(ctr + 1, pc, keys);
        PcEntry<R, Cost::A> en;
        en.m = draw_bits53_fast(ctr + 2, pc, keys);
        en.d = min(static_cast<int>(static_cast<double>(m1) * idx_scale), n - 1);
        const double x = box.point(en.d, bits_to_uniform(m2));
        bool ok;
        Cost::cache_common(static_cast<R>(x), en.d, n, en.t, ok);
        if (!ok) Cost::cache(static_cast<R>(x), en.d, n, en.t);
        buf[jj * 32 + lane] = en;
    }
}

template <class R, class Cost, int NT>
//  slot: the ring slot (of 3) holding round 0 (updated for the next call);
//  prefilled: round 0 is already there (made during the previous call);
//  prefetch_next: make round 0 of the same chains' next level (counter 0,
//  level + 1) ahead — during the second-to-last round when the last round
//  is short (its few trials would leave the consumer nothing to overlap),
//  else during the last round.
__device__ R pc_sweep(R* row, int n_rt, int family, R E, double temperature, uint32_t chain_base, uint32_t level,
                      uint32_t ctr0, int N, const Box& box, const PhiloxKeys& keys, uint32_t* mask,
                      size_t mask_stride, bool live, PcEntry<R, Cost::A>* buf, int& slot, bool prefilled,
                      bool prefetch_next, int lanes = 32) {
    constexpr int A = Cost::A;
    const int n = NT > 0 ? NT : n_rt;
    const float k2 = metropolis_k2(temperature); // log2(e) / T
    const bool producer = threadIdx.x >= 32;
    const int lane = threadIdx.x & 31;
    const int rounds = (N + 31) / 32;
    auto at = [&](int k) { return buf + ((slot + k) % 3) * 1024; }; // ring slot of round k
    if (!prefilled) {
        if (producer) pc_produce<R, Cost>(at(0), 0, N < 32 ? N : 32, n, chain_base, level, ctr0, box, keys, lanes);
        __syncthreads();
    }
    const bool short_last = rounds > 1 && N - 32 * (rounds - 1) <= 16;
    for (int k = 0; k < rounds; ++k) {
        const int jn = N - 32 * k < 32 ? N - 32 * k : 32;
        if (producer) {
            if (k + 1 < rounds) {
                const int j1 = 32 * (k + 1);
                pc_produce<R, Cost>(at(k + 1), j1, N - j1 < 32 ? N - j1 : 32, n, chain_base, level, ctr0, box, keys,
                                    lanes);
            }
            const bool early = short_last && k + 2 == rounds, late = !short_last && k + 1 == rounds;
            if (prefetch_next && (early || late))
                pc_produce<R, Cost>(at(rounds), 0, N < 32 ? N : 32, n, chain_base, level + 1, 0u, box, keys, lanes);
        } else if (live) {
            const PcEntry<R, A>* cur = at(k);
            uint32_t word = 0;
            // entry j+1 is loaded at the top of trial j (before this trial's
            // row stores, which the compiler cannot move it past), so its
            // shared-memory latency is off the chain's critical path
            PcEntry<R, A> nx = cur[lane];
            for (int j = 0; j < jn; ++j) {
                const PcEntry<R, A> en = nx;
                nx = cur[(j + 1 < jn ? j + 1 : j) * 32 + lane];
                R to[A];
#pragma unroll
                for (int a = 0; a < A; ++a) {
                    to[a] = row[en.d * A + a];
                    row[en.d * A + a] = en.t[a];
                }
                const R trial = Cost::template energy<NT>(row, n, family);
                int r = metropolis_fast<R>(trial, E, k2, metropolis_band(en.m));
                if (__any_sync(__activemask(), r < 0))
                    if (r < 0) r = Accept<R>::exact(static_cast<double>(trial) - static_cast<double>(E), temperature, en.m);
                if (r) {
                    E = trial;
                    word |= 1u << j;
                } else {
#pragma unroll
                    for (int a = 0; a < A; ++a) row[en.d * A + a] = to[a];
                }
            }
            mask[static_cast<size_t>(k) * mask_stride] = word;
        }
        __syncthreads();
    }
    slot = (slot + rounds) % 3; // where a prefetched next round 0 went
    return E;
}

// The consumer of pc_sweep with the deferred fold (engine.cuh, sweep_lazy):
// the ring entry's new term and the replaced term give the interval of the
// energy difference, and the consumer folds only to settle a straddling
// decision and once at the end of the level.  Producers are unchanged.
template <class R, class Cost, int NT>
__device__ R pc_sweep_lazy(R* row, int n_rt, int family, R E, double temperature, uint32_t chain_base,
                           uint32_t level, uint32_t ctr0, int N, const Box& box, const PhiloxKeys& keys,
                           uint32_t* mask, size_t mask_stride, bool live, PcEntry<R, Cost::A>* buf, int& slot,
                           bool prefilled, bool prefetch_next, R rr, R alpha, SweepStats& st, int lanes = 32) {
    using L = LazyOf<typename Cost::Fam>;
    static_assert(Cost::A == 1, "deferred fold: one accumulator");
    const int n = NT > 0 ? NT : n_rt;
    const float k2 = metropolis_k2(temperature);
    const bool producer = threadIdx.x >= 32;
    const int lane = threadIdx.x & 31;
    const int rounds = (N + 31) / 32;
    const R sa = L::sigma > 0 ? alpha : -alpha;
    bool have = true;
    auto at = [&](int k) { return buf + ((slot + k) % 3) * 1024; };
    if (!prefilled) {
        if (producer) pc_produce<R, Cost>(at(0), 0, N < 32 ? N : 32, n, chain_base, level, ctr0, box, keys, lanes);
        __syncthreads();
    }
    const bool short_last = rounds > 1 && N - 32 * (rounds - 1) <= 16;
    for (int k = 0; k < rounds; ++k) {
        const int jn = N - 32 * k < 32 ? N - 32 * k : 32;
        if (producer) {
            if (k + 1 < rounds) {
                const int j1 = 32 * (k + 1);
                pc_produce<R, Cost>(at(k + 1), j1, N - j1 < 32 ? N - j1 : 32, n, chain_base, level, ctr0, box, keys,
                                    lanes);
            }
            const bool early = short_last && k + 2 == rounds, late = !short_last && k + 1 == rounds;
            if (prefetch_next && (early || late))
                pc_produce<R, Cost>(at(rounds), 0, N < 32 ? N : 32, n, chain_base, level + 1, 0u, box, keys, lanes);
        } else if (live) {
            const PcEntry<R, 1>* cur = at(k);
            uint32_t word = 0;
            PcEntry<R, 1> nx = cur[lane];
            for (int j = 0; j < jn; ++j) {
                const PcEntry<R, 1> en = nx;
                nx = cur[(j + 1 < jn ? j + 1 : j) * 32 + lane];
                const R to = row[en.d];
                const MBand b = metropolis_band(en.m);
                const R q = (en.t[0] - to) * sa;
                const R hi = q + rr, lo = q - rr;
                int r = ((hi <= R(0)) | (static_cast<float>(hi) * k2 < b.lo))
                            ? 1
                            : (((lo > R(0)) & (static_cast<float>(lo) * k2 > b.hi)) ? 0 : -1);
                bool settled = false;
                if (__any_sync(__activemask(), r < 0)) {
                    if (__any_sync(__activemask(), (r < 0) & !have)) {
                        const R eo = Cost::template energy<NT>(row, n, family);
                        if (!have) {
                            E = eo;
                            have = true;
                        }
                    }
                    if (r < 0) row[en.d] = en.t[0];
                    const R et = Cost::template energy<NT>(row, n, family);
                    if (r < 0) {
                        int v = metropolis_fast<R>(et, E, k2, b);
                        if (v < 0)
                            v = Accept<R>::exact(static_cast<double>(et) - static_cast<double>(E), temperature, en.m);
                        if (v) E = et;
                        else row[en.d] = to;
                        r = v;
                        settled = true;
                        st.settles += 1;
                    }
                }
                if (r && !settled) {
                    row[en.d] = en.t[0];
                    have = false;
                }
                word |= static_cast<uint32_t>(r) << j;
            }
            mask[static_cast<size_t>(k) * mask_stride] = word;
        }
        __syncthreads();
    }
    if (!producer && live && __any_sync(__activemask(), !have)) {
        const R e = Cost::template energy<NT>(row, n, family);
        if (!have) E = e;
    }
    slot = (slot + rounds) % 3;
    return E;
}

// draw_random_start (engines.cpp:43-46): coordinate k uses draw k of (seed, c, 0)
__device__ __forceinline__ double random_start_coord(const EngineArgs& a, const Box& box,
                                                     uint32_t c, int k) {
    const uint64_t m = draw_bits53(static_cast<uint64_t>(k), c, 0, a.keys);
    return box.point(k, bits_to_uniform(m));
}

// Rebuild the end point of chain `cw` at level l into xs (shared), starting
// from the level's start point already in xs.  Warp 0 only.
static __device__ void replay_winner(const EngineArgs& a, const Box& box, double* xs, int level,
                              int32_t cw, const uint32_t* masks) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const int W = (a.N + 31) / 32;
    const uint64_t ctr0 = (level == 0 && a.random_start) ? static_cast<uint64_t>(a.n) : 0;
    const size_t cl = static_cast<size_t>(cw - a.chain_begin);
    for (int w = 0; w < W; ++w) {
        const uint32_t word = masks[static_cast<size_t>(w) * a.mask_stride + cl];
        const int j = w * 32 + lane;
        const bool acc = j < a.N && ((word >> lane) & 1u);
        int d = -1;
        double xv = 0;
        if (acc) {
            const uint64_t base = ctr0 + 3ull * static_cast<uint64_t>(j);
            const uint64_t m1 = draw_bits53(base, static_cast<uint32_t>(cw), level, a.keys);
            d = coordinate_index(bits_to_uniform(m1), a.n);
            const uint64_t m2 = draw_bits53(base + 1, static_cast<uint32_t>(cw), level, a.keys);
            xv = box.point(d, bits_to_uniform(m2));
        }
        const unsigned am = __ballot_sync(0xffffffffu, acc);
        if (acc) {
            const unsigned same = __match_any_sync(am, d);
            if (31 - __clz(same) == lane) xs[d] = xv; // last accepted write per coordinate
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Multi-GPU level minloc over peer memory (NVLink / NVSwitch)
//
// Every GPU owns a mailbox of 2 (level parity) x world records; a record is
// {seq, e, c, es, cs, x[n]}: the GPU's level winner (energy, global chain),
// its start-scan winner (level 0, random starts) and the winner's end point
// rebuilt by replay_winner.  Block 0 of each GPU stores its record into
// every peer's mailbox (plain stores through the peer mapping, then a
// system-scope fence and a release store of seq = epoch:level+1); every block
// of every GPU then acquires all `world` records of the level from its own
// mailbox and runs the same deterministic selection (better(): energy, then
// smallest global chain), so all GPUs continue from the same x* bit for bit.
// Parity double-buffering is safe for the same reason as cand[]: a GPU can
// only publish level l+2 after every GPU has published level l+1, which each
// does only after it has finished reading level l.
// ---------------------------------------------------------------------------

struct MailHeader {
    unsigned long long seq;
    double e;
    int32_t c;
    int32_t pad0;
    double es;
    int32_t cs;
    int32_t pad1;
};
constexpr size_t kMailHeaderBytes = 48;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

static __device__ void exchange_level(const EngineArgs& a, double* xs, Cand& w, Cand& ws, int l, Cand* scratch) {
    const int n = a.n, tid = threadIdx.x, B = blockDim.x;
    const size_t slot0 = static_cast<size_t>(l & 1) * a.world;
    const unsigned long long tag = (static_cast<unsigned long long>(a.epoch) << 32) | static_cast<unsigned>(l + 1);
    if (blockIdx.x == 0) {
        for (int p = 0; p < a.world; ++p) {
            char* rec = a.mail_peers[p] + (slot0 + a.rank) * a.rec_stride;
            double* rx = reinterpret_cast<double*>(rec + kMailHeaderBytes);
            for (int k = tid; k < n; k += B) rx[k] = xs[k];
            if (tid == 0) {
                MailHeader* h = reinterpret_cast<MailHeader*>(rec);
                h->e = w.e;
                h->c = w.c;
                h->es = ws.e;
                h->cs = ws.c;
            }
        }
        __threadfence_system();
        __syncthreads();
        if (tid == 0)
            for (int p = 0; p < a.world; ++p)
                st_release_sys(reinterpret_cast<unsigned long long*>(a.mail_peers[p] + (slot0 + a.rank) * a.rec_stride),
                               tag);
    }
    // acquire the level's records from this GPU's own mailbox
    Cand g = empty_cand(), gs = empty_cand();
    if (tid < a.world) {
        const char* rec = a.mail_self + (slot0 + tid) * a.rec_stride;
        const long long t0 = clock64();
        while (ld_acquire_sys(reinterpret_cast<const unsigned long long*>(rec)) != tag) {
            // a peer never arrived: report instead of hanging, and once the
            // run is known to be broken stop waiting at the later levels
            if (clock64() - t0 > a.spin_limit || *reinterpret_cast<volatile int*>(a.error_flag)) {
                atomicExch(a.error_flag, 1);
                break;
            }
        }
        const volatile MailHeader* h = reinterpret_cast<const volatile MailHeader*>(rec);
        g = Cand{h->e, h->c, tid};
        gs = Cand{h->es, h->cs, tid};
    }
    g = block_argmin(g, scratch);
    if (l == 0 && a.random_start) gs = block_argmin(gs, scratch);
    const volatile double* rx =
        reinterpret_cast<const volatile double*>(a.mail_self + (slot0 + g.aux) * a.rec_stride + kMailHeaderBytes);
    for (int k = tid; k < n; k += B) xs[k] = rx[k];
    __syncthreads();
    w = g;
    if (l == 0 && a.random_start) ws = gs;
}

// ---------------------------------------------------------------------------
// V2 persistent kernel
// ---------------------------------------------------------------------------

// Chain-pair traits: Cost = SepCost<float, F> runs two chains per thread
// (sweep_pair); everything else one chain per thread (sweep).
template <class Cost>
struct PairOf {
    static constexpr bool value = false;
};
template <template <class> class F>
struct PairOf<SepCost<float, F>> {
    static constexpr bool value = true;
    template <int NT>
    static __device__ void run(float* row, int n, float& eA, float& eB, double T, uint32_t cA, uint32_t cB,
                               uint32_t level, uint32_t ctr, int N, const Box& box, const PhiloxKeys& keys,
                               uint32_t* mA, uint32_t* mB, size_t ms) {
        sweep_pair<F, NT>(row, n, eA, eB, T, cA, cB, level, ctr, N, box, keys, mA, mB, ms);
    }
    template <int NT>
    static __device__ void run_x(float* row, int n, float& eA, float& eB, double T, uint32_t cA, uint32_t cB,
                                 uint32_t ctr, int N, const Box& box, const PhiloxKeys& keys, double* xa, double* xb,
                                 size_t xs) {
        sweep_pair<F, NT, true>(row, n, eA, eB, T, cA, cB, 0u, ctr, N, box, keys, nullptr, nullptr, 0, xa, xb, xs);
    }
    template <int NT>
    static __device__ void energy(const float* row, int n, float& eA, float& eB) {
        pair_energy<F<float>, NT>(row, n, eA, eB);
    }
};

// deferred-fold capability of a cost (SepCost of a LazyOf family)
template <class Cost>
struct LazyCost {
    static constexpr bool value = false;
};
template <class R, template <class> class F>
struct LazyCost<SepCost<R, F>> {
    static constexpr bool value = LazyOf<F<R>>::value;
    template <class T>
    using Fam = F<T>;
    static double radius(int n, const double* lo, const double* hi) {
        if constexpr (LazyOf<F<R>>::value) return lazy_radius<R, F>(n, lo, hi);
        else return -1.0;
    }
    static double alpha(int n) {
        if constexpr (LazyOf<F<R>>::value) return LazyOf<F<R>>::alpha(n);
        else return 0.0;
    }
};

// LZ: the deferred-fold sweep (sweep_lazy; Cost = SepCost of a LazyOf family)
template <class R, class Cost, int NT, bool G, bool PAIR, bool PC = false, bool LZ = false, bool UB = false>
__device__ __forceinline__ void v2_body(const EngineArgs& a) {
    constexpr int A = Cost::A;
    fn_param_init<Cost>(a.fparam);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::grid_group grid = cg::this_grid();
    const int B = blockDim.x, tid = threadIdx.x;
    const int n = a.n;
    Smem sm{smem_raw};
    // pair rows hold 2 n A interleaved values (chains A and B of the pair);
    // producer/consumer blocks keep rows for their consumer warp only
    const int S = G ? n * A : row_stride<R>(PAIR ? 2 * n : n, A);
    R* V = G ? nullptr : sm.take<R>(static_cast<size_t>(S) * (PC ? 32 : B));
    PcEntry<R, A>* pcbuf = PC ? sm.take<PcEntry<R, A>>(3 * 32 * 32) : nullptr;
    double* xs = sm.take<double>(n);
    R* vs = sm.take<R>(static_cast<size_t>(n) * A);
    double* lower = a.uniform_box ? nullptr : sm.take<double>(n);
    double* width = a.uniform_box ? nullptr : sm.take<double>(n);
    Cand* scratch = sm.take<Cand>(34);
    SharedScalars* sh = sm.take<SharedScalars>(1);

    Box box;
    load_box<R, Cost>(a, lower, width, box);
    for (int k = tid; k < n; k += B) xs[k] = a.start[k];
    __syncthreads();
    cache_point<R, Cost>(xs, vs, n, a.family);
    __syncthreads();
    if (tid == 0) {
        sh->estar = static_cast<double>(Cost::template energy<NT>(vs, n, a.family));
        sh->best_f = __longlong_as_double(0x7ff0000000000000ll);
        sh->best_c = 0;
        sh->fold_mode = 0;
        sh->lv_settles = 0;
        sh->lv_chains = 0;
    }
    __syncthreads();

    const size_t total_threads = static_cast<size_t>(gridDim.x) * B;
    const size_t gtid = static_cast<size_t>(blockIdx.x) * B + tid;
    const size_t W = static_cast<size_t>((a.N + 31) / 32);
    const size_t mask_buf = W * a.mask_stride;
    const auto row = RowSel<R, G>::make(V, S, a, gtid);
    SweepStats st{0, 0};
    int pc_slot = 0;            // producer/consumer ring state (PC mode)
    bool pc_prefilled = false;

    for (int l = 0; l < a.levels; ++l) {
        const double temperature = a.temps[l];
        const R estar = static_cast<R>(sh->estar);
        uint32_t* masks = a.masks + static_cast<size_t>(l & 1) * mask_buf;
        Cand best = empty_cand(), sbest = empty_cand();
        if constexpr (PC) {
            // warp 0 consumes (one chain per lane), warps 1..3 produce the
            // proposals; one group of 32 chains per block and round
            const int lane = tid & 31;
            const bool consumer = tid < 32;
            for (size_t g = blockIdx.x; g * 32 < a.chains_local; g += gridDim.x) {
                const size_t cl = g * 32 + lane;
                const bool live = consumer && cl < a.chains_local;
                const int glanes = static_cast<int>(a.chains_local - g * 32 < 32 ? a.chains_local - g * 32 : 32);
                const uint32_t c = static_cast<uint32_t>(a.chain_begin + (cl < a.chains_local ? cl : g * 32));
                R* prow = V + static_cast<size_t>(lane) * S;
                R e = 0;
                uint32_t ctr = 0;
                if (l == 0 && a.random_start) {
                    if (live) {
                        for (int k = 0; k < n; ++k) {
                            R t[A];
                            Cost::cache(static_cast<R>(random_start_coord(a, box, c, k)), k, n, t);
#pragma unroll
                            for (int q = 0; q < A; ++q) prow[k * A + q] = t[q];
                        }
                        e = Cost::template energy<NT>(prow, n, a.family);
                        st.draws += static_cast<uint64_t>(n);
                        const Cand s1 = start_cand(static_cast<double>(e), static_cast<int32_t>(c));
                        if (better(s1, sbest)) sbest = s1;
                    }
                    ctr = static_cast<uint32_t>(n);
                } else if (live) {
                    for (int k = 0; k < n * A; ++k) prow[k] = vs[k];
                    e = estar;
                }
                if (l == 0 && live) st.evals += 1; // the start evaluation (engines.cpp:157)
                // one chain group per block: the producers make the next
                // level's first round during this level's last one
                const bool one_group = static_cast<size_t>(gridDim.x) * 32 >= a.chains_local;
                if constexpr (LZ)
                    e = pc_sweep_lazy<R, Cost, NT>(prow, n, a.family, e, temperature,
                                                   static_cast<uint32_t>(a.chain_begin + g * 32), static_cast<uint32_t>(l),
                                                   ctr, a.N, box, a.keys, masks + cl, a.mask_stride, live, pcbuf, pc_slot,
                                                   one_group && pc_prefilled, one_group && l + 1 < a.levels,
                                                   static_cast<R>(a.lazy_r), static_cast<R>(a.lazy_alpha), st, glanes);
                else
                    e = pc_sweep<R, Cost, NT>(prow, n, a.family, e, temperature, static_cast<uint32_t>(a.chain_begin + g * 32),
                                              static_cast<uint32_t>(l), ctr, a.N, box, a.keys, masks + cl, a.mask_stride,
                                              live, pcbuf, pc_slot, one_group && pc_prefilled,
                                              one_group && l + 1 < a.levels, glanes);
                pc_prefilled = one_group && l + 1 < a.levels;
                if (live) {
                    st.evals += static_cast<uint64_t>(a.N);
                    st.draws += 3ull * static_cast<uint64_t>(a.N);
                    const Cand mine{static_cast<double>(e), static_cast<int32_t>(c), 0};
                    if (better(mine, best)) best = mine;
                }
            }
        } else if constexpr (PAIR && LZ) {
            // deferred fold on chain pairs: a warp takes 64 chains of the
            // level at a time (dynamic assignment, as in the one-chain
            // kernel below): lane l runs chains base + l (A) and base + 32 + l
            // (B); idle halves sweep a duplicate of chain `base` (identical
            // bits, nothing recorded; sweep_pair's mask words for it are the
            // live lane's own values)
            const bool fold_mode = sh->fold_mode;
            const uint64_t settles0 = st.settles;
            unsigned long long my_chains = 0;
            if (blockIdx.x == 0 && tid == 0) a.work[(l + 1) & 1] = 0;
            unsigned long long* wc = a.work + (l & 1);
            const int lane = tid & 31;
            float* prow = reinterpret_cast<float*>(row);
            for (;;) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(wc, 64ull);
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base >= a.chains_local) break;
                const bool vA = base + lane < a.chains_local, vB = base + 32 + lane < a.chains_local;
                const size_t clA = vA ? base + lane : base, clB = vB ? base + 32 + lane : base;
                const uint32_t cA = static_cast<uint32_t>(a.chain_begin + clA);
                const uint32_t cB = static_cast<uint32_t>(a.chain_begin + clB);
                float eA, eB;
                uint32_t ctr = 0;
                if (l == 0 && a.random_start) {
                    for (int k = 0; k < n; ++k) {
                        float ta[A], tb[A];
                        Cost::cache(static_cast<float>(random_start_coord(a, box, cA, k)), k, n, ta);
                        Cost::cache(static_cast<float>(random_start_coord(a, box, cB, k)), k, n, tb);
#pragma unroll
                        for (int q = 0; q < A; ++q) {
                            prow[2 * (k * A + q)] = ta[q];
                            prow[2 * (k * A + q) + 1] = tb[q];
                        }
                    }
                    PairOf<Cost>::template energy<NT>(prow, n, eA, eB);
                    ctr = static_cast<uint32_t>(n);
                    st.draws += static_cast<uint64_t>(n) * (vA + vB);
                    const Cand s1 = start_cand(static_cast<double>(eA), static_cast<int32_t>(cA));
                    if (vA && better(s1, sbest)) sbest = s1;
                    const Cand s2 = start_cand(static_cast<double>(eB), static_cast<int32_t>(cB));
                    if (vB && better(s2, sbest)) sbest = s2;
                } else {
                    unsigned long long* u = reinterpret_cast<unsigned long long*>(prow);
                    const float* vf = reinterpret_cast<const float*>(vs);
                    for (int e = 0; e < n * A; ++e) u[e] = f2_make(vf[e], vf[e]).v;
                    eA = eB = static_cast<float>(estar);
                }
                if (l == 0) st.evals += vA + vB; // the start evaluations (engines.cpp:157)
                if (!fold_mode) {
                    if constexpr (LazyCost<Cost>::value)
                        sweep_lazy_pair<LazyCost<Cost>::template Fam, NT>(
                            prow, n, eA, eB, temperature, cA, cB, static_cast<uint32_t>(l), ctr, a.N, box, a.keys,
                            vA ? masks + clA : nullptr, vB ? masks + clB : nullptr, a.mask_stride, st,
                            static_cast<float>(a.lazy_r), static_cast<float>(a.lazy_alpha), vA, vB);
                    my_chains += vA + vB;
                } else {
                    PairOf<Cost>::template run<NT>(prow, n, eA, eB, temperature, cA, cB, static_cast<uint32_t>(l), ctr,
                                                   a.N, box, a.keys, masks + clA, masks + clB, a.mask_stride);
                }
                st.evals += static_cast<uint64_t>(a.N) * (vA + vB);
                st.draws += 3ull * static_cast<uint64_t>(a.N) * (vA + vB);
                const Cand m1{static_cast<double>(eA), static_cast<int32_t>(cA), 0};
                if (vA && better(m1, best)) best = m1;
                const Cand m2{static_cast<double>(eB), static_cast<int32_t>(cB), 0};
                if (vB && better(m2, best)) best = m2;
            }
            if (!fold_mode) {
                atomicAdd(&sh->lv_settles, static_cast<unsigned long long>(st.settles - settles0));
                atomicAdd(&sh->lv_chains, my_chains);
            }
        } else if constexpr (PAIR) {
            // pair p = chains p and p + P (P = ceil(C/2)); an odd count leaves
            // the last pair's chain B a duplicate whose results are dropped
            // (its accept bits land in the padding columns of masks)
            const size_t P = (a.chains_local + 1) / 2;
            float* prow = reinterpret_cast<float*>(row);
            for (size_t p = gtid; p < P; p += total_threads) {
                const size_t clB = p + P;
                const bool vB = clB < a.chains_local;
                const uint32_t cA = static_cast<uint32_t>(a.chain_begin + p);
                const uint32_t cB = static_cast<uint32_t>(a.chain_begin + (vB ? clB : p));
                float eA, eB;
                uint32_t ctr = 0;
                if (l == 0 && a.random_start) {
                    for (int k = 0; k < n; ++k) {
                        float ta[A], tb[A];
                        Cost::cache(static_cast<float>(random_start_coord(a, box, cA, k)), k, n, ta);
                        Cost::cache(static_cast<float>(random_start_coord(a, box, cB, k)), k, n, tb);
#pragma unroll
                        for (int q = 0; q < A; ++q) {
                            prow[2 * (k * A + q)] = ta[q];
                            prow[2 * (k * A + q) + 1] = tb[q];
                        }
                    }
                    PairOf<Cost>::template energy<NT>(prow, n, eA, eB);
                    ctr = static_cast<uint32_t>(n);
                    st.draws += static_cast<uint64_t>(n) * (vB ? 2 : 1);
                    const Cand s1 = start_cand(static_cast<double>(eA), static_cast<int32_t>(cA));
                    if (better(s1, sbest)) sbest = s1;
                    const Cand s2 = start_cand(static_cast<double>(eB), static_cast<int32_t>(cB));
                    if (vB && better(s2, sbest)) sbest = s2;
                } else {
                    unsigned long long* u = reinterpret_cast<unsigned long long*>(prow);
                    const float* vf = reinterpret_cast<const float*>(vs);
                    for (int e = 0; e < n * A; ++e) u[e] = f2_make(vf[e], vf[e]).v;
                    eA = eB = static_cast<float>(estar);
                }
                if (l == 0) st.evals += vB ? 2 : 1; // the start evaluations (engines.cpp:157)
                PairOf<Cost>::template run<NT>(prow, n, eA, eB, temperature, cA, cB, static_cast<uint32_t>(l), ctr,
                                               a.N, box, a.keys, masks + p, masks + clB, a.mask_stride);
                st.evals += static_cast<uint64_t>(a.N) * (vB ? 2 : 1);
                st.draws += 3ull * static_cast<uint64_t>(a.N) * (vB ? 2 : 1);
                const Cand m1{static_cast<double>(eA), static_cast<int32_t>(cA), 0};
                if (better(m1, best)) best = m1;
                const Cand m2{static_cast<double>(eB), static_cast<int32_t>(cB), 0};
                if (vB && better(m2, best)) best = m2;
            }
        } else {
        // deferred fold: a block whose exact settles passed 2% of its trials
        // (each costs the warp two folds) sweeps with a fold per trial from
        // then on — temperatures only fall along the ladder, and the settle
        // rate with them (large n at low T); both sweeps are exact
        const bool fold_mode = LZ && sh->fold_mode;
        const uint64_t settles0 = st.settles;
        unsigned long long my_chains = 0;
        // live == false (deferred fold only): an idle lane of the last
        // group sweeps a duplicate of a live chain so the warp stays whole;
        // nothing of it is recorded
        auto one_chain = [&](size_t cl, bool live) {
            const uint32_t c = static_cast<uint32_t>(a.chain_begin + cl);
            const SweepStats st0 = st; // restored for an idle lane
            R e;
            uint32_t ctr = 0;
            if (l == 0 && a.random_start) {
                for (int k = 0; k < n; ++k) {
                    R t[A];
                    Cost::cache(static_cast<R>(random_start_coord(a, box, c, k)), k, n, t);
#pragma unroll
                    for (int q = 0; q < A; ++q) row[k * A + q] = t[q];
                }
                e = row_energy<Cost, NT>(row, n, a.family);
                ctr = static_cast<uint32_t>(n);
                st.draws += static_cast<uint64_t>(n);
                const Cand s = start_cand(static_cast<double>(e), static_cast<int32_t>(c));
                if (live && better(s, sbest)) sbest = s;
            } else {
                if constexpr (G) {
                    // HBM rows: whole 16-byte vectors (a warp writes 512
                    // contiguous bytes per store); the padding of the last
                    // vector is never read
                    using V = Vec16<R>;
                    for (int q = 0; q < (n * A + V::W - 1) / V::W; ++q) {
                        typename V::T v;
                        R* pv = reinterpret_cast<R*>(&v);
#pragma unroll
                        for (int i = 0; i < V::W; ++i) pv[i] = q * V::W + i < n * A ? vs[q * V::W + i] : R(0);
                        *reinterpret_cast<typename V::T*>(row.p + static_cast<size_t>(q) * row.s) = v;
                    }
                } else {
                    for (int k = 0; k < n * A; ++k) row[k] = vs[k];
                }
                e = estar;
            }
            if (l == 0) st.evals += 1; // the start evaluation (engines.cpp:157)
            bool lazy = false;
            if constexpr (LZ) lazy = !fold_mode;
            if (lazy) {
                if constexpr (LZ)
                    e = sweep_lazy<R, Cost, NT, decltype(row), UB>(row, n, a.family, e, temperature, c,
                                                                   static_cast<uint32_t>(l), ctr,
                                                a.N, box, a.keys, live ? masks + cl : nullptr, a.mask_stride,
                                                nullptr, 0, st, static_cast<R>(a.lazy_r),
                                                static_cast<R>(a.lazy_alpha));
                my_chains += live;
            } else {
                e = sweep<R, Cost, NT>(row, n, a.family, e, temperature, c, static_cast<uint32_t>(l), ctr,
                                       a.N, box, a.keys, live ? masks + cl : nullptr, a.mask_stride, nullptr, 0,
                                       st);
            }
            const Cand mine{static_cast<double>(e), static_cast<int32_t>(c), 0};
            if (live && better(mine, best)) best = mine;
            if (!live) st = st0;
        };
        if constexpr (LZ) {
            // Dynamic chain assignment: each warp takes the next 32 chains
            // of the level from a global counter (a chain's sweep time varies
            // with its exact-fold settles and the scheduler), so the level
            // ends one chain sweep after the last grab instead of after the
            // slowest warp's fixed share.  Level l uses work[l & 1]; block 0
            // clears the other counter, whose last use (level l - 1) ended
            // before this level's grid barrier and whose next use (level
            // l + 1) starts after the next one.
            if (blockIdx.x == 0 && tid == 0) a.work[(l + 1) & 1] = 0;
            unsigned long long* wc = a.work + (l & 1);
            const int lane = tid & 31;
            for (;;) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(wc, 32ull);
                base = __shfl_sync(0xffffffffu, base, 0);
                if (base >= a.chains_local) break;
                const bool live = base + lane < a.chains_local;
                one_chain(static_cast<size_t>(live ? base + lane : base), live);
            }
            if (!fold_mode) {
                atomicAdd(&sh->lv_settles, static_cast<unsigned long long>(st.settles - settles0));
                atomicAdd(&sh->lv_chains, my_chains);
            }
        } else {
            for (size_t cl = gtid; cl < a.chains_local; cl += total_threads) one_chain(cl, true);
        }
        }
        // block argmin -> cand[l&1][block]
        best = block_argmin(best, scratch);
        if (l == 0 && a.random_start) sbest = block_argmin(sbest, scratch);
        if (LZ && tid == 0) {
            if (a.lazy_adapt && sh->lv_settles * 50ull > sh->lv_chains * static_cast<unsigned long long>(a.N))
                sh->fold_mode = 1;
            sh->lv_settles = 0;
            sh->lv_chains = 0;
        }
        if (tid == 0) {
            a.cand[static_cast<size_t>(l & 1) * gridDim.x + blockIdx.x] = best;
            if (l == 0 && a.random_start) a.cand_start[blockIdx.x] = sbest;
        }
        grid.sync();

        // every block: global argmin over the block candidates
        Cand w = empty_cand(), ws = empty_cand();
        for (int i = tid; i < static_cast<int>(gridDim.x); i += B) {
            const Cand c = a.cand[static_cast<size_t>(l & 1) * gridDim.x + i];
            if (better(c, w)) w = c;
            if (l == 0 && a.random_start) {
                const Cand s = a.cand_start[i];
                if (better(s, ws)) ws = s;
            }
        }
        w = block_argmin(w, scratch);
        if (l == 0 && a.random_start) ws = block_argmin(ws, scratch);

        // the level's start point of the winner -> xs
        if (l == 0 && a.random_start)
            for (int k = tid; k < n; k += B) xs[k] = random_start_coord(a, box, w.c, k);
        __syncthreads();
        replay_winner(a, box, xs, l, w.c, masks);
        __syncthreads();
        if (a.world > 1) exchange_level(a, xs, w, ws, l, scratch); // the multi-GPU minloc (w, ws global)
        // level-0 best-so-far: the start scan of engines.cpp:161-167 — a strict
        // `<` against +inf in chain order, so NaN and +inf starts never count
        // (start_cand); with no qualifying start best_f stays +inf, the chain
        // 0 and best_x NaN (the reference leaves best_x empty)
        if (l == 0 && blockIdx.x == 0) {
            const bool have = a.random_start ? ws.c != INT32_MAX : sh->estar < kInf;
            for (int k = tid; k < n; k += B)
                a.best_x[k] = !have ? __longlong_as_double(0x7ff8000000000000ll)
                              : a.random_start ? random_start_coord(a, box, ws.c, k) : a.start[k];
            __syncthreads(); // every thread has read sh->estar
            if (tid == 0 && have) {
                sh->best_f = a.random_start ? ws.e : sh->estar;
                sh->best_c = a.random_start ? ws.c : 0;
            }
        }
        cache_point<R, Cost>(xs, vs, n, a.family);
        __syncthreads();
        if (tid == 0) sh->estar = w.e;
        __syncthreads();
        if (blockIdx.x == 0) {
            const bool improve = w.e < sh->best_f; // engines.cpp:193 (strict)
            if (improve)
                for (int k = tid; k < n; k += B) a.best_x[k] = xs[k];
            __syncthreads();
            if (tid == 0) {
                if (improve) {
                    sh->best_f = w.e;
                    sh->best_c = w.c;
                }
                a.trace_best[l] = sh->best_f;
                if (a.level_winner) a.level_winner[l] = w.c;
                if (a.level_winner_f) a.level_winner_f[l] = w.e;
            }
            __syncthreads();
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        a.out_scalars->best_f = sh->best_f;
        a.out_scalars->best_chain = sh->best_c;
    }
    // accounting: device-side totals of evaluations and draws
    __shared__ unsigned long long red_e, red_d, red_s;
    if (tid == 0) { red_e = 0; red_d = 0; red_s = 0; }
    __syncthreads();
    atomicAdd(&red_e, static_cast<unsigned long long>(st.evals));
    atomicAdd(&red_d, static_cast<unsigned long long>(st.draws));
    if (LZ) atomicAdd(&red_s, static_cast<unsigned long long>(st.settles));
    __syncthreads();
    if (tid == 0) {
        atomicAdd(&a.out_scalars->evaluations, red_e);
        atomicAdd(&a.out_scalars->rng_draws, red_d);
        if (LZ) atomicAdd(&a.out_scalars->exact_settles, red_s);
    }
}

template <class R, class Cost, int NT, bool G>
__global__ void __launch_bounds__(PSA_V2_MAX_THREADS, PSA_V2_MIN_BLOCKS) v2_kernel(const EngineArgs a) {
    v2_body<R, Cost, NT, G, false>(a);
}

// deferred fold on chain pairs (sweep_lazy_pair), shared-memory pair rows
template <class R, class Cost, int NT>
__global__ void __launch_bounds__(128, 2) v2_lazy_pair_kernel(const EngineArgs a) {
    v2_body<R, Cost, NT, false, true, false, true>(a);
}

// deferred fold (sweep_lazy): one chain per thread, rows in shared memory or
// HBM; UB: uniform box (the benchmark shapes), resolved at compile time
template <class R, class Cost, int NT, bool G, bool UB = false>
__global__ void __launch_bounds__(PSA_V2_MAX_THREADS, PSA_V2_MIN_BLOCKS) v2_lazy_kernel(const EngineArgs a) {
    v2_body<R, Cost, NT, G, false, false, true, UB>(a);
}

// producer/consumer blocks with the deferred-fold consumer (pc_sweep_lazy)
template <class R, class Cost, int NT>
__global__ void __launch_bounds__(256, 2) v2_lazy_pc_kernel(const EngineArgs a) {
    v2_body<R, Cost, NT, false, false, true, true>(a);
}

// producer/consumer blocks for small chain counts: warp 0 consumes, warps
// 1..3 produce (pc_sweep)
template <class R, class Cost, int NT>
__global__ void __launch_bounds__(256, 2) v2_pc_kernel(const EngineArgs a) {
    v2_body<R, Cost, NT, false, false, true>(a);
}

// chain pairs: 800+ bytes of shared state per thread at n = 100 leave room
// for 2 blocks of 128 per SM, so the register budget is 255
template <class R, class Cost, int NT>
__global__ void __launch_bounds__(128, 2) v2_pair_kernel(const EngineArgs a) {
    v2_body<R, Cost, NT, false, true>(a);
}

// ---------------------------------------------------------------------------
// V1 asynchronous kernel (engines.cpp:66-123)
// Each thread runs whole chains through the full ladder on stream (seed,c,0).
// Per level, the block folds its chains' running best into
// trace_cand[l][block]; at the end each thread's best end state goes to
// cand[gtid] with its point in xbest[gtid].  v1_finalize reduces both.
// ---------------------------------------------------------------------------

template <class R, class Cost, int NT, bool G>
__global__ void __launch_bounds__(256) v1_kernel(const EngineArgs a) {
    constexpr int A = Cost::A;
    fn_param_init<Cost>(a.fparam);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int B = blockDim.x, tid = threadIdx.x;
    const int n = a.n;
    Smem sm{smem_raw};
    const int S = G ? n * A : row_stride<R>(n, A);
    R* V = G ? nullptr : sm.take<R>(static_cast<size_t>(S) * B);
    double* xs = sm.take<double>(n);
    R* vs = sm.take<R>(static_cast<size_t>(n) * A);
    double* lower = a.uniform_box ? nullptr : sm.take<double>(n);
    double* width = a.uniform_box ? nullptr : sm.take<double>(n);
    Cand* scratch = sm.take<Cand>(34);
    SharedScalars* sh = sm.take<SharedScalars>(1);

    Box box;
    load_box<R, Cost>(a, lower, width, box);
    for (int k = tid; k < n; k += B) xs[k] = a.start[k];
    __syncthreads();
    cache_point<R, Cost>(xs, vs, n, a.family);
    __syncthreads();
    if (tid == 0) sh->estar = static_cast<double>(Cost::template energy<NT>(vs, n, a.family));
    __syncthreads();

    const size_t total_threads = static_cast<size_t>(gridDim.x) * B;
    const size_t gtid = static_cast<size_t>(blockIdx.x) * B + tid;
    const size_t rounds = (a.chains_local + total_threads - 1) / total_threads;
    const auto row = RowSel<R, G>::make(V, S, a, gtid);
    // the chain's double-precision point: written once per accepted move, so
    // it lives in HBM (SoA, stride = threads) and leaves shared memory to the
    // cached terms the fold reads on every trial
    double* xrow = a.xrows + gtid;
    const size_t xst = a.threads;
    SweepStats st{0, 0};
    Cand mybest = empty_cand();

    for (size_t r = 0; r < rounds; ++r) {
        const size_t cl = gtid + r * total_threads;
        const bool active = cl < a.chains_local;
        const uint32_t c = static_cast<uint32_t>(a.chain_begin + cl);
        R e = 0;
        uint32_t ctr = 0;
        if (active) {
            if (a.random_start) {
                for (int k = 0; k < n; ++k) {
                    const double xk = random_start_coord(a, box, c, k);
                    xrow[k * xst] = xk;
                    R t[A];
                    Cost::cache(static_cast<R>(xk), k, n, t);
#pragma unroll
                    for (int q = 0; q < A; ++q) row[k * A + q] = t[q];
                }
                e = row_energy<Cost, NT>(row, n, a.family);
                ctr = static_cast<uint32_t>(n);
                st.draws += static_cast<uint64_t>(n);
            } else {
                for (int k = 0; k < n; ++k) xrow[k * xst] = xs[k];
                for (int k = 0; k < n * A; ++k) row[k] = vs[k];
                e = static_cast<R>(sh->estar);
            }
            st.evals += 1;
        }
        double chain_best = static_cast<double>(e);
        for (int l = 0; l < a.levels; ++l) {
            if (active) {
                e = sweep<R, Cost, NT>(row, n, a.family, e, a.temps[l], c, 0, ctr, a.N, box, a.keys,
                                       nullptr, 0, xrow, xst, st);
                ctr += 3u * static_cast<uint32_t>(a.N);
                // std::min(chain_best, energy) (engines.cpp:94)
                if (static_cast<double>(e) < chain_best) chain_best = static_cast<double>(e);
            }
            // trace: min over chains of chain_best; std::min(m, v) skips NaN and
            // keeps the first (smallest chain) among equal values
            Cand tv = active && !is_nan(chain_best)
                          ? Cand{chain_best, static_cast<int32_t>(c), 0}
                          : empty_cand();
            tv = block_argmin(tv, scratch);
            if (tid == 0) {
                Cand* slot = &a.trace_cand[static_cast<size_t>(l) * gridDim.x + blockIdx.x];
                if (r == 0 || better(tv, *slot)) *slot = tv;
            }
        }
        if (active) {
            const Cand mine{static_cast<double>(e), static_cast<int32_t>(c), static_cast<int32_t>(gtid)};
            if (better(mine, mybest)) {
                mybest = mine;
                for (int k = 0; k < n; ++k)
                    a.xbest[gtid * static_cast<size_t>(n) + k] = xrow[k * xst];
            }
        }
    }
    const Cand b = block_argmin(mybest, scratch);
    if (tid == 0) a.cand[blockIdx.x] = b;

    __shared__ unsigned long long red_e, red_d;
    if (tid == 0) { red_e = 0; red_d = 0; }
    __syncthreads();
    atomicAdd(&red_e, static_cast<unsigned long long>(st.evals));
    atomicAdd(&red_d, static_cast<unsigned long long>(st.draws));
    __syncthreads();
    if (tid == 0) {
        atomicAdd(&a.out_scalars->evaluations, red_e);
        atomicAdd(&a.out_scalars->rng_draws, red_d);
    }
}

// V1 with producer/consumer warps (small chain counts, §2.4b): warp 0 runs
// 32 chains (one per lane) through the whole ladder, warps 1..3 make every
// trial's proposal 32 trials ahead (pc_produce on stream (seed, c, 0), whose
// counter runs on across levels).  The lanes move in lockstep, so each
// level's trace candidate is a warp argmin; points of the chains are kept in
// HBM and updated on accepted moves (the producers also store the proposed
// coordinate value).
template <class R, int A>
struct PcEntryX {
    PcEntry<R, A> p;
    double x; // the proposed coordinate value (compute_neighbour)
};

template <class R, class Cost>
__device__ void pc_produce_x(PcEntryX<R, Cost::A>* buf, long long j0, int jn, int n, uint32_t chain_base,
                             uint32_t ctr0, const Box& box, const PhiloxKeys& keys, int lanes = 32) {
    const int p = static_cast<int>(threadIdx.x) - 32, np = static_cast<int>(blockDim.x) - 32;
    const double idx_scale = static_cast<double>(n) * 0x1.0p-53;
    for (int e = p; e < lanes * jn; e += np) {
        const int jj = e / lanes, lane = e - jj * lanes;
        const PhiloxChain pc = philox_chain(chain_base + lane, 0u, keys);
        const uint32_t ctr = ctr0 + 3u * static_cast<uint32_t>(j0 + jj);
        const uint64_t m1 = draw_bits53_fast(ctr, pc, keys);
        const uint64_t m2 = draw_bits53_fast(ctr + 1, pc, keys);
        PcEntryX<R, Cost::A> en;
        en.p.m = draw_bits53_fast(ctr + 2, pc, keys);
        en.p.d = min(static_cast<int>(static_cast<double>(m1) * idx_scale), n - 1);
        en.x = box.point(en.p.d, bits_to_uniform(m2));
        bool ok;
        Cost::cache_common(static_cast<R>(en.x), en.p.d, n, en.p.t, ok);
        if (!ok) Cost::cache(static_cast<R>(en.x), en.p.d, n, en.p.t);
        buf[jj * 32 + lane] = en;
    }
}

// LZ: the consumer decides from the deferred-fold interval (sweep_lazy) and
// folds only to settle and at level ends (engines.cpp:90-106 reads the
// chain's energy there); v1_lazy_pc_kernel
template <class R, class Cost, int NT, bool LZ = false>
__global__ void __launch_bounds__(256, 2) v1_pc_kernel(const EngineArgs a) {
    constexpr int A = Cost::A;
    fn_param_init<Cost>(a.fparam);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int B = blockDim.x, tid = threadIdx.x, lane = tid & 31;
    const int n = a.n;
    Smem sm{smem_raw};
    const int S = row_stride<R>(n, A);
    R* V = sm.take<R>(static_cast<size_t>(S) * 32);
    PcEntryX<R, A>* buf = sm.take<PcEntryX<R, A>>(2 * 32 * 32);
    double* xs = sm.take<double>(n);
    R* vs = sm.take<R>(static_cast<size_t>(n) * A);
    double* lower = a.uniform_box ? nullptr : sm.take<double>(n);
    double* width = a.uniform_box ? nullptr : sm.take<double>(n);
    Cand* scratch = sm.take<Cand>(34);
    SharedScalars* sh = sm.take<SharedScalars>(1);

    Box box;
    load_box<R, Cost>(a, lower, width, box);
    for (int k = tid; k < n; k += B) xs[k] = a.start[k];
    __syncthreads();
    cache_point<R, Cost>(xs, vs, n, a.family);
    __syncthreads();
    if (tid == 0) sh->estar = static_cast<double>(Cost::template energy<NT>(vs, n, a.family));
    __syncthreads();

    const bool consumer = tid < 32, producer = !consumer;
    const size_t gslot = static_cast<size_t>(blockIdx.x) * 32 + lane; // this lane's xrows / xbest slot
    const size_t xst = a.threads;
    double* xrow = a.xrows + gslot;
    R* row = V + static_cast<size_t>(lane) * S;
    SweepStats st{0, 0};
    Cand mybest = empty_cand();
    const long long total = static_cast<long long>(a.levels) * a.N; // trials per chain
    const int rounds = static_cast<int>((total + 31) / 32);

    for (size_t g = blockIdx.x; g * 32 < a.chains_local; g += gridDim.x) {
        const size_t cl = g * 32 + lane;
        const bool live = consumer && cl < a.chains_local;
        const uint32_t chain_base = static_cast<uint32_t>(a.chain_begin + g * 32);
        const uint32_t c = static_cast<uint32_t>(a.chain_begin + (cl < a.chains_local ? cl : g * 32));
        R e = 0;
        uint32_t ctr0 = 0;
        if (a.random_start) {
            if (live) {
                for (int k = 0; k < n; ++k) {
                    const double xk = random_start_coord(a, box, c, k);
                    xrow[k * xst] = xk;
                    R t[A];
                    Cost::cache(static_cast<R>(xk), k, n, t);
#pragma unroll
                    for (int q = 0; q < A; ++q) row[k * A + q] = t[q];
                }
                e = Cost::template energy<NT>(row, n, a.family);
                st.draws += static_cast<uint64_t>(n);
            }
            ctr0 = static_cast<uint32_t>(n);
        } else if (live) {
            for (int k = 0; k < n; ++k) xrow[k * xst] = xs[k];
            for (int k = 0; k < n * A; ++k) row[k] = vs[k];
            e = static_cast<R>(sh->estar);
        }
        if (live) st.evals += 1;
        double chain_best = static_cast<double>(e);
        bool have = true; // LZ: e is the exact energy of the row
        const int glanes = static_cast<int>(a.chains_local - g * 32 < 32 ? a.chains_local - g * 32 : 32);
        if (producer)
            pc_produce_x<R, Cost>(buf, 0, total < 32 ? static_cast<int>(total) : 32, n, chain_base, ctr0, box, a.keys,
                                  glanes);
        __syncthreads();
        int level = 0, in_level = 0; // the trial's level and position in it
        float k2 = metropolis_k2(a.temps[0]);
        for (int k = 0; k < rounds; ++k) {
            const long long j0 = 32ll * k;
            const int jn = total - j0 < 32 ? static_cast<int>(total - j0) : 32;
            if (producer) {
                if (k + 1 < rounds) {
                    const long long j1 = j0 + 32;
                    pc_produce_x<R, Cost>(buf + ((k + 1) & 1) * 1024, j1, total - j1 < 32 ? static_cast<int>(total - j1) : 32,
                                          n, chain_base, ctr0, box, a.keys, glanes);
                }
            } else {
                const PcEntryX<R, A>* cur = buf + (k & 1) * 1024;
                PcEntryX<R, A> nx = cur[lane]; // entry j+1 loaded during trial j (pc_sweep)
                for (int j = 0; j < jn; ++j) {
                    const PcEntryX<R, A> en = nx;
                    nx = cur[(j + 1 < jn ? j + 1 : j) * 32 + lane];
                    if constexpr (LZ) {
                        if (live) {
                            using LF = LazyOf<typename Cost::Fam>;
                            const R sa = LF::sigma > 0 ? static_cast<R>(a.lazy_alpha) : -static_cast<R>(a.lazy_alpha);
                            const R rr = static_cast<R>(a.lazy_r);
                            const R to = row[en.p.d];
                            const MBand b = metropolis_band(en.p.m);
                            const R q = (en.p.t[0] - to) * sa;
                            const R hi = q + rr, lo = q - rr;
                            int r = ((hi <= R(0)) | (static_cast<float>(hi) * k2 < b.lo))
                                        ? 1
                                        : (((lo > R(0)) & (static_cast<float>(lo) * k2 > b.hi)) ? 0 : -1);
                            bool settled = false;
                            if (__any_sync(__activemask(), r < 0)) {
                                if (__any_sync(__activemask(), (r < 0) & !have)) {
                                    const R eo = Cost::template energy<NT>(row, n, a.family);
                                    if (!have) {
                                        e = eo;
                                        have = true;
                                    }
                                }
                                if (r < 0) row[en.p.d] = en.p.t[0];
                                const R et = Cost::template energy<NT>(row, n, a.family);
                                if (r < 0) {
                                    int v = metropolis_fast<R>(et, e, k2, b);
                                    if (v < 0)
                                        v = Accept<R>::exact(static_cast<double>(et) - static_cast<double>(e),
                                                             a.temps[level], en.p.m);
                                    if (v) e = et;
                                    else row[en.p.d] = to;
                                    r = v;
                                    settled = true;
                                }
                            }
                            if (r && !settled) {
                                row[en.p.d] = en.p.t[0];
                                have = false;
                            }
                            if (r) xrow[static_cast<size_t>(en.p.d) * xst] = en.x;
                        }
                    } else if (live) {
                        R to[A];
#pragma unroll
                        for (int q = 0; q < A; ++q) {
                            to[q] = row[en.p.d * A + q];
                            row[en.p.d * A + q] = en.p.t[q];
                        }
                        const R trial = Cost::template energy<NT>(row, n, a.family);
                        const double T = a.temps[level];
                        int r = metropolis_fast<R>(trial, e, k2, metropolis_band(en.p.m));
                        if (__any_sync(__activemask(), r < 0))
                            if (r < 0) r = Accept<R>::exact(static_cast<double>(trial) - static_cast<double>(e), T, en.p.m);
                        if (r) {
                            e = trial;
                            xrow[static_cast<size_t>(en.p.d) * xst] = en.x;
                        } else {
#pragma unroll
                            for (int q = 0; q < A; ++q) row[en.p.d * A + q] = to[q];
                        }
                    }
                    if (++in_level == a.N) {
                        if constexpr (LZ) { // the level-end energy is an exact fold
                            if (__any_sync(0xffffffffu, live && !have)) {
                                const R ef = Cost::template energy<NT>(row, n, a.family);
                                if (live && !have) {
                                    e = ef;
                                    have = true;
                                }
                            }
                        }
                        // level end (engines.cpp:90-106): std::min(chain_best, energy),
                        // then the warp's trace candidate (NaN skipped)
                        if (static_cast<double>(e) < chain_best) chain_best = static_cast<double>(e);
                        Cand tv = live && !is_nan(chain_best) ? Cand{chain_best, static_cast<int32_t>(c), 0}
                                                              : empty_cand();
                        tv = warp_argmin(tv);
                        if (lane == 0) {
                            Cand* slot = &a.trace_cand[static_cast<size_t>(level) * gridDim.x + blockIdx.x];
                            if (g == blockIdx.x || better(tv, *slot)) *slot = tv;
                        }
                        in_level = 0;
                        if (++level < a.levels) k2 = metropolis_k2(a.temps[level]);
                    }
                }
            }
            __syncthreads();
        }
        if (live) {
            st.evals += static_cast<uint64_t>(total);
            st.draws += 3ull * static_cast<uint64_t>(total);
            const Cand mine{static_cast<double>(e), static_cast<int32_t>(c), static_cast<int32_t>(gslot)};
            if (better(mine, mybest)) {
                mybest = mine;
                for (int k = 0; k < n; ++k) a.xbest[gslot * static_cast<size_t>(n) + k] = xrow[k * xst];
            }
        }
        __syncthreads();
    }
    const Cand b = block_argmin(mybest, scratch);
    if (tid == 0) a.cand[blockIdx.x] = b;

    __shared__ unsigned long long red_e, red_d;
    if (tid == 0) { red_e = 0; red_d = 0; }
    __syncthreads();
    atomicAdd(&red_e, static_cast<unsigned long long>(st.evals));
    atomicAdd(&red_d, static_cast<unsigned long long>(st.draws));
    __syncthreads();
    if (tid == 0) {
        atomicAdd(&a.out_scalars->evaluations, red_e);
        atomicAdd(&a.out_scalars->rng_draws, red_d);
    }
}

// V1 with chain pairs (binary32 separable families): thread t runs chains p
// and p + P (P = ceil(C/2)) through the whole ladder side by side
// (sweep_pair), each on its own stream (seed, c, 0); per level the block
// folds both chains' running best into the trace candidate.  Points live in
// HBM, one SoA row per chain of the pair (xrows[2][n][threads]).
template <class R, class Cost, int NT>
__global__ void __launch_bounds__(128, 3) v1_pair_kernel(const EngineArgs a) {
    constexpr int A = Cost::A;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int B = blockDim.x, tid = threadIdx.x;
    const int n = a.n;
    Smem sm{smem_raw};
    const int S = row_stride<float>(2 * n, A);
    float* V = sm.take<float>(static_cast<size_t>(S) * B);
    double* xs = sm.take<double>(n);
    float* vs = sm.take<float>(static_cast<size_t>(n) * A);
    double* lower = a.uniform_box ? nullptr : sm.take<double>(n);
    double* width = a.uniform_box ? nullptr : sm.take<double>(n);
    Cand* scratch = sm.take<Cand>(34);
    SharedScalars* sh = sm.take<SharedScalars>(1);

    Box box;
    load_box<float, Cost>(a, lower, width, box);
    for (int k = tid; k < n; k += B) xs[k] = a.start[k];
    __syncthreads();
    cache_point<float, Cost>(xs, vs, n, a.family);
    __syncthreads();
    if (tid == 0) sh->estar = static_cast<double>(Cost::template energy<NT>(vs, n, a.family));
    __syncthreads();

    const size_t total_threads = static_cast<size_t>(gridDim.x) * B;
    const size_t gtid = static_cast<size_t>(blockIdx.x) * B + tid;
    const size_t P = (a.chains_local + 1) / 2;
    const size_t rounds = (P + total_threads - 1) / total_threads;
    float* row = V + static_cast<size_t>(tid) * S;
    const size_t xst = a.threads;
    double* xa = a.xrows + gtid;
    double* xb = a.xrows + static_cast<size_t>(n) * xst + gtid;
    SweepStats st{0, 0};
    Cand mybest = empty_cand();

    for (size_t r = 0; r < rounds; ++r) {
        const size_t p = gtid + r * total_threads;
        const bool active = p < P;
        const bool vB = p + P < a.chains_local;
        const uint32_t cA = static_cast<uint32_t>(a.chain_begin + p);
        const uint32_t cB = static_cast<uint32_t>(a.chain_begin + (vB ? p + P : p));
        float eA = 0, eB = 0;
        uint32_t ctr = 0;
        if (active) {
            if (a.random_start) {
                for (int k = 0; k < n; ++k) {
                    const double ya = random_start_coord(a, box, cA, k), yb = random_start_coord(a, box, cB, k);
                    xa[k * xst] = ya;
                    xb[k * xst] = yb;
                    float ta[A], tb[A];
                    Cost::cache(static_cast<float>(ya), k, n, ta);
                    Cost::cache(static_cast<float>(yb), k, n, tb);
#pragma unroll
                    for (int q = 0; q < A; ++q) {
                        row[2 * (k * A + q)] = ta[q];
                        row[2 * (k * A + q) + 1] = tb[q];
                    }
                }
                PairOf<Cost>::template energy<NT>(row, n, eA, eB);
                ctr = static_cast<uint32_t>(n);
                st.draws += static_cast<uint64_t>(n) * (vB ? 2 : 1);
            } else {
                for (int k = 0; k < n; ++k) {
                    xa[k * xst] = xs[k];
                    xb[k * xst] = xs[k];
                }
                unsigned long long* u = reinterpret_cast<unsigned long long*>(row);
                for (int e = 0; e < n * A; ++e) u[e] = f2_make(vs[e], vs[e]).v;
                eA = eB = static_cast<float>(sh->estar);
            }
            st.evals += vB ? 2 : 1;
        }
        double bestA = eA, bestB = eB;
        for (int l = 0; l < a.levels; ++l) {
            if (active) {
                PairOf<Cost>::template run_x<NT>(row, n, eA, eB, a.temps[l], cA, cB, ctr, a.N, box, a.keys, xa, xb,
                                                 xst);
                ctr += 3u * static_cast<uint32_t>(a.N);
                st.evals += static_cast<uint64_t>(a.N) * (vB ? 2 : 1);
                st.draws += 3ull * static_cast<uint64_t>(a.N) * (vB ? 2 : 1);
                // std::min(chain_best, energy) (engines.cpp:94)
                if (static_cast<double>(eA) < bestA) bestA = eA;
                if (static_cast<double>(eB) < bestB) bestB = eB;
            }
            // trace: min over chains of the running best (std::min skips NaN
            // and keeps the smallest chain among equal values)
            Cand tv = active && !is_nan(bestA) ? Cand{bestA, static_cast<int32_t>(cA), 0} : empty_cand();
            const Cand tb = active && vB && !is_nan(bestB) ? Cand{bestB, static_cast<int32_t>(cB), 0} : empty_cand();
            if (better(tb, tv)) tv = tb;
            tv = block_argmin(tv, scratch);
            if (tid == 0) {
                Cand* slot = &a.trace_cand[static_cast<size_t>(l) * gridDim.x + blockIdx.x];
                if (r == 0 || better(tv, *slot)) *slot = tv;
            }
        }
        if (active) {
            const Cand ma{static_cast<double>(eA), static_cast<int32_t>(cA), static_cast<int32_t>(gtid)};
            if (better(ma, mybest)) {
                mybest = ma;
                for (int k = 0; k < n; ++k) a.xbest[gtid * static_cast<size_t>(n) + k] = xa[k * xst];
            }
            const Cand mb{static_cast<double>(eB), static_cast<int32_t>(cB), static_cast<int32_t>(gtid)};
            if (vB && better(mb, mybest)) {
                mybest = mb;
                for (int k = 0; k < n; ++k) a.xbest[gtid * static_cast<size_t>(n) + k] = xb[k * xst];
            }
        }
    }
    const Cand b = block_argmin(mybest, scratch);
    if (tid == 0) a.cand[blockIdx.x] = b;

    __shared__ unsigned long long red_e, red_d;
    if (tid == 0) { red_e = 0; red_d = 0; }
    __syncthreads();
    atomicAdd(&red_e, static_cast<unsigned long long>(st.evals));
    atomicAdd(&red_d, static_cast<unsigned long long>(st.draws));
    __syncthreads();
    if (tid == 0) {
        atomicAdd(&a.out_scalars->evaluations, red_e);
        atomicAdd(&a.out_scalars->rng_draws, red_d);
    }
}

// f(x_i) through the engine's own cache/energy path (one point per thread)
template <class R, class Cost>
__global__ void probe_evaluate(const EngineArgs a, const double* x, int count, double* out) {
    constexpr int A = Cost::A;
    fn_param_init<Cost>(a.fparam);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* V = reinterpret_cast<R*>(smem_raw);
    const int B = blockDim.x;
    R* row = V + static_cast<size_t>(threadIdx.x) * row_stride<R>(a.n, A);
    const int i = blockIdx.x * B + threadIdx.x;
    if (i >= count) return;
    for (int k = 0; k < a.n; ++k) {
        R t[A];
        Cost::cache(static_cast<R>(x[static_cast<size_t>(i) * a.n + k]), k, a.n, t);
#pragma unroll
        for (int q = 0; q < A; ++q) row[k * A + q] = t[q];
    }
    out[i] = static_cast<double>(Cost::template energy<0>(row, a.n, a.family));
}

// metropolis_sweep (sa_core.cpp:61-79) for ONE caller-held chain — the
// single-chain entry point of the C++ API (parsa::metropolis_sweep); the
// engines run their own fused sweeps.  One thread walks the stream from an
// arbitrary 64-bit counter.  The chain's cached values live in a global row;
// every trial re-folds the whole row, so the energy is chain_energy() of the
// point bit for bit, and the energy carried between trials is the caller's
// double (state.energy), exactly as the reference carries it.
template <class R, class Cost>
__global__ void sweep_one(const EngineArgs a, double* x, R* row, double* energy,
                          unsigned long long* counter, uint32_t chain, uint32_t level,
                          double temperature, int n_steps) {
    constexpr int A = Cost::A;
    fn_param_init<Cost>(a.fparam);
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int n = a.n;
    Box box;
    box.lower = a.lower;
    box.width = a.width;
    box.lo0 = 0;
    box.w0 = 0;
    box.uniform = false;
    for (int k = 0; k < n; ++k) {
        R t[A];
        Cost::cache(static_cast<R>(x[k]), k, n, t);
#pragma unroll
        for (int q = 0; q < A; ++q) row[k * A + q] = t[q];
    }
    double E = *energy;
    unsigned long long ctr = *counter;
    const float k2 = metropolis_k2(temperature); // log2(e) / T
    for (int s = 0; s < n_steps; ++s) {
        const int d = coordinate_index(bits_to_uniform(draw_bits53(ctr, chain, level, a.keys)), n);
        const double xv = box.point(d, bits_to_uniform(draw_bits53(ctr + 1, chain, level, a.keys)));
        const double xold = x[d];
        R to[A], tn[A];
        Cost::cache(static_cast<R>(xv), d, n, tn);
#pragma unroll
        for (int q = 0; q < A; ++q) {
            to[q] = row[d * A + q];
            row[d * A + q] = tn[q];
        }
        x[d] = xv;
        const double trial = static_cast<double>(Cost::template energy<0>(row, n, a.family));
        const uint64_t m3 = draw_bits53(ctr + 2, chain, level, a.keys);
        ctr += 3;
        int r = metropolis_fast<double>(trial, E, k2, metropolis_band(m3));
        if (r < 0) r = Accept<R>::exact(trial - E, temperature, m3);
        if (r) {
            E = trial;
        } else {
            x[d] = xold;
#pragma unroll
            for (int q = 0; q < A; ++q) row[d * A + q] = to[q];
        }
    }
    *energy = E;
    *counter = ctr;
}

// ---------------------------------------------------------------------------
// V0 latency path: run_sequential (engines.cpp:125-129) — ONE chain through
// the whole ladder, 114600 dependent trials for C1's ladder — for the affine
// families at n <= 32.  The chain lives in the registers of the consumer
// warp (lane k holds t_k and x_k); every lane runs the same scalar
// decision, so there is no vote: a trial is a broadcast read of its
// proposal, one shuffle for the replaced term, the deferred-fold interval
// test, and a predicated register move on acceptance.  Exact folds (settles,
// level ends) run in index order through shuffles.  Warps 1..3 produce the
// proposals (three Philox draws and the term) 32 trials ahead into a
// double-buffered ring.  Outputs are those of the V1 kernels (one block:
// trace candidates, end state, xbest slot 0), finalized by v1_finalize.
// ---------------------------------------------------------------------------
template <class R, class Cost>
__global__ void __launch_bounds__(128, 1) v0_kernel(const EngineArgs a) {
    using Fam = typename Cost::Fam;
    using L = LazyOf<Fam>;
    static_assert(Cost::A == 1, "deferred fold: one accumulator");
    __shared__ PcEntryX<R, 1> ring[2][32];
    __shared__ double lower_s[32], width_s[32];
    const int tid = threadIdx.x, lane = tid & 31;
    const int n = a.n; // <= 32 (plan_build)
    const bool producer = tid >= 32;
    Box box;
    if (tid < n && !a.uniform_box) {
        lower_s[tid] = a.lower[tid];
        width_s[tid] = a.width[tid];
    }
    box.lower = lower_s;
    box.width = width_s;
    box.lo0 = a.lo0;
    box.w0 = a.w0;
    box.uniform = a.uniform_box != 0;
    __syncthreads();
    const uint32_t c = a.chain_begin;
    const PhiloxChain pch = philox_chain(c, 0u, a.keys);
    const uint32_t ctr0 = a.random_start ? static_cast<uint32_t>(n) : 0u;
    const long long total = static_cast<long long>(a.levels) * a.N;
    const int rounds = static_cast<int>((total + 31) / 32);
    const double idx_scale = static_cast<double>(n) * 0x1.0p-53;
    // proposals for trials [32 k, 32 k + jn): one per producer thread
    auto produce = [&](int k) {
        const long long j0 = 32ll * k;
        const int jn = total - j0 < 32 ? static_cast<int>(total - j0) : 32;
        const int jj = tid - 32;
        if (jj < jn) {
            const uint32_t ctr = ctr0 + 3u * static_cast<uint32_t>(j0 + jj);
            const uint64_t m1 = draw_bits53_fast(ctr, pch, a.keys);
            const uint64_t m2 = draw_bits53_fast(ctr + 1, pch, a.keys);
            PcEntryX<R, 1> en;
            en.p.m = draw_bits53_fast(ctr + 2, pch, a.keys);
            en.p.d = min(static_cast<int>(static_cast<double>(m1) * idx_scale), n - 1);
            en.x = box.point(en.p.d, bits_to_uniform(m2));
            bool ok;
            Cost::cache_common(static_cast<R>(en.x), en.p.d, n, en.p.t, ok);
            if (!ok) Cost::cache(static_cast<R>(en.x), en.p.d, n, en.p.t);
            ring[k & 1][jj] = en;
        }
    };
    // the chain: lane k holds x_k and its term
    double x = 0;
    R t = 0;
    if (!producer && lane < n) {
        x = a.random_start ? random_start_coord(a, box, c, lane) : a.start[lane];
        R tt[1];
        Cost::cache(static_cast<R>(x), lane, n, tt);
        t = tt[0];
    }
    // exact energy in index order, lane dsub's term replaced by tsub
    auto fold_lanes = [&](R tsub, int dsub) {
        R acc[1] = {Fam::init(0, n)};
        for (int k = 0; k < n; ++k) {
            R v = __shfl_sync(0xffffffffu, t, k);
            if (k == dsub) v = tsub;
            acc[0] = fold<R>(Fam::op(0), acc[0], v);
        }
        return Fam::finish(acc, n);
    };
    R E = 0;
    if (!producer) E = fold_lanes(R(0), -1);
    bool have = true;
    double chain_best = static_cast<double>(E);
    uint64_t settles = 0;
    if (producer) produce(0);
    __syncthreads();
    int level = 0, in_level = 0;
    double T = a.temps[0];
    float k2 = metropolis_k2(T);
    const R sa = L::sigma > 0 ? static_cast<R>(a.lazy_alpha) : -static_cast<R>(a.lazy_alpha);
    const R rr = static_cast<R>(a.lazy_r);
    for (int k = 0; k < rounds; ++k) {
        const long long j0 = 32ll * k;
        const int jn = total - j0 < 32 ? static_cast<int>(total - j0) : 32;
        if (producer) {
            if (k + 1 < rounds) produce(k + 1);
        } else {
            const PcEntryX<R, 1>* cur = ring[k & 1];
            // the interval decision (sweep_lazy): 1 accept, 0 reject, -1 settle
            auto decide = [&](R tn, R to, const MBand& bb) {
                const R q = (tn - to) * sa;
                const R hi = q + rr, lo = q - rr;
                return ((hi <= R(0)) | (static_cast<float>(hi) * k2 < bb.lo))
                           ? 1
                           : (((lo > R(0)) & (static_cast<float>(lo) * k2 > bb.hi)) ? 0 : -1);
            };
            auto level_end = [&]() { // engines.cpp:90-106: the exact level-end energy
                if (!have) {
                    E = fold_lanes(R(0), -1);
                    have = true;
                }
                if (static_cast<double>(E) < chain_best) chain_best = static_cast<double>(E);
                if (lane == 0)
                    a.trace_cand[static_cast<size_t>(level) * gridDim.x + blockIdx.x] =
                        !is_nan(chain_best) ? Cand{chain_best, static_cast<int32_t>(c), 0} : empty_cand();
                in_level = 0;
                if (++level < a.levels) {
                    T = a.temps[level];
                    k2 = metropolis_k2(T);
                }
            };
            auto move = [&](const PcEntryX<R, 1>& en) {
                if (lane == en.p.d) {
                    t = en.p.t[0];
                    x = en.x;
                }
            };
            int j = 0;
            while (j < jn) {
                const PcEntryX<R, 1> e0 = cur[j];
                const MBand b0 = metropolis_band(e0.p.m);
                // two trials of one level at once: trial 1's decision is made
                // both for the term before trial 0 and for trial 0's new term
                // (same coordinate), then selected by trial 0's outcome — two
                // independent chains of work instead of one dependent chain
                if (j + 1 < jn && in_level + 2 <= a.N) {
                    const PcEntryX<R, 1> e1 = cur[j + 1];
                    const MBand b1 = metropolis_band(e1.p.m);
                    const R t0 = __shfl_sync(0xffffffffu, t, e0.p.d);
                    const R t1 = __shfl_sync(0xffffffffu, t, e1.p.d);
                    const int r0 = decide(e0.p.t[0], t0, b0);
                    const int r1a = decide(e1.p.t[0], t1, b1);
                    const int r1b = decide(e1.p.t[0], e0.p.t[0], b1);
                    const int r1 = (r0 == 1 && e1.p.d == e0.p.d) ? r1b : r1a;
                    if ((r0 >= 0) & (r1 >= 0)) { // warp-uniform
                        if (r0) {
                            move(e0);
                            have = false;
                        }
                        if (r1) {
                            move(e1);
                            have = false;
                        }
                        in_level += 2;
                        if (in_level == a.N) level_end();
                        j += 2;
                        continue;
                    }
                }
                // one trial, settling if needed
                const R to = __shfl_sync(0xffffffffu, t, e0.p.d);
                int r = decide(e0.p.t[0], to, b0);
                bool settled = false;
                if (r < 0) { // warp-uniform: every lane computed the same r
                    if (!have) {
                        E = fold_lanes(R(0), -1);
                        have = true;
                    }
                    const R et = fold_lanes(e0.p.t[0], e0.p.d);
                    int v = metropolis_fast<R>(et, E, k2, b0);
                    if (v < 0) v = Accept<R>::exact(static_cast<double>(et) - static_cast<double>(E), T, e0.p.m);
                    if (v) E = et;
                    r = v;
                    settled = true;
                    ++settles;
                }
                if (r) {
                    move(e0);
                    if (!settled) have = false;
                }
                if (++in_level == a.N) level_end();
                ++j;
            }
        }
        __syncthreads();
    }
    if (!producer) {
        if (lane < n) a.xbest[lane] = x; // slot 0 (engines.cpp:110-116: the end state)
        if (lane == 0) {
            a.cand[blockIdx.x] = Cand{static_cast<double>(E), static_cast<int32_t>(c), 0};
            atomicAdd(&a.out_scalars->evaluations, static_cast<unsigned long long>(1 + total));
            atomicAdd(&a.out_scalars->rng_draws,
                      static_cast<unsigned long long>(3 * total + (a.random_start ? n : 0)));
            atomicAdd(&a.out_scalars->exact_settles, static_cast<unsigned long long>(settles));
        }
    }
}

// ---------------------------------------------------------------------------
// Host-side dispatch over (precision, family)
// ---------------------------------------------------------------------------

template <class R, class Cost, int NT = 0>
struct KernelSet {
    static EngineKernels get() {
        EngineKernels k;
        k.v2 = reinterpret_cast<const void*>(&v2_kernel<R, Cost, NT, false>);
        k.v1 = reinterpret_cast<const void*>(&v1_kernel<R, Cost, NT, false>);
        k.v2g = reinterpret_cast<const void*>(&v2_kernel<R, Cost, 0, true>);
        k.v1g = reinterpret_cast<const void*>(&v1_kernel<R, Cost, 0, true>);
        k.smem_g = [](int n, int B, bool box) { return engine_smem_bytes<R, Cost::A>(n, B, box, false); };
        k.state_bytes = sizeof(R) * Cost::A;
        k.eval = reinterpret_cast<const void*>(&probe_evaluate<R, Cost>);
        k.sweep = reinterpret_cast<const void*>(&sweep_one<R, Cost>);
        k.smem_v2 = [](int n, int B, bool box) { return engine_smem_bytes<R, Cost::A>(n, B, box, true); };
        k.v2pc = reinterpret_cast<const void*>(&v2_pc_kernel<R, Cost, NT>);
        k.v1pc = reinterpret_cast<const void*>(&v1_pc_kernel<R, Cost, NT>);
        k.smem_v1pc = [](int n, int, bool box) {
            return engine_smem_bytes<R, Cost::A>(n, 32, box, true) + 16 + sizeof(PcEntryX<R, Cost::A>) * 2 * 32 * 32;
        };
        // rows for the consumer warp only, plus the 3 x 32 x 32 proposal ring
        k.smem_v2pc = [](int n, int, bool box) {
            return engine_smem_bytes<R, Cost::A>(n, 32, box, true) + 16 + sizeof(PcEntry<R, Cost::A>) * 3 * 32 * 32;
        };
        k.v2z = nullptr;
        k.v2zu = nullptr;
        k.v2gz = nullptr;
        k.v2gzu = nullptr;
        k.v2pcz = nullptr;
        k.v1pcz = nullptr;
        k.v0z = nullptr;
        k.v2pz = nullptr;
        k.lazy_radius = nullptr;
        k.lazy_alpha_of = nullptr;
        if constexpr (LazyCost<Cost>::value) {
            k.v2z = reinterpret_cast<const void*>(&v2_lazy_kernel<R, Cost, NT, false>);
            k.v2zu = reinterpret_cast<const void*>(&v2_lazy_kernel<R, Cost, NT, false, true>);
            k.v2gz = reinterpret_cast<const void*>(&v2_lazy_kernel<R, Cost, 0, true>);
            k.v2gzu = reinterpret_cast<const void*>(&v2_lazy_kernel<R, Cost, 0, true, true>);
            k.v2pcz = reinterpret_cast<const void*>(&v2_lazy_pc_kernel<R, Cost, NT>);
            k.v1pcz = reinterpret_cast<const void*>(&v1_pc_kernel<R, Cost, NT, true>);
            k.v0z = reinterpret_cast<const void*>(&v0_kernel<R, Cost>);
            k.lazy_radius = &LazyCost<Cost>::radius;
            k.lazy_alpha_of = &LazyCost<Cost>::alpha;
            if constexpr (PairOf<Cost>::value) k.v2pz = reinterpret_cast<const void*>(&v2_lazy_pair_kernel<R, Cost, NT>);
        }
        if constexpr (PairOf<Cost>::value) {
            k.v1p = reinterpret_cast<const void*>(&v1_pair_kernel<R, Cost, NT>);
            k.v2p = reinterpret_cast<const void*>(&v2_pair_kernel<R, Cost, NT>);
            k.smem_v2p = [](int n, int B, bool box) { return engine_smem_bytes<R, Cost::A>(n, B, box, true, true); };
        } else {
            k.v1p = nullptr;
            k.v2p = nullptr;
            k.smem_v2p = nullptr;
        }
        k.smem_v1 = [](int n, int B, bool box) { return engine_smem_bytes<R, Cost::A>(n, B, box, true); };
        k.smem_eval = [](int n, int B) { return sizeof(R) * size_t(row_stride<R>(n, Cost::A)) * B; };
        return k;
    }
};

// Dimensions of the benchmark configurations get a compile-time n
// (BASELINE.json: n = 10, 30, 100).
template <class R, template <class> class F>
EngineKernels sep_kernels(int n) {
    switch (n) {
    case 10: return KernelSet<R, SepCost<R, F>, 10>::get();
    case 30: return KernelSet<R, SepCost<R, F>, 30>::get();
    case 100: return KernelSet<R, SepCost<R, F>, 100>::get();
    // configs[3] (the hybrid's SA phase) runs normalized Schwefel at n = 500
    case 500:
        if constexpr (std::is_same<F<R>, Schwefel<R>>::value) return KernelSet<R, SepCost<R, F>, 500>::get();
        else return KernelSet<R, SepCost<R, F>>::get();
    default: return KernelSet<R, SepCost<R, F>>::get();
    }
}

// one kernel set per separable family (compile-time n for Schwefel) and one
// for all full-evaluation families; explicit instantiations live in
// engine_fam_*.cu
template <class R, template <class> class F>
EngineKernels sep_set(int n) {
    return sep_kernels<R, F>(n);
}
template <class R, template <class> class F>
EngineKernels sep_set_generic(int) {
    return KernelSet<R, SepCost<R, F>>::get();
}
template <class R>
EngineKernels full_set(int) {
    return KernelSet<R, FullCost<R>>::get();
}

} // namespace psa
