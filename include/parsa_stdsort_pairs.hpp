// parsa_stdsort_pairs.hpp — the libstdc++ introsort of parsa_stdsort.h over
// (key, id) pairs instead of ids looked up in a key array.
//
// Same algorithm, same comparisons (key < key), same element moves — so the
// resulting order, ties included, is exactly psa_std_sort's (checked on
// random tie-heavy inputs by tests/cxx/stdsort_pairs_check.cpp).  A
// comparison reads one 16-byte pair instead of an id and then its key, which
// halves the dependent shared-memory loads of the device Nelder–Mead's exact
// sort (the one-thread path taken when the simplex holds equal values).
#pragma once

#include "parsa_stdsort.h"

#ifndef PSA_PAIR_FN
#if defined(__CUDACC__)
#define PSA_PAIR_FN __host__ __device__ inline
#else
#define PSA_PAIR_FN inline
#endif
#endif

namespace psa_sort {

struct alignas(16) KeyId {
    double key;
    int id;
    int pad;
};

PSA_PAIR_FN bool less(const KeyId& a, const KeyId& b) { return a.key < b.key; }

PSA_PAIR_FN void swap(KeyId* v, int i, int j) {
    const KeyId t = v[i];
    v[i] = v[j];
    v[j] = t;
}

PSA_PAIR_FN void push_heap(KeyId* v, int first, int hole, int top, KeyId value) {
    int parent = (hole - 1) / 2;
    while (hole > top && less(v[first + parent], value)) {
        v[first + hole] = v[first + parent];
        hole = parent;
        parent = (hole - 1) / 2;
    }
    v[first + hole] = value;
}

PSA_PAIR_FN void adjust_heap(KeyId* v, int first, int hole, int len, KeyId value) {
    const int top = hole;
    int second = hole;
    while (second < (len - 1) / 2) {
        second = 2 * (second + 1);
        if (less(v[first + second], v[first + second - 1])) second--;
        v[first + hole] = v[first + second];
        hole = second;
    }
    if ((len & 1) == 0 && second == (len - 2) / 2) {
        second = 2 * (second + 1);
        v[first + hole] = v[first + second - 1];
        hole = second - 1;
    }
    push_heap(v, first, hole, top, value);
}

PSA_PAIR_FN void heap_sort(KeyId* v, int first, int last) {
    const int len = last - first;
    if (len >= 2) {
        int parent = (len - 2) / 2;
        for (;;) {
            const KeyId value = v[first + parent];
            adjust_heap(v, first, parent, len, value);
            if (parent == 0) break;
            parent--;
        }
    }
    while (last - first > 1) {
        --last;
        const KeyId value = v[last];
        v[last] = v[first];
        adjust_heap(v, first, 0, last - first, value);
    }
}

PSA_PAIR_FN void median_to_first(KeyId* v, int result, int a, int b, int c) {
    if (less(v[a], v[b])) {
        if (less(v[b], v[c])) swap(v, result, b);
        else if (less(v[a], v[c])) swap(v, result, c);
        else swap(v, result, a);
    } else if (less(v[a], v[c])) {
        swap(v, result, a);
    } else if (less(v[b], v[c])) {
        swap(v, result, c);
    } else {
        swap(v, result, b);
    }
}

PSA_PAIR_FN int unguarded_partition(KeyId* v, int first, int last, int pivot) {
    for (;;) {
        while (less(v[first], v[pivot])) ++first;
        --last;
        while (less(v[pivot], v[last])) --last;
        if (!(first < last)) return first;
        swap(v, first, last);
        ++first;
    }
}

PSA_PAIR_FN void introsort_loop(KeyId* v, int first, int last, int depth) {
    int stack_first[64], stack_last[64], stack_depth[64];
    int sp = 0;
    for (;;) {
        while (last - first > PSA_SORT_THRESHOLD) {
            if (depth == 0) {
                heap_sort(v, first, last);
                last = first;
                break;
            }
            --depth;
            const int mid = first + (last - first) / 2;
            median_to_first(v, first, first + 1, mid, last - 1);
            const int cut = unguarded_partition(v, first + 1, last, first);
            stack_first[sp] = first;
            stack_last[sp] = cut;
            stack_depth[sp] = depth;
            ++sp;
            first = cut;
        }
        if (sp == 0) return;
        --sp;
        first = stack_first[sp];
        last = stack_last[sp];
        depth = stack_depth[sp];
    }
}

PSA_PAIR_FN void linear_insert(KeyId* v, int last) {
    const KeyId val = v[last];
    int next = last - 1;
    while (less(val, v[next])) {
        v[last] = v[next];
        last = next;
        --next;
    }
    v[last] = val;
}

PSA_PAIR_FN void insertion_sort(KeyId* v, int first, int last) {
    if (first == last) return;
    for (int i = first + 1; i != last; ++i) {
        if (less(v[i], v[first])) {
            const KeyId val = v[i];
            for (int j = i; j > first; --j) v[j] = v[j - 1];
            v[first] = val;
        } else {
            linear_insert(v, i);
        }
    }
}

// std::sort(v, v + m) by key
PSA_PAIR_FN void sort(KeyId* v, int m) {
    if (m <= 1) return;
    introsort_loop(v, 0, m, psa_lg(m) * 2);
    if (m > PSA_SORT_THRESHOLD) {
        insertion_sort(v, 0, PSA_SORT_THRESHOLD);
        for (int i = PSA_SORT_THRESHOLD; i != m; ++i) linear_insert(v, i);
    } else {
        insertion_sort(v, 0, m);
    }
}

// ---------------------------------------------------------------------------
// The same sort as independent tasks (the device runs one task per lane).
//
// introsort_loop only ever works on disjoint ranges: a range larger than the
// threshold is either heap-sorted (depth budget spent) or split at a cut, and
// its two halves never interact again.  The final insertion sort cannot move
// an element across a cut either: everything left of a cut is not greater
// than the pivot and everything right of it not less (keys without NaN are
// strictly weakly ordered), and insertion only moves an element past a
// strictly greater one.  So running, for every range as soon as it exists,
// heap_sort / split and insertion_sort on every final range of at most
// PSA_SORT_THRESHOLD elements gives the order of sort() exactly, in any task
// order.  (Keys containing NaN take sort() itself.)
// ---------------------------------------------------------------------------

// one introsort_loop step on [first, last) with depth > 0: the cut
PSA_PAIR_FN int split(KeyId* v, int first, int last) {
    const int mid = first + (last - first) / 2;
    median_to_first(v, first, first + 1, mid, last - 1);
    return unguarded_partition(v, first + 1, last, first);
}

// the task of range [first, last) (size > threshold): calls emit(f, l, d)
// for each child range still above the threshold and insertion-sorts the rest
template <class Emit>
PSA_PAIR_FN void range_task(KeyId* v, int first, int last, int depth, Emit&& emit) {
    if (depth == 0) {
        heap_sort(v, first, last);
        return;
    }
    const int cut = split(v, first, last);
    if (cut - first > PSA_SORT_THRESHOLD) emit(first, cut, depth - 1);
    else insertion_sort(v, first, cut);
    if (last - cut > PSA_SORT_THRESHOLD) emit(cut, last, depth - 1);
    else insertion_sort(v, cut, last);
}

#if !defined(__CUDA_ARCH__)
// host emulation of the task form, breadth first (tests)
inline void sort_tasks(KeyId* v, int m) {
    if (m <= PSA_SORT_THRESHOLD) {
        insertion_sort(v, 0, m);
        return;
    }
    struct R { int f, l, d; };
    R cur[4096], nxt[4096];
    int nc = 1;
    cur[0] = R{0, m, psa_lg(m) * 2};
    while (nc > 0) {
        int nn = 0;
        for (int i = nc - 1; i >= 0; --i) // any order: process the level backwards
            range_task(v, cur[i].f, cur[i].l, cur[i].d, [&](int f, int l, int d) { nxt[nn++] = R{f, l, d}; });
        for (int i = 0; i < nn; ++i) cur[i] = nxt[i];
        nc = nn;
    }
}
#endif

#if defined(__CUDACC__)
// ---------------------------------------------------------------------------
// The same sort, warp-cooperative (device): sort() on (key, id) pairs with
// the whole warp instead of one lane per range — the order of sort()
// exactly, in any task order (see range_task above):
//  * a split's unguarded_partition is emulated with ballots.  With Ls the
//    ascending left-stop positions (!(v[i] < P)) and Rs the descending
//    right-stop positions (!(P < v[j])) of the ORIGINAL range, the two-pointer
//    scan swaps (Ls[k], Rs[k]) for every k < K, K the first k with
//    !(Ls[k] < Rs[k]) (both lists are monotone, and every swap touches only
//    positions both scans have already passed), and returns
//    K == 0 ? Ls[0] : min(Ls[K], Rs[K-1]) (position Rs[K-1] then holds a
//    left-stop value);
//  * heap_sort's make_heap runs the sift-downs of one tree depth in
//    parallel (their subtrees are disjoint, and the sequential loop visits
//    every deeper node first); its sort_heap phase stays on one lane;
//  * final insertion sorts run one range per lane.
// All 32 lanes call warp_sort; v, ls, rs (m ints each) and the range lists
// (WarpSortLists) are in shared memory.
// ---------------------------------------------------------------------------
struct WarpSortLists {
    int* cur;   // 3 ints per range: first, last, depth
    int* nxt;
    int* small; // 2 ints per final range (<= PSA_SORT_THRESHOLD elements)
};

__device__ inline int warp_partition(KeyId* v, int first, int last, int* ls, int* rs) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const double P = v[first].key;
    int nl = 0, nr = 0;
    for (int base = first + 1; base < last; base += 32) {
        const int i = base + lane;
        const bool in = i < last;
        const double k = in ? v[i].key : 0.0;
        const bool L = in && !(k < P);
        const bool R = in && !(P < k);
        const unsigned bl = __ballot_sync(0xffffffffu, L), br = __ballot_sync(0xffffffffu, R);
        if (L) ls[nl + __popc(bl & below)] = i;
        if (R) rs[nr + __popc(br & below)] = i; // ascending; Rs[k] = rs[nr - 1 - k]
        nl += __popc(bl);
        nr += __popc(br);
    }
    __syncwarp();
    const int mk = nl < nr ? nl : nr;
    int K = mk;
    for (int base = 0; base < mk; base += 32) {
        const int k = base + lane;
        const unsigned bf = __ballot_sync(0xffffffffu, k < mk && !(ls[k] < rs[nr - 1 - k]));
        if (bf) {
            K = base + __ffs(bf) - 1;
            break;
        }
    }
    for (int k = lane; k < K; k += 32) swap(v, ls[k], rs[nr - 1 - k]);
    __syncwarp();
    if (K == 0) return ls[0];
    const int r = rs[nr - K];
    return K < nl && ls[K] < r ? ls[K] : r;
}

// adjust_heap by the whole warp: the hole's descent follows, level by level,
// the child chosen by `second = right; if (v[right] < v[left]) second--` —
// a path that depends only on the heap, not on the value sifted.  The warp
// loads the 30 descendants of the current node four levels deep at once
// (lane j: depth L = floor(log2(j + 2)), offset o = j + 2 - 2^L, node
// (s + 1) 2^L - 1 + o), every odd lane (a right child) decides its pair,
// and the path through the four levels is read off one ballot; the chosen
// nodes move up into their parents' places in parallel (all loads precede
// all stores).  The descent stops where the sequential loop would
// (second >= (len - 1) / 2); the tail (a lone left child) and push_heap
// run on lane 0.  Same moves, same order of effect, as adjust_heap.
__device__ inline void warp_adjust_heap(KeyId* v, int first, int hole, int len, KeyId value) {
    const int lane = threadIdx.x & 31;
    KeyId* b = v + first;
    const int top = hole;
    const int lim = (len - 1) / 2;
    int second = hole;
    const int L = lane < 30 ? 31 - __clz(lane + 2) : 0;
    const int o = lane + 2 - (1 << L);
    while (second < lim) {
        const int node = ((second + 1) << L) - 1 + o;
        KeyId mine{0.0, 0, 0};
        if (lane < 30 && node < len) mine = b[node];
        const double sib = __shfl_up_sync(0xffffffffu, mine.key, 1);
        // odd o: a right child; it wins its pair unless it is less than the left
        const unsigned rw = __ballot_sync(0xffffffffu, lane < 30 && (o & 1) && !(mine.key < sib));
        // walk the (up to) four levels
        int path[4];
        int depth = 0, oo = 0, s = second;
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            if (s >= lim) break;
            const int right_lane = (1 << k) - 2 + 2 * oo + 1; // lane of the right child at depth k
            oo = 2 * oo + static_cast<int>((rw >> right_lane) & 1u);
            path[k - 1] = (1 << k) - 2 + oo; // lane of the chosen node
            s = ((second + 1) << k) - 1 + oo;
            depth = k;
        }
        __syncwarp(); // every lane's load precedes any store (racecheck)
        // moves: chosen node at depth k goes to its parent's place (the hole
        // for k = 1); lanes holding chosen nodes store in parallel
#pragma unroll
        for (int k = 1; k <= 4; ++k) {
            if (k <= depth && lane == path[k - 1]) {
                const int parent = k == 1 ? hole : ((second + 1) << (k - 1)) - 1 + (o >> 1);
                b[parent] = mine;
            }
        }
        hole = s;
        second = s;
        __syncwarp();
    }
    if (lane == 0) {
        if ((len & 1) == 0 && second == (len - 2) / 2) {
            second = 2 * (second + 1);
            b[hole] = b[second - 1];
            hole = second - 1;
        }
        push_heap(v, first, hole, top, value);
    }
    __syncwarp();
}

// ascending sort of [first, last) in place, for DISTINCT keys (any correct
// sort gives the same order then): the bitonic network in its all-ascending
// form (each merge starts by comparing every position with its mirror in the
// block), padded to a power of two with positions that act as +inf — with
// every comparator putting the smaller key first, a real element never moves
// into the padding
__device__ inline void warp_sort_distinct(KeyId* v, int first, int last) {
    const int lane = threadIdx.x & 31;
    const int m = last - first;
    int P = 1;
    while (P < m) P <<= 1;
    KeyId* b = v + first;
    auto cmpx = [&](int i, int l) { // i < l
        if (l < m) {
            const KeyId x = b[i], y = b[l];
            if (less(y, x)) {
                b[i] = y;
                b[l] = x;
            }
        }
    };
    for (int k = 2; k <= P; k <<= 1) {
        const int h = k >> 1;
        for (int t = lane; t < P / 2; t += 32) {
            const int blk = t / h, w = t - blk * h;
            cmpx(blk * k + w, blk * k + k - 1 - w);
        }
        __syncwarp();
        for (int j = k >> 2; j > 0; j >>= 1) {
            for (int t = lane; t < P / 2; t += 32) {
                const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                cmpx(i, i | j);
            }
            __syncwarp();
        }
    }
}

// heap_sort of [first, last).  tie_min: the smallest key that occurs more
// than once in the whole array (+inf: none; -inf, the default of warp_sort:
// unknown — every pop runs).  sort_heap pops the maximum
// each step, so once the root is below tie_min every remaining key is
// distinct and their heapsort order is simply ascending: the pops stop there
// and the rest is sorted directly — the same result, without the pops whose
// order no tie can observe.
__device__ inline void warp_heap_sort(KeyId* v, int first, int last, double tie_min) {
    const int lane = threadIdx.x & 31;
    const int len = last - first;
    if (len >= 2) {
        const int lastp = (len - 2) / 2;
        for (int d = 31 - __clz(lastp + 1); d >= 0; --d) { // deepest parents first
            const int lo = (1 << d) - 1, hi = min((1 << (d + 1)) - 2, lastp);
            for (int p = lo + lane; p <= hi; p += 32) {
                const KeyId value = v[first + p];
                adjust_heap(v, first, p, len, value);
            }
            __syncwarp();
        }
    }
    while (last - first > 1 && !(v[first].key < tie_min)) {
        --last;
        const KeyId value = v[last];
        __syncwarp();
        if (lane == 0) v[last] = v[first];
        __syncwarp();
        warp_adjust_heap(v, first, 0, last - first, value);
    }
    if (last - first > 1) warp_sort_distinct(v, first, last);
}

__device__ inline void warp_sort(KeyId* v, int m, int* ls, int* rs, WarpSortLists L,
                                 double tie_min = -__builtin_huge_val()) {
    const int lane = threadIdx.x & 31;
    if (m <= PSA_SORT_THRESHOLD) {
        if (lane == 0) insertion_sort(v, 0, m);
        __syncwarp();
        return;
    }
    int* cur = L.cur;
    int* nxt = L.nxt;
    if (lane == 0) {
        cur[0] = 0;
        cur[1] = m;
        cur[2] = psa_lg(m) * 2;
    }
    __syncwarp();
    int nc = 1;
    while (nc > 0) {
        int nn = 0, ns = 0; // warp-uniform
        for (int r = 0; r < nc; ++r) {
            const int f = cur[3 * r], l = cur[3 * r + 1], d = cur[3 * r + 2];
            if (d == 0) {
                warp_heap_sort(v, f, l, tie_min);
                continue;
            }
            if (lane == 0) median_to_first(v, f, f + 1, f + (l - f) / 2, l - 1);
            __syncwarp();
            const int cut = warp_partition(v, f, l, ls, rs);
            if (lane == 0) {
                if (cut - f > PSA_SORT_THRESHOLD) {
                    nxt[3 * nn] = f; nxt[3 * nn + 1] = cut; nxt[3 * nn + 2] = d - 1;
                } else {
                    L.small[2 * ns] = f; L.small[2 * ns + 1] = cut;
                }
                if (l - cut > PSA_SORT_THRESHOLD) {
                    const int q = nn + (cut - f > PSA_SORT_THRESHOLD);
                    nxt[3 * q] = cut; nxt[3 * q + 1] = l; nxt[3 * q + 2] = d - 1;
                } else {
                    const int q = ns + (cut - f <= PSA_SORT_THRESHOLD);
                    L.small[2 * q] = cut; L.small[2 * q + 1] = l;
                }
            }
            nn += (cut - f > PSA_SORT_THRESHOLD) + (l - cut > PSA_SORT_THRESHOLD);
            ns += (cut - f <= PSA_SORT_THRESHOLD) + (l - cut <= PSA_SORT_THRESHOLD);
            __syncwarp();
        }
        for (int i = lane; i < ns; i += 32) insertion_sort(v, L.small[2 * i], L.small[2 * i + 1]);
        __syncwarp();
        int* t = cur;
        cur = nxt;
        nxt = t;
        nc = nn;
    }
}
#endif

} // namespace psa_sort
