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

} // namespace psa_sort
