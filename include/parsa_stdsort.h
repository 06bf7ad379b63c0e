/*
 * parsa_stdsort.h — restatement of libstdc++'s std::sort (GCC 13,
 * bits/stl_algo.h + bits/stl_heap.h: introsort with median-of-three pivot,
 * depth limit 2*floor(log2 n), heapsort fallback, final insertion sort with
 * threshold 16) over an array of vertex ids ordered by key[id] with
 * comp(a, b) = key[a] < key[b].
 *
 * Why: the reference sorts the Nelder–Mead simplex with std::sort
 * (nelder_mead.cpp:60,111), which is not stable; when two vertices carry
 * equal values their relative order — and with it the summation order of
 * the next centroid — is whatever introsort produces.  Reproducing the
 * reference bit for bit therefore needs the same algorithm, not just any
 * sort.  Plain C so the CPU oracle and the device kernel share it
 * (PSA_SORT_FN adds __host__ __device__ under nvcc).
 */
#ifndef PARSA_STDSORT_H
#define PARSA_STDSORT_H

#ifndef PSA_SORT_FN
#if defined(__CUDACC__)
#define PSA_SORT_FN static __host__ __device__ inline
#else
#define PSA_SORT_FN static inline
#endif
#endif

#define PSA_SORT_THRESHOLD 16

PSA_SORT_FN int psa_sort_less(const double* key, int a, int b) { return key[a] < key[b]; }

PSA_SORT_FN void psa_sort_swap(int* v, int i, int j) {
    int t = v[i];
    v[i] = v[j];
    v[j] = t;
}

/* __push_heap */
PSA_SORT_FN void psa_push_heap(int* v, int first, int hole, int top, int value, const double* key) {
    int parent = (hole - 1) / 2;
    while (hole > top && psa_sort_less(key, v[first + parent], value)) {
        v[first + hole] = v[first + parent];
        hole = parent;
        parent = (hole - 1) / 2;
    }
    v[first + hole] = value;
}

/* __adjust_heap */
PSA_SORT_FN void psa_adjust_heap(int* v, int first, int hole, int len, int value, const double* key) {
    const int top = hole;
    int second = hole;
    while (second < (len - 1) / 2) {
        second = 2 * (second + 1);
        if (psa_sort_less(key, v[first + second], v[first + second - 1])) second--;
        v[first + hole] = v[first + second];
        hole = second;
    }
    if ((len & 1) == 0 && second == (len - 2) / 2) {
        second = 2 * (second + 1);
        v[first + hole] = v[first + second - 1];
        hole = second - 1;
    }
    psa_push_heap(v, first, hole, top, value, key);
}

/* __partial_sort(first, last, last) = __make_heap + __sort_heap */
PSA_SORT_FN void psa_heap_sort(int* v, int first, int last, const double* key) {
    const int len = last - first;
    if (len >= 2) {
        int parent = (len - 2) / 2;
        for (;;) {
            const int value = v[first + parent];
            psa_adjust_heap(v, first, parent, len, value, key);
            if (parent == 0) break;
            parent--;
        }
    }
    while (last - first > 1) {
        --last;
        const int value = v[last]; /* __pop_heap(first, last, last) */
        v[last] = v[first];
        psa_adjust_heap(v, first, 0, last - first, value, key);
    }
}

/* __move_median_to_first */
PSA_SORT_FN void psa_median_to_first(int* v, int result, int a, int b, int c, const double* key) {
    if (psa_sort_less(key, v[a], v[b])) {
        if (psa_sort_less(key, v[b], v[c])) psa_sort_swap(v, result, b);
        else if (psa_sort_less(key, v[a], v[c])) psa_sort_swap(v, result, c);
        else psa_sort_swap(v, result, a);
    } else if (psa_sort_less(key, v[a], v[c])) {
        psa_sort_swap(v, result, a);
    } else if (psa_sort_less(key, v[b], v[c])) {
        psa_sort_swap(v, result, c);
    } else {
        psa_sort_swap(v, result, b);
    }
}

/* __unguarded_partition */
PSA_SORT_FN int psa_unguarded_partition(int* v, int first, int last, int pivot, const double* key) {
    for (;;) {
        while (psa_sort_less(key, v[first], v[pivot])) ++first;
        --last;
        while (psa_sort_less(key, v[pivot], v[last])) --last;
        if (!(first < last)) return first;
        psa_sort_swap(v, first, last);
        ++first;
    }
}

PSA_SORT_FN int psa_lg(int n) {
    int r = 0;
    while (n > 1) {
        n >>= 1;
        ++r;
    }
    return r;
}

/* __introsort_loop, with the tail recursion on the right part kept as an
 * explicit stack (the left part is the loop, as in libstdc++) */
PSA_SORT_FN void psa_introsort_loop(int* v, int first, int last, int depth, const double* key) {
    int stack_first[64], stack_last[64], stack_depth[64];
    int sp = 0;
    for (;;) {
        while (last - first > PSA_SORT_THRESHOLD) {
            if (depth == 0) {
                psa_heap_sort(v, first, last, key);
                last = first; /* done with this range */
                break;
            }
            --depth;
            const int mid = first + (last - first) / 2;
            psa_median_to_first(v, first, first + 1, mid, last - 1, key);
            const int cut = psa_unguarded_partition(v, first + 1, last, first, key);
            /* recurse on [cut, last) first, then continue with [first, cut) */
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

/* __unguarded_linear_insert */
PSA_SORT_FN void psa_linear_insert(int* v, int last, const double* key) {
    const int val = v[last];
    int next = last - 1;
    while (psa_sort_less(key, val, v[next])) {
        v[last] = v[next];
        last = next;
        --next;
    }
    v[last] = val;
}

/* __insertion_sort */
PSA_SORT_FN void psa_insertion_sort(int* v, int first, int last, const double* key) {
    if (first == last) return;
    for (int i = first + 1; i != last; ++i) {
        if (psa_sort_less(key, v[i], v[first])) {
            const int val = v[i];
            for (int j = i; j > first; --j) v[j] = v[j - 1];
            v[first] = val;
        } else {
            psa_linear_insert(v, i, key);
        }
    }
}

/* std::sort(v, v + m) by key[] */
PSA_SORT_FN void psa_std_sort(int* v, int m, const double* key) {
    if (m <= 1) return;
    psa_introsort_loop(v, 0, m, psa_lg(m) * 2, key);
    if (m > PSA_SORT_THRESHOLD) {
        psa_insertion_sort(v, 0, PSA_SORT_THRESHOLD, key);
        for (int i = PSA_SORT_THRESHOLD; i != m; ++i) psa_linear_insert(v, i, key);
    } else {
        psa_insertion_sort(v, 0, m, key);
    }
}

#endif
