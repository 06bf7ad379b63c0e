// sort_probe.cu — the device exact sort of the Nelder-Mead kernel
// (psa_sort::warp_sort, include/parsa_stdsort_pairs.hpp) against the host
// restatement of libstdc++'s std::sort (psa_sort::sort) on random tie-heavy
// inputs, and its cycles on simplex-like inputs of 501 (key, id) pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include -o sort_probe sort_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

// the smallest key occurring more than once (+inf: none)
static double tie_min_of(const std::vector<double>& k, int m) {
    std::vector<double> s(k.begin(), k.begin() + m);
    std::sort(s.begin(), s.end());
    for (int i = 0; i + 1 < m; ++i)
        if (s[i] == s[i + 1]) return s[i];
    return INFINITY;
}

#include "parsa_stdsort.h"
#include "parsa_stdsort_pairs.hpp"

__global__ void heap_kernel(int m, int pf, long long* cyc) {
    __shared__ psa_sort::KeyId kp[1024];
    const int lane = threadIdx.x;
    for (int p = lane; p < m; p += 32) kp[p] = psa_sort::KeyId{static_cast<double>(p), p, 0};
    __syncwarp();
    long long t0 = clock64();
    // make_heap alone, then sort_heap alone
    if (lane == 0) {
        for (int parent = (m - 2) / 2;; --parent) {
            const psa_sort::KeyId value = kp[parent];
            psa_sort::adjust_heap(kp, 0, parent, m, value);
            if (parent == 0) break;
        }
    }
    __syncwarp();
    long long t1 = clock64();
    {
        int last = m;
        while (last > 1) {
            --last;
            const psa_sort::KeyId value = kp[last];
            __syncwarp();
            if (lane == 0) kp[last] = kp[0];
            __syncwarp();
            if (pf) psa_sort::warp_adjust_heap(kp, 0, 0, last, value);
            else if (lane == 0) psa_sort::adjust_heap(kp, 0, 0, last, value);
            __syncwarp();
        }
    }
    __syncwarp();
    long long t2 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

__global__ void sort_kernel(const double* keys, int m, int* out_ids, long long* cyc, double tie_min) {
    __shared__ psa_sort::KeyId kp[1024];
    __shared__ int ls[1024], rs[1024], lists[10 * 80];
    const int lane = threadIdx.x;
    for (int p = lane; p < m; p += 32) kp[p] = psa_sort::KeyId{keys[p], p, 0};
    __syncwarp();
    const psa_sort::WarpSortLists L{lists, lists + 3 * 80, lists + 6 * 80};
    const long long t0 = clock64();
    psa_sort::warp_sort(kp, m, ls, rs, L, tie_min);
    const long long t1 = clock64();
    for (int p = lane; p < m; p += 32) out_ids[p] = kp[p].id;
    if (lane == 0) *cyc = t1 - t0;
}

int main() {
    double* dk;
    int* di;
    long long* dc;
    cudaMalloc(&dk, 1024 * sizeof(double));
    cudaMalloc(&di, 1024 * sizeof(int));
    cudaMalloc(&dc, sizeof(long long));
    srand(7);
    int bad = 0, cases = 0;
    std::vector<double> keys(1024);
    std::vector<int> got(1024);
    for (int t = 0; t < 3000; ++t) {
        const int m = 1 + rand() % 1000;
        const int kinds = 1 + rand() % (t % 3 == 0 ? 3 : t % 3 == 1 ? 30 : 100000);
        for (int p = 0; p < m; ++p) keys[p] = rand() % kinds;
        if (t % 4 == 0) { // sorted prefix + one new element (the simplex case)
            std::vector<psa_sort::KeyId> s(m);
            for (int p = 0; p < m; ++p) s[p] = psa_sort::KeyId{keys[p], p, 0};
            psa_sort::sort(s.data(), m - 1);
            for (int p = 0; p < m - 1; ++p) keys[p] = s[p].key;
        }
        cudaMemcpy(dk, keys.data(), m * sizeof(double), cudaMemcpyHostToDevice);
        sort_kernel<<<1, 32>>>(dk, m, di, dc, t % 2 ? tie_min_of(keys, m) : -INFINITY);
        cudaMemcpy(got.data(), di, m * sizeof(int), cudaMemcpyDeviceToHost);
        std::vector<psa_sort::KeyId> want(m);
        for (int p = 0; p < m; ++p) want[p] = psa_sort::KeyId{keys[p], p, 0};
        psa_sort::sort(want.data(), m);
        ++cases;
        for (int p = 0; p < m; ++p)
            if (want[p].id != got[p]) {
                ++bad;
                break;
            }
    }
    std::printf("{\"cases\": %d, \"mismatches\": %d}\n", cases, bad);
    const char* names[] = {"sorted+new", "10 distinct", "all equal", "groups of 5"};
    for (int mode = 0; mode < 4; ++mode) {
        const int m = 501;
        for (int p = 0; p < m; ++p) {
            keys[p] = mode == 0 ? (p < m - 1 ? p : 100.5)
                      : mode == 1 ? (p < m - 1 ? p / 50 : 3.0)
                      : mode == 2 ? 1.0 : (p < m - 1 ? p / 5 : 50.0);
        }
        cudaMemcpy(dk, keys.data(), m * sizeof(double), cudaMemcpyHostToDevice);
        sort_kernel<<<1, 32>>>(dk, m, di, dc, tie_min_of(keys, m));
        long long c;
        cudaMemcpy(&c, dc, sizeof(c), cudaMemcpyDeviceToHost);
        std::printf("{\"input\": \"%s\", \"m\": 501, \"cycles\": %lld}\n", names[mode], c);
    }
    long long* d2;
    cudaMalloc(&d2, 16);
    for (int pf = 0; pf < 2; ++pf) {
        heap_kernel<<<1, 32>>>(354, pf, d2);
        long long h[2];
        cudaMemcpy(h, d2, 16, cudaMemcpyDeviceToHost);
        std::printf("{\"heap\": 354, \"prefetch\": %d, \"make_heap_cycles\": %lld, \"sort_heap_cycles\": %lld}\n", pf, h[0], h[1]);
    }
    return 0;
}
