// sort_probe.cu — cycles of the device exact introsort (warp-0 task form, as
// nelder_mead.cu's exact_sort_tasks) on simplex-like inputs of 501 (key, id)
// pairs: sorted with a new last element, heavy ties, all equal.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include -o sort_probe sort_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "parsa_stdsort.h"
#include "parsa_stdsort_pairs.hpp"

__device__ __noinline__ void tasks(psa_sort::KeyId* kp, int m, int* cur, int* nxt, int* count) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        cur[0] = 0;
        cur[1] = m;
        cur[2] = psa_lg(m) * 2;
    }
    int cnt = 1;
    __syncwarp();
    while (cnt > 0) {
        if (lane == 0) *count = 0;
        __syncwarp();
        for (int i = lane; i < cnt; i += 32)
            psa_sort::range_task(kp, cur[3 * i], cur[3 * i + 1], cur[3 * i + 2], [&](int f, int l, int d) {
                const int k = atomicAdd(count, 1);
                nxt[3 * k] = f;
                nxt[3 * k + 1] = l;
                nxt[3 * k + 2] = d;
            });
        __syncwarp();
        cnt = *count;
        __syncwarp();
        int* t = cur;
        cur = nxt;
        nxt = t;
    }
}

__global__ void probe(int mode, int m, long long* out, int* ok) {
    __shared__ psa_sort::KeyId kp[512];
    __shared__ int cur[3 * 512], nxt[3 * 512], count;
    const int lane = threadIdx.x;
    for (int p = lane; p < m; p += 32) {
        double k;
        if (mode == 0) k = p < m - 1 ? p : 100.5;          // sorted + new value
        else if (mode == 1) k = p < m - 1 ? p / 50 : 3.0;  // 10 distinct values
        else if (mode == 2) k = 1.0;                       // all equal
        else k = p < m - 1 ? p / 5 : 50.0;                 // groups of 5 ties
        kp[p] = psa_sort::KeyId{k, p, 0};
    }
    __syncwarp();
    const long long t0 = clock64();
    tasks(kp, m, cur, nxt, &count);
    __syncwarp();
    const long long t1 = clock64();
    if (lane == 0) {
        *out = t1 - t0;
        int good = 1;
        for (int p = 1; p < m; ++p) good &= !(kp[p].key < kp[p - 1].key);
        *ok = good;
    }
}

int main() {
    long long* d;
    int* ok;
    cudaMalloc(&d, 8);
    cudaMalloc(&ok, 4);
    const char* names[] = {"sorted+new", "10 distinct", "all equal", "groups of 5"};
    for (int mode = 0; mode < 4; ++mode) {
        probe<<<1, 32>>>(mode, 501, d, ok);
        long long c;
        int g;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&g, ok, 4, cudaMemcpyDeviceToHost);
        std::printf("{\"input\": \"%s\", \"m\": 501, \"cycles\": %lld, \"sorted\": %d}\n", names[mode], c, g);
    }
    return 0;
}
