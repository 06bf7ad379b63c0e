// latency_probe.cu — dependent-chain latencies that bound the Nelder-Mead
// centroid re-add (nelder_mead.cu): DADD, and the re-add's own pattern
// (index from shared memory, quotient from shared memory, DADD).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_probe latency_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void dadd_chain(double* out, double b, int iters, long long* cyc) {
    double a = threadIdx.x;
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) a = a + b;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    out[threadIdx.x] = a;
}

__global__ void readd_chain(double* out, int n, int reps, long long* cyc) {
    __shared__ int ord[512];
    __shared__ double Q[160 * 32];
    const int j = threadIdx.x;
    for (int i = j; i < 512; i += 32) ord[i] = (i * 37) % 160;
    for (int i = j; i < 160 * 32; i += 32) Q[i] = 1e-3 * i;
    __syncwarp();
    double c = 0;
    const long long t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < reps; ++r) {
        for (int p0 = 0; p0 < n; p0 += 16) {
            double q[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) q[i] = Q[ord[p0 + i] * 32 + j];
#pragma unroll
            for (int i = 0; i < 16; ++i) c += q[i];
        }
    }
    const long long t1 = clock64();
    if (j == 0) *cyc = t1 - t0;
    out[j] = c;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMalloc(&cyc, 2 * sizeof(long long));
    long long h[2];
    dadd_chain<<<1, 32>>>(out, 1.0, 1 << 14, cyc);
    readd_chain<<<1, 32>>>(out, 496, 64, cyc + 1);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    std::printf("{\"dadd_latency_cycles\": %.2f, \"readd_cycles_per_element\": %.2f}\n",
                double(h[0]) / (16.0 * (1 << 14)), double(h[1]) / (496.0 * 64));
    return 0;
}
