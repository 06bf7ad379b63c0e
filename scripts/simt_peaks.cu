// simt_peaks.cu — measured roofline denominators for the annealing engine.
//
// The engine is neither HBM- nor tensor-bound: its hot loop is the
// sequential fold over shared-memory cached terms (LDS.128 + FADD) plus the
// Philox integer work.  This measures, on the box, with CUDA events:
//   * shared-memory load bandwidth (LDS.128, conflict-free), bytes/s
//   * FP32 add issue rate (independent FADD chains), lane-ops/s
//   * 32x32->64 IMAD.WIDE.U32 rate (the Philox multiply), lane-ops/s
// and prints one JSON object (written to profiles/simt_peaks.json).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o simt_peaks simt_peaks.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#define CHECK(x)                                                                          \
    do {                                                                                  \
        cudaError_t e = (x);                                                              \
        if (e != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                  \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

constexpr int kIters = 4096;

__global__ void __launch_bounds__(512) smem_bw(float* out, int iters) {
    extern __shared__ float4 buf[];
    const int t = threadIdx.x;
    for (int i = t; i < 4096; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    // a warp reads 32 consecutive 16-byte vectors per instruction (4
    // conflict-free wavefronts); the address changes every iteration and the
    // loads are volatile so none can be hoisted or merged
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(buf));
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const unsigned idx = (t + 32 * q + 512 * it) & 4095;
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(base + 16 * idx));
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == -1.0f) out[0] = acc.x;
}

__global__ void __launch_bounds__(512) fadd_rate(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    const float b = out[1];
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = a[i] + b;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == -1.0f) out[0] = s;
}

__global__ void __launch_bounds__(512) imadwide_rate(uint32_t* out, int iters) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint64_t p = static_cast<uint64_t>(a[i]) * 0xD2511F53u;
                a[i] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p);
            }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0xdeadbeefu) out[0] = s;
}

template <class K, class... Args>
float time_ms(K kernel, dim3 g, dim3 b, size_t smem, Args... args) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) kernel<<<g, b, smem>>>(args...);
    cudaEventRecord(e0);
    kernel<<<g, b, smem>>>(args...);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    cudaDeviceProp p;
    CHECK(cudaGetDeviceProperties(&p, 0));
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int sms = p.multiProcessorCount;
    float* f;
    uint32_t* u;
    CHECK(cudaMalloc(&f, 64));
    CHECK(cudaMalloc(&u, 64));
    CHECK(cudaMemset(f, 0, 64));
    const int B = 512, G = sms * 4;
    CHECK(cudaFuncSetAttribute(smem_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    const float ms_s = time_ms(smem_bw, dim3(G), dim3(B), 65536, f, kIters);
    const double smem_bytes = double(G) * B * kIters * 16 * 16;
    const float ms_a = time_ms(fadd_rate, dim3(G), dim3(B), 0, f, kIters);
    const double fadds = double(G) * B * kIters * 16 * 8;
    const float ms_i = time_ms(imadwide_rate, dim3(G), dim3(B), 0, u, kIters);
    const double imads = double(G) * B * kIters * 16 * 8;
    CHECK(cudaGetLastError());
    std::printf("{\"device\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f,\n"
                " \"smem_bytes_per_s\": %.6e, \"smem_bytes_per_clk_per_sm_at_attr_clock\": %.2f,\n"
                " \"fp32_lane_ops_per_s\": %.6e, \"imad_wide_lane_ops_per_s\": %.6e,\n"
                " \"how\": \"scripts/simt_peaks.cu: %d blocks x %d threads, CUDA events, best of 1 after 3 warm-ups\"}\n",
                p.name, sms, clk_khz / 1e3, smem_bytes / (ms_s * 1e-3),
                smem_bytes / (ms_s * 1e-3) / (double(clk_khz) * 1e3 * sms), fadds / (ms_a * 1e-3),
                imads / (ms_i * 1e-3), G, B);
    return 0;
}
