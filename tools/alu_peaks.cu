// tools/alu_peaks.cu -- measured CUDA-core (non-tensor) peaks of this B200, for the ALU rooflines of the
// fixed-corotated and batched configs ("FP32/FP64 FLOP rate ... against *measured*
// CUDA-core peaks").  Not on the solve path.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_peaks tools/alu_peaks.cu
//   tools/alu_peaks > profiles/alu_peaks.json
//
// Each kernel runs ACC independent FMA chains per thread (enough to cover the pipe latency), grid = a
// multiple of the SM count x resident blocks.  FMA = 2 flops; a packed FFMA2 (fma.rn.f32x2, two FP32
// FMAs in one instruction) = 4 flops.  Burst = best of 10 launches of ~30 ms; sustained = the median
// rate over ~3 s of back-to-back launches (the power cap acts on the sustained figure).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
            return 1;                                                                        \
        }                                                                                    \
    } while (0)

constexpr int ACC = 16;

__global__ void ffma_kernel(float *out, int iters, float b, float c) {
    float a[ACC];
#pragma unroll
    for (int k = 0; k < ACC; ++k) a[k] = threadIdx.x * 1e-7f + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ACC; ++k) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(b), "f"(c));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < ACC; ++k) s += a[k];
    if (s == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_kernel(float *out, int iters, float b, float c) {
    unsigned long long a[ACC];
    float2 bb = make_float2(b, b), cc = make_float2(c, c);
    unsigned long long B = *reinterpret_cast<unsigned long long *>(&bb);
    unsigned long long Cc = *reinterpret_cast<unsigned long long *>(&cc);
#pragma unroll
    for (int k = 0; k < ACC; ++k) {
        float2 v = make_float2(threadIdx.x * 1e-7f + k, k * 0.5f);
        a[k] = *reinterpret_cast<unsigned long long *>(&v);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ACC; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(B), "l"(Cc));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < ACC; ++k) {
        float2 v = *reinterpret_cast<float2 *>(&a[k]);
        s += v.x + v.y;
    }
    if (s == 1234.5f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_kernel(float *out, int iters, double b, double c) {
    double a[ACC];
#pragma unroll
    for (int k = 0; k < ACC; ++k) a[k] = threadIdx.x * 1e-7 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ACC; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(b), "d"(c));
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < ACC; ++k) s += a[k];
    if (s == 1234.5) out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

struct Result {
    double burst, sustained, ms;
};

template <typename L>
static int measure(L launch, double flops_per_launch, Result &r) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    double best = 0.0, ms_best = 0.0;
    for (int i = 0; i < 10; ++i) {
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        double rate = flops_per_launch / (ms * 1e-3) / 1e12;
        if (rate > best) best = rate, ms_best = ms;
    }
    std::vector<double> rates;
    double total = 0.0;
    while (total < 3000.0) {
        CK(cudaEventRecord(e0));
        for (int k = 0; k < 10; ++k) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        total += ms;
        rates.push_back(10.0 * flops_per_launch / (ms * 1e-3) / 1e12);
    }
    std::sort(rates.begin(), rates.end());
    r = {best, rates[rates.size() / 2], ms_best};
    CK(cudaGetLastError());
    return 0;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float *out;
    CK(cudaMalloc(&out, sizeof(float) * 148 * 64 * 256 * 8));
    const int threads = 256, blocks = sms * 8;  // 64 warps per SM
    const double lanes = double(blocks) * threads;
    Result f32, f32x2, f64;
    int it32 = 20000, it64 = 2000;
    if (measure([&] { ffma_kernel<<<blocks, threads>>>(out, it32, 0.9999f, 1e-6f); }, lanes * it32 * ACC * 2.0, f32))
        return 1;
    if (measure([&] { ffma2_kernel<<<blocks, threads>>>(out, it32, 0.9999f, 1e-6f); }, lanes * it32 * ACC * 4.0,
                f32x2))
        return 1;
    if (measure([&] { dfma_kernel<<<blocks, threads>>>(out, it64, 0.9999, 1e-6); }, lanes * it64 * ACC * 2.0, f64))
        return 1;
    const double nominal32 = sms * 128.0 * 2.0 * clk * 1e3 / 1e12;
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"max_sm_clock_mhz\": %.0f,\n", prop.name, sms, clk / 1e3);
    printf("  \"how\": \"tools/alu_peaks.cu: %d independent FMA chains per thread, %d blocks x %d threads; "
           "FMA = 2 flops, FFMA2 = 4; burst = best of 10 launches, sustained = median over ~3 s back to back\",\n",
           ACC, blocks, threads);
    printf("  \"fp32_ffma_tflops\": %.3f, \"fp32_ffma_tflops_sustained\": %.3f,\n", f32.burst, f32.sustained);
    printf("  \"fp32_ffma2_tflops\": %.3f, \"fp32_ffma2_tflops_sustained\": %.3f,\n", f32x2.burst, f32x2.sustained);
    printf("  \"fp64_dfma_tflops\": %.3f, \"fp64_dfma_tflops_sustained\": %.3f,\n", f64.burst, f64.sustained);
    printf("  \"fp32_nominal_tflops_at_max_clock\": %.3f,\n", nominal32);
    printf("  \"launch_ms\": {\"ffma\": %.2f, \"ffma2\": %.2f, \"dfma\": %.2f}\n}\n", f32.ms, f32x2.ms, f64.ms);
    CK(cudaFree(out));
    return 0;
}
