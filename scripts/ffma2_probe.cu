// Throughput probe: scalar FFMA vs packed FFMA2 (fma.rn.f32x2, sm_100a) with
// 8 independent chains per thread; prints Tflop/s for each (nvcc -arch
// sm_100a, run on the GPU box).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long *>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2 *>(&v); }
__global__ void scalar_k(float *out, float a, float b, int iters) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fmaf_rn(x[i], a, b);
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void packed_k(float *out, float a, float b, int iters) {
    unsigned long long x[4];
    for (int i = 0; i < 4; ++i) x[i] = f2u(make_float2(threadIdx.x + 2 * i, threadIdx.x + 2 * i + 1));
    const unsigned long long A = f2u(make_float2(a, a)), B = f2u(make_float2(b, b));
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
    float s = 0; for (int i = 0; i < 4; ++i) { float2 v = u2f(x[i]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
    const int iters = 20000, blocks = 148 * 8, threads = 1024;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); scalar_k<<<blocks, threads>>>(o, 0.999f, 0.001f, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)blocks * threads;
        printf("scalar FFMA : %.1f Tflop/s (%.3f ms)\n", fl / ms / 1e9, ms);
        cudaEventRecord(e0); packed_k<<<blocks, threads>>>(o, 0.999f, 0.001f, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("packed FFMA2: %.1f Tflop/s (%.3f ms)\n", fl / ms / 1e9, ms);
    }
    return 0;
}
