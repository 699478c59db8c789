// Micro-benchmark: warp-level MMA throughput on B200 (sm_100a) for the LU's
// bulk update options: FP64 DMMA m8n8k4, TF32 m16n8k8 (FP32 accumulate),
// and plain FP32 FFMA, register operands, 8 independent accumulators per warp.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_rate.cu -o mma_rate
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_tf32(float* out, int iters) {
    unsigned a0 = __float_as_uint(1.0f + threadIdx.x * 1e-6f), a1 = a0, a2 = a0, a3 = a0;
    unsigned b0 = __float_as_uint(1.0f - threadIdx.x * 1e-6f), b1 = b0;
    float c[8][4];
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = c[q][2] = c[q][3] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, int iters) {
    float a = 1.0f + threadIdx.x * 1e-6f, b = 1.0f - threadIdx.x * 1e-6f;
    float c[16];
    for (int q = 0; q < 16; ++q) c[q] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) c[q] = fmaf(a, b, c[q]);
    }
    float s = 0.f;
    for (int q = 0; q < 16; ++q) s += c[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps = 4; warps <= 16; warps *= 2) {
        const int grid = sms * 2, block = warps * 32 / 2;
        float ms;
        k_dmma<<<grid, block>>>((double*)out, 16);
        cudaEventRecord(e0);
        k_dmma<<<grid, block>>>((double*)out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double dm = 2.0 * 256 * 8 * (double)iters * grid * (block / 32);
        k_tf32<<<grid, block>>>(out, 16);
        cudaEventRecord(e0);
        k_tf32<<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms2;
        cudaEventElapsedTime(&ms2, e0, e1);
        const double tf = 2.0 * 1024 * 8 * (double)iters * grid * (block / 32);
        k_ffma<<<grid, block>>>(out, 16);
        cudaEventRecord(e0);
        k_ffma<<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms3;
        cudaEventElapsedTime(&ms3, e0, e1);
        const double ff = 2.0 * 16 * (double)iters * grid * block;
        printf("warps/SM %2d: DMMA m8n8k4 %.1f TFLOP/s   TF32 m16n8k8 %.1f TFLOP/s   FP32 FFMA %.1f TFLOP/s\n", warps,
               dm / ms * 1e-9, tf / ms2 * 1e-9, ff / ms3 * 1e-9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
