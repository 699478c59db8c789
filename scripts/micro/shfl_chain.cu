// Microbenchmark: dependent shuffle-chain step cost vs warps per SM (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(float* out, int steps, int mode) {
    const int lane = threadIdx.x & 31;
    float acc = lane * 0.001f, f = 0.5f + lane * 1e-4f;
    __shared__ float sh[32 * 32];
    float* my = sh + (threadIdx.x >> 5) * 32;
    long long t0 = clock64();
    for (int s = 0; s < steps; s += 32) {
#pragma unroll
        for (int cc = 0; cc < 32; ++cc) {
            float yc;
            if (mode == 0) {
                yc = __shfl_sync(0xffffffffu, acc, cc);
            } else {
                if (lane == cc) my[cc] = acc;
                __syncwarp();
                yc = my[cc];
            }
            if (lane > cc) acc = fmaf(-f, yc, acc);
        }
    }
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 32 + (threadIdx.x >> 5)] = (float)(t1 - t0) / steps;
    if (acc == 123.f) out[0] = acc;
}
int main() {
    float* d; cudaMalloc(&d, 148 * 32 * 32 * 4);
    float h[148 * 32];
    for (int mode = 0; mode < 2; ++mode)
        for (int wps : {1, 4, 8, 16, 32}) {  // warps per SM (1 CTA per SM)
            chain<<<148, 32 * wps>>>(d, 32 * 256, mode);
            cudaDeviceSynchronize();
            chain<<<148, 32 * wps>>>(d, 32 * 256, mode);
            cudaMemcpy(h, d, 148 * wps * 4, cudaMemcpyDeviceToHost);
            double s = 0; for (int i = 0; i < 148 * wps; ++i) s += h[i];
            printf("mode %s warps/SM %2d: %.1f cycles per chain step per warp\n", mode ? "smem" : "shfl", wps, s / (148 * wps));
        }
}
