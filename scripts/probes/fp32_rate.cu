// FP32 pipe rate on this GPU: scalar FFMA vs packed FFMA2 vs FMUL, many
// independent chains per thread, 8 warps per SMSP.  nvcc -arch=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float *out, float a, float b, int iters) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            if (MODE == 0) {
                x[i] = __fmaf_rn(x[i], a, b);
                x[i + 1] = __fmaf_rn(x[i + 1], a, b);
            } else if (MODE == 1) {
                unsigned long long v = (unsigned long long)__float_as_uint(x[i]) |
                                       ((unsigned long long)__float_as_uint(x[i + 1]) << 32);
                unsigned long long aa = (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(a) << 32);
                unsigned long long bb = (unsigned long long)__float_as_uint(b) | ((unsigned long long)__float_as_uint(b) << 32);
                asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v) : "l"(aa), "l"(bb));
                x[i] = __uint_as_float((unsigned)v);
                x[i + 1] = __uint_as_float((unsigned)(v >> 32));
            } else {
                x[i] = __fmul_rn(x[i], a);
                x[i + 1] = __fmul_rn(x[i + 1], a);
            }
        }
    }
    float s = 0;
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float *o;
    cudaMalloc(&o, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    const char *names[3] = {"FFMA", "FFMA2", "FMUL"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 4, 256>>>(o, 0.999f, 0.001f, iters);
            if (mode == 1) k<1><<<148 * 4, 256>>>(o, 0.999f, 0.001f, iters);
            if (mode == 2) k<2><<<148 * 4, 256>>>(o, 0.999f, 0.001f, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double lane_ops = 148.0 * 4 * 256 * iters * 16;
            if (rep) printf("%s: %.3f ms, %.1f T lane-ops/s (%.2f lane-ops/clk/SM at 1.965 GHz)\n", names[mode], ms,
                            lane_ops / ms / 1e9, lane_ops / (ms * 1e-3) / 1.965e9 / 148);
        }
    }
    return 0;
}
