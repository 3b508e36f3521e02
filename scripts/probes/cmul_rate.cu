// Complex-multiply throughput on the FP32 pipe in the forms the fused pass
// programs use: planar packed (pcmul2) vs interleaved (cmul) vs scalar
// (cmul_s), with the phase as immediates or as registers (predicated
// selection).  8 float4 units per thread = 16 amplitudes, 8 warps / SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1805_00988_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "fused_dev.cuh"
using namespace qsb;
template <int MODE>
__global__ void k(float4 *out, int iters, float dxr, float dyr) {
    float4 v[8];
    for (int i = 0; i < 8; ++i) v[i] = make_float4(threadIdx.x * 1e-3f + i, 0.5f, 0.25f, i * 0.1f);
    const bool on = (threadIdx.x & 2) != 0;
    const float2 dr = make_float2(on ? dxr : 1.f, on ? dyr : 0.f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) v[i] = pcmul2(make_float2(0.99969881772994995117f, 0.024541229009628295898f), v[i]);
            if (MODE == 1) v[i] = pcmul2(dr, v[i]);
            if (MODE == 2) { cmul_s(make_float2(0.99969881772994995117f, 0.024541229009628295898f), v[i].x, v[i].y);
                             cmul_s(make_float2(0.99969881772994995117f, 0.024541229009628295898f), v[i].z, v[i].w); }
            if (MODE == 3) { cmul_s(dr, v[i].x, v[i].y); cmul_s(dr, v[i].z, v[i].w); }
            if (MODE == 4) { const float2 d = make_float2(0.99969881772994995117f, 0.024541229009628295898f);
                             float2 a = cmul(d, make_float2(v[i].x, v[i].y)), b = cmul(d, make_float2(v[i].z, v[i].w));
                             v[i] = make_float4(a.x, a.y, b.x, b.y); }
            if (MODE == 5) { float2 a = cmul(dr, make_float2(v[i].x, v[i].y)), b = cmul(dr, make_float2(v[i].z, v[i].w));
                             v[i] = make_float4(a.x, a.y, b.x, b.y); }
        }
    }
    for (int i = 0; i < 8; ++i) out[(blockIdx.x * blockDim.x + threadIdx.x) * 8 + i] = v[i];
}
int main() {
    float4 *o;
    cudaMalloc(&o, 148ull * 8 * 256 * 8 * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4000;
    const char *names[6] = {"planar pcmul2 imm", "planar pcmul2 reg", "scalar cmul_s imm", "scalar cmul_s reg",
                            "interleaved cmul imm", "interleaved cmul reg"};
    for (int warps = 4; warps <= 8; warps += 4)
    for (int mode = 0; mode < 6; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            const int blocks = 148 * 4 * warps / 8;
            cudaEventRecord(e0);
            switch (mode) {
                case 0: k<0><<<blocks, 256>>>(o, iters, 0.9f, 0.1f); break;
                case 1: k<1><<<blocks, 256>>>(o, iters, 0.9f, 0.1f); break;
                case 2: k<2><<<blocks, 256>>>(o, iters, 0.9f, 0.1f); break;
                case 3: k<3><<<blocks, 256>>>(o, iters, 0.9f, 0.1f); break;
                case 4: k<4><<<blocks, 256>>>(o, iters, 0.9f, 0.1f); break;
                case 5: k<5><<<blocks, 256>>>(o, iters, 0.9f, 0.1f); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double lane_ops = (double)blocks * 256 * iters * 16 * 4;  // 16 amplitudes x 4 ops
            if (rep) printf("warps/SMSP %d  %-22s %.3f ms  %.1f lane-ops/clk/SM\n", warps, names[mode], ms,
                            lane_ops / (ms * 1e-3) / 1.965e9 / 148);
        }
    }
    return 0;
}
