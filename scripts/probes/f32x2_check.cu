// Probe: packed f32x2 complex multiply/add vs the scalar __f*_rn form, bitwise.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include "common.cuh"
using namespace qsb;
__device__ float2 cmul_s(float2 g, float2 v) {
    return make_float2(__fmaf_rn(g.x, v.x, -__fmul_rn(g.y, v.y)), __fmaf_rn(g.x, v.y, __fmul_rn(g.y, v.x)));
}
__device__ uint32_t hsh(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdull; x^=x>>33; x*=0xc4ceb9fe1a85ec53ull; x^=x>>33; return (uint32_t)x; }
__device__ float rnd(uint64_t i){ uint32_t b=hsh(i); float f=__uint_as_float((b & 0x807fffffu) | ((120u + (b>>27 & 15u))<<23)); return f; }
__global__ void k(unsigned long long* bad, unsigned long long* bad_add, int mode) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    float2 g = make_float2(rnd(4*i), rnd(4*i+1)), v = make_float2(rnd(4*i+2), rnd(4*i+3));
    if (mode == 1) g.y = 0.f;
    if (mode == 2) { g.x = 0.70710677f; g.y = 0.f; }
    float2 a = cmul(g, v), b = cmul_s(g, v);
    if (__float_as_uint(a.x) != __float_as_uint(b.x) || __float_as_uint(a.y) != __float_as_uint(b.y)) atomicAdd(bad, 1ull);
    float2 c = cadd(a, v), d = make_float2(__fadd_rn(b.x, v.x), __fadd_rn(b.y, v.y));
    if (__float_as_uint(c.x) != __float_as_uint(d.x) || __float_as_uint(c.y) != __float_as_uint(d.y)) atomicAdd(bad_add, 1ull);
}
int main() {
    unsigned long long *d; cudaMalloc(&d, 16);
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(d, 0, 16);
        k<<<1 << 16, 256>>>(d, d + 1, mode);
        unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("mode %d: cmul mismatches %llu, cadd mismatches %llu of %d\n", mode, h[0], h[1], 1 << 24);
    }
    return 0;
}
