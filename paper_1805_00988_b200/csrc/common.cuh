// Shared device helpers for libqsb200 (sm_100a).
//
// Arithmetic contract: every complex product is evaluated exactly as numpy's
// complex64 SIMD multiply does on an FMA host (SURVEY.md Appendix A.1,
// re-verified by oracle/ tests):
//     (g * v).re = fma(g.re, v.re, -rn(g.im * v.im))
//     (g * v).im = fma(g.re, v.im,  rn(g.im * v.re))
// with the gate entry g as the left operand (pkg/src/pairsim/kernel.py:128-129),
// and the two products of a pair update added component-wise in fp32.
// Explicit rounding (packed .rn f32x2 PTX below) keeps nvcc from re-contracting
// the expression.
#pragma once

#ifdef __CUDACC_RTC__  // NVRTC (run-time compiled pass kernels): no host headers
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
#else
#include <cuda_runtime.h>
#include <stdint.h>

#include "qsb200.h"
#endif

namespace qsb {

// amplitudes per chunk of the exact sampling chain (csrc/measure.cu M1-M6); the
// fused passes' optional chunk-sum epilogue (QS_FUSED_CHUNK_SUMS) uses it too
constexpr int kCdfChunkLog = 12;


struct Gate2 {
    float2 a, b, c, d;
};

__host__ __device__ inline Gate2 gate_from(const float m[8]) {
    Gate2 g;
    g.a = make_float2(m[0], m[1]);
    g.b = make_float2(m[2], m[3]);
    g.c = make_float2(m[4], m[5]);
    g.d = make_float2(m[6], m[7]);
    return g;
}

// Packed fp32 pairs (sm_100a FMUL2 / FFMA2 / FADD2): each lane is an
// independent IEEE round-to-nearest operation, so a complex product needs two
// instructions instead of four with the same bits as the scalar form.  The
// lane swap (v.im, v.re) and the negated broadcast are free operand modifiers.
__device__ __forceinline__ unsigned long long f2_bits(float2 v) {
    return (unsigned long long)__float_as_uint(v.x) | ((unsigned long long)__float_as_uint(v.y) << 32);
}
__device__ __forceinline__ float2 f2_from(unsigned long long b) {
    return make_float2(__uint_as_float((unsigned)b), __uint_as_float((unsigned)(b >> 32)));
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(r);
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
    return f2_from(r);
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(r);
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(r);
}

// (re, im) = (fma(g.re, v.re, rn(-g.im * v.im)), fma(g.re, v.im, rn(g.im * v.re)));
// rn(-x) == -rn(x), so this is numpy's form bit for bit.  The two g.im
// products are scalar FMULs writing a fresh register pair (a packed FMUL2
// would need the lane-swapped (v.im, v.re), which ptxas tends to materialise
// with MOVs), then one FFMA2 with g.re broadcast: 3 instructions, no copies.
__device__ __forceinline__ float2 cmul(float2 g, float2 v) {
    const float2 t = make_float2(__fmul_rn(-g.y, v.y), __fmul_rn(g.y, v.x));
    return f2fma(make_float2(g.x, g.x), v, t);
}

__device__ __forceinline__ float2 cadd(float2 x, float2 y) { return f2add(x, y); }

// complex128 registers: numpy's complex128 multiply has the same form;
// explicit __d*_rn keeps nvcc / ptxas from contracting anything else
__device__ __forceinline__ double2 cmul_d(double2 g, double2 v) {
    return make_double2(__fma_rn(g.x, v.x, -__dmul_rn(g.y, v.y)), __fma_rn(g.x, v.y, __dmul_rn(g.y, v.x)));
}
__device__ __forceinline__ double2 cadd_d(double2 x, double2 y) {
    return make_double2(__dadd_rn(x.x, y.x), __dadd_rn(x.y, y.y));
}

// v_a' = a v_a + b v_b ; v_b' = d v_b + c v_a  (kernel.py:128-129)
__device__ __forceinline__ void pair_update(const Gate2 &g, float2 &va, float2 &vb) {
    float2 na = cadd(cmul(g.a, va), cmul(g.b, vb));
    float2 nb = cadd(cmul(g.d, vb), cmul(g.c, va));
    va = na;
    vb = nb;
}

// Lane-uniform form used by the shuffle path: own' = g1*own + g2*partner with
// (g1, g2) = (a, b) on the bit-clear side and (d, c) on the bit-set side.
__device__ __forceinline__ float2 lin2(float2 g1, float2 own, float2 g2, float2 partner) {
    return cadd(cmul(g1, own), cmul(g2, partner));
}

// Insert a 0 bit at position p (the paper's nth_cleared, kernel.py:31-37).
__device__ __forceinline__ uint64_t insert_zero(uint64_t i, int p) {
    uint64_t lo = i & ((1ull << p) - 1ull);
    return lo | ((i ^ lo) << 1);
}

// Up to kMaxFixed fixed bit positions, sorted ascending.
constexpr int kMaxFixed = 8;
struct FixedBits {
    int n;
    int pos[kMaxFixed];
};

__device__ __forceinline__ uint64_t deposit(uint64_t i, const FixedBits &fb) {
#pragma unroll
    for (int k = 0; k < kMaxFixed; ++k)
        if (k < fb.n) i = insert_zero(i, fb.pos[k]);
    return i;
}

__device__ __forceinline__ float4 ld_stream(const float4 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4 *p, float4 v) { __stcs(p, v); }

}  // namespace qsb
