// Device side of the K5 fused tile pass (see fused.cu for the design notes).
// Compiled twice: ahead of time into libqsb200.so (nvcc, the interpreter
// kernel k_fused) and at run time by NVRTC as the prelude of generated
// straight-line pass kernels (fused.cu: JIT).  Keep it NVRTC-clean: no host
// headers under __CUDACC_RTC__.
#pragma once

#include "common.cuh"

#ifdef __CUDACC_RTC__
typedef struct __align__(64) {
    unsigned long long opaque[16];
} CUtensorMap;
#else
#include <cuda.h>
#endif

namespace qsb {

constexpr int kLow = 6;      // local qubits 0..5 form one 512-B segment
constexpr int kMaxRegBits = 4;  // RB: 2^RB float4 per thread (RB = 3 or 4)
constexpr int kMaxK = 14;
constexpr int kMaxWarpBits = 5;

enum : int { kCplx = 0, kReal = 1, kHlike = 2, kSwap = 3 };

// One op, lowered to the layout of the stage it runs in (48 bytes, staged
// into shared memory once per CTA).
struct __align__(16) FOp {
    int variant;         // see kPhaseVariant
    uint32_t reg_need;   // register-index bits that must be set (warp-uniform)
    uint32_t tid_need;   // thread-id bits (lane | warp << 5) that must be set
    uint32_t half_need;  // odd half only (control / phase bit on local qubit 0)
    uint64_t ext_need;   // global qubits outside the tile that must be 1
    float one;           // == 1.0f, loaded at run time (see rsum / csub)
    int run;             // at a run head: number of consecutive ops with this variant
    float m[8];
};
// pair variants: ((slot + 1) * 4 + class) * 2 + has_need, slot -1 = half;
// phase variants: kPhaseVariant + reg_need * 2 + half_need
constexpr int kPhaseVariant = 64;

struct FStage {
    int rf[kMaxRegBits];   // f-bit (f = local >> 1) of register bit r
    int lf[5];             // f-bit of lane bit i
    int wf[kMaxWarpBits];  // f-bit of warp bit w
    int op_begin, op_end;
};

// Tile index -> global base: contiguous runs of non-tile qubits.
constexpr int kMaxRuns = 16;
struct Run {
    int src, dst, len;
};

constexpr int kMaxOps = 320;
constexpr int kNB = 3;  // tile buffers in the TMA ring
constexpr int kMaxStages = 48;
struct FParams {
    CUtensorMap tmap;  // 64-B aligned, first member
    int ncopies;       // TMA copies per tile (2^(row bits not in box dims 1-3))
    int crow[4];       // row-index bit of copy-index bit i
    int copy_f4;       // padded float4 per copy (2^(box row bits) * 33)
    uint32_t box_bytes;  // bytes one copy moves into shared memory
    int n, K, nwbits, nstages, nruns, nops;
    int dry;    // probes (QSB_FUSED_DRY): 1 skip the ops, 2 also the register stages, 3 also the stores,
                // 4 no HBM traffic at all (compute only; the register content is garbage)
    float one;  // == 1.0f, read at run time (the generated programs' rsum / csub)
    int l2hint;  // TMA copies with an L2 evict_first policy
    int combine;  // generated programs: combine runs of unit-modulus diagonal ops (exact = False)
    // >= 0: the register is |synth_basis> — the compute warps write each tile's
    // contents (zeros, 1 at the basis amplitude) instead of loading them
    // (qs_apply_fused_from_basis: reset + first pass in one HBM write)
    long long synth_basis;
    // non-null (the last launch group of a pass followed by a sample): each
    // tile's |a|^2 row sums (512-B rows of 64 amplitudes) are stored at
    // csum[index >> 6] before the tile is written back; the sampler reduces
    // them to its chunk sums instead of reading the register again
    double *csum;
    uint64_t ntiles;
    // Dynamic tile scheduler: the producers take tiles from this counter
    // (zero at launch; the last CTA to find it exhausted zeroes it again).
    unsigned long long *tile_ctr;
    int qpos[kMaxK];  // global qubit of local bit i
    Run runs[kMaxRuns];
    FStage stages[kMaxStages];
    FOp ops[kMaxOps];  // copied to shared memory once per CTA
};
// The whole table travels as the kernel parameter block (<= 32764 bytes since
// CUDA 12.1), so consecutive passes need no host synchronisation.
static_assert(sizeof(FParams) < 32000, "kernel parameter block too large");

// ---- PTX wrappers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// try_wait suspends in hardware between polls; after ~2^22 failed polls (far
// beyond any legitimate TMA latency) the kernel traps instead of hanging.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    for (uint32_t spins = 0;; ++spins) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred P;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P;\n"
            "}\n"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
        if (ok) return;
        if (spins > (1u << 22)) __trap();
    }
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tma_load_5d(void *smem_dst, const CUtensorMap *map, int row,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %2, %2, %2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(0), "r"(row), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap *map, int row, const void *smem_src) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %1, %1, %1, %2}], [%3];" ::"l"(map),
        "r"(0), "r"(row), "r"(smem_u32(smem_src))
        : "memory");
}
// The same copies with an L2 eviction-priority hint (each amplitude is read
// and written exactly once per pass: evict_first keeps the stream from
// displacing anything else in L2).
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_5d_hint(void *smem_dst, const CUtensorMap *map, int row,
                                                 uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %2, %2, %2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(0), "r"(row), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_5d_hint(const CUtensorMap *map, int row, const void *smem_src,
                                                  uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group.L2::cache_hint"
        " [%0, {%1, %1, %1, %1, %2}], [%3], %4;" ::"l"(map),
        "r"(0), "r"(row), "r"(smem_u32(smem_src)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---- exact pair updates per gate class ----------------------------------------
// real entry g (g.im == 0): fma(g, v.re, -rn(0*v.im)) == rn(g*v.re) and
// fma(g, v.im, rn(0*v.re)) == rn(g*v.im) for every nonzero result.
// ptxas (CUDA 12.9) contracts mul.rn.f32x2 feeding add.rn.f32x2 (and even
// fma.rn.f32x2(x, 1.0, y), which it first folds to an add) into one FFMA2,
// which would round a sum of two products once instead of three times.  The
// sums below are fma(x, one, y) / fma(y, -one, x) with `one` == 1.0f loaded
// from the op table at run time, so ptxas cannot fold them: exactly
// rn(x + y) / rn(x - y), and the products stay separately rounded.  The GPU
// parity tests compare every gate class bit for bit against the oracle.
__device__ __forceinline__ float2 rmul(float g, float2 v) { return f2mul(make_float2(g, g), v); }
__device__ __forceinline__ float2 rsum(float2 x, float2 y, float one) {
    return f2fma(x, make_float2(one, one), y);
}
__device__ __forceinline__ float2 csub(float2 x, float2 y, float one) {
    return f2fma(y, make_float2(-one, -one), x);
}

// A diagonal op inside a conditional block (a lane, warp or tile test):
// scalar FMUL / FFMA (the same four roundings per amplitude as cmul).
// ptxas writes a packed FFMA2 result into its addend's register pair, so
// after a branch every packed-updated pair needs two MOVs back into its home
// registers; the scalar form updates the amplitude in place (no copies).
__device__ __forceinline__ void cmul_s(float2 d, float &re, float &im) {
    const float t0 = __fmul_rn(-d.y, im), t1 = __fmul_rn(d.y, re);
    re = __fmaf_rn(d.x, re, t0);
    im = __fmaf_rn(d.x, im, t1);
}

template <int CLS>
__device__ __forceinline__ void pair_cls(const float *m, float one, float2 &va, float2 &vb) {
    if (CLS == kCplx) {
        float2 na = cadd(cmul(make_float2(m[0], m[1]), va), cmul(make_float2(m[2], m[3]), vb));
        float2 nb = cadd(cmul(make_float2(m[6], m[7]), vb), cmul(make_float2(m[4], m[5]), va));
        va = na;
        vb = nb;
    } else if (CLS == kReal) {
        float2 na = rsum(rmul(m[0], va), rmul(m[2], vb), one);
        float2 nb = rsum(rmul(m[6], vb), rmul(m[4], va), one);
        va = na;
        vb = nb;
    } else if (CLS == kHlike) {
        // c == a, d == -b: c*va == a*va and d*vb == -(b*vb) exactly
        float2 p = rmul(m[0], va), q = rmul(m[2], vb);
        va = rsum(p, q, one);
        vb = csub(p, q, one);
    } else {  // X: a == d == 0, b == c == 1 -> values swap
        float2 t = va;
        va = vb;
        vb = t;
    }
}

__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float4 mk4(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }

// T = register bit of the target (-1: the float4 half, local qubit 0);
// NEED: the op has a control / phase bit on the register index or the half
// (per-j warp-uniform tests); !NEED is the straight-line common case.
template <int T, int CLS, bool NEED, int RB>
__device__ __forceinline__ void apply_pair(const FOp &op, float4 (&v)[1 << RB]) {
    const uint32_t need = NEED ? op.reg_need : 0u;
    const bool odd_only = NEED && op.half_need != 0;
    const float one = op.one;
    float m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = (CLS == kSwap) ? 0.f : op.m[i];
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (T >= 0 && (j & (1 << T))) continue;
        if (NEED && (j & need) != need) continue;  // warp-uniform
        if (T < 0) {
            float2 a = lo2(v[j]), b = hi2(v[j]);
            pair_cls<CLS>(m, one, a, b);
            v[j] = mk4(a, b);
        } else {
            const int k = j | (1 << (T < 0 ? 0 : T));
            float2 a0 = lo2(v[j]), a1 = hi2(v[j]), b0 = lo2(v[k]), b1 = hi2(v[k]);
            if (!odd_only) pair_cls<CLS>(m, one, a0, b0);
            pair_cls<CLS>(m, one, a1, b1);
            v[j] = mk4(a0, a1);
            v[k] = mk4(b0, b1);
        }
    }
}

// Diagonal op: multiply the registers whose index has every bit of RNEED set
// (compile-time pattern) by d; ODD: only the odd half (phase bit on local 0).
// (Always under a per-op test: the scalar in-place form, see phase_cs.)
template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void apply_phase(const FOp &op, float4 (&v)[1 << RB]) {
    const float2 d = make_float2(op.m[6], op.m[7]);
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & RNEED) != RNEED) continue;
        if (!ODD) cmul_s(d, v[j].x, v[j].y);
        cmul_s(d, v[j].z, v[j].w);
    }
}

// Classes with a straight-line (no per-j test) body; the complex and swap
// bodies keep the per-j branch, which bounds ptxas' register demand there.
__device__ constexpr bool kStraight[4] = {false, true, true, false};

__device__ __forceinline__ bool op_ok(const FOp &op, uint32_t tid, uint64_t base) {
    return (tid & op.tid_need) == op.tid_need && (base & op.ext_need) == op.ext_need;
}

template <int T, int C, bool NEED, int RB>
__device__ __forceinline__ void run_pair(const FOp *ops, int len, uint32_t tid, uint64_t base,
                                         float4 (&v)[1 << RB]) {
    for (int k = 0; k < len; ++k)
        if (op_ok(ops[k], tid, base)) apply_pair<T, C, NEED, RB>(ops[k], v);
}

template <int R, bool ODD, int RB>
__device__ __forceinline__ void run_phase(const FOp *ops, int len, uint32_t tid, uint64_t base,
                                          float4 (&v)[1 << RB]) {
    for (int k = 0; k < len; ++k)
        if (op_ok(ops[k], tid, base)) apply_phase<R, ODD, RB>(ops[k], v);
}

// One dispatch per RUN of consecutive ops with the same variant (the host
// sets FOp::run at each run head): nvcc lowers the switch to a compare tree,
// so QFT-style streams of same-pattern phase ops pay for it once per run.
template <int RB>
__device__ __forceinline__ void apply_run(int variant, const FOp *ops, int len, uint32_t tid,
                                          uint64_t base, float4 (&v)[1 << RB]) {
    switch (variant) {
#define QSB_CASE(T, C)                                                                             \
    case (((T) + 1) * 4 + (C)) * 2 + 0:                                                            \
        if constexpr ((T) < RB) run_pair<(T), (C), !kStraight[C], RB>(ops, len, tid, base, v);      \
        break;                                                                                     \
    case (((T) + 1) * 4 + (C)) * 2 + 1:                                                            \
        if constexpr ((T) < RB) run_pair<(T), (C), true, RB>(ops, len, tid, base, v);               \
        break;
#define QSB_CASES(T) QSB_CASE(T, 0) QSB_CASE(T, 1) QSB_CASE(T, 2) QSB_CASE(T, 3)
        QSB_CASES(-1)
        QSB_CASES(0)
        QSB_CASES(1)
        QSB_CASES(2)
        QSB_CASES(3)
#undef QSB_CASES
#undef QSB_CASE
#define QSB_PH(R)                                                                       \
    case kPhaseVariant + (R) * 2 + 0:                                                    \
        if constexpr ((R) < (1 << RB)) run_phase<(R), false, RB>(ops, len, tid, base, v); \
        break;                                                                           \
    case kPhaseVariant + (R) * 2 + 1:                                                    \
        if constexpr ((R) < (1 << RB)) run_phase<(R), true, RB>(ops, len, tid, base, v);  \
        break;
        QSB_PH(0) QSB_PH(1) QSB_PH(2) QSB_PH(3) QSB_PH(4) QSB_PH(5) QSB_PH(6) QSB_PH(7)
        QSB_PH(8) QSB_PH(9) QSB_PH(10) QSB_PH(11) QSB_PH(12) QSB_PH(13) QSB_PH(14) QSB_PH(15)
#undef QSB_PH
        default: break;
    }
}

// Ahead-of-time program: walks the op table staged in shared memory.
struct Interp {
    static constexpr bool kPlanar = false;
    static constexpr bool kOwnsStages = false;  // the generic stage loop in fused_body
    template <int RB>
    static __device__ __forceinline__ void run(int, const FStage &st, const FOp *sops, uint32_t tid,
                                               uint64_t base, float, float4 (&v)[1 << RB]) {
        for (int o = st.op_begin; o < st.op_end;) {
            const int variant = sops[o].variant, len = sops[o].run;
            apply_run<RB>(variant, sops + o, len, tid, base, v);
            o += len;
        }
    }
};

// Compile-time forms for generated programs: target slot T (-1 = half),
// class, register-bit test RNEED and odd-half-only are template constants,
// the gate entries literals of the generated source.
template <int T, int CLS, int RNEED, bool ODD_ONLY, int RB>
__device__ __forceinline__ void pair_ct(const float (&m)[8], float one, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (T >= 0 && (j & (1 << T))) continue;
        if ((j & RNEED) != RNEED) continue;
        if (T < 0) {
            float2 a = lo2(v[j]), b = hi2(v[j]);
            pair_cls<CLS>(m, one, a, b);
            v[j] = mk4(a, b);
        } else {
            const int k = j | (1 << (T < 0 ? 0 : T));
            float2 a0 = lo2(v[j]), a1 = hi2(v[j]), b0 = lo2(v[k]), b1 = hi2(v[k]);
            if (!ODD_ONLY) pair_cls<CLS>(m, one, a0, b0);
            pair_cls<CLS>(m, one, a1, b1);
            v[j] = mk4(a0, a1);
            v[k] = mk4(b0, b1);
        }
    }
}

template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void phase_ct(float2 d, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & RNEED) != RNEED) continue;
        float2 a = lo2(v[j]), b = hi2(v[j]);
        if (!ODD) a = cmul(d, a);
        b = cmul(d, b);
        v[j] = mk4(a, b);
    }
}

// The same diagonal op inside a conditional block (cmul_s, above).
template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void phase_cs(float2 d, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & RNEED) != RNEED) continue;
        if (!ODD) cmul_s(d, v[j].x, v[j].y);
        cmul_s(d, v[j].z, v[j].w);
    }
}

// Predicated forms for ops whose test involves LANE bits (generated
// programs).  A divergent branch around each such op costs a BSSY/BSYNC
// reconvergence and splits the basic blocks ptxas schedules; instead every
// lane runs the body with an operand selected per lane:
// * phase: multiply by d where the test holds and by exactly (1, 0)
//   elsewhere: fma(1, re, -rn(0 * im)) == re and fma(1, im, rn(0 * re)) == im
//   for every finite value (only the sign of a zero result can differ: the
//   same freedom as the class shortcuts above), so the bits equal the
//   branch form;
// * swap (X / CX / CCX): select between the swapped and unswapped values.
template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void phase_sel(bool on, float2 d, float4 (&v)[1 << RB]) {
    const float2 e = make_float2(on ? d.x : 1.0f, on ? d.y : 0.0f);
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & RNEED) != RNEED) continue;
        if (!ODD) cmul_s(e, v[j].x, v[j].y);
        cmul_s(e, v[j].z, v[j].w);
    }
}
// the same with the packed product (FMUL, FMUL, FFMA2 per amplitude)
template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void phase_sel_ct(bool on, float2 d, float4 (&v)[1 << RB]) {
    phase_ct<RNEED, ODD, RB>(make_float2(on ? d.x : 1.0f, on ? d.y : 0.0f), v);
}

template <int T, int RNEED, bool ODD_ONLY, int RB>
__device__ __forceinline__ void swap_sel(bool on, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (T >= 0 && (j & (1 << T))) continue;
        if ((j & RNEED) != RNEED) continue;
        if (T < 0) {  // the two halves of one unit
            const float4 a = v[j];
            v[j] = make_float4(on ? a.z : a.x, on ? a.w : a.y, on ? a.x : a.z, on ? a.y : a.w);
        } else {
            const int k = j | (1 << (T < 0 ? 0 : T));
            const float4 a = v[j], b = v[k];
            if (ODD_ONLY) {
                v[j] = make_float4(a.x, a.y, on ? b.z : a.z, on ? b.w : a.w);
                v[k] = make_float4(b.x, b.y, on ? a.z : b.z, on ? a.w : b.w);
            } else {
                v[j] = make_float4(on ? b.x : a.x, on ? b.y : a.y, on ? b.z : a.z, on ? b.w : a.w);
                v[k] = make_float4(on ? a.x : b.x, on ? a.y : b.y, on ? a.z : b.z, on ? a.w : b.w);
            }
        }
    }
}

// ---- planar register layout (generated programs, phase-heavy passes) --------
// A 16-B unit holds two amplitudes (local qubit 0 = the half): interleaved
// (re0, im0, re1, im1) in memory.  Planar programs keep each unit as
// (re0, re1, im0, im1) in registers, so the real parts of both amplitudes
// form one packed register pair and the imaginary parts another: a complex
// product of both amplitudes is then four packed instructions (FMUL2 x 2,
// FFMA2 x 2) instead of six or eight, with every lane the same IEEE
// operation as the scalar form (bit-identical).  The units are transposed
// once after the first stage's load and back before the last stage's store;
// intermediate stages keep the planar order in shared memory (the unit
// addresses do not change).
__device__ __forceinline__ float4 to_planar(float4 u) { return make_float4(u.x, u.z, u.y, u.w); }
__device__ __forceinline__ float4 from_planar(float4 u) { return make_float4(u.x, u.z, u.y, u.w); }

// both halves multiplied by d: re' = fma(dx, re, -rn(dy im)), im' = fma(dx, im, rn(dy re))
__device__ __forceinline__ float4 pcmul2(float2 d, float4 u) {
    const float2 re = make_float2(u.x, u.y), im = make_float2(u.z, u.w);
    const float2 tr = f2mul(make_float2(-d.y, -d.y), im), ti = f2mul(make_float2(d.y, d.y), re);
    const float2 nr = f2fma(make_float2(d.x, d.x), re, tr), ni = f2fma(make_float2(d.x, d.x), im, ti);
    return make_float4(nr.x, nr.y, ni.x, ni.y);
}

template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void pphase(float2 d, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & RNEED) != RNEED) continue;
        if (ODD)
            cmul_s(d, v[j].y, v[j].w);  // the odd half only: (re1, im1)
        else
            v[j] = pcmul2(d, v[j]);
    }
}

template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void pphase_sel(bool on, float2 d, float4 (&v)[1 << RB]) {
    pphase<RNEED, ODD, RB>(make_float2(on ? d.x : 1.0f, on ? d.y : 0.0f), v);
}

// Combined diagonal run (opt-in, not bit-exact): multiply by e^{2 pi i t / 2^32}
// for an accumulated phase t in fixed-point turns (exact modular sum of the
// run's angles); one complex product per amplitude instead of one per op.
// (cos, sin) of an angle in fixed-point turns, and the product with it
__device__ __forceinline__ float2 turns_sincos(uint32_t t) {
    const float ang = (float)(int)t * 1.46291807926715968e-9f;  // 2 pi / 2^32
    float sn, cs;
    __sincosf(ang, &sn, &cs);
    return make_float2(cs, sn);
}
// product of two unit factors, rounding unconstrained (combined mode only)
__device__ __forceinline__ float2 cmul_any(float2 x, float2 y) {
    return make_float2(x.x * y.x - x.y * y.y, x.x * y.y + x.y * y.x);
}
__device__ __forceinline__ void turns_apply(float2 e, float &re, float &im) {
#ifdef QSB_TURNS_SCALAR
    const float nr = __fmaf_rn(re, e.x, -__fmul_rn(im, e.y));
    im = __fmaf_rn(re, e.y, __fmul_rn(im, e.x));
    re = nr;
#else
    const float2 r = cmul(e, make_float2(re, im));  // packed: FMUL, FMUL, FFMA2
    re = r.x;
    im = r.y;
#endif
}
__device__ __forceinline__ void turns_mul(uint32_t t, float &re, float &im) {
    const float ang = (float)(int)t * 1.46291807926715968e-9f;  // 2 pi / 2^32
    float sn, cs;
    __sincosf(ang, &sn, &cs);
    const float nr = __fmaf_rn(re, cs, -__fmul_rn(im, sn));
    im = __fmaf_rn(re, sn, __fmul_rn(im, cs));
    re = nr;
}

// The planar phase inside a (warp-uniform) branch: scalar in-place FMUL /
// FFMA per component (cmul_s), so the branch leaves every value in its home
// register (packed results land in fresh register pairs, which costs MOVs
// back at the join).
template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void pphase_cs(float2 d, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & RNEED) != RNEED) continue;
        if (!ODD) cmul_s(d, v[j].x, v[j].z);
        cmul_s(d, v[j].y, v[j].w);
    }
}

template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void pphase_sel_cs(bool on, float2 d, float4 (&v)[1 << RB]) {
    pphase_cs<RNEED, ODD, RB>(make_float2(on ? d.x : 1.0f, on ? d.y : 0.0f), v);
}

// Packed class bodies on a planar unit pair (a, b) = both halves of the
// pair's two amplitudes: same per-lane arithmetic as pair_cls.
template <int CLS>
__device__ __forceinline__ void ppair_cls(const float *m, float one, float4 &a, float4 &b) {
    const float2 ar = make_float2(a.x, a.y), ai = make_float2(a.z, a.w);
    const float2 br = make_float2(b.x, b.y), bi = make_float2(b.z, b.w);
    float2 nar, nai, nbr, nbi;
    if (CLS == kCplx) {
        const float4 p = pcmul2(make_float2(m[0], m[1]), a), q = pcmul2(make_float2(m[2], m[3]), b);
        const float4 r = pcmul2(make_float2(m[6], m[7]), b), t = pcmul2(make_float2(m[4], m[5]), a);
        nar = f2add(make_float2(p.x, p.y), make_float2(q.x, q.y));
        nai = f2add(make_float2(p.z, p.w), make_float2(q.z, q.w));
        nbr = f2add(make_float2(r.x, r.y), make_float2(t.x, t.y));
        nbi = f2add(make_float2(r.z, r.w), make_float2(t.z, t.w));
    } else if (CLS == kReal) {
        nar = rsum(rmul(m[0], ar), rmul(m[2], br), one);
        nai = rsum(rmul(m[0], ai), rmul(m[2], bi), one);
        nbr = rsum(rmul(m[6], br), rmul(m[4], ar), one);
        nbi = rsum(rmul(m[6], bi), rmul(m[4], ai), one);
    } else if (CLS == kHlike) {
        const float2 pr = rmul(m[0], ar), pi = rmul(m[0], ai), qr = rmul(m[2], br), qi = rmul(m[2], bi);
        nar = rsum(pr, qr, one);
        nai = rsum(pi, qi, one);
        nbr = csub(pr, qr, one);
        nbi = csub(pi, qi, one);
    } else {
        nar = br, nai = bi, nbr = ar, nbi = ai;
    }
    a = make_float4(nar.x, nar.y, nai.x, nai.y);
    b = make_float4(nbr.x, nbr.y, nbi.x, nbi.y);
}

// pair op on planar registers: T = register slot of the target (-1: the
// half), RNEED register-bit controls, ODD_ONLY a control on the half bit
template <int T, int CLS, int RNEED, bool ODD_ONLY, int RB>
__device__ __forceinline__ void ppair(const float (&m)[8], float one, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (T >= 0 && (j & (1 << T))) continue;
        if ((j & RNEED) != RNEED) continue;
        if (T < 0) {  // the two halves of one unit: (re0, im0) and (re1, im1)
            float2 a = make_float2(v[j].x, v[j].z), b = make_float2(v[j].y, v[j].w);
            pair_cls<CLS>(m, one, a, b);
            v[j] = make_float4(a.x, b.x, a.y, b.y);
        } else {
            const int k = j | (1 << (T < 0 ? 0 : T));
            if (ODD_ONLY) {
                float2 a = make_float2(v[j].y, v[j].w), b = make_float2(v[k].y, v[k].w);
                pair_cls<CLS>(m, one, a, b);
                v[j].y = a.x, v[j].w = a.y, v[k].y = b.x, v[k].w = b.y;
            } else {
                ppair_cls<CLS>(m, one, v[j], v[k]);
            }
        }
    }
}

template <int T, int RNEED, bool ODD_ONLY, int RB>
__device__ __forceinline__ void pswap_sel(bool on, float4 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (T >= 0 && (j & (1 << T))) continue;
        if ((j & RNEED) != RNEED) continue;
        if (T < 0) {
            const float4 a = v[j];  // (re0, re1, im0, im1) -> (re1, re0, im1, im0)
            v[j] = make_float4(on ? a.y : a.x, on ? a.x : a.y, on ? a.w : a.z, on ? a.z : a.w);
        } else {
            const int k = j | (1 << (T < 0 ? 0 : T));
            const float4 a = v[j], b = v[k];
            if (ODD_ONLY) {
                v[j] = make_float4(a.x, on ? b.y : a.y, a.z, on ? b.w : a.w);
                v[k] = make_float4(b.x, on ? a.y : b.y, b.z, on ? a.w : b.w);
            } else {
                v[j] = make_float4(on ? b.x : a.x, on ? b.y : a.y, on ? b.z : a.z, on ? b.w : a.w);
                v[k] = make_float4(on ? a.x : b.x, on ? a.y : b.y, on ? a.z : b.z, on ? a.w : b.w);
            }
        }
    }
}

__device__ __forceinline__ uint64_t tile_base(uint64_t t, const FParams &p) {
    uint64_t r = 0;
    for (int i = 0; i < p.nruns; ++i)
        r |= ((t >> p.runs[i].src) & ((1ull << p.runs[i].len) - 1ull)) << p.runs[i].dst;
    return r;
}

__device__ __forceinline__ uint32_t padded(uint32_t f) { return f + (f >> 5); }
// 128-bit shared-memory accesses for the generated stage loops: with literal
// offsets ptxas otherwise splits a float4 into two LDS.64 / STS.64 (to land
// the halves in the register pairs the packed ops want), which doubles the
// wavefronts and breaks the bank-conflict-free lane triples
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}
__device__ __forceinline__ double2 lds128d(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts128d(uint32_t a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
template <class V>
__device__ __forceinline__ V lds_unit(uint32_t a);
template <>
__device__ __forceinline__ float4 lds_unit<float4>(uint32_t a);
template <>
__device__ __forceinline__ double2 lds_unit<double2>(uint32_t a) {
    return lds128d(a);
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
template <>
__device__ __forceinline__ float4 lds_unit<float4>(uint32_t a) {
    return lds128(a);
}
__device__ __forceinline__ void sts_unit_(uint32_t a, float4 v) { sts128(a, v); }

__device__ __forceinline__ void sts_unit_(uint32_t a, double2 v) { sts128d(a, v); }
template <class V>
__device__ __forceinline__ void sts_unit(uint32_t a, V v) {
    sts_unit_(a, v);
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// A tile is a padded array of 16-B units: a complex64 register packs two
// amplitudes per unit (local qubit 0 = the unit's halves, 64 amplitudes per
// 512-B row), a complex128 register one (32 per row).
template <class V>
struct UnitTraits;
template <>
struct UnitTraits<float4> {
    static constexpr int kLowQ = 6;   // local qubits inside one 512-B row
    static constexpr int kHalf = 1;   // local qubit 0 lives inside the unit
};
template <>
struct UnitTraits<double2> {
    static constexpr int kLowQ = 5;
    static constexpr int kHalf = 0;
};

// complex128 forms for generated programs (generic 2x2, no class shortcuts:
// the sweep's exact arithmetic, pair_update_d in gates64.cu)
template <int T, int RNEED, int RB>
__device__ __forceinline__ void pair_ct_d(const double (&m)[8], double2 (&v)[1 << RB]) {
    const double2 ga = make_double2(m[0], m[1]), gb = make_double2(m[2], m[3]);
    const double2 gc = make_double2(m[4], m[5]), gd = make_double2(m[6], m[7]);
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if (j & (1 << T)) continue;
        if ((j & RNEED) != RNEED) continue;
        const int k = j | (1 << T);
        const double2 a = v[j], b = v[k];
        v[j] = cadd_d(cmul_d(ga, a), cmul_d(gb, b));
        v[k] = cadd_d(cmul_d(gd, b), cmul_d(gc, a));
    }
}

template <int RNEED, int RB>
__device__ __forceinline__ void phase_ct_d(double2 d, double2 (&v)[1 << RB]) {
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j)
        if ((j & RNEED) == RNEED) v[j] = cmul_d(d, v[j]);
}

// The kernel body, shared by the ahead-of-time interpreter kernel (Prog =
// Interp: op table in shared memory, one dispatch per run of ops) and the
// run-time compiled pass kernels (Prog = a generated straight-line program,
// fused.cu: JIT).  Everything but the op application is identical, so both
// give the same bits.
// The sampler's row sums of one finished tile (QS_FUSED_CHUNK_SUMS), by the
// producer warp just before it stores the tile: lane l adds up rows l, l+32,
// ... (32 padded 16-B units each; the 33-unit pitch keeps the lanes on
// distinct bank quads) and stores |a|^2 of the row's 64 amplitudes at
// csum[row index >> 6] — the compute warps' critical path is untouched.
template <int K, int kLowQ>
__device__ __forceinline__ void tile_row_sums(const float4 *buf, uint64_t base, const FParams &p, int lane) {
    constexpr int kRows = 1 << (K - kLowQ);
    for (int r = lane; r < kRows; r += 32) {
        const float4 *row = buf + r * 33;
        float a = 0.f, b = 0.f;
#pragma unroll 8
        for (int j = 0; j < 32; j += 2) {
            const float4 x = row[j], y = row[j + 1];
            a = __fmaf_rn(x.x, x.x, __fmaf_rn(x.y, x.y, __fmaf_rn(x.z, x.z, __fmaf_rn(x.w, x.w, a))));
            b = __fmaf_rn(y.x, y.x, __fmaf_rn(y.y, y.y, __fmaf_rn(y.z, y.z, __fmaf_rn(y.w, y.w, b))));
        }
        uint64_t g = base;
        for (int q = 0; q < K - kLowQ; ++q)
            if ((r >> q) & 1) g |= 1ull << p.qpos[kLowQ + q];
        p.csum[g >> kLowQ] = (double)(a + b);
    }
}

template <int K, int RB, class Prog, class V = float4>
__device__ __forceinline__ void fused_body(float4 *__restrict__ amps, const FParams &p) {
    constexpr int kLowQ = UnitTraits<V>::kLowQ;
    constexpr int kCompute = 1 << (K - UnitTraits<V>::kHalf - RB);  // compute threads
    constexpr int kSegs = 1 << (K - kLowQ);       // 512-B segments per tile
    constexpr int kBufF4 = kSegs * 33;            // padded float4 per buffer
    extern __shared__ __align__(128) float4 smem[];
    float4 *buf0 = smem;
    FOp *sops = (FOp *)(smem + kNB * kBufF4);
    __shared__ uint64_t full[kNB], done[kNB];
    __shared__ unsigned long long tile_id[kNB];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int b = 0; b < kNB; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&done[b], 1);
        }
        fence_mbar_init();
    }
    {  // stage the op table in shared memory
        const int4 *src = (const int4 *)p.ops;
        int4 *dst = (int4 *)sops;
        const int words = p.nops * (int)(sizeof(FOp) / 16);
        for (int i = tid; i < words; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();

    if (warp == kCompute / 32) {
        // ---------------- producer warp: TMA loads and stores ----------------
        // Tiles are handed out dynamically (one atomic per tile): the ops'
        // tile-uniform tests (controls / phase bits outside the tile) make
        // tiles unequal in work, and a static stride gives some CTAs only
        // heavy tiles (e.g. tile-index bits 0-1 are constant per CTA under a
        // stride of 148).  The tile index travels to the compute warps with
        // the buffer (tile_id[b], published by the full-barrier arrival);
        // ~0 ends the loop.
        const CUtensorMap *map = &p.tmap;
        const uint64_t pol = l2_evict_first();
        const int kCopyF4 = p.copy_f4;  // one 5-D box: 2^(box row bits) padded segments
        const uint32_t kBoxBytes = p.box_bytes;
        uint64_t pending[kNB];
        int i = 0;
        for (;; ++i) {
            const int b = i % kNB;
            float4 *buf = buf0 + b * kBufF4;
            // the next tile's index first (warp-wide), so that afterwards each
            // lane moves from its store copy to its load copy on its own: a
            // lane's load into a copy region waits only for ITS store of that
            // region to have been read out (no warp-wide barrier in between)
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(p.tile_ctr, 1ull);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (i >= kNB) {  // buffer b still holds tile i-kNB: write it back first
                mbar_wait(&done[b], ((i - kNB) / kNB) & 1);
                if constexpr (UnitTraits<V>::kHalf)
                    if (p.csum) tile_row_sums<K, kLowQ>(buf, pending[b], p, lane);
                const uint32_t row0 = (uint32_t)(pending[b] >> kLowQ);
                for (int c = lane; c < (p.dry >= 3 ? 0 : p.ncopies); c += 32) {
                    uint32_t row = row0;
                    for (int k = 0; k < 4; ++k) row |= (uint32_t)((c >> k) & 1) << p.crow[k];
                    if (p.l2hint)
                        tma_store_5d_hint(map, (int)row, buf + c * kCopyF4, pol);
                    else
                        tma_store_5d(map, (int)row, buf + c * kCopyF4);
                }
                bulk_commit();
            }
            if (t >= p.ntiles) {
                if (lane == 0) {
                    // every CTA draws exactly one index >= ntiles; the largest
                    // is the counter's last use in this launch
                    if (t == p.ntiles + gridDim.x - 1) *p.tile_ctr = 0ull;
                    tile_id[b] = ~0ull;
                    mbar_arrive(&full[b]);
                }
                break;
            }
            const uint64_t base = tile_base(t, p);
            pending[b] = base;
            if constexpr (UnitTraits<V>::kHalf) {
                if (p.synth_basis >= 0) {  // |basis>: no load — the compute warps write the tile
                    if (i >= kNB) bulk_wait_read0();  // this lane's stores of the buffer are read out
                    __syncwarp();
                    if (lane == 0) {
                        tile_id[b] = t;
                        mbar_arrive(&full[b]);  // the compute warps may overwrite the buffer
                    }
                    continue;
                }
            }
            if (lane == 0) {
                tile_id[b] = t;
                if (p.dry == 4)
                    mbar_arrive(&full[b]);  // probe: compute only, no HBM traffic
                else
                    mbar_arrive_expect_tx(&full[b], kBoxBytes * (uint32_t)p.ncopies);
            }
            const uint32_t row0 = (uint32_t)(base >> kLowQ);
            for (int c = lane; c < (p.dry == 4 ? 0 : p.ncopies); c += 32) {
                uint32_t row = row0;
                for (int k = 0; k < 4; ++k) row |= (uint32_t)((c >> k) & 1) << p.crow[k];
                if (i >= kNB && c == lane) bulk_wait_read0();  // this lane's store of the region is read out
                if (p.l2hint)
                    tma_load_5d_hint(buf + c * kCopyF4, map, (int)row, &full[b], pol);
                else
                    tma_load_5d(buf + c * kCopyF4, map, (int)row, &full[b]);
            }
        }
        // drain the last (up to) kNB - 1 tiles (tile i - kNB was stored above)
        for (int k = (i >= kNB ? i - kNB + 1 : 0); k < i; ++k) {
            const int b = k % kNB;
            mbar_wait(&done[b], (k / kNB) & 1);
            if constexpr (UnitTraits<V>::kHalf)
                if (p.csum) tile_row_sums<K, kLowQ>(buf0 + b * kBufF4, pending[b], p, lane);
            const uint32_t row0 = (uint32_t)(pending[b] >> kLowQ);
            for (int c = lane; c < (p.dry >= 3 ? 0 : p.ncopies); c += 32) {
                uint32_t row = row0;
                for (int q = 0; q < 4; ++q) row |= (uint32_t)((c >> q) & 1) << p.crow[q];
                if (p.l2hint)
                    tma_store_5d_hint(map, (int)row, buf0 + b * kBufF4 + c * p.copy_f4, pol);
                else
                    tma_store_5d(map, (int)row, buf0 + b * kBufF4 + c * p.copy_f4);
            }
            bulk_commit();
        }
        bulk_wait0();
        return;
    }

    // -------------------- compute warps: register stages --------------------
    // Generic loop (interpreter, probes): each thread's padded base per stage
    // depends only on its lane / warp bits, so it is built once per kernel
    // (local memory) instead of per stage and tile.
    uint32_t stage_pb[kMaxStages];
    for (int s = 0; s < p.nstages; ++s) {
        const FStage &st = p.stages[s];
        uint32_t fb = 0;
#pragma unroll
        for (int q = 0; q < 5; ++q) fb |= (uint32_t)((lane >> q) & 1) << st.lf[q];
        for (int q = 0; q < p.nwbits; ++q) fb |= (uint32_t)((warp >> q) & 1) << st.wf[q];
        stage_pb[s] = smem_u32(buf0) + padded(fb) * 16u;
    }
    for (int i = 0;; ++i) {
        const int b = i % kNB;
        float4 *tile = buf0 + b * kBufF4;
        mbar_wait(&full[b], (i / kNB) & 1);
        const uint64_t t = tile_id[b];
        if (t == ~0ull) break;
        const uint64_t base = tile_base(t, p);
        // |synth_basis> (qs_apply_fused_from_basis): the producer loaded
        // nothing; the compute warps write the tile as |basis> (zeros, 1 at
        // the basis amplitude when it lies in this tile) and the stages
        // proceed as after a load — the same threads write and then read, so
        // a named barrier orders them (no producer-written shared memory)
        if constexpr (UnitTraits<V>::kHalf) {
            if (p.synth_basis >= 0) {
                for (int u = tid; u < kBufF4; u += kCompute) tile[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                named_sync(1, kCompute);
                if (tid == 0) {
                    const uint64_t bb = (uint64_t)p.synth_basis;
                    uint64_t tmask = 0, local = 0;
                    for (int q = 0; q < K; ++q) {
                        tmask |= 1ull << p.qpos[q];
                        local |= ((bb >> p.qpos[q]) & 1ull) << q;
                    }
                    if ((bb & ~tmask) == base) {
                        float4 &w = tile[padded((uint32_t)(local >> 1))];
                        if (local & 1u)
                            w.z = 1.f;
                        else
                            w.x = 1.f;
                    }
                }
                named_sync(1, kCompute);
            }
        }
        bool staged = false;
        if constexpr (Prog::kOwnsStages) {  // generated program: literal stage layouts
            if (p.dry == 0 || p.dry == 4) {
                Prog::template run_stages<RB, kCompute>(tile, (uint32_t)tid, base, p.one, sops);
                staged = true;
            }
        }
        for (int s = 0; s < (staged || p.dry == 2 || p.dry == 3 ? 0 : p.nstages); ++s) {
            const FStage &st = p.stages[s];
            // byte address of this thread's unit 0 in buffer b, and the
            // register bits' byte strides
            const uint32_t pb = stage_pb[s] + (uint32_t)b * (uint32_t)kBufF4 * 16u;
            uint32_t rs[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) rs[r] = padded(1u << st.rf[r]) * 16u;
            V v[1 << RB];
#pragma unroll
            for (int j = 0; j < (1 << RB); ++j) {
                uint32_t a = pb;
#pragma unroll
                for (int r = 0; r < RB; ++r)
                    if (j & (1 << r)) a += rs[r];
                v[j] = lds_unit<V>(a);
            }
            if constexpr (Prog::kPlanar && UnitTraits<V>::kHalf) {
                if (s == 0) {
#pragma unroll
                    for (int j = 0; j < (1 << RB); ++j) v[j] = to_planar(v[j]);
                }
            }
            if (!p.dry || p.dry == 4) Prog::template run<RB>(s, st, sops, (uint32_t)tid, base, p.one, v);
            if constexpr (Prog::kPlanar && UnitTraits<V>::kHalf) {
                if (s + 1 == p.nstages) {
#pragma unroll
                    for (int j = 0; j < (1 << RB); ++j) v[j] = from_planar(v[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < (1 << RB); ++j) {
                uint32_t a = pb;
#pragma unroll
                for (int r = 0; r < RB; ++r)
                    if (j & (1 << r)) a += rs[r];
                sts_unit<V>(a, v[j]);
            }
            if (s + 1 < p.nstages) named_sync(1, kCompute);
        }
        fence_async_smem();  // generic-proxy smem writes -> visible to the bulk store
        named_sync(1, kCompute);
        if (tid == 0) mbar_arrive(&done[b]);
    }
}

template <int K, int RB>
__global__ void __maxnreg__(RB == 4 ? 168 : 96)
    k_fused(float4 *__restrict__ amps, const __grid_constant__ FParams p) {
    fused_body<K, RB, Interp>(amps, p);
}

}  // namespace qsb
