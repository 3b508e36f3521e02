// K5: fused tile pass for sm_100a (qs_apply_fused).
//
// A pass applies a run of gates with ONE read and ONE write of the register:
// the 2^n amplitudes are cut into 2^(n-K) tiles of 2^K amplitudes, where the
// K tile qubits Q = {0..5} + (K-6 chosen high qubits) hold every PAIR target
// of the pass.  Controls and phase bits may be anywhere (outside Q they are a
// per-tile predicate), so diagonal gates such as the QFT's controlled phases
// fuse into any pass.
//
// Data movement per tile (a persistent CTA loops over tiles):
//   HBM -> smem : TMA tensor copies (cp.async.bulk.tensor.5d, UTMALDG) over a
//                 per-pass 5-D tensor map: dim0 = the 64 contiguous amplitudes
//                 of local qubits 0..5 (box 66: the 2 out-of-bounds elements
//                 are zero-filled, giving one float4 of padding per 512-B
//                 segment so both register layouts below are bank-conflict
//                 free), dims 1-3 = three high tile qubits (size 2, stride
//                 2^q * 8 B), dim4 = the 512-B row index.  2^(K-9) copies of
//                 4.2 KB per tile, completion on an mbarrier (expect_tx).
//   smem <-> registers, one "stage" per register layout; every thread holds
//                 16 float4 = 32 amplitudes and every gate is applied inside a
//                 thread (no shuffles):
//                   LOW  stage: local qubit 0 = float4 half, 1..4 = register
//                                index -> gates on qubits 0..4
//                   HIGH stage: local qubit 0 = float4 half, 4 chosen qubits
//                                >= 5 = register index -> gates on those
//                 Lane / warp ids cover the remaining local qubits.
//   smem -> HBM : the same tensor map, cp.async.bulk.tensor store (UTMASTG;
//                 the padding elements are out of bounds and never written).
// One CTA per SM, warp-specialised: a producer warp drives the TMA for a
// double-buffered tile ring (load of tile i+1 and store of tile i-1 overlap
// the math on tile i; full/done mbarriers hand buffers back and forth) and
// 2^(K-5) compute threads run the register stages.
//
// Ops are applied in circuit order with the same per-pair arithmetic as the
// unfused sweep (common.cuh).  Gate-class specialisations (real entries,
// H-like a==c & d==-b, X) drop only products that are exactly ±0 or exact
// negations, so a fused pass equals the sequence of single-gate sweeps in
// every value (the sign of a zero amplitude is the only freedom).

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.h"

namespace qsb {

namespace {

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
constexpr int kPhaseVariant = 40;

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
    int ncopies;       // TMA copies per tile (2^(K-9))
    int crow[4];       // row-index bit of copy-index bit i
    int n, K, nwbits, nstages, nruns, nops;
    int dry;  // QSB_FUSED_DRY=1: move the tiles, skip the math (ring probe)
    uint64_t ntiles;
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
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gsrc, uint32_t bytes,
                                          uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_store(void *gdst, const void *smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
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
template <int RNEED, bool ODD, int RB>
__device__ __forceinline__ void apply_phase(const FOp &op, float4 (&v)[1 << RB]) {
    const float2 d = make_float2(op.m[6], op.m[7]);
#pragma unroll
    for (int j = 0; j < (1 << RB); ++j) {
        if ((j & RNEED) != RNEED) continue;
        float2 a = lo2(v[j]), b = hi2(v[j]);
        if (!ODD) a = cmul(d, a);
        b = cmul(d, b);
        v[j] = mk4(a, b);
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

__device__ __forceinline__ uint64_t tile_base(uint64_t t, const FParams &p) {
    uint64_t r = 0;
    for (int i = 0; i < p.nruns; ++i)
        r |= ((t >> p.runs[i].src) & ((1ull << p.runs[i].len) - 1ull)) << p.runs[i].dst;
    return r;
}

__device__ __forceinline__ uint32_t padded(uint32_t f) { return f + (f >> 5); }

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int K, int RB>
__global__ void __maxnreg__(RB == 4 ? 168 : 96)
    k_fused(float4 *__restrict__ amps, const __grid_constant__ FParams p) {
    constexpr int kCompute = 1 << (K - 1 - RB);   // compute threads
    constexpr int kSegs = 1 << (K - kLow);        // 512-B segments per tile
    constexpr int kBufF4 = kSegs * 33;            // padded float4 per buffer
    extern __shared__ __align__(128) float4 smem[];
    float4 *buf0 = smem;
    FOp *sops = (FOp *)(smem + kNB * kBufF4);
    __shared__ uint64_t full[kNB], done[kNB];

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
        const CUtensorMap *map = &p.tmap;
        constexpr int kCopyF4 = 8 * 33;  // one 5-D box: 8 padded segments
        constexpr uint32_t kBoxBytes = 8u * 66u * 8u;
        uint64_t pending[kNB];
        int i = 0;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++i) {
            const int b = i % kNB;
            float4 *buf = buf0 + b * kBufF4;
            if (i >= kNB) {  // buffer b still holds tile i-kNB: write it back first
                mbar_wait(&done[b], ((i - kNB) / kNB) & 1);
                const uint32_t row0 = (uint32_t)(pending[b] >> kLow);
                for (int c = lane; c < p.ncopies; c += 32) {
                    uint32_t row = row0;
                    for (int k = 0; k < 4; ++k) row |= (uint32_t)((c >> k) & 1) << p.crow[k];
                    tma_store_5d(map, (int)row, buf + c * kCopyF4);
                }
                bulk_commit();
                bulk_wait_read0();  // buffer b may be overwritten
                __syncwarp();
            }
            const uint64_t base = tile_base(t, p);
            pending[b] = base;
            if (lane == 0) mbar_arrive_expect_tx(&full[b], kBoxBytes * (uint32_t)p.ncopies);
            __syncwarp();
            const uint32_t row0 = (uint32_t)(base >> kLow);
            for (int c = lane; c < p.ncopies; c += 32) {
                uint32_t row = row0;
                for (int k = 0; k < 4; ++k) row |= (uint32_t)((c >> k) & 1) << p.crow[k];
                tma_load_5d(buf + c * kCopyF4, map, (int)row, &full[b]);
            }
        }
        // drain the last (up to) kNB tiles
        for (int k = (i >= kNB ? i - kNB : 0); k < i; ++k) {
            const int b = k % kNB;
            mbar_wait(&done[b], (k / kNB) & 1);
            const uint32_t row0 = (uint32_t)(pending[b] >> kLow);
            for (int c = lane; c < p.ncopies; c += 32) {
                uint32_t row = row0;
                for (int q = 0; q < 4; ++q) row |= (uint32_t)((c >> q) & 1) << p.crow[q];
                tma_store_5d(map, (int)row, buf0 + b * kBufF4 + c * kCopyF4);
            }
            bulk_commit();
        }
        bulk_wait0();
        return;
    }

    // -------------------- compute warps: register stages --------------------
    int i = 0;
    for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++i) {
        const int b = i % kNB;
        float4 *tile = buf0 + b * kBufF4;
        const uint64_t base = tile_base(t, p);
        mbar_wait(&full[b], (i / kNB) & 1);
        for (int s = 0; s < p.nstages; ++s) {
            const FStage &st = p.stages[s];
            uint32_t fb = 0;
#pragma unroll
            for (int q = 0; q < 5; ++q) fb |= (uint32_t)((lane >> q) & 1) << st.lf[q];
            for (int q = 0; q < p.nwbits; ++q) fb |= (uint32_t)((warp >> q) & 1) << st.wf[q];
            const uint32_t pb = padded(fb);
            uint32_t rs[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) rs[r] = padded(1u << st.rf[r]);
            float4 v[1 << RB];
#pragma unroll
            for (int j = 0; j < (1 << RB); ++j) {
                uint32_t a = pb;
#pragma unroll
                for (int r = 0; r < RB; ++r)
                    if (j & (1 << r)) a += rs[r];
                v[j] = tile[a];
            }
            if (!p.dry) {
                for (int o = st.op_begin; o < st.op_end;) {
                    const int variant = sops[o].variant, len = sops[o].run;
                    apply_run<RB>(variant, sops + o, len, (uint32_t)tid, base, v);
                    o += len;
                }
            }
#pragma unroll
            for (int j = 0; j < (1 << RB); ++j) {
                uint32_t a = pb;
#pragma unroll
                for (int r = 0; r < RB; ++r)
                    if (j & (1 << r)) a += rs[r];
                tile[a] = v[j];
            }
            if (s + 1 < p.nstages) named_sync(1, kCompute);
        }
        fence_async_smem();  // generic-proxy smem writes -> visible to the bulk store
        named_sync(1, kCompute);
        if (tid == 0) mbar_arrive(&done[b]);
    }
}

template <int K, int RB>
int launch_fused_k(qs_state *s, const FParams &p) {
    const size_t bufs = (size_t)kNB * (1u << (K - kLow)) * 33u * 16u;
    const size_t smem = bufs + (size_t)p.nops * sizeof(FOp);
    static int configured = -1;
    if (configured < (int)smem) {
        QS_CUDA(cudaFuncSetAttribute(k_fused<K, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(bufs + kMaxOps * sizeof(FOp))));
        configured = (int)(bufs + kMaxOps * sizeof(FOp));
    }
    uint64_t grid = (uint64_t)s->num_sms;
    if (grid > p.ntiles) grid = p.ntiles;
    k_fused<K, RB><<<(unsigned)grid, (1 << (K - 1 - RB)) + 32, smem, s->stream>>>((float4 *)s->amps, p);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

// ---- small registers (n <= 13): the whole state in shared memory ------------
// One CTA loads the register (<= 64 KB), applies every op in order with the
// exact pair/phase arithmetic of the sweep kernels, and writes it back: one
// launch per circuit instead of one per gate, for registers too small to fill
// the GPU anyway.
struct SOp {
    int kind, target;
    uint64_t ctrl_mask;
    float m[8];
};
constexpr int kSmallMaxOps = 640;
constexpr int kSmallMaxQubits = 13;
struct SParams {
    int n, nops;
    SOp ops[kSmallMaxOps];
};
static_assert(sizeof(SParams) < 32000, "kernel parameter block too large");

__global__ void __launch_bounds__(1024) k_small(float2 *__restrict__ amps,
                                                const __grid_constant__ SParams p) {
    extern __shared__ float2 sv[];
    const int N = 1 << p.n;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sv[i] = amps[i];
    __syncthreads();
    for (int o = 0; o < p.nops; ++o) {
        const SOp &op = p.ops[o];
        const uint32_t cm = (uint32_t)op.ctrl_mask;
        if (op.kind == QS_OP_PHASE) {
            const uint32_t mask = cm | (1u << op.target);
            const float2 d = make_float2(op.m[6], op.m[7]);
            for (int i = threadIdx.x; i < N; i += blockDim.x)
                if ((i & mask) == mask) sv[i] = cmul(d, sv[i]);
        } else {
            const Gate2 g = gate_from(op.m);
            const uint32_t tbit = 1u << op.target;
            for (int k = threadIdx.x; k < (N >> 1); k += blockDim.x) {
                const uint32_t a = (uint32_t)insert_zero((uint64_t)k, op.target);
                if ((a & cm) != cm) continue;
                float2 va = sv[a], vb = sv[a | tbit];
                pair_update(g, va, vb);
                sv[a] = va;
                sv[a | tbit] = vb;
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) amps[i] = sv[i];
}

int run_small(qs_state *s, const qs_op *ops, int nops) {
    static bool configured = false;
    if (!configured) {
        QS_CUDA(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(8u << kSmallMaxQubits)));
        configured = true;
    }
    SParams p;
    std::memset(&p, 0, sizeof p);
    p.n = s->num_qubits;
    const int threads = (1 << p.n) >= 2048 ? 1024 : ((1 << p.n) / 2 < 32 ? 32 : (1 << p.n) / 2);
    for (int base = 0; base < nops; base += kSmallMaxOps) {
        p.nops = nops - base < kSmallMaxOps ? nops - base : kSmallMaxOps;
        for (int i = 0; i < p.nops; ++i) {
            const qs_op &op = ops[base + i];
            p.ops[i].kind = op.kind;
            p.ops[i].target = op.target;
            p.ops[i].ctrl_mask = op.ctrl_mask;
            std::memcpy(p.ops[i].m, op.m, sizeof op.m);
        }
        k_small<<<1, threads, 8u << p.n, s->stream>>>(s->amps, p);
        QS_CUDA(cudaGetLastError());
    }
    return QS_OK;
}

int gate_class(const float m[8]) {
    const bool real = m[1] == 0.f && m[3] == 0.f && m[5] == 0.f && m[7] == 0.f;
    if (!real) return kCplx;
    if (m[0] == 0.f && m[6] == 0.f && m[2] == 1.f && m[4] == 1.f) return kSwap;
    if (m[4] == m[0] && m[6] == -m[2]) return kHlike;
    return kReal;
}

// Register layouts (f = local bit - 1; f has K-1 bits; RB register bits).
// An LDS/STS.128 phase serves 8 lanes; with the padded address f + (f >> 5)
// those 8 lanes hit 8 distinct bank quads iff lanes 0..2 vary f0..f2 (same
// padded row) or f5..f7 (distinct padding offsets).
//   LOW : regs f0..f(RB-1), lanes (f5, f6, f7, then the two lowest free bits),
//         warps = the remaining bits
//   HIGH: regs = RB chosen f-bits >= RB, lanes (f0, f1, f2, then the two
//         lowest free bits), warps = the remaining bits
void fill_lanes_warps(FStage &st, int K, int RB, const int *first3) {
    bool used[32] = {false};
    for (int r = 0; r < RB; ++r) used[st.rf[r]] = true;
    for (int i = 0; i < 3; ++i) {
        st.lf[i] = first3[i];
        used[first3[i]] = true;
    }
    int nl = 3, nw = 0;
    for (int f = 0; f < K - 1; ++f) {
        if (used[f]) continue;
        if (nl < 5)
            st.lf[nl++] = f;
        else
            st.wf[nw++] = f;
    }
}

FStage make_low_stage(int K, int RB) {
    FStage st;
    std::memset(&st, 0, sizeof st);
    for (int r = 0; r < RB; ++r) st.rf[r] = r;
    const int first3[3] = {5, 6, 7};
    fill_lanes_warps(st, K, RB, first3);
    return st;
}

FStage make_high_stage(int K, int RB, const std::vector<int> &rbits_f) {
    FStage st;
    std::memset(&st, 0, sizeof st);
    for (int r = 0; r < RB; ++r) st.rf[r] = rbits_f[r];
    const int first3[3] = {0, 1, 2};
    fill_lanes_warps(st, K, RB, first3);
    return st;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link dependency, so the library still loads on a GPU-less build host).
int encode_tile_map(qs_state *s, FParams &p) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        QS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn)
            return set_error(QS_ERR_CUDA, "cuTensorMapEncodeTiled entry point not available");
        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[5] = {64, 2, 2, 2, 1ull << (p.n - kLow)};
    const cuuint64_t strides[4] = {8ull << p.qpos[kLow], 8ull << p.qpos[kLow + 1],
                                   8ull << p.qpos[kLow + 2], 512ull};
    const cuuint32_t box[5] = {66, 2, 2, 2, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void *)s->amps, dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(QS_ERR_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
    p.ncopies = 1 << (p.K - kLow - 3);
    for (int k = 0; k < 4; ++k) p.crow[k] = (kLow + 3 + k < p.K) ? p.qpos[kLow + 3 + k] - kLow : 0;
    return QS_OK;
}

}  // namespace

int run_fused(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops) {
    const int n = s->num_qubits;
    uint64_t tile_mask = 0;
    for (int i = 0; i < ntile; ++i) {
        if (tile_qubits[i] < 0 || tile_qubits[i] >= n)
            return set_error(QS_ERR_INDEX, "tile qubit " + std::to_string(tile_qubits[i]) +
                                               " out of range");
        tile_mask |= 1ull << tile_qubits[i];
    }
    for (int i = 0; i < nops; ++i) {
        const qs_op &op = ops[i];
        if (op.kind != QS_OP_PAIR && op.kind != QS_OP_PHASE)
            return set_error(QS_ERR_VALUE, "unknown op kind");
        if (op.target < 0 || op.target >= n) return set_error(QS_ERR_INDEX, "op target out of range");
        if (n < 64 && (op.ctrl_mask >> n)) return set_error(QS_ERR_INDEX, "op control out of range");
        if ((op.ctrl_mask >> op.target) & 1ull)
            return set_error(QS_ERR_VALUE, "control and target must differ");
        if (op.kind == QS_OP_PAIR && !((tile_mask >> op.target) & 1ull))
            return set_error(QS_ERR_VALUE, "pair-op target " + std::to_string(op.target) +
                                               " is not a tile qubit");
        if (op.kind == QS_OP_PHASE &&
            !(op.m[0] == 1.f && op.m[1] == 0.f && op.m[2] == 0.f && op.m[3] == 0.f &&
              op.m[4] == 0.f && op.m[5] == 0.f))
            return set_error(QS_ERR_VALUE, "phase op needs a == 1 and b == c == 0");
    }
    const int K = __builtin_popcountll(tile_mask);
    const uint64_t low_mask = (1ull << kLow) - 1ull;
    const bool kernel_ok = n >= 10 && K >= 10 && K <= 13 && (tile_mask & low_mask) == low_mask;
    if (!kernel_ok && n <= kSmallMaxQubits) return run_small(s, ops, nops);
    if (!kernel_ok) {
        // Unsupported tile shape on a large register: one sweep per op — the
        // same arithmetic, one HBM pass per op.
        for (int i = 0; i < nops; ++i) {
            const qs_op &op = ops[i];
            int rc = op.kind == QS_OP_PHASE
                         ? launch_phase(s, op.ctrl_mask | (1ull << op.target),
                                        make_float2(op.m[6], op.m[7]))
                         : launch_sweep(s, op.target, op.ctrl_mask, op.m);
            if (rc) return rc;
        }
        return QS_OK;
    }

    FParams p;
    std::memset(&p, 0, sizeof p);
    p.n = n;
    p.K = K;
    // RB = register bits per thread: 4 (16 float4 per thread) by default; 3
    // (8 float4, twice the compute warps) with QSB_FUSED_RB=3 — measured
    // slower on B200 because the per-op overhead scales with the thread count.
    int RB = 4;
    {
        const char *r = std::getenv("QSB_FUSED_RB");
        if (r && *r == '3') RB = 3;
    }
    p.nwbits = K - 6 - RB;
    p.ntiles = 1ull << (n - K);
    {
        const char *d = std::getenv("QSB_FUSED_DRY");
        p.dry = d && *d == '1';
    }
    int local_of[64];
    for (int q = 0, i = 0; q < n; ++q) {
        local_of[q] = -1;
        if ((tile_mask >> q) & 1ull) {
            p.qpos[i] = q;
            local_of[q] = i++;
        }
    }
    {
        int rc = encode_tile_map(s, p);
        if (rc) return rc;
    }
    // tile index bits fill the non-tile qubits in order, as contiguous runs
    for (int q = 0, src = 0; q < n;) {
        if ((tile_mask >> q) & 1ull) {
            ++q;
            continue;
        }
        int len = 0;
        while (q + len < n && !((tile_mask >> (q + len)) & 1ull)) ++len;
        if (p.nruns == kMaxRuns) return set_error(QS_ERR_VALUE, "tile qubit set too fragmented");
        p.runs[p.nruns++] = Run{src, q, len};
        src += len;
        q += len;
    }

    // ---- stage planning -----------------------------------------------------
    // need: 0 = any stage (phase op / target on local qubit 0), 1 = LOW
    // (target on local 1..RB), 2 = HIGH holding the target's f-bit
    auto need_of = [&](const qs_op &op, int *fbit) -> int {
        if (op.kind != QS_OP_PAIR) return 0;
        const int lb = local_of[op.target];
        if (lb == 0) return 0;
        if (lb <= RB) return 1;
        *fbit = lb - 1;
        return 2;
    };
    std::vector<FStage> stages;
    std::vector<FOp> fops;
    int i = 0;
    while (i < nops) {
        // the layout follows the first op that constrains it
        int kind = 1;
        for (int j = i; j < nops; ++j) {
            int f = -1, nd = need_of(ops[j], &f);
            if (nd) {
                kind = nd;
                break;
            }
        }
        FStage st;
        if (kind == 1) {
            st = make_low_stage(K, RB);
        } else {
            std::vector<int> rb;
            for (int j = i; j < nops && (int)rb.size() < RB; ++j) {
                int f = -1, nd = need_of(ops[j], &f);
                if (nd == 1) break;
                if (nd == 2 && std::find(rb.begin(), rb.end(), f) == rb.end()) rb.push_back(f);
            }
            for (int f = RB; f < K - 1 && (int)rb.size() < RB; ++f)
                if (std::find(rb.begin(), rb.end(), f) == rb.end()) rb.push_back(f);
            std::sort(rb.begin(), rb.end());
            st = make_high_stage(K, RB, rb);
        }
        int reg_of[kMaxK], lane_of[kMaxK], warp_of[kMaxK];
        for (int f = 0; f < kMaxK; ++f) reg_of[f] = lane_of[f] = warp_of[f] = -1;
        for (int r = 0; r < RB; ++r) reg_of[st.rf[r]] = r;
        for (int l = 0; l < 5; ++l) lane_of[st.lf[l]] = l;
        for (int w = 0; w < p.nwbits; ++w) warp_of[st.wf[w]] = w;
        st.op_begin = (int)fops.size();
        for (; i < nops; ++i) {
            const qs_op &op = ops[i];
            int f = -1, nd = need_of(op, &f);
            if (nd == 1 && kind != 1) break;
            if (nd == 2 && (kind != 2 || reg_of[f] < 0)) break;
            FOp o;
            std::memset(&o, 0, sizeof o);
            std::memcpy(o.m, op.m, sizeof o.m);
            o.one = 1.0f;
            uint64_t need = op.ctrl_mask;
            if (op.kind == QS_OP_PHASE) need |= 1ull << op.target;
            for (int q = 0; q < n; ++q) {
                if (!((need >> q) & 1ull)) continue;
                const int lb = local_of[q];
                if (lb < 0)
                    o.ext_need |= 1ull << q;
                else if (lb == 0)
                    o.half_need = 1;
                else if (reg_of[lb - 1] >= 0)
                    o.reg_need |= 1u << reg_of[lb - 1];
                else if (lane_of[lb - 1] >= 0)
                    o.tid_need |= 1u << lane_of[lb - 1];
                else
                    o.tid_need |= 1u << (5 + warp_of[lb - 1]);
            }
            const int has_need = o.reg_need != 0 || o.half_need != 0;
            if (op.kind == QS_OP_PHASE) {
                o.variant = kPhaseVariant + (int)o.reg_need * 2 + (o.half_need ? 1 : 0);
            } else {
                const int lb = local_of[op.target];
                const int slot = lb == 0 ? -1 : reg_of[lb - 1];
                o.variant = ((slot + 1) * 4 + gate_class(op.m)) * 2 + has_need;
            }
            fops.push_back(o);
        }
        st.op_end = (int)fops.size();
        stages.push_back(st);
    }

    // ---- launch: consecutive stage groups within the op / stage limits ------
    size_t si = 0;
    while (si < stages.size()) {
        size_t sj = si;
        int nop = 0;
        while (sj < stages.size() && (int)(sj - si) < kMaxStages &&
               (nop + (stages[sj].op_end - stages[sj].op_begin) <= kMaxOps || sj == si)) {
            nop += stages[sj].op_end - stages[sj].op_begin;
            ++sj;
        }
        if (nop > kMaxOps) {  // one huge stage: split its op range
            FStage a = stages[si], b = stages[si];
            a.op_end = a.op_begin + kMaxOps;
            b.op_begin = a.op_end;
            stages[si] = a;
            stages.insert(stages.begin() + si + 1, b);
            continue;
        }
        p.nstages = (int)(sj - si);
        p.nops = nop;
        const int off = stages[si].op_begin;
        for (size_t k = si; k < sj; ++k) {
            p.stages[k - si] = stages[k];
            p.stages[k - si].op_begin -= off;
            p.stages[k - si].op_end -= off;
        }
        std::memcpy(p.ops, fops.data() + off, (size_t)nop * sizeof(FOp));
        for (int k = 0; k < p.nstages; ++k) {  // runs of equal variants, within a stage
            const FStage &st = p.stages[k];
            for (int o = st.op_begin; o < st.op_end;) {
                int e = o + 1;
                while (e < st.op_end && p.ops[e].variant == p.ops[o].variant) ++e;
                p.ops[o].run = e - o;
                o = e;
            }
        }
        int rc;
        switch (K) {
            case 10: rc = RB == 4 ? launch_fused_k<10, 4>(s, p) : launch_fused_k<10, 3>(s, p); break;
            case 11: rc = RB == 4 ? launch_fused_k<11, 4>(s, p) : launch_fused_k<11, 3>(s, p); break;
            case 12: rc = RB == 4 ? launch_fused_k<12, 4>(s, p) : launch_fused_k<12, 3>(s, p); break;
            default: rc = RB == 4 ? launch_fused_k<13, 4>(s, p) : launch_fused_k<13, 3>(s, p); break;
        }
        if (rc) return rc;
        si = sj;
    }
    return QS_OK;
}

}  // namespace qsb
