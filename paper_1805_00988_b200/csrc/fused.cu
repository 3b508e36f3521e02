// K5: fused tile pass for sm_100a (qs_apply_fused).
//
// A pass applies a run of gates with ONE read and ONE write of the register:
// the 2^n amplitudes are cut into 2^(n-K) tiles of 2^K amplitudes, where the
// K tile qubits Q = {0..5} + (K-6 chosen high qubits) are the qubits every
// PAIR op of the pass targets.  Controls and phase bits may be anywhere
// (outside Q they are a per-tile predicate), so diagonal gates such as the
// QFT's controlled phases fuse into any pass.
//
// Data movement per tile (a persistent CTA loops over tiles):
//   HBM -> smem : cp.async.bulk (TMA engine, UBLKCP) of 2^(K-6) contiguous
//                 512-B segments, completion on an mbarrier (expect_tx)
//   smem <-> registers, one "stage" per 4-bit register window: each thread
//                 holds 16 float4 (32 amplitudes).  Local qubit 0 is the
//                 float4 half, local qubits 1..5 are the lane id (gates there
//                 use __shfl_xor_sync), 4 high tile qubits are the register
//                 index and the remaining K-10 are the warp id.  Lanes always
//                 cover 512 contiguous bytes, so every shared-memory access is
//                 bank-conflict free with a dense layout.
//   smem -> HBM : cp.async.bulk store (bulk_group), drained before the next
//                 tile's load reuses the buffer.
// Two CTAs per SM overlap one tile's TMA traffic with the other's math.
//
// Ops are applied in circuit order with the same per-pair arithmetic as the
// unfused sweep (common.cuh), so a fused pass is bit-identical to the
// sequence of single-gate sweeps up to the sign of zero results (real-valued
// gates skip the products with a zero imaginary part; every nonzero value is
// identical).

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace qsb {

namespace {

constexpr int kLow = 6;     // local qubits 0..5 : float4 half + lane id
constexpr int kRegBits = 4; // 16 float4 per thread
constexpr int kMaxK = 14;
constexpr int kMaxWarpBits = kMaxK - kLow - kRegBits;  // 4

enum : int { kPair = 0, kPhase = 1 };
enum : int { kTHalf = 0, kTLane = 1, kTReg = 2 };

// One op, lowered to the layout of the stage it runs in.
struct FOp {
    int kind;         // kPair / kPhase
    int tclass;       // target class (pair): half / lane / reg
    int tidx;         // lane bit index (0..4) or register bit index (0..3)
    int real;         // all four entries real -> cheaper exact product
    uint32_t half_need, lane_need, reg_need, warp_need;  // controls (+ phase bits)
    uint64_t ext_need;                                   // global bits outside the tile
    float m[8];
};

struct FStage {
    int rbit[kRegBits];       // local bit of register bit r (>= 6)
    int wbit[kMaxWarpBits];   // local bit of warp bit w (>= 6)
    int op_begin, op_end;
};

// The whole op table travels as the kernel parameter block (<= 32 KB since
// CUDA 12.1), so consecutive passes need no host synchronisation.
constexpr int kMaxOps = 352;
constexpr int kMaxStages = 32;
struct FParams {
    int n, K, nwbits, nstages;
    uint64_t ntiles;
    uint64_t tile_mask;        // OR of 1 << qpos[i]
    int qpos[kMaxK];           // global qubit of local bit i
    FStage stages[kMaxStages];
    FOp ops[kMaxOps];
};
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
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
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
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// ---- exact products ---------------------------------------------------------
// For a real entry g (g.im == 0): fma(g.re, v.re, -rn(0*v.im)) == rn(g.re*v.re)
// and fma(g.re, v.im, rn(0*v.re)) == rn(g.re*v.im) for every nonzero result.
__device__ __forceinline__ float2 rmul(float g, float2 v) {
    return make_float2(__fmul_rn(g, v.x), __fmul_rn(g, v.y));
}
__device__ __forceinline__ void pair_real(const float *m, float2 &va, float2 &vb) {
    float2 na = cadd(rmul(m[0], va), rmul(m[2], vb));
    float2 nb = cadd(rmul(m[6], vb), rmul(m[4], va));
    va = na;
    vb = nb;
}
__device__ __forceinline__ void pair_any(const FOp &op, float2 &va, float2 &vb) {
    if (op.real) {
        pair_real(op.m, va, vb);
    } else {
        Gate2 g = gate_from(op.m);
        pair_update(g, va, vb);
    }
}
__device__ __forceinline__ float2 lin_any(const FOp &op, bool hi, float2 own, float2 partner) {
    // bit-clear side: a*own + b*partner ; bit-set side: d*own + c*partner
    const float *g1 = hi ? op.m + 6 : op.m + 0;
    const float *g2 = hi ? op.m + 4 : op.m + 2;
    if (op.real) return cadd(rmul(g1[0], own), rmul(g2[0], partner));
    return cadd(cmul(make_float2(g1[0], g1[1]), own), cmul(make_float2(g2[0], g2[1]), partner));
}

__device__ __forceinline__ float2 lo2(float4 v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(float4 v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float4 mk4(float2 a, float2 b) { return make_float4(a.x, a.y, b.x, b.y); }

template <int R>
__device__ __forceinline__ void op_reg(const FOp &op, float4 (&v)[16], bool thread_ok) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j & (1 << R)) continue;
        const int k = j | (1 << R);
        if (!thread_ok || (j & op.reg_need) != op.reg_need) continue;
        float2 a0 = lo2(v[j]), a1 = hi2(v[j]), b0 = lo2(v[k]), b1 = hi2(v[k]);
        if (!op.half_need) pair_any(op, a0, b0);
        pair_any(op, a1, b1);
        v[j] = mk4(a0, a1);
        v[k] = mk4(b0, b1);
    }
}

template <int B>
__device__ __forceinline__ void op_lane(const FOp &op, float4 (&v)[16], bool thread_ok, int lane) {
    const bool hi = (lane >> B) & 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        float4 y;
        y.x = __shfl_xor_sync(0xffffffffu, v[j].x, 1 << B);
        y.y = __shfl_xor_sync(0xffffffffu, v[j].y, 1 << B);
        y.z = __shfl_xor_sync(0xffffffffu, v[j].z, 1 << B);
        y.w = __shfl_xor_sync(0xffffffffu, v[j].w, 1 << B);
        if (!thread_ok || (j & op.reg_need) != op.reg_need) continue;
        float2 o0 = lo2(v[j]), o1 = hi2(v[j]);
        if (!op.half_need) o0 = lin_any(op, hi, o0, lo2(y));
        o1 = lin_any(op, hi, o1, hi2(y));
        v[j] = mk4(o0, o1);
    }
}

__device__ __forceinline__ void op_half(const FOp &op, float4 (&v)[16], bool thread_ok) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (!thread_ok || (j & op.reg_need) != op.reg_need) continue;
        float2 a = lo2(v[j]), b = hi2(v[j]);
        pair_any(op, a, b);
        v[j] = mk4(a, b);
    }
}

__device__ __forceinline__ void op_phase(const FOp &op, float4 (&v)[16], bool thread_ok) {
    const float2 d = make_float2(op.m[6], op.m[7]);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (!thread_ok || (j & op.reg_need) != op.reg_need) continue;
        float2 a = lo2(v[j]), b = hi2(v[j]);
        if (!op.half_need) a = cmul(d, a);
        b = cmul(d, b);
        v[j] = mk4(a, b);
    }
}

__device__ __forceinline__ uint64_t scatter_bits(uint64_t x, const int *pos, int npos) {
    uint64_t r = 0;
    for (int i = 0; i < npos; ++i) r |= ((x >> i) & 1ull) << pos[i];
    return r;
}

// global index of tile t: its bits go to the non-tile qubits, in order
__device__ __forceinline__ uint64_t tile_base(uint64_t t, int n, uint64_t tile_mask) {
    uint64_t r = 0;
    int k = 0;
    for (int q = 0; q < n; ++q)
        if (!((tile_mask >> q) & 1ull)) r |= ((t >> k++) & 1ull) << q;
    return r;
}

template <int K>
__global__ void __launch_bounds__(1 << (K - 5), (K >= 14 ? 1 : 2))
    k_fused(float4 *__restrict__ amps, const __grid_constant__ FParams p) {
    constexpr int kThreads = 1 << (K - 5);
    constexpr int kF4 = 1 << (K - 1);               // float4 per tile
    constexpr int kSegs = 1 << (K - kLow);          // 512-B segments per tile
    constexpr uint32_t kTileBytes = kF4 * 16u;
    extern __shared__ __align__(128) float4 tile[];
    __shared__ uint64_t bar;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();

    // segment h of tile t starts at global amplitude base | scatter(h, qpos[6..])
    const bool issuer = warp == 0;
    uint32_t parity = 0;
    for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const uint64_t base = tile_base(t, p.n, p.tile_mask);
        if (issuer) {
            bulk_wait_read0();  // previous tile's stores have drained this buffer
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&bar, kTileBytes);
            __syncwarp();
            for (int h = lane; h < kSegs; h += 32) {
                const uint64_t g = base | scatter_bits((uint64_t)h, p.qpos + kLow, K - kLow);
                bulk_load(tile + ((size_t)h << (kLow - 1)), amps + (g >> 1), 512u, &bar);
            }
        }
        mbar_wait(&bar, parity);
        parity ^= 1u;

        for (int s = 0; s < p.nstages; ++s) {
            const FStage st = p.stages[s];
            // float4 index of register slot j: lane | warp bits | register bits
            uint32_t fbase = (uint32_t)lane;
            for (int i = 0; i < p.nwbits; ++i)
                fbase |= (uint32_t)((warp >> i) & 1) << (st.wbit[i] - 1);
            uint32_t rs[kRegBits];
#pragma unroll
            for (int r = 0; r < kRegBits; ++r) rs[r] = 1u << (st.rbit[r] - 1);
            float4 v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                uint32_t f = fbase;
#pragma unroll
                for (int r = 0; r < kRegBits; ++r)
                    if (j & (1 << r)) f |= rs[r];
                v[j] = tile[f];
            }
            for (int o = st.op_begin; o < st.op_end; ++o) {
                const FOp op = p.ops[o];
                const bool ok = ((uint32_t)lane & op.lane_need) == op.lane_need &&
                                ((uint32_t)warp & op.warp_need) == op.warp_need &&
                                (base & op.ext_need) == op.ext_need;
                if (op.kind == kPhase) {
                    op_phase(op, v, ok);
                } else if (op.tclass == kTHalf) {
                    op_half(op, v, ok);
                } else if (op.tclass == kTLane) {
                    switch (op.tidx) {
                        case 0: op_lane<0>(op, v, ok, lane); break;
                        case 1: op_lane<1>(op, v, ok, lane); break;
                        case 2: op_lane<2>(op, v, ok, lane); break;
                        case 3: op_lane<3>(op, v, ok, lane); break;
                        default: op_lane<4>(op, v, ok, lane); break;
                    }
                } else {
                    switch (op.tidx) {
                        case 0: op_reg<0>(op, v, ok); break;
                        case 1: op_reg<1>(op, v, ok); break;
                        case 2: op_reg<2>(op, v, ok); break;
                        default: op_reg<3>(op, v, ok); break;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                uint32_t f = fbase;
#pragma unroll
                for (int r = 0; r < kRegBits; ++r)
                    if (j & (1 << r)) f |= rs[r];
                tile[f] = v[j];
            }
            __syncthreads();
        }

        fence_async_smem();  // generic-proxy smem writes -> visible to the bulk store
        __syncthreads();
        if (issuer) {
            for (int h = lane; h < kSegs; h += 32) {
                const uint64_t g = base | scatter_bits((uint64_t)h, p.qpos + kLow, K - kLow);
                bulk_store(amps + (g >> 1), tile + ((size_t)h << (kLow - 1)), 512u);
            }
            bulk_commit();
        }
    }
    if (issuer) bulk_wait0();
    (void)kThreads;
}

template <int K>
int launch_fused_k(qs_state *s, const FParams &p) {
    const size_t smem = (size_t)(1u << (K - 1)) * 16u;
    static bool configured = false;
    if (!configured) {
        QS_CUDA(cudaFuncSetAttribute(k_fused<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        configured = true;
    }
    uint64_t grid = (uint64_t)s->num_sms * 2;
    if (grid > p.ntiles) grid = p.ntiles;
    k_fused<K><<<(unsigned)grid, 1 << (K - 5), smem, s->stream>>>((float4 *)s->amps, p);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

bool is_real(const float m[8]) { return m[1] == 0.f && m[3] == 0.f && m[5] == 0.f && m[7] == 0.f; }

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
    const bool kernel_ok = n >= 10 && K >= 10 && K <= kMaxK && (tile_mask & low_mask) == low_mask;
    if (!kernel_ok) {
        // Registers below 10 qubits (or an unsupported tile shape): apply the
        // ops one sweep at a time — the same arithmetic, one pass per op.
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
    p.nwbits = K - kLow - kRegBits;
    p.ntiles = 1ull << (n - K);
    p.tile_mask = tile_mask;
    int local_of[64];
    for (int q = 0, i = 0; q < n; ++q) {
        local_of[q] = -1;
        if ((tile_mask >> q) & 1ull) {
            p.qpos[i] = q;
            local_of[q] = i++;
        }
    }

    // ---- stage planning: each stage holds 4 high local bits in registers ----
    std::vector<FStage> stages;
    std::vector<FOp> fops;
    const int nhigh = K - kLow;
    auto high_target = [&](const qs_op &op) -> int {
        if (op.kind != QS_OP_PAIR) return -1;
        int lb = local_of[op.target];
        return lb >= kLow ? lb : -1;
    };
    int i = 0;
    while (i < nops) {
        // choose the register window: the next distinct high targets, in order
        std::vector<int> rbits;
        for (int j = i; j < nops && (int)rbits.size() < kRegBits; ++j) {
            int hb = high_target(ops[j]);
            if (hb >= 0 && std::find(rbits.begin(), rbits.end(), hb) == rbits.end())
                rbits.push_back(hb);
        }
        for (int b = kLow; b < K && (int)rbits.size() < kRegBits; ++b)
            if (std::find(rbits.begin(), rbits.end(), b) == rbits.end()) rbits.push_back(b);
        std::sort(rbits.begin(), rbits.end());
        FStage st;
        std::memset(&st, 0, sizeof st);
        int rpos_of[kMaxK], wpos_of[kMaxK];
        for (int b = 0; b < kMaxK; ++b) rpos_of[b] = wpos_of[b] = -1;
        for (int r = 0; r < kRegBits; ++r) {
            st.rbit[r] = rbits[r];
            rpos_of[rbits[r]] = r;
        }
        for (int b = kLow, w = 0; b < K; ++b)
            if (rpos_of[b] < 0) {
                st.wbit[w] = b;
                wpos_of[b] = w++;
            }
        st.op_begin = (int)fops.size();
        // take ops while their pair target is representable in this stage
        for (; i < nops && (int)fops.size() - st.op_begin < kMaxOps; ++i) {
            const qs_op &op = ops[i];
            int hb = high_target(op);
            if (hb >= 0 && rpos_of[hb] < 0) break;
            FOp f;
            std::memset(&f, 0, sizeof f);
            f.kind = op.kind == QS_OP_PHASE ? kPhase : kPair;
            std::memcpy(f.m, op.m, sizeof f.m);
            f.real = is_real(op.m);
            uint64_t need = op.ctrl_mask;
            if (op.kind == QS_OP_PHASE) need |= 1ull << op.target;
            for (int q = 0; q < n; ++q) {
                if (!((need >> q) & 1ull)) continue;
                int lb = local_of[q];
                if (lb < 0)
                    f.ext_need |= 1ull << q;
                else if (lb == 0)
                    f.half_need = 1;
                else if (lb < kLow)
                    f.lane_need |= 1u << (lb - 1);
                else if (rpos_of[lb] >= 0)
                    f.reg_need |= 1u << rpos_of[lb];
                else
                    f.warp_need |= 1u << wpos_of[lb];
            }
            if (op.kind == QS_OP_PAIR) {
                int lb = local_of[op.target];
                if (lb == 0) {
                    f.tclass = kTHalf;
                } else if (lb < kLow) {
                    f.tclass = kTLane;
                    f.tidx = lb - 1;
                } else {
                    f.tclass = kTReg;
                    f.tidx = rpos_of[lb];
                }
            }
            fops.push_back(f);
        }
        st.op_end = (int)fops.size();
        stages.push_back(st);
        (void)nhigh;
    }
    // ---- launch: consecutive stage groups that fit one parameter block ----
    size_t si = 0;
    while (si < stages.size()) {
        size_t sj = si;
        int nop = 0;
        while (sj < stages.size() && (int)(sj - si) < kMaxStages &&
               nop + (stages[sj].op_end - stages[sj].op_begin) <= kMaxOps) {
            nop += stages[sj].op_end - stages[sj].op_begin;
            ++sj;
        }
        p.nstages = (int)(sj - si);
        const int off = stages[si].op_begin;
        for (size_t k = si; k < sj; ++k) {
            p.stages[k - si] = stages[k];
            p.stages[k - si].op_begin -= off;
            p.stages[k - si].op_end -= off;
        }
        std::memcpy(p.ops, fops.data() + off, (size_t)nop * sizeof(FOp));
        int rc;
        switch (K) {
            case 10: rc = launch_fused_k<10>(s, p); break;
            case 11: rc = launch_fused_k<11>(s, p); break;
            case 12: rc = launch_fused_k<12>(s, p); break;
            case 13: rc = launch_fused_k<13>(s, p); break;
            default: rc = launch_fused_k<14>(s, p); break;
        }
        if (rc) return rc;
        si = sj;
    }
    return QS_OK;
}

}  // namespace qsb
