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
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "fused_dev.cuh"
#include "internal.h"

namespace qsb {

// run-time compiled pass programs (jit.cu)
bool jit_enabled();
int jit_rb(int dflt);
void *jit_get(int device, const FParams &p, int K, int RB, size_t smem_max, bool wait,
              const qs_op64 *ops64 = nullptr);
void *jit_lookup(int device, const FParams &p, int K, int RB, const qs_op64 *ops64 = nullptr);
int jit_launch(qs_state *s, void *fn, const FParams &p, size_t smem, unsigned grid, unsigned block);

namespace {

// Persistent CTAs per SM: two for K <= 12 tiles (two 3-buffer rings fit in
// shared memory; the second CTA's warps run while the first waits at a stage
// barrier — measured 18% faster on QFT passes), one for K = 13.
// QSB_FUSED_CTAS_PER_SM overrides.
int ctas_per_sm(int K) {
    const char *e = std::getenv("QSB_FUSED_CTAS_PER_SM");
    const int v = e && *e ? std::atoi(e) : (K <= 12 ? 2 : 1);
    return v < 1 ? 1 : (v > 4 ? 4 : v);
}

template <int K, int RB>
int launch_fused_k(qs_state *s, const FParams &p) {
    const size_t bufs = (size_t)kNB * (1u << (K - kLow)) * 33u * 16u;
    const size_t smem = bufs + (size_t)p.nops * sizeof(FOp);
    if (int rc = ensure_smem_attr((const void *)k_fused<K, RB>, (int)(bufs + kMaxOps * sizeof(FOp)))) return rc;
    uint64_t grid = (uint64_t)s->num_sms * (uint64_t)ctas_per_sm(K);
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
    if (int rc = ensure_smem_attr((const void *)k_small, (int)(8u << kSmallMaxQubits))) return rc;
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
// An LDS/STS.128 phase serves 8 lanes; in the padded tile (33-unit rows) f-bit
// i moves the unit address by 1, 2, 4 mod 8 for i = 0, 1, 2 and for i = 5,
// 6, 7 (row strides 33, 66, 132) and by 0 mod 8 otherwise, so the 8 lanes hit
// 8 distinct bank quads iff lanes 0..2 take one f-bit of each class {0,5},
// {1,6}, {2,7}; lanes 3 and 4 are free.  Per stage plan_pass picks RB
// register bits (the stage's targets, then its most-tested bits), lanes 0..2
// from the classes, lanes 3-4 the least-tested free bits, warps the rest.

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
    // complex64: 64 amplitudes (8 B) per 512-B row; complex128: 32 (16 B);
    // either way 64 eight-byte elements per row, padded to 66 in shared
    // memory (box dim 0 runs 2 elements past the tensor's 64: zero-filled on
    // load, skipped on store).  Box dims 1-3 take the first three runs of
    // consecutive qubits among the tile's row bits (<= 8 bits each), so a
    // tile whose row qubits are one run (every H-layer pass) moves in ONE
    // copy; the row bits left over are enumerated by copies (ncopies, crow).
    const int low = s->prec == QS_DOUBLE ? 5 : kLow;
    const uint64_t ab = s->prec == QS_DOUBLE ? 16ull : 8ull;
    cuuint64_t dims[5] = {64, 1, 1, 1, 1ull << (p.n - low)};
    cuuint64_t strides[4] = {512ull, 512ull, 512ull, 512ull};
    cuuint32_t box[5] = {66, 1, 1, 1, 1};
    // QSB_FUSED_RUN_BOXES=0: one row bit per box dim (the round-1 form; probes)
    static const bool run_boxes = [] {
        const char *e = std::getenv("QSB_FUSED_RUN_BOXES");
        return !(e && e[0] == '0');
    }();
    int cov = 0;  // row bits covered by box dims 1-3
    for (int d = 1; d <= 3 && low + cov < p.K; ++d) {
        const int q0 = p.qpos[low + cov];
        int len = 1;
        while (run_boxes && len < 8 && low + cov + len < p.K && p.qpos[low + cov + len] == q0 + len) ++len;
        dims[d] = 1ull << len;
        box[d] = 1u << len;
        strides[d - 1] = ab << q0;
        cov += len;
    }
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void *)s->amps, dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(QS_ERR_CUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
    const int left = p.K - low - cov;  // row bits enumerated by copies
    if (left > 4) return set_error(QS_ERR_VALUE, "tile row bits too fragmented for the copy table");
    p.ncopies = 1 << left;
    p.copy_f4 = (1 << cov) * 33;
    p.box_bytes = (uint32_t)(1u << cov) * 66u * 8u;
    for (int k = 0; k < 4; ++k) p.crow[k] = (k < left) ? p.qpos[low + cov + k] - low : 0;
    return QS_OK;
}

}  // namespace

// Plan a validated pass (tile qubit set, ops in order) for RB register bits
// per thread: stage layouts and lowered ops, split into launch groups within
// the op / stage limits of one kernel parameter block.
static int plan_pass(qs_state *s, uint64_t tile_mask, const qs_op *ops, int nops, int RB,
                     std::vector<FParams> &groups, std::vector<int> *group_offsets = nullptr) {
    const int n = s->num_qubits;
    const int K = __builtin_popcountll(tile_mask);
    // 16-B units: complex64 packs local qubit 0 inside the unit (f = local - 1,
    // K - 1 unit bits); complex128 units hold one amplitude (f = local, K bits)
    const bool dbl = s->prec == QS_DOUBLE;
    const int FB = dbl ? K : K - 1;
    auto f_of = [&](int lb) { return dbl ? lb : lb - 1; };
    auto is_half = [&](int lb) { return !dbl && lb == 0; };
    std::unique_ptr<FParams> holder(new FParams);  // ~28 KB: off the stack
    FParams &p = *holder;
    std::memset(&p, 0, sizeof p);
    p.synth_basis = -1;  // load the tiles (qs_apply_fused_from_basis sets it on the first group)
    p.n = n;
    p.K = K;
    p.nwbits = FB - 5 - RB;
    p.ntiles = 1ull << (n - K);
    p.one = 1.0f;
    if (!s->tile_ctr) {  // first fused pass of this handle: the scheduler's counter
        DeviceGuard guard(s->device);
        QS_CUDA(pool_alloc(s->device, 256, (void **)&s->tile_ctr));  // cached: no cudaFree (device sync) per handle
        QS_CUDA(cudaMemsetAsync(s->tile_ctr, 0, 256, s->stream));
    }
    p.tile_ctr = s->tile_ctr;
    {
        const char *d = std::getenv("QSB_FUSED_DRY");
        p.dry = d && *d >= '1' && *d <= '4' ? *d - '0' : 0;
        const char *h = std::getenv("QSB_FUSED_L2HINT");
        p.l2hint = h && *h == '1';
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
    // need: 0 = any stage (phase op / target on local qubit 0), 2 = a stage
    // holding the target's f-bit in registers
    auto need_of = [&](const qs_op &op, int *fbit) -> int {
        if (op.kind != QS_OP_PAIR) return 0;
        const int lb = local_of[op.target];
        if (is_half(lb)) return 0;
        *fbit = f_of(lb);
        return 2;
    };
    // (1) stage layouts and op ranges: greedy over the PAIR ops in circuit
    // order.  A stage's register bits must hold the f-bit of every pair
    // target in it (half-bit targets are free) and leave one of the triples
    // {f0,f1,f2} / {f5,f6,f7} to lanes 0-2 (bank-conflict-free LDS/STS on
    // the padded layout); a stage ends when the next target does not fit.
    // (Low and high targets share a stage whenever they fit: a layered
    // circuit alternating them used to open a new stage per op, and every
    // stage is a shared-memory round trip of the whole tile.)
    struct Plan {
        std::vector<int> rb;    // register f-bits
        int begin, end, first;  // op range; first pair op with a register target
    };
    // An LDS/STS.128 quarter-warp (lanes 0..7) is bank-conflict-free iff the
    // 8 padded unit addresses differ mod 8.  With 33-unit padded rows, f-bit
    // i adds 1, 2, 4 mod 8 for i = 0, 1, 2 and for i = 5, 6, 7 (the row
    // strides 33, 66, 132) and 0 mod 8 otherwise: lanes 0..2 must take one
    // f-bit from each class {0,5}, {1,6}, {2,7} (8 conflict-free triples).
    // QSB_FUSED_NOBANK=1 (probe): ignore the bank classes — lanes take the
    // least-tested free bits, shared-memory accesses may conflict
    static const bool nobank = [] {
        const char *e = std::getenv("QSB_FUSED_NOBANK");
        return e && e[0] == '1';
    }();
    auto triple_ok = [&](const std::vector<int> &rb) {
        if (nobank) return true;
        for (int c = 0; c < 3; ++c) {
            const bool lo_free = std::find(rb.begin(), rb.end(), c) == rb.end();
            const bool hi_free = FB > c + 5 && std::find(rb.begin(), rb.end(), c + 5) == rb.end();
            if (!lo_free && !hi_free) return false;
        }
        return true;
    };
    // QSB_FUSED_STAGE_PAIRS=k (probe): at most k distinct pair-target bits
    // per register stage, so a phase-heavy pass re-lays its tile more often
    // and each stage's lanes can take bits its phases do not test
    static const int stage_pairs = [] {
        const char *e = std::getenv("QSB_FUSED_STAGE_PAIRS");
        return e && *e ? std::atoi(e) : 0;
    }();
    auto fits = [&](const std::vector<int> &rb, int f) {
        if (std::find(rb.begin(), rb.end(), f) != rb.end()) return true;
        if ((int)rb.size() >= RB) return false;
        std::vector<int> t = rb;
        t.push_back(f);
        return triple_ok(t);
    };
    std::vector<Plan> plans;
    {
        int i = 0;
        while (i < nops) {
            Plan pl;
            pl.begin = i;
            pl.first = nops;
            for (; i < nops; ++i) {
                int f = -1;
                if (!need_of(ops[i], &f)) continue;
                if (!fits(pl.rb, f)) break;
                if (stage_pairs > 0 && (int)pl.rb.size() >= stage_pairs &&
                    std::find(pl.rb.begin(), pl.rb.end(), f) == pl.rb.end())
                    break;
                if (pl.first == nops) pl.first = i;
                if (std::find(pl.rb.begin(), pl.rb.end(), f) == pl.rb.end()) pl.rb.push_back(f);
            }
            pl.end = i;
            plans.push_back(pl);
        }
    }
    // local f-bits an op tests (controls / phase bits; the half bit is free)
    auto test_fbits = [&](const qs_op &op) -> uint32_t {
        uint64_t need = op.ctrl_mask;
        if (op.kind == QS_OP_PHASE) need |= 1ull << op.target;
        uint32_t fb = 0;
        for (int q = 0; q < n; ++q)
            if (((need >> q) & 1ull) && local_of[q] >= 0 && !is_half(local_of[q]))
                fb |= 1u << f_of(local_of[q]);
        return fb;
    };
    auto in_regs = [&](const Plan &pl, uint32_t fb) -> int {
        int c = 0;
        for (int f : pl.rb) c += (fb >> f) & 1u;
        return c;
    };
    // (1b) free register slots take the f-bits the stage's ops test most (a
    // register-bit test is a compile-time mask; a lane-bit test idles half
    // the lanes), then the lowest free bits, always leaving a lane triple
    for (Plan &pl : plans) {
        int uses[32] = {0};
        for (int j = pl.begin; j < pl.end; ++j) {
            const uint32_t fb = test_fbits(ops[j]);
            for (int f = 0; f < FB; ++f) uses[f] += (fb >> f) & 1u;
        }
        std::vector<int> cand;
        for (int f = 0; f < FB; ++f) cand.push_back(f);
        std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) { return uses[x] > uses[y]; });
        for (int f : cand)
            if ((int)pl.rb.size() < RB && fits(pl.rb, f) &&
                std::find(pl.rb.begin(), pl.rb.end(), f) == pl.rb.end())
                pl.rb.push_back(f);
        if ((int)pl.rb.size() != RB) return set_error(QS_ERR_VALUE, "fused pass: no register layout for a stage");
        std::sort(pl.rb.begin(), pl.rb.end());
    }
    // (2) the unconstrained ops (phases, half-bit targets) between the last
    // pair op of stage s-1 and the first of stage s may run in either stage
    // (order is kept).  Move the trailing run to stage s when its bits are
    // register bits there more often: a register-bit test is free (compile-
    // time register mask), a lane-bit test costs a divergent full body.
    for (size_t s = 1; s < plans.size(); ++s) {
        Plan &a = plans[s - 1], &b = plans[s];
        int split = b.begin;
        while (split > a.begin && split - 1 >= a.first) {
            int f = -1;
            if (need_of(ops[split - 1], &f)) break;
            --split;
        }
        if (split < a.first) split = a.first + 1;
        if (split >= b.begin) continue;
        int score_a = 0, score_b = 0;
        for (int j = split; j < b.begin; ++j) {
            const uint32_t fb = test_fbits(ops[j]);
            score_a += in_regs(a, fb);
            score_b += in_regs(b, fb);
        }
        if (score_b > score_a) {
            a.end = split;
            b.begin = split;
        }
    }
    // (3) per stage: lanes 3 and 4 take the free f-bits its ops test least
    // (whole warps skip a failed warp-bit test; lanes diverge)
    std::vector<FStage> stages;
    std::vector<FOp> fops;
    for (const Plan &pl : plans) {
        int uses[32] = {0};
        for (int j = pl.begin; j < pl.end; ++j) {
            const uint32_t fb = test_fbits(ops[j]);
            for (int f = 0; f < FB; ++f) uses[f] += (fb >> f) & 1u;
        }
        FStage st;
        std::memset(&st, 0, sizeof st);
        for (int r = 0; r < RB; ++r) st.rf[r] = pl.rb[r];
        {
            // lanes 0..2: one f-bit of each class {0,5}, {1,6}, {2,7} (bank-
            // conflict-free, triple_ok), the one the stage's ops test less
            // when both are free of register bits
            bool used[32] = {false};
            for (int r = 0; r < RB; ++r) used[st.rf[r]] = true;
            for (int c = 0; c < (nobank ? 0 : 3); ++c) {
                const bool lo_free = !used[c], hi_free = FB > c + 5 && !used[c + 5];
                const int f = (!lo_free || (hi_free && uses[c + 5] < uses[c])) ? c + 5 : c;
                st.lf[c] = f;
                used[f] = true;
            }
            std::vector<int> fr;
            for (int f = 0; f < FB; ++f)
                if (!used[f]) fr.push_back(f);
            std::stable_sort(fr.begin(), fr.end(), [&](int x, int y) { return uses[x] < uses[y]; });
            const int nl = nobank ? 5 : 2;  // lanes still to assign
            for (int l = 0; l < nl; ++l) st.lf[5 - nl + l] = fr[l];
            std::vector<int> wb(fr.begin() + nl, fr.end());
            std::sort(wb.begin(), wb.end());
            for (int w = 0; w < (int)wb.size(); ++w) st.wf[w] = wb[w];
        }
        int reg_of[kMaxK], lane_of[kMaxK], warp_of[kMaxK];
        for (int f = 0; f < kMaxK; ++f) reg_of[f] = lane_of[f] = warp_of[f] = -1;
        for (int r = 0; r < RB; ++r) reg_of[st.rf[r]] = r;
        for (int l = 0; l < 5; ++l) lane_of[st.lf[l]] = l;
        for (int w = 0; w < p.nwbits; ++w) warp_of[st.wf[w]] = w;
        st.op_begin = (int)fops.size();
        for (int i = pl.begin; i < pl.end; ++i) {
            const qs_op &op = ops[i];
            FOp o;
            std::memset(&o, 0, sizeof o);
            std::memcpy(o.m, op.m, sizeof o.m);
            if (fault_flip_c() && op.kind == QS_OP_PAIR) {  // debug fault injection (QSB_FAULT_FLIP_C)
                o.m[4] = -o.m[4];
                o.m[5] = -o.m[5];
            }
            o.one = 1.0f;
            uint64_t need = op.ctrl_mask;
            if (op.kind == QS_OP_PHASE) need |= 1ull << op.target;
            for (int q = 0; q < n; ++q) {
                if (!((need >> q) & 1ull)) continue;
                const int lb = local_of[q];
                if (lb < 0)
                    o.ext_need |= 1ull << q;
                else if (is_half(lb))
                    o.half_need = 1;
                else if (reg_of[f_of(lb)] >= 0)
                    o.reg_need |= 1u << reg_of[f_of(lb)];
                else if (lane_of[f_of(lb)] >= 0)
                    o.tid_need |= 1u << lane_of[f_of(lb)];
                else
                    o.tid_need |= 1u << (5 + warp_of[f_of(lb)]);
            }
            const int has_need = o.reg_need != 0 || o.half_need != 0;
            if (op.kind == QS_OP_PHASE) {
                o.variant = kPhaseVariant + (int)o.reg_need * 2 + (o.half_need ? 1 : 0);
            } else {
                const int lb = local_of[op.target];
                const int slot = is_half(lb) ? -1 : reg_of[f_of(lb)];
                o.variant = ((slot + 1) * 4 + gate_class(o.m)) * 2 + has_need;
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
        if (group_offsets) group_offsets->push_back(off);  // FOp k of a group = op off + k
        for (int k = 0; k < p.nstages; ++k) {  // runs of equal variants, within a stage
            const FStage &st = p.stages[k];
            for (int o = st.op_begin; o < st.op_end;) {
                int e = o + 1;
                while (e < st.op_end && p.ops[e].variant == p.ops[o].variant) ++e;
                p.ops[o].run = e - o;
                o = e;
            }
        }
        if (const char *dump = std::getenv("QSB_FUSED_DUMP")) {  // planner debugging
            if (FILE *f = std::fopen(dump, "a")) {
                std::fprintf(f, "pass K=%d RB=%d nstages=%d nops=%d\n", K, RB, p.nstages, p.nops);
                for (int k = 0; k < p.nstages; ++k) {
                    const FStage &st = p.stages[k];
                    std::fprintf(f, "stage %d %d %d rf", k, st.op_begin, st.op_end);
                    for (int r = 0; r < RB; ++r) std::fprintf(f, " %d", st.rf[r]);
                    std::fprintf(f, " lf");
                    for (int l = 0; l < 5; ++l) std::fprintf(f, " %d", st.lf[l]);
                    std::fprintf(f, " wf");
                    for (int w = 0; w < p.nwbits; ++w) std::fprintf(f, " %d", st.wf[w]);
                    std::fprintf(f, "\n");
                    for (int o = st.op_begin; o < st.op_end; ++o)
                        std::fprintf(f, "op %d %d %u %u %u %llu\n", o, p.ops[o].variant, p.ops[o].reg_need,
                                     p.ops[o].tid_need, p.ops[o].half_need,
                                     (unsigned long long)p.ops[o].ext_need);
                }
                std::fclose(f);
            }
        }
        groups.push_back(p);
        si = sj;
    }
    return QS_OK;
}

int run_fused(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops, int flags,
              long long basis) {
    NvtxRange nvtx_range("qsb fused pass");
    const int n = s->num_qubits;
    // chunk sums for a following sample (qs_sample_prepare laid them out)
    double *const csum = (flags & QS_FUSED_CHUNK_SUMS) && s->prec != QS_DOUBLE ? s->csum_dst : nullptr;
    s->csum_ready = 0;  // the register changes: earlier sums are stale
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
    if (basis >= 0 && !kernel_ok) {  // no tile kernel to write |basis> with: reset, then the ops
        if (int rc = qs_reset(s, (uint64_t)basis)) return rc;
        basis = -1;
    }
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

    // Compiled straight-line programs (jit.cu) once every launch group's
    // program is ready; until then (compiles queued in the background) and
    // without NVRTC, the interpreter kernel.
    const size_t bufs = (size_t)kNB * (1u << (K - kLow)) * 33u * 16u;
    uint64_t grid = (uint64_t)s->num_sms * (uint64_t)ctas_per_sm(K);
    if (grid > (1ull << (n - K))) grid = 1ull << (n - K);
    cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s->stream, &capturing);
    const bool recording = capturing != cudaStreamCaptureStatusNone;  // CUDA graph: no compiles / loads
    if (jit_enabled()) {
        const char *jm = std::getenv("QSB_FUSED_JIT");
        const bool wait = jm && std::atoi(jm) >= 2 && !recording;
        // register bits per thread: 3 (twice the warps, shorter per-op bodies)
        // for phase-dominated passes, 4 otherwise (QSB_FUSED_JIT_RB overrides)
        int nphase = 0;
        for (int i = 0; i < nops; ++i) nphase += ops[i].kind == QS_OP_PHASE;
        const int jrb = jit_rb(2 * nphase > nops ? 3 : 4);
        std::vector<FParams> groups;
        if (plan_pass(s, tile_mask, ops, nops, jrb, groups) == QS_OK) {
            for (FParams &g : groups) g.combine = (flags & QS_FUSED_COMBINE_PHASES) ? 1 : 0;
            groups[0].synth_basis = basis;  // the first launch group writes |basis> (or loads: -1)
            groups.back().csum = csum;       // the last one leaves the sampler's chunk sums
            std::vector<void *> fns;
            for (const FParams &g : groups) {
                void *fn = recording ? jit_lookup(s->device, g, K, jrb)
                                     : jit_get(s->device, g, K, jrb, bufs + kMaxOps * sizeof(FOp), wait);
                if (!fn && wait) break;
                fns.push_back(fn);
            }
            bool all = fns.size() == groups.size();
            for (void *f : fns) all = all && f;
            if (all) {
                for (size_t i = 0; i < groups.size(); ++i) {
                    const int rc = jit_launch(s, fns[i], groups[i], bufs + (size_t)groups[i].nops * sizeof(FOp),
                                              (unsigned)grid, (1u << (K - 1 - jrb)) + 32u);
                    if (rc) return rc;
                }
                s->csum_ready = csum != nullptr;
                return QS_OK;
            }
        }
    }
    // RB = register bits per thread of the interpreter: 4 (16 float4 per
    // thread) by default; 3 (8 float4, twice the compute warps) with
    // QSB_FUSED_RB=3 — measured slower because the per-op overhead scales
    // with the thread count.
    int RB = 4;
    {
        const char *r = std::getenv("QSB_FUSED_RB");
        if (r && *r == '3') RB = 3;
    }
    std::vector<FParams> groups;
    {
        const int rc = plan_pass(s, tile_mask, ops, nops, RB, groups);
        if (rc) return rc;
    }
    groups[0].synth_basis = basis;
    groups.back().csum = csum;
    for (const FParams &g : groups) {
        int rc;
        switch (K) {
            case 10: rc = RB == 4 ? launch_fused_k<10, 4>(s, g) : launch_fused_k<10, 3>(s, g); break;
            case 11: rc = RB == 4 ? launch_fused_k<11, 4>(s, g) : launch_fused_k<11, 3>(s, g); break;
            case 12: rc = RB == 4 ? launch_fused_k<12, 4>(s, g) : launch_fused_k<12, 3>(s, g); break;
            default: rc = RB == 4 ? launch_fused_k<13, 4>(s, g) : launch_fused_k<13, 3>(s, g); break;
        }
        if (rc) return rc;
    }
    s->csum_ready = csum != nullptr;
    return QS_OK;
}

// complex128 registers: a planned pass as a compiled program over 16-B
// units (one amplitude each, csrc/fused_dev.cuh with V = double2).  Returns
// QS_OK once launched, 1 when the programs are not ready yet (the caller runs
// the ops as sweeps, same bits; compiles are queued), or an error code.
int run_fused_tiles_d(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op64 *ops, int nops) {
    const int n = s->num_qubits;
    uint64_t tile_mask = 0;
    for (int i = 0; i < ntile; ++i) {
        if (tile_qubits[i] < 0 || tile_qubits[i] >= n) return 1;
        tile_mask |= 1ull << tile_qubits[i];
    }
    const int K = __builtin_popcountll(tile_mask);
    if (n < 13 || K < 10 || K > 12 || (tile_mask & 31ull) != 31ull || !jit_enabled()) return 1;
    for (int i = 0; i < nops; ++i)
        if (ops[i].kind == QS_OP_PAIR && !((tile_mask >> ops[i].target) & 1ull)) return 1;
    std::vector<qs_op> ops32((size_t)nops);
    int nphase = 0;
    for (int i = 0; i < nops; ++i) {
        ops32[i].kind = ops[i].kind;
        ops32[i].target = ops[i].target;
        ops32[i].ctrl_mask = ops[i].ctrl_mask;
        for (int k = 0; k < 8; ++k) ops32[i].m[k] = (float)ops[i].m[k];
        nphase += ops[i].kind == QS_OP_PHASE;
    }
    const int RB = jit_rb(2 * nphase > nops ? 3 : 4);
    std::vector<FParams> groups;
    std::vector<int> offs;
    int rc = plan_pass(s, tile_mask, ops32.data(), nops, RB, groups, &offs);
    if (rc) return rc;
    cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s->stream, &capturing);
    const bool recording = capturing != cudaStreamCaptureStatusNone;
    const char *jm = std::getenv("QSB_FUSED_JIT");
    const bool wait = jm && std::atoi(jm) >= 2 && !recording;
    const size_t bufs = (size_t)kNB * (1u << (K - 5)) * 33u * 16u;
    std::vector<void *> fns;
    bool all = true;
    for (size_t g = 0; g < groups.size(); ++g) {
        void *f = recording ? jit_lookup(s->device, groups[g], K, RB, ops + offs[g])
                            : jit_get(s->device, groups[g], K, RB, bufs + kMaxOps * sizeof(FOp), wait, ops + offs[g]);
        all = all && f;
        fns.push_back(f);
    }
    if (!all) return 1;
    uint64_t grid = (uint64_t)s->num_sms;
    if (grid > (1ull << (n - K))) grid = 1ull << (n - K);
    for (size_t g = 0; g < groups.size(); ++g) {
        FParams q = groups[g];
        q.nops = 0;  // the program carries the entries: no op table to stage
        rc = jit_launch(s, fns[g], q, bufs, (unsigned)grid, (1u << (K - RB)) + 32u);
        if (rc) return rc;
    }
    return QS_OK;
}

}  // namespace qsb
