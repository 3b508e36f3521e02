// Gate sweeps (K1 single-qubit, K2/K3 controlled / doubly-controlled, K4
// phase) for sm_100a.
//
// Reference semantics: pkg/src/pairsim/kernel.py:108-165 — a sweep over the
// 2^(n-1) amplitude pairs (a, b = a | 1<<t) with a = nth_cleared(i, t),
// restricted to pairs whose control bits are 1.  Both amplitudes of a pair are
// read before either is written; pairs are disjoint, so stream order is the
// only barrier needed between sweeps.
//
// Layout in HBM: one contiguous complex64 array; a float4 holds the amplitude
// pair (2j, 2j+1).  A warp owns a 512-byte "row" of 64 amplitudes (32 float4,
// one per lane), which splits the index bits into three domains:
//   bit 0        -> the two halves of a lane's float4         (in-thread)
//   bits 1..5    -> the lane id                               (__shfl_xor_sync)
//   bits >= 6    -> the row index                             (two coalesced streams)
// Only the row bits are enumerated, so every warp access is a full 512-B
// coalesced request; controls on row bits shrink the enumeration (only the
// touched rows are read), controls on lane/half bits become predicates.
//
// Roofline: HBM.  Algorithmic bytes per sweep = 16 * 2^n for an uncontrolled
// gate (each amplitude read once and written once), 8 * 2^n controlled,
// 4 * 2^n doubly-controlled; the phase kernel touches only the amplitudes a
// diagonal gate changes.

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace qsb {

namespace {

constexpr int kThreads = 256;

int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    if (!v || !*v) return dflt;
    return std::atoi(v);
}

// ---------------------------------------------------------------------------
// Scalar path (registers with fewer than 7 qubits, i.e. fewer than two rows):
// one thread per enumerated pair.  Also the bit-for-bit cross-check of the
// vector paths in tests (QSB_FORCE_SCALAR=1).
__global__ void k_sweep_scalar(float2 *__restrict__ amps, uint64_t nitems, FixedBits fb,
                               uint64_t set_mask, uint64_t tbit, Gate2 g) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nitems;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a = deposit(i, fb) | set_mask;
        uint64_t b = a | tbit;
        float2 va = amps[a];
        float2 vb = amps[b];
        pair_update(g, va, vb);
        amps[a] = va;
        amps[b] = vb;
    }
}

// ---------------------------------------------------------------------------
// Target on a row bit (t >= 6): each lane streams float4 x from row R0 and y
// from row R1 = R0 | (1 << (t-6)), i.e. two coalesced 512-B streams 2^t
// amplitudes apart.  U row pairs per warp iteration keep 2U 16-B loads in
// flight per thread.
template <int U>
__global__ void __launch_bounds__(kThreads) k_sweep_high(float4 *__restrict__ s, uint64_t nitems,
                                                         FixedBits fb, uint64_t row_set,
                                                         uint64_t tstride, uint32_t lane_need,
                                                         int comp_ctrl, Gate2 g) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if ((lane & lane_need) != lane_need) return;  // lane fails a control on bits 1..5
    for (uint64_t base = warp * U; base < nitems; base += nwarps * U) {
        float4 x[U], y[U];
        uint64_t ia[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t item = base + u;
            ia[u] = ((deposit(item, fb) | row_set) << 5) | lane;
            if (item < nitems) {
                x[u] = ld_stream(s + ia[u]);
                y[u] = ld_stream(s + ia[u] + tstride);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u < nitems) {
                float2 a0 = make_float2(x[u].x, x[u].y), a1 = make_float2(x[u].z, x[u].w);
                float2 b0 = make_float2(y[u].x, y[u].y), b1 = make_float2(y[u].z, y[u].w);
                if (!comp_ctrl) pair_update(g, a0, b0);
                pair_update(g, a1, b1);
                st_stream(s + ia[u], make_float4(a0.x, a0.y, a1.x, a1.y));
                st_stream(s + ia[u] + tstride, make_float4(b0.x, b0.y, b1.x, b1.y));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Target on a lane / half bit (t <= 5): each warp reads one row (fully
// coalesced) and exchanges float4s with lane ^ (1 << (t-1)) through the
// register file; t == 0 pairs the two halves of one float4.  The gate
// coefficients are selected per lane so the update is divergence-free:
// bit-clear lanes compute a*own + b*partner, bit-set lanes d*own + c*partner.
template <int T, int U>
__global__ void __launch_bounds__(kThreads) k_sweep_low(float4 *__restrict__ s, uint64_t nitems,
                                                        FixedBits fb, uint64_t row_set,
                                                        uint32_t lane_need, int comp_ctrl, Gate2 g) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool lane_ok = (lane & lane_need) == lane_need;
    float2 g1 = g.a, g2 = g.b;
    if (T > 0 && ((lane >> (T - 1)) & 1u)) {
        g1 = g.d;
        g2 = g.c;
    }
    for (uint64_t base = warp * U; base < nitems; base += nwarps * U) {
        float4 x[U];
        uint64_t ia[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ia[u] = ((deposit(base + u, fb) | row_set) << 5) | lane;
            if (base + u < nitems) x[u] = ld_stream(s + ia[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u < nitems) {  // warp-uniform
                if (T == 0) {
                    float2 va = make_float2(x[u].x, x[u].y), vb = make_float2(x[u].z, x[u].w);
                    pair_update(g, va, vb);
                    x[u] = make_float4(va.x, va.y, vb.x, vb.y);
                } else {
                    const int m = 1 << (T > 0 ? T - 1 : 0);
                    float4 y;
                    y.x = __shfl_xor_sync(0xffffffffu, x[u].x, m);
                    y.y = __shfl_xor_sync(0xffffffffu, x[u].y, m);
                    y.z = __shfl_xor_sync(0xffffffffu, x[u].z, m);
                    y.w = __shfl_xor_sync(0xffffffffu, x[u].w, m);
                    float2 o0 = make_float2(x[u].x, x[u].y), o1 = make_float2(x[u].z, x[u].w);
                    if (!comp_ctrl) o0 = lin2(g1, o0, g2, make_float2(y.x, y.y));
                    o1 = lin2(g1, o1, g2, make_float2(y.z, y.w));
                    x[u] = make_float4(o0.x, o0.y, o1.x, o1.y);
                }
                if (lane_ok) st_stream(s + ia[u], x[u]);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Phase kernel (K4): a diagonal gate with a == 1, b == c == 0 only changes the
// amplitudes whose target (and control) bits are all 1: v_b' = d v_b (+ c v_a
// with c == 0, which adds a signed zero and leaves every value unchanged).
// Enumerates the float4s with the required bits set; mask bit 0 restricts the
// update to the odd half.
template <int U>
__global__ void __launch_bounds__(kThreads) k_phase(float4 *__restrict__ s, uint64_t nitems,
                                                    FixedBits fb, uint64_t vset, int odd_only,
                                                    float2 d) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = tid; base < nitems; base += nthreads * U) {
        float4 x[U];
        uint64_t iv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t item = base + u * nthreads;
            iv[u] = deposit(item, fb) | vset;
            if (item < nitems) x[u] = ld_stream(s + iv[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * nthreads < nitems) {
                float2 lo = make_float2(x[u].x, x[u].y), hi = make_float2(x[u].z, x[u].w);
                if (!odd_only) lo = cmul(d, lo);
                hi = cmul(d, hi);
                st_stream(s + iv[u], make_float4(lo.x, lo.y, hi.x, hi.y));
            }
        }
    }
}

__global__ void k_swap(float2 *__restrict__ amps, uint64_t nitems, FixedBits fb, uint64_t b1,
                       uint64_t b2) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nitems;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = deposit(i, fb);
        float2 x = amps[base | b1];
        float2 y = amps[base | b2];
        amps[base | b1] = y;
        amps[base | b2] = x;
    }
}

__global__ void k_set_one(float2 *amps, uint64_t idx) { amps[idx] = make_float2(1.0f, 0.0f); }

FixedBits make_fixed(const int *pos, int n) {
    FixedBits fb;
    fb.n = n;
    for (int i = 0; i < kMaxFixed; ++i) fb.pos[i] = i < n ? pos[i] : 0;
    // insertion sort, ascending (insert_zero must run low -> high)
    for (int i = 1; i < n; ++i)
        for (int j = i; j > 0 && fb.pos[j - 1] > fb.pos[j]; --j) {
            int t = fb.pos[j];
            fb.pos[j] = fb.pos[j - 1];
            fb.pos[j - 1] = t;
        }
    return fb;
}

// One-shot grids (one warp per U items, no grid-stride reuse) measured
// fastest on B200 for these streaming sweeps: 2.43-2.50 ms per 30-qubit sweep
// vs 2.6-2.8 ms with grids capped at 8-32 blocks/SM (scripts/sweep_tune.py).
// QSB_BLOCKS_PER_SM=k caps the grid at k blocks per SM (grid-stride loop).
unsigned grid_for(const qs_state *s, uint64_t work_threads) {
    const int per_sm = env_int("QSB_BLOCKS_PER_SM", 0);
    uint64_t want = (work_threads + kThreads - 1) / kThreads;
    const uint64_t cap = per_sm > 0 ? (uint64_t)s->num_sms * per_sm : 0x7fffffffull;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (unsigned)want;
}

template <int U>
int launch_high(qs_state *s, uint64_t nitems, FixedBits fb, uint64_t row_set, uint64_t tstride,
                uint32_t lane_need, int comp_ctrl, Gate2 g) {
    unsigned grid = grid_for(s, ((nitems + U - 1) / U) * 32);
    k_sweep_high<U><<<grid, kThreads, 0, s->stream>>>((float4 *)s->amps, nitems, fb, row_set,
                                                      tstride, lane_need, comp_ctrl, g);
    return QS_OK;
}

template <int T, int U>
int launch_low_t(qs_state *s, uint64_t nitems, FixedBits fb, uint64_t row_set, uint32_t lane_need,
                 int comp_ctrl, Gate2 g) {
    unsigned grid = grid_for(s, ((nitems + U - 1) / U) * 32);
    k_sweep_low<T, U><<<grid, kThreads, 0, s->stream>>>((float4 *)s->amps, nitems, fb, row_set,
                                                        lane_need, comp_ctrl, g);
    return QS_OK;
}

template <int U>
int launch_low(qs_state *s, int t, uint64_t nitems, FixedBits fb, uint64_t row_set,
               uint32_t lane_need, int comp_ctrl, Gate2 g) {
    switch (t) {
        case 0: return launch_low_t<0, U>(s, nitems, fb, row_set, lane_need, comp_ctrl, g);
        case 1: return launch_low_t<1, U>(s, nitems, fb, row_set, lane_need, comp_ctrl, g);
        case 2: return launch_low_t<2, U>(s, nitems, fb, row_set, lane_need, comp_ctrl, g);
        case 3: return launch_low_t<3, U>(s, nitems, fb, row_set, lane_need, comp_ctrl, g);
        case 4: return launch_low_t<4, U>(s, nitems, fb, row_set, lane_need, comp_ctrl, g);
        default: return launch_low_t<5, U>(s, nitems, fb, row_set, lane_need, comp_ctrl, g);
    }
}

}  // namespace

int launch_reset(qs_state *s, uint64_t basis) {
    if (s->prec == QS_DOUBLE) return launch_reset_d(s, basis);
    QS_CUDA(cudaMemsetAsync(s->amps, 0, 8ull << s->num_qubits, s->stream));
    k_set_one<<<1, 1, 0, s->stream>>>(s->amps, basis);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

int launch_phase(qs_state *s, uint64_t mask, float2 d) {
    const int n = s->num_qubits;
    // vector (float4) index space has n-1 bits; amplitude bit q>=1 -> vector bit q-1
    int pos[kMaxFixed];
    int np = 0;
    uint64_t vset = 0;
    for (int q = 1; q < n; ++q)
        if ((mask >> q) & 1ull) {
            if (np == kMaxFixed) return set_error(QS_ERR_VALUE, "too many control qubits");
            pos[np++] = q - 1;
            vset |= 1ull << (q - 1);
        }
    const int odd_only = (int)(mask & 1ull);
    uint64_t nitems = (n >= 1) ? (1ull << (n - 1 - np)) : 0;
    FixedBits fb = make_fixed(pos, np);
    constexpr int U = 2;
    unsigned grid = grid_for(s, (nitems + U - 1) / U);
    k_phase<U><<<grid, kThreads, 0, s->stream>>>((float4 *)s->amps, nitems, fb, vset, odd_only, d);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

int launch_sweep(qs_state *s, int target, uint64_t ctrl_mask, const float m_in[8]) {
    NvtxRange nvtx_range("qsb sweep");
    const int n = s->num_qubits;
    float mf[8];
    for (int i = 0; i < 8; ++i) mf[i] = m_in[i];
    const float *m = mf;
    const bool is_diag = mf[0] == 1.0f && mf[1] == 0.0f && mf[2] == 0.0f && mf[3] == 0.0f && mf[4] == 0.0f &&
                         mf[5] == 0.0f;
    if (fault_flip_c() && !is_diag) {  // debug fault injection (QSB_FAULT_FLIP_C)
        mf[4] = -mf[4];
        mf[5] = -mf[5];
    }
    const Gate2 g = gate_from(m);
    const uint64_t tbit = 1ull << target;
    int ncontrols = __builtin_popcountll(ctrl_mask);
    if (ncontrols + 1 > kMaxFixed) return set_error(QS_ERR_VALUE, "too many control qubits");

    // Diagonal phase gate (u1 / z / s / t and their controlled forms, the bulk
    // of the QFT): only the amplitudes with every mask bit set change.
    const bool phase = m[0] == 1.0f && m[1] == 0.0f && m[2] == 0.0f && m[3] == 0.0f &&
                       m[4] == 0.0f && m[5] == 0.0f;
    if (phase && !env_int("QSB_NO_PHASE", 0))
        return launch_phase(s, tbit | ctrl_mask, g.d);

    if (n < 7 || env_int("QSB_FORCE_SCALAR", 0)) {
        int pos[kMaxFixed];
        int np = 0;
        pos[np++] = target;
        for (int q = 0; q < n; ++q)
            if ((ctrl_mask >> q) & 1ull) pos[np++] = q;
        FixedBits fb = make_fixed(pos, np);
        uint64_t nitems = 1ull << (n - np);
        unsigned grid = grid_for(s, nitems);
        k_sweep_scalar<<<grid, kThreads, 0, s->stream>>>(s->amps, nitems, fb, ctrl_mask, tbit, g);
        QS_CUDA(cudaGetLastError());
        return QS_OK;
    }

    // split the controls into row bits (>= 6), lane bits (1..5) and half bit (0)
    int pos[kMaxFixed];
    int np = 0;
    uint64_t row_set = 0;
    uint32_t lane_need = 0;
    int comp_ctrl = 0;
    for (int q = 0; q < n; ++q) {
        if (!((ctrl_mask >> q) & 1ull)) continue;
        if (q >= 6) {
            pos[np++] = q - 6;
            row_set |= 1ull << (q - 6);
        } else if (q >= 1) {
            lane_need |= 1u << (q - 1);
        } else {
            comp_ctrl = 1;
        }
    }
    const uint64_t nrows = 1ull << (n - 6);
    const int U = env_int("QSB_SWEEP_U", 2);
    if (target >= 6) {
        pos[np++] = target - 6;
        FixedBits fb = make_fixed(pos, np);
        uint64_t nitems = nrows >> np;
        uint64_t tstride = (1ull << (target - 6)) * 32ull;
        if (U >= 4)
            launch_high<4>(s, nitems, fb, row_set, tstride, lane_need, comp_ctrl, g);
        else if (U == 1)
            launch_high<1>(s, nitems, fb, row_set, tstride, lane_need, comp_ctrl, g);
        else
            launch_high<2>(s, nitems, fb, row_set, tstride, lane_need, comp_ctrl, g);
    } else {
        FixedBits fb = make_fixed(pos, np);
        uint64_t nitems = nrows >> np;
        if (U >= 4)
            launch_low<4>(s, target, nitems, fb, row_set, lane_need, comp_ctrl, g);
        else if (U == 1)
            launch_low<1>(s, target, nitems, fb, row_set, lane_need, comp_ctrl, g);
        else
            launch_low<2>(s, target, nitems, fb, row_set, lane_need, comp_ctrl, g);
    }
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

int launch_swap(qs_state *s, int q1, int q2) {
    const int n = s->num_qubits;
    int pos[2] = {q1, q2};
    FixedBits fb = make_fixed(pos, 2);
    uint64_t nitems = 1ull << (n - 2);
    unsigned grid = grid_for(s, nitems);
    k_swap<<<grid, kThreads, 0, s->stream>>>(s->amps, nitems, fb, 1ull << q1, 1ull << q2);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

}  // namespace qsb
