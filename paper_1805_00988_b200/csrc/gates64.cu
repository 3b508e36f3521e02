// complex128 registers (pairsim Precision.DOUBLE, pkg/src/pairsim/state.py:25-42):
// gate sweeps, phase, qubit swap, reset and the single-launch small-register
// pass for sm_100a.
//
// Same pair-update semantics as gates.cu (pkg/src/pairsim/kernel.py:108-165),
// with the gate entries kept in fp64 (kernel.py:118-119 rounds them to the
// state's precision: no rounding for complex128).  numpy's complex128
// multiply on an FMA host has the same form as its complex64 one (re-probed
// here): (g*v).re = fma(g.re, v.re, -rn(g.im*v.im)),
// (g*v).im = fma(g.re, v.im, rn(g.im*v.re)); explicit __d*_rn intrinsics keep
// nvcc/ptxas from contracting anything else.
//
// Layout: one contiguous double2 per amplitude (16 B).  A warp owns a 512-B
// row of 32 amplitudes, so index bits 0..4 are the lane (shuffle path) and
// bits >= 5 the row (two coalesced streams 2^t apart).  Roofline: HBM,
// 32 * 2^n algorithmic bytes per uncontrolled sweep.

#include <cstdlib>
#include <cstring>
#include <memory>

#include "common.cuh"
#include "internal.h"

namespace qsb {

namespace {

constexpr int kThreads = 256;

struct Gate2d {
    double2 a, b, c, d;
};

Gate2d gate_from_d(const double m[8]) {
    Gate2d g;
    g.a = make_double2(m[0], m[1]);
    g.b = make_double2(m[2], m[3]);
    g.c = make_double2(m[4], m[5]);
    g.d = make_double2(m[6], m[7]);
    return g;
}

__device__ __forceinline__ void pair_update_d(const Gate2d &g, double2 &va, double2 &vb) {
    const double2 na = cadd_d(cmul_d(g.a, va), cmul_d(g.b, vb));
    const double2 nb = cadd_d(cmul_d(g.d, vb), cmul_d(g.c, va));
    va = na;
    vb = nb;
}

__device__ __forceinline__ double2 ld_cs(const double2 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_cs(double2 *p, double2 v) { __stcs(p, v); }

// registers with fewer than 6 qubits (less than one row) and QSB_FORCE_SCALAR
__global__ void k_sweep_scalar_d(double2 *__restrict__ amps, uint64_t nitems, FixedBits fb,
                                 uint64_t set_mask, uint64_t tbit, Gate2d g) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nitems;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = deposit(i, fb) | set_mask;
        double2 va = amps[a], vb = amps[a | tbit];
        pair_update_d(g, va, vb);
        amps[a] = va;
        amps[a | tbit] = vb;
    }
}

// target on a row bit (t >= 5): two coalesced 512-B streams 2^t amplitudes apart
template <int U>
__global__ void __launch_bounds__(kThreads) k_sweep_high_d(double2 *__restrict__ s, uint64_t nitems,
                                                           FixedBits fb, uint64_t row_set,
                                                           uint64_t tstride, uint32_t lane_need,
                                                           Gate2d g) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if ((lane & lane_need) != lane_need) return;
    for (uint64_t base = warp * U; base < nitems; base += nwarps * U) {
        double2 x[U], y[U];
        uint64_t ia[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ia[u] = ((deposit(base + u, fb) | row_set) << 5) | lane;
            if (base + u < nitems) {
                x[u] = ld_cs(s + ia[u]);
                y[u] = ld_cs(s + ia[u] + tstride);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u < nitems) {
                pair_update_d(g, x[u], y[u]);
                st_cs(s + ia[u], x[u]);
                st_cs(s + ia[u] + tstride, y[u]);
            }
        }
    }
}

// target on a lane bit (t <= 4): each warp reads one row and exchanges
// amplitudes with lane ^ (1 << t); bit-clear lanes compute a*own + b*partner,
// bit-set lanes d*own + c*partner (the same two products in the same order).
template <int T, int U>
__global__ void __launch_bounds__(kThreads) k_sweep_low_d(double2 *__restrict__ s, uint64_t nitems,
                                                          FixedBits fb, uint64_t row_set,
                                                          uint32_t lane_need, Gate2d g) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool lane_ok = (lane & lane_need) == lane_need;
    const bool upper = (lane >> T) & 1u;
    const double2 g1 = upper ? g.d : g.a, g2 = upper ? g.c : g.b;
    for (uint64_t base = warp * U; base < nitems; base += nwarps * U) {
        double2 x[U];
        uint64_t ia[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ia[u] = ((deposit(base + u, fb) | row_set) << 5) | lane;
            if (base + u < nitems) x[u] = ld_cs(s + ia[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u < nitems) {  // warp-uniform
                double2 y;
                y.x = __shfl_xor_sync(0xffffffffu, x[u].x, 1 << T);
                y.y = __shfl_xor_sync(0xffffffffu, x[u].y, 1 << T);
                x[u] = cadd_d(cmul_d(g1, x[u]), cmul_d(g2, y));
                if (lane_ok) st_cs(s + ia[u], x[u]);
            }
        }
    }
}

// diagonal gate (a == 1, b == c == 0): only amplitudes with every mask bit set
template <int U>
__global__ void __launch_bounds__(kThreads) k_phase_d(double2 *__restrict__ s, uint64_t nitems,
                                                      FixedBits fb, uint64_t set, double2 d) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = tid; base < nitems; base += nthreads * U) {
        double2 x[U];
        uint64_t iv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t item = base + u * nthreads;
            iv[u] = deposit(item, fb) | set;
            if (item < nitems) x[u] = ld_cs(s + iv[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (base + u * nthreads < nitems) st_cs(s + iv[u], cmul_d(d, x[u]));
    }
}

__global__ void k_swap_d(double2 *__restrict__ amps, uint64_t nitems, FixedBits fb, uint64_t b1,
                         uint64_t b2) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nitems;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = deposit(i, fb);
        const double2 x = amps[base | b1], y = amps[base | b2];
        amps[base | b1] = y;
        amps[base | b2] = x;
    }
}

__global__ void k_set_one_d(double2 *amps, uint64_t idx) { amps[idx] = make_double2(1.0, 0.0); }

FixedBits make_fixed_d(const int *pos, int n) {
    FixedBits fb;
    fb.n = n;
    for (int i = 0; i < kMaxFixed; ++i) fb.pos[i] = i < n ? pos[i] : 0;
    for (int i = 1; i < n; ++i)
        for (int j = i; j > 0 && fb.pos[j - 1] > fb.pos[j]; --j) {
            const int t = fb.pos[j];
            fb.pos[j] = fb.pos[j - 1];
            fb.pos[j - 1] = t;
        }
    return fb;
}

unsigned grid_d(uint64_t work_threads) {
    uint64_t want = (work_threads + kThreads - 1) / kThreads;
    if (want > 0x7fffffffull) want = 0x7fffffffull;
    return (unsigned)(want < 1 ? 1 : want);
}

template <int T>
void launch_low_d_t(qs_state *s, uint64_t nitems, FixedBits fb, uint64_t row_set, uint32_t lane_need,
                    const Gate2d &g) {
    constexpr int U = 2;
    k_sweep_low_d<T, U><<<grid_d(((nitems + U - 1) / U) * 32), kThreads, 0, s->stream>>>(
        amps_d(s), nitems, fb, row_set, lane_need, g);
}

// ---- single-launch pass for small registers (n <= 12: 64 KiB of smem) -------
constexpr int kSmallMaxQubitsD = 12;
constexpr int kSmallMaxOpsD = 320;
struct SOpD {
    int kind, target;
    uint64_t ctrl_mask;
    double m[8];
};
struct SParamsD {
    int n, nops;
    SOpD ops[kSmallMaxOpsD];
};
static_assert(sizeof(SParamsD) < 32000, "kernel parameter block too large");

__global__ void __launch_bounds__(1024) k_small_d(double2 *__restrict__ amps,
                                                  const __grid_constant__ SParamsD p) {
    extern __shared__ double2 sv[];
    const int N = 1 << p.n;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sv[i] = amps[i];
    __syncthreads();
    for (int o = 0; o < p.nops; ++o) {
        const SOpD &op = p.ops[o];
        const uint32_t cm = (uint32_t)op.ctrl_mask;
        if (op.kind == QS_OP_PHASE) {
            const uint32_t mask = cm | (1u << op.target);
            const double2 d = make_double2(op.m[6], op.m[7]);
            for (int i = threadIdx.x; i < N; i += blockDim.x)
                if ((i & mask) == mask) sv[i] = cmul_d(d, sv[i]);
        } else {
            Gate2d g;
            g.a = make_double2(op.m[0], op.m[1]);
            g.b = make_double2(op.m[2], op.m[3]);
            g.c = make_double2(op.m[4], op.m[5]);
            g.d = make_double2(op.m[6], op.m[7]);
            const uint32_t tbit = 1u << op.target;
            for (int k = threadIdx.x; k < (N >> 1); k += blockDim.x) {
                const uint32_t a = (uint32_t)insert_zero((uint64_t)k, op.target);
                if ((a & cm) != cm) continue;
                double2 va = sv[a], vb = sv[a | tbit];
                pair_update_d(g, va, vb);
                sv[a] = va;
                sv[a | tbit] = vb;
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) amps[i] = sv[i];
}

}  // namespace

int launch_reset_d(qs_state *s, uint64_t basis) {
    QS_CUDA(cudaMemsetAsync(s->amps, 0, 16ull << s->num_qubits, s->stream));
    k_set_one_d<<<1, 1, 0, s->stream>>>(amps_d(s), basis);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

int launch_phase_d(qs_state *s, uint64_t mask, double2 d) {
    const int n = s->num_qubits;
    int pos[kMaxFixed];
    int np = 0;
    for (int q = 0; q < n; ++q)
        if ((mask >> q) & 1ull) {
            if (np == kMaxFixed) return set_error(QS_ERR_VALUE, "too many control qubits");
            pos[np++] = q;
        }
    const uint64_t nitems = 1ull << (n - np);
    constexpr int U = 2;
    k_phase_d<U><<<grid_d((nitems + U - 1) / U), kThreads, 0, s->stream>>>(
        amps_d(s), nitems, make_fixed_d(pos, np), mask, d);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

int launch_sweep_d(qs_state *s, int target, uint64_t ctrl_mask, const double m[8]) {
    const int n = s->num_qubits;
    const Gate2d g = gate_from_d(m);
    const uint64_t tbit = 1ull << target;
    if (__builtin_popcountll(ctrl_mask) + 1 > kMaxFixed)
        return set_error(QS_ERR_VALUE, "too many control qubits");
    const bool phase = m[0] == 1.0 && m[1] == 0.0 && m[2] == 0.0 && m[3] == 0.0 && m[4] == 0.0 &&
                       m[5] == 0.0;
    const char *np_env = std::getenv("QSB_NO_PHASE");
    if (phase && !(np_env && *np_env == '1')) return launch_phase_d(s, tbit | ctrl_mask, g.d);

    const char *fs = std::getenv("QSB_FORCE_SCALAR");
    if (n < 6 || (fs && *fs == '1')) {
        int pos[kMaxFixed];
        int np = 0;
        pos[np++] = target;
        for (int q = 0; q < n; ++q)
            if ((ctrl_mask >> q) & 1ull) pos[np++] = q;
        const uint64_t nitems = 1ull << (n - np);
        k_sweep_scalar_d<<<grid_d(nitems), kThreads, 0, s->stream>>>(
            amps_d(s), nitems, make_fixed_d(pos, np), ctrl_mask, tbit, g);
        QS_CUDA(cudaGetLastError());
        return QS_OK;
    }
    // controls on row bits (>= 5) shrink the enumeration; lane bits are predicates
    int pos[kMaxFixed];
    int np = 0;
    uint64_t row_set = 0;
    uint32_t lane_need = 0;
    for (int q = 0; q < n; ++q) {
        if (!((ctrl_mask >> q) & 1ull)) continue;
        if (q >= 5) {
            pos[np++] = q - 5;
            row_set |= 1ull << (q - 5);
        } else {
            lane_need |= 1u << q;
        }
    }
    const uint64_t nrows = 1ull << (n - 5);
    if (target >= 5) {
        pos[np++] = target - 5;
        const uint64_t nitems = nrows >> np;
        constexpr int U = 2;
        k_sweep_high_d<U><<<grid_d(((nitems + U - 1) / U) * 32), kThreads, 0, s->stream>>>(
            amps_d(s), nitems, make_fixed_d(pos, np), row_set, (1ull << (target - 5)) * 32ull,
            lane_need, g);
    } else {
        const uint64_t nitems = nrows >> np;
        const FixedBits fb = make_fixed_d(pos, np);
        switch (target) {
            case 0: launch_low_d_t<0>(s, nitems, fb, row_set, lane_need, g); break;
            case 1: launch_low_d_t<1>(s, nitems, fb, row_set, lane_need, g); break;
            case 2: launch_low_d_t<2>(s, nitems, fb, row_set, lane_need, g); break;
            case 3: launch_low_d_t<3>(s, nitems, fb, row_set, lane_need, g); break;
            default: launch_low_d_t<4>(s, nitems, fb, row_set, lane_need, g); break;
        }
    }
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

int launch_swap_d(qs_state *s, int q1, int q2) {
    int pos[2] = {q1, q2};
    const uint64_t nitems = 1ull << (s->num_qubits - 2);
    k_swap_d<<<grid_d(nitems), kThreads, 0, s->stream>>>(amps_d(s), nitems, make_fixed_d(pos, 2),
                                                         1ull << q1, 1ull << q2);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

// Fused pass of a complex128 register: one shared-memory launch per <= 320 ops
// for n <= 12; otherwise the TMA tile pass as a compiled program (fused.cu:
// run_fused_tiles_d) when it is ready, else the ops in order through the
// sweep kernels.  Every op has the sweep arithmetic, so the
// result is the same as applying the ops one by one.
int run_fused_d(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op64 *ops, int nops) {
    const int n = s->num_qubits;
    for (int i = 0; i < nops; ++i) {
        const qs_op64 &op = ops[i];
        if (op.kind != QS_OP_PAIR && op.kind != QS_OP_PHASE) return set_error(QS_ERR_VALUE, "unknown op kind");
        if (op.target < 0 || op.target >= n) return set_error(QS_ERR_INDEX, "op target out of range");
        if (n < 64 && (op.ctrl_mask >> n)) return set_error(QS_ERR_INDEX, "op control out of range");
        if ((op.ctrl_mask >> op.target) & 1ull) return set_error(QS_ERR_VALUE, "control and target must differ");
        if (op.kind == QS_OP_PHASE && !(op.m[0] == 1.0 && op.m[1] == 0.0 && op.m[2] == 0.0 &&
                                        op.m[3] == 0.0 && op.m[4] == 0.0 && op.m[5] == 0.0))
            return set_error(QS_ERR_VALUE, "phase op needs a == 1 and b == c == 0");
    }
    if (n <= kSmallMaxQubitsD) {
        if (int rc = ensure_smem_attr((const void *)k_small_d, (int)(16u << kSmallMaxQubitsD))) return rc;
        // ~27 KB: on the heap, one per call (concurrent callers on other handles)
        std::unique_ptr<SParamsD> holder(new SParamsD());
        SParamsD &p = *holder;
        p.n = n;
        const int threads = (1 << n) >= 2048 ? 1024 : ((1 << n) / 2 < 32 ? 32 : (1 << n) / 2);
        for (int base = 0; base < nops; base += kSmallMaxOpsD) {
            p.nops = nops - base < kSmallMaxOpsD ? nops - base : kSmallMaxOpsD;
            for (int i = 0; i < p.nops; ++i) {
                const qs_op64 &op = ops[base + i];
                p.ops[i].kind = op.kind;
                p.ops[i].target = op.target;
                p.ops[i].ctrl_mask = op.ctrl_mask;
                std::memcpy(p.ops[i].m, op.m, sizeof op.m);
            }
            k_small_d<<<1, threads, 16u << n, s->stream>>>(amps_d(s), p);
            QS_CUDA(cudaGetLastError());
        }
        return QS_OK;
    }
    {  // a compiled tile pass (jit.cu) once its program is ready
        const int rc = run_fused_tiles_d(s, tile_qubits, ntile, ops, nops);
        if (rc == QS_OK) return QS_OK;
        if (rc != 1) return rc;
    }
    for (int i = 0; i < nops; ++i) {
        const qs_op64 &op = ops[i];
        const int rc = op.kind == QS_OP_PHASE
                           ? launch_phase_d(s, op.ctrl_mask | (1ull << op.target), make_double2(op.m[6], op.m[7]))
                           : launch_sweep_d(s, op.target, op.ctrl_mask, op.m);
        if (rc) return rc;
    }
    return QS_OK;
}

}  // namespace qsb
