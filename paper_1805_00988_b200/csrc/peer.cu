// Global-qubit gates of sharded registers as ONE kernel over peer memory.
//
// A register sharded on its top g qubits keeps rank r's slice in r's HBM.  A
// gate whose target is the global qubit of rank bit b pairs every amplitude
// of rank r with the amplitude at the same local index on partner r ^ (1<<b):
// the rank whose bit is 0 holds v_a, its partner v_b (kernel.py:108-132 with
// a = local index on the bit-0 rank).  Instead of swapping half a shard
// through NCCL and then sweeping locally (sharded.py's qubit-swap path), both
// ranks run this kernel at once on disjoint halves of the pair space: the
// local index space is split on one local bit s (the highest local bit that
// is not a control); the bit-0 rank updates the pairs with bit s = 0, its
// partner the pairs with bit s = 1.  Each rank reads and writes its own
// amplitude of a pair in its HBM and the partner's over NVLink (P2P loads and
// stores through a cudaIpc mapping of the partner's buffer), so the exchange
// and the arithmetic are one pass and nothing is staged.  Every pair is
// updated by exactly one rank with the sweep's arithmetic (pair_update), so
// the result is the unsharded register's bit for bit.  The caller orders the
// two ranks' streams (a barrier before and after the launch).
//
// Traffic per rank and gate: 1/2 shard read + written locally, 1/2 shard read
// + written over NVLink (NVLink-bound: 8 * 2^L bytes each way per GPU).

#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace qsb {

namespace {

template <int U>
__global__ void __launch_bounds__(256) k_peer_pair(float2 *__restrict__ own, float2 *__restrict__ peer,
                                                   uint64_t nitems, FixedBits fb, uint64_t set_mask,
                                                   int own_is_a, Gate2 g) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = tid; base < nitems; base += nthreads * U) {
        float2 x[U], y[U];
        uint64_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t item = base + u * nthreads;
            idx[u] = deposit(item, fb) | set_mask;
            if (item < nitems) {
                x[u] = __ldcs(own + idx[u]);
                y[u] = __ldcg(peer + idx[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * nthreads >= nitems) continue;
            float2 va = own_is_a ? x[u] : y[u];
            float2 vb = own_is_a ? y[u] : x[u];
            pair_update(g, va, vb);
            __stcs(own + idx[u], own_is_a ? va : vb);
            __stcg(peer + idx[u], own_is_a ? vb : va);
        }
    }
}

// The same pair update on 16-B units (two amplitudes, local bit 0 free): one
// 16-B access per amplitude pair and side instead of two 8-B ones, so each
// NVLink request carries twice the payload.  Items enumerate units; the
// fixed bits (controls, the split bit) are deposited into unit indices.
template <int U>
__global__ void __launch_bounds__(256) k_peer_pair16(float4 *__restrict__ own, float4 *__restrict__ peer,
                                                     uint64_t nitems, FixedBits fb, uint64_t set_mask,
                                                     int own_is_a, Gate2 g) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = tid; base < nitems; base += nthreads * U) {
        float4 x[U], y[U];
        uint64_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t item = base + u * nthreads;
            idx[u] = deposit(item, fb) | set_mask;
            if (item < nitems) {
                x[u] = __ldcs(own + idx[u]);
                y[u] = __ldcg(peer + idx[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * nthreads >= nitems) continue;
            const float4 a = own_is_a ? x[u] : y[u], b = own_is_a ? y[u] : x[u];
            float2 a0 = make_float2(a.x, a.y), a1 = make_float2(a.z, a.w);
            float2 b0 = make_float2(b.x, b.y), b1 = make_float2(b.z, b.w);
            pair_update(g, a0, b0);
            pair_update(g, a1, b1);
            const float4 na = make_float4(a0.x, a0.y, a1.x, a1.y), nb = make_float4(b0.x, b0.y, b1.x, b1.y);
            __stcs(own + idx[u], own_is_a ? na : nb);
            __stcg(peer + idx[u], own_is_a ? nb : na);
        }
    }
}

// complex128 shards: the same pair update on 16-B amplitudes (the sweep's
// fp64 arithmetic, gates64.cu pair_update_d)
struct PeerGateD {
    double2 a, b, c, d;
};

template <int U>
__global__ void __launch_bounds__(256) k_peer_pair_d(double2 *__restrict__ own, double2 *__restrict__ peer,
                                                     uint64_t nitems, FixedBits fb, uint64_t set_mask,
                                                     int own_is_a, PeerGateD g) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = tid; base < nitems; base += nthreads * U) {
        double2 x[U], y[U];
        uint64_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t item = base + u * nthreads;
            idx[u] = deposit(item, fb) | set_mask;
            if (item < nitems) {
                x[u] = __ldcs(own + idx[u]);
                y[u] = __ldcg(peer + idx[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * nthreads >= nitems) continue;
            const double2 va = own_is_a ? x[u] : y[u], vb = own_is_a ? y[u] : x[u];
            const double2 na = cadd_d(cmul_d(g.a, va), cmul_d(g.b, vb));
            const double2 nb = cadd_d(cmul_d(g.d, vb), cmul_d(g.c, va));
            __stcs(own + idx[u], own_is_a ? na : nb);
            __stcg(peer + idx[u], own_is_a ? nb : na);
        }
    }
}

// Qubit-swap exchange over peer memory: own[i] <-> peer[i] for i < n units
// of 16 B (two complex64 amplitudes).  Both partners run it at once on
// disjoint halves of the exchanged range, so the swap is one pass with no
// staging buffer and no copy-back (the NCCL path stages the received half
// and copies it into place: an extra half-shard of HBM traffic).
template <int U>
__global__ void __launch_bounds__(256) k_peer_swap(float4 *__restrict__ own, float4 *__restrict__ peer,
                                                   uint64_t n) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = tid; base < n; base += nthreads * U) {
        float4 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * nthreads;
            if (i < n) {
                x[u] = __ldcs(own + i);
                y[u] = __ldcg(peer + i);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * nthreads;
            if (i < n) {
                __stcs(own + i, y[u]);
                __stcg(peer + i, x[u]);
            }
        }
    }
}

__global__ void k_peer_swap8(float2 *__restrict__ own, float2 *__restrict__ peer, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float2 a = own[i], b = peer[i];
        own[i] = b;
        peer[i] = a;
    }
}

unsigned grid_for(const qs_state *s, uint64_t items, int per_thread) {
    uint64_t blocks = (items + 256ull * per_thread - 1) / (256ull * per_thread);
    if (blocks > (uint64_t)s->num_sms * 8) blocks = (uint64_t)s->num_sms * 8;
    return (unsigned)(blocks < 1 ? 1 : blocks);
}

}  // namespace

// own[i] <-> peer[i], i < count amplitudes, on s's stream (caller: device guard)
int launch_peer_swap(qs_state *s, float2 *own, float2 *peer, uint64_t count) {
    if (count == 0) return QS_OK;
    if ((((uintptr_t)own | (uintptr_t)peer) & 15u) == 0 && (count & 1ull) == 0) {
        constexpr int U = 4;
        const uint64_t n = count >> 1;
        k_peer_swap<U><<<grid_for(s, n, U), 256, 0, s->stream>>>((float4 *)own, (float4 *)peer, n);
    } else {
        k_peer_swap8<<<grid_for(s, count, 1), 256, 0, s->stream>>>(own, peer, count);
    }
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

}  // namespace qsb

using namespace qsb;

extern "C" {

int qs_ipc_handle(qs_state *s, void *out) {
    if (!s) return set_error(QS_ERR_NULL, "null qs_state handle");
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    DeviceGuard guard(s->device);
    cudaIpcMemHandle_t h;
    QS_CUDA(cudaIpcGetMemHandle(&h, s->amps));
    s->ipc_exported = 1;
    std::memcpy(out, &h, sizeof h);
    return QS_OK;
}

int qs_ipc_open(int device, const void *handle, void **out) {
    if (!handle || !out) return set_error(QS_ERR_NULL, "null handle or output pointer");
    DeviceGuard guard(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    QS_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    return QS_OK;
}

int qs_ipc_close(int device, void *ptr) {
    if (!ptr) return QS_OK;
    DeviceGuard guard(device);
    QS_CUDA(cudaIpcCloseMemHandle(ptr));
    return QS_OK;
}

static int apply_gate_peer(qs_state *s, void *peer_amps, int own_is_a, uint64_t ctrl_mask, const float *m,
                           const double *md) {
    if (!s) return set_error(QS_ERR_NULL, "null qs_state handle");
    if (!peer_amps || (!m && !md)) return set_error(QS_ERR_NULL, "null peer buffer or gate matrix");
    const bool dbl = s->prec == QS_DOUBLE;
    const int L = s->num_qubits;
    if (L < 64 && (ctrl_mask >> L)) return set_error(QS_ERR_INDEX, "local control out of range");
    if (__builtin_popcountll(ctrl_mask) + 1 > kMaxFixed) return set_error(QS_ERR_VALUE, "too many control qubits");
    // split bit: the highest local bit that is not a control
    int sbit = -1;
    for (int q = L - 1; q >= 0; --q)
        if (!((ctrl_mask >> q) & 1ull)) {
            sbit = q;
            break;
        }
    int pos[kMaxFixed];
    int np = 0;
    uint64_t set_mask = ctrl_mask;
    for (int q = 0; q < L; ++q)
        if ((ctrl_mask >> q) & 1ull) pos[np++] = q;
    if (sbit >= 0) {
        pos[np++] = sbit;
        if (!own_is_a) set_mask |= 1ull << sbit;
    } else if (!own_is_a) {
        return QS_OK;  // every local bit is a control: the bit-0 rank does the single pair
    }
    // sort the fixed positions ascending for deposit()
    for (int i = 1; i < np; ++i)
        for (int j = i; j > 0 && pos[j - 1] > pos[j]; --j) {
            const int t = pos[j];
            pos[j] = pos[j - 1];
            pos[j - 1] = t;
        }
    DeviceGuard guard(s->device);
    constexpr int U = 4;
    if (dbl) {  // complex128: 16-B amplitudes
        double e[8];
        for (int i = 0; i < 8; ++i) e[i] = md ? md[i] : (double)m[i];
        PeerGateD g{make_double2(e[0], e[1]), make_double2(e[2], e[3]), make_double2(e[4], e[5]),
                    make_double2(e[6], e[7])};
        FixedBits fb;
        fb.n = np;
        for (int i = 0; i < kMaxFixed; ++i) fb.pos[i] = i < np ? pos[i] : 0;
        const uint64_t nitems = 1ull << (L - np);
        k_peer_pair_d<U><<<grid_for(s, nitems, U), 256, 0, s->stream>>>((double2 *)s->amps, (double2 *)peer_amps,
                                                                         nitems, fb, set_mask, own_is_a, g);
        QS_CUDA(cudaGetLastError());
        return QS_OK;
    }
    float mf[8];
    for (int i = 0; i < 8; ++i) mf[i] = m ? m[i] : (float)md[i];
    const bool wide = np == 0 || pos[0] > 0;  // local bit 0 free: 16-B units
    FixedBits fb;
    fb.n = np;
    for (int i = 0; i < kMaxFixed; ++i) fb.pos[i] = i < np ? pos[i] - (wide ? 1 : 0) : 0;
    const Gate2 g = gate_from(mf);
    if (wide) {
        const uint64_t nitems = 1ull << (L - 1 - np);
        k_peer_pair16<U><<<grid_for(s, nitems, U), 256, 0, s->stream>>>(
            (float4 *)s->amps, (float4 *)peer_amps, nitems, fb, set_mask >> 1, own_is_a, g);
    } else {
        const uint64_t nitems = 1ull << (L - np);
        k_peer_pair<U><<<grid_for(s, nitems, U), 256, 0, s->stream>>>(s->amps, (float2 *)peer_amps, nitems, fb,
                                                                       set_mask, own_is_a, g);
    }
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

int qs_apply_gate_peer(qs_state *s, void *peer_amps, int own_is_a, uint64_t ctrl_mask, const float m[8]) {
    return apply_gate_peer(s, peer_amps, own_is_a, ctrl_mask, m, nullptr);
}

int qs_apply_gate_peer_f64(qs_state *s, void *peer_amps, int own_is_a, uint64_t ctrl_mask, const double m[8]) {
    return apply_gate_peer(s, peer_amps, own_is_a, ctrl_mask, nullptr, m);
}

int qs_swap_peer(qs_state *s, void *peer_amps, uint64_t own_offset, uint64_t peer_offset, uint64_t count) {
    if (!s) return set_error(QS_ERR_NULL, "null qs_state handle");
    if (!peer_amps) return set_error(QS_ERR_NULL, "null peer buffer");
    const uint64_t dim = 1ull << s->num_qubits;
    if (own_offset > dim || count > dim - own_offset) return set_error(QS_ERR_INDEX, "swap range out of bounds");
    if (count == 0) return QS_OK;
    DeviceGuard guard(s->device);
    if (s->prec == QS_DOUBLE)  // 16-B amplitudes = two float2 units each
        return launch_peer_swap(s, s->amps + 2 * own_offset, (float2 *)peer_amps + 2 * peer_offset, 2 * count);
    return launch_peer_swap(s, s->amps + own_offset, (float2 *)peer_amps + peer_offset, count);
}

}  // extern "C"
