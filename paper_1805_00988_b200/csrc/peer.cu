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

}  // namespace

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

int qs_apply_gate_peer(qs_state *s, void *peer_amps, int own_is_a, uint64_t ctrl_mask, const float m[8]) {
    if (!s) return set_error(QS_ERR_NULL, "null qs_state handle");
    if (!peer_amps || !m) return set_error(QS_ERR_NULL, "null peer buffer or gate matrix");
    if (s->prec != QS_SINGLE) return set_error(QS_ERR_VALUE, "peer gates need complex64 shards");
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
    FixedBits fb;
    fb.n = np;
    for (int i = 0; i < kMaxFixed; ++i) fb.pos[i] = i < np ? pos[i] : 0;
    const uint64_t nitems = 1ull << (L - np);
    DeviceGuard guard(s->device);
    constexpr int U = 4;
    uint64_t blocks = (nitems + 256ull * U - 1) / (256ull * U);
    if (blocks > (uint64_t)s->num_sms * 8) blocks = (uint64_t)s->num_sms * 8;
    if (blocks < 1) blocks = 1;
    k_peer_pair<U><<<(unsigned)blocks, 256, 0, s->stream>>>(s->amps, (float2 *)peer_amps, nitems, fb, set_mask,
                                                             own_is_a, gate_from(m));
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

}  // extern "C"
