// A register sharded over several GPUs driven by ONE process (SURVEY 8(b)
// qs_create_sharded, 8(e) "Driver: a single process drives all devices").
//
// Layout (as paper_1805_00988_b200/sharded.py): P = 2^g shards, shard r holds
// the contiguous slice [r 2^L, (r+1) 2^L) of the PHYSICAL index space, L =
// n - g; physical positions L..n-1 are the rank bits.  A logical -> physical
// qubit map is kept here and updated lazily:
//
// * a gate on local qubits runs on every shard with no communication;
//   controls on global qubits are shard predicates;
// * a diagonal gate keeps the data in place: re-targeted to one of its local
//   bits, or — all its bits global — a whole-shard multiply on the shards
//   whose rank bits satisfy it (same per-amplitude product, no exchange);
// * a pair gate on a global qubit either swaps that position with local
//   position L-1 (the qubit swap: partners exchange the contiguous half of
//   their slice whose bit L-1 differs from their rank bit) and then runs
//   locally, or (peer gates on) updates the pairs across the two shards in
//   one kernel over peer memory (csrc/peer.cu, qs_apply_gate_peer).
//
// Data movement of a swap: NCCL send/recv between the partners' devices (one
// communicator per device from ncclCommInitAll, libnccl loaded with dlopen)
// through a staging buffer, or a peer-memory swap kernel (qs_swap_peer) when
// NCCL is unavailable, the devices repeat (several shards on one GPU) or it
// is requested (QSB_SHARD_EXCHANGE=p2p / qs_sharded_set_mode).  Every pair
// update is the sweep's arithmetic, so results equal the unsharded
// register's bit for bit.
//
// Readout un-permutes the qubit map (local swap kernels + exchanges), then
// reads the shards in rank order; sampling chains the exact sequential CDF
// across shards (qs_cdf_extend semantics) and draws on every shard.

#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <nccl.h>  // types only: libnccl is loaded at run time

#include "internal.h"

namespace qsb {

int launch_peer_swap(qs_state *s, float2 *own, float2 *peer, uint64_t count);  // peer.cu

namespace {

struct Nccl {
    bool ok = false;
    ncclResult_t (*init_all)(ncclComm_t *, int, const int *);
    ncclResult_t (*destroy)(ncclComm_t);
    ncclResult_t (*group_start)();
    ncclResult_t (*group_end)();
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    const char *(*err)(ncclResult_t);
};

Nccl load_nccl() {
    Nccl n;
    void *h = nullptr;
    for (const char *nm : {"libnccl.so.2", "libnccl.so"})
        if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return n;
    n.init_all = (decltype(n.init_all))dlsym(h, "ncclCommInitAll");
    n.destroy = (decltype(n.destroy))dlsym(h, "ncclCommDestroy");
    n.group_start = (decltype(n.group_start))dlsym(h, "ncclGroupStart");
    n.group_end = (decltype(n.group_end))dlsym(h, "ncclGroupEnd");
    n.send = (decltype(n.send))dlsym(h, "ncclSend");
    n.recv = (decltype(n.recv))dlsym(h, "ncclRecv");
    n.err = (decltype(n.err))dlsym(h, "ncclGetErrorString");
    n.ok = n.init_all && n.destroy && n.group_start && n.group_end && n.send && n.recv && n.err;
    return n;
}

const Nccl &nccl() {
    static const Nccl n = load_nccl();
    return n;
}

int nccl_fail(ncclResult_t r, const char *what) {
    return set_error(QS_ERR_CUDA, std::string("NCCL error in ") + what + ": " + nccl().err(r));
}

#define QS_NCCL(call)                                          \
    do {                                                       \
        ncclResult_t _r = (call);                              \
        if (_r != ncclSuccess) return nccl_fail(_r, #call);     \
    } while (0)

bool is_phase(const float m[8]) {
    return m[0] == 1.f && m[1] == 0.f && m[2] == 0.f && m[3] == 0.f && m[4] == 0.f && m[5] == 0.f;
}

constexpr uint64_t kStagingAmps = 1ull << 26;  // 512 MiB of complex64 per shard (NCCL path)

}  // namespace
}  // namespace qsb

using namespace qsb;

struct qs_sharded {
    int n = 0, g = 0, L = 0, P = 0;
    std::vector<qs_state *> shards;
    std::vector<int> devs;
    std::vector<int> pos, at;  // pos[logical] = physical, at[physical] = logical
    std::vector<ncclComm_t> comms;
    std::vector<cudaEvent_t> ev;
    std::vector<float2 *> staging;
    int exchange = QS_EXCHANGE_P2P;
    int peer_gates = 0;
    bool p2p_ok = true;  // every shard's device can load / store every other's memory
    uint64_t swaps = 0, peer_gate_count = 0;
};

namespace {

// stream of shard `a` waits for everything queued so far on shard `b`
int order_after(qs_sharded *h, int a, int b) {
    if (a == b) return QS_OK;
    {
        DeviceGuard guard(h->devs[b]);
        QS_CUDA(cudaEventRecord(h->ev[b], h->shards[b]->stream));
    }
    DeviceGuard guard(h->devs[a]);
    QS_CUDA(cudaStreamWaitEvent(h->shards[a]->stream, h->ev[b], 0));
    return QS_OK;
}

int order_pair(qs_sharded *h, int a, int b) {
    if (int rc = order_after(h, a, b)) return rc;
    return order_after(h, b, a);
}

bool local(const qs_sharded *h, int q) { return h->pos[q] < h->L; }

void swap_physical(qs_sharded *h, int p1, int p2) {
    const int a = h->at[p1], b = h->at[p2];
    h->at[p1] = b;
    h->at[p2] = a;
    h->pos[a] = p2;
    h->pos[b] = p1;
}

// Exchange for swapping physical position L + rank_bit with L - 1: partner
// shards r (rank bit 0) and r2 = r | 1 << rank_bit trade r's half with bit
// L-1 = 1 and r2's half with bit L-1 = 0 (sharded.py exchange_plan).
int exchange(qs_sharded *h, int rank_bit) {
    NvtxRange nvtx_range("qsb sharded exchange");
    const uint64_t half = 1ull << (h->L - 1);
    const int bit = 1 << rank_bit;
    if (h->exchange == QS_EXCHANGE_NCCL) {
        const Nccl &nc = nccl();
        for (int r = 0; r < h->P; ++r)
            if (!h->staging[r]) {
                DeviceGuard guard(h->devs[r]);
                QS_CUDA(cudaMalloc((void **)&h->staging[r], 8ull * std::min<uint64_t>(half, kStagingAmps)));
            }
        const uint64_t step = std::min<uint64_t>(half, kStagingAmps);
        for (uint64_t c = 0; c < half; c += step) {
            QS_NCCL(nc.group_start());
            for (int r = 0; r < h->P; ++r) {
                const int partner = r ^ bit;
                const uint64_t off = (r & bit) ? 0 : half;  // the half whose bit L-1 differs from ours
                QS_NCCL(nc.send(h->shards[r]->amps + off + c, 2 * step, ncclFloat32, partner, h->comms[r],
                                h->shards[r]->stream));
                QS_NCCL(nc.recv(h->staging[r], 2 * step, ncclFloat32, partner, h->comms[r], h->shards[r]->stream));
            }
            QS_NCCL(nc.group_end());
            for (int r = 0; r < h->P; ++r) {
                const uint64_t off = (r & bit) ? 0 : half;
                DeviceGuard guard(h->devs[r]);
                QS_CUDA(cudaMemcpyAsync(h->shards[r]->amps + off + c, h->staging[r], 8 * step,
                                        cudaMemcpyDeviceToDevice, h->shards[r]->stream));
            }
        }
        return QS_OK;
    }
    // peer memory: each partner swaps half of the exchanged range
    for (int r = 0; r < h->P; ++r) {
        if (r & bit) continue;
        const int r2 = r | bit;
        if (int rc = order_pair(h, r, r2)) return rc;
        const uint64_t first = half - half / 2;  // r's share; r2 takes the rest
        {
            DeviceGuard guard(h->devs[r]);
            if (int rc = launch_peer_swap(h->shards[r], h->shards[r]->amps + half, h->shards[r2]->amps, first))
                return rc;
        }
        if (half > first) {
            DeviceGuard guard(h->devs[r2]);
            if (int rc = launch_peer_swap(h->shards[r2], h->shards[r2]->amps + first,
                                          h->shards[r]->amps + half + first, half - first))
                return rc;
        }
        if (int rc = order_pair(h, r, r2)) return rc;
    }
    return QS_OK;
}

int swap_local_global(qs_sharded *h, int loc, int glob) {
    const int s = h->L - 1;
    if (loc != s) {
        for (int r = 0; r < h->P; ++r) {
            DeviceGuard guard(h->devs[r]);
            if (int rc = launch_swap(h->shards[r], loc, s)) return rc;
        }
        swap_physical(h, loc, s);
    }
    if (int rc = exchange(h, glob - h->L)) return rc;
    swap_physical(h, glob, s);
    ++h->swaps;
    if (loc != s) {
        for (int r = 0; r < h->P; ++r) {
            DeviceGuard guard(h->devs[r]);
            if (int rc = launch_swap(h->shards[r], loc, s)) return rc;
        }
        swap_physical(h, loc, s);
    }
    return QS_OK;
}

int ensure_local(qs_sharded *h, int q) {
    if (local(h, q)) return QS_OK;
    const int p = h->pos[q];
    if (int rc = exchange(h, p - h->L)) return rc;
    swap_physical(h, p, h->L - 1);
    ++h->swaps;
    return QS_OK;
}

// Restore the identity qubit map (readout), as ShardedState.canonicalize.
int canonicalize(qs_sharded *h) {
    for (int p = 0; p < h->n; ++p) {
        if (h->at[p] == p) continue;
        const int pp = h->pos[p];  // logical qubit p now sits at physical pp
        int rc = QS_OK;
        if (p < h->L && pp < h->L) {
            for (int r = 0; r < h->P && !rc; ++r) {
                DeviceGuard guard(h->devs[r]);
                rc = launch_swap(h->shards[r], p, pp);
            }
            if (!rc) swap_physical(h, p, pp);
        } else if (p >= h->L && pp >= h->L) {
            rc = swap_local_global(h, h->L - 1, p);
            if (!rc) rc = swap_local_global(h, h->L - 1, pp);
            if (!rc) rc = swap_local_global(h, h->L - 1, p);
        } else if (p < h->L) {
            rc = swap_local_global(h, p, pp);
        } else {
            rc = swap_local_global(h, pp, p);
        }
        if (rc) return rc;
    }
    return QS_OK;
}

int sync_all(qs_sharded *h) {
    for (int r = 0; r < h->P; ++r) {
        DeviceGuard guard(h->devs[r]);
        QS_CUDA(cudaStreamSynchronize(h->shards[r]->stream));
    }
    return QS_OK;
}

int apply(qs_sharded *h, int target, int nctrl, const int *ctrl, const float m[8]) {
    if (!h) return set_error(QS_ERR_NULL, "null qs_sharded handle");
    if (!m) return set_error(QS_ERR_NULL, "null gate matrix");
    int qs[3] = {target, nctrl > 0 ? ctrl[0] : -1, nctrl > 1 ? ctrl[1] : -1};
    for (int i = 0; i <= nctrl; ++i)
        if (qs[i] < 0 || qs[i] >= h->n)
            return set_error(QS_ERR_INDEX, "qubit " + std::to_string(qs[i]) + " out of range for " +
                                               std::to_string(h->n) + " qubits");
    for (int i = 0; i <= nctrl; ++i)
        for (int j = i + 1; j <= nctrl; ++j)
            if (qs[i] == qs[j]) return set_error(QS_ERR_VALUE, "control and target must differ");
    const bool phase = is_phase(m);
    int t = target;
    std::vector<int> controls(ctrl, ctrl + nctrl);
    if (phase && !local(h, t)) {
        // diagonal: symmetric in its bits; keep the data in place
        for (int i = 0; i <= nctrl; ++i)
            if (local(h, qs[i])) {
                t = qs[i];
                controls.clear();
                for (int j = 0; j <= nctrl; ++j)
                    if (j != i) controls.push_back(qs[j]);
                break;
            }
        if (!local(h, t)) {  // every bit global: a whole-shard multiply where they are all 1
            uint64_t need = 0;
            for (int i = 0; i <= nctrl; ++i) need |= 1ull << (h->pos[qs[i]] - h->L);
            for (int r = 0; r < h->P; ++r)
                if (((uint64_t)r & need) == need) {
                    DeviceGuard guard(h->devs[r]);
                    if (int rc = launch_phase(h->shards[r], 0, make_float2(m[6], m[7]))) return rc;
                }
            return QS_OK;
        }
    }
    auto split = [&](uint64_t *cmask, uint64_t *need) {
        *cmask = 0;
        *need = 0;
        for (int c : controls) {
            const int pc = h->pos[c];
            if (pc < h->L)
                *cmask |= 1ull << pc;
            else
                *need |= 1ull << (pc - h->L);
        }
    };
    if (!phase && !local(h, t) && h->peer_gates) {
        uint64_t cmask, need;
        split(&cmask, &need);
        const int bit = 1 << (h->pos[t] - h->L);
        for (int r = 0; r < h->P; ++r) {
            if ((r & bit) || ((uint64_t)r & need) != need) continue;
            const int r2 = r | bit;
            if (int rc = order_pair(h, r, r2)) return rc;
            if (int rc = qs_apply_gate_peer(h->shards[r], h->shards[r2]->amps, 1, cmask, m)) return rc;
            if (int rc = qs_apply_gate_peer(h->shards[r2], h->shards[r]->amps, 0, cmask, m)) return rc;
            if (int rc = order_pair(h, r, r2)) return rc;
        }
        ++h->peer_gate_count;
        return QS_OK;
    }
    if (int rc = ensure_local(h, t)) return rc;
    uint64_t cmask, need;
    split(&cmask, &need);
    const int tp = h->pos[t];
    for (int r = 0; r < h->P; ++r) {
        if (((uint64_t)r & need) != need) continue;
        DeviceGuard guard(h->devs[r]);
        if (int rc = launch_sweep(h->shards[r], tp, cmask, m)) return rc;
    }
    return QS_OK;
}

template <class F>
int for_range(qs_sharded *h, uint64_t offset, uint64_t count, F &&fn) {
    const uint64_t dim = 1ull << h->n, sd = 1ull << h->L;
    if (offset > dim || count > dim - offset) return set_error(QS_ERR_INDEX, "amplitude range out of bounds");
    if (int rc = canonicalize(h)) return rc;
    for (int r = 0; r < h->P; ++r) {
        const uint64_t lo = std::max<uint64_t>(offset, (uint64_t)r * sd);
        const uint64_t hi = std::min<uint64_t>(offset + count, (uint64_t)(r + 1) * sd);
        if (lo >= hi) continue;
        if (int rc = fn(r, lo - (uint64_t)r * sd, hi - lo, lo - offset)) return rc;
    }
    return QS_OK;
}

}  // namespace

extern "C" {

int qs_create_sharded(int num_qubits, int nshards, const int *devs, uint64_t memory_budget, qs_sharded **out) {
    if (!out || !devs) return set_error(QS_ERR_NULL, "null device list or output pointer");
    *out = nullptr;
    if (nshards < 1 || (nshards & (nshards - 1))) return set_error(QS_ERR_VALUE, "shard count must be a power of two");
    int g = 0;
    while ((1 << g) < nshards) ++g;
    if (num_qubits < 1 || num_qubits - g < 1 || num_qubits > 62)
        return set_error(QS_ERR_VALUE, "need 1 <= num_qubits - log2(shards) and num_qubits <= 62");
    int ndev = 0;
    QS_CUDA(cudaGetDeviceCount(&ndev));
    for (int r = 0; r < nshards; ++r)
        if (devs[r] < 0 || devs[r] >= ndev) return set_error(QS_ERR_INDEX, "device " + std::to_string(devs[r]) + " out of range");
    std::unique_ptr<qs_sharded> h(new qs_sharded());
    h->n = num_qubits;
    h->g = g;
    h->L = num_qubits - g;
    h->P = nshards;
    h->devs.assign(devs, devs + nshards);
    for (int q = 0; q < num_qubits; ++q) {
        h->pos.push_back(q);
        h->at.push_back(q);
    }
    auto fail = [&](int rc) {
        qs_sharded_destroy(h.release());
        return rc;
    };
    h->shards.assign(nshards, nullptr);
    h->ev.assign(nshards, nullptr);
    h->staging.assign(nshards, nullptr);
    for (int r = 0; r < nshards; ++r) {
        if (int rc = qs_create(h->L, devs[r], memory_budget, &h->shards[r])) return fail(rc);
        DeviceGuard guard(devs[r]);
        if (cudaEventCreateWithFlags(&h->ev[r], cudaEventDisableTiming) != cudaSuccess)
            return fail(cuda_fail(cudaGetLastError(), "cudaEventCreateWithFlags"));
    }
    // peer access between distinct devices (P2P kernels over NVLink)
    bool distinct = true, p2p = true;
    for (int a = 0; a < nshards; ++a)
        for (int b = 0; b < nshards; ++b) {
            if (a == b) continue;
            if (devs[a] == devs[b]) {
                distinct = false;
                continue;
            }
            int can = 0;
            cudaDeviceCanAccessPeer(&can, devs[a], devs[b]);
            if (!can) {
                p2p = false;
                continue;
            }
            DeviceGuard guard(devs[a]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(devs[b], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) p2p = false;
            cudaGetLastError();
        }
    // NCCL communicators (one per device) when every shard has its own GPU
    const char *want = std::getenv("QSB_SHARD_EXCHANGE");
    const bool force_p2p = want && (!std::strcmp(want, "p2p") || !std::strcmp(want, "peer"));
    if (distinct && nshards > 1 && !force_p2p && nccl().ok) {
        h->comms.assign(nshards, nullptr);
        const ncclResult_t r = nccl().init_all(h->comms.data(), nshards, devs);
        if (r == ncclSuccess) {
            h->exchange = QS_EXCHANGE_NCCL;
        } else {
            h->comms.clear();
        }
    }
    h->p2p_ok = p2p;  // repeated devices are trivially peers; distinct ones need P2P access
    if (h->exchange != QS_EXCHANGE_NCCL && !p2p && nshards > 1)
        return fail(set_error(QS_ERR_CUDA, "shards cannot exchange data: no NCCL communicator and no peer access"));
    if (const char *pg = std::getenv("QSB_SHARD_PEER")) h->peer_gates = *pg == '1' && (p2p || !distinct);
    if (int rc = qs_sharded_reset(h.get(), 0)) return fail(rc);
    *out = h.release();
    return QS_OK;
}

int qs_sharded_destroy(qs_sharded *h) {
    if (!h) return QS_OK;
    for (int r = 0; r < (int)h->shards.size(); ++r)
        if (h->shards[r]) {
            DeviceGuard guard(h->devs[r]);
            cudaStreamSynchronize(h->shards[r]->stream);
        }
    for (ncclComm_t c : h->comms)
        if (c) nccl().destroy(c);
    for (int r = 0; r < (int)h->shards.size(); ++r) {
        DeviceGuard guard(h->devs[r]);
        if (h->staging[r]) cudaFree(h->staging[r]);
        if (h->ev[r]) cudaEventDestroy(h->ev[r]);
        if (h->shards[r]) qs_destroy(h->shards[r]);
    }
    delete h;
    return QS_OK;
}

int qs_sharded_info(const qs_sharded *h, int *num_qubits, int *nshards, int *shard_qubits) {
    if (!h) return set_error(QS_ERR_NULL, "null qs_sharded handle");
    if (num_qubits) *num_qubits = h->n;
    if (nshards) *nshards = h->P;
    if (shard_qubits) *shard_qubits = h->L;
    return QS_OK;
}

int qs_sharded_shard(qs_sharded *h, int rank, qs_state **out) {
    if (!h || !out) return set_error(QS_ERR_NULL, "null handle or output pointer");
    if (rank < 0 || rank >= h->P) return set_error(QS_ERR_INDEX, "shard index out of range");
    *out = h->shards[rank];
    return QS_OK;
}

int qs_sharded_set_mode(qs_sharded *h, int peer_gates, int exchange) {
    if (!h) return set_error(QS_ERR_NULL, "null qs_sharded handle");
    if (exchange == QS_EXCHANGE_NCCL && h->comms.empty())
        return set_error(QS_ERR_VALUE, "no NCCL communicators (devices repeat or libnccl missing)");
    if ((exchange == QS_EXCHANGE_P2P || peer_gates == 1) && !h->p2p_ok)
        return set_error(QS_ERR_VALUE, "peer-memory kernels need P2P access between every pair of devices");
    if (exchange == QS_EXCHANGE_NCCL || exchange == QS_EXCHANGE_P2P) h->exchange = exchange;
    if (peer_gates >= 0) h->peer_gates = peer_gates != 0;
    return QS_OK;
}

int qs_sharded_stats(const qs_sharded *h, uint64_t *swaps, uint64_t *peer_gates, int *exchange) {
    if (!h) return set_error(QS_ERR_NULL, "null qs_sharded handle");
    if (swaps) *swaps = h->swaps;
    if (peer_gates) *peer_gates = h->peer_gate_count;
    if (exchange) *exchange = h->exchange;
    return QS_OK;
}

int qs_sharded_reset(qs_sharded *h, uint64_t basis) {
    if (!h) return set_error(QS_ERR_NULL, "null qs_sharded handle");
    if (h->n < 64 && (basis >> h->n)) return set_error(QS_ERR_INDEX, "basis index out of range");
    for (int q = 0; q < h->n; ++q) h->pos[q] = h->at[q] = q;
    const uint64_t owner = basis >> h->L, local_idx = basis & ((1ull << h->L) - 1ull);
    for (int r = 0; r < h->P; ++r) {
        DeviceGuard guard(h->devs[r]);
        if ((uint64_t)r == owner) {
            if (int rc = launch_reset(h->shards[r], local_idx)) return rc;
        } else {
            QS_CUDA(cudaMemsetAsync(h->shards[r]->amps, 0, state_bytes(h->shards[r]), h->shards[r]->stream));
        }
    }
    return QS_OK;
}

int qs_sharded_apply_gate(qs_sharded *h, int target, const float m[8]) { return apply(h, target, 0, nullptr, m); }

int qs_sharded_apply_controlled_gate(qs_sharded *h, int control, int target, const float m[8]) {
    return apply(h, target, 1, &control, m);
}

int qs_sharded_apply_controlled_controlled_gate(qs_sharded *h, int c1, int c2, int target, const float m[8]) {
    const int c[2] = {c1, c2};
    return apply(h, target, 2, c, m);
}

int qs_sharded_qubit_map(const qs_sharded *h, int32_t *pos) {
    if (!h || !pos) return set_error(QS_ERR_NULL, "null handle or output buffer");
    for (int q = 0; q < h->n; ++q) pos[q] = h->pos[q];
    return QS_OK;
}

int qs_sharded_localize(qs_sharded *h, int qubit) {
    if (!h) return set_error(QS_ERR_NULL, "null qs_sharded handle");
    if (qubit < 0 || qubit >= h->n) return set_error(QS_ERR_INDEX, "qubit out of range");
    return ensure_local(h, qubit);
}

int qs_sharded_synchronize(qs_sharded *h) {
    if (!h) return set_error(QS_ERR_NULL, "null qs_sharded handle");
    return sync_all(h);
}

int qs_sharded_get_amplitudes(qs_sharded *h, uint64_t offset, uint64_t count, void *host) {
    if (!h || !host) return set_error(QS_ERR_NULL, "null handle or host buffer");
    return for_range(h, offset, count, [&](int r, uint64_t loff, uint64_t cnt, uint64_t out_off) {
        return qs_get_amplitudes(h->shards[r], loff, cnt, (char *)host + 8 * out_off);
    });
}

int qs_sharded_set_amplitudes(qs_sharded *h, uint64_t offset, uint64_t count, const void *host) {
    if (!h || !host) return set_error(QS_ERR_NULL, "null handle or host buffer");
    return for_range(h, offset, count, [&](int r, uint64_t loff, uint64_t cnt, uint64_t in_off) {
        return qs_set_amplitudes(h->shards[r], loff, cnt, (const char *)host + 8 * in_off);
    });
}

int qs_sharded_probabilities(qs_sharded *h, uint64_t offset, uint64_t count, double *host) {
    if (!h || !host) return set_error(QS_ERR_NULL, "null handle or host buffer");
    return for_range(h, offset, count, [&](int r, uint64_t loff, uint64_t cnt, uint64_t out_off) {
        return qs_probabilities(h->shards[r], loff, cnt, host + out_off);
    });
}

int qs_sharded_norm_squared(qs_sharded *h, double *out) {
    if (!h || !out) return set_error(QS_ERR_NULL, "null handle or output pointer");
    double s = 0.0;
    for (int r = 0; r < h->P; ++r) {
        double v = 0.0;
        if (int rc = qs_norm_squared(h->shards[r], &v)) return rc;
        s += v;
    }
    *out = s;
    return QS_OK;
}

// pairsim.measure.sample (measure.py:76-85) over the whole register: the
// exact sequential CDF continues shard to shard in index order.
int qs_sharded_sample(qs_sharded *h, const qs_pcg64 *rng, int64_t k, int64_t *out) {
    if (!h || !rng || !out) return set_error(QS_ERR_NULL, "null handle, rng or output buffer");
    if (k < 1) return set_error(QS_ERR_VALUE, "n_samples must be >= 1");
    if (int rc = canonicalize(h)) return rc;
    std::vector<double> start(h->P);
    double s = 0.0;
    for (int r = 0; r < h->P; ++r) {
        start[r] = s;
        if (int rc = qs_cdf_extend(h->shards[r], s, &s)) return rc;
    }
    if (!(s > 0.0)) return set_error(QS_ERR_DEGENERATE, "all outcome probabilities are zero");
    std::vector<int64_t> part((size_t)k);
    for (int64_t i = 0; i < k; ++i) out[i] = -1;
    for (int r = 0; r < h->P; ++r) {
        if (int rc = qs_sample_shard(h->shards[r], rng, k, start[r], s, (uint64_t)r << h->L, 1ull << h->n,
                                     r == h->P - 1, part.data()))
            return rc;
        for (int64_t i = 0; i < k; ++i) out[i] = std::max(out[i], part[i]);
    }
    return QS_OK;
}

}  // extern "C"
