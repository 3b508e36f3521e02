// libqsb200 runtime: handle lifecycle, validation, error reporting and the
// extern "C" entry points declared in include/qsb200.h.
//
// Validation order and messages follow the reference functions each entry
// point replaces (cited per function) so the Python layer can re-raise the
// same exception types.

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace qsb {

static thread_local std::string g_last_error;

int set_error(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

// cudaFuncSetAttribute applies to the current device's context only: track
// the dynamic shared-memory limit already set per (kernel, device) and raise
// it when a launch needs more (thread-safe; one entry per device a kernel
// has run on).
int ensure_smem_attr(const void *fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> done;
    int dev = 0;
    QS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    int &have = done[{fn, dev}];
    if (have >= bytes) return QS_OK;
    QS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
    return QS_OK;
}

bool fault_flip_c() {
    static const bool on = [] {
        const char *e = std::getenv("QSB_FAULT_FLIP_C");
        return e && *e == '1';
    }();
    return on;
}

int cuda_fail(cudaError_t e, const char *what) {
    std::string m = std::string("CUDA error in ") + what + ": " + cudaGetErrorName(e) + " (" +
                    cudaGetErrorString(e) + ")";
    return set_error(QS_ERR_CUDA, m);
}

int ensure_scratch(qs_state *s, size_t bytes) {
    if (s->scratch_bytes >= bytes) return QS_OK;
    // grow geometrically in 2-MiB steps: requests that creep up (k-dependent
    // sample outputs) would otherwise reallocate (and synchronise) each time,
    // and round sizes let the device buffer cache reuse blocks across handles
    if (s->scratch_bytes && bytes < s->scratch_bytes + s->scratch_bytes / 2)
        bytes = s->scratch_bytes + s->scratch_bytes / 2;
    bytes = (bytes + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
    if (s->scratch) {
        QS_CUDA(cudaStreamSynchronize(s->stream));
        s->csum_dst = nullptr;  // a prepared chunk-sum array lived in the old buffer
        s->csum_ready = 0;
        pool_free(s->device, s->scratch, s->scratch_bytes);
        s->scratch = nullptr;
        s->scratch_bytes = 0;
    }
    QS_CUDA(pool_alloc(s->device, bytes, &s->scratch));
    s->scratch_bytes = bytes;
    return QS_OK;
}

int ensure_pinned(qs_state *s, size_t bytes) {
    if (s->pinned_bytes >= bytes) return QS_OK;
    if (s->pinned_bytes && bytes < s->pinned_bytes + s->pinned_bytes / 2)
        bytes = s->pinned_bytes + s->pinned_bytes / 2;
    bytes = (bytes + (64u << 10) - 1) & ~(size_t)((64u << 10) - 1);
    if (s->pinned) {
        QS_CUDA(cudaStreamSynchronize(s->stream));
        QS_CUDA(cudaFreeHost(s->pinned));
        s->pinned = nullptr;
        s->pinned_bytes = 0;
    }
    QS_CUDA(cudaMallocHost(&s->pinned, bytes));
    s->pinned_bytes = bytes;
    return QS_OK;
}

static std::string format_bytes(unsigned long long b) {
    // decimal units, 4 significant digits (pkg/src/pairsim/state.py:86-97)
    if (b < 1000ull) return std::to_string(b) + " B";
    const char *units[] = {"kB", "MB", "GB", "TB", "PB", "EB"};
    double v = (double)b;
    int u = 0;
    for (u = 0; u < 6; ++u) {
        v /= 1000.0;
        if (v < 1000.0 || u == 5) break;
    }
    char buf[64];
    int digits = v < 10 ? 3 : (v < 100 ? 2 : 1);
    snprintf(buf, sizeof buf, "%.*f", digits, v);
    std::string t(buf);
    while (!t.empty() && t.back() == '0') t.pop_back();
    if (!t.empty() && t.back() == '.') t.pop_back();
    return t + " " + units[u];
}

}  // namespace qsb

using namespace qsb;

#define CHECK_HANDLE(s) \
    if (!(s)) return set_error(QS_ERR_NULL, "null qs_state handle")

static int check_qubit(const qs_state *s, int q, const char *what) {
    if (q < 0 || q >= s->num_qubits)
        return set_error(QS_ERR_INDEX, std::string(what) + " " + std::to_string(q) +
                                           " out of range for " + std::to_string(s->num_qubits) +
                                           " qubits");
    return QS_OK;
}

extern "C" {

int qs_abi_version(void) { return QSB200_ABI_VERSION; }

const char *qs_last_error(void) { return g_last_error.c_str(); }

int qs_device_count(int *out) {
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *out = 0;
        cudaGetLastError();
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    *out = n;
    return QS_OK;
}

// new_state: pkg/src/pairsim/state.py:122-143
int qs_create(int num_qubits, int device, uint64_t memory_budget, qs_state **out) {
    return qs_create_ex(num_qubits, device, memory_budget, QS_SINGLE, out);
}

static int create_impl(int num_qubits, int device, uint64_t memory_budget, int precision, qs_state **out,
                       bool init);

int qs_create_ex(int num_qubits, int device, uint64_t memory_budget, int precision, qs_state **out) {
    return create_impl(num_qubits, device, memory_budget, precision, out, true);
}

// A register whose contents are left undefined: for a circuit whose first
// fused pass writes its start state anyway (qs_apply_fused_from_basis) —
// pairsim's new_state + run_circuit without the separate clear.
int qs_create_uninit(int num_qubits, int device, uint64_t memory_budget, int precision, qs_state **out) {
    return create_impl(num_qubits, device, memory_budget, precision, out, false);
}

static int create_impl(int num_qubits, int device, uint64_t memory_budget, int precision, qs_state **out,
                       bool init) {
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    *out = nullptr;
    if (num_qubits < 1) return set_error(QS_ERR_VALUE, "num_qubits must be >= 1");
    if (precision != QS_SINGLE && precision != QS_DOUBLE)
        return set_error(QS_ERR_VALUE, "precision must be QS_SINGLE or QS_DOUBLE");
    const int shift = precision == QS_DOUBLE ? 4 : 3;  // log2 bytes per amplitude
    if (num_qubits > 300)
        return set_error(QS_ERR_CAPACITY, std::to_string(num_qubits) +
                                              " qubits is past the supported limit of 300");
    int ndev = 0;
    QS_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_error(QS_ERR_VALUE, "device " + std::to_string(device) + " not present (" +
                                           std::to_string(ndev) + " devices)");
    DeviceGuard guard(device);
    // Default budget: 75% of free HBM (cached register buffers count as free).
    // Registers up to 256 MiB skip the (slow) free-memory query: if such a
    // request does not fit, cudaMalloc fails and CapacityError is raised anyway.
    unsigned long long budget = memory_budget;
    if (!budget) {
        if (num_qubits <= 25) {
            budget = ~0ull;
        } else {
            size_t free_b = 0, total_b = 0;
            QS_CUDA(cudaMemGetInfo(&free_b, &total_b));
            budget = (unsigned long long)(free_b + pool_cached(device)) * 3 / 4;
        }
    }
    // need_bytes = memory_required // 8 = (8 or 16) * 2^n (state.py:71-83, 134)
    const unsigned long long need_b = num_qubits > 59 ? 0ull : (1ull << (num_qubits + shift));
    if (num_qubits > 59 || need_b > budget) {
        std::string need = num_qubits > 59 ? std::string("more than 2^63 bytes")
                                           : format_bytes(need_b) + " (" + std::to_string(need_b) +
                                                 " bytes)";
        return set_error(QS_ERR_CAPACITY, std::to_string(num_qubits) + " qubits need " + need +
                                              "; memory budget is " + format_bytes(budget));
    }
    qs_state *s = new qs_state();
    std::memset(s, 0, sizeof *s);
    s->num_qubits = num_qubits;
    s->device = device;
    s->prec = precision;
    cudaError_t e = pool_alloc(device, need_b, (void **)&s->amps);
    if (e != cudaSuccess) {
        delete s;
        cudaGetLastError();
        return set_error(QS_ERR_CAPACITY, std::string("cudaMalloc of ") + std::to_string(need_b) +
                                              " bytes failed: " + cudaGetErrorString(e));
    }
    e = stream_acquire(device, &s->stream);
    if (e != cudaSuccess) {
        pool_free(device, s->amps, need_b);
        delete s;
        return cuda_fail(e, "cudaStreamCreateWithFlags");
    }
    cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device);
    int rc = init ? launch_reset(s, 0) : QS_OK;
    if (rc != QS_OK) {
        stream_release(device, s->stream);
        pool_free(device, s->amps, need_b);
        delete s;
        return rc;
    }
    *out = s;
    return QS_OK;
}

int qs_destroy(qs_state *s) {
    if (!s) return QS_OK;
    DeviceGuard guard(s->device);
    cudaStreamSynchronize(s->stream);  // the buffers may be recycled right away
    if (s->ipc_exported)
        cudaFree(s->amps);
    else
        pool_free(s->device, s->amps, state_bytes(s));
    pool_free(s->device, s->scratch, s->scratch_bytes);
    if (s->ops_dev) cudaFree(s->ops_dev);
    if (s->tile_ctr) pool_free(s->device, s->tile_ctr, 256);  // zero again once its last pass finished
    if (s->pinned) cudaFreeHost(s->pinned);
    stream_release(s->device, s->stream);
    delete s;
    return QS_OK;
}

int qs_num_qubits(const qs_state *s, int *out) {
    CHECK_HANDLE(s);
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    *out = s->num_qubits;
    return QS_OK;
}

int qs_precision(const qs_state *s, int *out) {
    CHECK_HANDLE(s);
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    *out = s->prec;
    return QS_OK;
}

int qs_device(const qs_state *s, int *out) {
    CHECK_HANDLE(s);
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    *out = s->device;
    return QS_OK;
}

int qs_device_pointer(qs_state *s, void **out) {
    CHECK_HANDLE(s);
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    *out = s->amps;
    return QS_OK;
}

int qs_stream(qs_state *s, void **out) {
    CHECK_HANDLE(s);
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    *out = (void *)s->stream;
    return QS_OK;
}

int qs_reset(qs_state *s, uint64_t basis) {
    CHECK_HANDLE(s);
    if (basis >> s->num_qubits)
        return set_error(QS_ERR_INDEX, "basis index " + std::to_string(basis) +
                                           " out of range [0, " +
                                           std::to_string(1ull << s->num_qubits) + ")");
    DeviceGuard guard(s->device);
    return launch_reset(s, basis);
}

int qs_synchronize(qs_state *s) {
    CHECK_HANDLE(s);
    DeviceGuard guard(s->device);
    QS_CUDA(cudaStreamSynchronize(s->stream));
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

// Gate entry points share the reference's check order (kernel.py:115-116,
// 145-150) and dispatch on the register's precision: complex64 sweeps take
// float32 entries (np.complex64-rounded), complex128 sweeps fp64 entries.
static int check_gate(const qs_state *s, const void *m, int target, int nctrl, const int *ctrl) {
    CHECK_HANDLE(s);
    if (!m) return set_error(QS_ERR_NULL, "null gate matrix");
    int rc = check_qubit(s, target, "target");
    if (rc) return rc;
    for (int i = 0; i < nctrl; ++i) {
        rc = check_qubit(s, ctrl[i], "control");
        if (rc) return rc;
    }
    for (int i = 0; i < nctrl; ++i)
        if (ctrl[i] == target) return set_error(QS_ERR_VALUE, "control and target must differ");
    if (nctrl == 2 && ctrl[0] == ctrl[1]) return set_error(QS_ERR_VALUE, "the two controls must differ");
    return QS_OK;
}

static int sweep_f32(qs_state *s, int target, uint64_t cmask, const float m[8]) {
    DeviceGuard guard(s->device);
    if (s->prec == QS_DOUBLE) {
        double md[8];
        for (int i = 0; i < 8; ++i) md[i] = (double)m[i];  // exact widening
        return launch_sweep_d(s, target, cmask, md);
    }
    return launch_sweep(s, target, cmask, m);
}

static int sweep_f64(qs_state *s, int target, uint64_t cmask, const double m[8]) {
    DeviceGuard guard(s->device);
    if (s->prec == QS_DOUBLE) return launch_sweep_d(s, target, cmask, m);
    float mf[8];
    for (int i = 0; i < 8; ++i) mf[i] = (float)m[i];  // round to nearest, as np.complex64(x)
    return launch_sweep(s, target, cmask, mf);
}

// apply_gate: pkg/src/pairsim/kernel.py:108-132
int qs_apply_gate(qs_state *s, int target, const float m[8]) {
    int rc = check_gate(s, m, target, 0, nullptr);
    return rc ? rc : sweep_f32(s, target, 0ull, m);
}

int qs_apply_gate_f64(qs_state *s, int target, const double m[8]) {
    int rc = check_gate(s, m, target, 0, nullptr);
    return rc ? rc : sweep_f64(s, target, 0ull, m);
}

// apply_controlled_gate: pkg/src/pairsim/kernel.py:135-165 (same check order)
int qs_apply_controlled_gate(qs_state *s, int control, int target, const float m[8]) {
    int rc = check_gate(s, m, target, 1, &control);
    return rc ? rc : sweep_f32(s, target, 1ull << control, m);
}

int qs_apply_controlled_gate_f64(qs_state *s, int control, int target, const double m[8]) {
    int rc = check_gate(s, m, target, 1, &control);
    return rc ? rc : sweep_f64(s, target, 1ull << control, m);
}

int qs_apply_controlled_controlled_gate(qs_state *s, int c1, int c2, int target,
                                        const float m[8]) {
    const int c[2] = {c1, c2};
    int rc = check_gate(s, m, target, 2, c);
    return rc ? rc : sweep_f32(s, target, (1ull << c1) | (1ull << c2), m);
}

int qs_apply_controlled_controlled_gate_f64(qs_state *s, int c1, int c2, int target,
                                            const double m[8]) {
    const int c[2] = {c1, c2};
    int rc = check_gate(s, m, target, 2, c);
    return rc ? rc : sweep_f64(s, target, (1ull << c1) | (1ull << c2), m);
}

int qs_apply_fused_ex(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops,
                      int flags) {
    CHECK_HANDLE(s);
    if (nops == 0) return QS_OK;
    if (!ops || !tile_qubits) return set_error(QS_ERR_NULL, "null op list or tile qubit list");
    DeviceGuard guard(s->device);
    if (s->prec == QS_DOUBLE) {  // exact widening of the float32 entries
        std::vector<qs_op64> wide((size_t)nops);
        for (int i = 0; i < nops; ++i) {
            wide[i].kind = ops[i].kind;
            wide[i].target = ops[i].target;
            wide[i].ctrl_mask = ops[i].ctrl_mask;
            for (int k = 0; k < 8; ++k) wide[i].m[k] = (double)ops[i].m[k];
        }
        return run_fused_d(s, tile_qubits, ntile, wide.data(), nops);
    }
    return run_fused(s, tile_qubits, ntile, ops, nops, flags);
}

int qs_apply_fused_from_basis(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops,
                              int flags, uint64_t basis) {
    CHECK_HANDLE(s);
    if (s->num_qubits < 64 && basis >= (1ull << s->num_qubits))
        return set_error(QS_ERR_INDEX, "basis index out of range");
    if (nops == 0 || s->prec == QS_DOUBLE) {  // nothing to fuse with / complex128: reset, then the pass
        if (int rc = qs_reset(s, basis)) return rc;
        return qs_apply_fused_ex(s, tile_qubits, ntile, ops, nops, flags);
    }
    if (!ops || !tile_qubits) return set_error(QS_ERR_NULL, "null op list or tile qubit list");
    DeviceGuard guard(s->device);
    return run_fused(s, tile_qubits, ntile, ops, nops, flags, (long long)basis);
}

int qs_apply_fused(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops) {
    return qs_apply_fused_ex(s, tile_qubits, ntile, ops, nops, 0);
}

int qs_apply_fused_f64(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op64 *ops,
                       int nops) {
    CHECK_HANDLE(s);
    if (nops == 0) return QS_OK;
    if (!ops || !tile_qubits) return set_error(QS_ERR_NULL, "null op list or tile qubit list");
    DeviceGuard guard(s->device);
    if (s->prec == QS_DOUBLE) return run_fused_d(s, tile_qubits, ntile, ops, nops);
    std::vector<qs_op> narrow((size_t)nops);
    for (int i = 0; i < nops; ++i) {
        narrow[i].kind = ops[i].kind;
        narrow[i].target = ops[i].target;
        narrow[i].ctrl_mask = ops[i].ctrl_mask;
        for (int k = 0; k < 8; ++k) narrow[i].m[k] = (float)ops[i].m[k];
    }
    return run_fused(s, tile_qubits, ntile, narrow.data(), nops);
}

int qs_swap_qubits(qs_state *s, int q1, int q2) {
    CHECK_HANDLE(s);
    int rc = check_qubit(s, q1, "qubit");
    if (rc) return rc;
    rc = check_qubit(s, q2, "qubit");
    if (rc) return rc;
    if (q1 == q2) return QS_OK;
    DeviceGuard guard(s->device);
    const int lo = q1 < q2 ? q1 : q2, hi = q1 < q2 ? q2 : q1;
    return s->prec == QS_DOUBLE ? launch_swap_d(s, lo, hi) : launch_swap(s, lo, hi);
}

static int check_range(const qs_state *s, uint64_t offset, uint64_t count) {
    uint64_t dim = 1ull << s->num_qubits;
    if (offset > dim || count > dim - offset)
        return set_error(QS_ERR_INDEX, "amplitude range [" + std::to_string(offset) + ", " +
                                           std::to_string(offset + count) + ") out of range [0, " +
                                           std::to_string(dim) + ")");
    return QS_OK;
}

int qs_get_amplitudes(qs_state *s, uint64_t offset, uint64_t count, void *host) {
    CHECK_HANDLE(s);
    int rc = check_range(s, offset, count);
    if (rc) return rc;
    if (count == 0) return QS_OK;
    if (!host) return set_error(QS_ERR_NULL, "null host buffer");
    DeviceGuard guard(s->device);
    QS_CUDA(cudaMemcpyAsync(host, (char *)s->amps + offset * amp_bytes(s), count * amp_bytes(s), cudaMemcpyDeviceToHost,
                            s->stream));
    QS_CUDA(cudaStreamSynchronize(s->stream));
    return QS_OK;
}

int qs_set_amplitudes(qs_state *s, uint64_t offset, uint64_t count, const void *host) {
    CHECK_HANDLE(s);
    int rc = check_range(s, offset, count);
    if (rc) return rc;
    if (count == 0) return QS_OK;
    if (!host) return set_error(QS_ERR_NULL, "null host buffer");
    DeviceGuard guard(s->device);
    QS_CUDA(cudaMemcpyAsync((char *)s->amps + offset * amp_bytes(s), host, count * amp_bytes(s), cudaMemcpyHostToDevice,
                            s->stream));
    // the caller may reuse `host` as soon as we return
    QS_CUDA(cudaStreamSynchronize(s->stream));
    return QS_OK;
}

int qs_set_amplitudes_async(qs_state *s, uint64_t offset, uint64_t count, const void *host) {
    CHECK_HANDLE(s);
    int rc = check_range(s, offset, count);
    if (rc) return rc;
    if (count == 0) return QS_OK;
    if (!host) return set_error(QS_ERR_NULL, "null host buffer");
    DeviceGuard guard(s->device);
    QS_CUDA(cudaMemcpyAsync((char *)s->amps + offset * amp_bytes(s), host, count * amp_bytes(s), cudaMemcpyHostToDevice,
                            s->stream));
    return QS_OK;
}

int qs_get_amplitudes_async(qs_state *s, uint64_t offset, uint64_t count, void *host) {
    CHECK_HANDLE(s);
    int rc = check_range(s, offset, count);
    if (rc) return rc;
    if (count == 0) return QS_OK;
    if (!host) return set_error(QS_ERR_NULL, "null host buffer");
    DeviceGuard guard(s->device);
    QS_CUDA(cudaMemcpyAsync(host, (char *)s->amps + offset * amp_bytes(s), count * amp_bytes(s), cudaMemcpyDeviceToHost,
                            s->stream));
    return QS_OK;
}

int qs_probabilities(qs_state *s, uint64_t offset, uint64_t count, double *host) {
    CHECK_HANDLE(s);
    int rc = check_range(s, offset, count);
    if (rc) return rc;
    if (count == 0) return QS_OK;
    if (!host) return set_error(QS_ERR_NULL, "null host buffer");
    DeviceGuard guard(s->device);
    return run_probabilities(s, offset, count, host);
}

int qs_norm_squared(qs_state *s, double *out) {
    CHECK_HANDLE(s);
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    DeviceGuard guard(s->device);
    return run_norm(s, out);
}

// sample: pkg/src/pairsim/measure.py:76-85
int qs_sample(qs_state *s, const qs_pcg64 *rng, int64_t k, int64_t *out) {
    CHECK_HANDLE(s);
    if (k < 1) return set_error(QS_ERR_VALUE, "n_samples must be >= 1");
    if (!rng || !out) return set_error(QS_ERR_NULL, "null rng or output buffer");
    DeviceGuard guard(s->device);
    return run_sample(s, rng, k, out);
}

int qs_sample_prepare(qs_state *s, int64_t k) {
    CHECK_HANDLE(s);
    if (k < 1) return set_error(QS_ERR_VALUE, "n_samples must be >= 1");
    DeviceGuard guard(s->device);
    double *csum = nullptr;
    int rc = run_sample_prepare(s, k, &csum);
    s->csum_dst = csum;
    return rc;
}

int qs_sample_ex(qs_state *s, const qs_pcg64 *rng, int64_t k, int64_t *out, int flags) {
    CHECK_HANDLE(s);
    if (k < 1) return set_error(QS_ERR_VALUE, "n_samples must be >= 1");
    if (!rng || !out) return set_error(QS_ERR_NULL, "null rng or output buffer");
    DeviceGuard guard(s->device);
    return run_sample(s, rng, k, out, (flags & QS_SAMPLE_SUMS_READY) != 0);
}

// measure_collapse: pkg/src/pairsim/measure.py:88-99
int qs_measure_collapse(qs_state *s, const qs_pcg64 *rng, int64_t *outcome) {
    CHECK_HANDLE(s);
    if (!rng || !outcome) return set_error(QS_ERR_NULL, "null rng or output pointer");
    DeviceGuard guard(s->device);
    int64_t m = 0;
    int rc = run_sample(s, rng, 1, &m);
    if (rc) return rc;
    rc = launch_reset(s, (uint64_t)m);
    if (rc) return rc;
    *outcome = m;
    return QS_OK;
}

int qs_cdf_extend(qs_state *s, double start, double *end) {
    CHECK_HANDLE(s);
    if (!end) return set_error(QS_ERR_NULL, "null output pointer");
    DeviceGuard guard(s->device);
    return run_cdf_extend(s, start, end);
}

int qs_sample_shard(qs_state *s, const qs_pcg64 *rng, int64_t k, double start, double total,
                    uint64_t index_base, uint64_t global_dim, int is_last, int64_t *out) {
    CHECK_HANDLE(s);
    if (k < 1) return set_error(QS_ERR_VALUE, "n_samples must be >= 1");
    if (!rng || !out) return set_error(QS_ERR_NULL, "null rng or output buffer");
    const uint64_t dim = 1ull << s->num_qubits;
    if (global_dim < dim || index_base > global_dim - dim)
        return set_error(QS_ERR_INDEX, "slice [index_base, index_base + 2^n) outside global_dim");
    DeviceGuard guard(s->device);
    return run_sample_shard(s, rng, k, start, total, index_base, global_dim, is_last, out);
}

}  // extern "C"

// ---- CUDA graphs: record a run of gate launches once, replay it -------------
// For launch-bound registers (small n, many gates) a recorded gate sequence
// replays as one graph launch.  Only asynchronous calls may be recorded: gate,
// fused-pass, reset and amplitude-upload calls; getters (which synchronise)
// fail while recording.
struct qs_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int device = 0;
};

extern "C" {

int qs_begin_capture(qs_state *s) {
    CHECK_HANDLE(s);
    DeviceGuard guard(s->device);
    // relaxed: a handle destroyed elsewhere in the recording thread (cudaFree
    // of its buffer) must not invalidate the recording
    QS_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeRelaxed));
    return QS_OK;
}

int qs_end_capture(qs_state *s, qs_graph **out) {
    CHECK_HANDLE(s);
    if (!out) return set_error(QS_ERR_NULL, "null output pointer");
    *out = nullptr;
    DeviceGuard guard(s->device);
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(s->stream, &g);
    cudaGetLastError();  // a call that broke the recording must not poison later checks
    if (ec != cudaSuccess) return cuda_fail(ec, "cudaStreamEndCapture");
    qs_graph *h = new qs_graph();
    h->graph = g;
    h->device = s->device;
    cudaError_t e = cudaGraphInstantiate(&h->exec, g, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        delete h;
        return cuda_fail(e, "cudaGraphInstantiate");
    }
    *out = h;
    return QS_OK;
}

int qs_graph_launch(qs_state *s, qs_graph *g) {
    CHECK_HANDLE(s);
    if (!g) return set_error(QS_ERR_NULL, "null graph");
    if (g->device != s->device) return set_error(QS_ERR_VALUE, "graph was recorded on another device");
    DeviceGuard guard(s->device);
    QS_CUDA(cudaGraphLaunch(g->exec, s->stream));
    return QS_OK;
}

int qs_graph_destroy(qs_graph *g) {
    if (!g) return QS_OK;
    DeviceGuard guard(g->device);
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return QS_OK;
}

}  // extern "C"
