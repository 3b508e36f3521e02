// Host-side internals shared by the libqsb200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "qsb200.h"

struct qs_state {
    int num_qubits;
    int device;
    float2 *amps;          // 2^n amplitudes, 256-B aligned (cudaMalloc); double2 when prec == 1
    int prec;              // QS_SINGLE (complex64) or QS_DOUBLE (complex128)
    cudaStream_t stream;   // all work on this handle is ordered on it
    int num_sms;
    // measurement scratch (lazily grown; freed with the handle)
    void *scratch;
    size_t scratch_bytes;
    void *pinned;          // small pinned host buffer for results
    size_t pinned_bytes;
    // fused-pass op buffer (device copy of qs_op arrays)
    void *ops_dev;
    size_t ops_bytes;
    // fused-pass tile scheduler counter (lazily allocated, zero between launches)
    unsigned long long *tile_ctr;
    // the register buffer was exported with cudaIpcGetMemHandle: other
    // processes may still map it, so it is freed, never recycled by the pool
    int ipc_exported;
    // the last fused pass (QS_FUSED_CHUNK_SUMS) left the sampler's chunk sums
    // (M1) in scratch; consumed / cleared by the next sample or pass
    int csum_ready;
    double *csum_dst;  // qs_sample_prepare's chunk-sum array in scratch (nullptr: none)
};

#include <nvtx3/nvToolsExt.h>  // header-only; a no-op unless a tool (ncu / nsys) is attached

namespace qsb {

// NVTX range for the duration of a scope (SURVEY 5 tracing: per pass,
// exchange, readout) — visible to ncu --nvtx / nsys timelines.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int set_error(int code, const std::string &msg);

// bytes per amplitude: 8 (complex64) or 16 (complex128)
inline uint64_t amp_bytes(const qs_state *s) { return s->prec == QS_DOUBLE ? 16ull : 8ull; }
inline uint64_t state_bytes(const qs_state *s) { return amp_bytes(s) << s->num_qubits; }
inline double2 *amps_d(const qs_state *s) { return reinterpret_cast<double2 *>(s->amps); }
int cuda_fail(cudaError_t e, const char *what);
// Fault injection for the parity suite (the sign-flipped `c` of
// pkg/tests/test_cli.py:151-160): QSB_FAULT_FLIP_C=1 negates the c entry of
// every pair gate in the sweep and fused paths.  Debug only.
bool fault_flip_c();
// raise a kernel's max dynamic shared memory on the current device (once per size)
int ensure_smem_attr(const void *fn, int bytes);

// RAII guard: switch to the handle's device for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int ensure_scratch(qs_state *s, size_t bytes);
int ensure_pinned(qs_state *s, size_t bytes);

// device-memory / stream caches (pool.cu)
cudaError_t pool_alloc(int device, size_t bytes, void **out);
void pool_free(int device, void *ptr, size_t bytes);
size_t pool_cached(int device);
void pool_trim(int device);
cudaError_t stream_acquire(int device, cudaStream_t *out);
void stream_release(int device, cudaStream_t s);

// kernels (gates.cu / measure.cu / fused.cu)
int launch_sweep(qs_state *s, int target, uint64_t ctrl_mask, const float m[8]);
int launch_phase(qs_state *s, uint64_t mask, float2 d);
int launch_swap(qs_state *s, int q1, int q2);
int launch_reset(qs_state *s, uint64_t basis);
// complex128 registers (gates64.cu)
int launch_sweep_d(qs_state *s, int target, uint64_t ctrl_mask, const double m[8]);
int launch_phase_d(qs_state *s, uint64_t mask, double2 d);
int launch_swap_d(qs_state *s, int q1, int q2);
int launch_reset_d(qs_state *s, uint64_t basis);
int run_fused_d(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op64 *ops, int nops);
int run_fused_tiles_d(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op64 *ops, int nops);
int run_probabilities(qs_state *s, uint64_t offset, uint64_t count, double *host);
int run_norm(qs_state *s, double *out);
int run_sample(qs_state *s, const qs_pcg64 *rng, int64_t k, int64_t *out, bool sums_ready = false);
int run_sample_prepare(qs_state *s, int64_t k, double **csum);
int run_cdf_extend(qs_state *s, double start, double *end);
int run_sample_shard(qs_state *s, const qs_pcg64 *rng, int64_t k, double start, double total,
                     uint64_t base, uint64_t gdim, int is_last, int64_t *out);
int run_fused(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops, int flags = 0,
              long long basis = -1);

}  // namespace qsb

#define QS_CUDA(call)                                          \
    do {                                                       \
        cudaError_t _e = (call);                               \
        if (_e != cudaSuccess) return qsb::cuda_fail(_e, #call); \
    } while (0)
