/*
 * qsb200.h — C ABI of the B200-native state-vector backend (libqsb200.so).
 *
 * The reference (pairsim, /root/reference/pkg/src/pairsim) has no FFI: its
 * boundary is a Python function API over a host numpy buffer.  This header is
 * the native seam that the Python host layer (paper_1805_00988_b200/) binds
 * with ctypes; every entry point below names the reference function whose
 * semantics it reproduces.
 *
 * Conventions
 *   - Amplitudes are complex64 (interleaved (re, im) float32) or, for
 *     registers created with QS_DOUBLE, complex128 (interleaved float64) —
 *     pairsim's Precision.SINGLE / DOUBLE (pkg/src/pairsim/state.py:25-42).
 *     Qubit t = bit t of the basis index (pkg/src/pairsim/state.py:3-5).
 *   - A 2x2 gate [[a, b], [c, d]] is passed as float m[8] =
 *     {a.re, a.im, b.re, b.im, c.re, c.im, d.re, d.im}, already rounded to
 *     float32 exactly as `np.complex64(x)` rounds (pkg/src/pairsim/kernel.py:118-119).
 *   - Every call returns an int status; 0 = QS_OK.  On failure the message is
 *     available from qs_last_error() (thread-local).
 *   - A handle owns one device buffer and one CUDA stream.  Mutating calls are
 *     asynchronous on that stream (stream order is the sweep barrier of
 *     pkg/src/pairsim/kernel.py:244-245); getters synchronize.  One host thread
 *     per handle at a time.
 */
#ifndef QSB200_H
#define QSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSB200_ABI_VERSION 2

/* Register precision (pkg/src/pairsim/state.py:25-42). */
enum { QS_SINGLE = 0, QS_DOUBLE = 1 };

/* Status codes.  The Python layer maps them onto the reference's exception
 * taxonomy (pkg/src/pairsim/errors.py:4-37). */
enum {
    QS_OK = 0,
    QS_ERR_INDEX = 1,      /* IndexError: qubit or basis index out of range   */
    QS_ERR_VALUE = 2,      /* ValueError: control == target, n < 1, k < 1 ... */
    QS_ERR_CAPACITY = 3,   /* CapacityError: register over the memory budget  */
    QS_ERR_DEGENERATE = 4, /* DegenerateStateError: all probabilities zero    */
    QS_ERR_CUDA = 5,       /* CUDA runtime failure (message has the details)  */
    QS_ERR_NULL = 6        /* null handle or output pointer                   */
};

typedef struct qs_state qs_state;

/* numpy PCG64 generator state (bit_generator.state["state"]), split into
 * 64-bit halves.  Draws are (next64 >> 11) * 2^-53, exactly numpy's
 * Generator.random() (pkg/src/pairsim/measure.py:81-82). */
typedef struct {
    uint64_t state_hi, state_lo;
    uint64_t inc_hi, inc_lo;
} qs_pcg64;

/* One operation of a fused pass (qs_apply_fused). */
enum {
    QS_OP_PAIR = 0,  /* 2x2 pair update on `target` under `ctrl_mask`           */
    QS_OP_PHASE = 1  /* amps with every bit of (1<<target | ctrl_mask) set are
                        multiplied by d; requires a == 1, b == c == 0          */
};

typedef struct {
    int32_t kind;       /* QS_OP_PAIR or QS_OP_PHASE                              */
    int32_t target;     /* global qubit index                                     */
    uint64_t ctrl_mask; /* global control qubits (all must be 1); excludes target */
    float m[8];         /* gate entries, as for qs_apply_gate                      */
} qs_op;

/* The same op with fp64 gate entries (complex128 registers). */
typedef struct {
    int32_t kind;
    int32_t target;
    uint64_t ctrl_mask;
    double m[8];
} qs_op64;

/* ---- library ------------------------------------------------------------ */
int qs_abi_version(void);
const char *qs_last_error(void);
int qs_device_count(int *out);
/* Return cached register buffers / streams of `device` (all devices when
 * device < 0) to the driver.  Destroyed handles park their buffers in a
 * bounded per-device cache (QSB_CACHE_BYTES, default 1/4 of HBM) so that
 * new_state-style create/destroy cycles skip cudaMalloc/cudaFree. */
int qs_release_cached(int device);
/* Page-locked host memory (cudaMallocHost): readouts into it (qs_probabilities,
 * qs_get_amplitudes) go straight to it by DMA, without staging copies or page
 * faults — for callers that read large registers repeatedly. */
int qs_host_alloc(uint64_t bytes, void **out);
int qs_host_free(void *ptr);

/* ---- lifecycle: pkg/src/pairsim/state.py:122-143 (new_state) ------------ */
/* Allocates 8 * 2^n bytes on `device` and initialises |0...0>.
 * memory_budget == 0 selects the default budget: 75% of the device's free
 * memory (the GPU analogue of default_memory_budget, state.py:114-119).
 * Fails with QS_ERR_CAPACITY *before* allocating when over budget; a budget
 * equal to the need is allowed (pkg/tests/test_state.py:45-52). */
int qs_create(int num_qubits, int device, uint64_t memory_budget, qs_state **out);
/* As qs_create with an explicit precision (QS_SINGLE or QS_DOUBLE); a
 * complex128 register needs 16 * 2^n bytes (memory_required, state.py:71-83). */
int qs_create_ex(int num_qubits, int device, uint64_t memory_budget, int precision, qs_state **out);
/* qs_create_ex with the register's contents left undefined (no clear): for a
 * circuit whose first fused pass writes its start state anyway
 * (qs_apply_fused_from_basis).  Reading it before that is unspecified. */
int qs_create_uninit(int num_qubits, int device, uint64_t memory_budget, int precision, qs_state **out);
int qs_precision(const qs_state *s, int *out);
int qs_destroy(qs_state *s);
int qs_num_qubits(const qs_state *s, int *out);
int qs_device(const qs_state *s, int *out);
/* Raw device pointer / cudaStream_t of the handle (for transports and
 * device-side timing; the pointer stays owned by the handle). */
int qs_device_pointer(qs_state *s, void **out);
int qs_stream(qs_state *s, void **out);
/* Overwrite the register with basis state |basis> (amps = e_basis). */
int qs_reset(qs_state *s, uint64_t basis);
int qs_synchronize(qs_state *s);

/* ---- gates: pkg/src/pairsim/kernel.py:108-165 --------------------------- */
/* apply_gate (kernel.py:108-132): per pair (a, b = a|1<<t):
 *   v_a' = m_a v_a + m_b v_b ;  v_b' = m_d v_b + m_c v_a   (pre-update values) */
int qs_apply_gate(qs_state *s, int target, const float m[8]);
/* apply_controlled_gate (kernel.py:135-165): same update where bit `control`
 * is 1; QS_ERR_INDEX out of range, QS_ERR_VALUE when control == target. */
int qs_apply_controlled_gate(qs_state *s, int control, int target, const float m[8]);
/* Doubly-controlled update (QCGPU's apply_controlled_controlled_gate; no
 * pairsim counterpart): the update where bits c1 and c2 are both 1. */
int qs_apply_controlled_controlled_gate(qs_state *s, int c1, int c2, int target, const float m[8]);
/* fp64 gate entries: exact on a complex128 register; rounded to float32 (as
 * np.complex64(x) rounds, kernel.py:118-119) on a complex64 register.  The
 * float32 entry points above widen exactly on a complex128 register. */
int qs_apply_gate_f64(qs_state *s, int target, const double m[8]);
int qs_apply_controlled_gate_f64(qs_state *s, int control, int target, const double m[8]);
int qs_apply_controlled_controlled_gate_f64(qs_state *s, int c1, int c2, int target,
                                            const double m[8]);
/* Fused pass: one HBM read+write of the register applies `ops` in order,
 * bit-identical to applying them one by one.  `tile_qubits` (ntile entries,
 * must contain 0..5 when num_qubits >= 6) is the set of qubits held in each
 * on-chip tile; every QS_OP_PAIR target must be in it (controls and phase
 * bits may be anywhere). */
int qs_apply_fused(qs_state *s, const int32_t *tile_qubits, int ntile,
                   const qs_op *ops, int nops);
/* qs_apply_fused with flags.  QS_FUSED_COMBINE_PHASES (opt-in, NOT
 * bit-exact): in the compiled pass programs, each run of consecutive
 * unit-modulus diagonal ops (u1 / z / s / t and controlled forms) becomes one
 * complex product per amplitude by the run's accumulated phase (angles summed
 * exactly in fixed-point turns) instead of one product per op; results agree
 * with the sequential ops to rounding (~1e-6 relative; tested at the
 * north_star rtol 1e-5).  complex128 registers ignore the flag. */
enum { QS_FUSED_COMBINE_PHASES = 1, QS_FUSED_CHUNK_SUMS = 2 };
int qs_apply_fused_ex(qs_state *s, const int32_t *tile_qubits, int ntile,
                      const qs_op *ops, int nops, int flags);
/* qs_reset(s, basis) followed by qs_apply_fused_ex(...), as ONE HBM write:
 * the pass's tiles are written as |basis> (zeros, 1 at the basis amplitude)
 * instead of being loaded, so the register is never cleared separately.
 * Same result bit for bit.  Falls back to the two calls when the pass has
 * no tile kernel (small registers, unusual tile shapes) or is complex128.
 * New entry point; pairsim's equivalent is new_state + run_circuit
 * (pkg/src/pairsim/state.py:122-143, circuits.py:171-192). */
int qs_apply_fused_from_basis(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops,
                              int flags, uint64_t basis);
/* Fused pass with fp64 gate entries (the form a complex128 register takes;
 * on a complex64 register the entries are rounded to float32 and the call
 * is qs_apply_fused). */
int qs_apply_fused_f64(qs_state *s, const int32_t *tile_qubits, int ntile,
                       const qs_op64 *ops, int nops);
/* Fused passes are compiled at run time into straight-line kernels (NVRTC,
 * host worker threads); until a pass's program is ready it runs on the
 * interpreter kernel, with the same bits.  Wait for every queued compile and
 * load the programs of `device` (< 0: all).  Not needed for correctness. */
int qs_jit_sync(int device);
/* Pass programs this process compiled with NVRTC, loaded from the on-disk
 * program cache (QSB_JIT_CACHE_DIR / ~/.cache/qsb200-jit; QSB_JIT_CACHE=0
 * disables it), and failed to build. */
int qs_jit_stats(uint64_t *compiled, uint64_t *cache_hits, uint64_t *failed);
/* Drop queued compiles, let an in-flight one finish and stop the compile
 * threads (call before process teardown; the Python layer registers it with
 * atexit).  Later fused passes run on the interpreter kernel. */
int qs_jit_shutdown(void);
/* Swap qubits q1 and q2 (a basis permutation; used by the sharded layer). */
int qs_swap_qubits(qs_state *s, int q1, int q2);

/* ---- readout: state.py:146-161, measure.py:29-99 ------------------------- */
/* `host` holds `count` amplitudes of the register's precision (float pairs
 * for QS_SINGLE, double pairs for QS_DOUBLE). */
int qs_get_amplitudes(qs_state *s, uint64_t offset, uint64_t count, void *host);
int qs_set_amplitudes(qs_state *s, uint64_t offset, uint64_t count, const void *host);
/* Asynchronous variants: enqueue the copy on the handle's stream and return.
 * `host` must stay valid (and, for full overlap, be pinned) until the next
 * qs_synchronize on this handle. */
int qs_set_amplitudes_async(qs_state *s, uint64_t offset, uint64_t count, const void *host);
int qs_get_amplitudes_async(qs_state *s, uint64_t offset, uint64_t count, void *host);
/* probabilities (measure.py:29-34): p[j] = re^2 + im^2 in fp64, bit-exact
 * (complex128: rn(rn(re*re) + rn(im*im)), numpy's three separate roundings). */
int qs_probabilities(qs_state *s, uint64_t offset, uint64_t count, double *host);
/* norm_squared (state.py:146-151): fp64 sum of |a|^2 (tree order). */
int qs_norm_squared(qs_state *s, double *out);
/* sample (measure.py:76-85): k draws from `rng` against the normalised
 * sequential fp64 CDF, searchsorted(side="right"), clamped to dim-1.
 * out[i] is the outcome of draw i.  Bit-exact with the reference for the
 * same generator state.  QS_ERR_DEGENERATE when all probabilities are 0. */
int qs_sample(qs_state *s, const qs_pcg64 *rng, int64_t k, int64_t *out);
/* A circuit's last fused pass feeding a sample: qs_sample_prepare(h, k) lays
 * out the sampler's scratch for k draws and zeroes its chunk sums; the next
 * fused pass with QS_FUSED_CHUNK_SUMS adds each tile's |a|^2 row sums into
 * them as it writes the tile back (no extra read of the register), and
 * qs_sample_ex(..., QS_SAMPLE_SUMS_READY) skips its own chunk-sum pass (M1).
 * The sums only seed the exact chain's guesses: draws are bit-identical to
 * qs_sample either way. */
enum { QS_SAMPLE_SUMS_READY = 1 };
int qs_sample_prepare(qs_state *s, int64_t k);
int qs_sample_ex(qs_state *s, const qs_pcg64 *rng, int64_t k, int64_t *out, int flags);
/* measure_collapse (measure.py:88-99): one draw, then amps = e_outcome. */
int qs_measure_collapse(qs_state *s, const qs_pcg64 *rng, int64_t *outcome);

/* ---- sharded registers (one slice of a larger logical register) ---------- */
/* The exact sequential cumsum of this register's probabilities continued from
 * `start` (the running value after all earlier slices): *end = final value.
 * Chaining slices reproduces numpy's cumsum over the concatenation bit for bit. */
int qs_cdf_extend(qs_state *s, double start, double *end);
/* Draws against the global normalised CDF when this register is the slice
 * [index_base, index_base + 2^n) of a global_dim register whose running sum
 * enters the slice at `start` and ends at `total` (last slice: is_last = 1).
 * out[i] = global outcome of draw i if it falls in this slice, else -1; each
 * draw falls in exactly one slice.  Same draws as qs_sample for the same rng. */
int qs_sample_shard(qs_state *s, const qs_pcg64 *rng, int64_t k, double start, double total,
                    uint64_t index_base, uint64_t global_dim, int is_last, int64_t *out);

/* ---- CUDA graphs: record a gate sequence once, replay it --------------------- */
/* Between qs_begin_capture and qs_end_capture, the asynchronous calls on the
 * handle (gates, fused passes, reset, uploads) are recorded instead of run;
 * qs_graph_launch replays them as one graph launch on the same handle (the
 * recording addresses the capturing handle's buffer).  Getters synchronise and fail while
 * recording.  For launch-bound (small) registers and repeated circuits. */
typedef struct qs_graph qs_graph;
int qs_begin_capture(qs_state *s);
int qs_end_capture(qs_state *s, qs_graph **out);
int qs_graph_launch(qs_state *s, qs_graph *g);
int qs_graph_destroy(qs_graph *g);

/* ---- global-qubit gates over peer memory (sharded registers) --------------- */
/* cudaIpc handle (64 bytes) of the register's device buffer, and mapping a
 * partner process's handle into this process on `device` (NVLink P2P). */
int qs_ipc_handle(qs_state *s, void *out64);
int qs_ipc_open(int device, const void *handle64, void **out);
int qs_ipc_close(int device, void *ptr);
/* The pair update of apply_gate / apply_controlled_gate (kernel.py:108-165)
 * for a target on a GLOBAL qubit of a sharded register, in one kernel: this
 * shard and `peer_amps` (the partner shard, same local index space) hold the
 * two amplitudes of every pair; own_is_a = 1 on the shard whose rank bit is 0.
 * Both partners call it concurrently; each updates half of the pairs (split
 * on the highest local non-control bit), reading and writing the partner's
 * amplitudes through peer memory.  ctrl_mask = local control bits (controls
 * on other global qubits are rank predicates of the caller).  The caller
 * orders the two shards' streams before and after. */
int qs_apply_gate_peer(qs_state *s, void *peer_amps, int own_is_a, uint64_t ctrl_mask, const float m[8]);
/* The same with fp64 entries (complex128 shards; on complex64 shards the
 * entries are rounded to float32).  qs_swap_peer works on either precision. */
int qs_apply_gate_peer_f64(qs_state *s, void *peer_amps, int own_is_a, uint64_t ctrl_mask, const double m[8]);
/* Qubit-swap exchange over peer memory (the data movement of a global-target
 * swap, sharded.py's exchange_plan): amplitudes [own_offset, own_offset +
 * count) of this shard trade places with [peer_offset, peer_offset + count)
 * of the partner's, in one kernel on this handle's stream (16-B accesses, no
 * staging buffer).  Partners split the exchanged range between them and call
 * it concurrently on disjoint parts; the caller orders both streams before
 * and after. */
int qs_swap_peer(qs_state *s, void *peer_amps, uint64_t own_offset, uint64_t peer_offset, uint64_t count);

/* ---- registers sharded over several GPUs by ONE process ----------------------
 * SURVEY 8(b) qs_create_sharded / 8(e): n qubits over nshards = 2^g shards on
 * the top g qubits, shard r (the slice [r 2^L, (r+1) 2^L), L = n - g) on
 * device devs[r] (devices may repeat: several shards per GPU).  Same gate and
 * readout semantics as the single-device calls (the pairsim functions they
 * cite); a gate on a global qubit swaps it with local qubit L-1 through an
 * exchange of half of each partner shard (NCCL send/recv over NVLink with one
 * communicator per device from ncclCommInitAll, libnccl loaded at run time;
 * or a peer-memory swap kernel), or with peer gates on runs one pair kernel
 * over peer memory.  Readout un-permutes the lazy qubit map.  memory_budget
 * applies per shard (0: 75% of each device's free memory).
 * Reference anchor: paper_1805_00988_b200/sharded.py (the torch.distributed
 * multi-process form of the same layout). */
typedef struct qs_sharded qs_sharded;
enum { QS_EXCHANGE_NCCL = 1, QS_EXCHANGE_P2P = 2 };
int qs_create_sharded(int num_qubits, int nshards, const int *devs, uint64_t memory_budget, qs_sharded **out);
int qs_sharded_destroy(qs_sharded *h);
int qs_sharded_info(const qs_sharded *h, int *num_qubits, int *nshards, int *shard_qubits);
int qs_sharded_shard(qs_sharded *h, int rank, qs_state **out);
/* peer_gates: 1 on, 0 off, -1 unchanged; exchange: QS_EXCHANGE_NCCL / _P2P (0: unchanged) */
int qs_sharded_set_mode(qs_sharded *h, int peer_gates, int exchange);
int qs_sharded_stats(const qs_sharded *h, uint64_t *swaps, uint64_t *peer_gates, int *exchange);
int qs_sharded_reset(qs_sharded *h, uint64_t basis);
int qs_sharded_apply_gate(qs_sharded *h, int target, const float m[8]);
int qs_sharded_apply_controlled_gate(qs_sharded *h, int control, int target, const float m[8]);
int qs_sharded_apply_controlled_controlled_gate(qs_sharded *h, int c1, int c2, int target, const float m[8]);
int qs_sharded_synchronize(qs_sharded *h);
/* The lazy qubit map (pos[logical] = physical position; >= shard_qubits =
 * global) and a qubit swap bringing `qubit` to a local position: with
 * qs_sharded_shard, what a caller needs to run fused passes of local ops on
 * the shards between global-target gates (multigpu.MultiDeviceState.run). */
int qs_sharded_qubit_map(const qs_sharded *h, int32_t *pos);
int qs_sharded_localize(qs_sharded *h, int qubit);
int qs_sharded_get_amplitudes(qs_sharded *h, uint64_t offset, uint64_t count, void *host);
int qs_sharded_set_amplitudes(qs_sharded *h, uint64_t offset, uint64_t count, const void *host);
int qs_sharded_probabilities(qs_sharded *h, uint64_t offset, uint64_t count, double *host);
int qs_sharded_norm_squared(qs_sharded *h, double *out);
int qs_sharded_sample(qs_sharded *h, const qs_pcg64 *rng, int64_t k, int64_t *out);

#ifdef __cplusplus
}
#endif

#endif /* QSB200_H */
