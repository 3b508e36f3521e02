// Probability / measurement chain (K7-K10) for sm_100a.
//
// probabilities (pkg/src/pairsim/measure.py:29-34): p = re*re + im*im in fp64.
// Both squares of a float32 are exact in fp64, so one __dadd_rn reproduces
// numpy bit for bit.
//
// sample (measure.py:68-85) draws u = (pcg64_next >> 11) * 2^-53 and returns
// searchsorted(cdf / cdf[-1], u, side="right") clamped to dim-1, where cdf is
// numpy's *sequential* fp64 cumsum.  A parallel scan rounds differently, so
// the device reproduces the sequential sum exactly with a shift-equivariance
// argument:
//
//   Inside one binade [2^e, 2^(e+1)) doubles lie on a grid of spacing
//   u = ulp(2^e), and round-to-nearest onto that grid commutes with shifts by
//   even multiples of u (odd multiples flip ties-to-even).  So if a chunk's
//   sequential trajectory is computed from a guessed start g0 (an even grid
//   point) and from g1 = g0 + u, and both trajectories stay inside the binade,
//   then the trajectory from the true start s = g0 + m*u (same binade) is the
//   g0 trajectory shifted by m*u when m is even and the g1 trajectory shifted
//   by (m-1)*u when m is odd — exactly, including every rounding.
//
// Pipeline (C = 4096 amplitudes per chunk):
//   M1 k_chunk_sums   parallel fp64 chunk sums (any order: guesses only)
//   M2 scan_guess     two-level exclusive scan of the sums -> guessed chunk starts
//   M3 k_trajectories both guessed trajectories per chunk (warp-transposed
//                     through shared memory so HBM reads stay coalesced)
//   M4 true chunk starts: the parity of s's mantissa selects the
//                     trajectory, end = s + D exactly — composed as parity
//                     maps over blocks of chunks (k_block_maps / k_block_walk
//                     / k_block_fill); chunks that cross a binade (or whose
//                     guess fell in the wrong binade) are re-summed
//                     sequentially from s
//   M5 k_chunk_last   normalised CDF value at each chunk end
//   M6 k_draws        per draw: PCG64 jump-ahead, binary search over chunk
//                     ends, then the sequential in-chunk walk from the exact
//                     chunk start to the first fl(cdf/total) > u.
// No N-sized CDF is materialised; every value compared against u equals the
// reference's cdf[j] / total bit for bit.

#include <sys/mman.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace qsb {

namespace {

constexpr int kChunkLog = 12;  // 4096 amplitudes per chunk
static_assert(kChunkLog == kCdfChunkLog, "fused-pass chunk sums use the sampler's chunk size");

__device__ __forceinline__ double prob(float2 a) {
    double re = (double)a.x, im = (double)a.y;
    return __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
}
// complex128 (measure.py:31-34 on a complex128 array): re*re, im*im and their
// sum are three separately rounded numpy passes.
__device__ __forceinline__ double prob(double2 a) {
    return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

// A = float2 (complex64 register) or double2 (complex128 register)
template <class A>
__global__ void k_probs(const A *__restrict__ amps, double *__restrict__ out, uint64_t count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = prob(amps[i]);
}

// ---- norm: fixed-shape two-pass tree reduction (deterministic) -------------
constexpr int kNormBlocks = 1024;
constexpr int kNormThreads = 256;

__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? sh[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

template <class A>
__global__ void k_norm_partial(const A *__restrict__ amps, uint64_t n, double *partial) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        acc += prob(amps[i]);
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void k_norm_final(const double *partial, int n, double *out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) *out = acc;
}

// ---- M1: chunk sums ---------------------------------------------------------
template <class A>
__global__ void k_chunk_sums(const A *__restrict__ amps, int clog, double *__restrict__ csum) {
    __shared__ double sh[32];
    const uint64_t c = blockIdx.x;
    const uint64_t C = 1ull << clog;
    const A *p = amps + (c << clog);
    double acc = 0.0;
    for (uint64_t j = threadIdx.x; j < C; j += blockDim.x) acc += prob(p[j]);
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) csum[c] = acc;
}
// complex64 with 4096-amplitude chunks: 16-B loads, all eight of a thread's
// loads in flight at once (the sums are guesses: any order will do)
__global__ void __launch_bounds__(256) k_chunk_sums_f4(const float4 *__restrict__ amps, double *__restrict__ csum) {
    __shared__ double sh[32];
    const float4 *p = amps + (blockIdx.x << (kChunkLog - 1));
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldcs(p + threadIdx.x + 256 * i);
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += prob(make_float2(v[i].x, v[i].y)) + prob(make_float2(v[i].z, v[i].w));
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) csum[blockIdx.x] = acc;
}

// ---- M2: exclusive scan of chunk sums -> guessed chunk starts ----------------
// Only a GUESS of every chunk's start is needed (M3-M5 resolve the exact
// sequential values), so any summation order will do; a sum of non-negative
// terms is 0 exactly when every term is 0, which is all M3 relies on.  Two
// levels: per-segment sums (coalesced), one block scanning the segment sums,
// then each segment's in-block scan plus its offset.
constexpr int kScanThreads = 256, kScanPer = 8, kScanSeg = kScanThreads * kScanPer;

__device__ __forceinline__ double block_excl_scan(double v, double *warp_tot, double &total) {
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (unsigned)o) inc += t;
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    double base = 0.0, all = 0.0;
    const unsigned nw = blockDim.x >> 5;
    for (unsigned i = 0; i < nw; ++i) {
        if (i == w) base = all;
        all += warp_tot[i];
    }
    __syncthreads();
    total = all;
    return base + inc - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_seg_sums(const double *__restrict__ csum, uint64_t nch,
                                                                double *__restrict__ ssum) {
    __shared__ double wt[kScanThreads / 32];
    const uint64_t lo = (uint64_t)blockIdx.x * kScanSeg;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        const uint64_t i = lo + (uint64_t)j * kScanThreads + threadIdx.x;
        if (i < nch) acc += csum[i];
    }
    double total;
    block_excl_scan(acc, wt, total);
    if (threadIdx.x == 0) ssum[blockIdx.x] = total;
}

// one block: in-place exclusive scan of the nseg segment sums
__global__ void __launch_bounds__(1024) k_scan_seg_top(double *__restrict__ ssum, uint64_t nseg) {
    __shared__ double wt[32];
    const uint64_t per = (nseg + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = threadIdx.x * per;
    const uint64_t hi = lo + per < nseg ? lo + per : nseg;
    double acc = 0.0;
    for (uint64_t i = lo; i < hi; ++i) acc += ssum[i];
    double total;
    double run = block_excl_scan(acc, wt, total);
    for (uint64_t i = lo; i < hi; ++i) {
        const double t = ssum[i];
        ssum[i] = run;
        run += t;
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_seg_apply(const double *__restrict__ csum, uint64_t nch,
                                                                 const double *__restrict__ soff,
                                                                 double *__restrict__ g) {
    __shared__ double tile[kScanSeg];
    __shared__ double wt[kScanThreads / 32];
    const uint64_t lo = (uint64_t)blockIdx.x * kScanSeg;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {  // coalesced load, then each thread owns 8 consecutive chunks
        const uint64_t i = lo + (uint64_t)j * kScanThreads + threadIdx.x;
        tile[j * kScanThreads + threadIdx.x] = i < nch ? csum[i] : 0.0;
    }
    __syncthreads();
    double v[kScanPer], acc = 0.0;
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        v[j] = tile[threadIdx.x * kScanPer + j];
        acc += v[j];
    }
    double total;
    double run = soff[blockIdx.x] + block_excl_scan(acc, wt, total);
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        tile[threadIdx.x * kScanPer + j] = run;
        run += v[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        const uint64_t i = lo + (uint64_t)j * kScanThreads + threadIdx.x;
        if (i < nch) g[i] = tile[j * kScanThreads + threadIdx.x];
    }
}

static void scan_guess(const double *csum, uint64_t nch, double *seg_tmp, double *g, cudaStream_t st) {
    const uint64_t nseg = (nch + kScanSeg - 1) / kScanSeg;
    k_scan_seg_sums<<<(unsigned)nseg, kScanThreads, 0, st>>>(csum, nch, seg_tmp);
    k_scan_seg_top<<<1, 1024, 0, st>>>(seg_tmp, nseg);
    k_scan_seg_apply<<<(unsigned)nseg, kScanThreads, 0, st>>>(csum, nch, seg_tmp, g);
}

// binade helpers on the bit pattern of a non-negative double
__device__ __forceinline__ double binade_hi(double g) {
    const uint64_t bits = (uint64_t)__double_as_longlong(g);
    const uint64_t E = bits >> 52;
    if (E <= 1) return __longlong_as_double((long long)(2ull << 52));  // 2^-1021
    return __longlong_as_double((long long)((E + 1) << 52));
}
__device__ __forceinline__ double binade_lo(double g) {
    const uint64_t bits = (uint64_t)__double_as_longlong(g);
    const uint64_t E = bits >> 52;
    if (E <= 1) return 0.0;
    return __longlong_as_double((long long)(E << 52));
}

enum : int { kFlagOk = 1, kFlagExact0 = 2, kFlagWalked = 4, kFlagFineAbs = 8 };
// kFlagWalked: the chunk was re-summed sequentially (binade crossing);
// kFlagFineAbs: its fine starts (fine0) hold the exact running values
// themselves (recorded by that walk), not trajectory offsets
// Fine starts: M3 also keeps both trajectories (minus their guesses) at every
// 256th amplitude of a 4096-amplitude chunk, so a draw can start its exact
// walk at the last of the chunk's 16 sub-blocks whose running value is still
// <= u instead of at the chunk start (16x less walking per draw).
// Fine starts: the exact running value every 2^kFineLog amplitudes of a
// chunk, so a draw walks at most 64 amplitudes.  Stored coarse-first: the 16
// values at multiples of 256 in slots 0..15, then per 256-block the three at
// +64 / +128 / +192 (slots 16 + 3 q + r - 1): a draw reads the 16 coarse
// values, then 3 fine ones.  Slot-major in memory (value (chunk, slot) at
// slot * nch + chunk), so M3's lanes — 32 consecutive chunks — write each
// slot as one coalesced 256-B row.
constexpr int kFineLog = 6, kFinePer = 1 << (kChunkLog - kFineLog);
constexpr int kCoarseStep = 4, kCoarse = kFinePer / kCoarseStep;  // 16 coarse values (every 256)
__host__ __device__ __forceinline__ int fine_slot(int i) {  // i: position / 64
    return (i & (kCoarseStep - 1)) == 0 ? i / kCoarseStep
                                        : kCoarse + (kCoarseStep - 1) * (i / kCoarseStep) + (i & (kCoarseStep - 1)) - 1;
}

// ---- M3: guessed trajectories -------------------------------------------------
// One warp owns 32 consecutive chunks; every 32-element step the warp loads a
// 32x32 tile (each row = 32 consecutive amplitudes of one chunk, a coalesced
// 256-B read), converts to probabilities in shared memory, and lane L walks
// row L sequentially with both chains.
constexpr int kTrajWarps = 4;
template <class A>
__global__ void __launch_bounds__(kTrajWarps * 32)
    k_trajectories(const A *__restrict__ amps, uint64_t nch, int clog, double start,
                   const double *__restrict__ g, double *__restrict__ g0out,
                   double *__restrict__ d0, double *__restrict__ d1, double *__restrict__ hiout,
                   int *__restrict__ flags, double *__restrict__ fine0, double *__restrict__ fine1) {
    __shared__ double tile[kTrajWarps][32][33];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t first = ((uint64_t)blockIdx.x * kTrajWarps + w) * 32;
    if (first >= nch) return;
    const uint64_t my = first + lane;
    const uint64_t C = 1ull << clog;
    const bool active = my < nch;

    // g[my] = prefix of the chunk sums before this chunk; it is exactly 0
    // iff every earlier probability is 0, in which case the true running
    // value at the chunk start is exactly `start` (the CDF value carried in
    // from an earlier shard; 0 for a whole register).
    const double prefix = active ? g[my] : 0.0;
    const bool exact0 = (my == 0) || prefix == 0.0;
    const double gg = __dadd_rn(start, prefix);
    double g0 = gg, g1 = gg, hi = 0.0;
    if (!exact0) {
        g0 = __longlong_as_double(__double_as_longlong(gg) & ~1ll);
        g1 = __longlong_as_double(__double_as_longlong(g0) + 1ll);
        hi = binade_hi(g0);
    } else {
        g0 = start;
        g1 = start;
    }
    double t0 = g0, t1 = g1;
    // an exact0 chunk's running values ARE the CDF (its true start is
    // `start`): record them absolutely (kFlagFineAbs), position 0 included
    if (fine0 && active && exact0) fine0[my] = g0;  // slot 0
    const int rows = (int)((nch - first) < 32 ? (nch - first) : 32);
    for (uint64_t j0 = 0; j0 < C; j0 += 32) {
        const int width = (int)((C - j0) < 32 ? (C - j0) : 32);
        // eight rows' loads in flight before their squares are stored (a
        // load-then-store per row waited a full memory latency per row)
        for (int r0 = 0; r0 < rows; r0 += 8) {
            A a[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (r0 + q < rows && lane < width) a[q] = amps[((first + r0 + q) << clog) + j0 + lane];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (r0 + q < rows) tile[w][r0 + q][lane] = lane < width ? prob(a[q]) : 0.0;
        }
        __syncwarp();
        if (active) {
            for (int j = 0; j < width; ++j) {
                const double p = tile[w][lane][j];
                t0 = __dadd_rn(t0, p);
                t1 = __dadd_rn(t1, p);
            }
            const uint64_t pos = j0 + 32;  // elements summed so far
            if (fine0 && (pos & ((1u << kFineLog) - 1)) == 0 && pos < C) {
                if (exact0) {
                    fine0[(uint64_t)fine_slot((int)(pos >> kFineLog)) * nch + my] = t0;
                } else {
                    fine0[(uint64_t)fine_slot((int)(pos >> kFineLog)) * nch + my] = __dsub_rn(t0, g0);  // exact in the binade
                    fine1[(uint64_t)fine_slot((int)(pos >> kFineLog)) * nch + my] = __dsub_rn(t1, g1);
                }
            }
        }
        __syncwarp();
    }
    if (!active) return;
    g0out[my] = g0;
    if (exact0) {
        d0[my] = t0;  // exact end when the true start is 0
        d1[my] = t0;
        hiout[my] = 0.0;
        flags[my] = kFlagExact0 | (fine0 ? kFlagFineAbs : 0);
    } else {
        d0[my] = __dsub_rn(t0, g0);  // exact: same grid, same binade
        d1[my] = __dsub_rn(t1, g1);
        hiout[my] = hi;
        flags[my] = (t0 < hi && t1 < hi) ? kFlagOk : 0;
    }
}

// M3 for complex64 registers of >= 2^17 amplitudes (whole warps of 4096-
// amplitude chunks): the same trajectories, but each warp streams its 32
// chunks through a shared-memory ring (kTbStages deep) of 1-D bulk copies (one
// 512-B row per lane and stage, completion on an mbarrier), so a row block is
// in flight while the previous one is summed.  The register-staged form above
// kept only eight rows of loads in flight per warp and was memory-latency
// bound (ncu: long_scoreboard 50% of stalls, 2.1 ms at n = 30).
#ifndef QSB_TB_COLS
#define QSB_TB_COLS 64
#endif
#ifndef QSB_TB_STAGES
#define QSB_TB_STAGES 2
#endif
constexpr int kTbCols = QSB_TB_COLS;         // amplitudes per row and stage (512 B; 256-B rows x 4 stages: 1.37 -> 1.89 ms)
constexpr int kTbStages = QSB_TB_STAGES;     // ring depth (3 stages, 4 warps/SM: 1.67 ms vs 1.37 with 2 stages, 6 warps/SM)
constexpr int kTbPitch4 = kTbCols / 2 + 1;   // padded row pitch in float4 (odd: lanes on distinct bank quads)
constexpr int kTbStage4 = 32 * kTbPitch4;

__device__ __forceinline__ uint32_t tb_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tb_wait(uint64_t *bar, uint32_t parity) {
    for (uint32_t spins = 0;; ++spins) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0, 1, 0, P;\n}\n"
            : "=r"(ok)
            : "r"(tb_smem(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (spins > (1u << 22)) __trap();
    }
}
// stage the row block `col` (kTbCols amplitudes of each of the warp's 32 chunks)
__device__ __forceinline__ void tb_issue(const float2 *__restrict__ rows, uint64_t *bar, float4 *stage, int col,
                                         int lane) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the stage
    __syncwarp();
    if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tb_smem(bar)),
                     "r"(32u * kTbCols * 8u)
                     : "memory");
    __syncwarp();
    const float2 *src = rows + ((uint64_t)lane << kChunkLog) + (uint64_t)col * kTbCols;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            tb_smem(stage + lane * kTbPitch4)),
        "l"(src), "r"((uint32_t)(kTbCols * 8)), "r"(tb_smem(bar))
        : "memory");
}

__global__ void __launch_bounds__(32)
    k_trajectories_bulk(const float2 *__restrict__ amps, uint64_t nch, double start, const double *__restrict__ g,
                        double *__restrict__ g0out, double *__restrict__ d0, double *__restrict__ d1,
                        double *__restrict__ hiout, int *__restrict__ flags, double *__restrict__ fine0,
                        double *__restrict__ fine1) {
    extern __shared__ __align__(128) float4 tb_dyn[];  // kTbStages x kTbStage4 (dynamic: may exceed 48 KB)
    float4(*ring)[kTbStage4] = reinterpret_cast<float4(*)[kTbStage4]>(tb_dyn);
    __shared__ __align__(8) uint64_t bar[kTbStages];
    const int lane = threadIdx.x;
    const uint64_t first = (uint64_t)blockIdx.x * 32;
    const uint64_t my = first + lane;
    const float2 *rows = amps + (first << kChunkLog);
    if (lane == 0) {
        for (int st = 0; st < kTbStages; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tb_smem(&bar[st])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    for (int st = 0; st < kTbStages; ++st) tb_issue(rows, &bar[st], ring[st], st, lane);

    // prologue and epilogue as in k_trajectories
    const double prefix = g[my];
    const bool exact0 = (my == 0) || prefix == 0.0;
    const double gg = __dadd_rn(start, prefix);
    double g0 = start, g1 = start, hi = 0.0;
    if (!exact0) {
        g0 = __longlong_as_double(__double_as_longlong(gg) & ~1ll);
        g1 = __longlong_as_double(__double_as_longlong(g0) + 1ll);
        hi = binade_hi(g0);
    }
    double t0 = g0, t1 = g1;
    if (fine0 && exact0) fine0[my] = g0;  // slot 0
    constexpr int kCols = (1 << kChunkLog) / kTbCols;
    constexpr int kFineEvery = (1 << kFineLog) / kTbCols;
    for (int c = 0; c < kCols; ++c) {
        const int st = c % kTbStages;
        tb_wait(&bar[st], (uint32_t)(c / kTbStages) & 1u);
        const float4 *row = ring[st] + lane * kTbPitch4;
#pragma unroll 8
        for (int j = 0; j < kTbCols / 2; ++j) {
            const float4 q = row[j];
            const double p0 = prob(make_float2(q.x, q.y)), p1 = prob(make_float2(q.z, q.w));
            t0 = __dadd_rn(t0, p0);
            t1 = __dadd_rn(t1, p0);
            t0 = __dadd_rn(t0, p1);
            t1 = __dadd_rn(t1, p1);
        }
        if (c + kTbStages < kCols) tb_issue(rows, &bar[st], ring[st], c + kTbStages, lane);
        if (fine0 && (c + 1) % kFineEvery == 0 && c + 1 < kCols) {
            const int f = (c + 1) / kFineEvery;
            if (exact0) {
                fine0[(uint64_t)fine_slot(f) * nch + my] = t0;
            } else {
                fine0[(uint64_t)fine_slot(f) * nch + my] = __dsub_rn(t0, g0);  // exact while in the binade
                fine1[(uint64_t)fine_slot(f) * nch + my] = __dsub_rn(t1, g1);
            }
        }
    }
    g0out[my] = g0;
    if (exact0) {
        d0[my] = t0;
        d1[my] = t0;
        hiout[my] = 0.0;
        flags[my] = kFlagExact0 | (fine0 ? kFlagFineAbs : 0);
    } else {
        d0[my] = __dsub_rn(t0, g0);
        d1[my] = __dsub_rn(t1, g1);
        hiout[my] = hi;
        flags[my] = (t0 < hi && t1 < hi) ? kFlagOk : 0;
    }
}

// ---- M4: resolve true chunk starts ------------------------------------------
// Inside one binade a double's bit pattern is linear in its value (step u).
// A chunk whose trajectory check passes moves the running value s to
// s + d[parity(s)] exactly, i.e. its bit pattern by an integer inc[parity],
// and the parity of the result follows from that.  Such parity maps
// (inc0, inc1) compose associatively — (A then B)(p) = A_p + B[(p + A_p) & 1]
// — so a block of chunks whose guesses share one binade reduces to one map
// (M4a, a block scan that also keeps every chunk's exclusive prefix map);
// one warp walks the blocks (M4b: a single step per regular block — its start
// and end must lie in that binade — while a block holding a binade crossing,
// a failed trajectory or the exact-zero prefix is walked chunk by chunk with
// the exact sequential fallback); and every chunk start of a regular block is
// its block start plus the prefix map (M4c).  The values are the ones the
// chunk-by-chunk walk produces, bit for bit.
constexpr int kMapBlock = 256;

struct PMap {
    long long a0, a1;  // bit-pattern increment from an even / odd start
};
__device__ __forceinline__ PMap pcompose(PMap x, PMap y) {  // x, then y
    PMap r;
    r.a0 = x.a0 + ((x.a0 & 1) ? y.a1 : y.a0);
    r.a1 = x.a1 + (((1 + x.a1) & 1) ? y.a1 : y.a0);
    return r;
}

__global__ void __launch_bounds__(kMapBlock)
    k_block_maps(uint64_t nch, const double *__restrict__ g0, const double *__restrict__ d0,
                 const double *__restrict__ d1, const int *__restrict__ flags, long long *__restrict__ pmap,
                 long long *__restrict__ bmap) {
    __shared__ PMap wsum[kMapBlock / 32];
    __shared__ long long sE;
    const uint64_t k = blockIdx.x * (uint64_t)kMapBlock + threadIdx.x;
    const bool in = k < nch;
    long long E = -1;
    PMap m{0, 0};
    bool ok = true;
    if (in) {
        const int f = flags[k];
        const double g = g0[k];
        const long long gb = __double_as_longlong(g);
        E = (long long)((unsigned long long)gb >> 52);
        ok = (f & kFlagOk) && !(f & kFlagExact0) && E >= 2;
        if (ok) {  // t0 = g0 + d0 and t1 = g1 + d1 are exact (same grid, same binade)
            m.a0 = __double_as_longlong(__dadd_rn(g, d0[k])) - gb;
            m.a1 = __double_as_longlong(__dadd_rn(__longlong_as_double(gb + 1), d1[k])) - (gb + 1);
        }
    }
    // a block of exact0 chunks (every earlier probability zero: only its last
    // chunk can hold a nonzero sum): every chunk starts at the carried-in
    // start, the block ends at the last chunk's exact end (bmap kind 2)
    if (__syncthreads_and(!in || (flags[k] & kFlagExact0))) {
        if (in) {
            pmap[2 * k] = 0;
            pmap[2 * k + 1] = 0;
        }
        const uint64_t last = (blockIdx.x + 1) * (uint64_t)kMapBlock < nch ? (blockIdx.x + 1) * (uint64_t)kMapBlock - 1
                                                                        : nch - 1;
        if (k == last) {
            bmap[4 * blockIdx.x + 0] = __double_as_longlong(d0[k]);
            bmap[4 * blockIdx.x + 3] = 2;
        }
        return;
    }
    if (threadIdx.x == 0) sE = E;
    __syncthreads();
    ok = ok && (!in || E == sE);
    if (!__syncthreads_and(ok)) {
        if (threadIdx.x == 0) bmap[4 * blockIdx.x + 3] = 0;
        return;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    PMap inc = m;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        PMap x;
        x.a0 = __shfl_up_sync(0xffffffffu, inc.a0, o);
        x.a1 = __shfl_up_sync(0xffffffffu, inc.a1, o);
        if (lane >= o) inc = pcompose(x, inc);
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    PMap pre{0, 0};
    for (int i = 0; i < w; ++i) pre = pcompose(pre, wsum[i]);
    PMap ex;
    ex.a0 = __shfl_up_sync(0xffffffffu, inc.a0, 1);
    ex.a1 = __shfl_up_sync(0xffffffffu, inc.a1, 1);
    if (lane == 0) ex = PMap{0, 0};
    ex = pcompose(pre, ex);
    if (in) {
        pmap[2 * k] = ex.a0;
        pmap[2 * k + 1] = ex.a1;
    }
    if (threadIdx.x == kMapBlock - 1) {
        const PMap tot = pcompose(pre, inc);
        bmap[4 * blockIdx.x + 0] = tot.a0;
        bmap[4 * blockIdx.x + 1] = tot.a1;
        bmap[4 * blockIdx.x + 2] = sE;
        bmap[4 * blockIdx.x + 3] = 1;
    }
}

// One warp re-sums a chunk exactly (a binade crossing): the lanes load and
// square its amplitudes into shared memory (coalesced, in parallel — each
// |a|^2 is one rounding either way), lane 0 adds them in order (the
// sequential cumsum) and keeps the exact running value every 2^kFineLog
// amplitudes as the chunk's fine starts, so draws landing in it walk at most
// 2^kFineLog amplitudes.  Returns the end value in every lane.
template <class A>
__device__ double warp_walk_chunk(const A *__restrict__ amps, uint64_t chunk, int clog, double s, double *sp,
                                  double *fine_abs, uint64_t fstride, uint64_t *bar, uint32_t &phase) {
    const int lane = threadIdx.x & 31;
    const int C = 1 << clog;
    const A *p = amps + ((uint64_t)chunk << clog);
    if (sizeof(A) == sizeof(double) && clog == kChunkLog) {
        // one 32-KB bulk copy of the chunk into sp (a complex64 amplitude and
        // its fp64 probability are both 8 B), then each lane squares its own
        // slots in place: one memory latency instead of C/32 dependent loads
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tb_smem(bar)),
                         "r"((uint32_t)(C * 8))
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    tb_smem(sp)),
                "l"(p), "r"((uint32_t)(C * 8)), "r"(tb_smem(bar))
                : "memory");
        }
        tb_wait(bar, phase);
        phase ^= 1u;
        const A *raw = reinterpret_cast<const A *>(sp);
#pragma unroll 8
        for (int j = lane; j < (1 << kChunkLog); j += 32) {
            const A a = raw[j];
            sp[j] = prob(a);
        }
    } else {
        for (int j = lane; j < C; j += 32) sp[j] = prob(p[j]);
    }
    __syncwarp();
    // sub-blocks of 256 amplitudes (one per lane, 16 per chunk); fine starts
    // every 64 (kFineLog): at each sub-block start and at +64/+128/+192
    constexpr int S = 1 << (kFineLog + 2);
    constexpr int kSub = S >> kFineLog;  // fine starts per sub-block
    const int nsb = C / S;
    double res = s;
    if (nsb < 2) {  // short chunk: plain sequential sum (fine starts only for full chunks)
        if (lane == 0)
            for (int j = 0; j < C; ++j) res = __dadd_rn(res, sp[j]);
        __syncwarp();
        return __shfl_sync(0xffffffffu, res, 0);
    }
    // The M3/M4 argument one level down: sub-block L's sequential sum from an
    // even / odd start g0, g1 = g0 + ulp near its guessed start (the chunk
    // start plus a plain sum of the earlier sub-blocks) is, while both
    // trajectories stay in g0's binade, the true sum's offset for a true
    // start of that parity in that binade (so are its partial sums at +64,
    // +128, +192: the fine starts inside the sub-block); lane 0 then chains
    // the sub-blocks exactly and re-sums in order only those that leave their
    // binade.
    const double *q = sp + (lane < nsb ? lane : 0) * S;
    double bs = 0.0;  // this sub-block's plain sum (for the guess only)
    if (lane < nsb)
        for (int j = 0; j < S; ++j) bs += q[j];
    double pre = bs;  // inclusive warp scan -> exclusive prefix (guess)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double x = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += x;
    }
    pre -= bs;
    double g0 = 0.0, d0 = 0.0, d1 = 0.0, hi = 0.0;
    double m0[kSub - 1], m1[kSub - 1];  // partial offsets at +64, +128, +192
    int ok = 0;
    if (lane < nsb) {
        const double gg = __dadd_rn(s, pre);
        g0 = __longlong_as_double(__double_as_longlong(gg) & ~1ll);
        const double g1 = __longlong_as_double(__double_as_longlong(g0) + 1ll);
        hi = binade_hi(g0);
        double t0 = g0, t1 = g1;
#pragma unroll
        for (int r = 0; r < kSub; ++r) {
            for (int j = r << kFineLog; j < (r + 1) << kFineLog; ++j) {
                t0 = __dadd_rn(t0, q[j]);
                t1 = __dadd_rn(t1, q[j]);
            }
            if (r + 1 < kSub) {
                m0[r] = __dsub_rn(t0, g0);
                m1[r] = __dsub_rn(t1, g1);
            }
        }
        d0 = __dsub_rn(t0, g0);
        d1 = __dsub_rn(t1, g1);
        ok = t0 < hi && t1 < hi;
    }
    for (int L = 0; L < nsb; ++L) {
        const double lg0 = __shfl_sync(0xffffffffu, g0, L), ld0 = __shfl_sync(0xffffffffu, d0, L);
        const double ld1 = __shfl_sync(0xffffffffu, d1, L), lhi = __shfl_sync(0xffffffffu, hi, L);
        const int lok = __shfl_sync(0xffffffffu, ok, L);
        double lm0[kSub - 1], lm1[kSub - 1];
#pragma unroll
        for (int r = 0; r < kSub - 1; ++r) {
            lm0[r] = __shfl_sync(0xffffffffu, m0[r], L);
            lm1[r] = __shfl_sync(0xffffffffu, m1[r], L);
        }
        if (lane == 0) {
            if (fine_abs) fine_abs[(uint64_t)fine_slot(L * kSub) * fstride] = res;
            const bool odd = (__double_as_longlong(res) & 1ll) != 0;
            const double en = __dadd_rn(res, odd ? ld1 : ld0);
            if (lok && res >= binade_lo(lg0) && res < lhi && en < lhi) {
                // the whole sub-block stays in the binade: its inner fine
                // starts are the start plus the trajectory's partial offsets
                if (fine_abs) {
#pragma unroll
                    for (int r = 0; r < kSub - 1; ++r)
                        fine_abs[(uint64_t)fine_slot(L * kSub + r + 1) * fstride] = __dadd_rn(res, odd ? lm1[r] : lm0[r]);
                }
                res = en;
            } else {  // the sub-block leaves its binade (or the guess missed): sum it in order
                const double *r = sp + L * S;
                for (int j = 0; j < S; j += 8) {
                    double pr[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) pr[u] = r[j + u];
#pragma unroll
                    for (int u = 0; u < 8; ++u) res = __dadd_rn(res, pr[u]);
                    const int done = j + 8;
                    if (fine_abs && (done & ((1 << kFineLog) - 1)) == 0 && done < S)
                        fine_abs[(uint64_t)fine_slot(L * kSub + (done >> kFineLog)) * fstride] = res;
                }
            }
        }
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, res, 0);
}

template <class A>
__global__ void __launch_bounds__(32)
    k_block_walk(const A *__restrict__ amps, uint64_t nch, int clog, double s_start,
                 const double *__restrict__ g0, const double *__restrict__ d0, const double *__restrict__ d1,
                 const double *__restrict__ hi, int *__restrict__ flags,
                 const long long *__restrict__ bmap, uint64_t nblk, double *__restrict__ sblock,
                 double *__restrict__ start, double *__restrict__ total, unsigned long long *__restrict__ nslow,
                 double *__restrict__ fine0, double *__restrict__ fine1) {
    __shared__ double sd0[kMapBlock], sd1[kMapBlock], shi[kMapBlock], slo[kMapBlock], sg0[kMapBlock];
    __shared__ int sfl[kMapBlock];
    __shared__ __align__(16) double sprob[1 << kChunkLog];
    __shared__ __align__(8) uint64_t wbar;
    uint32_t wphase = 0;
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tb_smem(&wbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    double s = s_start;  // identical in every lane
    unsigned long long slow = 0;
    for (uint64_t b0 = 0; b0 < nblk; b0 += 32) {
        long long F0 = 0, F1 = 0, E = -1, reg = 0;
        if (b0 + lane < nblk) {
            const long long *q = bmap + 4 * (b0 + lane);
            reg = q[3];
            if (reg) {
                F0 = q[0];
                F1 = q[1];
                E = q[2];
            }
        }
        const int cnt = (int)((nblk - b0) < 32 ? (nblk - b0) : 32);
        for (int i = 0; i < cnt; ++i) {
            const long long f0 = __shfl_sync(0xffffffffu, F0, i), f1 = __shfl_sync(0xffffffffu, F1, i);
            const long long e = __shfl_sync(0xffffffffu, E, i), r = __shfl_sync(0xffffffffu, reg, i);
            const uint64_t b = b0 + i;
            const long long sb = __double_as_longlong(s);
            const long long eb = sb + ((sb & 1) ? f1 : f0);
            if (r == 2 && s == s_start) {  // exact0 block: its chunks start at s_start
                if (lane == 0) sblock[b] = s;
                s = __longlong_as_double(f0);
                continue;
            }
            if (r == 1 && (sb >> 52) == e && (eb >> 52) == e) {  // start and end inside the block's binade
                if (lane == 0) sblock[b] = s;
                s = __longlong_as_double(eb);
                continue;
            }
            // irregular block (a binade crossing, a failed trajectory or the
            // exact-zero prefix inside): stage its chunk data; each lane
            // composes the parity maps of its 8 consecutive chunks when they
            // are valid and share one binade (the M4a argument on a segment),
            // the warp steps through the 32 segments — one step per uniform
            // segment — and lane 0 walks only the other segments chunk by
            // chunk (re-summing, with the whole warp, a chunk that crosses)
            if (lane == 0) sblock[b] = -1.0;
            const uint64_t k0 = b * kMapBlock;
            const int m = (int)((nch - k0) < (uint64_t)kMapBlock ? (nch - k0) : kMapBlock);
            for (int j = lane; j < m; j += 32) {
                sd0[j] = d0[k0 + j];
                sd1[j] = d1[k0 + j];
                shi[j] = hi[k0 + j];
                sg0[j] = g0[k0 + j];
                slo[j] = binade_lo(sg0[j]);
                sfl[j] = flags[k0 + j];
            }
            __syncwarp();
            constexpr int kSeg = kMapBlock / 32;
            const int c0 = lane * kSeg, c1 = c0 + kSeg < m ? c0 + kSeg : m;
            PMap seg{0, 0};
            long long segE = -1;
            bool seg_ok = c0 < c1;
            for (int j = c0; j < c1 && seg_ok; ++j) {
                const long long gb = __double_as_longlong(sg0[j]);
                const long long E = (long long)((unsigned long long)gb >> 52);
                const int f = sfl[j];
                if (!(f & kFlagOk) || (f & kFlagExact0) || E < 2 || (j > c0 && E != segE)) {
                    seg_ok = false;
                    break;
                }
                segE = E;
                PMap mj;
                mj.a0 = __double_as_longlong(__dadd_rn(sg0[j], sd0[j])) - gb;
                mj.a1 = __double_as_longlong(__dadd_rn(__longlong_as_double(gb + 1), sd1[j])) - (gb + 1);
                seg = pcompose(seg, mj);
            }
            double seg_start = -1.0;  // this lane's segment start when taken in one step
            for (int L = 0; L * kSeg < m; ++L) {
                const int l0 = L * kSeg, l1 = l0 + kSeg < m ? l0 + kSeg : m;
                const long long a0 = __shfl_sync(0xffffffffu, seg.a0, L), a1 = __shfl_sync(0xffffffffu, seg.a1, L);
                const long long e = __shfl_sync(0xffffffffu, segE, L);
                const bool sok = __shfl_sync(0xffffffffu, (int)seg_ok, L) != 0;
                const long long sb = __double_as_longlong(s);
                const long long eb = sb + ((sb & 1) ? a1 : a0);
                if (sok && (sb >> 52) == e && (eb >> 52) == e) {  // start and end inside the segment's binade
                    if (lane == L) seg_start = s;
                    s = __longlong_as_double(eb);
                    continue;
                }
                // lane 0 runs through the segment's valid chunks alone; the
                // warp joins only for a chunk that must be re-summed
                for (int j = l0; j < l1;) {
                    int bad = l1;
                    if (lane == 0) {
                        // software-pipelined: chunk j+1's shared-memory values
                        // load while chunk j's add / compares (the only work
                        // that waits for s) run
                        double na0 = sd0[j], na1 = sd1[j], nh = shi[j], nl = slo[j];
                        int nf = sfl[j];
                        for (; j < l1; ++j) {
                            const double x0 = na0, x1 = na1, h = nh, l = nl;
                            const int f = nf;
                            if (j + 1 < l1) {
                                na0 = sd0[j + 1];
                                na1 = sd1[j + 1];
                                nh = shi[j + 1];
                                nl = slo[j + 1];
                                nf = sfl[j + 1];
                            }
                            start[k0 + j] = s;
                            double en;
                            bool valid;
                            if (f & kFlagExact0) {
                                valid = (s == s_start);
                                en = x0;
                            } else {
                                const bool odd = (__double_as_longlong(s) & 1ll) != 0;
                                en = __dadd_rn(s, odd ? x1 : x0);
                                valid = (f & kFlagOk) && s >= l && s < h && en < h;
                            }
                            if (!valid) {
                                bad = j;
                                break;
                            }
                            s = en;
                        }
                    }
                    bad = __shfl_sync(0xffffffffu, bad, 0);
                    s = __shfl_sync(0xffffffffu, s, 0);
                    if (bad >= l1) break;
                    const bool record = fine0 && clog == kChunkLog;
                    s = warp_walk_chunk(amps, k0 + bad, clog, s, sprob,
                                        record ? fine0 + (k0 + bad) : nullptr, nch, &wbar, wphase);
                    if (lane == 0) {
                        ++slow;
                        flags[k0 + bad] = sfl[bad] | kFlagWalked | (record ? kFlagFineAbs : 0);
                    }
                    __syncwarp();
                    j = bad + 1;
                }
                s = __shfl_sync(0xffffffffu, s, 0);
            }
            // the chunk starts of the segments taken in one step: the segment
            // start plus each chunk's map, in order (exact, same binade)
            if (seg_start >= 0.0) {
                long long cb = __double_as_longlong(seg_start);
                for (int j = c0; j < c1; ++j) {
                    start[k0 + j] = __longlong_as_double(cb);
                    const long long gb = __double_as_longlong(sg0[j]);
                    const long long inc = (cb & 1) ? __double_as_longlong(__dadd_rn(__longlong_as_double(gb + 1), sd1[j])) - (gb + 1)
                                                   : __double_as_longlong(__dadd_rn(sg0[j], sd0[j])) - gb;
                    cb += inc;
                }
            }
            __syncwarp();
            s = __shfl_sync(0xffffffffu, s, 0);
        }
    }
    if (lane == 0) {
        *total = s;
        *nslow = slow;
    }
}

__global__ void __launch_bounds__(kMapBlock)
    k_block_fill(uint64_t nch, const double *__restrict__ sblock, const long long *__restrict__ pmap,
                 double *__restrict__ start) {
    const double sb = sblock[blockIdx.x];
    if (sb < 0.0) return;  // walked chunk by chunk in M4b
    const uint64_t k = blockIdx.x * (uint64_t)kMapBlock + threadIdx.x;
    if (k >= nch) return;
    const long long bits = __double_as_longlong(sb);
    start[k] = __longlong_as_double(bits + ((bits & 1) ? pmap[2 * k + 1] : pmap[2 * k]));
}

// ---- M5: normalised CDF value at each chunk end --------------------------------
// `end` = this register's final running value; `gtotal` = the global last
// CDF value used to normalise (0: use `end`, i.e. a whole register).
__global__ void k_chunk_last(const double *__restrict__ start, uint64_t nch,
                             const double *__restrict__ end, double gtotal,
                             double *__restrict__ last) {
    const double t = gtotal > 0.0 ? gtotal : *end;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < nch;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const double e = (k + 1 < nch) ? start[k + 1] : *end;
        last[k] = __ddiv_rn(e, t);
    }
}

// ---- PCG64 (numpy's default bit generator, XSL-RR 128/64) -------------------
typedef unsigned __int128 u128;
__device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }
__device__ __forceinline__ uint64_t pcg_output(u128 st) {
    const uint64_t x = (uint64_t)(st >> 64) ^ (uint64_t)st;
    const unsigned rot = (unsigned)(st >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}
// state after `delta` LCG steps (Brown's jump-ahead)
__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
    const u128 mult = mk128(2549297995355413924ull, 4865540595714422341ull);
    u128 acc_mult = 1, acc_plus = 0, cur_mult = mult, cur_plus = inc;
    while (delta) {
        if (delta & 1ull) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

// Smallest non-negative double S with fl(S / t) > u, as the condition the
// reference's searchsorted applies to each normalised CDF value (measure.py:
// 80-83: cdf /= total, then the first value > u).  fl(s / t) is monotone in
// s (t > 0) and the bit patterns of non-negative doubles are ordered like
// their values, so S is found by galloping from fl(u t) and bisecting bit
// patterns — a few divisions per draw instead of one per amplitude walked;
// `fl(s / t) > u` is then exactly `s >= S`.  u < 1, so fl(t / t) = 1 > u
// bounds the search.
__device__ double cdf_cut(double u, double t) {
    const long long top = __double_as_longlong(t);
    auto pred = [&](long long b) { return __ddiv_rn(__longlong_as_double(b), t) > u; };
    const double g0 = __dmul_rn(u, t);
    long long g = g0 > 0.0 ? __double_as_longlong(g0) : 0ll;
    if (g > top) g = top;
    long long lo, hi;  // pred(hi) holds; pred(lo) fails (lo = -1: below every s)
    if (pred(g)) {
        hi = g;
        long long step = 1;
        lo = g - 1;
        while (lo >= 0 && pred(lo)) {
            hi = lo;
            step <<= 1;
            lo = hi - step;
        }
        if (lo < 0) lo = -1;
    } else {
        lo = g;
        long long step = 1;
        hi = g + 1;
        while (hi < top && !pred(hi)) {
            lo = hi;
            step <<= 1;
            hi = lo + step;
        }
        if (hi > top) hi = top;
    }
    while (hi - lo > 1) {
        const long long mid = lo + (hi - lo) / 2;
        if (pred(mid))
            hi = mid;
        else
            lo = mid;
    }
    return __longlong_as_double(hi);
}

// ---- M6: draws ---------------------------------------------------------------------
// Draw i resolves in this register iff fl(s_start / t) <= u (no earlier
// register holds a value above u) and u < last[nch-1] (or this is the last
// register); otherwise out[i] = -1.  Outcomes are offset by `base` and
// clamped to `gdim - 1` (measure.py:83).
template <class A>
__global__ void k_draws(const A *__restrict__ amps, uint64_t nch, int clog, uint64_t dim,
                        const double *__restrict__ start, const double *__restrict__ last,
                        const double *__restrict__ end, double gtotal, double s_start,
                        uint64_t base, uint64_t gdim, int is_last, qs_pcg64 rng, int64_t k,
                        int64_t *__restrict__ out, const int *__restrict__ flags,
                        const double *__restrict__ fine0, const double *__restrict__ fine1) {
    const double t = gtotal > 0.0 ? gtotal : *end;
    const double u_lo = __ddiv_rn(s_start, t);
    const u128 st0 = mk128(rng.state_hi, rng.state_lo);
    const u128 inc = mk128(rng.inc_hi, rng.inc_lo);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        const u128 st = pcg_advance(st0, inc, (uint64_t)i + 1ull);  // step, then output
        const double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
        if (u < u_lo || (!is_last && !(last[nch - 1] > u))) {
            out[i] = -1;
            continue;
        }
        // first chunk whose last normalised value exceeds u
        uint64_t lo = 0, hi = nch;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (last[mid] > u)
                hi = mid;
            else
                lo = mid + 1;
        }
        uint64_t idx = dim;  // searchsorted returns dim when every value <= u
        if (lo < nch) {
            const uint64_t C = 1ull << clog;
            const A *p = amps + (lo << clog);
            double s = start[lo];
            const double cut = cdf_cut(u, t);  // fl(s / t) > u  <=>  s >= cut
            // the same sequential sum, 8 probabilities loaded ahead of the
            // chain (the loads do not depend on s; a one-at-a-time loop
            // waits a memory latency per amplitude)
            uint64_t j = 0, hit = C;
            if (fine0 && clog == kChunkLog) {
                const int f = flags[lo];
                // the chunk's fine starts, coarse-first: the 16 values at
                // multiples of 256 (8 16-B loads issued together), then the
                // 3 inside the chosen 256-block; the values are
                // non-decreasing, so each level's pick is the count of
                // leading values below the cut
                const bool absf = (f & kFlagFineAbs) != 0;
                const bool traj = !absf && (f & kFlagOk) && !(f & (kFlagExact0 | kFlagWalked));
                if (absf || traj) {
                    const double *fb = (absf || !(__double_as_longlong(s) & 1ll) ? fine0 : fine1) + lo;
                    double fv[kCoarse];  // slot-major: value (lo, slot) at slot * nch + lo
#pragma unroll
                    for (int q = 0; q < kCoarse; ++q) fv[q] = fb[(uint64_t)q * nch];
                    // absolute (a walked / exact0 chunk: running values before
                    // amplitude 64 i) or start + trajectory offset (M3, M4)
                    double fs = absf ? fv[0] : s;
                    int qb = 0;
                    bool go = true;
#pragma unroll
                    for (int q = 1; q < kCoarse; ++q) {
                        const double v = absf ? fv[q] : __dadd_rn(s, fv[q]);
                        go = go && v < cut;
                        if (go) {
                            qb = q;
                            fs = v;
                        }
                    }
                    const double *ff = fb + (uint64_t)(kCoarse + (kCoarseStep - 1) * qb) * nch;
                    double fw[kCoarseStep - 1];
#pragma unroll
                    for (int r = 0; r < kCoarseStep - 1; ++r) fw[r] = ff[(uint64_t)r * nch];
                    int rb = 0;
                    go = true;
#pragma unroll
                    for (int r = 0; r < kCoarseStep - 1; ++r) {
                        const double v = absf ? fw[r] : __dadd_rn(s, fw[r]);
                        go = go && v < cut;
                        if (go) {
                            rb = r + 1;
                            fs = v;
                        }
                    }
                    j = (uint64_t)(qb * kCoarseStep + rb) << kFineLog;
                    s = fs;
                }
            }
            if constexpr (std::is_same<A, float2>::value) {
                // 16 probabilities per batch from 8 float4 loads (j is a
                // multiple of 256 here, the chunk 32-KB aligned)
                const float4 *p4 = reinterpret_cast<const float4 *>(p);
                for (; j + 16 <= C && hit == C; j += 16) {
                    float4 w[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) w[q] = p4[(j >> 1) + q];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const double pa = prob(make_float2(w[q].x, w[q].y)), pb = prob(make_float2(w[q].z, w[q].w));
                        if (hit == C) {
                            s = __dadd_rn(s, pa);
                            if (s >= cut) hit = j + 2 * q;
                        }
                        if (hit == C) {
                            s = __dadd_rn(s, pb);
                            if (s >= cut) hit = j + 2 * q + 1;
                        }
                    }
                }
            }
            for (; j + 8 <= C && hit == C; j += 8) {
                double pr[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pr[q] = prob(p[j + q]);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (hit == C) {
                        s = __dadd_rn(s, pr[q]);
                        if (s >= cut) hit = j + q;
                    }
                }
            }
            for (; j < C && hit == C; ++j) {
                s = __dadd_rn(s, prob(p[j]));
                if (s >= cut) hit = j;
            }
            idx = (lo << clog) + hit;
        }
        idx += base;
        out[i] = (int64_t)(idx < gdim - 1 ? idx : gdim - 1);
    }
}

}  // namespace

// probabilities into a (pageable) host array: |a|^2 pieces computed on the
// device, copied D2H into two pinned staging buffers, and drained to `host`
// by a team of host threads (each copies its slice of every piece) while the
// next piece is in flight.  The team lives for the whole call: spawning
// threads per piece cost more than the copies.
int run_probabilities(qs_state *s, uint64_t offset, uint64_t count, double *host) {
    NvtxRange nvtx_range("qsb probabilities");
    uint64_t piece = 1ull << 23;  // 64 MiB of fp64 per staging round
    if (const char *e = std::getenv("QSB_PROB_PIECE_LOG")) piece = 1ull << std::atoi(e);
    const uint64_t step = count < piece ? count : piece;
    int rc = ensure_scratch(s, 2 * step * sizeof(double));
    if (rc) return rc;
    {
        // pinned destination (qs_host_alloc / cudaHostRegister): |a|^2 pieces
        // go straight to it by DMA, no staging copy and no page faults
        cudaPointerAttributes attr;
        if (cudaPointerGetAttributes(&attr, host) == cudaSuccess && attr.type == cudaMemoryTypeHost) {
            double *dev[2] = {(double *)s->scratch, (double *)s->scratch + step};
            for (uint64_t done = 0, i = 0; done < count; done += step, ++i) {
                const uint64_t m = (count - done) < step ? (count - done) : step;
                unsigned grid = (unsigned)((m + 255) / 256);
                if (grid > (unsigned)s->num_sms * 16) grid = s->num_sms * 16;
                double *d = dev[i & 1];
                if (s->prec == QS_DOUBLE)
                    k_probs<<<grid, 256, 0, s->stream>>>(amps_d(s) + offset + done, d, m);
                else
                    k_probs<<<grid, 256, 0, s->stream>>>(s->amps + offset + done, d, m);
                QS_CUDA(cudaGetLastError());
                QS_CUDA(cudaMemcpyAsync(host + done, d, m * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
            }
            QS_CUDA(cudaStreamSynchronize(s->stream));
            return QS_OK;
        }
        cudaGetLastError();
    }
    rc = ensure_pinned(s, 2 * step * sizeof(double));
    if (rc) return rc;
    // A fresh numpy result page-faults 4-KiB pages during the host copy: ask
    // for transparent huge pages on its 2-MiB-aligned interior.
    if (count * sizeof(double) >= (64u << 20) && !(std::getenv("QSB_PROB_THP") && std::getenv("QSB_PROB_THP")[0] == '0')) {
        const uintptr_t a = ((uintptr_t)host + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
        const uintptr_t z = ((uintptr_t)(host + count)) & ~(uintptr_t)((2u << 20) - 1);
        if (z > a) madvise((void *)a, z - a, MADV_HUGEPAGE);
    }
    double *dev[2] = {(double *)s->scratch, (double *)s->scratch + step};
    double *pin[2] = {(double *)s->pinned, (double *)s->pinned + step};
    cudaEvent_t ev[2];
    QS_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    QS_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    const uint64_t npieces = (count + step - 1) / step;
    auto enqueue = [&](uint64_t i) -> int {
        const uint64_t done = i * step, m = (count - done) < step ? (count - done) : step;
        const int b = (int)(i & 1);
        unsigned grid = (unsigned)((m + 255) / 256);
        if (grid > (unsigned)s->num_sms * 16) grid = s->num_sms * 16;
        if (s->prec == QS_DOUBLE)
            k_probs<<<grid, 256, 0, s->stream>>>(amps_d(s) + offset + done, dev[b], m);
        else
            k_probs<<<grid, 256, 0, s->stream>>>(s->amps + offset + done, dev[b], m);
        QS_CUDA(cudaGetLastError());
        QS_CUDA(cudaMemcpyAsync(pin[b], dev[b], m * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        QS_CUDA(cudaEventRecord(ev[b], s->stream));
        return QS_OK;
    };
    // copy team: worker t copies slice t of piece `ready`, then counts itself done
    unsigned hw = std::thread::hardware_concurrency();
    int nt = count * sizeof(double) < (16u << 20) ? 0 : (int)(hw > 16 ? 16 : (hw < 2 ? 2 : hw));
    if (const char *e = std::getenv("QSB_PROB_THREADS")) nt = nt ? std::atoi(e) : 0;  // probes
    std::atomic<long long> ready{-1};
    std::atomic<int> finished{0};
    std::atomic<bool> stop{false};
    auto piece_len = [&](uint64_t i) { return (count - i * step) < step ? (count - i * step) : step; };
    std::vector<std::thread> team;
    for (int t = 0; t < nt; ++t)
        team.emplace_back([&, t] {
            long long seen = -1;
            for (;;) {
                long long r;
                while ((r = ready.load(std::memory_order_acquire)) == seen && !stop.load(std::memory_order_acquire))
                    std::this_thread::yield();
                if (r == seen) return;  // stop
                seen = r;
                const uint64_t len = piece_len((uint64_t)r) * sizeof(double);
                const uint64_t per = (len / nt + 63) & ~(uint64_t)63;
                const uint64_t lo = (uint64_t)t * per, hi = lo + per < len ? lo + per : len;
                if (lo < hi)
                    std::memcpy((char *)(host + (uint64_t)r * step) + lo, (const char *)pin[r & 1] + lo, hi - lo);
                finished.fetch_add(1, std::memory_order_acq_rel);
            }
        });
    int err = QS_OK;
    for (uint64_t i = 0; i < npieces && i < 2 && !err; ++i) err = enqueue(i);
    for (uint64_t i = 0; i < npieces && !err; ++i) {
        if (cudaEventSynchronize(ev[i & 1]) != cudaSuccess) {
            err = cuda_fail(cudaGetLastError(), "cudaEventSynchronize");
            break;
        }
        if (nt) {
            ready.store((long long)i, std::memory_order_release);
            while (finished.load(std::memory_order_acquire) < (int)((i + 1) * nt)) std::this_thread::yield();
        } else {
            std::memcpy(host + i * step, pin[i & 1], piece_len(i) * sizeof(double));
        }
        if (i + 2 < npieces) err = enqueue(i + 2);  // buffer i & 1 is free again
    }
    stop.store(true, std::memory_order_release);
    for (auto &x : team) x.join();
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    return err;
}

int run_norm(qs_state *s, double *out) {
    int rc = ensure_scratch(s, (kNormBlocks + 1) * sizeof(double));
    if (rc) return rc;
    double *partial = (double *)s->scratch;
    const uint64_t n = 1ull << s->num_qubits;
    if (s->prec == QS_DOUBLE)
        k_norm_partial<<<kNormBlocks, kNormThreads, 0, s->stream>>>(amps_d(s), n, partial);
    else
        k_norm_partial<<<kNormBlocks, kNormThreads, 0, s->stream>>>(s->amps, n, partial);
    k_norm_final<<<1, kNormThreads, 0, s->stream>>>(partial, kNormBlocks, partial + kNormBlocks);
    QS_CUDA(cudaGetLastError());
    rc = ensure_pinned(s, sizeof(double));
    if (rc) return rc;
    QS_CUDA(cudaMemcpyAsync(s->pinned, partial + kNormBlocks, sizeof(double),
                            cudaMemcpyDeviceToHost, s->stream));
    QS_CUDA(cudaStreamSynchronize(s->stream));
    *out = *(double *)s->pinned;
    return QS_OK;
}

// Scratch layout of the exact-CDF chain for one register.
struct CdfScratch {
    int clog;
    uint64_t nch;
    double *csum, *g0, *d0, *d1, *hi, *start, *last, *end, *sblock, *fine0, *fine1;
    unsigned long long *nslow;
    long long *pmap, *bmap;
    uint64_t nblk;
    int *flags;
    int64_t *dout;
};

static int cdf_scratch(qs_state *s, int64_t k, CdfScratch &c) {
    const int n = s->num_qubits;
    const uint64_t dim = 1ull << n;
    c.clog = n < kChunkLog ? n : kChunkLog;
    c.nch = dim >> c.clog;
    const uint64_t nch = c.nch;
    c.nblk = (nch + kMapBlock - 1) / kMapBlock;
    // csum, g0, d0, d1, hi, start, last (doubles) + end + nslow, prefix maps
    // (2 per chunk), block maps (4 per block), block starts + flags + outcomes
    // + fine starts (two trajectories x 16 per chunk) when there are draws
    const bool fine = k > 0 && c.clog == kChunkLog;
    const size_t nd = 7 * nch + 2 + 2 * nch + 5 * c.nblk + (fine ? 2 * kFinePer * nch + 8 : 0);
    const size_t bytes = nd * sizeof(double) + nch * sizeof(int) + 64 + (size_t)k * sizeof(int64_t);
    int rc = ensure_scratch(s, bytes);
    if (rc) return rc;
    double *b = (double *)s->scratch;
    c.csum = b;
    c.g0 = b + nch;
    c.d0 = b + 2 * nch;
    c.d1 = b + 3 * nch;
    c.hi = b + 4 * nch;
    c.start = b + 5 * nch;
    c.last = b + 6 * nch;
    c.end = b + 7 * nch;
    c.nslow = (unsigned long long *)(b + 7 * nch + 1);
    c.pmap = (long long *)(b + 7 * nch + 2);
    c.bmap = c.pmap + 2 * nch;
    c.sblock = (double *)(c.bmap + 4 * c.nblk);
    // fine values 64-B aligned
    c.fine0 = fine ? (double *)(((uintptr_t)(c.sblock + c.nblk) + 63) & ~(uintptr_t)63) : nullptr;
    c.fine1 = fine ? c.fine0 + kFinePer * nch : nullptr;
    c.flags = (int *)(b + nd);
    c.dout = (int64_t *)((char *)c.flags + ((nch * sizeof(int) + 63) & ~(size_t)63));
    return QS_OK;
}

// M1..M4: exact sequential running sum over the register, continuing from
// `s_start`; leaves chunk starts in c.start and the final value in *c.end.
static bool traj_regs() {
    static const bool on = [] {
        const char *e = std::getenv("QSB_TRAJ_REGS");
        return e && *e && *e != '0';
    }();
    return on;
}

template <class A>
static int cdf_chain_t(qs_state *s, const A *amps, const CdfScratch &c, double s_start, bool sums_ready) {
    // M1, unless the circuit's last fused pass already accumulated the chunk
    // sums (qs_sample_prepare + QS_FUSED_CHUNK_SUMS: they are guesses only)
    if (sums_ready) {
    } else if (sizeof(A) == sizeof(float2) && c.clog == kChunkLog)
        k_chunk_sums_f4<<<(unsigned)c.nch, 256, 0, s->stream>>>((const float4 *)amps, c.csum);
    else
        k_chunk_sums<<<(unsigned)c.nch, 256, 0, s->stream>>>(amps, c.clog, c.csum);
    scan_guess(c.csum, c.nch, c.d0, c.start, s->stream);  // guessed prefixes -> start[] (d0: segment sums)
    {
        const uint64_t warps = (c.nch + 31) / 32;
        const unsigned blocks = (unsigned)((warps + kTrajWarps - 1) / kTrajWarps);
        bool bulk = false;
        if constexpr (std::is_same<A, float2>::value)  // QSB_TRAJ_REGS=1: the register-staged form (probes)
            bulk = c.clog == kChunkLog && c.nch % 32 == 0 && !traj_regs();
        if constexpr (std::is_same<A, float2>::value) {
            if (bulk) {
                constexpr int kRingBytes = kTbStages * kTbStage4 * 16;
                if (int rc = ensure_smem_attr((const void *)k_trajectories_bulk, kRingBytes)) return rc;
                k_trajectories_bulk<<<(unsigned)(c.nch / 32), 32, kRingBytes, s->stream>>>(
                    amps, c.nch, s_start, c.start, c.g0, c.d0, c.d1, c.hi, c.flags, c.fine0, c.fine1);
            }
        }
        if (!bulk)
            k_trajectories<<<blocks, kTrajWarps * 32, 0, s->stream>>>(
                amps, c.nch, c.clog, s_start, c.start, c.g0, c.d0, c.d1, c.hi, c.flags, c.fine0, c.fine1);
    }
    k_block_maps<<<(unsigned)c.nblk, kMapBlock, 0, s->stream>>>(c.nch, c.g0, c.d0, c.d1, c.flags, c.pmap,
                                                                 c.bmap);
    k_block_walk<<<1, 32, 0, s->stream>>>(amps, c.nch, c.clog, s_start, c.g0, c.d0, c.d1, c.hi, c.flags,
                                          c.bmap, c.nblk, c.sblock, c.start, c.end, c.nslow, c.fine0, c.fine1);
    k_block_fill<<<(unsigned)c.nblk, kMapBlock, 0, s->stream>>>(c.nch, c.sblock, c.pmap, c.start);
    QS_CUDA(cudaGetLastError());
    return QS_OK;
}

static int cdf_chain(qs_state *s, const CdfScratch &c, double s_start, bool sums_ready = false) {
    return s->prec == QS_DOUBLE ? cdf_chain_t(s, (const double2 *)amps_d(s), c, s_start, false)
                                : cdf_chain_t(s, (const float2 *)s->amps, c, s_start, sums_ready);
}

// M5 + M6 and the copy-out shared by qs_sample / qs_sample_shard.
static int draw(qs_state *s, const CdfScratch &c, const qs_pcg64 *rng, int64_t k, double s_start,
                double gtotal, uint64_t base, uint64_t gdim, int is_last, int64_t *out,
                double *end_out) {
    {
        unsigned grid = (unsigned)((c.nch + 255) / 256);
        if (grid > 4096) grid = 4096;
        k_chunk_last<<<grid, 256, 0, s->stream>>>(c.start, c.nch, c.end, gtotal, c.last);
    }
    {
        unsigned grid = (unsigned)((k + 127) / 128);
        if (grid > (unsigned)s->num_sms * 16) grid = s->num_sms * 16;
        if (s->prec == QS_DOUBLE)
            k_draws<<<grid, 128, 0, s->stream>>>(amps_d(s), c.nch, c.clog, 1ull << s->num_qubits,
                                                 c.start, c.last, c.end, gtotal, s_start, base, gdim,
                                                 is_last, *rng, k, c.dout, c.flags, c.fine0, c.fine1);
        else
            k_draws<<<grid, 128, 0, s->stream>>>(s->amps, c.nch, c.clog, 1ull << s->num_qubits,
                                                 c.start, c.last, c.end, gtotal, s_start, base, gdim,
                                                 is_last, *rng, k, c.dout, c.flags, c.fine0, c.fine1);
    }
    QS_CUDA(cudaGetLastError());
    int rc = ensure_pinned(s, sizeof(double));
    if (rc) return rc;
    QS_CUDA(cudaMemcpyAsync(s->pinned, c.end, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    QS_CUDA(cudaMemcpyAsync(out, c.dout, (size_t)k * sizeof(int64_t), cudaMemcpyDeviceToHost,
                            s->stream));
    QS_CUDA(cudaStreamSynchronize(s->stream));
    *end_out = *(double *)s->pinned;
    return QS_OK;
}

// Scratch for k draws laid out and the chunk sums zeroed, so that the next
// fused pass can accumulate them (QS_FUSED_CHUNK_SUMS) and qs_sample_ex skip
// M1.  *csum: where that pass adds (nullptr when this register's sampler has
// no such chunks: complex128 or fewer than 2^12 amplitudes).
int run_sample_prepare(qs_state *s, int64_t k, double **csum) {
    *csum = nullptr;
    s->csum_ready = 0;
    if (s->prec == QS_DOUBLE || s->num_qubits < kChunkLog) return QS_OK;
    CdfScratch c;
    int rc = cdf_scratch(s, k, c);
    if (rc) return rc;
    // the pass's row sums (2^(n-6) doubles) go where M3 later writes the fine
    // starts (2 x 64 per chunk = 2^(n-5) doubles): free until then
    *csum = c.fine0;
    s->csum_dst = c.fine0;
    return QS_OK;
}

// M1 from the row sums a fused pass left (64 rows of 64 amplitudes per chunk)
__global__ void k_rows_to_chunks(const double *__restrict__ rows, uint64_t nch, double *__restrict__ csum) {
    const uint64_t c = blockIdx.x * (uint64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
    if (c >= nch) return;
    const int lane = threadIdx.x & 31;
    double v = rows[(c << 6) + lane] + rows[(c << 6) + 32 + lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) csum[c] = v;
}

int run_sample(qs_state *s, const qs_pcg64 *rng, int64_t k, int64_t *out, bool sums_ready) {
    NvtxRange nvtx_range("qsb sample");
    // the sums are guesses only (M2-M4 resolve the exact starts whatever they
    // are), so this is a shortcut, never a correctness condition
    bool ready = sums_ready && s->csum_ready && s->csum_dst != nullptr;
    s->csum_ready = 0;
    void *before = s->scratch;
    CdfScratch c;
    int rc = cdf_scratch(s, k, c);
    if (rc) return rc;
    if (s->scratch != before || c.fine0 != s->csum_dst) ready = false;  // reallocated: the row sums are gone
    if (ready)
        k_rows_to_chunks<<<(unsigned)((c.nch + 7) / 8), 256, 0, s->stream>>>(c.fine0, c.nch, c.csum);
    rc = cdf_chain(s, c, 0.0, ready);
    if (rc) return rc;
    double tot = 0.0;
    const uint64_t dim = 1ull << s->num_qubits;
    rc = draw(s, c, rng, k, 0.0, 0.0, 0, dim, 1, out, &tot);
    if (rc) return rc;
    if (!(tot > 0.0))  // measure.py:71-72
        return set_error(QS_ERR_DEGENERATE, "all outcome probabilities are zero");
    return QS_OK;
}

int run_cdf_extend(qs_state *s, double start, double *end) {
    CdfScratch c;
    int rc = cdf_scratch(s, 0, c);
    if (rc) return rc;
    rc = cdf_chain(s, c, start);
    if (rc) return rc;
    rc = ensure_pinned(s, sizeof(double));
    if (rc) return rc;
    QS_CUDA(cudaMemcpyAsync(s->pinned, c.end, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    QS_CUDA(cudaStreamSynchronize(s->stream));
    *end = *(double *)s->pinned;
    return QS_OK;
}

int run_sample_shard(qs_state *s, const qs_pcg64 *rng, int64_t k, double start, double total,
                     uint64_t base, uint64_t gdim, int is_last, int64_t *out) {
    if (!(total > 0.0)) return set_error(QS_ERR_DEGENERATE, "all outcome probabilities are zero");
    CdfScratch c;
    int rc = cdf_scratch(s, k, c);
    if (rc) return rc;
    rc = cdf_chain(s, c, start);
    if (rc) return rc;
    double end = 0.0;
    return draw(s, c, rng, k, start, total, base, gdim, is_last, out, &end);
}

}  // namespace qsb
