// Probe: TMA tile ring throughput (data only, in place) for 2^12-amplitude
// tiles of a 30-qubit complex64 register, as a function of the row width
// (2^R contiguous amplitudes per row) and of where the tile's high qubits
// sit.  Answers whether a pass whose tile rows are 64 B (R = 3: nine new
// qubits per pass at K = 12) streams as fast as the 512-B-row passes (R = 6).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring64 ring64.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int kNB = 3, kBufBytes = 33792, kConsumers = 4;

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t par) {
    for (;;) {
        uint32_t ok;
        asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}\n"
                     : "=r"(ok) : "r"(su(bar)), "r"(par) : "memory");
        if (ok) return;
    }
}

struct P {
    CUtensorMap map;
    int nd;          // tensor dims
    int tdim[2];     // which dims carry the tile index (lo, hi); -1 none
    int tbits[2];    // bits of the tile index per such dim
    uint64_t ntiles;
    unsigned long long *ctr;
    int touch;
    unsigned box_bytes;
};

__device__ __forceinline__ void coords(const P &p, uint64_t t, int c[5]) {
    for (int i = 0; i < 5; ++i) c[i] = 0;
    if (p.tdim[0] >= 0) c[p.tdim[0]] = (int)(t & ((1ull << p.tbits[0]) - 1));
    if (p.tdim[1] >= 0) c[p.tdim[1]] = (int)(t >> p.tbits[0]);
}

__global__ void __launch_bounds__(32 * (kConsumers + 1)) k_ring(const __grid_constant__ P p) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full[kNB], done[kNB];
    __shared__ unsigned long long tid_[kNB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int b = 0; b < kNB; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[b])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&done[b])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kConsumers) {
        if (lane) return;
        uint64_t pend[kNB];
        int i = 0;
        for (;; ++i) {
            const int b = i % kNB;
            unsigned char *buf = sm + b * kBufBytes;
            const unsigned long long t = atomicAdd(p.ctr, 1ull);
            if (i >= kNB) {
                wait(&done[b], ((i - kNB) / kNB) & 1);
                int c[5];
                coords(p, pend[b], c);
                asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                             ::"l"(&p.map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su(buf)) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            if (t >= p.ntiles) {
                tid_[b] = ~0ull;
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&full[b])) : "memory");
                break;
            }
            pend[b] = t;
            tid_[b] = t;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[b])), "r"(p.box_bytes) : "memory");
            int c[5];
            coords(p, t, c);
            asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                         ::"r"(su(buf)), "l"(&p.map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su(&full[b])) : "memory");
        }
        for (int k = (i >= kNB ? i - kNB + 1 : 0); k < i; ++k) {
            const int b = k % kNB;
            wait(&done[b], (k / kNB) & 1);
            int c[5];
            coords(p, pend[b], c);
            asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                         ::"l"(&p.map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(su(sm + b * kBufBytes))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return;
    }
    for (int i = 0;; ++i) {
        const int b = i % kNB;
        wait(&full[b], (i / kNB) & 1);
        if (tid_[b] == ~0ull) break;
        if (p.touch) {
            float4 *v = (float4 *)(sm + b * kBufBytes);
            for (int j = threadIdx.x; j < 32768 / 16; j += 32 * kConsumers) {
                float4 x = v[j];
                x.x = -x.x;
                v[j] = x;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumers));
        if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&done[b])) : "memory");
    }
}

// tile = rows of 2^R amplitudes x the contiguous high-qubit run [h, h + K - R)
static int make(P &p, void *base, int n, int K, int R, int h, CUtensorMapSwizzle swz, int pad) {
    cuuint64_t dims[5];
    cuuint64_t str[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    int nd = 0;
    dims[nd] = 1ull << R; box[nd] = (1u << R) + (pad ? 2 : 0); ++nd;
    const int hb = K - R;
    int left = hb, at = h;
    while (left > 0) {
        const int w = left > 8 ? 8 : left;
        dims[nd] = 1ull << w; box[nd] = 1u << w; str[nd - 1] = 8ull << at; ++nd;
        left -= w; at += w;
    }
    p.tdim[0] = p.tdim[1] = -1;
    p.tbits[0] = p.tbits[1] = 0;
    int q = 0;
    if (h > R) { dims[nd] = 1ull << (h - R); box[nd] = 1; str[nd - 1] = 8ull << R; p.tdim[q] = nd; p.tbits[q] = h - R; ++q; ++nd; }
    if (h + hb < n) { dims[nd] = 1ull << (n - h - hb); box[nd] = 1; str[nd - 1] = 8ull << (h + hb); p.tdim[q] = nd; p.tbits[q] = n - h - hb; ++q; ++nd; }
    if (q == 1 && p.tdim[0] < 0) { p.tdim[0] = p.tdim[1]; p.tbits[0] = p.tbits[1]; p.tdim[1] = -1; }
    while (nd < 5) { dims[nd] = 1; box[nd] = 1; str[nd - 1] = str[nd - 2] * 2; ++nd; }
    p.nd = nd;
    p.box_bytes = (unsigned)(box[0] * 8u * (1u << (K - R)));
    p.ntiles = 1ull << (n - K);
    CUresult r = cuTensorMapEncodeTiled(&p.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d (R=%d h=%d)\n", (int)r, R, h); return 1; }
    return 0;
}

int main() {
    const int n = 30, K = 12;
    void *a;
    CK(cudaMalloc(&a, 8ull << n));
    CK(cudaMemset(a, 0, 8ull << n));
    unsigned long long *ctr;
    CK(cudaMalloc(&ctr, 8));
    CK(cudaMemset(ctr, 0, 8));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = kNB * kBufBytes;
    CK(cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    struct Cfg { int R, h, touch; CUtensorMapSwizzle swz; const char *name; int pad; };
    std::vector<Cfg> cfgs = {
        {6, 24, 0, CU_TENSOR_MAP_SWIZZLE_NONE, "512B rows, tile hi 24-29", 0},
        {6, 24, 0, CU_TENSOR_MAP_SWIZZLE_NONE, "512B rows padded 66, tile hi 24-29", 1},
        {6, 12, 0, CU_TENSOR_MAP_SWIZZLE_NONE, "512B rows, tile hi 12-17", 0},
        {6, 12, 0, CU_TENSOR_MAP_SWIZZLE_NONE, "512B rows padded 66, tile hi 12-17", 1},
        {6, 6, 0, CU_TENSOR_MAP_SWIZZLE_NONE, "512B rows, tile 0-11", 0},
        {6, 6, 0, CU_TENSOR_MAP_SWIZZLE_NONE, "512B rows padded 66, tile 0-11", 1},
        {6, 24, 1, CU_TENSOR_MAP_SWIZZLE_NONE, "512B rows padded 66 + touch, tile hi 24-29", 1},
        {6, 24, 0, CU_TENSOR_MAP_SWIZZLE_128B, "512B rows swizzle128?, tile hi 24-29", 0},
    };
    for (int occ = 2; occ >= 1; --occ) {
        for (auto &c : cfgs) {
            P p;
            if (make(p, a, n, K, c.R, c.h, c.swz, c.pad)) continue;
            p.ctr = ctr;
            p.touch = c.touch;
            const int grid = sms * occ;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int w = 0; w < 2; ++w) {
                CK(cudaMemset(ctr, 0, 8));
                k_ring<<<grid, 32 * (kConsumers + 1), smem>>>(p);
            }
            CK(cudaDeviceSynchronize());
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                CK(cudaMemset(ctr, 0, 8));
                cudaEventRecord(e0);
                k_ring<<<grid, 32 * (kConsumers + 1), smem>>>(p);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            CK(cudaGetLastError());
            printf("{\"cfg\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"TBps\": %.2f}\n", c.name, occ, best,
                   16.0 * (1ull << n) / best / 1e9);
        }
    }
    return 0;
}
