// Probe: does compute-sanitizer racecheck model mbarrier ordering?  Warp 1
// reads a shared buffer, then arrives on an mbarrier; warp 0 waits on it and
// then overwrites the buffer.  Correct (release/acquire through the
// mbarrier); a report here means racecheck does not see that ordering.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(float *out) {
    __shared__ float buf[256];
    __shared__ uint64_t bar;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = (float)i;
    __syncthreads();
    if (w == 1) {  // consumer: read, then arrive
        float s = 0.f;
        for (int i = lane; i < 256; i += 32) s += buf[i];
        out[lane] = s;
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
    } else if (w == 0) {  // producer: wait, then overwrite
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.u32 %0,1,0,P;\n}\n"
                         : "=r"(ok) : "r"(su(&bar)) : "memory");
        for (int i = lane; i < 256; i += 32) buf[i] = 0.f;
        __syncwarp();
        out[32 + lane] = buf[lane];
    }
}
int main() {
    float *o;
    cudaMalloc(&o, 64 * sizeof(float));
    k<<<1, 64>>>(o);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
