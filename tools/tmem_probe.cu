// tmem_probe.cu -- tcgen05.ld throughput (TMEM -> registers) with 4 or 8 warps, 32x32b.x32 loads, and the
// tcgen05.st throughput; clock64 per warp.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NW>
__global__ void k(int iters, long long* out, float* sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + 256 * (warp >> 2);
    float acc = 0.f;
    uint32_t r[32];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t a = t + 32 * (i & 3);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                       "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                       "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                       "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(a));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
    }
    long long t1 = clock64();
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t a = t + 32 * (i & 3);
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(acc + j);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                     :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                       "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
                       "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
                       "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
                       "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    long long t3 = clock64();
    if ((threadIdx.x & 31) == 0) { out[2 * warp] = t1 - t0; out[2 * warp + 1] = t3 - t2; }
    sink[threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "r"(512));
}
template <int NW> void run(int iters) {
    long long* d; float* s; long long h[32];
    cudaMalloc(&d, 256); cudaMalloc(&s, 4096);
    k<NW><<<1, 32 * NW>>>(iters, d, s);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16 * NW, cudaMemcpyDeviceToHost);
    long long ld = 0, st = 0;
    for (int w = 0; w < NW; ++w) { ld = ld > h[2 * w] ? ld : h[2 * w]; st = st > h[2 * w + 1] ? st : h[2 * w + 1]; }
    const double bytes = (double)NW * iters * 4096;
    printf("%d warps x %d x (32x32b.x32 = 4 KB): ld %lld cyc -> %.1f B/cyc/SM (%.0f cyc per warp-load); st %lld cyc -> %.1f B/cyc/SM\n",
           NW, iters, ld, bytes / ld, (double)ld / iters, st, bytes / st);
    cudaFree(d); cudaFree(s);
}
int main() { run<4>(2048); run<8>(2048); run<4>(2048); return 0; }
