// tma_bench.cu -- HBM -> shared-memory staging bandwidth of cp.async.bulk (TMA 1-D) by copy size and
// in-flight depth, and of 16-byte cp.async, with no compute: the ceiling for the inner kernel's staging.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each CTA streams `per_cta` bytes as `chunk`-byte bulk copies, `depth` stages of `stage_bytes`
__global__ void bulk_kernel(const char* src, size_t per_cta, int chunk, int stage_bytes, int depth, int issuers, float* sink) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[8];
    const char* base = src + blockIdx.x * per_cta;
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int nstages = (int)(per_cta / stage_bytes);
    const int per_stage = stage_bytes / chunk;
    auto issue = [&](int s) {
        const int slot = s % depth;
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[slot])), "r"(stage_bytes));
        __syncwarp();
        if (threadIdx.x < issuers)
            for (int c = threadIdx.x; c < per_stage; c += issuers)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(s32(sm + slot * stage_bytes + c * chunk)), "l"(base + (size_t)s * stage_bytes + (size_t)c * chunk),
                             "r"(chunk), "r"(s32(&bar[slot])) : "memory");
    };
    if (threadIdx.x < 32)
        for (int s = 0; s < depth && s < nstages; ++s) issue(s);
    float acc = 0.f;
    for (int s = 0; s < nstages; ++s) {
        const int slot = s % depth;
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                     ::"r"(s32(&bar[slot])), "r"((s / depth) & 1) : "memory");
        acc += reinterpret_cast<float*>(sm + slot * stage_bytes)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x < 32 && s + depth < nstages) issue(s + depth);
    }
    if (acc == 1234.f) sink[0] = acc;
}

__global__ void cpasync_kernel(const char* src, size_t per_cta, int stage_bytes, int depth, float* sink) {
    extern __shared__ __align__(128) char sm[];
    const char* base = src + blockIdx.x * per_cta;
    const int nstages = (int)(per_cta / stage_bytes);
    auto issue = [&](int s) {
        const int slot = s % depth;
        for (int c = threadIdx.x; c < stage_bytes / 16; c += blockDim.x)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(sm + slot * stage_bytes + c * 16)),
                         "l"(base + (size_t)s * stage_bytes + c * 16) : "memory");
        asm volatile("cp.async.commit_group;");
    };
    for (int s = 0; s < depth - 1 && s < nstages; ++s) issue(s);
    float acc = 0.f;
    for (int s = 0; s < nstages; ++s) {
        if (s + depth - 1 < nstages) issue(s + depth - 1); else asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group %0;" ::"n"(2));
        __syncthreads();
        acc += reinterpret_cast<float*>(sm + (s % depth) * stage_bytes)[threadIdx.x];
        __syncthreads();
    }
    if (acc == 1234.f) sink[0] = acc;
}

int main() {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t total = (size_t)2 << 30;
    char* src; CK(cudaMalloc(&src, total)); CK(cudaMemset(src, 1, total));
    float* sink; CK(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(cpasync_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    printf("[");
    bool first = true;
    struct Cfg { int chunk, stage, depth, ctas_per_sm, issuers; };
    Cfg cfgs[] = {{1024, 32768, 2, 2, 1}, {1024, 32768, 2, 2, 32}, {1024, 32768, 3, 2, 32}, {1024, 16384, 4, 2, 32},
                  {4096, 32768, 2, 2, 32}, {16384, 32768, 2, 2, 1}, {32768, 32768, 2, 2, 1}, {32768, 32768, 3, 2, 1},
                  {32768, 32768, 6, 1, 1}, {256, 32768, 2, 2, 32}, {1024, 8192, 4, 4, 32}, {16384, 16384, 4, 2, 1}};
    for (const Cfg& c : cfgs) {
        const int grid = sms * c.ctas_per_sm;
        const size_t per_cta = (total / grid) / c.stage * c.stage;
        const size_t smem = (size_t)c.stage * c.depth;
        float best = 1e9, ms;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0);
            bulk_kernel<<<grid, 128, smem>>>(src, per_cta, c.chunk, c.stage, c.depth, c.issuers, sink);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("%s{\"engine\": \"bulk\", \"chunk\": %d, \"stage\": %d, \"depth\": %d, \"ctas_per_sm\": %d, \"issuers\": %d, \"GBs\": %.1f}",
               first ? "" : ",\n", c.chunk, c.stage, c.depth, c.ctas_per_sm, c.issuers, per_cta * grid / best / 1e6);
        first = false;
    }
    int cfg2[][3] = {{32768, 3, 2}, {16384, 4, 2}, {32768, 4, 1}};
    for (auto& c : cfg2) {
        const int grid = sms * c[2];
        const size_t per_cta = (total / grid) / c[0] * c[0];
        float best = 1e9, ms;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0);
            cpasync_kernel<<<grid, 256, (size_t)c[0] * c[1]>>>(src, per_cta, c[0], c[1], sink);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf(",\n{\"engine\": \"cp.async16\", \"stage\": %d, \"depth\": %d, \"ctas_per_sm\": %d, \"GBs\": %.1f}", c[0], c[1], c[2],
               per_cta * grid / best / 1e6);
    }
    printf("]\n");
    return 0;
}
