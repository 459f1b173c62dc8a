// microbench.cu -- on-box throughput probes that decide the kernel design:
// FP32 FFMA, legacy mma.sync (tf32 m16n8k8, bf16 m16n8k16), and a streaming HBM read.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void mma_tf32_kernel(float* out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
    float d[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(d[k][0]), "+f"(d[k][1]), "+f"(d[k][2]), "+f"(d[k][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mma_bf16_kernel(float* out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
    float d[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(d[k][0]), "+f"(d[k][1]), "+f"(d[k][2]), "+f"(d[k][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// latency: one warp, one dependent chain of mma.sync
__global__ void mma_lat_kernel(float* out, int iters, long long* cycles) {
    uint32_t a0 = threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
    float d[4] = {};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    out[threadIdx.x] = d[0] + d[1] + d[2] + d[3];
}

__global__ void read_kernel(const float4* __restrict__ in, size_t n, float* out) {
    float acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldg(in + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
    float* out;
    CK(cudaMalloc(&out, 1 << 26));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // FFMA: 148*4 blocks x 256 threads x iters*16*8 FMAs
    {
        int iters = 4096, blocks = sms * 8, threads = 256;
        ffma_kernel<<<blocks, threads>>>(out, 16, 1.0001f, 0.5f);
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>(out, iters, 1.0001f, 0.5f);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * blocks * threads * (double)iters * 16 * 8;
        printf(", \"ffma_tflops\": %.2f", fl / ms / 1e9);
    }
    {
        int iters = 8192, blocks = sms * 8, threads = 256;
        mma_tf32_kernel<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        mma_tf32_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * 8 * 8 * (blocks * threads / 32.0) * iters * 4;
        printf(", \"mma_sync_tf32_tflops\": %.2f", fl / ms / 1e9);
    }
    {
        int iters = 8192, blocks = sms * 8, threads = 256;
        mma_bf16_kernel<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        mma_bf16_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * 8 * 16 * (blocks * threads / 32.0) * iters * 4;
        printf(", \"mma_sync_bf16_tflops\": %.2f", fl / ms / 1e9);
    }
    {
        long long* cyc;
        CK(cudaMalloc(&cyc, 8));
        mma_lat_kernel<<<1, 32>>>(out, 1000, cyc);
        long long c = 0;
        CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
        printf(", \"mma_sync_tf32_latency_cycles\": %.1f", c / 1000.0);
    }
    {
        size_t bytes = (size_t)4 << 30;
        float4* in;
        CK(cudaMalloc(&in, bytes));
        CK(cudaMemset(in, 0, bytes));
        read_kernel<<<sms * 8, 512>>>(in, bytes / 16, out);
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            read_kernel<<<sms * 8, 512>>>(in, bytes / 16, out);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf(", \"hbm_read_gbs\": %.1f", bytes / best / 1e6);
        cudaFree(in);
    }
    printf("}\n");
    return 0;
}
