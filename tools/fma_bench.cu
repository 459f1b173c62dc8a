// fma_bench.cu -- FP32 issue-rate microbenchmarks on B200: 3-register FFMA vs FFMA2 (fma.rn.f32x2), and LDS.128
// wavefront cost for the broadcast patterns the warp-per-pair kernels use.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

// 16 independent accumulators, multiplicands in registers (varying per lane so nothing folds to constants)
__global__ void ffma3_kernel(float* out, int iters) {
    float a[16], x = threadIdx.x * 1e-3f, y = 1.0f - threadIdx.x * 1e-4f;
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = j * 0.1f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = fmaf(x, a[j], y);
            x = x * 1.0000001f;   // keeps x live and non-constant
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__global__ void ffma2_kernel(float* out, int iters) {
    unsigned long long a[16];
    float2 xv = make_float2(threadIdx.x * 1e-3f, threadIdx.x * 2e-3f), yv = make_float2(1.0f, 0.5f);
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = f2u(make_float2(j * 0.1f, j * 0.2f));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            unsigned long long x = f2u(xv), y = f2u(yv);
#pragma unroll
            for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(a[j]) : "l"(x), "l"(y));
            xv.x *= 1.0000001f;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) { float2 v = *reinterpret_cast<float2*>(&a[j]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// LDS.128: each lane reads 16 B at base + (lane / group) * stride floats (group lanes share an address)
__global__ void lds_kernel(float* out, int iters, int group, int stride) {
    __shared__ __align__(16) float sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int off = ((lane / group) * stride) & 8191 & ~3;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            float4 v = *reinterpret_cast<const float4*>(sm + ((off + 4 * r) & 8191));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        off ^= 64;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// LDS.64 / LDS.32 with fragment-like patterns: lane reads base + (lane / 4) * stride + 2 * (lane % 4) floats
template <int W>
__global__ void ldsw_kernel(float* out, int iters, int stride) {
    __shared__ __align__(16) float sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int off = ((lane >> 2) * stride + (W == 2 ? 2 * (lane & 3) : (lane & 3))) & 8191;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            if (W == 2) {
                float2 v = *reinterpret_cast<const float2*>(sm + ((off + 8 * r) & 8191));
                acc += v.x * v.y;
            } else {
                acc += sm[(off + 8 * r) & 8191];
            }
        }
        off ^= 64;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void mma_tput_kernel(float* out, int iters) {
    float d[8][4] = {};
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256, iters = 4096;
    float ms;
    printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
    ffma3_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); ffma3_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"ffma3_tflops\": %.2f", 2.0 * blocks * threads * (double)iters * 8 * 16 / ms / 1e9);
    ffma2_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); ffma2_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"ffma2_tflops\": %.2f", 4.0 * blocks * threads * (double)iters * 8 * 16 / ms / 1e9);
    // LDS.128 patterns: cycles per warp-instruction per SM = elapsed_cycles * sms / total warp instructions
    const int pats[][2] = {{1, 4}, {4, 36}, {8, 36}, {4, 4}, {8, 4}, {32, 0}, {2, 4}, {4, 68}, {1, 36}};
    for (auto& p : pats) {
        lds_kernel<<<blocks, threads>>>(out, 16, p[0], p[1]);
        cudaEventRecord(e0); lds_kernel<<<blocks, threads>>>(out, 1024, p[0], p[1]); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double winst = (double)blocks * (threads / 32) * 1024 * 16;
        printf(", \"lds128_g%d_s%d_clk_per_inst_per_sm\": %.3f", p[0], p[1], ms * 1e-3 * clk * 1e3 * sms / winst);
    }
    for (int stride : {8, 24, 40, 36}) {
        ldsw_kernel<2><<<blocks, threads>>>(out, 16, stride);
        cudaEventRecord(e0); ldsw_kernel<2><<<blocks, threads>>>(out, 1024, stride); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double winst = (double)blocks * (threads / 32) * 1024 * 16;
        printf(", \"lds64_frag_s%d_clk_per_inst_per_sm\": %.3f", stride, ms * 1e-3 * clk * 1e3 * sms / winst);
        ldsw_kernel<1><<<blocks, threads>>>(out, 16, stride);
        cudaEventRecord(e0); ldsw_kernel<1><<<blocks, threads>>>(out, 1024, stride); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"lds32_frag_s%d_clk_per_inst_per_sm\": %.3f", stride, ms * 1e-3 * clk * 1e3 * sms / winst);
    }
    for (int bpsm : {1, 2, 4, 8}) {
        mma_tput_kernel<<<sms * bpsm, 128>>>(out, 16);
        cudaEventRecord(e0); mma_tput_kernel<<<sms * bpsm, 128>>>(out, 2048); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = (double)sms * bpsm * 4 * 2048 * 8;
        printf(", \"mma_tf32_warps_per_sm_%d_tflops\": %.1f", bpsm * 4, mmas * 2 * 16 * 8 * 8 / ms / 1e9);
    }
    printf("}\n");
    return 0;
}
