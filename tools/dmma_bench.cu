// dmma_bench.cu -- FP64 tensor-core (mma.sync m8n8k4 f64) and f32->f64 conversion throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_kernel(double* out, int iters) {
    double d[8][2] = {};
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void cvt_kernel(const float* in, double* out, int iters) {
    float x[8];
    for (int j = 0; j < 8; ++j) x[j] = in[(threadIdx.x + j) & 255];
    double s = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { s += (double)x[j]; x[j] = __int_as_float(__float_as_int(x[j]) ^ 1); }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_kernel(double* out, int iters) {
    double a[8], x = threadIdx.x * 1e-3, y = 1.0;
    for (int j = 0; j < 8; ++j) a[j] = j;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(x, a[j], y);
    double s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; float* in;
    cudaMalloc(&out, 148 * 32 * 1024 * sizeof(double)); cudaMalloc(&in, 1024 * sizeof(float));
    cudaMemset(in, 0, 1024 * sizeof(float));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    printf("{");
    for (int wps : {4, 8, 16}) {
        dmma_kernel<<<sms * wps / 4, 128>>>(out, 16);
        cudaEventRecord(e0); dmma_kernel<<<sms * wps / 4, 128>>>(out, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("\"dmma_warps_per_sm_%d_tflops\": %.2f, ", wps, 2.0 * sms * wps * 4096.0 * 8 * 256 / ms / 1e9);
    }
    cvt_kernel<<<sms * 8, 256>>>(in, out, 16);
    cudaEventRecord(e0); cvt_kernel<<<sms * 8, 256>>>(in, out, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("\"f32_to_f64_plus_dadd_per_clk_per_sm\": %.2f, ", (double)sms * 8 * 256 * 4096 * 8 / (ms * 1e-3) / sms / 1.965e9);
    dfma_kernel<<<sms * 8, 256>>>(out, 16);
    cudaEventRecord(e0); dfma_kernel<<<sms * 8, 256>>>(out, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("\"dfma_tflops\": %.2f}\n", 2.0 * sms * 8 * 256 * 4096.0 * 8 / ms / 1e9);
    return 0;
}
