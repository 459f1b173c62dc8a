// inner_small.cu -- ttc_inner for tiny batches (B <= 4, e.g. C1's single pair): the kernel's time is then its
// latency, not its throughput.  The streaming kernels fetch core n when step n needs it, one DRAM round trip
// per step; here one CTA per pair issues ALL of both trains' loads at once (cp.async, both trains in shared
// memory, one round trip in total), then sweeps the N steps out of shared memory with the whole CTA:
//   W[r, i, q] = sum_p Z[r, p] Y_n[p, i, q],   Z'[s, q] = sum_{r, i} X_n[r, i, s] W[r, i, q]
// (the north-star recurrence Z_n = sum_i X_n[:,i,:]^T Z_{n-1} Y_n[:,i,:], Z_0 = [1]; R1), fp32 FMA in a fixed
// order (bitwise deterministic).
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void stage(float* dst, const float* src, int n) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
        for (int e = threadIdx.x; e < (n >> 2); e += blockDim.x) cp_async16(dst + 4 * e, src + 4 * e);
        for (int e = (n & ~3) + threadIdx.x; e < n; e += blockDim.x) cp_async4(dst + e, src + e);
    } else {
        for (int e = threadIdx.x; e < n; e += blockDim.x) cp_async4(dst + e, src + e);
    }
}

__global__ void __launch_bounds__(kThreads) inner_small_kernel(const InnerArgs a, SmallLayout L) {
    extern __shared__ __align__(16) float sm[];
    __shared__ int32_t rx[TTC_MAX_ORDER + 1], ry[TTC_MAX_ORDER + 1];
    __shared__ int64_t xo[TTC_MAX_ORDER + 1], yo[TTC_MAX_ORDER + 1];
    const int b = a.order ? a.order[blockIdx.x] : (int)blockIdx.x, N = a.N;
    for (int k = threadIdx.x; k <= N; k += blockDim.x) {
        rx[k] = a.x.ranks ? a.x.ranks[(int64_t)b * (N + 1) + k] : ((k == 0 || k == N) ? 1 : a.x.urank);
        ry[k] = a.y.ranks ? a.y.ranks[(int64_t)b * (N + 1) + k] : ((k == 0 || k == N) ? 1 : a.y.urank);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        xo[0] = yo[0] = 0;
        for (int k = 0; k < N; ++k) {
            xo[k + 1] = xo[k] + (int64_t)rx[k] * a.dims[k] * rx[k + 1];
            yo[k + 1] = yo[k] + (int64_t)ry[k] * a.dims[k] * ry[k + 1];
        }
    }
    __syncthreads();
    float* xs = sm;                       // X train, L.xmax floats
    float* ys = xs + L.xmax;              // Y train, L.ymax floats
    float* W = ys + L.ymax;               // L.wmax floats
    float* Z = W + L.wmax;                // two L.zmax buffers
    float* Zn = Z + L.zmax;
    stage(xs, a.x.cores + (a.x.offsets ? a.x.offsets[b] : (int64_t)b * a.x.train_elems), (int)xo[N]);
    stage(ys, a.y.cores + (a.y.offsets ? a.y.offsets[b] : (int64_t)b * a.y.train_elems), (int)yo[N]);
    if (threadIdx.x == 0) Z[0] = 1.f;     // Z_0 = [1]
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int n = 0; n < N; ++n) {
        const int R = rx[n], S = rx[n + 1], P = ry[n], Q = ry[n + 1], I = a.dims[n];
        const float* X = xs + xo[n];      // X_n[r, i, s] at r + R (i + I s)
        const float* Y = ys + yo[n];      // Y_n[p, i, q] at p + P (i + I q)
        const int RI = R * I;
        for (int e = threadIdx.x; e < RI * Q; e += blockDim.x) {   // W[r + R (i + I q)], e = r + R iq
            const int iq = e / R, r = e - iq * R;
            const float* y = Y + P * iq;
            float acc = 0.f;
            for (int p = 0; p < P; ++p) acc = fmaf(Z[r + R * p], y[p], acc);
            W[e] = acc;
        }
        __syncthreads();
        // Z'[s + S q] = sum_k X[k + RI s] W[k + RI q] (K = (r, i) contiguous in both): 8 lanes per output split
        // k and combine by shuffles (a short dependent chain instead of RI serial FMAs); fixed order
        for (int e0 = threadIdx.x >> 3; e0 < ((S * Q + 3) & ~3); e0 += blockDim.x >> 3) {
            const int sub = threadIdx.x & 7, e = min(e0, S * Q - 1);
            const int q = e / S, s = e - q * S;
            const float* x = X + RI * s;
            const float* w = W + RI * q;
            float acc = 0.f;
            for (int k = sub; k < RI; k += 8) acc = fmaf(x[k], w[k], acc);
            acc += __shfl_xor_sync(0xffffffffu, acc, 4);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            if (sub == 0 && e0 < S * Q) Zn[e] = acc;
        }
        __syncthreads();
        float* t = Z; Z = Zn; Zn = t;
    }
    if (threadIdx.x == 0) a.out[b] = Z[0];
}

}  // namespace

cudaError_t launch_inner_small(const InnerArgs& a, const SmallLayout& L, cudaStream_t s) {
    const size_t smem = sizeof(float) * (size_t)(L.xmax + L.ymax + L.wmax + 2 * L.zmax);
    cudaError_t e = cudaFuncSetAttribute(inner_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    inner_small_kernel<<<a.B, kThreads, smem, s>>>(a, L);
    return cudaGetLastError();
}

}  // namespace ttc
