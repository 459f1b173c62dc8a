// inner_generic.cu -- general-shape tt_inner kernel (any ranks <= TTC_MAX_RANK, any mode sizes).
//
// Computes the sweep Z_n = sum_i X_n[:,i,:]^T Z_{n-1} Y_n[:,i,:] (ttc.h / PAPER.md:50-51, 318-320) for one
// pair per CTA.  Z lives in shared memory; cores are read straight from global memory (L1/L2 cached);
// the i range is processed in chunks so the intermediate W fits a fixed shared buffer.  This is the
// always-correct path for shapes the specialised kernels (inner_fast.cu) do not cover.
//
// Per step the association is chosen per pair: with F the core multiplied into Z first
// and G the other one,
//   W[g, i, f'] = sum_f Z[g, f] F[f, i, f']            then   Z'[g', f'] = sum_{g, i} G[g, i, g'] W[g, i, f'].
// W-first: F = Y, G = X (cost I R P (P' + ... ));  V-first: F = X, G = Y.  Z is always stored with the X
// bond fastest: Z[r + R p].
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void load_ranks(const TrainDev& t, int b, int N, int32_t* dst) {
    for (int n = threadIdx.x; n <= N; n += blockDim.x)
        dst[n] = t.ranks ? t.ranks[(int64_t)b * (N + 1) + n] : ((n == 0 || n == N) ? 1 : t.urank);
}

__device__ __forceinline__ int64_t train_base(const TrainDev& t, int b) {
    return t.offsets ? t.offsets[b] : (int64_t)b * t.train_elems;
}

__global__ void __launch_bounds__(kThreads) inner_generic_kernel(const InnerArgs a) {
    extern __shared__ float smem[];
    __shared__ int32_t rx[TTC_MAX_ORDER + 1], ry[TTC_MAX_ORDER + 1];
    float* Z = smem;
    float* Zn = Z + a.zmax;
    float* W = Zn + a.zmax;
    const int b = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
    const int N = a.N;
    load_ranks(a.x, b, N, rx);
    load_ranks(a.y, b, N, ry);
    if (threadIdx.x == 0) Z[0] = 1.0f;
    const float* xc = a.x.cores + train_base(a.x, b);
    const float* yc = a.y.cores + train_base(a.y, b);
    __syncthreads();

    for (int n = 0; n < N; ++n) {
        const int R = rx[n], S = rx[n + 1], P = ry[n], Q = ry[n + 1], I = a.dims[n];
        // per-i MACs of each association: W-first R*P*Q + R*S*Q, V-first R*P*S + P*S*Q
        const bool vfirst = (R * P * S + P * S * Q) < (R * P * Q + R * S * Q);
        const float* F = vfirst ? xc : yc;
        const float* G = vfirst ? yc : xc;
        const int Fa = vfirst ? R : P, Fb = vfirst ? S : Q;
        const int Ga = vfirst ? P : R, Gb = vfirst ? Q : S;
        const int zg = vfirst ? R : 1, zf = vfirst ? 1 : R;          // Z[g, f] = Z[g*zg + f*zf]
        for (int e = threadIdx.x; e < S * Q; e += blockDim.x) Zn[e] = 0.0f;
        const int ic_max = max(1, min(I, a.wbuf / (Ga * Fb)));
        for (int i0 = 0; i0 < I; i0 += ic_max) {
            const int ic = min(ic_max, I - i0);
            // W[g + Ga*(ii + ic*fb)] = sum_f Z[g, f] * F[f, i0+ii, fb]
            const int nw = Ga * ic * Fb;
            for (int e = threadIdx.x; e < nw; e += blockDim.x) {
                const int g = e % Ga;
                const int t = e / Ga;
                const int ii = t % ic, fb = t / ic;
                const float* f_col = F + (int64_t)Fa * ((i0 + ii) + (int64_t)I * fb);
                float acc = 0.0f;
                for (int f = 0; f < Fa; ++f) acc = fmaf(Z[g * zg + f * zf], __ldg(f_col + f), acc);
                W[e] = acc;
            }
            __syncthreads();
            // Zn[g', f'] += sum_{g, ii} G[g, i0+ii, g'] * W[g, ii, f']
            for (int e = threadIdx.x; e < Gb * Fb; e += blockDim.x) {
                const int gb = e % Gb, fb = e / Gb;
                float acc = 0.0f;
                for (int ii = 0; ii < ic; ++ii) {
                    const float* g_col = G + (int64_t)Ga * ((i0 + ii) + (int64_t)I * gb);
                    const float* w_col = W + Ga * (ii + ic * fb);
                    for (int g = 0; g < Ga; ++g) acc = fmaf(__ldg(g_col + g), w_col[g], acc);
                }
                const int idx = vfirst ? (fb + Fb * gb) : (gb + Gb * fb);   // X bond fastest
                Zn[idx] += acc;
            }
            __syncthreads();
        }
        float* t = Z; Z = Zn; Zn = t;
        xc += (int64_t)R * I * S;
        yc += (int64_t)P * I * Q;
    }
    if (threadIdx.x == 0) a.out[b] = Z[0];
}

}  // namespace

cudaError_t launch_inner_generic(const InnerArgs& a, cudaStream_t s) {
    const size_t smem = sizeof(float) * (2 * (size_t)a.zmax + (size_t)a.wbuf);
    cudaError_t e = cudaFuncSetAttribute(inner_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    inner_generic_kernel<<<a.B, kThreads, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ttc
