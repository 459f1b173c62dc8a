// reconstruct.cu -- dense tensors of a batch of trains (ttc.h: ttc_reconstruct; Eq. 9, and
// Alg. 2 steps 5-6: reconstruct, then permute).  One CTA per train:
//   Left  = X_1 ... X_k          (prod_{n<=k} I_n  x  R_k), built left to right in shared memory
//   Right = X_{k+1} ... X_N      (R_k  x  prod_{n>k} I_n), built right to left in shared memory
//   D[row, col] = sum_r Left[row, r] Right[r, col]    (a register-tiled FP32 product)
// with row = (i_1..i_k) and col = (i_{k+1}..i_N) little-endian; the output address of (row, col) is
// offr[row] + offc[col] (the permuted Eq. 2 strides), so the permutation of step 6 costs nothing extra.
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 256;

// Packed FP32 pair (FFMA2, sm_100a): acc.{x,y} accumulate the even / odd terms of a dot product.
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void fma2(unsigned long long& acc, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ float hsum2(unsigned long long v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo + hi;
}

// Left[row][r] (row stride Rk), Right stored transposed Rt[col][r] (col stride Rk): both contiguous along r.
__global__ void __launch_bounds__(kThreads) reconstruct_kernel(const ReconArgs a) {
    extern __shared__ float sm[];
    __shared__ int32_t rk[TTC_MAX_ORDER + 1];
    __shared__ int64_t co[TTC_MAX_ORDER + 1];
    const int b = blockIdx.x, N = a.N, k = a.k;
    for (int n = threadIdx.x; n <= N; n += blockDim.x)
        rk[n] = (n == 0 || n == N) ? 1 : (a.t.ranks ? a.t.ranks[(int64_t)b * (N + 1) + n] : a.t.urank);
    __syncthreads();
    if (threadIdx.x == 0) {
        co[0] = 0;
        for (int n = 0; n < N; ++n) co[n + 1] = co[n] + (int64_t)rk[n] * a.dims[n] * rk[n + 1];
    }
    __syncthreads();
    const float* G = a.t.cores + (a.t.offsets ? a.t.offsets[b] : (int64_t)b * a.t.train_elems);
    float* out = a.out + (a.out_offsets ? a.out_offsets[b] : (int64_t)b * a.pair_elems);
    const int Rk = rk[k];
    const int rows = a.rows, cols = a.cols;
    float* L = sm;                                  // rows x Rk (row stride Rk)
    float* Rt = L + a.lbuf;                         // cols x Rk (col stride Rk)
    float* T = Rt + a.rbuf;                         // Left's build temporary
    float* T2 = T + a.t1;                           // Right's build temporary
    int32_t* offr = reinterpret_cast<int32_t*>(T2 + a.t2);
    int32_t* offc = offr + rows;
    // output offsets of the row / column multi-indices (permuted Eq. 2 strides)
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        int64_t o = 0;
        int q = r;
        for (int n = 0; n < k; ++n) { const int i = q % a.dims[n]; q /= a.dims[n]; o += (int64_t)i * a.ostride[n]; }
        offr[r] = (int32_t)o;
    }
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
        int64_t o = 0;
        int q = c;
        for (int n = k; n < N; ++n) { const int i = q % a.dims[n]; q /= a.dims[n]; o += (int64_t)i * a.ostride[n]; }
        offc[c] = (int32_t)o;
    }
    // ---- Left = X_1 .. X_k: P[row][s], row = (i_1..i_j) little-endian; the last product lands in L
    {
        float* cur = (k % 2 == 1) ? L : T;          // k - 1 products follow: alternate so the last writes L
        int prow = a.dims[0];
        const float* X1 = G + co[0];                // X_1[0, i, s] at i + I_1 s
        for (int e = threadIdx.x; e < prow * rk[1]; e += blockDim.x) {
            const int i = e / rk[1], s = e - i * rk[1];
            cur[e] = __ldg(X1 + i + a.dims[0] * s);
        }
        for (int j = 1; j < k; ++j) {
            __syncthreads();
            float* nxt = (cur == L) ? T : L;
            const float* Xj = G + co[j];            // X_j[r, i, s] at r + R (i + I s)
            const int R = rk[j], S = rk[j + 1], I = a.dims[j];
            const int nrow = prow * I;
            for (int e = threadIdx.x; e < nrow * S; e += blockDim.x) {
                const int row = e / S, s = e - row * S;
                const int i = row / prow, pr = row - i * prow;
                const float* x = Xj + R * (i + I * s);
                const float* p = cur + (size_t)pr * R;
                float acc = 0.f;
#pragma unroll 4
                for (int r = 0; r < R; ++r) acc = fmaf(p[r], __ldg(x + r), acc);
                nxt[e] = acc;
            }
            cur = nxt;
            prow = nrow;
        }
    }
    // ---- Right = X_{k+1} .. X_N: Q[col][r], col = (i_j..i_N) little-endian; the last product lands in Rt
    if (k == N) {                                   // N = 1: no right block, Right = [1]
        if (threadIdx.x == 0) Rt[0] = 1.f;
    } else {
        const int nR = N - k;                       // cores in the right block
        float* cur = (nR % 2 == 1) ? Rt : T2;
        int pcol = a.dims[N - 1];
        const float* XN = G + co[N - 1];            // X_N[r, i, 0] at r + R i
        const int RN = rk[N - 1];
        for (int e = threadIdx.x; e < pcol * RN; e += blockDim.x) cur[e] = __ldg(XN + e);   // [i][r] = X_N[r, i]
        for (int j = N - 2; j >= k; --j) {
            __syncthreads();
            float* nxt = (cur == Rt) ? T2 : Rt;
            const float* Xj = G + co[j];
            const int R = rk[j], S = rk[j + 1], I = a.dims[j];
            const int ncol = I * pcol;
            for (int e = threadIdx.x; e < ncol * R; e += blockDim.x) {
                const int col = e / R, r = e - col * R;
                const int pc = col / I, i = col - pc * I;
                const float* q = cur + (size_t)pc * S;
                const float* x = Xj + r + R * i;    // X_j[r, i, s] at x + R I s
                const int xst = R * I;
                float acc = 0.f;
#pragma unroll 4
                for (int s = 0; s < S; ++s, x += xst) acc = fmaf(__ldg(x), q[s], acc);
                nxt[e] = acc;
            }
            cur = nxt;
            pcol = ncol;
        }
    }
    __syncthreads();
    // ---- D = Left Right in 64 x 64 output tiles, 4 x 4 per thread (rows tx + 16 a, cols ty + 16 b).  With
    // Rk % 4 == 0 the operands are read 4 r at a time (LDS.128) and the products accumulate pairwise (even / odd
    // r) with FFMA2: 8 loads per 32 packed FMAs.
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const bool vec = (Rk & 3) == 0;
    for (int r0 = 0; r0 < rows; r0 += 64)
        for (int c0 = 0; c0 < cols; c0 += 64) {
            const float* lp[4];
            const float* rp[4];
#pragma unroll
            for (int a2 = 0; a2 < 4; ++a2) lp[a2] = L + (size_t)min(r0 + tx + 16 * a2, rows - 1) * Rk;
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) rp[b2] = Rt + (size_t)min(c0 + ty + 16 * b2, cols - 1) * Rk;
            float res[4][4];
            if (vec) {
                unsigned long long acc[4][4];
#pragma unroll
                for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
                    for (int b2 = 0; b2 < 4; ++b2) acc[a2][b2] = 0ull;
                for (int r = 0; r < Rk; r += 4) {
                    float4 lv[4], rv[4];
#pragma unroll
                    for (int a2 = 0; a2 < 4; ++a2) lv[a2] = *reinterpret_cast<const float4*>(lp[a2] + r);
#pragma unroll
                    for (int b2 = 0; b2 < 4; ++b2) rv[b2] = *reinterpret_cast<const float4*>(rp[b2] + r);
#pragma unroll
                    for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
                        for (int b2 = 0; b2 < 4; ++b2) {
                            fma2(acc[a2][b2], pk(lv[a2].x, lv[a2].y), pk(rv[b2].x, rv[b2].y));
                            fma2(acc[a2][b2], pk(lv[a2].z, lv[a2].w), pk(rv[b2].z, rv[b2].w));
                        }
                }
#pragma unroll
                for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
                    for (int b2 = 0; b2 < 4; ++b2) res[a2][b2] = hsum2(acc[a2][b2]);
            } else {
#pragma unroll
                for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
                    for (int b2 = 0; b2 < 4; ++b2) res[a2][b2] = 0.f;
                for (int r = 0; r < Rk; ++r) {
                    float lv[4], rv[4];
#pragma unroll
                    for (int a2 = 0; a2 < 4; ++a2) lv[a2] = lp[a2][r];
#pragma unroll
                    for (int b2 = 0; b2 < 4; ++b2) rv[b2] = rp[b2][r];
#pragma unroll
                    for (int a2 = 0; a2 < 4; ++a2)
#pragma unroll
                        for (int b2 = 0; b2 < 4; ++b2) res[a2][b2] = fmaf(lv[a2], rv[b2], res[a2][b2]);
                }
            }
            int orow[4];
#pragma unroll
            for (int a2 = 0; a2 < 4; ++a2) {
                const int r = r0 + tx + 16 * a2;
                orow[a2] = r < rows ? offr[r] : -1;
            }
#pragma unroll
            for (int b2 = 0; b2 < 4; ++b2) {
                const int c = c0 + ty + 16 * b2;
                if (c >= cols) continue;
                float* oc = out + offc[c];
#pragma unroll
                for (int a2 = 0; a2 < 4; ++a2)
                    if (orow[a2] >= 0) __stcs(oc + orow[a2], res[a2][b2]);
            }
        }
}

}  // namespace

cudaError_t launch_reconstruct(const ReconArgs& a, size_t smem_bytes, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(reconstruct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    reconstruct_kernel<<<a.B, kThreads, smem_bytes, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ttc
