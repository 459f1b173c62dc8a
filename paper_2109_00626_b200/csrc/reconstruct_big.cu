// reconstruct_big.cu -- dense tensors of trains too large for reconstruct.cu's one-CTA-per-train shared-memory
// kernel (ttc.h: ttc_reconstruct_ws; Eq. 9, and Alg. 2 steps 5-6).  Example
// 2's outputs: X x_1^1 Y of two 20 x 20 x 20 x 5 tensors is a 20 x 20 x 5 x 20 x 20 x 5 train
// with ranks up to 100 (4,000,000 entries), of two 20 x 20 x 20 x 5 x 4 tensors an order-8 train of 64,000,000.
//
// The same split as reconstruct.cu -- Left = X_1 ... X_k (prod_{n<=k} I_n x R_k), Right = X_{k+1} ... X_N
// (R_k x prod_{n>k} I_n), D = Left Right -- but the partial products live in a caller-owned workspace and every
// product is its own launch of one tiled FP32 GEMM, C (M x N) = A (M x K) B (K x N), all column-major, in the
// layouts the Eq. 2 core layout (element [r, i, s] at r + R_{n-1}(i + I_n s)) gives for free:
//   left step   L_{j+1} (pre_j x I_j R_{j+1}) = L_j (pre_j x R_j)       X_j (R_j x I_j R_{j+1})   [L_1 = X_1]
//   right step  Q_j (R_j I_j x suf_{j+1})     = X_j (R_j I_j x R_{j+1}) Q_{j+1} (R_{j+1} x suf_{j+1})
//                                                                                          [Q_{N-1} = X_N]
//   final       D[row, col] = L_k Q_k, stored at offr(row) + offc(col) (the permuted Eq. 2 strides: step 6's
//               permutation costs nothing extra), the output tile staged in shared memory so that the stores
//               run along whichever side holds the output's stride-1 mode.
// (0-based in the code: modes 0..N-1, pre_j = prod_{n<j} I_n, suf_j = prod_{n>=j} I_n, ranks R_0..R_N.)
// One grid per launch spans the largest product of the batch; CTAs past their own pair's tiles return.
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kT = 64;        // output tile kT x kT
constexpr int kQ = 16;        // K chunk
constexpr int kThreads = 256;

__device__ __forceinline__ int rank_of(const ReconBigArgs& a, int b, int n) {
    return (n == 0 || n == a.N) ? 1 : (a.t.ranks ? a.t.ranks[(int64_t)b * (a.N + 1) + n] : a.t.urank);
}

// offset of core n inside pair b's train
__device__ __forceinline__ int64_t core_off(const ReconBigArgs& a, int b, int n) {
    int64_t o = 0;
    int rp = 1;
    for (int m = 0; m < n; ++m) {
        const int r = rank_of(a, b, m + 1);
        o += (int64_t)rp * a.dims[m] * r;
        rp = r;
    }
    return o;
}

// kind 0: left step j (produces L_{j+1}); kind 1: right step j (produces Q_j); kind 2: the final product.
__global__ void __launch_bounds__(kThreads) recon_big_kernel(const ReconBigArgs a, int kind, int j) {
    __shared__ float As[kQ][kT + 4];
    __shared__ float Bs[kQ][kT + 4];
    __shared__ float Cs[kT][kT + 1];
    __shared__ int64_t offr[kT], offc[kT];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int N = a.N, k = a.k;
    for (int b = blockIdx.y; b < a.B; b += gridDim.y) {
        const float* cores = a.t.cores + (a.t.offsets ? a.t.offsets[b] : (int64_t)b * a.t.train_elems);
        float* lbuf = a.ws + (int64_t)b * (2 * a.ws_left + 2 * a.ws_right);   // [2][ws_left]
        float* rbuf = lbuf + 2 * a.ws_left;                                     // [2][ws_right]
        const float *A, *Bm;
        float* C = nullptr;
        int64_t M, Nc;
        int K;
        if (kind == 0) {
            A = j == 1 ? cores : lbuf + a.ws_left * ((j - 1) & 1);
            M = a.pre[j];
            K = rank_of(a, b, j);
            Bm = cores + core_off(a, b, j);
            Nc = (int64_t)a.dims[j] * rank_of(a, b, j + 1);
            C = lbuf + a.ws_left * (j & 1);
        } else if (kind == 1) {
            A = cores + core_off(a, b, j);
            M = (int64_t)rank_of(a, b, j) * a.dims[j];
            K = rank_of(a, b, j + 1);
            Bm = j + 1 == N - 1 ? cores + core_off(a, b, N - 1) : rbuf + a.ws_right * ((j + 1) & 1);
            Nc = a.suf[j + 1];
            C = rbuf + a.ws_right * (j & 1);
        } else {
            A = k == 1 ? cores : lbuf + a.ws_left * ((k - 1) & 1);
            M = a.pre[k];
            K = rank_of(a, b, k);
            Bm = k == N - 1 ? cores + core_off(a, b, N - 1) : rbuf + a.ws_right * (k & 1);
            Nc = a.suf[k];
        }
        const int64_t tm = (M + kT - 1) / kT, tn = (Nc + kT - 1) / kT;
        if ((int64_t)blockIdx.x >= tm * tn) continue;   // uniform per CTA: no barrier is skipped by part of it
        const int64_t m0 = (blockIdx.x % tm) * kT, n0 = (blockIdx.x / tm) * kT;
        float acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
        for (int q0 = 0; q0 < K; q0 += kQ) {
#pragma unroll
            for (int it = 0; it < 4; ++it) {
                const int e = tid + kThreads * it;
                const int am = e & 63, aq = e >> 6;          // A: 64 rows x 16 k, rows fastest
                As[aq][am] = (m0 + am < M && q0 + aq < K) ? A[(m0 + am) + M * (int64_t)(q0 + aq)] : 0.f;
                const int bq = e & 15, bn = e >> 4;          // B: 16 k x 64 columns, k fastest
                Bs[bq][bn] = (q0 + bq < K && n0 + bn < Nc) ? Bm[(q0 + bq) + (int64_t)K * (n0 + bn)] : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                float av[4], bv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) av[u] = As[q][tx + 16 * u];
#pragma unroll
                for (int v = 0; v < 4; ++v) bv[v] = Bs[q][ty + 16 * v];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
            }
            __syncthreads();
        }
        if (kind != 2) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int64_t m = m0 + tx + 16 * u, n = n0 + ty + 16 * v;
                    if (m < M && n < Nc) C[m + M * n] = acc[u][v];
                }
            continue;
        }
        // ---- final: output addresses of the tile's rows (modes 0..k-1) and columns (modes k..N-1)
        if (tid < kT) {
            int64_t q = m0 + tid, o = 0;
            for (int n = 0; n < k; ++n) {
                o += (q % a.dims[n]) * a.ostride[n];
                q /= a.dims[n];
            }
            offr[tid] = o;
        } else if (tid < 2 * kT) {
            int64_t q = n0 + tid - kT, o = 0;
            for (int n = k; n < N; ++n) {
                o += (q % a.dims[n]) * a.ostride[n];
                q /= a.dims[n];
            }
            offc[tid - kT] = o;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) Cs[tx + 16 * u][ty + 16 * v] = acc[u][v];
        __syncthreads();
        float* out = a.out + (a.out_offsets ? a.out_offsets[b] : (int64_t)b * a.pair_elems);
        for (int e = tid; e < kT * kT; e += kThreads) {
            const int r = a.row_fast ? (e & 63) : (e >> 6), c = a.row_fast ? (e >> 6) : (e & 63);
            if (m0 + r < M && n0 + c < Nc) __stcs(out + offr[r] + offc[c], Cs[r][c]);
        }
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_reconstruct_big(const ReconBigArgs& a, cudaStream_t s) {
    const unsigned gy = (unsigned)(a.B < 65535 ? a.B : 65535);
    auto go = [&](int kind, int j, int64_t tiles) -> cudaError_t {
        if (tiles <= 0) return cudaSuccess;
        if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
        recon_big_kernel<<<dim3((unsigned)tiles, gy), kThreads, 0, s>>>(a, kind, j);
        return cudaGetLastError();
    };
    cudaError_t e;
    for (int j = 1; j < a.k; ++j)
        if ((e = go(0, j, a.tiles_left[j])) != cudaSuccess) return e;
    for (int j = a.N - 2; j >= a.k; --j)
        if ((e = go(1, j, a.tiles_right[j])) != cudaSuccess) return e;
    return go(2, 0, a.tiles_final);
}

}  // namespace ttc
