// reconstruct.cu -- dense tensors of a batch of trains (ttc.h: ttc_reconstruct; Eq. 9, and
// Alg. 2 steps 5-6: reconstruct, then permute).  One CTA per train:
//   Left  = X_1 ... X_k          (prod_{n<=k} I_n  x  R_k), built left to right in shared memory
//   Right = X_{k+1} ... X_N      (R_k  x  prod_{n>k} I_n), built right to left in shared memory
//   D[row, col] = sum_r Left[row, r] Right[r, col]    (a register-tiled FP32 product)
// with row = (i_1..i_k) and col = (i_{k+1}..i_N) little-endian; the output address of (row, col) is
// offr[row] + offc[col] (the permuted Eq. 2 strides), so the permutation of step 6 costs nothing extra.
// Each core of a build step is first copied (coalesced) into shared memory, re-laid so that the threads of a
// warp read it along odd strides (conflict-free), then the step's outputs are dot products over shared memory.
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

// D = Left Right in 64 x (16 TM) output tiles.  Thread (tx, ty) owns rows r0 + 4 tx + {0..3} (one 16-byte
// load of Left^T per r: Left is kept transposed, Lt[r][row] with row stride ldL) and columns c0 + ty + 16 b,
// b < TM (Right as Rt[col][r]: one 16-byte load per 4 r when Rk % 4 == 0).  Row pairs accumulate with FFMA2
// (fma.rn.f32x2, the column value broadcast), so a thread's result for one column is a float4 of 4 consecutive
// rows: one streaming 16-byte store when those rows are contiguous in the output (unpermuted leading modes).
__device__ __forceinline__ float2 up(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
template <int TM>
__device__ __forceinline__ void d_tiles(const float* Lt, int ldL, const float* Rt, int Rk, int rows, int cols,
                                        const int32_t* offr, const int32_t* offc, float* out) {
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const bool vec = (Rk & 3) == 0;
    for (int r0 = 0; r0 < rows; r0 += 64)
        for (int c0 = 0; c0 < cols; c0 += 16 * TM) {
            const int row = r0 + 4 * tx;
            const float* lt = Lt + row;
            const float* rp[TM];
#pragma unroll
            for (int b2 = 0; b2 < TM; ++b2) rp[b2] = Rt + (size_t)min(c0 + ty + 16 * b2, cols - 1) * Rk;
            unsigned long long acc[2][TM];
#pragma unroll
            for (int b2 = 0; b2 < TM; ++b2) acc[0][b2] = acc[1][b2] = 0ull;
            if (vec) {
                for (int r = 0; r < Rk; r += 4) {
                    float4 lq[4], rv[TM];
#pragma unroll
                    for (int q = 0; q < 4; ++q) lq[q] = *reinterpret_cast<const float4*>(lt + (size_t)(r + q) * ldL);
#pragma unroll
                    for (int b2 = 0; b2 < TM; ++b2) rv[b2] = *reinterpret_cast<const float4*>(rp[b2] + r);
#pragma unroll
                    for (int b2 = 0; b2 < TM; ++b2) {
                        const float w[4] = {rv[b2].x, rv[b2].y, rv[b2].z, rv[b2].w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            fma2(acc[0][b2], pk(lq[q].x, lq[q].y), pk(w[q], w[q]));
                            fma2(acc[1][b2], pk(lq[q].z, lq[q].w), pk(w[q], w[q]));
                        }
                    }
                }
            } else {
                for (int r = 0; r < Rk; ++r) {
                    const float4 l = *reinterpret_cast<const float4*>(lt + (size_t)r * ldL);
#pragma unroll
                    for (int b2 = 0; b2 < TM; ++b2) {
                        const float w = rp[b2][r];
                        fma2(acc[0][b2], pk(l.x, l.y), pk(w, w));
                        fma2(acc[1][b2], pk(l.z, l.w), pk(w, w));
                    }
                }
            }
            if (row >= rows) continue;
            const int o0 = offr[row];
            const bool v4 = row + 3 < rows && offr[row + 1] == o0 + 1 && offr[row + 2] == o0 + 2 && offr[row + 3] == o0 + 3;
#pragma unroll
            for (int b2 = 0; b2 < TM; ++b2) {
                const int c = c0 + ty + 16 * b2;
                if (c >= cols) continue;
                float* oc = out + offc[c];
                const float2 lo = up(acc[0][b2]), hi = up(acc[1][b2]);
                if (v4 && (reinterpret_cast<uintptr_t>(oc + o0) & 15u) == 0) {
                    __stcs(reinterpret_cast<float4*>(oc + o0), make_float4(lo.x, lo.y, hi.x, hi.y));
                } else {
                    const float v[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (row + u < rows) __stcs(oc + offr[row + u], v[u]);
                }
            }
        }
}

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Left[row][r] (row stride Rk), Right stored transposed Rt[col][r] (col stride Rk): both contiguous along r.
__global__ void __launch_bounds__(kThreads, 2) reconstruct_kernel(const ReconArgs a) {
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
    float* L = sm;                                  // Left^T: Rk x rows (row stride ldL); partials [row][s]
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
    float* XS = reinterpret_cast<float*>(offc + cols);   // the staged core of the current build step
    // ---- Left = X_1 .. X_k: P[row][s], row = (i_1..i_j) little-endian; the last product lands in L,
    // transposed (Lt[s][row], row stride ldL)
    const int ldL = a.ldl;
    {
        float* cur = (k % 2 == 1) ? L : T;          // k - 1 products follow: alternate so the last writes L
        int prow = a.dims[0];
        const float* X1 = G + co[0];                // X_1[0, i, s] at i + I_1 s
        if (k == 1) {
            for (int e = threadIdx.x; e < prow * rk[1]; e += blockDim.x) {
                const int s = e / prow, i = e - s * prow;
                cur[s * ldL + i] = __ldg(X1 + e);
            }
        } else {
            for (int e = threadIdx.x; e < prow * rk[1]; e += blockDim.x) {
                const int i = e / rk[1], s = e - i * rk[1];
                cur[e] = __ldg(X1 + i + a.dims[0] * s);
            }
        }
        for (int j = 1; j < k; ++j) {
            const float* Xj = G + co[j];            // X_j[r, i, s] at r + R (i + I s)
            const int R = rk[j], S = rk[j + 1], I = a.dims[j], Rp = R | 1;
            __syncthreads();                        // cur written, XS free
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            for (int s = 0; s < S; ++s)             // XS[(i S + s) Rp + r] = X_j[r, i, s]
                for (int i = warp; i < I; i += nw)
                    for (int r = lane; r < R; r += 32) cp_async4(XS + (i * S + s) * Rp + r, Xj + r + R * (i + I * s));
            cp_wait_all();
            __syncthreads();
            float* nxt = (cur == L) ? T : L;
            const bool last = j == k - 1;           // writes Left^T
            const int nrow = prow * I, ig = (I + 3) >> 2;
            // thread: (pr, i0..i0+3, s), s fastest across threads (XS rows Rp apart: odd stride, no conflicts)
            for (int e = threadIdx.x; e < prow * ig * S; e += blockDim.x) {
                const int s = e % S, t = e / S, gi = t % ig, pr = t / ig, i0 = 4 * gi;
                const float* p = cur + (size_t)pr * R;
                const float* x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] = XS + (min(i0 + u, I - 1) * S + s) * Rp;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 2
                for (int r = 0; r < R; ++r) {
                    const float pv = p[r];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = fmaf(pv, x[u][r], acc[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u < I) {
                        const int row = pr + prow * (i0 + u);
                        nxt[last ? s * ldL + row : row * S + s] = acc[u];
                    }
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
            const float* Xj = G + co[j];
            const int R = rk[j], S = rk[j + 1], I = a.dims[j], Sp = S | 1;
            __syncthreads();
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
            for (int s = warp; s < S; s += nw)      // XS[(r + R i) Sp + s] = X_j[r, i, s]
                for (int ri = lane; ri < R * I; ri += 32) cp_async4(XS + ri * Sp + s, Xj + ri + R * I * s);
            cp_wait_all();
            __syncthreads();
            float* nxt = (cur == Rt) ? T2 : Rt;
            const int ncol = I * pcol, ig = (I + 3) >> 2;
            // thread: (r, i0..i0+3, pc), r fastest across threads (XS rows Sp apart: odd stride, no conflicts)
            for (int e = threadIdx.x; e < pcol * ig * R; e += blockDim.x) {
                const int r = e % R, t = e / R, gi = t % ig, pc = t / ig, i0 = 4 * gi;
                const float* q = cur + (size_t)pc * S;
                const float* x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) x[u] = XS + (r + R * min(i0 + u, I - 1)) * Sp;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 2
                for (int s2 = 0; s2 < S; ++s2) {
                    const float qv = q[s2];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = fmaf(x[u][s2], qv, acc[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u < I) nxt[(i0 + u + I * pc) * R + r] = acc[u];
            }
            cur = nxt;
            pcol = ncol;
        }
    }
    __syncthreads();
    // ---- D = Left Right in 64 x (16 TM) output tiles (TM = 5 when 80-wide tiles waste less of the ragged edge)
    if (a.tm == 5) d_tiles<5>(L, ldL, Rt, Rk, rows, cols, offr, offc, out);
    else d_tiles<4>(L, ldL, Rt, Rk, rows, cols, offr, offc, out);
}

}  // namespace

cudaError_t launch_reconstruct(const ReconArgs& a, size_t smem_bytes, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(reconstruct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    reconstruct_kernel<<<a.B, kThreads, smem_bytes, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ttc
