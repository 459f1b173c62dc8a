// ttsvd_big.cu -- TT-SVD (Alg. 1) of tensors too large for the shared-memory kernels of
// ttsvd.cu (more than 16,384 elements, or an unfolding whose smaller side exceeds 64: Example 2's cases (ii)
// 20 x 20 x 20 x 5 and (iii) 20 x 20 x 20 x 5 x 4, whose middle unfoldings are 400 x 100 and
// 400 x 400).  One CTA per tensor over a caller-owned fp64 workspace (ttc_tt_svd_workspace).
//
// Each step n factors the unfolding Z (m x c, column-major: the Eq. 2 order of the remaining modes) by ONE-SIDED
// Jacobi (Hestenes) on the matrix A whose s = min(m, c) columns are orthogonalised:
//   m <= c:  A = Z^T (c x m).  A V has orthogonal columns  =>  V = U (left singular vectors of Z) and
//            (A V)^T = U^T Z = S V'^T, the next unfolding, directly.
//   m >  c:  A = Z   (m x c).  Z V = U S  =>  U = columns of Z V / sigma, next unfolding S V^T.
// Rotations of column pairs in the parallel round-robin order (one warp per pair, s/2 pairs per round), until a
// sweep rotates nothing (|a_p . a_q| <= 1e-15 sqrt(|a_p|^2 |a_q|^2)); singular values = norms of A V's columns.
// The delta-truncated rank, the 1e-7 singular-value floor (R25) and the sign convention (R24: the largest-magnitude
// entry of every left singular vector positive, the matching row of S V^T flipped with it) are Alg. 1's as the
// oracle reads them (oracle/ttsvd.py).  Alg. 2 step 1's permutation is folded into the first read.
//
// Every pass over A and V goes through L2 / HBM (a 400 x 400 fp64 A is 1.25 MB): this path is for the paper's
// Example 2 sizes, not a hot loop.
#include <cmath>

#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kBigThreads = 512;
constexpr int kBigWarps = kBigThreads / 32;
constexpr double kSigmaFloor = 1e-7;   // R25
constexpr int kMaxSweeps = 60;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// round-robin tournament: the player at position pos in round r (position 0 fixed, the others rotate)
__device__ __forceinline__ int rr_player(int pos, int r, int S) { return pos == 0 ? 0 : ((pos - 1 + r) % (S - 1)) + 1; }

__global__ void __launch_bounds__(kBigThreads) ttsvd_big_kernel(const TtsvdArgs a, double* ws, int64_t ws_per) {
    __shared__ double sig[kTtsvdBigMaxSide];
    __shared__ int ord[kTtsvdBigMaxSide];
    __shared__ double sgn[kTtsvdBigMaxSide];
    __shared__ double red[kBigWarps];
    __shared__ int rotated, rank_s;
    const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = a.N, elems = a.elems;
    double* Z = ws + (int64_t)b * ws_per;   // current unfolding, column-major
    double* A = Z + elems;                  // the matrix whose columns are orthogonalised
    double* V = A + elems;                  // accumulated rotations (s x s)
    const float* src = a.dense + (int64_t)b * elems;
    float* core = a.cores + (int64_t)b * a.train_cap;
    int32_t* rk = a.ranks + (int64_t)b * (N + 1);

    // ---- Z_0 = X^rho (Alg. 2 step 1's permutation folded into the gather), ||X||^2
    double nrm = 0.0;
    for (int e = tid; e < elems; e += kBigThreads) {
        int q = e;
        int64_t off = 0;
        for (int k = 0; k < N; ++k) {
            const int ik = q % a.dims[k];
            q /= a.dims[k];
            off += (int64_t)ik * a.in_stride[k];
        }
        const double v = src[off];
        Z[e] = v;
        nrm += v * v;
    }
    nrm = warp_sum(nrm);
    if (lane == 0) red[warp] = nrm;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kBigWarps; ++w) t += red[w];
        red[0] = t;
        rk[0] = 1;
        rk[N] = 1;
    }
    __syncthreads();
    const double delta2 = a.eps2 * red[0];   // (eps / sqrt(N - 1))^2 ||X||^2
    __syncthreads();

    int Rp = 1;                 // R_{n-1}
    int64_t cur = elems;        // elements of the current unfolding
    int64_t coff = 0;           // offset of core n in the train
    for (int n = 0; n + 1 < N; ++n) {
        const int m = Rp * a.dims[n];
        const int c = (int)(cur / m);
        const bool wide = m <= c;            // A = Z^T
        const int s = wide ? m : c, L = wide ? c : m;
        // A (L x s, column-major) and V = I (s x s)
        for (int64_t e = tid; e < (int64_t)L * s; e += kBigThreads) {
            const int row = (int)(e % L), col = (int)(e / L);
            A[e] = wide ? Z[col + (int64_t)m * row] : Z[e];
        }
        for (int64_t e = tid; e < (int64_t)s * s; e += kBigThreads) V[e] = (e % s) == (e / s) ? 1.0 : 0.0;
        __syncthreads();
        // ---- one-sided Jacobi sweeps
        const int S = s + (s & 1);
        for (int sweep = 0; sweep < kMaxSweeps && s > 1; ++sweep) {
            if (tid == 0) rotated = 0;
            __syncthreads();
            for (int r = 0; r < S - 1; ++r) {
                for (int k = warp; k < S / 2; k += kBigWarps) {
                    const int p = rr_player(k, r, S), q = rr_player(S - 1 - k, r, S);
                    if (p >= s || q >= s) continue;
                    double* ap = A + (int64_t)L * p;
                    double* aq = A + (int64_t)L * q;
                    double al = 0.0, be = 0.0, ga = 0.0;
                    for (int e = lane; e < L; e += 32) {
                        const double x = ap[e], y = aq[e];
                        al = fma(x, x, al);
                        be = fma(y, y, be);
                        ga = fma(x, y, ga);
                    }
                    al = warp_sum(al);
                    be = warp_sum(be);
                    ga = warp_sum(ga);
                    if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
                    const double zeta = (be - al) / (2.0 * ga);
                    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
                    for (int e = lane; e < L; e += 32) {
                        const double x = ap[e], y = aq[e];
                        ap[e] = cs * x - sn * y;
                        aq[e] = sn * x + cs * y;
                    }
                    double* vp = V + (int64_t)s * p;
                    double* vq = V + (int64_t)s * q;
                    for (int e = lane; e < s; e += 32) {
                        const double x = vp[e], y = vq[e];
                        vp[e] = cs * x - sn * y;
                        vq[e] = sn * x + cs * y;
                    }
                    if (lane == 0) rotated = 1;
                }
                __syncthreads();
            }
            if (!rotated) break;
            __syncthreads();
        }
        // ---- singular values (column norms), descending order (ties: lower index first)
        for (int j = warp; j < s; j += kBigWarps) {
            const double* aj = A + (int64_t)L * j;
            double v = 0.0;
            for (int e = lane; e < L; e += 32) v = fma(aj[e], aj[e], v);
            v = warp_sum(v);
            if (lane == 0) sig[j] = sqrt(v);
        }
        __syncthreads();
        for (int j = tid; j < s; j += kBigThreads) {
            int pos = 0;
            for (int k = 0; k < s; ++k) pos += (sig[k] > sig[j]) || (sig[k] == sig[j] && k < j);
            ord[pos] = j;
        }
        __syncthreads();
        // ---- delta-truncated rank (R23) with the singular-value floor (R25)
        if (tid == 0) {
            const double s0 = sig[ord[0]];
            int R = 1;
            if (s0 > 0.0) {
                int keep = 0;
                for (int k = 0; k < s; ++k) keep += sig[ord[k]] > kSigmaFloor * s0;
                // tail = sum_{j >= R} s_j^2 over every singular value (the below-floor ones included), shrinking R
                // while the discarded part stays within delta^2 (R23; oracle/ttsvd.py delta_rank)
                double tail = 0.0;
                for (int k = keep; k < s; ++k) tail += sig[ord[k]] * sig[ord[k]];
                R = keep;
                while (R > 1) {
                    const double sr = sig[ord[R - 1]];
                    if (tail + sr * sr > delta2) break;
                    tail += sr * sr;
                    --R;
                }
            }
            rank_s = R;
            rk[n + 1] = R;
        }
        __syncthreads();
        const int R = rank_s;
        // ---- core n = U (m x R) with the sign convention: column k is V[:, ord[k]] (wide) or A[:, ord[k]] / sigma
        for (int k = warp; k < R; k += kBigWarps) {
            const int j = ord[k];
            const double inv = wide ? 1.0 : (sig[j] > 0.0 ? 1.0 / sig[j] : 0.0);
            const double* u = wide ? V + (int64_t)s * j : A + (int64_t)L * j;
            double best = -1.0;
            int bi = 0;
            for (int e = lane; e < m; e += 32) {
                const double v = fabs(u[e]);
                if (v > best) { best = v; bi = e; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            const double sg = u[bi] < 0.0 ? -1.0 : 1.0;
            if (lane == 0) sgn[k] = sg;
            for (int e = lane; e < m; e += 32) core[coff + e + (int64_t)m * k] = (float)(sg * inv * u[e]);
        }
        __syncthreads();
        // ---- next unfolding Z' = S V^T (R x c, column-major), reshaped to (R I_{n+1}) x rest by the index order
        for (int64_t e = tid; e < (int64_t)R * c; e += kBigThreads) {
            const int k = (int)(e % R), col = (int)(e / R);
            const int j = ord[k];
            Z[e] = wide ? sgn[k] * A[col + (int64_t)L * j] : sgn[k] * sig[j] * V[col + (int64_t)s * j];
        }
        __syncthreads();
        coff += (int64_t)m * R;
        Rp = R;
        cur = (int64_t)R * c;
    }
    // ---- last core: G^(N) = Z (R_{N-1} x I_N x 1)
    for (int64_t e = tid; e < cur; e += kBigThreads) core[coff + e] = (float)Z[e];
}

}  // namespace

int64_t ttsvd_big_ws_per(int32_t elems, int32_t gmax) {
    return 2 * (int64_t)elems + (int64_t)gmax * gmax + 16;   // doubles per tensor: Z, A, V (+ padding)
}

cudaError_t launch_ttsvd_big(const TtsvdArgs& a, double* ws, cudaStream_t s) {
    ttsvd_big_kernel<<<a.B, kBigThreads, 0, s>>>(a, ws, ttsvd_big_ws_per(a.elems, a.gmax));
    return cudaGetLastError();
}

}  // namespace ttc
