// ttsvd.cu -- batched TT-SVD (ttc.h: ttc_tt_svd; Alg. 1), optionally of the permuted tensor
// X^rho of Alg. 2 step 1.  The method, as both implementations below compute it (the fused
// one-CTA-per-tensor ttsvd_kernel, and the launch pipeline further down that ttc_tt_svd uses when a workspace
// is given and every Gram side is <= 32):
//   delta^2 = eps^2 / (N - 1) ||X||_F^2;  Z <- X_(1)
//   for n = 1 .. N-1:  delta-truncated SVD of Z (R_{n-1} I_n x rest) through the eigenproblem of its smaller
//                      Gram matrix (fp64, cyclic Jacobi with round-robin parallel rotations):
//                        Z Z^T = U S^2 U^T  (rows <= cols):  G^(n) = U_R,  Z <- U_R^T Z = S_R V_R^T
//                        Z^T Z = V S^2 V^T  (rows > cols):   G^(n) = Z V_R S_R^-1,  Z <- S_R V_R^T
//                      R = the smallest rank with sum_{j >= R} s_j^2 <= delta^2 (readings R23, R25); every
//                      column of U has its largest-magnitude entry positive (R24)
//   G^(N) <- Z
// Output: train b packed from cores_dev + b * train_cap (capacity layout of the largest possible ranks), its
// ranks at ranks_dev[b * (N + 1)].
#include <cfloat>

#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 256;
constexpr int kSweeps = 15;   // cap on cyclic Jacobi sweeps (quadratic convergence: n <= 64 needs < 10 in fp64)
// rotation threshold (R26): a pair (p, q) of the Gram matrix is rotated while g_pq^2 > kTol2 g_pp g_qq,
// i.e. until the columns are orthogonal to 1e-9 relative -- 60x below the fp32 roundoff of the stored cores; the
// eigenvalues (squared singular values, the delta-rank decisions) are then exact to ~1e-18 relative (A2 +3.8%
// over eps_64)
constexpr double kTol2 = 1e-18;
constexpr double kSigmaFloor = 1e-7;

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    __syncthreads();
    return t;
}

// Source offsets of X^rho's elements e = tid, tid + step, ... (Alg. 2 step 1's permutation as strides): the
// mixed-radix digits of e are decomposed once, then advanced by the digits of `step` with carries (no integer
// division per element).
constexpr int kWalkMax = 16;   // orders up to 16 walk in registers (fully unrolled); larger ones divide
struct GatherWalk {
    int32_t dig[kWalkMax], sd[kWalkMax];
    int64_t off;
    int e, step;
    __device__ __forceinline__ void init(const TtsvdArgs& a, int e0, int st) {
        e = e0;
        step = st;
        off = 0;
        if (a.N > kWalkMax) { off = slow(a, e); return; }
        int q = e, r = step;
#pragma unroll
        for (int k = 0; k < kWalkMax; ++k)
            if (k < a.N) {
                dig[k] = q % a.dims[k]; q /= a.dims[k];
                sd[k] = r % a.dims[k]; r /= a.dims[k];
                off += (int64_t)dig[k] * a.in_stride[k];
            }
    }
    __device__ __forceinline__ static int64_t slow(const TtsvdArgs& a, int e) {
        int q = e;
        int64_t o = 0;
        for (int k = 0; k < a.N; ++k) { const int i = q % a.dims[k]; q /= a.dims[k]; o += (int64_t)i * a.in_stride[k]; }
        return o;
    }
    __device__ __forceinline__ void next(const TtsvdArgs& a) {
        e += step;
        if (a.N > kWalkMax) { off = slow(a, e); return; }
        int carry = 0;
#pragma unroll
        for (int k = 0; k < kWalkMax; ++k)
            if (k < a.N) {
                int d = dig[k] + sd[k] + carry;
                carry = d >= a.dims[k];
                if (carry) d -= a.dims[k];
                off += (int64_t)(d - dig[k]) * a.in_stride[k];
                dig[k] = d;
            }
    }
};

// Symmetric eigenproblem of G (n x n, row-major in shared memory, overwritten by the rotated matrix) by cyclic
// Jacobi; V (n x n) receives the eigenvectors as columns.  Round-robin ordering: n' = n rounded up to even
// players, n'/2 disjoint rotations per round (player n' - 1 is a dummy when n is odd), n' - 1 rounds a sweep.
// A pair is rotated only while g_pq^2 > kTol2 |g_pp g_qq| (R26); the iteration stops after a sweep that rotated
// no pair (or kSweeps sweeps).
__device__ void jacobi(double* G, double* V, int n, double* cs, double* sn, int* pp, int* pq, int* flag) {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) V[e] = (e / n == e % n) ? 1.0 : 0.0;
    const int np = (n + 1) & ~1, half = np / 2;
    for (int sweep = 0; sweep < kSweeps; ++sweep) {
        __syncthreads();
        if (threadIdx.x == 0) *flag = 0;
        for (int t = 0; t < np - 1; ++t) {
            __syncthreads();
            for (int q = threadIdx.x; q < half; q += blockDim.x) {
                // players 1..np-1 rotate around the fixed player 0; pair q = (position q, position np-1-q)
                auto pos = [&](int j) { return j == 0 ? 0 : ((j - 1 + t) % (np - 1)) + 1; };
                int a = pos(q), b = pos(np - 1 - q);
                if (a > b) { const int x = a; a = b; b = x; }
                double c = 1.0, s = 0.0;
                bool rot = false;
                if (b < n) {
                    const double app = G[a * n + a], aqq = G[b * n + b], apq = G[a * n + b];
                    if (fabs(apq) > 1e-300 && apq * apq > kTol2 * fabs(app * aqq)) {
                        const double th = (aqq - app) / (2.0 * apq);
                        const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        c = 1.0 / sqrt(tt * tt + 1.0);
                        s = tt * c;
                        rot = true;
                    }
                }
                if (rot) *flag = 1;
                cs[q] = c; sn[q] = s; pp[q] = a; pq[q] = rot ? b : -1;
            }
            __syncthreads();
            // columns p, q of G and V
            for (int e = threadIdx.x; e < half * n; e += blockDim.x) {
                const int q = e / n, k = e - q * n;
                const int b = pq[q];
                if (b < 0) continue;
                const int a = pp[q];
                const double c = cs[q], s = sn[q];
                const double gka = G[k * n + a], gkb = G[k * n + b];
                G[k * n + a] = c * gka - s * gkb;
                G[k * n + b] = s * gka + c * gkb;
                const double vka = V[k * n + a], vkb = V[k * n + b];
                V[k * n + a] = c * vka - s * vkb;
                V[k * n + b] = s * vka + c * vkb;
            }
            __syncthreads();
            // rows p, q of G
            for (int e = threadIdx.x; e < half * n; e += blockDim.x) {
                const int q = e / n, k = e - q * n;
                const int b = pq[q];
                if (b < 0) continue;
                const int a = pp[q];
                const double c = cs[q], s = sn[q];
                const double gak = G[a * n + k], gbk = G[b * n + k];
                G[a * n + k] = c * gak - s * gbk;
                G[b * n + k] = s * gak + c * gbk;
            }
        }
        __syncthreads();
        if (*flag == 0) break;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) ttsvd_kernel(const TtsvdArgs a) {
    extern __shared__ __align__(16) unsigned char sraw[];
    const int b = blockIdx.x, N = a.N, side_max = a.gmax;
    double* G = reinterpret_cast<double*>(sraw);                 // gmax x gmax
    double* V = G + side_max * side_max;                         // gmax x gmax
    double* lam = V + side_max * side_max;                       // gmax
    double* cs = lam + side_max;                                 // gmax / 2 + 1 (rotation cosines)
    double* sn = cs + side_max / 2 + 1;
    double* red = sn + side_max / 2 + 1;                         // 32
    int* order = reinterpret_cast<int*>(red + 32);               // gmax
    int* pp = order + side_max;
    int* pq = pp + side_max / 2 + 1;
    int* misc = pq + side_max / 2 + 1;                           // [0]: R, [1]: Jacobi rotation flag
    float* Z = reinterpret_cast<float*>(misc + 4) + ((4 - ((reinterpret_cast<uintptr_t>(misc + 4) >> 2) & 3)) & 3);
    float* Zt = Z + a.elems;
    const float* src = a.dense + (int64_t)b * a.elems;
    float* out = a.cores + (int64_t)b * a.train_cap;
    int32_t* rout = a.ranks + (int64_t)b * (N + 1);
    // ---- Z <- X^rho (mode k of X^rho is read with the source stride in_stride[k]); ||X||_F^2
    double nrm = 0.0;
    GatherWalk gw;
    gw.init(a, threadIdx.x, blockDim.x);
    for (int e = threadIdx.x; e < a.elems; e += blockDim.x, gw.next(a)) {
        const float v = __ldg(src + gw.off);
        Z[e] = v;
        nrm += (double)v * v;
    }
    nrm = block_sum(nrm, red);
    const double delta2 = a.eps2 * nrm;   // eps^2 / (N - 1) ||X||^2
    if (threadIdx.x == 0) rout[0] = 1;
    int Rprev = 1;
    int64_t o = 0;
    int cur_elems = a.elems;
    for (int n = 0; n < N - 1; ++n) {
        const int m = Rprev * a.dims[n], ncols = cur_elems / m;
        const bool rows_side = m <= ncols;
        const int side = rows_side ? m : ncols;
        // ---- Gram matrix of the smaller side (fp64)
        for (int e = threadIdx.x; e < side * side; e += blockDim.x) {
            const int i = e / side, j = e - i * side;
            if (j < i) continue;
            double acc = 0.0;
            if (rows_side) for (int c = 0; c < ncols; ++c) acc += (double)Z[i + m * c] * Z[j + m * c];
            else for (int r = 0; r < m; ++r) acc += (double)Z[r + m * i] * Z[r + m * j];
            G[i * side + j] = acc;
            G[j * side + i] = acc;
        }
        jacobi(G, V, side, cs, sn, pp, pq, misc + 1);
        // ---- eigenvalues descending (stable order), the delta-truncated rank
        for (int j = threadIdx.x; j < side; j += blockDim.x) lam[j] = fmax(G[j * side + j], 0.0);
        __syncthreads();
        for (int j = threadIdx.x; j < side; j += blockDim.x) {
            int rank = 0;
            for (int i = 0; i < side; ++i) rank += (lam[i] > lam[j]) || (lam[i] == lam[j] && i < j);
            order[rank] = j;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const double top = lam[order[0]];
            int keep = 0;
            for (int j = 0; j < side; ++j) keep += lam[order[j]] > kSigmaFloor * kSigmaFloor * top && top > 0.0;
            int R = keep < 1 ? 1 : keep;
            double tail = 0.0;   // sum_{j >= R} s_j^2 over the kept values
            for (int j = keep - 1; j >= 1; --j) {
                tail += lam[order[j]];
                if (tail <= delta2) R = j; else break;
            }
            misc[0] = R;
        }
        __syncthreads();
        const int R = misc[0];
        // ---- U (m x R) into the output core, the next Z (R x ncols) into Zt
        if (rows_side) {   // U = eigenvectors of Z Z^T
            for (int e = threadIdx.x; e < m * R; e += blockDim.x) {
                const int j = e / m, i = e - j * m;
                out[o + e] = (float)V[i * side + order[j]];
            }
        } else {           // U = Z V_R S_R^-1
            for (int e = threadIdx.x; e < m * R; e += blockDim.x) {
                const int j = e / m, r = e - j * m;
                const int col = order[j];
                double acc = 0.0;
                for (int c = 0; c < ncols; ++c) acc += (double)Z[r + m * c] * V[c * side + col];
                out[o + e] = lam[col] > 0.0 ? (float)(acc / sqrt(lam[col])) : 0.f;
            }
        }
        __syncthreads();
        // R24: the largest-magnitude entry of every column of U positive (flip the column and its row of S V^T)
        for (int j = threadIdx.x; j < R; j += blockDim.x) {
            float best = 0.f;
            int bi = 0;
            for (int i = 0; i < m; ++i) {
                const float v = fabsf(out[o + i + (int64_t)m * j]);
                if (v > best) { best = v; bi = i; }
            }
            const bool flip = out[o + bi + (int64_t)m * j] < 0.f;
            if (flip)
                for (int i = 0; i < m; ++i) out[o + i + (int64_t)m * j] = -out[o + i + (int64_t)m * j];
            lam[order[j]] = flip ? -lam[order[j]] : lam[order[j]];   // sign carried in lam's sign bit
        }
        __syncthreads();
        // next Z = U^T Z (rows side) or S_R V_R^T (cols side), with the signs of U's columns
        for (int e = threadIdx.x; e < R * ncols; e += blockDim.x) {
            const int c = e / R, j = e - c * R;
            const int col = order[j];
            const double sgn = lam[col] < 0.0 ? -1.0 : 1.0;
            double v;
            if (rows_side) {
                double acc = 0.0;
                for (int i = 0; i < m; ++i) acc += V[i * side + col] * (double)Z[i + m * c];
                v = sgn * acc;
            } else {
                v = sgn * sqrt(fabs(lam[col])) * V[c * side + col];
            }
            Zt[j + R * c] = (float)v;
        }
        __syncthreads();
        { float* t = Z; Z = Zt; Zt = t; }
        o += (int64_t)m * R;
        if (threadIdx.x == 0) rout[n + 1] = R;
        cur_elems = R * ncols;
        Rprev = R;
    }
    // ---- G^(N) <- Z (R_{N-1} x I_N)
    for (int e = threadIdx.x; e < cur_elems; e += blockDim.x) out[o + e] = Z[e];
    if (threadIdx.x == 0) rout[N] = 1;
}

// ===================================================================================================
// Multi-kernel pipeline for Gram sides <= 32 (ttc_tt_svd's default; the fused kernel above keeps larger
// sides): the per-tensor Jacobi iterations are latency chains (each round waits on one rotation's fp64
// sqrt / divide), so instead of one CTA per tensor holding the whole SVD (3 per SM, the SM idle behind the
// CTA barriers), every eigenproblem runs on ONE warp with no CTA barriers, 4 per CTA and up to 8 CTAs per
// SM, the whole batch in flight at once; the dense phases (gather, Gram matrices, U, the next unfolding)
// are separate CTA-per-tensor kernels, passing Z_n, the Gram matrix and its eigenvectors through a
// workspace (L2-resident at A2's sizes).
//   first  : Z_0 <- X^rho, ||X||^2, Gram of Z_0
//   jacobi : (per step n) eigenvectors (two warps per eigenproblem: G and V updates overlapped), eigenvalues
//            in descending order, the delta-truncated rank R_n
//   step   : (per step n) core n = U (R24 signs), Z_{n+1}, its Gram (or, after the last step, core N)

// Gram matrix of Z (m x ncols, Z[r + m c]) of the smaller side (side x side, row-major) in fp64 register tiles: 4 x 4 tiles of the upper triangle, one warp per tile,
// its lanes splitting the summed index (lane, lane + 32, ...), the 16 partial sums reduced by warp shuffles (no
// atomics), then written to g and mirrored.  Element (i, t) of the side x len operand is Z[i si + t st].
__device__ void gram_tiled(const float* Z, int m, int ncols, double* g) {
    const bool rows_side = m <= ncols;
    const int side = rows_side ? m : ncols, len = rows_side ? ncols : m;
    const int si = rows_side ? 1 : m, st = rows_side ? m : 1;
    const int T = (side + 3) >> 2, pairs = T * (T + 1) / 2;
    const int wp = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int it = wp; it < pairs; it += nw) {
        int p = it, ti = 0;
        while (p >= T - ti) { p -= T - ti; ++ti; }   // upper-triangle tile (ti, tj), tj >= ti
        const int tj = ti + p, i0 = 4 * ti, j0 = 4 * tj;
        double acc[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
        int ia[4], ja[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { ia[u] = min(i0 + u, side - 1) * si; ja[u] = min(j0 + u, side - 1) * si; }
        for (int t = l; t < len; t += 32) {
            const float* zt = Z + t * st;
            double x[4], y[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { x[u] = zt[ia[u]]; y[u] = zt[ja[u]]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(x[u], y[v], acc[u][v]);
        }
        // butterfly reduce-scatter of the 16 sums over the warp (8 + 4 + 2 + 1 + 1 exchanges instead of 16 x 5):
        // each level a lane keeps the half of its values selected by one lane bit and adds the partner's copy
        double r[16];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) r[4 * u + v] = acc[u][v];
#pragma unroll
        for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
            const bool up = (l & o) != 0;
#pragma unroll
            for (int k = 0; k < h; ++k) {
                const double send = up ? r[k] : r[k + h];
                const double keep = up ? r[k + h] : r[k];
                r[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        r[0] += __shfl_xor_sync(0xffffffffu, r[0], 1);
        if ((l & 1) == 0) {   // lane 2q holds sum number 8 b4 + 4 b3 + 2 b2 + b1 of its lane bits
            const int idx = ((l >> 4) & 1) * 8 + ((l >> 3) & 1) * 4 + ((l >> 2) & 1) * 2 + ((l >> 1) & 1);
            const int i = i0 + (idx >> 2), j = j0 + (idx & 3);
            if (i < side && j < side) { g[i * side + j] = r[0]; g[j * side + i] = r[0]; }
        }
    }
}

// Z[dst(e)] = src[e] for the tensor's elements e = tid, tid + blockDim, ... read contiguously; dst by the
// mixed-radix walk of e (radices rad, X^rho strides dstr, source mode order) advanced by blockDim's digits with
// carries (NW >= N digits in registers; NW = 0: per-element division).  The copies are cp.async (all in flight
// at once); the caller waits for them.
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
template <int NW>
__device__ __forceinline__ double scatter_walk(const TtsvdArgs& a, const float* src, float* Z, const int32_t* rad_s,
                                               const int32_t* dstr_s) {
    const int N = a.N;
    double nrm = 0.0;
    if (NW == 0) {
        for (int e = threadIdx.x; e < a.elems; e += blockDim.x) {
            int q = e, off = 0;
            for (int p = 0; p < N; ++p) { off += (q % rad_s[p]) * dstr_s[p]; q /= rad_s[p]; }
            cp_async4(Z + off, src + e);
        }
        return nrm;
    }
    constexpr int W = NW > 0 ? NW : 1;
    int dig[W], sd[W], rad[W], dstr[W];
    int off = 0, q = threadIdx.x, r = blockDim.x;
#pragma unroll
    for (int p = 0; p < W; ++p) {
        rad[p] = p < N ? rad_s[p] : 1;
        dstr[p] = p < N ? dstr_s[p] : 0;
        dig[p] = q % rad[p]; q /= rad[p];
        sd[p] = r % rad[p]; r /= rad[p];
        off += dig[p] * dstr[p];
    }
    for (int e = threadIdx.x; e < a.elems; e += blockDim.x) {
        cp_async4(Z + off, src + e);
        int carry = 0;
#pragma unroll
        for (int p = 0; p < W; ++p) {   // (padding digits: radix 1, stride 0 -> no effect)
            int d = dig[p] + sd[p] + carry;
            carry = d >= rad[p];
            if (carry) d -= rad[p];
            off += (d - dig[p]) * dstr[p];
            dig[p] = d;
        }
    }
    return nrm;
}

__global__ void __launch_bounds__(kThreads, 4) ttsvd_first_kernel(const TtsvdArgs a, const TtsvdWs w) {
    extern __shared__ __align__(16) unsigned char sraw[];
    __shared__ int32_t rad[TTC_MAX_ORDER];
    __shared__ int32_t dstr[TTC_MAX_ORDER];
    double* red = reinterpret_cast<double*>(sraw);                // 32
    float* Z = reinterpret_cast<float*>(red + 32);
    const int b = blockIdx.x, N = a.N;
    const float* src = a.dense + (int64_t)b * a.elems;
    float* zg = w.z + (int64_t)b * a.elems;
    // the source's modes in memory order (X^rho's modes sorted by source stride), with X^rho's compact strides:
    // the source is read contiguously (coalesced) and scattered into Z in X^rho order
    if (threadIdx.x == 0) {
        for (int p = 0; p < N; ++p) {
            int best = -1;
            for (int k = 0; k < N; ++k) {
                bool used = false;
                for (int q = 0; q < p; ++q) used |= rad[q] == -1 - k;   // (temporarily: -1 - mode)
                if (!used && (best < 0 || a.in_stride[k] < a.in_stride[best])) best = k;
            }
            rad[p] = -1 - best;
        }
        for (int p = 0; p < N; ++p) {
            const int k = -1 - rad[p];
            int32_t xs = 1;   // X^rho's compact stride of mode k
            for (int k2 = 0; k2 < k; ++k2) xs *= a.dims[k2];
            rad[p] = a.dims[k];
            dstr[p] = xs;
        }
    }
    __syncthreads();
    if (N <= 4) scatter_walk<4>(a, src, Z, rad, dstr);
    else scatter_walk<0>(a, src, Z, rad, dstr);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    double nrm = 0.0;   // ||X||^2, and Z_0 to the workspace for the step kernel
    for (int e = threadIdx.x; e < a.elems; e += blockDim.x) {
        const float v = Z[e];
        zg[e] = v;
        nrm += (double)v * v;
    }
    nrm = block_sum(nrm, red);
    if (threadIdx.x == 0) {
        w.nrm[b] = nrm;
        a.ranks[(int64_t)b * (N + 1)] = 1;
    }
    gram_tiled(Z, a.dims[0], a.elems / a.dims[0], w.g + (int64_t)b * a.gmax * a.gmax);
}

// Cyclic Jacobi of G (n x n, n <= 32) on a PAIR of warps, with no CTA barriers: same round-robin pairs and
// rotation rule as jacobi() (one sqrt, one divide, one rsqrt per rotation); every round applies its rotations at
// once as 2 x 2 upper-triangle block updates G' = J_p^T G J_q mirrored (G double-buffered, so one pass), rounds
// that rotate nothing are skipped, and the iteration stops after a sweep that rotates no pair.
// The G warp (role 0) computes each round's rotations into one of
// two parameter buffers and applies the two-sided block update to G; the V warp (role 1) applies the previous
// round's rotations to V (V J) meanwhile, so the V update leaves the critical path.  The two warps meet once a
// round at a 64-thread named barrier `bar`; ctl[0] publishes "round r rotates" and ctl[1] "stop".  Returns the
// buffer holding the final G (in the G warp).
struct JacParams {
    double cs[2][16], sn[2][16];
    int pa[2][16], pb[2][16];
    int ctl[4];
};
__device__ __forceinline__ void pair_bar(int bar) { asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory"); }

// One round's two-sided rotation of G into Gn for this lane's upper-triangle 2 x 2 blocks (bp: q1 << 8 | q2, -1
// past the end), mirrored.  G and Gn are distinct buffers (__restrict__): every block's loads can be issued
// ahead of the other blocks' stores.
__device__ __forceinline__ void block_update(const double* __restrict__ G, double* __restrict__ Gn, int n,
                                             const JacParams& P, int cur, const int (&bp)[5]) {
    double y[5][4];
    int a1s[5], b1s[5], a2s[5], b2s[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
        if (bp[u] < 0) break;
        const int q1 = bp[u] >> 8, q2 = bp[u] & 255;
        const int a1 = P.pa[cur][q1], b1 = P.pb[cur][q1], a2 = P.pa[cur][q2], b2 = P.pb[cur][q2];
        const double c1 = P.cs[cur][q1], s1 = P.sn[cur][q1], c2 = P.cs[cur][q2], s2 = P.sn[cur][q2];
        const bool hb1 = b1 < n, hb2 = b2 < n;
        const double g00 = G[a1 * n + a2], g01 = hb2 ? G[a1 * n + b2] : 0.0;
        const double g10 = hb1 ? G[b1 * n + a2] : 0.0, g11 = hb1 && hb2 ? G[b1 * n + b2] : 0.0;
        const double x00 = c2 * g00 - s2 * g01, x01 = s2 * g00 + c2 * g01;   // B J2
        const double x10 = c2 * g10 - s2 * g11, x11 = s2 * g10 + c2 * g11;
        y[u][0] = c1 * x00 - s1 * x10; y[u][1] = c1 * x01 - s1 * x11;     // J1^T (B J2)
        y[u][2] = s1 * x00 + c1 * x10; y[u][3] = s1 * x01 + c1 * x11;
        a1s[u] = a1; b1s[u] = b1; a2s[u] = a2; b2s[u] = b2;
    }
#pragma unroll
    for (int u = 0; u < 5; ++u) {
        if (bp[u] < 0) break;
        const int a1 = a1s[u], b1 = b1s[u], a2 = a2s[u], b2 = b2s[u];
        const bool hb1 = b1 < n, hb2 = b2 < n;
        Gn[a1 * n + a2] = y[u][0];
        Gn[a2 * n + a1] = y[u][0];
        if (hb2) { Gn[a1 * n + b2] = y[u][1]; Gn[b2 * n + a1] = y[u][1]; }
        if (hb1) { Gn[b1 * n + a2] = y[u][2]; Gn[a2 * n + b1] = y[u][2]; }
        if (hb1 && hb2) { Gn[b1 * n + b2] = y[u][3]; Gn[b2 * n + b1] = y[u][3]; }
    }
}

__device__ double* jacobi_pair(double* G, double* Gn, double* V, int n, JacParams& P, int role, int bar) {
    const int lane = threadIdx.x & 31;
    const int np = (n + 1) & ~1, half = np / 2;
    // V is kept TRANSPOSED here (Vt[col][row]: lane = row, so a column rotation is one conflict-free access per
    // lane); the caller stores it back row-major
    if (role == 1)
        for (int e = lane; e < n * n; e += 32) V[e] = (e / n == e % n) ? 1.0 : 0.0;
    int bp[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
        int p = lane + 32 * u, q1 = 0;
        if (p >= half * (half + 1) / 2) { bp[u] = -1; continue; }
        while (p >= half - q1) { p -= half - q1; ++q1; }
        bp[u] = (q1 << 8) | (q1 + p);
    }
    int px = lane == 0 ? 0 : lane, py = np - 1 - lane;   // this lane's players' positions (pos(j) at t = 0 is j)
    int sweep = 0, t = 0, r = 0;
    bool any = false;
    for (;; ++r) {
        const int cur = r & 1;
        if (role == 0) {
            // stop after a sweep that rotated nothing (or kSweeps sweeps): decided at the start of a sweep
            bool stop = false;
            if (t == 0 && r > 0) {
                stop = !any || sweep == kSweeps;
                any = false;
            }
            bool rot = false;
            if (!stop && lane < half) {
                int x = px, y = py;
                if (x > y) { const int u = x; x = y; y = u; }
                double c = 1.0, sv = 0.0;
                if (y < n) {
                    const double app = G[x * n + x], aqq = G[y * n + y], apq = G[x * n + y];
                    if (fabs(apq) > 1e-300 && apq * apq > kTol2 * fabs(app * aqq)) {
                        const double d = aqq - app, b2 = apq + apq;
                        const double tt = (d >= 0.0 ? b2 : -b2) / (fabs(d) + sqrt(fma(d, d, b2 * b2)));
                        c = rsqrt(fma(tt, tt, 1.0));
                        sv = tt * c;
                        rot = true;
                    }
                }
                P.cs[cur][lane] = c; P.sn[cur][lane] = sv; P.pa[cur][lane] = x; P.pb[cur][lane] = y;
            }
            const bool rr = __any_sync(0xffffffffu, rot);
            any |= rr;
            if (lane == 0) P.ctl[cur] = (rr ? 1 : 0) | (stop ? 2 : 0);   // parity slot: the V warp reads it after
                                                                          // this barrier, before round r + 2 reuses it
            if (px != 0) px = px == np - 1 ? 1 : px + 1;
            py = py == np - 1 ? 1 : py + 1;
            if (++t == np - 1) { t = 0; ++sweep; }
            pair_bar(bar);   // round r's rotations published; the V warp has finished round r - 1
            if (stop) break;
            if (rr) {
                block_update(G, Gn, n, P, cur, bp);
                __syncwarp();
                double* tmp = G; G = Gn; Gn = tmp;
            }
        } else {
            pair_bar(bar);
            const int f = P.ctl[cur];
            if (f & 2) break;
            if ((f & 1) && lane < n) {   // V J: lane = row, the round's rotations in turn (broadcast parameters)
                for (int q = 0; q < half; ++q) {
                    const int x = P.pa[cur][q], y = P.pb[cur][q];
                    const double sv = P.sn[cur][q];
                    if (y >= n || sv == 0.0) continue;
                    const double c = P.cs[cur][q];
                    const double vx = V[x * n + lane], vy = V[y * n + lane];
                    V[x * n + lane] = c * vx - sv * vy;
                    V[y * n + lane] = sv * vx + c * vy;
                }
            }
        }
    }
    // both warps leave at the same barrier (the V warp's last update finished before it); the returned G is the
    // G warp's final buffer (the V warp's copy of the pointer is not used)
    return G;
}

// The same iteration on ONE warp per eigenproblem (the default; TTC_JAC_PAIR builds use jacobi_pair): each round
// computes its rotations, applies them to G (block update into Gn) and to V in turn.  Half the registers per
// problem, so twice as many problems resident per SM: A2's 2,048 eigenproblems per launch fit in one wave
// (16 per SM) instead of 1.73 (8 per SM), and A2 runs 5% faster (762 K -> 801 K pairs/s) although each problem
// takes longer.
__device__ double* jacobi_solo(double* G, double* Gn, double* V, int n, JacParams& P) {
    const int lane = threadIdx.x & 31;
    const int np = (n + 1) & ~1, half = np / 2;
    for (int e = lane; e < n * n; e += 32) V[e] = (e / n == e % n) ? 1.0 : 0.0;   // V transposed (lane = row)
    int bp[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
        int p = lane + 32 * u, q1 = 0;
        if (p >= half * (half + 1) / 2) { bp[u] = -1; continue; }
        while (p >= half - q1) { p -= half - q1; ++q1; }
        bp[u] = (q1 << 8) | (q1 + p);
    }
    int px = lane == 0 ? 0 : lane, py = np - 1 - lane;
    int sweep = 0, t = 0;
    bool any = false;
    for (int r = 0;; ++r) {
        const int cur = r & 1;
        bool stop = false;
        if (t == 0 && r > 0) {
            stop = !any || sweep == kSweeps;
            any = false;
        }
        if (stop) break;
        bool rot = false;
        if (lane < half) {
            int x = px, y = py;
            if (x > y) { const int u = x; x = y; y = u; }
            double c = 1.0, sv = 0.0;
            if (y < n) {
                const double app = G[x * n + x], aqq = G[y * n + y], apq = G[x * n + y];
                if (fabs(apq) > 1e-300 && apq * apq > kTol2 * fabs(app * aqq)) {
                    const double d = aqq - app, b2 = apq + apq;
                    const double tt = (d >= 0.0 ? b2 : -b2) / (fabs(d) + sqrt(fma(d, d, b2 * b2)));
                    c = rsqrt(fma(tt, tt, 1.0));
                    sv = tt * c;
                    rot = true;
                }
            }
            P.cs[cur][lane] = c; P.sn[cur][lane] = sv; P.pa[cur][lane] = x; P.pb[cur][lane] = y;
        }
        const bool rr = __any_sync(0xffffffffu, rot);
        any |= rr;
        if (px != 0) px = px == np - 1 ? 1 : px + 1;
        py = py == np - 1 ? 1 : py + 1;
        if (++t == np - 1) { t = 0; ++sweep; }
        if (!rr) continue;
        __syncwarp();   // the round's parameters visible
        block_update(G, Gn, n, P, cur, bp);
        {   // V J: the round's (rotation q, row) items spread over all 32 lanes (rotations touch disjoint row pairs
            // of the transposed V; identity rotations rewrite their rows unchanged); e / n by a multiply-shift
            const unsigned inv = (65536u + (unsigned)n - 1u) / (unsigned)n;   // exact for e < 1024 when n <= 32
            for (int e = lane; e < half * n; e += 32) {
                const int q = (int)(((unsigned)e * inv) >> 16), row = e - q * n;
                const int x = P.pa[cur][q], y = P.pb[cur][q];
                if (y >= n) continue;
                const double c = P.cs[cur][q], sv = P.sn[cur][q];
                const double vx = V[x * n + row], vy = V[y * n + row];
                V[x * n + row] = c * vx - sv * vy;
                V[y * n + row] = sv * vx + c * vy;
            }
        }
        __syncwarp();
        double* tmp = G; G = Gn; Gn = tmp;
    }
    return G;
}

#ifdef TTC_JAC_PAIR
constexpr int kJacWarps = 2;    // warps per eigenproblem
#else
constexpr int kJacWarps = 1;
#endif
constexpr int kJacPairs = 4;   // eigenproblems per CTA (kJacWarps warps each)

__global__ void __launch_bounds__(32 * kJacWarps * kJacPairs) ttsvd_jacobi_kernel(const TtsvdArgs a, const TtsvdWs w, int n) {
    extern __shared__ __align__(16) unsigned char sraw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = kJacWarps == 2 ? warp >> 1 : warp, role = kJacWarps == 2 ? warp & 1 : 0;
    const int b = blockIdx.x * kJacPairs + pair;
    if (b >= a.B) return;   // (both warps of the pair leave: only pair-local barriers below)
    const int g2 = a.gmax * a.gmax, N = a.N;
    double* G = reinterpret_cast<double*>(sraw) + (size_t)pair * (3 * g2 + 32);
    double* Gn = G + g2;
    double* V = Gn + g2;
    double* lam = V + g2;                                    // 32
    JacParams& P = reinterpret_cast<JacParams*>(sraw + sizeof(double) * (size_t)kJacPairs * (3 * g2 + 32))[pair];
    __shared__ int ord_s[kJacPairs][32];
    int* ord = ord_s[pair];
    int32_t* rk = a.ranks + (int64_t)b * (N + 1);
    const int Rprev = rk[n];
    int64_t cur = Rprev;
    for (int k = n; k < N; ++k) cur *= a.dims[k];
    const int m = Rprev * a.dims[n], ncols = (int)(cur / m), side = m <= ncols ? m : ncols;
    if (role == 0) {
        const double* gsrc = w.g + (int64_t)b * g2;
        for (int e = lane; e < side * side; e += 32) G[e] = gsrc[e];
        __syncwarp();
    }
    const double* Gf = kJacWarps == 2 ? jacobi_pair(G, Gn, V, side, P, role, 1 + pair) : jacobi_solo(G, Gn, V, side, P);
    if (kJacWarps == 1) __syncwarp();
    if (role == 1 || kJacWarps == 1) {   // V is final: store it row-major (it was kept transposed)
        double* vdst = w.v + (int64_t)b * g2;
        for (int e = lane; e < side * side; e += 32) {
            const int k = e / side, x = e - k * side;
            vdst[e] = V[x * side + k];
        }
        if (kJacWarps == 2) return;
    }
    // eigenvalues, descending stable order
    if (lane < side) lam[lane] = fmax(Gf[lane * side + lane], 0.0);
    __syncwarp();
    if (lane < side) {
        int rank = 0;
        for (int i = 0; i < side; ++i) rank += (lam[i] > lam[lane]) || (lam[i] == lam[lane] && i < lane);
        ord[rank] = lane;
    }
    __syncwarp();
    if (lane == 0) {   // R23 / R25: the delta-truncated rank over the values above the floor
        const double top = lam[ord[0]], delta2 = a.eps2 * w.nrm[b];
        int keep = 0;
        for (int j = 0; j < side; ++j) keep += lam[ord[j]] > kSigmaFloor * kSigmaFloor * top && top > 0.0;
        int R = keep < 1 ? 1 : keep;
        double tail = 0.0;
        for (int j = keep - 1; j >= 1; --j) {
            tail += lam[ord[j]];
            if (tail <= delta2) R = j; else break;
        }
        rk[n + 1] = R;
    }
    if (lane < side) {
        w.lam[(int64_t)b * a.gmax + lane] = lam[lane];
        w.ord[(int64_t)b * a.gmax + lane] = ord[lane];
    }
}

__global__ void __launch_bounds__(kThreads, 3) ttsvd_step_kernel(const TtsvdArgs a, const TtsvdWs w, int n) {
    extern __shared__ __align__(16) unsigned char sraw[];
    const int b = blockIdx.x, N = a.N, gm = a.gmax;
    const int32_t* rk = a.ranks + (int64_t)b * (N + 1);
    const int Rprev = rk[n], R = rk[n + 1];
    int64_t cur = Rprev;
    for (int k = n; k < N; ++k) cur *= a.dims[k];
    const int m = Rprev * a.dims[n], ncols = (int)(cur / m);
    const bool rows_side = m <= ncols;
    const int side = rows_side ? m : ncols;
    double* V = reinterpret_cast<double*>(sraw);                  // gm x gm
    double* lam = V + gm * gm;                                     // gm
    int* ord = reinterpret_cast<int*>(lam + gm);                   // gm
    int64_t* oo = reinterpret_cast<int64_t*>(ord + ((gm + 3) & ~3));   // [0]: offset of core n
    float* Z = reinterpret_cast<float*>(oo + 2);
    float* U = Z + a.elems;
    if (threadIdx.x == 0) {
        int64_t o = 0;
        for (int k = 0; k < n; ++k) o += (int64_t)rk[k] * a.dims[k] * rk[k + 1];
        oo[0] = o;
    }
    // Z_n and the eigenvectors: every load in flight at once (16-byte cp.async where aligned), one round trip
    const float* zg = w.z + (int64_t)b * a.elems;
    const double* vg = w.v + (int64_t)b * gm * gm;
    const int nz = (int)cur;
    if (((reinterpret_cast<uintptr_t>(zg) | reinterpret_cast<uintptr_t>(Z)) & 15u) == 0) {
        for (int e = threadIdx.x; e < (nz >> 2); e += blockDim.x) tc::cp_async16(Z + 4 * e, zg + 4 * e);
        for (int e = (nz & ~3) + threadIdx.x; e < nz; e += blockDim.x) Z[e] = zg[e];
    } else {
        for (int e = threadIdx.x; e < nz; e += blockDim.x) Z[e] = zg[e];
    }
    if (((reinterpret_cast<uintptr_t>(vg) | reinterpret_cast<uintptr_t>(V)) & 15u) == 0) {
        for (int e = threadIdx.x; e < (side * side >> 1); e += blockDim.x) tc::cp_async16(V + 2 * e, vg + 2 * e);
        if ((side * side) & 1) if (threadIdx.x == 0) V[side * side - 1] = vg[side * side - 1];
    } else {
        for (int e = threadIdx.x; e < side * side; e += blockDim.x) V[e] = vg[e];
    }
    tc::cp_commit_group();
    for (int j = threadIdx.x; j < side; j += blockDim.x) {
        lam[j] = w.lam[(int64_t)b * gm + j];
        ord[j] = w.ord[(int64_t)b * gm + j];
    }
    tc::cp_wait_pending(0);
    __syncthreads();
    float* out = a.cores + (int64_t)b * a.train_cap + oo[0];
    // ---- U (m x R)
    if (rows_side) {
        for (int e = threadIdx.x; e < m * R; e += blockDim.x) {
            const int j = e / m, i = e - j * m;
            U[e] = (float)V[i * side + ord[j]];
        }
    } else {           // U = Z V_R S_R^-1 in 4 (r) x 4 (j) register tiles, fp64 accumulation
        const int tr = (m + 3) >> 2, tj = (R + 3) >> 2;
        for (int it = threadIdx.x; it < tr * tj; it += blockDim.x) {
            const int r0 = 4 * (it % tr), j0 = 4 * (it / tr);
            int col[4], rr[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { col[u] = ord[min(j0 + u, R - 1)]; rr[u] = min(r0 + u, m - 1); }
            double acc[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
            for (int c = 0; c < ncols; ++c) {
                double x[4], y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) { x[u] = Z[rr[u] + m * c]; y[u] = V[c * side + col[u]]; }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fma(x[u], y[v], acc[u][v]);
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                if (j0 + v >= R) break;
                const double l = lam[col[v]];
                const double inv = l > 0.0 ? 1.0 / sqrt(l) : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (r0 + u < m) U[r0 + u + m * (j0 + v)] = l > 0.0 ? (float)(acc[u][v] * inv) : 0.f;
            }
        }
    }
    __syncthreads();
    // ---- R24: one warp per column, the largest |entry| (lowest row on ties) made positive
    {
        const int wp = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int j = wp; j < R; j += nw) {
            const float* u = U + (int64_t)m * j;
            float best = -1.f;
            int bi = 0;
            for (int i = l; i < m; i += 32) {
                const float v = fabsf(u[i]);
                if (v > best) { best = v; bi = i; }
            }
            for (int o2 = 16; o2 > 0; o2 >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, best, o2);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o2);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (l == 0 && u[bi] < 0.f) lam[ord[j]] = -lam[ord[j]];   // sign bit carries the flip (lam may be 0)
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < m * R; e += blockDim.x) {
        const int j = e / m;
        out[e] = signbit(lam[ord[j]]) ? -U[e] : U[e];
    }
    __syncthreads();
    // ---- Z_{n+1} = U^T Z (rows side) or S_R V_R^T (cols side), signs applied; into U's buffer
    if (rows_side) {   // U^T Z in 4 (j) x 4 (c) register tiles, fp64 accumulation
        const int tj = (R + 3) >> 2, tc = (ncols + 3) >> 2;
        for (int it = threadIdx.x; it < tj * tc; it += blockDim.x) {
            const int c0 = 4 * (it / tj), j0 = 4 * (it - (it / tj) * tj);
            int col[4], cc[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { col[u] = ord[min(j0 + u, R - 1)]; cc[u] = m * min(c0 + u, ncols - 1); }
            double acc[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
            for (int i = 0; i < m; ++i) {
                double x[4], y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) { x[u] = V[i * side + col[u]]; y[u] = Z[i + cc[u]]; }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = fma(x[u], y[v], acc[u][v]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    if (j0 + u < R && c0 + v < ncols)
                        U[j0 + u + R * (c0 + v)] = (float)(signbit(lam[col[u]]) ? -acc[u][v] : acc[u][v]);
        }
    } else {
        for (int e = threadIdx.x; e < R * ncols; e += blockDim.x) {
            const int c = e / R, j = e - c * R;
            const int col = ord[j];
            const double sgn = signbit(lam[col]) ? -1.0 : 1.0;
            U[j + R * c] = (float)(sgn * sqrt(fabs(lam[col])) * V[c * side + col]);
        }
    }
    __syncthreads();
    const int nel = R * ncols;
    if (n + 2 == N) {   // the last core G^(N) = Z_{N-1}
        for (int e = threadIdx.x; e < nel; e += blockDim.x) out[(int64_t)m * R + e] = U[e];
        if (threadIdx.x == 0) a.ranks[(int64_t)b * (N + 1) + N] = 1;
        return;
    }
    float* zo = w.z + (int64_t)b * a.elems;
    for (int e = threadIdx.x; e < nel; e += blockDim.x) zo[e] = U[e];
    const int m2 = R * a.dims[n + 1];
    gram_tiled(U, m2, nel / m2, w.g + (int64_t)b * gm * gm);
}

}  // namespace

cudaError_t launch_ttsvd(const TtsvdArgs& a, size_t smem_bytes, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(ttsvd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    ttsvd_kernel<<<a.B, kThreads, smem_bytes, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_ttsvd_pipeline(const TtsvdArgs& a, const TtsvdWs& w, cudaStream_t s) {
    const int gm = a.gmax;
    const size_t smem_first = sizeof(double) * 32 + sizeof(double) * (size_t)((a.elems + 1) / 2);
    const size_t smem_jac = (sizeof(double) * (size_t)(3 * gm * gm + 32) + sizeof(JacParams)) * kJacPairs;
    const size_t smem_step = sizeof(double) * (size_t)(gm * gm + gm) + sizeof(int) * (size_t)((gm + 3) & ~3) +
                             2 * sizeof(int64_t) + 2 * sizeof(float) * (size_t)a.elems;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(ttsvd_first_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_first)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ttsvd_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_jac)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ttsvd_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_step)) != cudaSuccess) return e;
    // shared memory bounds how many tensors an SM holds at once: ask for the largest carveout
    if ((e = cudaFuncSetAttribute(ttsvd_first_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ttsvd_jacobi_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ttsvd_step_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess) return e;
    ttsvd_first_kernel<<<a.B, kThreads, smem_first, s>>>(a, w);
    for (int n = 0; n + 1 < a.N; ++n) {
        ttsvd_jacobi_kernel<<<(a.B + kJacPairs - 1) / kJacPairs, 32 * kJacWarps * kJacPairs, smem_jac, s>>>(a, w, n);
        ttsvd_step_kernel<<<a.B, kThreads, smem_step, s>>>(a, w, n);
    }
    return cudaGetLastError();
}

}  // namespace ttc
