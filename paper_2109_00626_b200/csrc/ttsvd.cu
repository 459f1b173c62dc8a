// ttsvd.cu -- batched TT-SVD (ttc.h: ttc_tt_svd; Alg. 1), optionally of the permuted tensor
// X^rho of Alg. 2 step 1.  One CTA per tensor, the whole tensor in shared memory:
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

#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 256;
constexpr int kSweeps = 15;   // cap on cyclic Jacobi sweeps (quadratic convergence: n <= 64 needs < 10 in fp64)
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

// Symmetric eigenproblem of G (n x n, row-major in shared memory, overwritten by the rotated matrix) by cyclic
// Jacobi; V (n x n) receives the eigenvectors as columns.  Round-robin ordering: n' = n rounded up to even
// players, n'/2 disjoint rotations per round (player n' - 1 is a dummy when n is odd), n' - 1 rounds a sweep.
// A pair is rotated only while |g_pq| > eps_64 sqrt(|g_pp g_qq|) (below that the rotation changes nothing at
// fp64 precision); the iteration stops after a sweep that rotated no pair (or kSweeps sweeps).
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
                    if (fabs(apq) > 1e-300 && fabs(apq) > DBL_EPSILON * sqrt(fabs(app * aqq))) {
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
    for (int e = threadIdx.x; e < a.elems; e += blockDim.x) {
        int q = e;
        int64_t o = 0;
        for (int k = 0; k < N; ++k) { const int i = q % a.dims[k]; q /= a.dims[k]; o += (int64_t)i * a.in_stride[k]; }
        const float v = __ldg(src + o);
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

}  // namespace

cudaError_t launch_ttsvd(const TtsvdArgs& a, size_t smem_bytes, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(ttsvd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    ttsvd_kernel<<<a.B, kThreads, smem_bytes, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ttc
