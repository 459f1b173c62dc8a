// reconstruct.cu -- dense tensors of a batch of trains (ttc.h: ttc_reconstruct; Eq. 9, and
// Alg. 2 steps 5-6: reconstruct, then permute).  One CTA per train:
//   Left  = X_1 ... X_k          (prod_{n<=k} I_n  x  R_k), built left to right in shared memory
//   Right = X_{k+1} ... X_N      (R_k  x  prod_{n>k} I_n), built right to left in shared memory
//   D[row, col] = sum_r Left[row, r] Right[r, col]
// with row = (i_1..i_k) (little-endian, or big-endian when that puts the output's stride-1 mode first) and
// col = (i_{k+1}..i_N) little-endian; the output address of (row, col) is
// offr[row] + offc[col] (the permuted Eq. 2 strides), so the permutation of step 6 costs nothing extra.
//
// Every product -- each build step and D itself -- is one register-tiled FP32 GEMM, out(m, n) = sum_q
// At[q][m] B[n][q], with both operands in shared memory in layouts the Eq. 2 core layout gives for free:
//   Left step  P_{j+1}^T[s][(pr, i)] = sum_r P_j^T[r][pr] X_j[(i, s)][r]     (X_j as stored: [i + I s][r])
//   Right step Q_{j}[(i, pc)][r]     = sum_s X_j^T[s][(r, i)] Q_{j+1}[pc][s] (X_j as stored: [s][r + R i])
//   D          D[row][col]           = sum_r Left^T[r][row] Right[col][r]
// so each core is staged with a plain contiguous cp.async copy (no transposition), the partial products are
// kept transposed / untransposed as the next GEMM reads them, and one tile routine serves all three.
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 256;

// Packed FP32 pair (FFMA2, sm_100a).
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void fma2(unsigned long long& acc, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ float2 up(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ float4 lds4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ float lds1(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Contiguous copy of n floats global -> shared (16-byte pieces when both ends are aligned).
__device__ __forceinline__ void stage(float* dst, const float* src, int n) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
        for (int e = threadIdx.x; e < (n >> 2); e += blockDim.x) cp_async16(dst + 4 * e, src + 4 * e);
        for (int e = (n & ~3) + threadIdx.x; e < n; e += blockDim.x) cp_async4(dst + e, src + e);
    } else {
        for (int e = threadIdx.x; e < n; e += blockDim.x) cp_async4(dst + e, src + e);
    }
}

// Per-tile row state and per-column-tile column state of the store functors below.
struct RowSt {
    int m0, a, b;
};
struct ColSt {
    float* p;
    int a;   // < 0: column past N (nothing stored)
};

// Thread grid of one GEMM: txn = lx wx threads along m (4 rows each), tyn = (32 / lx) (8 / wx) along n (tm
// columns each, 4 or 5); a warp covers lx x (32 / lx) of it, so its At loads touch lx distinct 16-byte quads and
// its B loads 32 / lx distinct columns.  Chosen per product shape by a cost model: tiles x max(FFMA2 time,
// shared-memory wavefronts) per k, FFMA2 ~ tm and wavefronts ~ max(1, lx / 8) + tm / 4 max(1, ly / 8).
struct Grid {
    int lx, wx, tm;
};
// The 40 candidates (lx, wx, tm) are scored by the first 40 threads in parallel; *best (shared, initialised to
// ~0 by the caller before a barrier) receives the winner packed as cost << 8 | candidate.
__device__ __forceinline__ Grid grid_of(int c) { return Grid{1 << (c >> 3), 1 << ((c >> 1) & 3), 4 + (c & 1)}; }
__device__ __forceinline__ void score_grid(int M, int N, unsigned* best) {
    const int c = threadIdx.x;
    if (c >= 40) return;
    const Grid g = grid_of(c);
    const int ly = 32 / g.lx, txn = g.lx * g.wx, tyn = ly * (8 / g.wx), tm = g.tm;
    const int tiles = ((M + 4 * txn - 1) / (4 * txn)) * ((N + tyn * tm - 1) / (tyn * tm));
    // per-k cost in quarter units: FFMA2 4 tm; shared-memory wavefronts: the At load 2 (8 units), the B loads 2
    // each (4 when all 32 lanes read distinct columns, lx = 1), tm / 4 of them
    const int wf = 8 + (ly == 32 ? 4 : 2) * tm;
    atomicMin(best, ((unsigned)min(tiles * max(4 * tm, wf), 0xffffff) << 8) | (unsigned)c);
}

// out(m, n) = sum_{q < K} At[q lda + m] B[n ldb + q] for m < M, n < N.  Thread (tx, ty) of the grid owns
// m0 + {0..3} (m0 = mt + 4 tx, one 16-byte At load per q when lda % 4 == 0; At must be readable up to row
// m = 4 txn ceil(M / (4 txn)) - 1 < M + 512) and n = nt + ty + tyn b, b < TM (one 16-byte B load per 4 q when ldb, K % 4
// == 0; columns past N re-read column N - 1).  The m pairs accumulate with FFMA2 (the B value broadcast);
// st.row(m0) once per tile, then st(row state, n, v) stores the thread's 4 results of column n.
template <int TM, class Store>
__device__ __forceinline__ void tile_gemm(const Grid g, const float* At, int lda, const float* B, int ldb, int M,
                                          int N, int K, const Store& st) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, ly = 32 / g.lx;
    const int txn = g.lx * g.wx, tyn = ly * (8 / g.wx);
    // within the warp, tx from lane bits 1.. and ty from bit 0 and the bits above tx: each half-warp's At and B
    // addresses then come in adjacent-lane runs or alternate lane by lane, which LDS.128 serves in one wavefront
    // per half-warp (tools/lds_bench.cu; tx = lane & (lx - 1) would cost two for lx >= 4)
    int ltx = 0, lty = lane;
    if (g.lx > 1) {
        ltx = (lane >> 1) & (g.lx - 1);
        lty = (lane & 1) | ((lane >> (1 + __ffs(g.lx) - 1)) << 1);
    }
    const int tx = (warp % g.wx) * g.lx + ltx, ty = (warp / g.wx) * ly + lty;
    const bool vecA = (lda & 3) == 0, vecB = ((ldb | K) & 3) == 0;
    const uint32_t A0 = sa(At), B0 = sa(B);
    const int la = 4 * lda;   // bytes per q row of At
    // column tiles outer: the B addresses and the column halves of the output addresses are set once per column
    // tile and reused down all its row tiles
    for (int nt = 0; nt < N; nt += tyn * TM) {
        uint32_t bp[TM];
        ColSt cs[TM];
#pragma unroll
        for (int b2 = 0; b2 < TM; ++b2) {
            const int n = nt + ty + tyn * b2;
            bp[b2] = B0 + 4u * (uint32_t)(min(n, N - 1) * ldb);
            cs[b2] = n < N ? st.col(n) : ColSt{nullptr, -1};
        }
        for (int mt = 0; mt < M; mt += 4 * txn) {
            const int m0 = mt + 4 * tx;
            uint32_t ap = A0 + 4u * m0;
            unsigned long long acc[2][TM];
#pragma unroll
            for (int b2 = 0; b2 < TM; ++b2) acc[0][b2] = acc[1][b2] = 0ull;
            if (vecA && vecB) {
                for (int q = 0; q < K; q += 4, ap += 4 * la) {
                    float4 a4[4], b4[TM];
#pragma unroll
                    for (int u = 0; u < 4; ++u) a4[u] = lds4(ap + u * la);
#pragma unroll
                    for (int b2 = 0; b2 < TM; ++b2) b4[b2] = lds4(bp[b2] + 4 * q);
#pragma unroll
                    for (int b2 = 0; b2 < TM; ++b2) {
                        const float w[4] = {b4[b2].x, b4[b2].y, b4[b2].z, b4[b2].w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            fma2(acc[0][b2], pk(a4[u].x, a4[u].y), pk(w[u], w[u]));
                            fma2(acc[1][b2], pk(a4[u].z, a4[u].w), pk(w[u], w[u]));
                        }
                    }
                }
            } else {
                for (int q = 0; q < K; ++q, ap += la) {
                    float4 a;
                    if (vecA) a = lds4(ap);
                    else a = make_float4(lds1(ap), lds1(ap + 4), lds1(ap + 8), lds1(ap + 12));
#pragma unroll
                    for (int b2 = 0; b2 < TM; ++b2) {
                        const float w = lds1(bp[b2] + 4 * q);
                        fma2(acc[0][b2], pk(a.x, a.y), pk(w, w));
                        fma2(acc[1][b2], pk(a.z, a.w), pk(w, w));
                    }
                }
            }
            if (m0 >= M) continue;
            const auto rs = st.row(m0);
#pragma unroll
            for (int b2 = 0; b2 < TM; ++b2) {
                if (cs[b2].a < 0) continue;
                const float2 lo = up(acc[0][b2]), hi = up(acc[1][b2]);
                st(rs, cs[b2], make_float4(lo.x, lo.y, hi.x, hi.y));
            }
        }
    }
}
template <class Store>
__device__ __forceinline__ void gemm(const Grid g, const float* At, int lda, const float* B, int ldb, int M, int N,
                                     int K, const Store& st) {
    if (g.tm == 5) tile_gemm<5>(g, At, lda, B, ldb, M, N, K, st);
    else tile_gemm<4>(g, At, lda, B, ldb, M, N, K, st);
}

// Stores of the three GEMM kinds: row(m0) once per tile, col(n) once per column tile, then (row, col, v) for
// the thread's 4 results (rows m0..m0+3) of column n.  Rows m0 + u >= M are dropped.
struct StoreLeft {   // P'^T[s][row] (row stride ld), m = pr, n = i + I s; row = pr + prow i, or i + I pr (rev)
    float* out;
    int ld, prow, I, M;
    bool rev;
    __device__ __forceinline__ RowSt row(int m0) const { return RowSt{m0, m0 + 3 < M ? 4 : M - m0, 0}; }
    __device__ __forceinline__ ColSt col(int n) const {
        const int s = n / I, i = n - s * I;
        return ColSt{out + (size_t)s * ld + (rev ? i : prow * i), 0};
    }
    __device__ __forceinline__ void operator()(const RowSt& rs, const ColSt& c, float4 v) const {
        const float w[4] = {v.x, v.y, v.z, v.w};
        if (rev) {   // the new mode fastest: the 4 rows are I apart
            float* o = c.p + I * rs.m0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (u < rs.a) o[I * u] = w[u];
            return;
        }
        float* o = c.p + rs.m0;
        if (rs.a == 4 && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
            *reinterpret_cast<float4*>(o) = v;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (u < rs.a) o[u] = w[u];
        }
    }
};
struct StoreRight {  // Q'[i + I pc][r] (row stride R), m = r + R i, n = pc
    float* out;
    int R, I, M;
    __device__ __forceinline__ RowSt row(int m0) const {
        const int i0 = m0 / R;
        return RowSt{m0, i0, m0 - i0 * R};
    }
    __device__ __forceinline__ ColSt col(int n) const { return ColSt{out + (size_t)I * n * R, 0}; }
    __device__ __forceinline__ void operator()(const RowSt& rs, const ColSt& c, float4 v) const {
        const float w[4] = {v.x, v.y, v.z, v.w};
        if (rs.b + 3 < R) {   // the 4 rows lie in one row of Q' (M = R I, so m0 + 3 < M as well)
            float* o = c.p + (size_t)rs.a * R + rs.b;
            if ((reinterpret_cast<uintptr_t>(o) & 15u) == 0) { *reinterpret_cast<float4*>(o) = v; return; }
#pragma unroll
            for (int u = 0; u < 4; ++u) o[u] = w[u];
            return;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int m = rs.m0 + u;
            if (m >= M) break;
            const int i = m / R, r = m - i * R;
            c.p[(size_t)i * R + r] = w[u];
        }
    }
};
struct StoreD {      // out[offr[row] + offc[col]], m = row, n = col (streaming 16-byte stores when contiguous)
    float* out;
    const int32_t* offr;
    const int32_t* offc;
    int M;
    __device__ __forceinline__ RowSt row(int m0) const {   // (bit 31 of offr[m0], m0 % 4 == 0: rows m0..m0+3
        const int o = offr[m0];                                   //  contiguous, set by the kernel's setup pass)
        return RowSt{m0, o & 0x7fffffff, (int)((unsigned)o >> 31)};
    }
    __device__ __forceinline__ ColSt col(int n) const { return ColSt{out + offc[n], 0}; }
    __device__ __forceinline__ void operator()(const RowSt& rs, const ColSt& c, float4 v) const {
        float* o = c.p + rs.a;
        if (rs.b && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
            __stcs(reinterpret_cast<float4*>(o), v);
            return;
        }
        const float w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (rs.m0 + u < M) __stcs(c.p + (offr[rs.m0 + u] & 0x7fffffff), w[u]);
    }
};

__global__ void __launch_bounds__(kThreads, 2) reconstruct_kernel(const ReconArgs a) {
    extern __shared__ float sm[];
    __shared__ int32_t rk[TTC_MAX_ORDER + 1];
    __shared__ int64_t co[TTC_MAX_ORDER + 1];
    __shared__ unsigned gsel[2];                // packed grid choices (score_grid), alternating between GEMMs
    const int b = blockIdx.x, N = a.N, k = a.k;
    for (int n = threadIdx.x; n <= N; n += blockDim.x)
        rk[n] = (n == 0 || n == N) ? 1 : (a.t.ranks ? a.t.ranks[(int64_t)b * (N + 1) + n] : a.t.urank);
    __syncthreads();
    const int rows = a.rows, cols = a.cols;
    int gi = 0;                                 // gsel slot of the next GEMM
    if (threadIdx.x == 0) {
        gsel[0] = gsel[1] = ~0u;
        co[0] = 0;
        for (int n = 0; n < N; ++n) co[n + 1] = co[n] + (int64_t)rk[n] * a.dims[n] * rk[n + 1];
    }
    const float* G = a.t.cores + (a.t.offsets ? a.t.offsets[b] : (int64_t)b * a.t.train_elems);
    float* out = a.out + (a.out_offsets ? a.out_offsets[b] : (int64_t)b * a.pair_elems);
    float* L = sm;                          // Left^T: Rk x rows, row stride ldl; left partials likewise
    float* Rt = L + a.lbuf;                 // Right: [col][r], row stride Rk; right partials likewise
    float* T = Rt + a.rbuf;                 // Left's build temporary
    float* T2 = T + a.t1;                   // Right's build temporary
    int32_t* offr = reinterpret_cast<int32_t*>(T2 + a.t2);
    int32_t* offc = offr + rows;
    float* XS = reinterpret_cast<float*>(offc + cols);   // the staged core of the current build step
    XS = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(XS) + 15) & ~uintptr_t(15));
    // output offsets of the row / column multi-indices (permuted Eq. 2 strides)
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        int64_t o = 0;
        int q = r;
        if (a.lrev) {   // rows enumerate the left modes big-endian (mode k fastest)
            for (int n = k - 1; n >= 0; --n) { const int i = q % a.dims[n]; q /= a.dims[n]; o += (int64_t)i * a.ostride[n]; }
        } else {
            for (int n = 0; n < k; ++n) { const int i = q % a.dims[n]; q /= a.dims[n]; o += (int64_t)i * a.ostride[n]; }
        }
        offr[r] = (int32_t)o;
    }
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
        int64_t o = 0;
        int q = c;
        for (int n = k; n < N; ++n) { const int i = q % a.dims[n]; q /= a.dims[n]; o += (int64_t)i * a.ostride[n]; }
        offc[c] = (int32_t)o;
    }
    __syncthreads();
    // row quads m0 = 4t whose four output rows are consecutive: flagged in bit 31 of offr[m0] (offsets < 2^31), so
    // the D epilogue decides a 16-byte store with one shared load instead of four
    for (int t = threadIdx.x; 4 * t + 3 < rows; t += blockDim.x) {
        const int m0 = 4 * t, o0 = offr[m0];
        if (offr[m0 + 1] == o0 + 1 && offr[m0 + 2] == o0 + 2 && offr[m0 + 3] == o0 + 3)
            offr[m0] = (int32_t)((unsigned)o0 | 0x80000000u);
    }
    __syncthreads();
    const int Rk = rk[k];
    // ---- Left: P_1^T[s][i] = X_1[0, i, s] (as stored), then P_{j+1}^T = GEMM(P_j^T, X_j) for j = 2..k
    {
        float* cur = (k % 2 == 1) ? L : T;  // k - 1 products follow: alternate so the last writes L
        int prow = a.dims[0], ld = a.ld[0];
        const float* X1 = G + co[0];
        for (int e = threadIdx.x; e < prow * rk[1]; e += blockDim.x) {
            const int s = e / prow, i = e - s * prow;
            cur[s * ld + i] = __ldg(X1 + e);
        }
        for (int j = 1; j < k; ++j) {
            const int R = rk[j], S = rk[j + 1], I = a.dims[j];
            stage(XS, G + co[j], R * I * S);   // [i + I s][r]
            score_grid(prow, I * S, &gsel[gi]);
            cp_wait_all();
            __syncthreads();                   // cur and XS ready
            float* nxt = (cur == L) ? T : L;
            const int nld = a.ld[j];
            const Grid g = grid_of(gsel[gi] & 255u);
            if (threadIdx.x == 0) gsel[gi ^ 1] = ~0u;   // the slot after next is reset behind the next barrier
            gi ^= 1;
            gemm(g, cur, ld, XS, R, prow, I * S, R, StoreLeft{nxt, nld, prow, I, prow, a.lrev != 0});
            __syncthreads();                   // XS free, nxt complete
            cur = nxt;
            prow *= I;
            ld = nld;
        }
    }
    // ---- Right: Q_N[i][r] = X_N[r, i, 0] (as stored), then Q_j = GEMM(X_j^T, Q_{j+1}) for j = N-1..k+1
    if (k == N) {                           // N = 1: no right block, Right = [1]
        if (threadIdx.x == 0) Rt[0] = 1.f;
    } else {
        const int nR = N - k;
        float* cur = (nR % 2 == 1) ? Rt : T2;
        int pcol = a.dims[N - 1];
        const float* XN = G + co[N - 1];
        for (int e = threadIdx.x; e < pcol * rk[N - 1]; e += blockDim.x) cur[e] = __ldg(XN + e);
        for (int j = N - 2; j >= k; --j) {
            const int R = rk[j], S = rk[j + 1], I = a.dims[j];
            stage(XS, G + co[j], R * I * S);   // [s][r + R i]
            score_grid(R * I, pcol, &gsel[gi]);
            cp_wait_all();
            __syncthreads();
            float* nxt = (cur == Rt) ? T2 : Rt;
            const Grid g = grid_of(gsel[gi] & 255u);
            if (threadIdx.x == 0) gsel[gi ^ 1] = ~0u;
            gi ^= 1;
            gemm(g, XS, R * I, cur, S, R * I, pcol, S, StoreRight{nxt, R, I, R * I});
            __syncthreads();
            cur = nxt;
            pcol *= I;
        }
    }
    score_grid(rows, cols, &gsel[gi]);
    __syncthreads();
    // ---- D = Left Right, written through the permuted output offsets
    gemm(grid_of(gsel[gi] & 255u), L, a.ldl, Rt, Rk, rows, cols, Rk, StoreD{out, offr, offc, rows});
}

}  // namespace

cudaError_t launch_reconstruct(const ReconArgs& a, size_t smem_bytes, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(reconstruct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    reconstruct_kernel<<<a.B, kThreads, smem_bytes, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ttc
