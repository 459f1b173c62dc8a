// splice.cu -- the paper's TTCP construction for a pair of end modes (ttc.h: ttc_splice_plan_create; Alg. 2
// steps 4-5, on TT operands): K = A_x^T A_y (Eq. 12), then the output chain
//   [X free cores (reversed and rank-transposed when n = 1)]  K  [Y free cores (reversed when m = M)]
// with K absorbed into the next core (else the previous one).  One CTA per pair: K in shared memory, then every
// output core streamed in Eq. 2 order (consecutive threads write consecutive elements; reversed cores gather
// their source, which is small and L1/L2-resident; the absorbing core is a sum over K's inner bond).  Output
// bytes ~ input bytes: bound by HBM traffic, not arithmetic.
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 128;
constexpr int kMagicMax = 4096;

// c_div[d] = ceil(2^32 / d): n / d == __umulhi(n, c_div[d]) for n < 2^32 / d (d >= 2); d = 1 handled apart.
struct DivTable {
    unsigned v[kMagicMax + 1];
    constexpr DivTable() : v() {
        for (int d = 2; d <= kMagicMax; ++d) v[d] = (unsigned)((0x100000000ull + d - 1) / d);
    }
};
__constant__ DivTable c_div = DivTable();


// One output core, prepared per pair by thread l (core l): the (reversed) source core C[u, i, v] (A x Id x B)
// at src + cu u + ci i + cv v; kind 0 copy, 1 rank-transposed copy, 2 K absorbed from the left, 3 K absorbed
// from the right.
struct CoreDesc {
    int64_t soff;
    int32_t fromx, kind, A, Id, B, cu, ci, cv, tot;
    uint32_t mdiv0, mdiv1;   // magic divisors of the element decomposition (e / rows, col / Id)
};

struct SpliceCtx {
    int32_t rx[kMaxContractOrder + 1], ry[kMaxContractOrder + 1];
    int64_t xo[kMaxContractOrder + 1], yo[kMaxContractOrder + 1];
    CoreDesc cd[kMaxLadder];
};

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
// Contiguous copy of n floats global -> shared (16-byte pieces when both ends are aligned).
__device__ __forceinline__ void stage(float* dst, const float* src, int n) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
        for (int e = threadIdx.x; e < (n >> 2); e += blockDim.x) cp_async16(dst + 4 * e, src + 4 * e);
        for (int e = (n & ~3) + threadIdx.x; e < n; e += blockDim.x) cp_async4(dst + e, src + e);
    } else {
        for (int e = threadIdx.x; e < n; e += blockDim.x) cp_async4(dst + e, src + e);
    }
}

// Loads of the cores: from the staged shared copy, or through the read-only path from global memory.
template <bool STAGED>
__device__ __forceinline__ float ldc(const float* p) {
    if (STAGED) return *p;
    return __ldg(p);
}

template <bool STAGED>
__device__ __forceinline__ void splice_body(const SpliceArgs& a, SpliceCtx& c, const float* xg, const float* yg,
                                            float* Ks, float* out) {
    // ---- step 4: K[r, p] = sum_i A_x[i, r] A_y[i, p]  (Eq. 12)
    const int Rk = a.n == 1 ? c.rx[1] : c.rx[a.N - 1], Pk = a.m == 1 ? c.ry[1] : c.ry[a.M - 1];
    const int I = a.xdims[a.n - 1];
    const float* Ax = xg + c.xo[a.n - 1];   // n = 1: [0, i, r] at i + I r;   n = N: [r, i, 0] at r + Rk i
    const float* Ay = yg + c.yo[a.m - 1];
    for (int e = threadIdx.x; e < Rk * Pk; e += blockDim.x) {
        const int r = e % Rk, p = e / Rk;
        float acc = 0.f;
        for (int i = 0; i < I; ++i) {
            const float u = a.n == 1 ? ldc<STAGED>(Ax + i + I * r) : ldc<STAGED>(Ax + r + Rk * i);
            const float v = a.m == 1 ? ldc<STAGED>(Ay + i + I * p) : ldc<STAGED>(Ay + p + Pk * i);
            acc = fmaf(u, v, acc);
        }
        Ks[e] = acc;
    }
    __syncthreads();
    if (a.L == 0) {   // N = M = 1: the scalar K
        if (threadIdx.x == 0) out[0] = Ks[0];
        return;
    }
    // ---- step 5: the output chain (element e = row + rows (i + Id col'): e / rows and col / Id by IMAD.HI),
    // streaming stores (the output is not re-read by this kernel)
    int64_t doff = 0;
    for (int l = 0; l < a.L; ++l) {
        const CoreDesc& d = c.cd[l];
        const float* G = (d.fromx ? xg : yg) + d.soff;
        float* dst = out + doff;
        const int tot = d.tot, kind = d.kind, Id = d.Id;
        doff += tot;
        if (kind == 0) {                                   // plain copy of the core
            if (((reinterpret_cast<uintptr_t>(G) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0 && (tot & 3) == 0) {
                const float4* g4 = reinterpret_cast<const float4*>(G);
                float4* d4 = reinterpret_cast<float4*>(dst);
                for (int e = threadIdx.x; e < tot / 4; e += blockDim.x) __stcs(d4 + e, STAGED ? g4[e] : __ldg(g4 + e));
            } else {
                for (int e = threadIdx.x; e < tot; e += blockDim.x) __stcs(dst + e, ldc<STAGED>(G + e));
            }
            continue;
        }
        const int rows = kind == 2 ? Rk : d.A;
        const unsigned m0 = d.mdiv0, m1 = d.mdiv1;
        const int cu = d.cu, ci = d.ci, cv = d.cv;
        if ((rows & 3) == 0 && (Rk & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
            // 4 consecutive rows of one column per thread: the index math, the K column (kind 2) or row (kind 3)
            // and the C fibre (kind 2) are shared by the 4 outputs; one 16-byte streaming store
            for (int e = 4 * threadIdx.x; e < tot; e += 4 * blockDim.x) {
                const int col = m0 ? (int)__umulhi((unsigned)e, m0) : e, row = e - col * rows;
                const int w = m1 ? (int)__umulhi((unsigned)col, m1) : col, i = col - w * Id;
                float v[4];
                if (kind == 1) {
                    const float* g = G + cu * row + ci * i + cv * w;
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = ldc<STAGED>(g + cu * u);
                } else if (kind == 2) {
                    const float* g = G + ci * i + cv * w;
                    v[0] = v[1] = v[2] = v[3] = 0.f;
                    for (int p = 0; p < d.A; ++p) {
                        const float gp = ldc<STAGED>(g + cu * p);
                        const float4 k4 = *reinterpret_cast<const float4*>(Ks + row + Rk * p);
                        v[0] = fmaf(k4.x, gp, v[0]); v[1] = fmaf(k4.y, gp, v[1]);
                        v[2] = fmaf(k4.z, gp, v[2]); v[3] = fmaf(k4.w, gp, v[3]);
                    }
                } else {
                    const float* g = G + cu * row + ci * i;
                    v[0] = v[1] = v[2] = v[3] = 0.f;
                    for (int r = 0; r < d.B; ++r) {
                        const float kr = Ks[r + Rk * w];
#pragma unroll
                        for (int u = 0; u < 4; ++u) v[u] = fmaf(ldc<STAGED>(g + cu * u + cv * r), kr, v[u]);
                    }
                }
                __stcs(reinterpret_cast<float4*>(dst + e), make_float4(v[0], v[1], v[2], v[3]));
            }
            continue;
        }
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
            const int col = m0 ? (int)__umulhi((unsigned)e, m0) : e, row = e - col * rows;
            const int w = m1 ? (int)__umulhi((unsigned)col, m1) : col, i = col - w * Id;
            float v;
            if (kind == 1) {                               // rank-transposed copy: [u, i, v] = G[v, i, u]
                v = ldc<STAGED>(G + cu * row + ci * i + cv * w);
            } else if (kind == 2) {                        // sum_p K[r, p] C[p, i, w]   (A == Pk)
                const float* g = G + ci * i + cv * w;
                v = 0.f;
                for (int p = 0; p < d.A; ++p) v = fmaf(Ks[row + Rk * p], ldc<STAGED>(g + cu * p), v);
            } else {                                       // sum_r C[u, i, r] K[r, w]   (B == Rk)
                const float* g = G + cu * row + ci * i;
                v = 0.f;
                for (int r = 0; r < d.B; ++r) v = fmaf(ldc<STAGED>(g + cv * r), Ks[r + Rk * w], v);
            }
            __stcs(dst + e, v);
        }
    }
}

__global__ void __launch_bounds__(kThreads) splice_kernel(const SpliceArgs a) {
    extern __shared__ __align__(16) float sm[];
    __shared__ SpliceCtx c;
    const int b = blockIdx.x, N = a.N, M = a.M;
    // ranks and core offsets of both trains (two warps in parallel)
    for (int k = threadIdx.x; k <= N; k += blockDim.x)
        c.rx[k] = a.x.ranks ? a.x.ranks[(int64_t)b * (N + 1) + k] : ((k == 0 || k == N) ? 1 : a.x.urank);
    for (int k = threadIdx.x; k <= M; k += blockDim.x)
        c.ry[k] = a.y.ranks ? a.y.ranks[(int64_t)b * (M + 1) + k] : ((k == 0 || k == M) ? 1 : a.y.urank);
    __syncthreads();
    if (threadIdx.x == 0) {
        c.xo[0] = 0;
        for (int k = 0; k < N; ++k) c.xo[k + 1] = c.xo[k] + (int64_t)c.rx[k] * a.xdims[k] * c.rx[k + 1];
    } else if (threadIdx.x == 32) {
        c.yo[0] = 0;
        for (int k = 0; k < M; ++k) c.yo[k + 1] = c.yo[k] + (int64_t)c.ry[k] * a.ydims[k] * c.ry[k + 1];
    }
    __syncthreads();
    const float* xg = a.x.cores + (a.x.offsets ? a.x.offsets[b] : (int64_t)b * a.x.train_elems);
    const float* yg = a.y.cores + (a.y.offsets ? a.y.offsets[b] : (int64_t)b * a.y.train_elems);
    float* out = a.out + (a.out_offsets ? a.out_offsets[b] : (int64_t)b * a.out_pair_elems);
    float* Ks = sm;                                          // K: Rk x Pk, column-major
    float* xs = sm + a.k4;                                   // the staged trains (stage_x, stage_y floats)
    float* ys = xs + a.stage_x;
    if (a.stage_x) {   // one round trip for all of the pair's loads
        stage(xs, xg, (int)c.xo[N]);
        stage(ys, yg, (int)c.yo[M]);
    }
    // output core descriptors, one thread per core
    for (int l = threadIdx.x; l < a.L; l += blockDim.x) {
        CoreDesc& d = c.cd[l];
        const bool xsrc = a.src[l] > 0;
        const int s = (xsrc ? a.src[l] : -a.src[l]) - 1;
        const int32_t* rr = xsrc ? c.rx : c.ry;
        const int a0 = rr[s], Id = xsrc ? a.xdims[s] : a.ydims[s], b0 = rr[s + 1];
        const bool rv = a.rev[l] != 0;
        const int Rk = a.n == 1 ? c.rx[1] : c.rx[N - 1], Pk = a.m == 1 ? c.ry[1] : c.ry[M - 1];
        d.fromx = xsrc;
        d.soff = xsrc ? c.xo[s] : c.yo[s];
        d.A = rv ? b0 : a0;
        d.B = rv ? a0 : b0;
        d.Id = Id;
        d.cu = rv ? a0 * Id : 1;
        d.ci = a0;
        d.cv = rv ? 1 : a0 * Id;
        d.kind = l == a.nx ? 2 : (a.nx == a.L && l == a.L - 1) ? 3 : (rv ? 1 : 0);
        const int rows = d.kind == 2 ? Rk : d.A, cols = d.kind == 3 ? Pk : d.B;
        d.tot = rows * Id * cols;
        d.mdiv0 = rows >= 2 ? c_div.v[rows] : 0u;
        d.mdiv1 = Id >= 2 ? c_div.v[Id] : 0u;
    }
    if (a.stage_x) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        splice_body<true>(a, c, xs, ys, Ks, out);
    } else {
        __syncthreads();
        splice_body<false>(a, c, xg, yg, Ks, out);
    }
}

}  // namespace

cudaError_t launch_splice(const SpliceArgs& a, size_t smem_bytes, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(splice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    splice_kernel<<<a.B, kThreads, smem_bytes, s>>>(a);
    return cudaGetLastError();
}

}  // namespace ttc
