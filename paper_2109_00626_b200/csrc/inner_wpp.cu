// inner_wpp.cu -- tt_inner, one warp per pair, for bond ranks <= 32 (BASELINE.json C5: N = 64, I = 2, ranks drawn
// from {8, 16, 24, 32} per bond; also C1).  Same sweep as ttc.h:
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :],  out = Z_N.
// Long trains of small steps: any per-step barrier or sub-KB TMA copy would dominate, so every warp works
// alone on its own pair:
//   * staging: the warp prefetches its own future steps with 16-byte cp.async into a private ring in shared
//     memory (cores packed back to back, several steps deep), one commit group per step;
//   * the rank products run on the tensor cores (3xTF32 mma.sync m16n8k8) with the cheaper association per
//     step (W-first: F = Y, G = X; V-first: F = X, G = Y), padded to 16-row / 8-col tiles;
//   * Z lives in a private 32 x 33 scratch tile in canonical orientation (X bond fastest): each step reads its
//     B fragments in whatever orientation its association needs and writes Z' back.
// Numerics as inner_fast.cu: B operands and core values split round-to-nearest, each tensor-core group of at
// most two k8 blocks added to fp32 with a round-to-nearest FADD.
#include <algorithm>
#include <cstdio>

#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

using namespace tc;

constexpr int kWarps = 4;     // warps per CTA (independent)
constexpr int kZS = 33;       // scratch row stride
constexpr int kDepth = 4;     // steps in flight per warp (issued, not yet computed)

struct WppArgs {
    int ring;        // floats of one warp's ring
    int warp_floats; // ring + Z scratch + in-flight queue
};

__device__ __forceinline__ void cp16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait(int pending) {
    switch (pending) {   // wait until at most `pending` of this thread's newest groups are still in flight
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    }
}

__device__ __forceinline__ int wrank(const TrainDev& t, int b, int N, int n) {
    if (n == 0 || n == N) return 1;
    return t.ranks ? __ldg(t.ranks + (int64_t)b * (N + 1) + n) : t.urank;
}
__device__ __forceinline__ int64_t wbase(const TrainDev& t, int b) {
    return t.offsets ? __ldg(t.offsets + b) : (int64_t)b * t.train_elems;
}

// A fragment of a core packed in shared memory (element [u, i, v] at u + Ga (i + I v)):
//   a0 = G[u0+2t, i, v0+g]  a1 = G[u0+2t, i, v0+g+8]  a2 = G[u0+2t+1, i, v0+g]  a3 = G[u0+2t+1, i, v0+g+8]
__device__ __forceinline__ AFrag wpp_afrag(const float* G, int Ga, int Gb, int I, int i, int u0, int v0, int g, int t) {
    const int u = u0 + 2 * t, v1 = v0 + g, v2 = v1 + 8;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    if (u < Ga) {
        if ((Ga & 1) == 0) {   // u even and Ga even: (u, u+1) both in range and 8-byte aligned
            if (v1 < Gb) { const float2 x = *reinterpret_cast<const float2*>(G + u + Ga * (i + I * v1)); a[0] = x.x; a[2] = x.y; }
            if (v2 < Gb) { const float2 x = *reinterpret_cast<const float2*>(G + u + Ga * (i + I * v2)); a[1] = x.x; a[3] = x.y; }
        } else {
            const bool u1 = u + 1 < Ga;
            if (v1 < Gb) { a[0] = G[u + Ga * (i + I * v1)]; if (u1) a[2] = G[u + 1 + Ga * (i + I * v1)]; }
            if (v2 < Gb) { a[1] = G[u + Ga * (i + I * v2)]; if (u1) a[3] = G[u + 1 + Ga * (i + I * v2)]; }
        }
    }
    AFrag f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f.hi[k] = hi_bits(a[k]);
        f.lo[k] = lo_bits(a[k], f.hi[k]);
    }
    return f;
}

// One step of one pair for one warp.  F: core multiplied into Z first (Fa x I x Fb), G: the other (Ga x I x Gb).
// zs: canonical Z (x + kZS y); vf: V-first (then Z[g, f] = zs[f + kZS g], else zs[g + kZS f]).
__device__ __forceinline__ void wpp_step(const float* F, int Fa, int Fb, const float* G, int Ga, int Gb, int I, bool vf,
                                         float* zs, int lane) {
    const int lg = lane >> 2, t = lane & 3;
    const int kf_n = (Fa + 7) >> 3, ng_n = (Ga + 7) >> 3, mq_n = (Fb + 15) >> 4, mg_n = (Gb + 15) >> 4;
    float acc[2][4][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[m][q][c] = 0.f;
    for (int i = 0; i < I; ++i) {
        // ---- GEMM-1: w[mq][ng] = sum_kf A_F(i, mq, kf) B_Z(kf, ng), B_Z(kf, ng) = Z[g = 8ng + lg, f = 8kf + 2t + j]
        float w[2][4][4];
#pragma unroll
        for (int mq = 0; mq < 2; ++mq)
#pragma unroll
            for (int ng = 0; ng < 4; ++ng)
#pragma unroll
                for (int c = 0; c < 4; ++c) w[mq][ng][c] = 0.f;
#pragma unroll
        for (int kp = 0; kp < 4; kp += 2) {
            if (kp >= kf_n) break;
            float tg[2][4][4];
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
                const int kf = kp + sub;
                if (kf >= kf_n) break;
                BFrag zb[4];
#pragma unroll
                for (int ng = 0; ng < 4; ++ng) {
                    if (ng >= ng_n) break;
                    const int gg = 8 * ng + lg, f0 = 8 * kf + 2 * t;
                    float z0 = 0.f, z1 = 0.f;
                    if (gg < Ga) {
                        if (f0 < Fa) z0 = vf ? zs[f0 + kZS * gg] : zs[gg + kZS * f0];
                        if (f0 + 1 < Fa) z1 = vf ? zs[f0 + 1 + kZS * gg] : zs[gg + kZS * (f0 + 1)];
                    }
                    zb[ng] = split_b(z0, z1);
                }
#pragma unroll
                for (int mq = 0; mq < 2; ++mq) {
                    if (mq >= mq_n) break;
                    const AFrag A = wpp_afrag(F, Fa, Fb, I, i, 8 * kf, 16 * mq, lg, t);
#pragma unroll
                    for (int ng = 0; ng < 4; ++ng) {
                        if (ng >= ng_n) break;
                        if (sub == 0) mma3<true>(tg[mq][ng], A, zb[ng]);
                        else mma3<false>(tg[mq][ng], A, zb[ng]);
                    }
                }
            }
#pragma unroll
            for (int mq = 0; mq < 2; ++mq)
#pragma unroll
                for (int ng = 0; ng < 4; ++ng)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (mq < mq_n && ng < ng_n) w[mq][ng][c] += tg[mq][ng][c];
        }
        // ---- GEMM-2: acc[mg][nf] += sum_kg A_G(i, mg, kg) B_W(kg, nf), B_W(kg, nf) = w[nf/2][kg][2 (nf%2) + j]
#pragma unroll
        for (int kp = 0; kp < 4; kp += 2) {
            if (kp >= ng_n) break;
            float tg[2][4][4];
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
                const int kg = kp + sub;
                if (kg >= ng_n) break;
                BFrag Bw[4];
#pragma unroll
                for (int nf = 0; nf < 4; ++nf) Bw[nf] = split_b(w[nf >> 1][kg][2 * (nf & 1)], w[nf >> 1][kg][2 * (nf & 1) + 1]);
#pragma unroll
                for (int mg = 0; mg < 2; ++mg) {
                    if (mg >= mg_n) break;
                    const AFrag A = wpp_afrag(G, Ga, Gb, I, i, 8 * kg, 16 * mg, lg, t);
#pragma unroll
                    for (int nf = 0; nf < 4; ++nf) {
                        if (8 * nf >= Fb) break;
                        if (sub == 0) mma3<true>(tg[mg][nf], A, Bw[nf]);
                        else mma3<false>(tg[mg][nf], A, Bw[nf]);
                    }
                }
            }
#pragma unroll
            for (int mg = 0; mg < 2; ++mg)
#pragma unroll
                for (int nf = 0; nf < 4; ++nf)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (mg < mg_n && 8 * nf < Fb) acc[mg][nf][c] += tg[mg][nf][c];
        }
    }
    __syncwarp();   // every lane has read the old Z
    // ---- Z'[g', f'] -> canonical scratch (g' on G's right bond, f' on F's right bond)
#pragma unroll
    for (int mg = 0; mg < 2; ++mg)
#pragma unroll
        for (int nf = 0; nf < 4; ++nf)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int gg = 16 * mg + lg + 8 * (c >> 1), ff = 8 * nf + 2 * t + (c & 1);
                if (gg < Gb && ff < Fb) zs[vf ? (ff + kZS * gg) : (gg + kZS * ff)] = acc[mg][nf][c];
            }
    __syncwarp();
}

// Per-warp cursor over this warp's (pair, step) sequence.
struct WCursor {
    int k, b, n, R, P;
    int64_t xo, yo;
    bool valid;
};
__device__ __forceinline__ void wc_pair(const InnerArgs& a, WCursor& c, int gw, int nw) {
    const int idx = gw + c.k * nw;
    c.valid = idx < a.B;
    if (!c.valid) return;
    c.b = a.order ? __ldg(a.order + idx) : idx;
    c.n = 0;
    c.R = 1;
    c.P = 1;
    c.xo = wbase(a.x, c.b);
    c.yo = wbase(a.y, c.b);
}

struct InFlight {
    int start;          // ring offset (floats) of X, Y follows
    int b, n, R, P, S, Q, I;
    unsigned end;       // monotone ring position after this step
};

__global__ void __launch_bounds__(32 * kWarps) inner_wpp_kernel(const InnerArgs a, const WppArgs w) {
    extern __shared__ __align__(16) float smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* ring = smem + warp * w.warp_floats;
    float* zs = ring + w.ring;
    InFlight* q = reinterpret_cast<InFlight*>(zs + ((32 * kZS + 3) & ~3));   // kDepth entries, warp-private
    const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
    WCursor ic;
    ic.k = 0;
    wc_pair(a, ic, gw, nw);
    unsigned head = 0, tail = 0;   // monotone ring positions (floats)
    int qh = 0, qn = 0;            // in-flight queue: oldest entry index, count
    const unsigned RING = (unsigned)w.ring;
    while (true) {
        // ---- issue future steps while they fit
        while (ic.valid && qn < kDepth) {
            const int I = a.dims[ic.n];
            const int S = wrank(a.x, ic.b, a.N, ic.n + 1), Q = wrank(a.y, ic.b, a.N, ic.n + 1);
            const int nx = ic.R * I * S, ny = ic.P * I * Q;
            const unsigned need = (unsigned)((nx + 3) & ~3) + (unsigned)((ny + 3) & ~3);
            unsigned start = head;
            if ((start % RING) + need > RING) start = (start / RING + 1) * RING;   // do not wrap a step
            if (qn == 0) tail = start;                                              // empty ring: the skip is free
            if (start + need - tail > RING) break;                                  // no room yet
            float* dst = ring + (start % RING);
            const float* xs = a.x.cores + ic.xo;
            const float* ys = a.y.cores + ic.yo;
            const int nxp = (nx + 3) & ~3;
            if (((nx | ny) & 3) == 0 && ((reinterpret_cast<uintptr_t>(xs) | reinterpret_cast<uintptr_t>(ys)) & 15u) == 0) {
                for (int e = 4 * lane; e < nx; e += 128) cp16(dst + e, xs + e);
                for (int e = 4 * lane; e < ny; e += 128) cp16(dst + nxp + e, ys + e);
            } else {   // unaligned core sizes (rank-1 boundaries with odd I): plain copies, visible after syncwarp
                for (int e = lane; e < nx; e += 32) dst[e] = __ldg(xs + e);
                for (int e = lane; e < ny; e += 32) dst[nxp + e] = __ldg(ys + e);
            }
            cp_commit();
            if (lane == 0) {
                InFlight f;
                f.start = (int)(start % RING);
                f.b = ic.b; f.n = ic.n; f.R = ic.R; f.P = ic.P; f.S = S; f.Q = Q; f.I = I;
                f.end = start + need;
                q[(qh + qn) % kDepth] = f;
            }
            ++qn;
            head = start + need;
            ic.xo += nx;
            ic.yo += ny;
            ic.R = S;
            ic.P = Q;
            if (++ic.n == a.N) {
                ++ic.k;
                wc_pair(a, ic, gw, nw);
            }
        }
        if (qn == 0) break;
        // ---- compute the oldest step
        cp_wait(qn - 1);
        __syncwarp();
        const InFlight f = q[qh];
        const float* X = ring + f.start;
        const float* Y = X + ((f.R * f.I * f.S + 3) & ~3);
        if (f.n == 0) {   // Z_0 = [1]
            if (lane == 0) zs[0] = 1.0f;
            __syncwarp();
        }
        const bool vf = (f.R * f.P * f.S + f.P * f.S * f.Q) < (f.R * f.P * f.Q + f.R * f.S * f.Q);
        if (vf) wpp_step(X, f.R, f.S, Y, f.P, f.Q, f.I, true, zs, lane);
        else wpp_step(Y, f.P, f.Q, X, f.R, f.S, f.I, false, zs, lane);
#ifdef TTC_WPP_DEBUG
        if (lane == 0 && f.b == 0)
            printf("n=%d R=%d P=%d S=%d Q=%d I=%d start=%d end=%u head=%u tail=%u qn=%d vf=%d z00=%g\n", f.n, f.R, f.P, f.S,
                   f.Q, f.I, f.start, f.end, head, tail, qn, (int)vf, zs[0]);
#endif
        if (f.n == a.N - 1 && lane == 0) a.out[f.b] = zs[0];
        __syncwarp();
        tail = f.end;
        qh = (qh + 1) % kDepth;
        --qn;
    }
    cp_wait(0);
}

}  // namespace

// Ring sized for the largest step of the batch (X + Y cores) and at least twice the average.
// Ring of max(max step + 8, 4096) floats: at least one step of the largest shape, typically two to three of C5's.
static int64_t wpp_ring(int max_rank, int max_dim) {
    const int64_t max_step = 2 * (int64_t)max_rank * max_dim * max_rank + 8;
    return (std::max<int64_t>(max_step, 4096) + 3) & ~3;
}

bool inner_wpp_supported(const InnerArgs& a, int max_rank) {
    if (max_rank > 32 || a.N < 1) return false;
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = std::max(max_dim, (int)a.dims[n]);
    const int64_t warp_floats = wpp_ring(max_rank, max_dim) + ((32 * kZS + 3) & ~3) + kDepth * (int64_t)sizeof(InFlight) / 4;
    return sizeof(float) * warp_floats * kWarps <= 200 * 1024;
}

cudaError_t launch_inner_wpp(const InnerArgs& a, int max_rank, cudaStream_t s) {
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = std::max(max_dim, (int)a.dims[n]);
    WppArgs w;
    w.ring = (int)wpp_ring(max_rank, max_dim);
    w.warp_floats = w.ring + ((32 * kZS + 3) & ~3) + (int)(kDepth * sizeof(InFlight) / 4);
    const size_t smem = sizeof(float) * (size_t)w.warp_floats * kWarps;
    cudaError_t e = cudaFuncSetAttribute(inner_wpp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_wpp_kernel, 32 * kWarps, smem)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int want = (a.B + kWarps - 1) / kWarps;
    const int grid = want < sms * per_sm ? want : sms * per_sm;
    inner_wpp_kernel<<<grid, 32 * kWarps, smem, s>>>(a, w);
    return cudaGetLastError();
}

}  // namespace ttc
