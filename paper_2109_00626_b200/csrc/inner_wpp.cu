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
constexpr int kZsl = 32 * kZS; // offset of the lo half of the pre-split scratch
constexpr int kDepth = 4;     // steps in flight per warp (issued, not yet computed)
constexpr int kTail = 640;    // slack floats after a warp's region: unguarded reads of a partial M tile

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

// Full-tile variant of wpp_step for steps whose four bond ranks are multiples of 8 (C5's {8,16,24,32}):
// K blocks and N tiles are exact, so fragment loads, B reads and Z writes need no guards; rows of a 16-row
// M tile beyond the rank read padding / neighbouring data that only reaches output rows never read (the warp's
// region is followed by kTail floats of slack so such reads stay inside shared memory).  Tiles are skipped by
// warp-uniform branches, never by per-element predicates.
__device__ __forceinline__ AFrag wpp_afrag_full(const float* G, int Ga, int I, int i, int u0, int v0, int g, int t) {
    const float* p1 = G + u0 + 2 * t + Ga * (i + I * (v0 + g));
    const float* p2 = p1 + Ga * I * 8;
    const float2 x1 = *reinterpret_cast<const float2*>(p1);
    const float2 x2 = *reinterpret_cast<const float2*>(p2);
    AFrag f;
    const float a[4] = {x1.x, x2.x, x1.y, x2.y};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f.hi[k] = hi_bits(a[k]);
        f.lo[k] = lo_bits(a[k], f.hi[k]);
    }
    return f;
}

// U consecutive slices i0 .. i0+U-1 of a full-tile step in lockstep (the slices' GEMM chains are independent until
// they reach acc).  U = 1 is used: U = 2 spilled registers and measured slower on C5.
template <int U>
__device__ __forceinline__ void wpp_slices(const float* F, int Fa, const float* G, int Ga, int I, int i0, int kf_n, int ng_n,
                                           int mq_n, int mg_n, int nf_n, int sg, int sf, const uint32_t* zsh,
                                           const uint32_t* zsl, int lg, int t, float (&acc)[2][4][4]) {
    // ---- GEMM-1: w[x][mq][ng] = sum_kf A_F(i0+x, mq, kf) B_Z(kf, ng); two k-blocks per tensor-core group
    float w[U][2][4][4];
#pragma unroll
    for (int mq = 0; mq < 2; ++mq) {
        if (mq >= mq_n) break;
#pragma unroll
        for (int kp = 0; kp < 4; kp += 2) {
            if (kp >= kf_n) break;
            const bool two = kp + 1 < kf_n;
            AFrag A0[U], A1[U];
#pragma unroll
            for (int x = 0; x < U; ++x) {
                A0[x] = wpp_afrag_full(F, Fa, I, i0 + x, 8 * kp, 16 * mq, lg, t);
                A1[x] = A0[x];
                if (two) A1[x] = wpp_afrag_full(F, Fa, I, i0 + x, 8 * kp + 8, 16 * mq, lg, t);
            }
#pragma unroll
            for (int ng = 0; ng < 4; ++ng) {
                if (ng >= ng_n) break;
                const int gg = 8 * ng + lg, f0 = 8 * kp + 2 * t;
                const int i0z = gg * sg + f0 * sf, i1z = i0z + sf;
                BFrag B0, B1;
                B0.hi[0] = zsh[i0z]; B0.hi[1] = zsh[i1z]; B0.lo[0] = zsl[i0z]; B0.lo[1] = zsl[i1z];
                if (two) {
                    const int j0 = i0z + 8 * sf, j1 = j0 + sf;
                    B1.hi[0] = zsh[j0]; B1.hi[1] = zsh[j1]; B1.lo[0] = zsl[j0]; B1.lo[1] = zsl[j1];
                }
#pragma unroll
                for (int x = 0; x < U; ++x) {
                    float tg[4];
                    if (two) mma6<true>(tg, A0[x], B0, A1[x], B1);
                    else mma3<true>(tg, A0[x], B0);
#pragma unroll
                    for (int c = 0; c < 4; ++c) w[x][mq][ng][c] = (kp == 0) ? tg[c] : w[x][mq][ng][c] + tg[c];
                }
            }
        }
    }
    // ---- GEMM-2: acc[mg][nf] += sum_x sum_kg A_G(i0+x, mg, kg) B_W(x, kg, nf)
#pragma unroll
    for (int mg = 0; mg < 2; ++mg) {
        if (mg >= mg_n) break;
#pragma unroll
        for (int kp = 0; kp < 4; kp += 2) {
            if (kp >= ng_n) break;
            const bool two = kp + 1 < ng_n;
            AFrag A0[U], A1[U];
#pragma unroll
            for (int x = 0; x < U; ++x) {
                A0[x] = wpp_afrag_full(G, Ga, I, i0 + x, 8 * kp, 16 * mg, lg, t);
                A1[x] = A0[x];
                if (two) A1[x] = wpp_afrag_full(G, Ga, I, i0 + x, 8 * kp + 8, 16 * mg, lg, t);
            }
#pragma unroll
            for (int nf = 0; nf < 4; ++nf) {
                if (nf >= nf_n) break;
                float tg[U][4];
#pragma unroll
                for (int x = 0; x < U; ++x) {
                    const BFrag B0 = split_b(w[x][nf >> 1][kp][2 * (nf & 1)], w[x][nf >> 1][kp][2 * (nf & 1) + 1]);
                    if (two) {
                        const BFrag B1 = split_b(w[x][nf >> 1][kp + 1][2 * (nf & 1)], w[x][nf >> 1][kp + 1][2 * (nf & 1) + 1]);
                        mma6<true>(tg[x], A0[x], B0, A1[x], B1);
                    } else {
                        mma3<true>(tg[x], A0[x], B0);
                    }
                }
#pragma unroll
                for (int x = 0; x < U; ++x)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[mg][nf][c] += tg[x][c];
            }
        }
    }
}

// zsh / zsl: Z pre-split (hi, lo as the tensor core consumes them), written once per step.
__device__ __forceinline__ void wpp_step_full(const float* F, int Fa, int Fb, const float* G, int Ga, int Gb, int I,
                                              bool vf, uint32_t* zsh, uint32_t* zsl, int lane) {
    const int lg = lane >> 2, t = lane & 3;
    const int kf_n = Fa >> 3, ng_n = Ga >> 3, mq_n = (Fb + 15) >> 4, mg_n = (Gb + 15) >> 4, nf_n = Fb >> 3;
    // scratch index of Z[g, f]: W-first g + kZS f, V-first f + kZS g
    const int sg = vf ? kZS : 1, sf = vf ? 1 : kZS;
    float acc[2][4][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[m][q][c] = 0.f;
    for (int i = 0; i < I; ++i) wpp_slices<1>(F, Fa, G, Ga, I, i, kf_n, ng_n, mq_n, mg_n, nf_n, sg, sf, zsh, zsl, lg, t, acc);
    __syncwarp();   // every lane has read the old Z
    // ---- Z'[g', f'] -> canonical scratch, split once; rows g' >= Gb of a partial M tile are written too
#pragma unroll
    for (int mg = 0; mg < 2; ++mg) {
        if (mg >= mg_n) break;
#pragma unroll
        for (int nf = 0; nf < 4; ++nf) {
            if (nf >= nf_n) break;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int gg = 16 * mg + lg + 8 * (c >> 1), ff = 8 * nf + 2 * t + (c & 1);
                const uint32_t h = hi_bits(acc[mg][nf][c]);
                zsh[gg * sg + ff * sf] = h;
                zsl[gg * sg + ff * sf] = lo_bits(acc[mg][nf][c], h);
            }
        }
    }
    __syncwarp();
}

// Boundary steps on the FP32 pipe (rank-1 bonds make every tensor-core tile mostly padding).
// First step (R = P = 1): Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q] -- Eq. 12's K -- into the canonical scratch.
template <bool SPLIT>
__device__ __forceinline__ void wpp_first(const float* X, const float* Y, int S, int Q, int I, float* zs, int lane) {
    for (int e = lane; e < S * Q; e += 32) {
        const int sidx = e % S, q = e / S;
        float d = 0.f;
        for (int i = 0; i < I; ++i) d = fmaf(X[i + I * sidx], Y[i + I * q], d);
        if (SPLIT) {   // pre-split scratch: hi in zs, lo in zs + kZsl
            const uint32_t h = hi_bits(d);
            reinterpret_cast<uint32_t*>(zs)[sidx + kZS * q] = h;
            reinterpret_cast<uint32_t*>(zs)[kZsl + sidx + kZS * q] = lo_bits(d, h);
        } else {
            zs[sidx + kZS * q] = d;
        }
    }
    __syncwarp();
}
// Last step (S = Q = 1): Z_N = sum_{r,p} Z[r,p] sum_i X_N[r,i,0] Y_N[p,i,0] (warp-reduced, fixed order).
// With R = P = 1 (N == 1) this is the dot product sum_i x_i y_i.
template <bool SPLIT>
__device__ __forceinline__ float wpp_last(const float* X, const float* Y, int R, int P, int I, bool first, const float* zs,
                                          int lane) {
    float v = 0.f;
    for (int e = lane; e < R * P; e += 32) {
        const int r = e % R, p = e / R;
        float d = 0.f;
        for (int i = 0; i < I; ++i) d = fmaf(X[r + R * i], Y[p + P * i], d);
        float z = 1.0f;
        if (!first) z = SPLIT ? zs[r + kZS * p] + zs[kZsl + r + kZS * p] : zs[r + kZS * p];   // hi + lo = Z exactly
        v = fmaf(z, d, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
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

template <bool FULL>
__global__ void __launch_bounds__(32 * kWarps, 2) inner_wpp_kernel(const InnerArgs a, const WppArgs w) {
    extern __shared__ __align__(16) float smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* ring = smem + warp * w.warp_floats;
    float* zs = ring + w.ring;
    InFlight* q = reinterpret_cast<InFlight*>(zs + 2 * ((32 * kZS + 3) & ~3));   // kDepth entries, warp-private
    const int gw = blockIdx.x * kWarps + warp, nw = gridDim.x * kWarps;
    WCursor ic;
    ic.k = 0;
    wc_pair(a, ic, gw, nw);
    unsigned head = 0, tail = 0;   // monotone ring positions (floats)
    unsigned head_off = 0;         // head's offset inside the ring
    int qh = 0, qn = 0;            // in-flight queue: oldest entry index, count
    const unsigned RING = (unsigned)w.ring;
    while (true) {
        // ---- issue future steps while they fit
        while (ic.valid && qn < kDepth) {
            const int I = a.dims[ic.n];
            const int S = wrank(a.x, ic.b, a.N, ic.n + 1), Q = wrank(a.y, ic.b, a.N, ic.n + 1);
            const int nx = ic.R * I * S, ny = ic.P * I * Q;
            const unsigned need = (unsigned)((nx + 3) & ~3) + (unsigned)((ny + 3) & ~3);
            unsigned start = head, start_off = head_off;
            if (start_off + need > RING) { start += RING - start_off; start_off = 0; }   // do not wrap a step
            if (qn == 0) tail = start;                                                  // empty ring: the skip is free
            if (start + need - tail > RING) break;                                      // no room yet
            float* dst = ring + start_off;
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
                f.start = (int)start_off;
                f.b = ic.b; f.n = ic.n; f.R = ic.R; f.P = ic.P; f.S = S; f.Q = Q; f.I = I;
                f.end = start + need;
                q[(qh + qn) % kDepth] = f;
            }
            ++qn;
            head = start + need;
            head_off = start_off + need;
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
        const bool vf = (f.R * f.P * f.S + f.P * f.S * f.Q) < (f.R * f.P * f.Q + f.R * f.S * f.Q);
        if (f.n == a.N - 1) {
            const float v = wpp_last<FULL>(X, Y, f.R, f.P, f.I, f.n == 0, zs, lane);
            if (lane == 0) zs[0] = v;
            __syncwarp();
        } else if (f.n == 0) {
            wpp_first<FULL>(X, Y, f.S, f.Q, f.I, zs, lane);
        } else if (FULL) {   // every interior rank of the batch is a multiple of 8 (host-checked)
            uint32_t* zh = reinterpret_cast<uint32_t*>(zs);
            if (vf) wpp_step_full(X, f.R, f.S, Y, f.P, f.Q, f.I, true, zh, zh + kZsl, lane);
            else wpp_step_full(Y, f.P, f.Q, X, f.R, f.S, f.I, false, zh, zh + kZsl, lane);
        } else {
            if (vf) wpp_step(X, f.R, f.S, Y, f.P, f.Q, f.I, true, zs, lane);
            else wpp_step(Y, f.P, f.Q, X, f.R, f.S, f.I, false, zs, lane);
        }
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
    const int64_t warp_floats = wpp_ring(max_rank, max_dim) + 2 * ((32 * kZS + 3) & ~3) + kDepth * (int64_t)sizeof(InFlight) / 4 + kTail;
    return sizeof(float) * warp_floats * kWarps <= 200 * 1024;
}

template <bool FULL>
cudaError_t launch_wpp_t(const InnerArgs& a, int max_rank, cudaStream_t s) {
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = std::max(max_dim, (int)a.dims[n]);
    WppArgs w;
    w.ring = (int)wpp_ring(max_rank, max_dim);
    w.warp_floats = w.ring + 2 * ((32 * kZS + 3) & ~3) + (int)(kDepth * sizeof(InFlight) / 4) + kTail;
    const size_t smem = sizeof(float) * (size_t)w.warp_floats * kWarps;
    cudaError_t e = cudaFuncSetAttribute(inner_wpp_kernel<FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_wpp_kernel<FULL>, 32 * kWarps, smem)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int want = (a.B + kWarps - 1) / kWarps;
    const int grid = want < sms * per_sm ? want : sms * per_sm;
    inner_wpp_kernel<FULL><<<grid, 32 * kWarps, smem, s>>>(a, w);
    return cudaGetLastError();
}

cudaError_t launch_inner_wpp(const InnerArgs& a, int max_rank, bool ranks_mult8, cudaStream_t s) {
    return ranks_mult8 ? launch_wpp_t<true>(a, max_rank, s) : launch_wpp_t<false>(a, max_rank, s);
}

}  // namespace ttc
