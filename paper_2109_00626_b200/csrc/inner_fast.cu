// inner_fast.cu -- tt_inner for bond ranks <= 32 (BASELINE.json C1, C2, C5): persistent CTAs, cores staged
// HBM -> shared memory by the TMA bulk-copy engine (cp.async.bulk + mbarrier, double-buffered across steps
// and across pairs), rank products on the tensor cores as 3xTF32 mma.sync m16n8k8.
//
// The sweep (ttc.h), per mode n, with F the core multiplied into Z first and G the
// other one (W-first: F = Y, G = X;  V-first: F = X, G = Y -- the cheaper association per step):
//   GEMM-1  W^T[(i,f'), g] = sum_f F[f,i,f'] Z[g,f]       M = f' (16-row tiles), N = g (8-col), K = f
//   GEMM-2  Z'[g', f']    += sum_g G[g,i,g'] W[g,i,f']    M = g' (16-row tiles), N = f' (8-col), K = g
// Work split: the (slice i, 16-wide f' block) units of a step are spread over the 4 warps; each warp keeps
// its partial Z' in registers, the partials are summed through shared memory once per step (fixed order:
// every warp reconstructs the identical Z, so the result is deterministic).
// Fragment algebra (g = lane/4, t = lane%4; C fragment c_{2h+j} = C[g + 8h, 2t + j]): GEMM-1's C fragments
// are GEMM-2's B fragments unchanged when the k index inside each k8 block is permuted (k-slot t <-> 2t,
// k-slot t+4 <-> 2t+1); the A fragments (core values from shared memory) use the same permutation.
// Numerics: x = hi + lo (hi = rna_tf32(x), lo = rna_tf32(x - hi)), A*B ~= A_lo B_hi + A_hi B_lo + A_hi B_hi,
// each group of three MMAs starts from zero and is added to the fp32 accumulator with a round-to-nearest
// FADD (the tensor core's internal fp32 accumulation truncates).
// Shared-memory core layout: plane v (fixed last index) of a core at v * PS, PS = padded plane stride with
// PS = 8 (mod 32) floats, so the 8 rows of an A fragment fall in distinct banks.
#include <cstdlib>
#include <cstring>

#include "ttc_internal.h"
#include "tc_common.cuh"

namespace ttc {
namespace {

#ifndef TTC_RM16_MAXNREG
#define TTC_RM16_MAXNREG 96
#endif

using namespace tc;

// A fragment of a core staged in shared memory (element [u,i,v] at base + v*PS + i*Ga + u) for
// sum_u G[u,i,v] * B[u,.] with M = v (rows v0+g, v0+g+8) and K = u (k8 block at u0, permuted):
//   a0 = G[u0+2t, i, v0+g]  a1 = G[u0+2t, i, v0+g+8]  a2 = G[u0+2t+1, i, v0+g]  a3 = G[u0+2t+1, i, v0+g+8]
struct SmemCore {
    const float* base;
    int Ga, Gb, PS;
};
// Rows of one (i, 16-row block) of a core, ready for k-block loads.
struct ARows {
    const float* p1;   // &G[2t, i, v0+g]
    const float* p2;   // &G[2t, i, v0+g+8]
    bool ok1, ok2;
};
__device__ __forceinline__ ARows a_rows(const SmemCore& c, int i, int v0, int g, int t) {
    ARows r;
    r.p1 = c.base + (v0 + g) * c.PS + i * c.Ga + 2 * t;
    r.p2 = r.p1 + 8 * c.PS;
    r.ok1 = v0 + g < c.Gb;
    r.ok2 = v0 + g + 8 < c.Gb;
    return r;
}
// FULL: Ga is a multiple of 8 (K fully in range) -- rows beyond Gb are read unpredicated (they only feed
// output rows that are never used).  Otherwise every element is predicated.
template <bool FULL>
__device__ __forceinline__ void load_a(const SmemCore& c, const ARows& r, int u0, int t, float (&a)[4]) {
    if (FULL) {
        const float2 x1 = *reinterpret_cast<const float2*>(r.p1 + u0);
        const float2 x2 = *reinterpret_cast<const float2*>(r.p2 + u0);
        a[0] = x1.x; a[2] = x1.y; a[1] = x2.x; a[3] = x2.y;
    } else {
        const int u = u0 + 2 * t;
        const bool u0ok = u < c.Ga, u1ok = u + 1 < c.Ga;
        a[0] = (u0ok && r.ok1) ? r.p1[u0] : 0.f;
        a[2] = (u1ok && r.ok1) ? r.p1[u0 + 1] : 0.f;
        a[1] = (u0ok && r.ok2) ? r.p2[u0] : 0.f;
        a[3] = (u1ok && r.ok2) ? r.p2[u0 + 1] : 0.f;
    }
}

// Walks the CTA's (pair, step) sequence.
struct Cursor {
    int k, b, n, R, P;
    int64_t xo, yo;
    bool valid;
};

__device__ __forceinline__ int rank_at(const TrainDev& t, int b, int N, int n) {
    if (n == 0 || n == N) return 1;
    return t.ranks ? __ldg(t.ranks + (int64_t)b * (N + 1) + n) : t.urank;
}
__device__ __forceinline__ int64_t train_base(const TrainDev& t, int b) {
    return t.offsets ? __ldg(t.offsets + b) : (int64_t)b * t.train_elems;
}
__device__ __forceinline__ void cursor_pair(const InnerArgs& a, Cursor& c) {
    const int idx = blockIdx.x + c.k * gridDim.x;
    c.valid = idx < a.B;
    if (!c.valid) return;
    c.b = a.order ? __ldg(a.order + idx) : idx;
    c.n = 0;
    c.R = 1;
    c.P = 1;
    c.xo = train_base(a.x, c.b);
    c.yo = train_base(a.y, c.b);
}

// Geometry of one step, computed once by the issuing warp and read by every warp from a shared ring.
struct StepInfo {
    int R, P, S, Q, I, psx, psy;
    int b;        // pair
    int flags;    // bit0: V-first association, bit1: planes bulk-copyable, bit2: first step, bit3: last step
    int pad;
    int64_t xo, yo;
};

__device__ __forceinline__ void cursor_next(const InnerArgs& a, Cursor& c, int S, int Q) {
    const int I = a.dims[c.n];
    c.xo += (int64_t)c.R * I * S;
    c.yo += (int64_t)c.P * I * Q;
    c.R = S;
    c.P = Q;
    if (++c.n == a.N) {
        ++c.k;
        cursor_pair(a, c);
    }
}

// Warp 0: records step `c` in the ring and stages its planes into `stage` (plane v of each core at v * PS):
// one TMA bulk copy (cp.async.bulk) per plane, issued by the 32 lanes in parallel, completing on `bar`.
// Steps whose planes are not 16-byte copyable arrive without data (the compute side then copies them).
__device__ __forceinline__ void issue_step(const InnerArgs& a, Cursor& c, StepInfo* info, float* stage, uint64_t* bar,
                                           int x_floats) {
    const int lane = threadIdx.x & 31;
    const int I = a.dims[c.n];
    const int S = rank_at(a.x, c.b, a.N, c.n + 1), Q = rank_at(a.y, c.b, a.N, c.n + 1);
    const int R = c.R, P = c.P;
    const int ix = I * R, iy = I * P;
    const float* xs = a.x.cores + c.xo;
    const float* ys = a.y.cores + c.yo;
    const bool ok = ((ix & 3) == 0) && ((iy & 3) == 0) && ((reinterpret_cast<uintptr_t>(xs) & 15u) == 0) &&
                    ((reinterpret_cast<uintptr_t>(ys) & 15u) == 0);
    const int psx = plane_stride(ix), psy = plane_stride(iy);
    if (lane == 0) {
        StepInfo si;
        si.R = R; si.P = P; si.S = S; si.Q = Q; si.I = I; si.psx = psx; si.psy = psy; si.b = c.b; si.pad = 0;
        // per-slice MACs of the two associations: W-first R*P*Q + R*S*Q, V-first R*P*S + P*S*Q
        const bool vf = (R * P * S + P * S * Q) < (R * P * Q + R * S * Q);
        si.flags = (vf ? 1 : 0) | (ok ? 2 : 0) | (c.n == 0 ? 4 : 0) | (c.n == a.N - 1 ? 8 : 0);
        si.xo = c.xo; si.yo = c.yo;
        *info = si;
        if (ok) {
            fence_proxy_async();
            mbar_arrive_expect_tx(bar, (uint32_t)(4 * (ix * S + iy * Q)));
        } else {
            mbar_arrive(bar);
        }
    }
    __syncwarp();
    if (ok) {
        for (int v = lane; v < S + Q; v += 32) {
            if (v < S) bulk_g2s(stage + v * psx, xs + (int64_t)v * ix, 4u * ix, bar);
            else bulk_g2s(stage + x_floats + (v - S) * psy, ys + (int64_t)(v - S) * iy, 4u * iy, bar);
        }
    }
    cursor_next(a, c, S, Q);
}

struct Layout {
    int stage_floats, x_floats;   // per stage: X region then Y region
};

constexpr int kEnd = 16;   // StepInfo flag: no more steps for this CTA

// U work units (slice i, 16-wide f' block) of one step, processed in lockstep for instruction-level
// parallelism: GEMM-1 into w (C fragments), then GEMM-2 accumulating into acc (static indices only).
// Each GEMM accumulates at most two k8 blocks (six MMAs) inside the tensor core before a round-to-nearest
// FADD into the fp32 accumulator.
template <int RM, int U, bool FULL>
__device__ __forceinline__ void step_units(const SmemCore& Fc, const SmemCore& Gc, const int (&ui)[U], const int (&mq)[U],
                                           int kf_n, int ng_n, int mg_n, int Fb, int lg, int t,
                                           const BFrag (&zb)[RM / 8][RM / 8], float (&acc)[RM / 16][RM / 8][4]) {
    constexpr int NT = RM / 8, MT = RM / 16;
    // ---- GEMM-1: w[x][ng] = sum_kf A_F(mq, kf) B_Z(kf, ng), two k8 blocks per tensor-core group
    float w[U][NT][4];
    ARows fr[U];
#pragma unroll
    for (int x = 0; x < U; ++x) fr[x] = a_rows(Fc, ui[x], 16 * mq[x], lg, t);
#pragma unroll
    for (int kp = 0; kp < NT; kp += 2) {
        if (kp >= kf_n) break;
        float tg[U][NT][4];
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
            const int kf = kp + sub;
            if (kf >= kf_n) break;
            AFrag A[U];
#pragma unroll
            for (int x = 0; x < U; ++x) {
                float fa[4];
                load_a<FULL>(Fc, fr[x], 8 * kf, t, fa);
                A[x] = split_a(fa);
            }
#pragma unroll
            for (int ng = 0; ng < NT; ++ng) {
                if (ng >= ng_n) break;
#pragma unroll
                for (int x = 0; x < U; ++x) {
                    if (sub == 0) mma3<true>(tg[x][ng], A[x], zb[kf][ng]);
                    else mma3<false>(tg[x][ng], A[x], zb[kf][ng]);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < U; ++x)
#pragma unroll
            for (int ng = 0; ng < NT; ++ng)
#pragma unroll
                for (int c = 0; c < 4; ++c) w[x][ng][c] = (kp == 0) ? tg[x][ng][c] : w[x][ng][c] + tg[x][ng][c];
    }
    // ---- GEMM-2: acc[mg][2 mq + h] += sum_kg A_G(mg, kg) B_W(kg, h),  B_W(kg, h) = w[kg][2h + j]
#pragma unroll
    for (int mg = 0; mg < MT; ++mg) {
        if (mg >= mg_n) break;
        ARows gr[U];
#pragma unroll
        for (int x = 0; x < U; ++x) gr[x] = a_rows(Gc, ui[x], 16 * mg, lg, t);
#pragma unroll
        for (int kp = 0; kp < NT; kp += 2) {
            if (kp >= ng_n) break;
            float tg[U][2][4];
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
                const int kg = kp + sub;
                if (kg >= ng_n) break;
                AFrag A[U];
#pragma unroll
                for (int x = 0; x < U; ++x) {
                    float ga[4];
                    load_a<FULL>(Gc, gr[x], 8 * kg, t, ga);
                    A[x] = split_a(ga);
                }
#pragma unroll
                for (int x = 0; x < U; ++x)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const BFrag B = split_b(w[x][kg][2 * h], w[x][kg][2 * h + 1]);
                        if (sub == 0) mma3<true>(tg[x][h], A[x], B);
                        else mma3<false>(tg[x][h], A[x], B);
                    }
            }
#pragma unroll
            for (int x = 0; x < U; ++x)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int mqq = 0; mqq < MT; ++mqq) {   // static index into acc
                        if (mqq != mq[x] || 16 * mqq + 8 * h >= Fb) continue;
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[mg][2 * mqq + h][c] += tg[x][h][c];
                    }
        }
    }
}

// Interior step of a rank-16 batch (R = P = S = Q = 16, W-first): the same two GEMMs as step_units with
// every bound a compile-time constant -- no predicates, no partial tiles.  U slices i in lockstep.
template <int U>
__device__ __forceinline__ void interior16(const float* F, int psF, const float* G, int psG, const int (&ui)[U], int lg,
                                           int t, const BFrag (&zb)[2][2], float (&acc)[1][2][4]) {
    float w[U][2][4];
#pragma unroll
    for (int x = 0; x < U; ++x) {   // GEMM-1: W^T[(i, q), r] = sum_p Y[p, i, q] Z[r, p]
        const float* p1 = F + lg * psF + ui[x] * 16 + 2 * t;
        const float* p2 = p1 + 8 * psF;
        AFrag A[2];
#pragma unroll
        for (int kf = 0; kf < 2; ++kf) {
            const float2 a1 = *reinterpret_cast<const float2*>(p1 + 8 * kf);
            const float2 a2 = *reinterpret_cast<const float2*>(p2 + 8 * kf);
            const float fa[4] = {a1.x, a2.x, a1.y, a2.y};
            A[kf] = split_a_trunc(fa);
        }
#pragma unroll
        for (int ng = 0; ng < 2; ++ng) {
            mma3<true>(w[x][ng], A[0], zb[0][ng]);
            mma3<false>(w[x][ng], A[1], zb[1][ng]);
        }
    }
#pragma unroll
    for (int x = 0; x < U; ++x) {   // GEMM-2: Z'[s, q] += sum_r X[r, i, s] W[r, i, q]
        const float* p1 = G + lg * psG + ui[x] * 16 + 2 * t;
        const float* p2 = p1 + 8 * psG;
        AFrag A[2];
#pragma unroll
        for (int kg = 0; kg < 2; ++kg) {
            const float2 a1 = *reinterpret_cast<const float2*>(p1 + 8 * kg);
            const float2 a2 = *reinterpret_cast<const float2*>(p2 + 8 * kg);
            const float ga[4] = {a1.x, a2.x, a1.y, a2.y};
            A[kg] = split_a_trunc(ga);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const BFrag B0 = split_b(w[x][0][2 * h], w[x][0][2 * h + 1]);
            const BFrag B1 = split_b(w[x][1][2 * h], w[x][1][2 * h + 1]);
            float tg[4];
            mma3<true>(tg, A[0], B0);
            mma3<false>(tg, A[1], B1);
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[0][h][c] += tg[c];
        }
    }
}

// zfrag slot e (next step's B fragment: jj = e & 1, lane = (e >> 1) & 31, ng = (e >> 6) % NT, kf = (e >> 6) / NT)
// -> offset of the same Z entry in this step's fragment-native partials, or -1 if outside the ranks.
template <int NT>
__device__ __forceinline__ int zfrag_source(int e, bool vf, bool vfn, int Gan, int Fan) {
    const int jj = e & 1, ln = (e >> 1) & 31, blk = e >> 6;
    const int ng = blk % NT, kf = blk / NT;
    const int gq = 8 * ng + (ln >> 2), fq = 8 * kf + 2 * (ln & 3) + jj;   // next step's (g, f)
    if (gq >= Gan || fq >= Fan) return -1;
    // canonical (x, y) of that Z entry, then this step's output coordinates (g', f')
    const int xb = vfn ? fq : gq, yb = vfn ? gq : fq;
    const int g2 = vf ? yb : xb, f2 = vf ? xb : yb;
    const int mg = g2 >> 4, hh = (g2 >> 3) & 1, nf = f2 >> 3;
    const int l2 = ((g2 & 7) << 2) | ((f2 & 7) >> 1), cc = (hh << 1) | (f2 & 1);
    return ((mg * NT + nf) * 32 + l2) * 4 + cc;
}

__device__ __forceinline__ void bar_compute(int threads) { asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory"); }

// Warp-specialised: warps 0..WARPS-1 compute, warp WARPS produces (TMA bulk copies into a 2-stage ring,
// full/empty mbarriers).  Per step: units -> fragment-native partials -> reduction straight into the next
// step's GEMM-1 B-fragment layout (zfrag), two named barriers among the compute warps.
template <int RM, int WARPS>
__global__ void __launch_bounds__(32 * (WARPS + 1)) __maxnreg__(RM == 16 ? TTC_RM16_MAXNREG : 255) inner_tc_kernel(const InnerArgs a, const Layout lay) {
    constexpr int NT = RM / 8;     // k8 blocks / 8-col tiles over one bond
    constexpr int MT = RM / 16;    // 16-row tiles over one bond
    constexpr int CT = 32 * WARPS; // compute threads
    constexpr int PART = MT * NT * 32 * 4;   // floats of one warp's partial (fragment-native)
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t full[2], empty[2];
    __shared__ __align__(16) StepInfo ring[4];
    float* stages = smem;
    float* zpart = smem + 2 * lay.stage_floats;   // [WARPS][MT][NT][32 lanes][4]
    float* zfrag = zpart + WARPS * PART;          // [NT kf][NT ng][32 lanes][2]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lg = lane >> 2, t = lane & 3;

    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&empty[0], WARPS);
        mbar_init(&empty[1], WARPS);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == WARPS) {   // ------------------------------------------------------------ producer warp
        Cursor ic;
        ic.k = 0;
        cursor_pair(a, ic);
        for (int j = 0;; ++j) {
            const int st = j & 1;
            if (j >= 2) mbar_wait(&empty[st], ((j >> 1) - 1) & 1);
            if (!ic.valid) {
                if (lane == 0) {
                    ring[j & 3].flags = kEnd;
                    mbar_arrive(&full[st]);
                }
                break;
            }
            issue_step(a, ic, &ring[j & 3], stages + st * lay.stage_floats, &full[st], lay.x_floats);
        }
        return;
    }

    // ------------------------------------------------------------------------------------- compute warps
    constexpr int SLOTS = (NT * NT * 64 + CT - 1) / CT;   // zfrag slots per thread
    int plain_off[SLOTS];   // reduction sources of this thread's slots for W-first steps at full rank
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
        const int e = threadIdx.x + k * CT;
        plain_off[k] = e < NT * NT * 64 ? zfrag_source<NT>(e, false, false, RM, RM) : -1;
    }
    float acc[MT][NT][4];
    for (int j = 0;; ++j) {
        const int st = j & 1;
        mbar_wait(&full[st], (j >> 1) & 1);
        const StepInfo si = ring[j & 3];
        if (si.flags & kEnd) break;
        float* stage = stages + st * lay.stage_floats;
        const int R = si.R, P = si.P, S = si.S, Q = si.Q, I = si.I;
        const bool vf = si.flags & 1;
        if ((si.flags & 2) == 0) {   // synchronous fallback copy (odd plane sizes / alignment)
            const float* xs = a.x.cores + si.xo;
            const float* ys = a.y.cores + si.yo;
            for (int e = threadIdx.x; e < I * R * S; e += CT) {
                const int v = e / (I * R), w = e - v * (I * R);
                stage[v * si.psx + w] = __ldg(xs + e);
            }
            for (int e = threadIdx.x; e < I * P * Q; e += CT) {
                const int v = e / (I * P), w = e - v * (I * P);
                stage[lay.x_floats + v * si.psy + w] = __ldg(ys + e);
            }
            bar_compute(CT);
        }
        const SmemCore Fc = vf ? SmemCore{stage, R, S, si.psx} : SmemCore{stage + lay.x_floats, P, Q, si.psy};
        const SmemCore Gc = vf ? SmemCore{stage + lay.x_floats, P, Q, si.psy} : SmemCore{stage, R, S, si.psx};
        const int Fa = Fc.Ga, Fb = Fc.Gb, Ga = Gc.Ga, Gb = Gc.Gb;
        // GEMM-1 B fragments: zb[kf][ng] = split of Z[g = 8 ng + lg, f = 8 kf + 2t + j]
        BFrag zb[NT][NT];
#pragma unroll
        for (int kf = 0; kf < NT; ++kf)
#pragma unroll
            for (int ng = 0; ng < NT; ++ng) {
                float2 v2;
                if (si.flags & 4) v2 = make_float2((kf == 0 && ng == 0 && lane == 0) ? 1.0f : 0.0f, 0.0f);   // Z_0 = [1]
                else v2 = *reinterpret_cast<const float2*>(zfrag + ((kf * NT + ng) * 32 + lane) * 2);
                zb[kf][ng] = split_b(v2.x, v2.y);
            }
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int q = 0; q < NT; ++q)
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) acc[m][q][cc] = 0.f;
        const int kf_n = (Fa + 7) >> 3, ng_n = (Ga + 7) >> 3, mq_n = (Fb + 15) >> 4, mg_n = (Gb + 15) >> 4;
        // this warp's units u = warp, warp + WARPS, ... < I * mq_n as (i = u % I, mq = u / I)
        int ui = warp, umq = 0;
        while (ui >= I) { ui -= I; ++umq; }
        auto next_unit = [&](int& i, int& m) {
            i += WARPS;
            while (i >= I) { i -= I; ++m; }
        };
        if (RM == 16 && !vf && R == 16 && P == 16 && S == 16 && Q == 16) {
            // lean interior path: units are the slices i = warp, warp + WARPS, ...
            const float* Fp = stage + lay.x_floats;
            int i = warp;
            for (; i + WARPS < I; i += 2 * WARPS) {
                const int uu[2] = {i, i + WARPS};
                interior16<2>(Fp, si.psy, stage, si.psx, uu, lg, t, reinterpret_cast<const BFrag(&)[2][2]>(zb), reinterpret_cast<float(&)[1][2][4]>(acc));
            }
            if (i < I) {
                const int uu[1] = {i};
                interior16<1>(Fp, si.psy, stage, si.psx, uu, lg, t, reinterpret_cast<const BFrag(&)[2][2]>(zb), reinterpret_cast<float(&)[1][2][4]>(acc));
            }
        } else if (((Fa & 7) == 0) && ((Ga & 7) == 0)) {
            while (umq < mq_n) {
                int i2 = ui, m2 = umq;
                next_unit(i2, m2);
                if (m2 < mq_n) {   // two independent units in lockstep: twice the ILP
                    const int uu[2] = {ui, i2}, mm[2] = {umq, m2};
                    step_units<RM, 2, true>(Fc, Gc, uu, mm, kf_n, ng_n, mg_n, Fb, lg, t, zb, acc);
                    next_unit(i2, m2);
                } else {
                    const int uu[1] = {ui}, mm[1] = {umq};
                    step_units<RM, 1, true>(Fc, Gc, uu, mm, kf_n, ng_n, mg_n, Fb, lg, t, zb, acc);
                }
                ui = i2; umq = m2;
            }
        } else {
            while (umq < mq_n) {
                const int uu[1] = {ui}, mm[1] = {umq};
                step_units<RM, 1, false>(Fc, Gc, uu, mm, kf_n, ng_n, mg_n, Fb, lg, t, zb, acc);
                next_unit(ui, umq);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);   // this warp is done with the stage
        // ---- phase A: this warp's partial Z' in fragment-native order (one 16-byte store per fragment)
        float* zw = zpart + warp * PART;
#pragma unroll
        for (int mg = 0; mg < MT; ++mg)
#pragma unroll
            for (int nf = 0; nf < NT; ++nf)
                *reinterpret_cast<float4*>(zw + ((mg * NT + nf) * 32 + lane) * 4) =
                    make_float4(acc[mg][nf][0], acc[mg][nf][1], acc[mg][nf][2], acc[mg][nf][3]);
        bar_compute(CT);   // (1) partials visible
        if (si.flags & 8) {   // Z_N = Z'[0, 0]: fragment (0, 0), lane 0, element 0
            if (threadIdx.x == 0) {
                float v = 0.f;
#pragma unroll
                for (int w = 0; w < WARPS; ++w) v += zpart[w * PART];
                a.out[si.b] = v;
            }
        } else {
            // ---- phase B: reduce the partials (fixed order) directly into the next step's B fragments
            mbar_wait(&full[st ^ 1], ((j + 1) >> 1) & 1);   // next step's geometry (and data) are ready
            const StepInfo sn = ring[(j + 1) & 3];
            const bool vfn = sn.flags & 1;
            const int Gan = vfn ? sn.P : sn.R, Fan = vfn ? sn.R : sn.P;
            const bool plain = !vf && !vfn && Gan == RM && Fan == RM;   // precomputed mapping
#pragma unroll
            for (int k = 0; k < SLOTS; ++k) {
                const int e = threadIdx.x + k * CT;
                if (e >= NT * NT * 64) break;
                const int off = plain ? plain_off[k] : zfrag_source<NT>(e, vf, vfn, Gan, Fan);
                float v = 0.f;
                if (off >= 0) {
#pragma unroll
                    for (int w = 0; w < WARPS; ++w) v += zpart[w * PART + off];
                }
                zfrag[e] = v;
            }
        }
        bar_compute(CT);   // (2) zfrag visible; zpart free
    }
}

template <int RM, int WARPS>
size_t tc_smem_bytes(const InnerArgs& a, Layout* lay) {
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = a.dims[n] > max_dim ? a.dims[n] : max_dim;
    lay->x_floats = RM * plane_stride(max_dim * RM);
    lay->stage_floats = 2 * lay->x_floats;
    return sizeof(float) * (2 * (size_t)lay->stage_floats + (size_t)WARPS * (RM / 16) * (RM / 8) * 128 +
                           (size_t)(RM / 8) * (RM / 8) * 64);
}

template <int RM, int WARPS>
cudaError_t launch_tc(const InnerArgs& a, cudaStream_t s) {
    Layout lay;
    const size_t smem = tc_smem_bytes<RM, WARPS>(a, &lay);
    cudaError_t e = cudaFuncSetAttribute(inner_tc_kernel<RM, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_tc_kernel<RM, WARPS>, 32 * (WARPS + 1), smem)) !=
        cudaSuccess)
        return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int grid = a.B < sms * per_sm ? a.B : sms * per_sm;
    inner_tc_kernel<RM, WARPS><<<grid, 32 * (WARPS + 1), smem, s>>>(a, lay);
    return cudaGetLastError();
}

}  // namespace

// Shared-memory need: two stages of RM x plane_stride(max I * RM) per core plus the Z buffers.
bool inner_fast_supported(const InnerArgs& a, int max_rank, bool uniform) {
    (void)uniform;
    if (max_rank > 32) return false;
    Layout lay;
    const size_t smem = max_rank <= 16 ? tc_smem_bytes<16, 8>(a, &lay) : tc_smem_bytes<32, 4>(a, &lay);
    return smem <= 220 * 1024;
}

cudaError_t launch_inner_fast(const InnerArgs& a, int max_rank, bool uniform, cudaStream_t s) {
    (void)uniform;
    return max_rank <= 16 ? launch_tc<16, 8>(a, s) : launch_tc<32, 4>(a, s);
}

}  // namespace ttc
