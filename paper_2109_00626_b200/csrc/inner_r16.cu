// inner_r16.cu -- tt_inner specialised for batches whose trains all have the rank profile (1, 16, ..., 16, 1)
// (BASELINE.json C2: N = 8, I = 16, R = 16).  Same sweep as ttc.h / inner_fast.cu:
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :],  out = Z_N.
// Persistent CTAs, warp-specialised:
//   * producer warp: TMA bulk copies (cp.async.bulk) of each step's two cores into a 2-stage ring (interior
//     cores one copy per plane into padded planes, boundary cores one contiguous copy), full/empty mbarriers;
//   * 8 compute warps:
//       first step  Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q]  (Eq. 12's K = A_x^T A_y) on the FP32 pipe, written
//                   straight into the next step's B-fragment layout;
//       interior    the two rank-16 GEMMs of a slice i on the tensor cores (3xTF32 mma.sync m16n8k8, every bound
//                   a compile-time constant), slices spread over the warps, partials reduced through shared
//                   memory in a fixed order into the next step's B fragments;
//       last step   Z_N = sum_{r,p} Z[r,p] sum_i X_N[r,i,0] Y_N[p,i,0] on the FP32 pipe + a fixed-order
//                   block reduction.
// Every core byte is read from HBM exactly once; nothing is written but the result.
#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

using namespace tc;

constexpr int kCW = 8;          // compute warps
constexpr int kCT = 32 * kCW;   // compute threads = zfrag slots (2 x 2 fragments x 64)
constexpr int kPart = 2 * 32 * 4;   // floats of one warp's partial Z' (2 n-tiles, fragment-native)
constexpr int kEnd = 1 << 30;
#ifndef TTC_R16_STAGES
#define TTC_R16_STAGES 3
#endif
constexpr int kStages = TTC_R16_STAGES;   // TMA ring depth (steps in flight per CTA)

struct R16Step {
    int b, n, I, flags;   // flags: 1 first step, 2 last step, kEnd: no more steps
    int64_t xo, yo;
};

struct R16Layout {
    int ps_max;      // plane stride for the largest I
    int x_floats;    // X region of a stage (16 planes)
    int stage_floats;
};

struct R16Cursor {
    int k, b, n;
    int64_t xo, yo;
    bool valid;
};

__device__ __forceinline__ void r16_pair(const InnerArgs& a, R16Cursor& c) {
    const int idx = blockIdx.x + c.k * gridDim.x;
    c.valid = idx < a.B;
    if (!c.valid) return;
    c.b = a.order ? __ldg(a.order + idx) : idx;
    c.n = 0;
    c.xo = a.x.offsets ? __ldg(a.x.offsets + c.b) : (int64_t)c.b * a.x.train_elems;
    c.yo = a.y.offsets ? __ldg(a.y.offsets + c.b) : (int64_t)c.b * a.y.train_elems;
}

// Producer: record the step and stage its cores.  Interior cores: plane v (16 of them, I*16 floats each) at
// v * ps (ps = 8 mod 32: conflict-free fragment loads); boundary cores (16*I floats) copied contiguously.
__device__ __forceinline__ void r16_issue(const InnerArgs& a, R16Cursor& c, R16Step* info, float* stage, uint64_t* bar,
                                          const R16Layout& lay) {
    const int lane = threadIdx.x & 31;
    const int I = a.dims[c.n];
    const bool first = c.n == 0, last = c.n == a.N - 1;
    const float* xs = a.x.cores + c.xo;
    const float* ys = a.y.cores + c.yo;
    const int plane = 16 * I;
    if (lane == 0) {
        R16Step s;
        s.b = c.b; s.n = c.n; s.I = I; s.flags = (first ? 1 : 0) | (last ? 2 : 0); s.xo = c.xo; s.yo = c.yo;
        *info = s;
        fence_proxy_async();
        const int floats = (first || last) ? 2 * plane : 2 * 16 * plane;
        mbar_arrive_expect_tx(bar, 4u * floats);
    }
    __syncwarp();
    if (first || last) {
        if (lane == 0) bulk_g2s(stage, xs, 4u * plane, bar);
        if (lane == 1) bulk_g2s(stage + lay.x_floats, ys, 4u * plane, bar);
    } else {
        const int ps = plane_stride(plane);
        if (lane < 16) bulk_g2s(stage + lane * ps, xs + (int64_t)lane * plane, 4u * plane, bar);
        else bulk_g2s(stage + lay.x_floats + (lane - 16) * ps, ys + (int64_t)(lane - 16) * plane, 4u * plane, bar);
    }
    // advance
    const int64_t core = (first || last) ? plane : 16 * plane;
    c.xo += core;
    c.yo += core;
    if (++c.n == a.N) {
        ++c.k;
        r16_pair(a, c);
    }
}

// One interior slice pair/single, identical arithmetic to inner_fast.cu's interior16.
template <int U>
__device__ __forceinline__ void r16_units(const float* F, const float* G, int ps, const int (&ui)[U], int lg, int t,
                                          const BFrag (&zb)[2][2], float (&acc)[2][4]) {
    float w[U][2][4];
#pragma unroll
    for (int x = 0; x < U; ++x) {   // GEMM-1: W^T[(i, q), r] = sum_p Y[p, i, q] Z[r, p]
        const float* p1 = F + lg * ps + ui[x] * 16 + 2 * t;
        const float* p2 = p1 + 8 * ps;
        AFrag A[2];
#pragma unroll
        for (int kf = 0; kf < 2; ++kf) {
            const float2 a1 = *reinterpret_cast<const float2*>(p1 + 8 * kf);
            const float2 a2 = *reinterpret_cast<const float2*>(p2 + 8 * kf);
            const float fa[4] = {a1.x, a2.x, a1.y, a2.y};
            A[kf] = split_a_trunc(fa);
        }
#pragma unroll
        for (int ng = 0; ng < 2; ++ng) mma6<true>(w[x][ng], A[0], zb[0][ng], A[1], zb[1][ng]);
    }
#pragma unroll
    for (int x = 0; x < U; ++x) {   // GEMM-2: Z'[s, q] += sum_r X[r, i, s] W[r, i, q]
        const float* p1 = G + lg * ps + ui[x] * 16 + 2 * t;
        const float* p2 = p1 + 8 * ps;
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
            mma6<true>(tg, A[0], B0, A[1], B1);
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[h][c] += tg[c];
        }
    }
}

__global__ void __maxnreg__(96) inner_r16_kernel(const InnerArgs a, const R16Layout lay) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ __align__(16) R16Step ring[8];
    __shared__ float red[kCW];
    float* stages = smem;
    float* zpart = smem + kStages * lay.stage_floats;   // [kCW][2 n-tiles][32 lanes][4]
    float* zfrag = zpart + kCW * kPart;           // [kf][ng][32 lanes][2]: B fragments of Z for the next step
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int k = 0; k < kStages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCW) {   // ------------------------------------------------------------------ producer warp
        R16Cursor ic;
        ic.k = 0;
        r16_pair(a, ic);
        for (int j = 0;; ++j) {
            const int st = j % kStages;
            if (j >= kStages) mbar_wait(&empty[st], ((j / kStages) - 1) & 1);
            if (!ic.valid) {
                if (lane == 0) {
                    ring[j & 7].flags = kEnd;
                    mbar_arrive(&full[st]);
                }
                break;
            }
            r16_issue(a, ic, &ring[j & 7], stages + st * lay.stage_floats, &full[st], lay);
        }
        return;
    }

    // ------------------------------------------------------------------------------------------ compute
    const int tid = threadIdx.x, lg = lane >> 2, t = lane & 3;
    // this thread's zfrag slot e = tid: Z entry (g, f) = (8 ng + ln/4, 8 kf + 2 (ln%4) + jj) and its source in a
    // warp's fragment-native partial Z' (C fragment of n-tile nf = f / 8: lane 4 (g%8) + (f%8)/2, element
    // 2 (g/8) + f%2)
    const int e_jj = tid & 1, e_ln = (tid >> 1) & 31, e_ng = (tid >> 6) & 1, e_kf = tid >> 7;
    const int zg = 8 * e_ng + (e_ln >> 2), zf = 8 * e_kf + 2 * (e_ln & 3) + e_jj;
    const int src = ((zf >> 3) * 32 + ((zg & 7) << 2) + ((zf & 7) >> 1)) * 4 + ((zg >> 3) << 1) + (zf & 1);

    for (int j = 0;; ++j) {
        const int st = j % kStages;
        mbar_wait(&full[st], (j / kStages) & 1);
        const R16Step si = ring[j & 7];
        if (si.flags == kEnd) break;
        const float* X = stages + st * lay.stage_floats;
        const float* Y = X + lay.x_floats;
        const int I = si.I;
        if (si.flags & 2) {
            // ---- last step: Z_N = sum_{r,p} Z[r,p] sum_i X_N[r,i] Y_N[p,i]; this thread owns Z[zg, zf]
            float v = 0.f;
            if (si.flags & 1) {   // N == 1 cannot reach this kernel; kept for completeness
                v = 0.f;
            } else {
                float d = 0.f;
                for (int i = 0; i < I; ++i) d = fmaf(X[zg + 16 * i], Y[zf + 16 * i], d);
                v = zfrag[tid] * d;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[warp] = v;
            bar_named(1, kCT);
            if (tid == 0) {
                float s = 0.f;
#pragma unroll
                for (int w = 0; w < kCW; ++w) s += red[w];
                a.out[si.b] = s;
            }
            bar_named(1, kCT);
            continue;
        }
        if (si.flags & 1) {
            // ---- first step: Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q] (= A_x^T A_y, Eq. 12) into slot tid
            float d = 0.f;
            for (int i = 0; i < I; ++i) d = fmaf(X[i + I * zg], Y[i + I * zf], d);
            zfrag[tid] = d;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            bar_named(1, kCT);
            continue;
        }
        // ---- interior step
        BFrag zb[2][2];
#pragma unroll
        for (int kf = 0; kf < 2; ++kf)
#pragma unroll
            for (int ng = 0; ng < 2; ++ng) {
                const float2 v2 = *reinterpret_cast<const float2*>(zfrag + ((kf * 2 + ng) * 32 + lane) * 2);
                zb[kf][ng] = split_b(v2.x, v2.y);
            }
        float acc[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[h][c] = 0.f;
        const int ps = plane_stride(16 * I);
        int i = warp;
        for (; i + kCW < I; i += 2 * kCW) {
            const int uu[2] = {i, i + kCW};
            r16_units<2>(Y, X, ps, uu, lg, t, zb, acc);
        }
        if (i < I) {
            const int uu[1] = {i};
            r16_units<1>(Y, X, ps, uu, lg, t, zb, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        float* zw = zpart + warp * kPart;
#pragma unroll
        for (int h = 0; h < 2; ++h)
            *reinterpret_cast<float4*>(zw + (h * 32 + lane) * 4) = make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]);
        bar_named(1, kCT);   // partials visible
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kCW; ++w) v += zpart[w * kPart + src];
        zfrag[tid] = v;
        bar_named(1, kCT);   // next step's B fragments visible; partials free
    }
}

}  // namespace

bool inner_r16_supported(const InnerArgs& a, bool uniform_r16) {
    if (!uniform_r16 || a.N < 2) return false;
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = a.dims[n] > max_dim ? a.dims[n] : max_dim;
    // two stages of 2 x 16 padded planes + partials + fragments
    const size_t smem = sizeof(float) * (kStages * (size_t)2 * 16 * plane_stride(16 * max_dim) + kCW * kPart + kCT);
    return smem <= 112 * 1024;   // two CTAs per SM
}

cudaError_t launch_inner_r16(const InnerArgs& a, cudaStream_t s) {
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = a.dims[n] > max_dim ? a.dims[n] : max_dim;
    R16Layout lay;
    lay.ps_max = plane_stride(16 * max_dim);
    lay.x_floats = 16 * lay.ps_max;
    lay.stage_floats = 2 * lay.x_floats;
    const size_t smem = sizeof(float) * (kStages * (size_t)lay.stage_floats + kCW * kPart + kCT);
    cudaError_t e = cudaFuncSetAttribute(inner_r16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inner_r16_kernel, 32 * (kCW + 1), smem)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int grid = a.B < sms * per_sm ? a.B : sms * per_sm;
    inner_r16_kernel<<<grid, 32 * (kCW + 1), smem, s>>>(a, lay);
    return cudaGetLastError();
}

}  // namespace ttc
