// inner_r16.cu -- tt_inner specialised for batches whose trains all have the rank profile (1, 16, ..., 16, 1)
// (BASELINE.json C2: N = 8, I = 16, R = 16).  Same sweep as ttc.h / inner_fast.cu:
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :],  out = Z_N.
// Persistent CTAs, warp-specialised:
//   * producer warp: TMA bulk copies (cp.async.bulk) of each INTERIOR step's two cores into a kStages-deep ring
//     (one copy per plane into padded planes), full/empty mbarriers; the two rank-1 boundary cores of a pair
//     (1 KB each per train for I = 16) are only prefetched into L2 (cp.async.bulk.prefetch.L2) -- a boundary
//     step in the ring would occupy a whole stage for 1/16 of its data and leave the next pair's first
//     interior stage issued just one short step ahead of its use (an exposed HBM latency per pair);
//   * 8 compute warps, per pair:
//       first core  Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q]  (Eq. 12's K = A_x^T A_y) on the FP32 pipe from
//                   global (L2-resident) memory, written straight into the next step's B-fragment layout,
//                   overlapping the first interior stage's arrival;
//       interior    the two rank-16 GEMMs of a slice i on the tensor cores (3xTF32 mma.sync m16n8k8, every bound
//                   a compile-time constant), slices spread over the warps, partials reduced through shared
//                   memory in a fixed order into the next step's B fragments;
//       last core   fused into the last interior step's reduction: each thread holds one entry Z_{N-1}[r, p] and
//                   multiplies it by sum_i X_N[r,i,0] Y_N[p,i,0] (FP32, from L2), then a fixed-order block
//                   reduction.
// Every core byte is read from HBM exactly once; nothing is written but the result.  Needs N >= 3.
#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

using namespace tc;

constexpr int kCW = 8;          // compute warps
constexpr int kCT = 32 * kCW;   // compute threads = zfrag slots (2 x 2 fragments x 64)
constexpr int kPart = 2 * 32 * 4;   // floats of one warp's partial Z' (2 n-tiles, fragment-native)
#ifndef TTC_R16_STAGES
#define TTC_R16_STAGES 3
#endif
constexpr int kStages = TTC_R16_STAGES;   // TMA ring depth (interior steps in flight per CTA)

struct R16Layout {
    int ps_max;      // plane stride for the largest I
    int x_floats;    // X region of a stage (16 planes)
    int stage_floats;
};

// The k-th pair of this CTA (pairs blockIdx.x, blockIdx.x + gridDim.x, ...): index b and core offsets.
struct R16Pair {
    int b;
    int64_t xo, yo;
    bool valid;
};
__device__ __forceinline__ R16Pair r16_pair(const InnerArgs& a, int k) {
    R16Pair p;
    const int idx = blockIdx.x + k * gridDim.x;
    p.valid = idx < a.B;
    if (!p.valid) return p;
    p.b = a.order ? __ldg(a.order + idx) : idx;
    p.xo = a.x.offsets ? __ldg(a.x.offsets + p.b) : (int64_t)p.b * a.x.train_elems;
    p.yo = a.y.offsets ? __ldg(a.y.offsets + p.b) : (int64_t)p.b * a.y.train_elems;
    return p;
}

__device__ __forceinline__ void prefetch_l2(const float* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Producer: stage interior core n (planes of 16 x I floats: plane v at v * ps, ps = 8 mod 32 so that fragment
// loads are conflict-free), X planes then Y planes.
__device__ __forceinline__ void r16_issue(const float* xs, const float* ys, int I, float* stage, uint64_t* bar,
                                          const R16Layout& lay) {
    const int lane = threadIdx.x & 31;
    const int plane = 16 * I;
    if (lane == 0) mbar_arrive_expect_tx(bar, 4u * 2 * 16 * plane);
    __syncwarp();
    const int ps = plane_stride(plane);
    if (lane < 16) bulk_g2s(stage + lane * ps, xs + (int64_t)lane * plane, 4u * plane, bar);
    else bulk_g2s(stage + lay.x_floats + (lane - 16) * ps, ys + (int64_t)(lane - 16) * plane, 4u * plane, bar);
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
    __shared__ float red[kCW];
    float* stages = smem;
    float* zpart = smem + kStages * lay.stage_floats;   // [kCW][2 n-tiles][32 lanes][4]
    float* zfrag = zpart + kCW * kPart;           // [kf][ng][32 lanes][2]: B fragments of Z for the next step
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N, I0 = a.dims[0], IL = a.dims[N - 1];

    if (threadIdx.x == 0) {
        for (int k = 0; k < kStages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCW) {   // ------------------------------------------------------------------ producer warp
        int j = 0;
        for (int k = 0;; ++k) {
            const R16Pair p = r16_pair(a, k);
            if (!p.valid) break;
            const float* xs = a.x.cores + p.xo;
            const float* ys = a.y.cores + p.yo;
            // boundary cores -> L2 (the compute warps read them with plain loads)
            if (lane == 0) prefetch_l2(xs, 4u * 16 * I0);
            if (lane == 1) prefetch_l2(ys, 4u * 16 * I0);
            int64_t off = 16 * (int64_t)I0;
            for (int n = 1; n < N - 1; ++n, ++j) {
                const int st = j % kStages;
                if (j >= kStages) mbar_wait(&empty[st], ((j / kStages) - 1) & 1);
                const int I = a.dims[n];
                r16_issue(xs + off, ys + off, I, stages + st * lay.stage_floats, &full[st], lay);
                off += 256 * (int64_t)I;
            }
            if (lane == 0) prefetch_l2(xs + off, 4u * 16 * IL);
            if (lane == 1) prefetch_l2(ys + off, 4u * 16 * IL);
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

    int j = 0;
    for (int k = 0;; ++k) {
        const R16Pair p = r16_pair(a, k);
        if (!p.valid) break;
        const float* xs = a.x.cores + p.xo;
        const float* ys = a.y.cores + p.yo;
        {   // ---- first core: Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q] (= A_x^T A_y, Eq. 12) into slot tid.
            // Safe to overwrite zfrag: every warp passed the previous pair's partials barrier, after its last read.
            const float* xr = xs + I0 * zg;
            const float* yr = ys + I0 * zf;
            float d = 0.f;
            if ((I0 & 3) == 0) {
                for (int i = 0; i < I0; i += 4) {
                    const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + i));
                    const float4 yv = __ldg(reinterpret_cast<const float4*>(yr + i));
                    d = fmaf(xv.x, yv.x, d);
                    d = fmaf(xv.y, yv.y, d);
                    d = fmaf(xv.z, yv.z, d);
                    d = fmaf(xv.w, yv.w, d);
                }
            } else {
                for (int i = 0; i < I0; ++i) d = fmaf(__ldg(xr + i), __ldg(yr + i), d);
            }
            zfrag[tid] = d;
            bar_named(1, kCT);
        }
        int64_t off = 16 * (int64_t)I0;
        for (int n = 1; n < N - 1; ++n, ++j) {
            const int st = j % kStages;
            const int I = a.dims[n];
            off += 256 * (int64_t)I;
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
            mbar_wait(&full[st], (j / kStages) & 1);
            const float* X = stages + st * lay.stage_floats;
            const float* Y = X + lay.x_floats;
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
            if (n < N - 2) {
                bar_named(1, kCT);   // partials visible
                float v = 0.f;
#pragma unroll
                for (int w = 0; w < kCW; ++w) v += zpart[w * kPart + src];
                zfrag[tid] = v;
                bar_named(1, kCT);   // next step's B fragments visible; partials free
            } else {
                // ---- last core fused: Z_N = sum_{r,p} Z_{N-1}[r,p] sum_i X_N[r,i,0] Y_N[p,i,0]; this thread owns
                // Z_{N-1}[zg, zf].  The L2 loads are issued before the barrier.
                const float* xl = xs + off;
                const float* yl = ys + off;
                float d = 0.f;
                for (int i2 = 0; i2 < IL; ++i2) d = fmaf(__ldg(xl + zg + 16 * i2), __ldg(yl + zf + 16 * i2), d);
                bar_named(1, kCT);   // partials visible
                float v = 0.f;
#pragma unroll
                for (int w = 0; w < kCW; ++w) v += zpart[w * kPart + src];
                v *= d;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) red[warp] = v;
                bar_named(1, kCT);   // red visible; partials free
                if (tid == 0) {
                    float s = 0.f;
#pragma unroll
                    for (int w = 0; w < kCW; ++w) s += red[w];
                    a.out[p.b] = s;
                }
            }
        }
    }
}

}  // namespace

bool inner_r16_supported(const InnerArgs& a, bool uniform_r16) {
    if (!uniform_r16 || a.N < 3) return false;
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
