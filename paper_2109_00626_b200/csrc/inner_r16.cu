// inner_r16.cu -- tt_inner specialised for batches whose trains all have the rank profile (1, 16, ..., 16, 1)
// (BASELINE.json C2: N = 8, I = 16, R = 16).  Same sweep as ttc.h / inner_fast.cu:
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :],  out = Z_N.
// Persistent CTAs (three per SM for mode sizes up to 16, two up to 26: three pairs in flight per SM), warp-specialised:
//   * producer warp: TMA bulk copies (cp.async.bulk) of each INTERIOR step's two cores into a kStages-deep ring
//     (one copy per plane into padded planes), full/empty mbarriers;
//   * boundary warp: the two rank-1 cores of each pair (1 KB per core and train for I = 16 -- as a ring stage
//     they would occupy a whole stage for 1/16 of its data and leave the next pair's first interior stage issued
//     one short step ahead of its use), one pair ahead, on the FP32 pipe from global memory:
//       Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q]   (Eq. 12's K = A_x^T A_y), in B-fragment slot order;
//       D[r, p]   = sum_i X_N[r,i,0] Y_N[p,i,0],  so that  Z_N = sum_{r,p} Z_{N-1}[r,p] D[r,p];
//   * 4 compute warps: per interior step the two rank-16 GEMMs of each slice i on the tensor cores (3xTF32
//     mma.sync m16n8k8, ldmatrix for the Y operand, every bound a compile-time constant), slices spread over
//     the warps, partials reduced through shared memory in a fixed order into the next step's B fragments; the
//     last interior step's reduction is fused with the last core (multiply by D, fixed-order block reduction).
// Every core byte is read from HBM exactly once; nothing is written but the result.  Needs N >= 3.
#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

using namespace tc;

// 4 compute warps per CTA and several CTAs per SM (independent pairs in flight, a 4-warp barrier per reduction)
// measured better than 8 warps per CTA: C2 23.7 M (8 warps, 3 stages, 2 CTAs / SM) -> 26.5 M (4 warps, 3 stages,
// 2 CTAs) -> 27.3 M pairs/s (4 warps, 2 stages, 3 CTAs); 2 warps per CTA 24.1 M, 1 warp 9.1 M.
#ifndef TTC_R16_CW
#define TTC_R16_CW 4
#endif
constexpr int kCW = TTC_R16_CW;     // compute warps
constexpr int kCT = 32 * kCW;       // compute threads
constexpr int kSlots = 256;         // zfrag slots (2 x 2 fragments x 64)
constexpr int kSPT = kSlots / kCT;  // slots per compute thread
static_assert(kSlots % kCT == 0, "slots per thread");
constexpr int kPart = 2 * 32 * 4;   // floats of one warp's partial Z' (2 n-tiles, fragment-native)
constexpr int kScrLd = 17;                // row stride of the boundary warp's scratch cores (16 + 1)
constexpr int kScr = 2 * 16 * kScrLd;     // floats of the scratch

struct R16Layout {
    int ps_max;      // plane stride for the largest I
    int x_floats;    // X region of a stage (16 planes)
    int stage_floats;
    int scratch;     // 1: the boundary warp stages its cores in shared memory (I_1, I_N <= 16)
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

// Plane strides: X planes at = 8 mod 32 floats (conflict-free 8-byte B-fragment loads), Y planes at = 4 mod 8
// floats (the 8 rows of an ldmatrix phase fall in 8 distinct 16-byte bank groups).
__host__ __device__ __forceinline__ int ps_x(int floats) { return plane_stride(floats); }
__host__ __device__ __forceinline__ int ps_y(int floats) {
    int ps = (floats + 3) & ~3;
    return (ps & 7) ? ps : ps + 4;
}

// Bulk copy with an L2 evict-first policy: every core byte is read exactly once, so it should not displace
// anything in L2.
__device__ __forceinline__ void bulk_g2s_once(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Producer: stage interior core n (planes of 16 x I floats at the strides above), X planes then Y planes.
__device__ __forceinline__ void r16_issue(const float* xs, const float* ys, int I, float* stage, uint64_t* bar,
                                          const R16Layout& lay, uint64_t pol) {
    const int lane = threadIdx.x & 31;
    const int plane = 16 * I;
    if (lane == 0) mbar_arrive_expect_tx(bar, 4u * 2 * 16 * plane);
    __syncwarp();
    if (lane < 16) bulk_g2s_once(stage + lane * ps_x(plane), xs + (int64_t)lane * plane, 4u * plane, bar, pol);
    else bulk_g2s_once(stage + lay.x_floats + (lane - 16) * ps_y(plane), ys + (int64_t)(lane - 16) * plane, 4u * plane,
                       bar, pol);
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const float* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
// 3xTF32 parts of data read from shared memory: hi = the raw bits (the tensor core truncates to tf32),
// lo = x - trunc(x) exactly.
__device__ __forceinline__ uint32_t lo_trunc(uint32_t x) {
    return __float_as_uint(__uint_as_float(x) - __uint_as_float(x & 0xffffe000u));
}

// U slices of one interior step (mode index i = ui[x]):
//   GEMM-1  Wt[q, r] = sum_p Y[p, i, q] Z[r, p]:   A = Y_i (m = q: plane, k = p: contiguous) by ldmatrix in natural
//           k order; B = Z from zfrag (b0 = Z[8ng + g, 8kf + t], b1 = Z[8ng + g, 8kf + t + 4]).
//   GEMM-2  Zt'[q, s] += sum_r Wt[q, r] X[r, i, s]: A = GEMM-1's C fragments re-read as k-permuted A fragments
//           (k slot t <-> r = 2t, slot t + 4 <-> r = 2t + 1: {c0, c2, c1, c3}); B = X_i with the same permutation,
//           b0, b1 = X[8kb + 2t, i, 8ns + g], X[8kb + 2t + 1, i, 8ns + g]: one 8-byte load lands in fragment order.
// yl: this lane's ldmatrix row address (row q = (lane & 7) + 8 ((lane >> 3) & 1), k offset 4 (lane >> 4)) at i = 0,
// xl: this lane's X address (plane g, element 2t) at i = 0.
template <int U>
__device__ __forceinline__ void r16_units(const float* yl, const float* xl, int psx, const int (&ui)[U],
                                          const BFrag (&zb)[2][2], float (&acc)[2][4]) {
    float w[U][2][4];
#pragma unroll
    for (int x = 0; x < U; ++x) {
        AFrag A[2];
#pragma unroll
        for (int kf = 0; kf < 2; ++kf) {
            ldsm_x4(A[kf].hi, yl + ui[x] * 16 + 8 * kf);
#pragma unroll
            for (int c = 0; c < 4; ++c) A[kf].lo[c] = lo_trunc(A[kf].hi[c]);
        }
#pragma unroll
        for (int ng = 0; ng < 2; ++ng) mma6<true>(w[x][ng], A[0], zb[0][ng], A[1], zb[1][ng]);
    }
#pragma unroll
    for (int x = 0; x < U; ++x) {
        AFrag Aw[2];
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
            const float c4[4] = {w[x][kb][0], w[x][kb][2], w[x][kb][1], w[x][kb][3]};
            Aw[kb] = split_a(c4);
        }
#pragma unroll
        for (int ns = 0; ns < 2; ++ns) {
            BFrag B[2];
#pragma unroll
            for (int kb = 0; kb < 2; ++kb) {
                const uint2 v = *reinterpret_cast<const uint2*>(xl + 8 * ns * psx + ui[x] * 16 + 8 * kb);
                B[kb].hi[0] = v.x;
                B[kb].hi[1] = v.y;
                B[kb].lo[0] = lo_trunc(v.x);
                B[kb].lo[1] = lo_trunc(v.y);
            }
            float tg[4];
            mma6<true>(tg, Aw[0], B[0], Aw[1], B[1]);
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[ns][c] += tg[c];
        }
    }
}

// zfrag slot e = [kf][ng][ln][jj] holds Z[zg, zf] = Z[8 ng + ln/4, 8 kf + ln%4 + 4 jj] (zg on X's bond, zf on Y's):
// the B fragments of the next GEMM-1 (b0 = Z[8ng + g, 8kf + t], b1 = Z[8ng + g, 8kf + t + 4]).
__device__ __forceinline__ void slot_entry(int e, int& zg, int& zf) {
    const int jj = e & 1, ln = (e >> 1) & 31, ng = (e >> 6) & 1, kf = e >> 7;
    zg = 8 * ng + (ln >> 2);
    zf = 8 * kf + (ln & 3) + 4 * jj;
}

constexpr int kStages = 2;   // TMA ring depth (interior steps in flight per CTA)

__global__ void __maxnreg__(96) inner_r16_kernel(const InnerArgs a, const R16Layout lay) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ __align__(8) uint64_t z1full, z1empty, dfull, dempty;
    __shared__ float red[kCW];
    float* stages = smem;
    float* zpart = smem + kStages * lay.stage_floats;   // [kCW][2 n-tiles][32 lanes][4]
    float* zfrag = zpart + kCW * kPart;           // [slot]: B fragments of Z for the next step
    float* z1buf = zfrag + kSlots;                // [slot]: Z_1 of the next pair (boundary warp)
    float* dbuf = z1buf + kSlots;                 // [slot]: sum_i X_N[zg,i,0] Y_N[zf,i,0] of the next pair
    float* scr = lay.scratch ? dbuf + kSlots : nullptr;   // boundary warp: two 16 x kScrLd cores (I_1, I_N <= 16)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N, I0 = a.dims[0], IL = a.dims[N - 1];

    if (threadIdx.x == 0) {
        for (int k = 0; k < kStages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], kCW);
        }
        mbar_init(&z1full, 32);
        mbar_init(&dfull, 32);
        mbar_init(&z1empty, 1);
        mbar_init(&dempty, 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCW) {   // ------------------------------------------------------------------ producer warp
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        int j = 0;
        for (int k = 0;; ++k) {
            const R16Pair p = r16_pair(a, k);
            if (!p.valid) break;
            const float* xs = a.x.cores + p.xo;
            const float* ys = a.y.cores + p.yo;
            int64_t off = 16 * (int64_t)I0;
            for (int n = 1; n < N - 1; ++n, ++j) {
                const int st = j % kStages;
                if (j >= kStages) mbar_wait(&empty[st], ((j / kStages) - 1) & 1);
                const int I = a.dims[n];
                r16_issue(xs + off, ys + off, I, stages + st * lay.stage_floats, &full[st], lay, pol);
                off += 256 * (int64_t)I;
            }
        }
        return;
    }
    if (warp == kCW + 1) {   // ------------------------------------------------------------- boundary warp
        // The two rank-1 cores of each pair on the FP32 pipe, one pair ahead of the compute warps, from global
        // memory (1 KB per core and train for I = 16: a TMA stage would be 1/16 full):
        //   Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q]  (Eq. 12's K = A_x^T A_y)          -> z1buf
        //   D[r, p]   = sum_i X_N[r,i,0] Y_N[p,i,0]  (so that Z_N = sum_{r,p} Z_{N-1}[r,p] D[r,p])  -> dbuf
        int64_t last = 16 * (int64_t)I0;
        for (int n = 1; n < N - 1; ++n) last += 256 * (int64_t)a.dims[n];
        for (int k = 0;; ++k) {
            const R16Pair p = r16_pair(a, k);
            if (!p.valid) break;
            const float* xs = a.x.cores + p.xo;
            const float* ys = a.y.cores + p.yo;
            if (scr) {
                // both cores of a boundary step into the scratch as rows of 16 (+1 pad: conflict-free reads) --
                // all loads of a core pair in flight at once -- then the 256 dot products from shared memory
                //   Z_1: row s of X_1 = X_1[0, :, s] (contiguous), row q of Y_1 likewise
                for (int e = lane; e < 16 * I0; e += 32) {
                    const int s_ = e / I0, i = e - s_ * I0;
                    scr[s_ * kScrLd + i] = __ldg(xs + e);
                    scr[16 * kScrLd + s_ * kScrLd + i] = __ldg(ys + e);
                }
                __syncwarp();
                if (k > 0) mbar_wait(&z1empty, (k - 1) & 1);
                for (int e = lane; e < kSlots; e += 32) {
                    int zg, zf;
                    slot_entry(e, zg, zf);
                    const float* xr = scr + zg * kScrLd;
                    const float* yr = scr + 16 * kScrLd + zf * kScrLd;
                    float d = 0.f;
                    for (int i = 0; i < I0; ++i) d = fmaf(xr[i], yr[i], d);
                    z1buf[e] = d;
                }
                mbar_arrive(&z1full);
                __syncwarp();
                //   D: row r of X_N = X_N[r, :, 0] (stride 16 in memory), row p of Y_N likewise
                const float* xl = xs + last;
                const float* yl = ys + last;
                for (int e = lane; e < 16 * IL; e += 32) {
                    const int r = e & 15, i = e >> 4;
                    scr[r * kScrLd + i] = __ldg(xl + e);
                    scr[16 * kScrLd + r * kScrLd + i] = __ldg(yl + e);
                }
                __syncwarp();
                if (k > 0) mbar_wait(&dempty, (k - 1) & 1);
                for (int e = lane; e < kSlots; e += 32) {
                    int zg, zf;
                    slot_entry(e, zg, zf);
                    const float* xr = scr + zg * kScrLd;
                    const float* yr = scr + 16 * kScrLd + zf * kScrLd;
                    float d = 0.f;
                    for (int i = 0; i < IL; ++i) d = fmaf(xr[i], yr[i], d);
                    dbuf[e] = d;
                }
                __syncwarp();
                mbar_arrive(&dfull);
                continue;
            }
            if (k > 0) mbar_wait(&z1empty, (k - 1) & 1);
            for (int e = lane; e < kSlots; e += 32) {
                int zg, zf;
                slot_entry(e, zg, zf);
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
                z1buf[e] = d;
            }
            mbar_arrive(&z1full);
            if (k > 0) mbar_wait(&dempty, (k - 1) & 1);
            const float* xl = xs + last;
            const float* yl = ys + last;
            for (int e = lane; e < kSlots; e += 32) {
                int zg, zf;
                slot_entry(e, zg, zf);
                float d = 0.f;
                for (int i = 0; i < IL; ++i) d = fmaf(__ldg(xl + zg + 16 * i), __ldg(yl + zf + 16 * i), d);
                dbuf[e] = d;
            }
            mbar_arrive(&dfull);
        }
        return;
    }

    // ------------------------------------------------------------------------------------------ compute
    const int tid = threadIdx.x, lg = lane >> 2, t = lane & 3;
    // this thread's zfrag slots are tid + kCT u; the source of slot (zg, zf) in a warp's fragment-native partial
    // Zt'[q = zf, s = zg] is the C fragment of n-tile zg / 8: lane 4 (zf % 8) + (zg % 8) / 2, element
    // 2 (zf / 8) + zg % 2
    int src[kSPT];
#pragma unroll
    for (int u = 0; u < kSPT; ++u) {
        int zg, zf;
        slot_entry(tid + kCT * u, zg, zf);
        src[u] = ((zg >> 3) * 32 + ((zf & 7) << 2) + ((zg & 7) >> 1)) * 4 + ((zf >> 3) << 1) + (zg & 1);
    }
    const int yrow = (lane & 7) + 8 * ((lane >> 3) & 1), ykoff = 4 * (lane >> 4);

    int j = 0;
    for (int k = 0;; ++k) {
        const R16Pair p = r16_pair(a, k);
        if (!p.valid) break;
        mbar_wait(&z1full, k & 1);   // Z_1 of this pair in z1buf
        for (int n = 1; n < N - 1; ++n, ++j) {
            const int st = j % kStages;
            const int I = a.dims[n];
            // ---- interior step
            const float* zsrc = n == 1 ? z1buf : zfrag;
            BFrag zb[2][2];
#pragma unroll
            for (int kf = 0; kf < 2; ++kf)
#pragma unroll
                for (int ng = 0; ng < 2; ++ng) {
                    const float2 v2 = *reinterpret_cast<const float2*>(zsrc + ((kf * 2 + ng) * 32 + lane) * 2);
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
            const int psx = ps_x(16 * I);
            const float* yl = Y + yrow * ps_y(16 * I) + ykoff;
            const float* xl = X + lg * psx + 2 * t;
            int i = warp;
            for (; i + kCW < I; i += 2 * kCW) {
                const int uu[2] = {i, i + kCW};
                r16_units<2>(yl, xl, psx, uu, zb, acc);
            }
            if (i < I) {
                const int uu[1] = {i};
                r16_units<1>(yl, xl, psx, uu, zb, acc);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            float* zw = zpart + warp * kPart;
#pragma unroll
            for (int h = 0; h < 2; ++h)
                *reinterpret_cast<float4*>(zw + (h * 32 + lane) * 4) = make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]);
            bar_named(1, kCT);   // partials visible; every warp is done with zfrag / z1buf
            if (n == 1 && tid == 0) mbar_arrive(&z1empty);
            float vs[kSPT];
#pragma unroll
            for (int u = 0; u < kSPT; ++u) {
                vs[u] = 0.f;
#pragma unroll
                for (int w = 0; w < kCW; ++w) vs[u] += zpart[w * kPart + src[u]];
            }
            if (n < N - 2) {
#pragma unroll
                for (int u = 0; u < kSPT; ++u) zfrag[tid + kCT * u] = vs[u];
                bar_named(1, kCT);   // next step's B fragments visible; partials free
            } else {
                // ---- last core: Z_N = sum_{r,p} Z_{N-1}[r,p] D[r,p]; this thread owns its slots of Z_{N-1}
                mbar_wait(&dfull, k & 1);
                float v = 0.f;
#pragma unroll
                for (int u = 0; u < kSPT; ++u) v = fmaf(vs[u], dbuf[tid + kCT * u], v);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) red[warp] = v;
                bar_named(1, kCT);   // red visible; partials and dbuf free
                if (tid == 0) {
                    mbar_arrive(&dempty);
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

namespace {
// Shared-memory bytes of a configuration (without the boundary scratch) and the per-CTA budget at `ctas` per SM
// (228 KB less 1 KB reserved and ~0.3 KB static shared memory per CTA).
size_t r16_smem(int stages, int max_dim) {
    return sizeof(float) * (stages * (size_t)16 * (ps_x(16 * max_dim) + ps_y(16 * max_dim)) + kCW * kPart + 3 * kSlots);
}
size_t r16_budget(int ctas) { return (size_t)(228 * 1024 / ctas - 1024 - 320); }
// CTAs per SM with the 2-stage ring: 3 (mode sizes <= 16, C2), else 2 (<= 26); a 3-stage ring at 2 CTAs per SM
// never fits where 2 stages at 3 do not
bool r16_config(int max_dim, int* ctas) {
    for (int c = 3; c >= 2; --c)
        if (r16_smem(kStages, max_dim) <= r16_budget(c)) {
            *ctas = c;
            return true;
        }
    return false;
}
}  // namespace

bool inner_r16_supported(const InnerArgs& a, bool uniform_r16) {
    if (!uniform_r16 || a.N < 3) return false;
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = a.dims[n] > max_dim ? a.dims[n] : max_dim;
    int ctas;
    return r16_config(max_dim, &ctas);
}

cudaError_t launch_inner_r16(const InnerArgs& a, cudaStream_t s) {
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = a.dims[n] > max_dim ? a.dims[n] : max_dim;
    int ctas = 3;
    if (!r16_config(max_dim, &ctas)) return cudaErrorInvalidConfiguration;
    R16Layout lay;
    lay.ps_max = ps_x(16 * max_dim);
    lay.x_floats = 16 * lay.ps_max;
    lay.stage_floats = lay.x_floats + 16 * ps_y(16 * max_dim);
    size_t smem = r16_smem(kStages, max_dim);
    // the boundary warp's scratch only where it still fits the budget
    lay.scratch = (a.dims[0] <= 16 && a.dims[a.N - 1] <= 16 && smem + sizeof(float) * kScr <= r16_budget(ctas)) ? 1 : 0;
    if (lay.scratch) smem += sizeof(float) * kScr;
    auto kern = inner_r16_kernel;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * (kCW + 2), smem)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int grid = a.B < sms * per_sm ? a.B : sms * per_sm;
    kern<<<grid, 32 * (kCW + 2), smem, s>>>(a, lay);
    return cudaGetLastError();
}

}  // namespace ttc
