// inner_r64.cu -- tt_inner specialised for batches whose trains all have the rank profile (1, 64, ..., 64, 1)
// (BASELINE.json C4: N = 16, I = 4, R = 64 -- "the tensor-core path").  Same sweep as ttc.h:
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :],  out = Z_N.
// One persistent CTA per SM, warp-specialised:
//   * producer warp: TMA bulk copies (cp.async.bulk, one per plane) of Y_n into the Y buffer and X_n into the
//     X buffer (one buffer each, 66 KB, planes padded to a stride = 8 mod 32 floats);
//   * 8 compute warps, per interior step:
//       phase 1 (needs Y_n only)  GEMM-1  W^T[(i,q), r] = sum_p Y_n[p,i,q] Z[r,p]   -> W kept in registers;
//                                 the Y buffer is released, Y_{n+1} streams in during phase 2
//       phase 2 (needs X_n only)  GEMM-2  Z'[s, q]    += sum_r X_n[r,i,s] W[r,i,q] -> per-warp partial;
//                                 the X buffer is released, X_{n+1} streams in during the next phase 1
//     warp w owns the 16-column block q in [16 (w/2), 16 (w/2) + 16) and the slices i = w%2, w%2 + 2, ...;
//     the two partials of a block are summed in a fixed order and split (3xTF32 hi / lo) once into the
//     next step's B-fragment layout.  Tensor cores: 3xTF32 mma.sync m16n8k8 (the per-pair chain has no
//     shared operand to batch over, and GEMM-1's M = 16 rows per (i, q-block) unit).
//   * boundary steps (R_0 = 1, R_N = 1) on the FP32 pipe.
#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

using namespace tc;

constexpr int kR = 64;
constexpr int kCW = 8;                 // compute warps
constexpr int kCT = 32 * kCW;
constexpr int kPart = 4 * 2 * 32 * 4;  // one warp's partial Z' block: 4 m-tiles (s) x 2 n-tiles (q) x 32 lanes x 4
constexpr int kZf = 8 * 8 * 32 * 4;    // B fragments of Z: 8 k-blocks (p) x 8 n-tiles (r) x 32 lanes x {hi0,hi1,lo0,lo1}
constexpr int kEnd = 1 << 30;

struct R64Step {
    int b, n, I, flags;   // flags: 1 first step, 2 last step, kEnd: no more steps
};

struct R64Layout {
    int core_floats;   // one padded core buffer (64 planes)
};

struct R64Cursor {
    int k, b, n;
    int64_t xo, yo;
    bool valid;
};

__device__ __forceinline__ void r64_pair(const InnerArgs& a, R64Cursor& c) {
    const int idx = blockIdx.x + c.k * gridDim.x;
    c.valid = idx < a.B;
    if (!c.valid) return;
    c.b = a.order ? __ldg(a.order + idx) : idx;
    c.n = 0;
    c.xo = a.x.offsets ? __ldg(a.x.offsets + c.b) : (int64_t)c.b * a.x.train_elems;
    c.yo = a.y.offsets ? __ldg(a.y.offsets + c.b) : (int64_t)c.b * a.y.train_elems;
}

// Producer: stage one core (interior: 64 planes of I*64 floats at stride ps; boundary: contiguous).
__device__ __forceinline__ void r64_stage(const float* src, int I, bool boundary, float* dst, uint64_t* bar) {
    const int lane = threadIdx.x & 31;
    const int plane = kR * I;
    if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, 4u * (boundary ? plane : kR * plane));
    }
    __syncwarp();
    if (boundary) {
        if (lane == 0) bulk_g2s(dst, src, 4u * plane, bar);
    } else {
        const int ps = plane_stride(plane);
        for (int v = lane; v < kR; v += 32) bulk_g2s(dst + v * ps, src + (int64_t)v * plane, 4u * plane, bar);
    }
}

__global__ void __maxnreg__(168) inner_r64_kernel(const InnerArgs a, const R64Layout lay) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t xfull, yfull, xempty, yempty;
    __shared__ __align__(16) R64Step ring[2];
    __shared__ float red[kCW];
    float* xbuf = smem;
    float* ybuf = smem + lay.core_floats;
    float* zpart = ybuf + lay.core_floats;                              // [kCW][kPart]
    uint32_t* zfrag = reinterpret_cast<uint32_t*>(zpart + kCW * kPart);  // [kf][ng][lane][4]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&xfull, 1);
        mbar_init(&yfull, 1);
        mbar_init(&xempty, kCW);
        mbar_init(&yempty, kCW);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kCW) {   // ------------------------------------------------------------------ producer warp
        R64Cursor c;
        c.k = 0;
        r64_pair(a, c);
        for (int j = 0;; ++j) {
            if (j >= 1) mbar_wait(&yempty, (j - 1) & 1);
            if (!c.valid) {
                if (lane == 0) {
                    ring[j & 1].flags = kEnd;
                    mbar_arrive(&yfull);
                }
                break;
            }
            const int I = a.dims[c.n];
            const bool first = c.n == 0, last = c.n == a.N - 1;
            if (lane == 0) {
                R64Step s;
                s.b = c.b; s.n = c.n; s.I = I; s.flags = (first ? 1 : 0) | (last ? 2 : 0);
                ring[j & 1] = s;
            }
            __syncwarp();
            r64_stage(a.y.cores + c.yo, I, first || last, ybuf, &yfull);
            if (j >= 1) mbar_wait(&xempty, (j - 1) & 1);
            r64_stage(a.x.cores + c.xo, I, first || last, xbuf, &xfull);
            const int64_t core = (first || last) ? (int64_t)kR * I : (int64_t)kR * kR * I;
            c.xo += core;
            c.yo += core;
            if (++c.n == a.N) {
                ++c.k;
                r64_pair(a, c);
            }
        }
        return;
    }

    // ------------------------------------------------------------------------------------------ compute
    const int tid = threadIdx.x, lg = lane >> 2, t = lane & 3;
    const int mq = warp >> 1, ipar = warp & 1;   // this warp's q block and slice parity
    for (int j = 0;; ++j) {
        mbar_wait(&yfull, j & 1);
        const R64Step si = ring[j & 1];
        if (si.flags == kEnd) break;
        const int I = si.I;
        if (si.flags & 1) {
            // ---- first step: Z_1[s, q] = sum_i X_1[0,i,s] Y_1[0,i,q] (Eq. 12's K) -> B fragments (hi, lo)
            mbar_wait(&xfull, j & 1);
            for (int slot = tid; slot < 8 * 8 * 32; slot += kCT) {
                const int ln = slot & 31, ng = (slot >> 5) & 7, kf = slot >> 8;
                const int g = 8 * ng + (ln >> 2), f0 = 8 * kf + 2 * (ln & 3);
                float d0 = 0.f, d1 = 0.f;
                for (int i = 0; i < I; ++i) {
                    const float xv = xbuf[i + I * g];
                    d0 = fmaf(xv, ybuf[i + I * f0], d0);
                    d1 = fmaf(xv, ybuf[i + I * (f0 + 1)], d1);
                }
                const uint32_t h0 = hi_bits(d0), h1 = hi_bits(d1);
                reinterpret_cast<uint4*>(zfrag)[slot] = make_uint4(h0, h1, lo_bits(d0, h0), lo_bits(d1, h1));
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&yempty);
                mbar_arrive(&xempty);
            }
            bar_named(1, kCT);
            continue;
        }
        if (si.flags & 2) {
            // ---- last step: Z_N = sum_{r,p} Z[r,p] sum_i X_N[r,i] Y_N[p,i]
            mbar_wait(&xfull, j & 1);
            float v = 0.f;
            for (int slot = tid; slot < 8 * 8 * 32; slot += kCT) {
                const int ln = slot & 31, ng = (slot >> 5) & 7, kf = slot >> 8;
                const int g = 8 * ng + (ln >> 2), f0 = 8 * kf + 2 * (ln & 3);
                const uint4 zf = reinterpret_cast<const uint4*>(zfrag)[slot];
                const float z0 = __uint_as_float(zf.x) + __uint_as_float(zf.z);   // hi + lo = Z exactly
                const float z1 = __uint_as_float(zf.y) + __uint_as_float(zf.w);
                float d0 = 0.f, d1 = 0.f;
                for (int i = 0; i < I; ++i) {
                    const float xv = xbuf[g + kR * i];
                    d0 = fmaf(xv, ybuf[f0 + kR * i], d0);
                    d1 = fmaf(xv, ybuf[f0 + 1 + kR * i], d1);
                }
                v = fmaf(z0, d0, v);
                v = fmaf(z1, d1, v);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&yempty);
                mbar_arrive(&xempty);
            }
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
        // ---- interior step: this warp's slices i = ipar, ipar + 2, ... (two at a time), q block mq
        const int ps = plane_stride(kR * I);
        float acc[4][2][4];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[m][h][c] = 0.f;
        bool x_ready = false;
        for (int i0 = ipar; i0 < I; i0 += 4) {
            const bool two = i0 + 2 < I;
            const int iu[2] = {i0, two ? i0 + 2 : i0};
            // ---- phase 1: GEMM-1  w[x][ng] = sum_kf A_Y(x, kf) B_Z(kf, ng), two k-blocks per tensor-core group
            float w[2][8][4];
            const float* yp[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) yp[x] = ybuf + (16 * mq + lg) * ps + iu[x] * kR + 2 * t;
#pragma unroll
            for (int kf = 0; kf < 8; kf += 2) {
                AFrag A[2][2];   // [unit][sub]
#pragma unroll
                for (int x = 0; x < 2; ++x)
#pragma unroll
                    for (int sub = 0; sub < 2; ++sub) {
                        const float2 a1 = *reinterpret_cast<const float2*>(yp[x] + 8 * (kf + sub));
                        const float2 a2 = *reinterpret_cast<const float2*>(yp[x] + 8 * ps + 8 * (kf + sub));
                        const float fa[4] = {a1.x, a2.x, a1.y, a2.y};
                        A[x][sub] = split_a_trunc(fa);
                    }
#pragma unroll
                for (int ng = 0; ng < 8; ++ng) {
                    BFrag B[2];
#pragma unroll
                    for (int sub = 0; sub < 2; ++sub) {
                        const uint4 zf = reinterpret_cast<const uint4*>(zfrag)[((kf + sub) * 8 + ng) * 32 + lane];
                        B[sub].hi[0] = zf.x; B[sub].hi[1] = zf.y; B[sub].lo[0] = zf.z; B[sub].lo[1] = zf.w;
                    }
#pragma unroll
                    for (int x = 0; x < 2; ++x) {
                        if (x == 1 && !two) break;
                        float tg[4];
                        mma6<true>(tg, A[x][0], B[0], A[x][1], B[1]);
#pragma unroll
                        for (int c = 0; c < 4; ++c) w[x][ng][c] = (kf == 0) ? tg[c] : w[x][ng][c] + tg[c];
                    }
                }
            }
            if (i0 + 4 >= I) {   // the warp's last GEMM-1 of this step: release the Y buffer
                __syncwarp();
                if (lane == 0) mbar_arrive(&yempty);
            }
            if (!x_ready) {
                mbar_wait(&xfull, j & 1);
                x_ready = true;
            }
            // ---- phase 2: GEMM-2  acc[mg][h] += sum_kg A_X(mg, kg) B_W(kg, h),  B_W(kg, h) = w[kg][2h + j]
            // per k-block pair: 8 independent (mg, h) tensor-core chains over (unit, sub), then one FADD each
#pragma unroll
            for (int kg = 0; kg < 8; kg += 2) {
                float tg[4][2][4];
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    if (x == 1 && !two) break;
                    BFrag Bw[2][2];   // [sub][h]
#pragma unroll
                    for (int sub = 0; sub < 2; ++sub)
#pragma unroll
                        for (int h = 0; h < 2; ++h) Bw[sub][h] = split_b(w[x][kg + sub][2 * h], w[x][kg + sub][2 * h + 1]);
#pragma unroll
                    for (int mg = 0; mg < 4; ++mg) {
                        const float* xp = xbuf + (16 * mg + lg) * ps + iu[x] * kR + 2 * t + 8 * kg;
#pragma unroll
                        for (int sub = 0; sub < 2; ++sub) {
                            const float2 a1 = *reinterpret_cast<const float2*>(xp + 8 * sub);
                            const float2 a2 = *reinterpret_cast<const float2*>(xp + 8 * ps + 8 * sub);
                            const float ga[4] = {a1.x, a2.x, a1.y, a2.y};
                            const AFrag A = split_a_trunc(ga);
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                if (x == 0 && sub == 0) mma3<true>(tg[mg][h], A, Bw[sub][h]);
                                else mma3<false>(tg[mg][h], A, Bw[sub][h]);
                            }
                        }
                    }
                }
#pragma unroll
                for (int mg = 0; mg < 4; ++mg)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[mg][h][c] += tg[mg][h][c];
            }
        }
        if (ipar >= I) {   // (I < 2) this warp had no slice: still release / acquire
            if (lane == 0) mbar_arrive(&yempty);
            mbar_wait(&xfull, j & 1);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty);
        // ---- partial Z'[s, q-block] (fragment-native) -> reduce pairs of warps -> next step's B fragments
        float* zw = zpart + warp * kPart;
#pragma unroll
        for (int mg = 0; mg < 4; ++mg)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                *reinterpret_cast<float4*>(zw + ((mg * 2 + h) * 32 + lane) * 4) =
                    make_float4(acc[mg][h][0], acc[mg][h][1], acc[mg][h][2], acc[mg][h][3]);
        bar_named(1, kCT);
        for (int slot = tid; slot < 8 * 8 * 32; slot += kCT) {
            // slot (kf, ng, ln): Z[g, f0 + jj] with g = 8 ng + ln/4 (X bond), f0 = 8 kf + 2 (ln%4) (Y bond)
            const int ln = slot & 31, ng = (slot >> 5) & 7, kf = slot >> 8;
            const int g = 8 * ng + (ln >> 2), f0 = 8 * kf + 2 * (ln & 3);
            const int qb = f0 >> 4;   // q block -> warps 2 qb, 2 qb + 1
            const int mg = g >> 4, hh = (g >> 3) & 1, h = (f0 >> 3) & 1;
            const int l2 = ((g & 7) << 2) | ((f0 & 7) >> 1);
            const int off = ((mg * 2 + h) * 32 + l2) * 4 + (hh << 1);   // + jj
            const float2 v0 = *reinterpret_cast<const float2*>(zpart + (2 * qb) * kPart + off);
            const float2 v1 = *reinterpret_cast<const float2*>(zpart + (2 * qb + 1) * kPart + off);
            const float z0 = v0.x + v1.x, z1 = v0.y + v1.y;
            const uint32_t h0 = hi_bits(z0), h1 = hi_bits(z1);
            reinterpret_cast<uint4*>(zfrag)[slot] = make_uint4(h0, h1, lo_bits(z0, h0), lo_bits(z1, h1));
        }
        bar_named(1, kCT);
    }
}

}  // namespace

bool inner_r64_supported(const InnerArgs& a, bool uniform_r64) {
    if (!uniform_r64 || a.N < 2) return false;
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = a.dims[n] > max_dim ? a.dims[n] : max_dim;
    const size_t smem = sizeof(float) * (2 * (size_t)kR * plane_stride(kR * max_dim) + kCW * kPart + kZf);
    return smem <= 226 * 1024;
}

cudaError_t launch_inner_r64(const InnerArgs& a, cudaStream_t s) {
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = a.dims[n] > max_dim ? a.dims[n] : max_dim;
    R64Layout lay;
    lay.core_floats = kR * plane_stride(kR * max_dim);
    const size_t smem = sizeof(float) * (2 * (size_t)lay.core_floats + kCW * kPart + kZf);
    cudaError_t e = cudaFuncSetAttribute(inner_r64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    const int grid = a.B < sms ? a.B : sms;
    inner_r64_kernel<<<grid, 32 * (kCW + 1), smem, s>>>(a, lay);
    return cudaGetLastError();
}

}  // namespace ttc
