// EXPERIMENT, not built (tools/experiments/): measured slower than inner_r16.cu (DESIGN.md §6 C2 notes) and kept
// for the record.  To try it: copy into csrc/, declare inner_r16w_supported / launch_inner_r16w in ttc_internal.h
// and dispatch to it for uniform rank-16 batches.
// inner_r16w.cu -- tt_inner for uniform rank-16 trains (BASELINE.json C2: N = 8, I = 16, R = 16), ONE WARP PER PAIR.
// Same sweep and the same 3xTF32 mma.sync arithmetic as inner_r16.cu (ttc.h; Fig. 1b / Eq. 12 chained):
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :],  out = Z_N,
// but a warp sweeps its pair alone, slice by slice, so that nothing is shared between warps (no CTA barrier, no
// cross-warp reduction) and many pairs are in flight per SM:
//   * staging: each warp's lane 0 streams its pair's slices (X_n[:, i, :], Y_n[:, i, :]: 16 x 16 floats each, rows
//     1 KB apart in HBM) into a private ring of kSlots slots with TMA tensor copies; one 3-D map per operand buffer:
//     (16 floats, 16 rows @ 64 I bytes, n / 4 @ 16 bytes), boxes (20 or 24, 16, 1) whose last 4 / 8 floats per row
//     lie past the first dimension (zero-filled, never read from HBM): rows land 80 B (Y: ldmatrix, 8 rows in 8
//     distinct bank groups) or 96 B (X: 8-byte fragment loads, conflict-free per half-warp) apart;
//   * boundary cores (X_1, Y_1 and X_N, Y_N, 16 I floats each, contiguous) by 1-D bulk copies into two buffers,
//     refilled for the warp's next pair as soon as this pair no longer needs them;
//   * per interior step: Z as the B fragments of GEMM-1 in registers; per pair of slices GEMM-1 (W = Z Y_i) and
//     GEMM-2 (Z' += X_i^T W) as in inner_r16.cu; at the step end Z' (C fragments) goes through 1 KB of the warp's
//     shared memory to become the next step's B fragments; the first step's Z_1 = A_x^T A_y and the last step's
//     D = X_N . Y_N (Eq. 12) are formed by each lane for exactly the 8 entries it needs.
// Needs N >= 3, every interior mode of the same size I <= 16, 16-byte aligned cores (host-checked).
#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

using namespace tc;

#ifndef TTC_R16W_SLOTS
#define TTC_R16W_SLOTS 4
#endif
#ifndef TTC_R16W_WARPS
#define TTC_R16W_WARPS 4
#endif
constexpr int kSlots = TTC_R16W_SLOTS;       // ring slots (slices staged ahead, 2 consumed at a time)
constexpr int kYLd = 20, kXLd = 24;          // row strides of the staged Y / X slice tiles (floats)
constexpr int kYTile = 16 * kYLd, kXTile = 16 * kXLd;
constexpr int kSlotFloats = kYTile + kXTile; // 704 floats = 2816 B (a multiple of 128)
constexpr int kWarps = TTC_R16W_WARPS;       // independent warps per CTA (one pair each at a time)

struct R16wLayout {
    int bnd;          // floats of one boundary buffer (2 cores)
    int warp_floats;  // shared floats per warp
};

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const float* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ uint32_t lo_trunc(uint32_t x) {
    return __float_as_uint(__uint_as_float(x) - __uint_as_float(x & 0xffffe000u));
}

// U slices: yl[x] = this lane's ldmatrix row address in slice x's Y tile, xl[x] its X fragment address (see
// inner_r16.cu r16_units: identical arithmetic with per-slice tiles instead of planes).
template <int U>
__device__ __forceinline__ void slices(const float* const (&yl)[U], const float* const (&xl)[U],
                                       const BFrag (&zb)[2][2], float (&acc)[2][4]) {
    float w[U][2][4];
#pragma unroll
    for (int x = 0; x < U; ++x) {
        AFrag A[2];
#pragma unroll
        for (int kf = 0; kf < 2; ++kf) {
            ldsm_x4(A[kf].hi, yl[x] + 8 * kf);
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
                const uint2 v = *reinterpret_cast<const uint2*>(xl[x] + 8 * ns * kXLd + 8 * kb);
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

// The slice stream of one warp: its pairs blockIdx.x * kWarps + warp + k * (gridDim.x * kWarps), interior cores
// n = 1 .. N-2, slices i = 0 .. I-1, in consumption order.
struct Stream {
    int k, n, i;      // pair ordinal, core, slice
    int b;            // pair index (-1: exhausted)
    int64_t xo, yo;   // offsets of core n
};
__device__ __forceinline__ int pair_index(const InnerArgs& a, int k) {
    const int idx = (int)(blockIdx.x * kWarps + (threadIdx.x >> 5)) + k * (int)(gridDim.x * kWarps);
    return idx < a.B ? (a.order ? __ldg(a.order + idx) : idx) : -1;
}
__device__ __forceinline__ int64_t fbase(const TrainDev& t, int b) {
    return t.offsets ? __ldg(t.offsets + b) : (int64_t)b * t.train_elems;
}
__device__ __forceinline__ void stream_pair(const InnerArgs& a, Stream& s) {
    s.b = pair_index(a, s.k);
    if (s.b < 0) return;
    s.n = 1;
    s.i = 0;
    s.xo = fbase(a.x, s.b) + 16 * (int64_t)a.dims[0];
    s.yo = fbase(a.y, s.b) + 16 * (int64_t)a.dims[0];
}
__device__ __forceinline__ void stream_next(const InnerArgs& a, Stream& s, int I) {
    if (++s.i < I) return;
    s.i = 0;
    s.xo += 256 * (int64_t)I;
    s.yo += 256 * (int64_t)I;
    if (++s.n < a.N - 1) return;
    ++s.k;
    stream_pair(a, s);
}

// boundary cores of pair b: first (X_1, Y_1: 16 I_1 floats each) or last (X_N, Y_N: 16 I_N floats each)
__device__ __forceinline__ void issue_bnd(const InnerArgs& a, int b, bool last, float* dst, uint64_t* bar) {
    const int I = last ? a.dims[a.N - 1] : a.dims[0];
    const uint32_t bytes = 4u * 16u * (uint32_t)I;
    const int64_t xo = fbase(a.x, b) + (last ? a.x.train_elems - 16 * I : 0);
    const int64_t yo = fbase(a.y, b) + (last ? a.y.train_elems - 16 * I : 0);
    mbar_arrive_expect_tx(bar, 2 * bytes);
    bulk_g2s(dst, a.x.cores + xo, bytes, bar);
    bulk_g2s(dst + 16 * I, a.y.cores + yo, bytes, bar);
}

__global__ void __launch_bounds__(32 * kWarps) inner_r16w_kernel(const InnerArgs a, const R16wLayout lay,
                                                                 const __grid_constant__ CUtensorMap tmx,
                                                                 const __grid_constant__ CUtensorMap tmy) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t bars[kWarps][kSlots + 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    float* ring = smem + (size_t)warp * lay.warp_floats;          // kSlots x (Y tile, X tile)
    float* zp = ring + kSlots * kSlotFloats;                       // 256 floats: Z' in C-fragment order
    float* bf = zp + 256;                                          // first cores (X_1, Y_1)
    float* bl = bf + lay.bnd;                                      // last cores (X_N, Y_N)
    uint64_t* full = bars[warp];
    uint64_t* bfull = bars[warp] + kSlots;                         // [0]: first cores, [1]: last cores
    const int N = a.N, I = a.dims[1], I0 = a.dims[0], IL = a.dims[N - 1];
    const int per_pair = (N - 2) * I;                              // slices per pair

    if (lane == 0) {
        for (int i = 0; i < kSlots + 2; ++i) mbar_init(full + i, 1);
        fence_mbar_init();
    }
    __syncwarp();
    Stream is;                 // issue cursor (lane 0's view is the one used; every lane tracks it identically)
    is.k = 0;
    stream_pair(a, is);
    if (is.b < 0) return;
    uint32_t issued = 0;
    auto issue_one = [&]() {   // the next slice of the stream into slot issued % kSlots (lane 0 issues)
        if (is.b < 0) return;
        if (lane == 0) {
            float* slot = ring + (issued % kSlots) * kSlotFloats;
            uint64_t* bar = full + issued % kSlots;
            fence_proxy_async();
            mbar_arrive_expect_tx(bar, 4u * kSlotFloats);
            tma_3d(slot, &tmy, 0, 0, (int)((is.yo + 16 * is.i) >> 2), bar);
            tma_3d(slot + kYTile, &tmx, 0, 0, (int)((is.xo + 16 * is.i) >> 2), bar);
        }
        ++issued;
        stream_next(a, is, I);
    };
    if (lane == 0) {
        issue_bnd(a, is.b, false, bf, bfull);
        issue_bnd(a, is.b, true, bl, bfull + 1);
    }
    for (int s = 0; s < kSlots; ++s) issue_one();

    // the zp source of Z entry (zg, zf) (Zt'[q = zf, s = zg] as C fragments: lane 4 (zf % 8) + (zg % 8) / 2,
    // element 2 (zf / 8) + zg % 2); this lane's B-fragment entries: zg = 8 ng + g, zf = 8 kf + t + 4 jj
    int src[2][2][2];
#pragma unroll
    for (int kf = 0; kf < 2; ++kf)
#pragma unroll
        for (int ng = 0; ng < 2; ++ng)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int zg = 8 * ng + g, zf = 8 * kf + t + 4 * jj;
                src[kf][ng][jj] = ((zg >> 3) * 32 + ((zf & 7) << 2) + ((zg & 7) >> 1)) * 4 + ((zf >> 3) << 1) + (zg & 1);
            }
    const int yrow = (lane & 7) + 8 * ((lane >> 3) & 1), ykoff = 4 * (lane >> 4);
    uint32_t consumed = 0;
    for (int k = 0;; ++k) {
        const int b = pair_index(a, k);
        if (b < 0) break;
        // ---- first step: Z_1[zg][zf] = sum_i X_1[0, i, zg] Y_1[0, i, zf] (Eq. 12's K) for this lane's 8 entries
        mbar_wait(bfull, k & 1);
        BFrag zb[2][2];
        {
            float zv[2][2][2];
#pragma unroll
            for (int kf = 0; kf < 2; ++kf)
#pragma unroll
                for (int ng = 0; ng < 2; ++ng)
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const float* xr = bf + I0 * (8 * ng + g);
                        const float* yr = bf + 16 * I0 + I0 * (8 * kf + t + 4 * jj);
                        float d = 0.f;
                        for (int i = 0; i < I0; ++i) d = fmaf(xr[i], yr[i], d);
                        zv[kf][ng][jj] = d;
                    }
#pragma unroll
            for (int kf = 0; kf < 2; ++kf)
#pragma unroll
                for (int ng = 0; ng < 2; ++ng) zb[kf][ng] = split_b(zv[kf][ng][0], zv[kf][ng][1]);
        }
        __syncwarp();   // the first cores are read: refill with the next pair's
        {
            const int nb = pair_index(a, k + 1);
            if (nb >= 0 && lane == 0) issue_bnd(a, nb, false, bf, bfull);
        }
        for (int n = 1; n < N - 1; ++n) {
            float acc[2][4];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[h][c] = 0.f;
            int i = 0;
            for (; i + 1 < I; i += 2) {
                const float* ys[2];
                const float* xs[2];
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const uint32_t c = consumed + x;
                    mbar_wait(full + c % kSlots, (c / kSlots) & 1);
                    const float* slot = ring + (c % kSlots) * kSlotFloats;
                    ys[x] = slot + yrow * kYLd + ykoff;
                    xs[x] = slot + kYTile + g * kXLd + 2 * t;
                }
                slices<2>(ys, xs, zb, acc);
                __syncwarp();
                consumed += 2;
                issue_one();
                issue_one();
            }
            if (i < I) {
                mbar_wait(full + consumed % kSlots, (consumed / kSlots) & 1);
                const float* slot = ring + (consumed % kSlots) * kSlotFloats;
                const float* ys[1] = {slot + yrow * kYLd + ykoff};
                const float* xs[1] = {slot + kYTile + g * kXLd + 2 * t};
                slices<1>(ys, xs, zb, acc);
                __syncwarp();
                consumed += 1;
                issue_one();
            }
            // ---- Z_n: C fragments -> the warp's shared memory -> this lane's entries
#pragma unroll
            for (int h = 0; h < 2; ++h)
                *reinterpret_cast<float4*>(zp + (h * 32 + lane) * 4) = make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]);
            __syncwarp();
            float zv[2][2][2];
#pragma unroll
            for (int kf = 0; kf < 2; ++kf)
#pragma unroll
                for (int ng = 0; ng < 2; ++ng)
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) zv[kf][ng][jj] = zp[src[kf][ng][jj]];
            __syncwarp();   // zp free for the next step
            if (n < N - 2) {
#pragma unroll
                for (int kf = 0; kf < 2; ++kf)
#pragma unroll
                    for (int ng = 0; ng < 2; ++ng) zb[kf][ng] = split_b(zv[kf][ng][0], zv[kf][ng][1]);
            } else {
                // ---- last core: Z_N = sum_{r,p} Z_{N-1}[r,p] D[r,p], D[r,p] = sum_i X_N[r,i,0] Y_N[p,i,0]
                mbar_wait(bfull + 1, k & 1);
                float v = 0.f;
#pragma unroll
                for (int kf = 0; kf < 2; ++kf)
#pragma unroll
                    for (int ng = 0; ng < 2; ++ng)
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const int zg = 8 * ng + g, zf = 8 * kf + t + 4 * jj;
                            float d = 0.f;
                            for (int ii = 0; ii < IL; ++ii) d = fmaf(bl[zg + 16 * ii], bl[16 * IL + zf + 16 * ii], d);
                            v = fmaf(zv[kf][ng][jj], d, v);
                        }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) a.out[b] = v;
                __syncwarp();   // the last cores are read: refill with the next pair's
                const int nb = pair_index(a, k + 1);
                if (nb >= 0 && lane == 0) issue_bnd(a, nb, true, bl, bfull + 1);
            }
        }
    }
    (void)per_pair;
}

}  // namespace

bool inner_r16w_supported(const InnerArgs& a, bool uniform_r16, bool aligned16, int64_t nx, int64_t ny) {
    if (!uniform_r16 || !aligned16 || a.N < 3 || !encode_fn()) return false;
    const int I = a.dims[1];
    if (I < 1 || I > 16) return false;
    for (int n = 1; n < a.N - 1; ++n)
        if (a.dims[n] != I) return false;
    if (a.dims[0] > 64 || a.dims[a.N - 1] > 64) return false;
    return nx / 4 < (int64_t(1) << 31) && ny / 4 < (int64_t(1) << 31);
}

cudaError_t launch_inner_r16w(const InnerArgs& a, int64_t nx, int64_t ny, cudaStream_t s) {
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const int I = a.dims[1];
    CUtensorMap tmx, tmy;
    for (int buf = 0; buf < 2; ++buf) {
        const cuuint64_t dims[3] = {16, 16, (cuuint64_t)((buf ? ny : nx) / 4)};
        const cuuint64_t strides[2] = {(cuuint64_t)64 * I, 16};   // row (s or q) stride 16 I floats; 16-byte units
        const cuuint32_t box[3] = {(cuuint32_t)(buf ? kYLd : kXLd), 16, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(buf ? &tmy : &tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(buf ? a.y.cores : a.x.cores),
                dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    R16wLayout lay;
    const int bmax = a.dims[0] > a.dims[a.N - 1] ? a.dims[0] : a.dims[a.N - 1];
    lay.bnd = 2 * 16 * bmax;
    lay.warp_floats = (kSlots * kSlotFloats + 256 + 2 * lay.bnd + 31) & ~31;   // 128-byte aligned per warp
    const size_t smem = sizeof(float) * (size_t)kWarps * lay.warp_floats;
    cudaError_t e = cudaFuncSetAttribute(inner_r16w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(inner_r16w_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess)
        return e;
    int dev = 0, sms = 0, occ = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, inner_r16w_kernel, 32 * kWarps, smem)) != cudaSuccess)
        return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int ctas_needed = (a.B + kWarps - 1) / kWarps;
    const int grid = ctas_needed < sms * occ ? ctas_needed : sms * occ;
    inner_r16w_kernel<<<grid, 32 * kWarps, smem, s>>>(a, lay, tmx, tmy);
    return cudaGetLastError();
}

}  // namespace ttc
