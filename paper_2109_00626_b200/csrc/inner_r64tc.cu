// inner_r64tc.cu -- tt_inner for uniform rank-64 trains with mode sizes I_n = 4 (BASELINE.json C4: N = 16, I = 4,
// R = 64, "the tensor-core path") on the 5th-generation tensor cores: tcgen05.mma kind::tf32 with the
// accumulators in tensor memory, operands staged by TMA (cp.async.bulk.tensor) in the 128-byte-swizzled K-major
// layout the MMA reads.  Same sweep as ttc.h:
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :]  (Fig. 1b / Eq. 12 chained),  out = Z_N.
//
// Interior step n, in two GEMM families (Eq. 2 layout: Y_n[p, i, q] at p + 64 i + 256 q, X_n[r, i, s] likewise):
//   GEMM-1, per half h (slices i = 2h, 2h+1), M = 128:
//       D1_h[m = q + 64 i'][r] = sum_p Y_n[p, 2h+i', q] Z[r][p]        (= W_i[r][q], W_i = Z Y_n[:, i, :])
//       A = the Y_n slice pair as 128 rows x 64 p (a 3-D TMA box: p fastest, then q, then i'), B = Z (64 r x 64 p)
//   GEMM-2, per slice i, M = 128 (the raw rows and the lo rows of A stacked):
//       D2[s][q] += sum_r X_n[r, i, s] W_i[r][q]                        (= Z_n after the four slices)
//       A = [X_n[:, i, :]^T raw; its lo part] as 128 rows (8-row groups alternating, 2-D TMA boxes of 8 rows s x
//       32 r), B = W_i (64 q x 64 r, written by threads); a raw row's and its lo row's sums are added by a shuffle
// 3xTF32: an input core value x (TMA-staged) is fed as its raw bits (the tensor core truncates them to tf32 --
// measured, tools/tc05_probe.cu) and as lo = RN_tf32(x - trunc_tf32(x)); the operands the threads write (Z, W)
// as hi = RN_tf32(x) and lo = x - hi; a.b ~ a_hi b_hi + a_lo b_hi + a_hi b_lo with every dropped or rounded term of
// random sign.  Accumulation stays in TMEM over the whole K (measured as accurate as
// sequential fp32 round-to-nearest, tools/tc05_probe.cu).
//
// Warp roles (one persistent CTA per SM, pairs assigned statically):
//   warp 0  TMA producer: 12 ring entries per step (4 Y tiles of 16 KB, 8 X K-chunks of 8 KB) into a 4-slot ring
//           (+ the pair's boundary cores, 4 KB)
//   warp 1  TMEM allocator and MMA issuer (one thread)
//   warps 2-5 epilogue warps (one per TMEM sub-partition): the D1 -> W (hi, lo) and D2 -> Z (hi, lo)
//            epilogues through tcgen05.ld (partial accumulators summed in fp32), the boundary steps
//            (Z_1 = A_x^T A_y, Eq. 12, and the final scalar) on the FP32 pipe
//   warps 6-7 lo workers: the lo parts of the staged inputs (Y: 3-buffer lo ring; X: into the entry's own slot)
#include <cuda.h>
#include <cstdio>

#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

using namespace tc;

constexpr int kTile = 16384;                      // bytes of one ring slot
#ifndef TTC_R64TC_RAW
#define TTC_R64TC_RAW 4
#endif
#ifndef TTC_R64TC_LO
#define TTC_R64TC_LO 3
#endif
constexpr int kRaw = TTC_R64TC_RAW, kLo = TTC_R64TC_LO;   // ring depths (staged entries / the Y entries' lo parts)
#ifndef TTC_R64TC_LO_WARPS
#define TTC_R64TC_LO_WARPS 2
#endif
constexpr int kLoWarps = TTC_R64TC_LO_WARPS;       // lo workers (warps 6 ..); 4 measured 0.94M vs 1.69M pairs/s
                                                   // (168 registers: the epilogue spills)
constexpr int kThreads = 32 * (6 + kLoWarps);      // TMA, MMA, 4 epilogue warps, the lo workers
// ring entries per interior step: 4 Y tiles (a half's K-chunk: 128 rows x 32 p, 16 KB; its lo part in the lo ring),
// then 8 X entries (slice i, K-chunk kc: 64 rows s x 32 r, 8 KB) whose lo parts share the slot: 8-row groups
// alternate raw, lo, raw, lo ... 1 KB each, so that GEMM-2's A operand [X_i^T raw; X_i^T lo] is ONE M = 128
// operand (8-row groups 1 KB apart) and a raw row and its lo row sit 8 TMEM lanes apart in the same warp
constexpr int kYPerStep = 4, kEntriesPerStep = 12;

// shared-memory layout (bytes from the 1024-aligned base)
constexpr int kOffRaw = 0;
constexpr int kOffLo = kOffRaw + kRaw * kTile;
// B operands written by the threads (32 KB each): per 32-wide K-chunk kc, 64 hi rows then 64 lo rows (16 KB), so
// that one N = 128 MMA reads [B_hi | B_lo] and one N = 64 MMA reads B_hi
constexpr int kOffB2 = kOffLo + kLo * kTile;      // 2 buffers: W_i as the GEMM-2 B operand (buffer i & 1)
constexpr int kOffB1 = kOffB2 + 4 * kTile;        // Z as the GEMM-1 B operand
constexpr int kOffBnd = kOffB1 + 2 * kTile;       // 2 buffers x {X_1, Y_1, X_N, Y_N} x 1 KB
constexpr int kOffRed = kOffBnd + 2 * 4096;       // 4 floats: the final reduction
constexpr int kOffBar = kOffRed + 64;
// barrier indices
constexpr int FULL = 0, EMPTY = FULL + kRaw, LO_READY = EMPTY + kRaw, LO_FREE = LO_READY + kRaw,
              D1_FULL = LO_FREE + kLo, D1_EMPTY = D1_FULL + 2, B2_READY = D1_EMPTY + 2, B2_FREE = B2_READY + 2,
              D2_FULL = B2_FREE + 2, B1_READY = D2_FULL + 1, BND_FULL = B1_READY + 1, BND_EMPTY = BND_FULL + 2,
              D2P_FULL = BND_EMPTY + 2, D2P_EMPTY = D2P_FULL + 2;
constexpr int kNumBars = D2P_EMPTY + 2;
constexpr int kSmemBytes = kOffBar + 8 * kNumBars + 16 + 1024;   // + TMEM address slot + alignment slack
static_assert(kSmemBytes <= 227 * 1024, "shared memory");

// TMEM columns (512 allocated).  The tensor core's accumulation into TMEM truncates (measured: -5.6e-8 relative per
// accumulating MMA on positive sums, tools/tc05_probe.cu), so long chains are split: the large a_hi b_hi products
// accumulate in short chains -- GEMM-1 8 MMAs per half, GEMM-2 4 per (slice, K-chunk) -- and the small cross terms
// (2^-11 smaller, their truncation negligible) in separate accumulators; the converters add the partials in fp32
// round-to-nearest.
// Each accumulator is a 128-column block: a_hi b_hi in columns 0..63, the cross terms in 64..127 (one N = 128 MMA
// a_hi [b_hi | b_lo] writes both, one N = 64 MMA adds a_lo b_hi to the second half).
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kD1 = 0;       // + 128 h: GEMM-1 of half h (M = 128)
constexpr uint32_t kD2 = 256;     // + 128 (i & 1): GEMM-2 of slice i (M = 128): lane 16 g + e (e < 8) the raw row
                                  // s = 8 g + e, lane 16 g + 8 + e its lo row; columns 0..63 x b_hi, 64..127 x b_lo

// TTC_R64_PROF builds: clock64 time each role spends in each barrier wait, printed by CTA 0 at the end
#ifdef TTC_R64_PROF
#define PW(slot, call) do { const long long t0_ = clock64(); call; prof[slot] += clock64() - t0_; } while (0)
#else
#define PW(slot, call) call
#endif

struct TcArgs {
    int32_t B, N;
    int64_t pair_elems;       // floats per train (packed)
    const float* x;
    const float* y;
    float* out;
    const int32_t* order;
};

__device__ __forceinline__ uint64_t* bar_at(unsigned char* base, int i) {
    return reinterpret_cast<uint64_t*>(base + kOffBar) + i;
}

// ---- tcgen05 / TMA wrappers -----------------------------------------------------------------------------
// K-major SWIZZLE_128B operand descriptor (rows of 128 B, 8-row groups 1024 B apart), sm_100 version bit
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dt), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 32 consecutive TMEM columns of this warp's 32 lanes (thread t <-> lane t of the warp's sub-partition)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// lo part of a 3xTF32 split: x - trunc_tf32(x) (exact), rounded to nearest tf32 (so the tensor core's own
// truncation of it is exact and the remaining error has a random sign)
__device__ __forceinline__ float lo_rn(float x) {
    const float l = x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
    return __uint_as_float((__float_as_uint(l) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ float4 lo_rn4(float4 v) { return make_float4(lo_rn(v.x), lo_rn(v.y), lo_rn(v.z), lo_rn(v.w)); }
// split of the operands the threads write (Z, W): hi = RN_tf32(x), lo = x - hi (exact; the tensor core truncates
// it).  lo has a random sign, so the dropped lo_a lo_b term and lo's truncation are unbiased (a truncation split
// on both sides biases every product by ~2^-22 |ab| and drifted 6e-5 over C4's 14 steps on self pairs).
__device__ __forceinline__ void split_rn4(float4 v, float4& hi, float4& lo) {
    hi.x = __uint_as_float((__float_as_uint(v.x) + 0x1000u) & 0xffffe000u);
    hi.y = __uint_as_float((__float_as_uint(v.y) + 0x1000u) & 0xffffe000u);
    hi.z = __uint_as_float((__float_as_uint(v.z) + 0x1000u) & 0xffffe000u);
    hi.w = __uint_as_float((__float_as_uint(v.w) + 0x1000u) & 0xffffe000u);
    lo = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
}

// byte offset of the hi part of element (row, k) of a thread-written B operand (lo: + 8192)
__device__ __forceinline__ uint32_t bb_off(int row, int k) {
    return (uint32_t)((k >> 5) * 16384 + row * 128 + ((((k >> 2) & 7) ^ (row & 7)) << 4) + ((k & 3) << 2));
}
__device__ __forceinline__ float4 f4(const uint32_t* v) {
    return make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3]));
}
__device__ __forceinline__ float4 sel4(bool s, float4 a, float4 b) {
    return make_float4(s ? a.x : b.x, s ? a.y : b.y, s ? a.z : b.z, s ? a.w : b.w);
}
// one thread writes 32 values (row `row`, K = k0 .. k0 + 31) of a B operand as hi + lo.  Within each pair of 16-byte
// chunks, rows with bit 3 set store the odd chunk first: rows r and r + 8 (same swizzle phase) then never hit the
// same bank group in one instruction (16 consecutive rows per warp store: conflict-free).
__device__ __forceinline__ void write_b32(unsigned char* buf, int row, int k0, const float4 (&f)[8]) {
    const bool sw = (row >> 3) & 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 2 * u + (e ^ (int)sw);
            const float4 v = sel4(sw == (bool)e, f[2 * u], f[2 * u + 1]);   // chunk c's data
            float4 h, l;
            split_rn4(v, h, l);
            const uint32_t off = bb_off(row, k0 + 4 * c);
            *reinterpret_cast<float4*>(buf + off) = h;
            *reinterpret_cast<float4*>(buf + off + 8192) = l;
        }
    }
}

struct Cursor {       // the static pair sequence of this CTA
    int it, b;
    bool valid;
};
__device__ __forceinline__ void pair_at(const TcArgs& a, int it, Cursor& c) {
    const int idx = blockIdx.x + it * gridDim.x;
    c.it = it;
    c.valid = idx < a.B;
    c.b = c.valid ? (a.order ? __ldg(a.order + idx) : idx) : 0;
}

__global__ void __launch_bounds__(kThreads, 1)
inner_r64tc_kernel(const TcArgs a, const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays a shared pointer
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + kOffBar + 8 * kNumBars);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    const int steps = N - 2;                      // interior steps per pair

    if (threadIdx.x == 0) {
        for (int i = 0; i < kRaw; ++i) { mbar_init(bar_at(sm, FULL + i), 1); mbar_init(bar_at(sm, EMPTY + i), 1); }
        for (int i = 0; i < kRaw; ++i) mbar_init(bar_at(sm, LO_READY + i), kLoWarps);   // per ring slot
        for (int i = 0; i < kLo; ++i) mbar_init(bar_at(sm, LO_FREE + i), 1);            // per lo buffer
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar_at(sm, D2P_FULL + i), 1); mbar_init(bar_at(sm, D2P_EMPTY + i), 4);
            mbar_init(bar_at(sm, D1_FULL + i), 1); mbar_init(bar_at(sm, D1_EMPTY + i), 4);
            mbar_init(bar_at(sm, B2_READY + i), 2); mbar_init(bar_at(sm, B2_FREE + i), 1);
            mbar_init(bar_at(sm, BND_FULL + i), 1); mbar_init(bar_at(sm, BND_EMPTY + i), 4);
        }
        mbar_init(bar_at(sm, D2_FULL), 1);
        mbar_init(bar_at(sm, B1_READY), 4);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(tslot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
#ifdef TTC_R64_PROF
    long long prof[20] = {0};
    const long long tstart = clock64();
#endif

    if (warp == 0) {
        // ================================================================ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&tmy)) : "memory");
            uint32_t k = 0;
            Cursor c;
            for (int it = 0;; ++it) {
                pair_at(a, it, c);
                if (!c.valid) break;
                const int j = it & 1;
                PW(0, mbar_wait(bar_at(sm, BND_EMPTY + j), ((it >> 1) & 1) ^ 1));
                unsigned char* bnd = sm + kOffBnd + j * 4096;
                const float* xb = a.x + (int64_t)c.b * a.pair_elems;
                const float* yb = a.y + (int64_t)c.b * a.pair_elems;
                mbar_arrive_expect_tx(bar_at(sm, BND_FULL + j), 4096);
                bulk_g2s(bnd, xb, 1024, bar_at(sm, BND_FULL + j));
                bulk_g2s(bnd + 1024, yb, 1024, bar_at(sm, BND_FULL + j));
                bulk_g2s(bnd + 2048, xb + a.pair_elems - 256, 1024, bar_at(sm, BND_FULL + j));
                bulk_g2s(bnd + 3072, yb + a.pair_elems - 256, 1024, bar_at(sm, BND_FULL + j));
                // row (of 256 floats) of core n = 1..N-2 of this pair: (b pair_elems + 256 + (n - 1) 16384) / 256
                const int64_t row0 = ((int64_t)c.b * a.pair_elems + 256) / 256;
                for (int n = 0; n < steps; ++n) {
                    const int row = (int)(row0 + 64 * n);
                    for (int t = 0; t < kEntriesPerStep; ++t, ++k) {
                        const int s = k % kRaw;
                        PW(1, mbar_wait(bar_at(sm, EMPTY + s), ((k / kRaw) & 1) ^ 1));
                        unsigned char* dst = sm + kOffRaw + s * kTile;
                        uint64_t* fb = bar_at(sm, FULL + s);
                        if (t < kYPerStep) {   // Y half t/2, K-chunk t%2: box (32 p, 2 i, 64 q)
                            mbar_arrive_expect_tx(fb, kTile);
                            tc::tma_3d(dst, &tmy, 32 * (t & 1), row, 2 * (t >> 1), fb);
                        } else {               // X slice e/2, K-chunk e%2: one box (32 r, 64 s) into the slot's first
                            const int e = t - kYPerStep;   // 8 KB (the lo workers spread the 8-row groups)
                            mbar_arrive_expect_tx(fb, kTile / 2);
                            tc::tma_2d(dst, &tmx, 64 * (e >> 1) + 32 * (e & 1), row, fb);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================================================================ MMA issuer
        if (lane == 0) {
            const uint32_t id1w = idesc_tf32(128, 128), id1 = idesc_tf32(128, 64);
            const uint32_t sbase = smem_u32(sm);
            const uint32_t b1 = sbase + kOffB1;
            uint32_t k = 0, v = 0, ky = 0;   // entry counter, interior-step counter, Y-entry counter
            Cursor c;
            for (int it = 0;; ++it) {
                pair_at(a, it, c);
                if (!c.valid) break;
                for (int n = 0; n < steps; ++n, ++v) {
                    PW(2, mbar_wait(bar_at(sm, B1_READY), v & 1));
                    // ---- GEMM-1, halves h = 0, 1 (M = 128: rows i' + 2q)
                    for (int h = 0; h < 2; ++h) {
                        PW(3, mbar_wait(bar_at(sm, D1_EMPTY + h), (v & 1) ^ 1));
                        const uint32_t d = tmem + kD1 + 128 * h;
                        for (int kc = 0; kc < 2; ++kc, ++k) {
                            PW(4, mbar_wait(bar_at(sm, FULL + k % kRaw), (k / kRaw) & 1));
                            PW(5, mbar_wait(bar_at(sm, LO_READY + k % kRaw), (k / kRaw) & 1));
                            tc_fence_after();
                            const uint32_t ar = sbase + kOffRaw + (k % kRaw) * kTile;
                            const uint32_t al = sbase + kOffLo + (ky % kLo) * kTile;
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint64_t A = desc_sw128(ar + 32 * kk), Al = desc_sw128(al + 32 * kk);
                                const uint64_t B = desc_sw128(b1 + 16384 * kc + 32 * kk);   // [Z_hi | Z_lo]
                                mma_tf32(d, A, B, id1w, (kc | kk) ? 1u : 0u);             // a_hi [b_hi | b_lo]
                                mma_tf32(d + 64, Al, B, id1, 1u);                         // + a_lo b_hi
                            }
                            // free this entry's slot and lo buffer as soon as its own MMAs are done
                            mma_commit(bar_at(sm, EMPTY + k % kRaw));
                            mma_commit(bar_at(sm, LO_FREE + ky % kLo));
                            ++ky;
                        }
                        mma_commit(bar_at(sm, D1_FULL + h));
                    }
                    // ---- GEMM-2, slices i = 0..3: one M = 128 MMA per K-block, A = [X_i^T raw; X_i^T lo] (8-row groups
                    //      interleaved), B = [W_hi | W_lo]: 8 MMAs a slice (16 with an M = 64 raw and a separate lo MMA;
                    //      the MMA issue is the kernel's pace), each slice's chain 8 MMAs long as in GEMM-1
                    for (int i = 0; i < 4; ++i) {
                        const int j = i & 1;
                        PW(8, mbar_wait(bar_at(sm, B2_READY + j), (2 * v + (i >> 1)) & 1));
                        PW(9, mbar_wait(bar_at(sm, D2P_EMPTY + j), ((2 * v + (i >> 1)) & 1) ^ 1));
                        const uint32_t br = sbase + kOffB2 + j * 2 * kTile;
                        const uint32_t d = tmem + kD2 + 128 * j;
                        for (int kc = 0; kc < 2; ++kc, ++k) {
                            PW(6, mbar_wait(bar_at(sm, FULL + k % kRaw), (k / kRaw) & 1));
                            PW(7, mbar_wait(bar_at(sm, LO_READY + k % kRaw), (k / kRaw) & 1));
                            tc_fence_after();
                            const uint32_t ar = sbase + kOffRaw + (k % kRaw) * kTile;
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint64_t A = desc_sw128(ar + 32 * kk);
                                const uint64_t B = desc_sw128(br + 16384 * kc + 32 * kk);   // [W_hi | W_lo]
                                mma_tf32(d, A, B, id1w, (kc | kk) ? 1u : 0u);
                            }
                            mma_commit(bar_at(sm, EMPTY + k % kRaw));
                        }
                        mma_commit(bar_at(sm, B2_FREE + j));
                        mma_commit(bar_at(sm, D2P_FULL + j));
                    }
                }
            }
        }
    } else if (warp >= 6) {
        // ================================================================ lo workers (warps 6, 7)
        // the lo part of every staged input tile, in the order the MMA issuer consumes them (elementwise: the lo
        // tile has the raw tile's byte layout); all loads of a thread's share are issued before any store
        constexpr int kLoT = 32 * kLoWarps;       // lo threads
        const int ct = threadIdx.x - 192;         // 0 .. kLoT - 1
        uint32_t ktot = 0;
        for (int idx = blockIdx.x; idx < a.B; idx += gridDim.x) ktot += (uint32_t)steps * kEntriesPerStep;
        uint32_t ky = 0;
        for (uint32_t k = 0; k < ktot; ++k) {
            const int s = k % kRaw;
            PW(10, mbar_wait(bar_at(sm, FULL + s), (k / kRaw) & 1));
            const float4* src = reinterpret_cast<const float4*>(sm + kOffRaw + s * kTile);
            if ((k % kEntriesPerStep) < kYPerStep) {   // Y entry: its 16 KB lo part into the lo ring (same layout)
                const int l = ky % kLo;
                PW(11, mbar_wait(bar_at(sm, LO_FREE + l), ((ky / kLo) & 1) ^ 1));
                ++ky;
                float4* dst = reinterpret_cast<float4*>(sm + kOffLo + l * kTile);
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    float4 r[kTile / 16 / (2 * kLoT)];
#pragma unroll
                    for (int e = 0; e < kTile / 16 / (2 * kLoT); ++e) r[e] = src[ct + kLoT * (2 * e + hf)];
#pragma unroll
                    for (int e = 0; e < kTile / 16 / (2 * kLoT); ++e) dst[ct + kLoT * (2 * e + hf)] = lo_rn4(r[e]);
                }
            } else {   // X entry: the 8 KB raw box (64 rows) read whole, then raw 8-row group g rewritten at 2 KB g and
                       // its lo part at 2 KB g + 1 KB (1 KB swizzle atoms: the swizzle phase is kept)
                float4 r[kTile / 32 / kLoT];
#pragma unroll
                for (int e = 0; e < kTile / 32 / kLoT; ++e) r[e] = src[ct + kLoT * e];
                __syncwarp();
                bar_named(2, kLoT);   // every lo thread has read the box before any group moves
                float4* dst = reinterpret_cast<float4*>(sm + kOffRaw + s * kTile);
#pragma unroll
                for (int e = 0; e < kTile / 32 / kLoT; ++e) {
                    const int q = ct + kLoT * e;                     // float4 index within the 8 KB of raw data
                    const int o = ((q >> 6) << 7) + (q & 63);
                    dst[o] = r[e];
                    dst[o + 64] = lo_rn4(r[e]);
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_at(sm, LO_READY + s));
        }
    } else {
        // ================================================================ epilogue warps (warps 2..5)
        const int ct = threadIdx.x - 64;          // 0..127
        const int sp = warp & 3;                  // TMEM sub-partition of this warp (lanes 32 sp .. 32 sp + 31)
        const uint32_t tl = tmem + ((uint32_t)(32 * sp) << 16);
        unsigned char* b1 = sm + kOffB1;
        float* red = reinterpret_cast<float*>(sm + kOffRed);
        uint32_t v = 0;
        Cursor c;
        for (int it = 0;; ++it) {
            pair_at(a, it, c);
            if (!c.valid) break;
            const int jb = it & 1;
            const float* bnd = reinterpret_cast<const float*>(sm + kOffBnd + jb * 4096);
            PW(12, mbar_wait(bar_at(sm, BND_FULL + jb), (it >> 1) & 1));
            // ---- first step: Z_1[s][q] = sum_i X_1[0, i, s] Y_1[0, i, q]  (Eq. 12's K), into B1 (raw, lo)
            {
                const int s = ct & 63, q0 = 32 * (ct >> 6);
                const float4 xs = reinterpret_cast<const float4*>(bnd)[s];
                uint32_t zv[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const float4 yq = reinterpret_cast<const float4*>(bnd + 256)[q0 + q];
                    float z = xs.x * yq.x;
                    z = fmaf(xs.y, yq.y, z);
                    z = fmaf(xs.z, yq.z, z);
                    z = fmaf(xs.w, yq.w, z);
                    zv[q] = __float_as_uint(z);
                }
                float4 f[8];
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4) f[c4] = f4(zv + 4 * c4);
                write_b32(b1, s, q0, f);
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_at(sm, B1_READY));
            }
            for (int n = 0; n < steps; ++n, ++v) {
                // ---- epilogue 1: D1[h] row m = q + 64 i' of this lane (m = 32 sp + lane) -> W_{2h+i'} into B2[i']:
                // warps sp = 0, 1 own slice 2h, warps 2, 3 slice 2h + 1 (32 consecutive rows q per warp store)
                const int q = 32 * (sp & 1) + lane, ip = sp >> 1;
                auto write_w = [&](int h) {       // a_hi b_hi partial + cross terms, 32 columns at a time, split
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        uint32_t t0[32], t1[32];
                        tmem_ld32(tl + kD1 + 128 * h + 32 * hh, t0);
                        tmem_ld32(tl + kD1 + 128 * h + 64 + 32 * hh, t1);
                        tmem_wait_ld();
                        float4 f[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            f[c].x = __uint_as_float(t0[4 * c]) + __uint_as_float(t1[4 * c]);
                            f[c].y = __uint_as_float(t0[4 * c + 1]) + __uint_as_float(t1[4 * c + 1]);
                            f[c].z = __uint_as_float(t0[4 * c + 2]) + __uint_as_float(t1[4 * c + 2]);
                            f[c].w = __uint_as_float(t0[4 * c + 3]) + __uint_as_float(t1[4 * c + 3]);
                        }
                        write_b32(sm + kOffB2 + ip * 2 * kTile, q, 32 * hh, f);
                    }
                };
                // GEMM-2 slice sums of TMEM lane 32 sp + lane: the raw row s (lane bit 3 clear) or the lo row of s (set),
                // s = 16 sp + 8 (lane >> 4) + lane % 8
                float zacc[64];
                auto add_slice = [&](int i) {
                    const int j = i & 1;
                    PW(13, mbar_wait(bar_at(sm, D2P_FULL + j), (2 * v + (i >> 1)) & 1));
                    tc_fence_after();
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        uint32_t p0[32], p1[32];
                        tmem_ld32(tl + kD2 + 128 * j + 32 * hh, p0);
                        tmem_ld32(tl + kD2 + 128 * j + 64 + 32 * hh, p1);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const float t = __uint_as_float(p0[e]) + __uint_as_float(p1[e]);
                            zacc[32 * hh + e] = i ? zacc[32 * hh + e] + t : t;
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_at(sm, D2P_EMPTY + j));
                };
                PW(14, mbar_wait(bar_at(sm, D1_FULL + 0), v & 1));
                PW(15, mbar_wait(bar_at(sm, B2_FREE + ip), ((2 * v) & 1) ^ 1));
                tc_fence_after();
                write_w(0);
                tc_fence_before();
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(bar_at(sm, D1_EMPTY + 0));
                    mbar_arrive(bar_at(sm, B2_READY + ip));
                }
                // ---- epilogue 1b: D1[1] -> W_2 into B2[0] (after GEMM-2 slice 0), W_3 into B2[1] (after slice 1)
                PW(16, mbar_wait(bar_at(sm, D1_FULL + 1), v & 1));
                for (int j = 0; j < 2; ++j) {
                    PW(17, mbar_wait(bar_at(sm, B2_FREE + j), ((2 * v + 1) & 1) ^ 1));
                    add_slice(j);                                 // slice j is done (B2[j] is free)
                    if (ip == j) {
                        tc_fence_after();
                        write_w(1);
                        tc_fence_before();
                        fence_proxy_async();
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(bar_at(sm, B2_READY + j));
                            mbar_arrive(bar_at(sm, D1_EMPTY + 1));
                        }
                    }
                }
                add_slice(2);
                add_slice(3);
                // ---- epilogue 2: Z_n row s = raw-row sums + lo-row sums (lanes 8 apart)
                uint32_t z0[32], z1[32];     // (slice 3 read above: every MMA of the step is complete)
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    z0[e] = __float_as_uint(zacc[e] + __shfl_xor_sync(0xffffffffu, zacc[e], 8));
                    z1[e] = __float_as_uint(zacc[32 + e] + __shfl_xor_sync(0xffffffffu, zacc[32 + e], 8));
                }
                // both lanes of a pair now hold row s: the raw lane writes its columns 0..31, the lo lane 32..63
                const int s = 16 * sp + 8 * (lane >> 4) + (lane & 7);
                const bool upper = (lane & 8) != 0;
                if (n + 1 < steps) {
                    float4 f[8];
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) f[c4] = sel4(upper, f4(z1 + 4 * c4), f4(z0 + 4 * c4));
                    write_b32(b1, s, upper ? 32 : 0, f);
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_at(sm, B1_READY));
                } else {
                    // ---- last step: out = sum_{s,q} Z[s][q] sum_i X_N[s, i, 0] Y_N[q, i, 0] (each lane of a pair
                    //      takes half of row s's columns)
                    float acc = 0.f;
                    {
                        const float* xN = bnd + 512;
                        const float* yN = bnd + 768 + (upper ? 32 : 0);
                        const float x0 = xN[s], x1 = xN[s + 64], x2 = xN[s + 128], x3 = xN[s + 192];
#pragma unroll
                        for (int qq = 0; qq < 32; ++qq) {
                            float t = x0 * yN[qq];
                            t = fmaf(x1, yN[qq + 64], t);
                            t = fmaf(x2, yN[qq + 128], t);
                            t = fmaf(x3, yN[qq + 192], t);
                            acc = fmaf(__uint_as_float(upper ? z1[qq] : z0[qq]), t, acc);
                        }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    if (lane == 0) red[sp] = acc;
                    bar_named(1, 128);
                    if (ct == 0) a.out[c.b] = (red[0] + red[1]) + (red[2] + red[3]);
                    bar_named(1, 128);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_at(sm, BND_EMPTY + jb));
                }
            }
        }
    }
#ifdef TTC_R64_PROF
    if (blockIdx.x == 0 && lane == 0 && (warp <= 2 || warp == 6)) {
        prof[19] = clock64() - tstart;
        printf("r64tc prof warp %d total %lld | %lld %lld | %lld %lld %lld %lld %lld %lld %lld %lld | %lld %lld | "
               "%lld %lld %lld %lld %lld %lld %lld\n", warp, prof[19], prof[0], prof[1], prof[2], prof[3], prof[4],
               prof[5], prof[6], prof[7], prof[8], prof[9], prof[10], prof[11], prof[12], prof[13], prof[14],
               prof[15], prof[16], prof[17], prof[18]);
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(kTmemCols));
}

}  // namespace

// ---- host: tensor maps through the driver entry point (no link-time dependency on libcuda)
EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

bool inner_r64tc_supported(const InnerArgs& a, bool uniform_r64) {
    if (!uniform_r64 || a.N < 3 || a.x.offsets || a.y.offsets) return false;
    for (int n = 0; n < a.N; ++n)
        if (a.dims[n] != 4) return false;
    if ((reinterpret_cast<uintptr_t>(a.x.cores) | reinterpret_cast<uintptr_t>(a.y.cores)) & 15u) return false;
    const int64_t rows = (int64_t)a.B * a.x.train_elems / 256;
    return rows < (int64_t(1) << 31);
}

cudaError_t launch_inner_r64tc(const InnerArgs& a, cudaStream_t s) {
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    const int64_t pe = a.x.train_elems;            // 256 + (N - 2) 16384 + 256 floats per train
    const cuuint64_t rows = (cuuint64_t)((int64_t)a.B * pe / 256);
    CUtensorMap tmx, tmy;
    {   // X: rows of 256 floats (r + 64 i for one s), box 32 x 64 rows (one K-chunk of one slice)
        const cuuint64_t dims[2] = {256, rows};
        const cuuint64_t strides[1] = {1024};
        const cuuint32_t box[2] = {32, 64};
        const cuuint32_t es[2] = {1, 1};
        if (enc(&tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.x.cores), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {   // Y: (p: 64, q-row: rows @ 1024 B, i: 4 @ 256 B), box (32 p, 64 q, 2 i) -> SMEM rows q + 64 i'
        const cuuint64_t dims[3] = {64, rows, 4};
        const cuuint64_t strides[2] = {1024, 256};
        const cuuint32_t box[3] = {32, 64, 2};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(&tmy, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(a.y.cores), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    TcArgs t;
    t.B = a.B;
    t.N = a.N;
    t.pair_elems = pe;
    t.x = a.x.cores;
    t.y = a.y.cores;
    t.out = a.out;
    t.order = a.order;
    cudaError_t e = cudaFuncSetAttribute(inner_r64tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    const int grid = a.B < sms ? a.B : sms;
    inner_r64tc_kernel<<<grid, kThreads, kSmemBytes, s>>>(t, tmx, tmy);
    return cudaGetLastError();
}

}  // namespace ttc
