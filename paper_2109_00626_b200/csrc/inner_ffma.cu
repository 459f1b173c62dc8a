// inner_ffma.cu -- tt_inner, one warp per pair on the FP32 pipe, for interior bond ranks that are multiples of 8
// and <= 32 (BASELINE.json C5: N = 64, I = 2, ranks drawn from {8, 16, 24, 32} per bond).  Same sweep as ttc.h:
//   Z_0 = [1],  Z_n = sum_i X_n[:, i, :]^T Z_{n-1} Y_n[:, i, :]   (Fig. 1b / Eq. 12 chained),  out = Z_N.
//
// Why FP32 and not the tensor cores here: C5's steps are tiny (8..32-wide) and rectangular, so 16-row mma
// tiles pad 20% of the work away and 3xTF32 triples the rest; measured legacy mma.sync tf32 (279 TF) then
// caps the sweep near 10 M pairs/s, while FFMA at 72 TF caps it near 23 M pairs/s.
//
// Per step, with the cheaper association (F = the core multiplied into Z first, G = the other one):
//   GEMM-1 (per slice i):  W_i[g, f'] = sum_f Z[g, f] F[f, i, f']          (Ga x Fb, K = Fa)
//   GEMM-2 (per slice i):  Z'[g', f'] += sum_g G[g, i, g'] W_i[g, f']      (Gb x Fb, K = Ga)
// W-first: F = Y, G = X (Z indexed [x bond][y bond]); V-first: F = X, G = Y (Z stored transposed).
// Every operand is read along its contraction index, which is the contiguous one in the paper's core
// layout (Eq. 2), so each lane loads 4 K-values with one 16-byte LDS and does 4 FFMA per output it owns.
// Lane (lg = lane / 4, lf = lane % 4) owns rows lg + 8a and columns lf + 4b of each output tile.
//
// Staging: the warp copies its own future steps into a private ring, with 4 floats of padding after every
// contiguous run (F: runs of Fa, G: runs of Ga*I) so that the 8 (or 4) distinct runs one LDS.128 touches fall into
// distinct bank groups -- interior operands by TMA tensor boxes (FfMaps below: the padding is the out-of-range
// tail of each box row, zero-filled), boundary cores and batches whose run lengths overflow the map table by
// 16-byte cp.async; Z and W are kept with padded row strides likewise.
// Pairs are assigned statically: warp w of W takes positions w, 2W-1-w, 2W+w, 4W-1-w, ... of the work list
// (a "snake" over the cost-descending list of ttc_inner_ordered balances heterogeneous pairs); no global state,
// so concurrent launches and graph replays on several streams are independent (re-entrant, ttc.h).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tc_common.cuh"
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kPad = 4;
#ifndef TTC_FFMA_Q
#define TTC_FFMA_Q 4
#endif
constexpr int kQ = TTC_FFMA_Q;          // staged steps in flight per warp (queue entries)

constexpr int kMagicMax = 1024;          // exact-division table: q in [2, kMagicMax]

// c_magic[q] = ceil(2^32 / q): e / q == __umulhi(e, c_magic[q]) for every e < 2^32 / q (q >= 2).
struct MagicTable {
    unsigned v[kMagicMax + 1];
    constexpr MagicTable() : v() {
        for (int q = 2; q <= kMagicMax; ++q) v[q] = (unsigned)((0x100000000ull + q - 1) / q);
    }
};
__constant__ MagicTable c_magic = MagicTable();

struct FfArgs {
    int ring;         // floats of one warp's ring
    int zbuf, wbuf;   // floats of the Z and W buffers
    int warp_floats;  // ring + Z + W + queue
};

// TMA staging (kTma): one 3-D tensor map per operand buffer and run length L (the contiguous runs an operand is
// staged in: F runs of Fa floats, G runs of Ga I floats).  Map (L, 8, n / 4) with strides (4 L, 16) bytes and a
// box of (L + 4, 8, 1): the box starting at coordinate (0, 0, o / 4) is the 8 runs of L floats from float o on,
// written to shared memory as rows of L + 4 floats -- the padded layout -- with the 4 floats past each run
// outside the map's first dimension (zero-filled, never read from global memory).  Any 16-byte aligned start is
// reachable through the third coordinate (runs of 8 rows: every interior F and G operand has a multiple of 8).
constexpr int kMaxMaps = 16;
constexpr int kMaxRunQ = 63;      // L / 4 <= 63 (the box's first dimension L + 4 <= 256)
struct FfMaps {
    CUtensorMap m[kMaxMaps];
    unsigned char ix[2][kMaxRunQ + 1];   // [X / Y][L / 4] -> map index
};

struct FStep {
    int start;        // ring offset (floats) of the F region (boundary steps: X), G (Y) follows
    int b, n, R, P, S, Q, I;
    int vf;           // interior: V-first (F = X); boundary: unused
    int part;         // interior: 0 the whole step, 1 its F operand only (GEMM-1), 2 its G operand only (GEMM-2)
    int znext;        // orientation the next step wants Z in (1: transposed, V-first next)
    unsigned end;     // monotone ring position after this step
};

__device__ __forceinline__ int frank(const TrainDev& t, int b, int N, int n) {
    if (n <= 0 || n >= N) return 1;
    return t.ranks ? __ldg(t.ranks + (int64_t)b * (N + 1) + n) : t.urank;
}
__device__ __forceinline__ int64_t fbase(const TrainDev& t, int b) {
    return t.offsets ? __ldg(t.offsets + b) : (int64_t)b * t.train_elems;
}
// V-first (X multiplied into Z first) iff it is strictly cheaper: I S P (R + Q) < I R Q (P + S)
__device__ __forceinline__ int vfirst(int R, int P, int S, int Q) { return S * P * (R + Q) < R * Q * (P + S); }

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// Packed FP32 pair (FFMA2 on sm_100a: two FMAs per issue slot at the same FP32 throughput, measured
// tools/fma_bench.cu).  acc.{x,y} accumulate the even / odd k terms of a dot product.
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void fma2(unsigned long long& acc, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ float hsum2(unsigned long long v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo + hi;
}
// acc += a.xy * b.xy, a.zw * b.zw (pairwise): the 4-term dot product in two FFMA2
__device__ __forceinline__ void dot4x2(unsigned long long& acc, const float4 a, const float4 b) {
    fma2(acc, pk(a.x, a.y), pk(b.x, b.y));
    fma2(acc, pk(a.z, a.w), pk(b.z, b.w));
}

// Copy `runs` runs of `run` floats (run % 4 == 0) from contiguous global memory into shared memory with a run
// stride of run + kPad (run / 4 in [2, kMagicMax]): e / (run / 4) is one IMAD.HI with the magic table.
__device__ __forceinline__ void stage_padded(float* dst, const float* src, int runs, int run, int lane) {
    const unsigned q = (unsigned)run >> 2;
    const unsigned div = c_magic.v[q];
    const unsigned chunks = (unsigned)runs * q;
#pragma unroll 1
    for (unsigned e = lane; e < chunks; e += 32) {
        const unsigned c = __umulhi(e, div);
        const unsigned o = e - c * q;
        tc::cp_async16(dst + c * (run + kPad) + 4 * o, src + 4 * e);
    }
}
__device__ __forceinline__ void stage_plain(float* dst, const float* src, int n, int lane) {
    if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
#pragma unroll 1
        for (int e = 4 * lane; e < n; e += 128) tc::cp_async16(dst + e, src + e);
    } else {   // odd boundary sizes (N = 1, I odd): plain copies, visible after the consumer's __syncwarp
#pragma unroll 1
        for (int e = lane; e < n; e += 32) dst[e] = __ldg(src + e);
    }
}

// Register-tiled block product and store: for rows lg + 8a (a < TA) and columns c0 + lf + 4b (b < NB),
//   out[row * rs + col * cs + (col / I) * ci] = sum_k A[row][k] B[col][k]
// A rows and B columns are contiguous along k (strides sA / sB, 16-byte aligned).  The (col / I) term inserts
// the W buffer's column padding (ci = 0: none).  The next k-chunk's operands are loaded before the current
// chunk's FFMAs issue (software pipelining: LDS latency hides behind 4 TA NB FFMAs).  Only the 8
// instantiations below exist, inside one non-inlined ff_gemm, for every shape and both GEMMs: the hot code
// stays inside the SM's instruction caches (~6 KB L0, 32 KB L1.5) although every warp runs another shape.
template <int TA, int NB>
__device__ __forceinline__ void block_fma(const float* __restrict__ A, int sA, const float* __restrict__ B, int sB, int K,
                                          float* __restrict__ out, int rs, int cs, int ci, unsigned idiv, int c0,
                                          int lg, int lf) {
    unsigned long long acc[TA][NB];
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[a][b] = 0ull;
    const float* Ap[TA];
    const float* Bp[NB];
#pragma unroll
    for (int a = 0; a < TA; ++a) Ap[a] = A + 8 * a * sA;
#pragma unroll
    for (int b = 0; b < NB; ++b) Bp[b] = B + (c0 + lf + 4 * b) * sB;
    // two k-chunks per iteration (K % 8 == 0): loads at immediate offsets +0 / +4 of pointers advanced once per
    // iteration; the next iteration's first chunk is loaded while the second chunk computes (the final prefetch
    // reads the 4 padding floats after every row / column: in bounds, discarded)
    const float* ap[TA];
    const float* bq[NB];
#pragma unroll
    for (int a = 0; a < TA; ++a) ap[a] = Ap[a];
#pragma unroll
    for (int b = 0; b < NB; ++b) bq[b] = Bp[b];
    float4 za[TA], fb[NB];
#pragma unroll
    for (int a = 0; a < TA; ++a) za[a] = ld4(ap[a]);
#pragma unroll
    for (int b = 0; b < NB; ++b) fb[b] = ld4(bq[b]);
#pragma unroll 1
    for (int k = 0; k < K; k += 8) {
        float4 zb[TA], gb[NB];
#pragma unroll
        for (int a = 0; a < TA; ++a) zb[a] = ld4(ap[a] + 4);
#pragma unroll
        for (int b = 0; b < NB; ++b) gb[b] = ld4(bq[b] + 4);
#pragma unroll
        for (int a = 0; a < TA; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b) dot4x2(acc[a][b], za[a], fb[b]);
#pragma unroll
        for (int a = 0; a < TA; ++a) { ap[a] += 8; za[a] = ld4(ap[a]); }
#pragma unroll
        for (int b = 0; b < NB; ++b) { bq[b] += 8; fb[b] = ld4(bq[b]); }
#pragma unroll
        for (int a = 0; a < TA; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b) dot4x2(acc[a][b], zb[a], gb[b]);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const unsigned col = c0 + lf + 4 * b;
        const int cbase = col * cs + (ci ? (int)__umulhi(col, idiv) * ci : 0);
#pragma unroll
        for (int a = 0; a < TA; ++a) out[(lg + 8 * a) * rs + cbase] = hsum2(acc[a][b]);
    }
}

// All column blocks of one row count: 4 lane-columns per block, a 2-column tail.
template <int TA>
__device__ __forceinline__ void gemm_rows(const float* A, int sA, const float* B, int sB, int K, int ncols, float* out,
                                          int rs, int cs, int ci, unsigned idiv, int lg, int lf) {
    int cb = 0;
    for (; cb + 4 <= ncols; cb += 4) block_fma<TA, 4>(A, sA, B, sB, K, out, rs, cs, ci, idiv, 4 * cb, lg, lf);
    if (cb < ncols) block_fma<TA, 2>(A, sA, B, sB, K, out, rs, cs, ci, idiv, 4 * cb, lg, lf);
}

// out = A B^T over rows < 8 TA and columns < 4 ncols (ncols even); one dispatch on the row count per GEMM.
__device__ __noinline__ void ff_gemm(const float* A, int sA, const float* B, int sB, int K, int TA, int ncols,
                                     float* out, int rs, int cs, int ci, unsigned idiv, int lane) {
    // lane -> (row group lg, column group lf): lg from lane bits 1-3, lf from bits 0 and 4.  An LDS.128 costs one
    // shared-memory wavefront per half-warp only when each half-warp's addresses come in runs of adjacent lanes
    // or alternate lane by lane (tools/lds_bench.cu: lane >> 2 -> 2 wavefronts, lane & 3 -> 4); this mapping
    // gives 2 for both the A (row) and the B (column) loads (lg = lane >> 2, lf = lane & 3: 2 and 4).
    const int lg = (lane >> 1) & 7, lf = (lane & 1) | ((lane >> 4) << 1);
    A += lg * sA;
    if (TA >= 3) {
        if (TA == 4) gemm_rows<4>(A, sA, B, sB, K, ncols, out, rs, cs, ci, idiv, lg, lf);
        else gemm_rows<3>(A, sA, B, sB, K, ncols, out, rs, cs, ci, idiv, lg, lf);
    } else {
        if (TA == 2) gemm_rows<2>(A, sA, B, sB, K, ncols, out, rs, cs, ci, idiv, lg, lf);
        else gemm_rows<1>(A, sA, B, sB, K, ncols, out, rs, cs, ci, idiv, lg, lf);
    }
}

// One interior step.  Z: [g][f] with row stride Fa + kPad.  GEMM-1 writes W[g + Ga c + kPad (c / I)] for F
// column c = i + I f' (so that GEMM-2 reads W column f' as one contiguous run over (g, i)); GEMM-2 writes Z'
// in the orientation the next step reads: same (flip = 0): [g'][f'] stride Fb + kPad; flip: [f'][g'] stride
// Gb + kPad.
__device__ __forceinline__ void ff_step1(const float* F, int Fa, int Fb, int Ga, int I, const float* Z, float* W,
                                         int lane) {
    const unsigned idiv = I == 1 ? 0u : c_magic.v[I];
    const int sF = Fa + kPad;
    // GEMM-1: W[g, c] = sum_f Z[g, f] F[f, c]     (Ga x I Fb, K = Fa)
    ff_gemm(Z, sF, F, sF, Fa, Ga >> 3, (I * Fb) >> 2, W, 1, I == 1 ? Ga + kPad : Ga, I == 1 ? 0 : kPad, idiv, lane);
    __syncwarp();
}
__device__ __forceinline__ void ff_step2(int Fb, const float* G, int Ga, int Gb, int I, float* Z, const float* W,
                                         int flip, int lane) {
    const int sG = Ga * I + kPad, sW = Ga * I + kPad;
    // GEMM-2: Z'[g', f'] = sum_(g,i) G[(g,i), g'] W[(g,i), f']   (Gb x Fb, K = Ga I)
    ff_gemm(G, sG, W, sW, Ga * I, Gb >> 3, Fb >> 2, Z, flip ? 1 : Fb + kPad, flip ? Gb + kPad : 1, 0, 0u, lane);
    __syncwarp();
}

// First step (R = P = 1): Z_1[s, q] = sum_i X_1[0, i, s] Y_1[0, i, q] -- Eq. 12's K -- stored for the next step:
// znext = 0: Z[s][q] stride Q + kPad, znext = 1: Z[q][s] stride S + kPad.
// (The two boundary steps run once per pair: kept out of line, so that the steady-state step loop stays compact in
// the instruction caches -- measured +4.5% on C5.)
__device__ __noinline__ void ff_first(const float* X, const float* Y, int S, int Q, int I, int znext, float* Z,
                                         int lane) {
#pragma unroll 1
    for (int q = 0; q < Q; ++q)
        for (int s = lane; s < S; s += 32) {
            float d = 0.f;
            for (int i = 0; i < I; ++i) d = fmaf(X[i + I * s], Y[i + I * q], d);
            Z[znext ? q * (S + kPad) + s : s * (Q + kPad) + q] = d;
        }
    __syncwarp();
}
// Last step (S = Q = 1): Z_N = sum_{r,p} Z[r,p] sum_i X_N[r,i,0] Y_N[p,i,0], Z[r][p] stride P + kPad (first:
// N = 1, Z_0 = 1).  Warp-reduced in a fixed order.
__device__ __noinline__ float ff_last(const float* X, const float* Y, int R, int P, int I, bool first, const float* Z,
                                         int lane) {
    float v = 0.f;
    for (int p = 0; p < P; ++p)
        for (int r = lane; r < R; r += 32) {
            float d = 0.f;
            for (int i = 0; i < I; ++i) d = fmaf(X[r + R * i], Y[p + P * i], d);
            v = fmaf(first ? 1.0f : Z[r * (P + kPad) + p], d, v);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct FCursor {
    int b, n, R, P;
    int64_t xo, yo;
    bool valid;
    bool half;        // the current step is split and its F part is staged: G next
    unsigned k;       // pairs taken so far by this warp
};

// This warp's next pair (static snake assignment over the work list); its rank rows go to rk (X: rk[0..N],
// Y: rk[N+1..2N+1]).
__device__ __forceinline__ void fc_pop(const InnerArgs& a, const FfArgs&, FCursor& c, int* rk, int lane) {
    const unsigned W = gridDim.x, w = blockIdx.x;
    const unsigned t = c.k * W + ((c.k & 1u) ? W - 1u - w : w);
    ++c.k;
    c.valid = t < (unsigned)a.B;
    if (!c.valid) return;
    c.b = a.order ? __ldg(a.order + t) : (int)t;
    const int N = a.N;
    __syncwarp();   // every lane is done reading the previous pair's ranks
    for (int n = lane; n <= N; n += 32) {
        rk[n] = frank(a.x, c.b, N, n);
        rk[N + 1 + n] = frank(a.y, c.b, N, n);
    }
    __syncwarp();
    // the association of every interior step at once (bit n of vfm: step n is V-first), one ballot per 32 steps
    unsigned* vfm = reinterpret_cast<unsigned*>(rk + 2 * (N + 1));
    for (int n0 = 0; n0 < N; n0 += 32) {
        const int n = n0 + lane;
        const bool v = n >= 1 && n + 1 < N && vfirst(rk[n], rk[N + 1 + n], rk[n + 1], rk[N + 2 + n]);
        const unsigned m = __ballot_sync(0xffffffffu, v);
        if (lane == 0) vfm[n0 >> 5] = m;
    }
    __syncwarp();
    c.n = 0;
    c.half = false;
    c.R = 1;
    c.P = 1;
    c.xo = fbase(a.x, c.b);
    c.yo = fbase(a.y, c.b);
}

// One warp per CTA (warps never synchronise with each other); several CTAs per SM, as shared memory allows.
template <bool kTma>
__global__ void __launch_bounds__(32)
inner_ffma_kernel(const InnerArgs a, const FfArgs w, const __grid_constant__ FfMaps maps) {
    extern __shared__ __align__(128) float smem[];
    const int lane = threadIdx.x & 31;
    float* ring = smem;
    float* Z = ring + w.ring;
    float* W = Z + w.zbuf;
    FStep* q = reinterpret_cast<FStep*>(W + w.wbuf);
    uint64_t* bars = reinterpret_cast<uint64_t*>(q + kQ);   // kTma: one mbarrier per queue entry
    int* rk = reinterpret_cast<int*>(bars + kQ);
    const int N = a.N;
    const unsigned* vfm = reinterpret_cast<const unsigned*>(rk + 2 * (N + 1));   // fc_pop's association bits
    unsigned phase = 0;                                      // kTma: parity bit per queue entry
    if (kTma) {
        if (lane == 0) {
            for (int i = 0; i < kQ; ++i) tc::mbar_init(bars + i, 1);
            tc::fence_mbar_init();
        }
        __syncwarp();
    }
    FCursor ic;
    ic.k = 0;
    fc_pop(a, w, ic, rk, lane);
    unsigned head = 0, tail = 0, head_off = 0;
    int qh = 0, qn = 0;
    const unsigned RING = (unsigned)w.ring;
    while (true) {
        // ---- stage future steps while they fit
        while (ic.valid && qn < kQ) {
            const int n = ic.n, I = a.dims[n];
            const int R = ic.R, P = ic.P;
            const int S = rk[n + 1], Q = rk[N + 2 + n];
            const bool boundary = n == 0 || n == N - 1;
            int vf = 0, need, part = 0;
            if (boundary) {
                need = ((R * I * S + 3) & ~3) + ((P * I * Q + 3) & ~3);
                if (kTma) need = (need + 31) & ~31;   // every step starts on 128 bytes (TMA destinations)
            } else {
                vf = (vfm[n >> 5] >> (n & 31)) & 1u;
                const int Fa = vf ? R : P, Fb = vf ? S : Q, Ga = vf ? P : R, Gb = vf ? Q : S;
                const int needF = I * Fb * (Fa + kPad), needG = Gb * (Ga * I + kPad);
                need = needF + needG;
                if ((unsigned)need > RING) {   // a step larger than the ring: its F and G operands one after the other
                    part = ic.half ? 2 : 1;
                    need = part == 1 ? needF : needG;
                }
            }
            const int tx = need;                      // bytes / 4 the step's TMA boxes deliver (interior)
            if (kTma) need = (need + 31) & ~31;
            unsigned start = head, start_off = head_off;
            if (start_off + need > RING) { start += RING - start_off; start_off = 0; }   // never wrap a step
            if (qn == 0) tail = start;
            if (start + need - tail > RING) break;                                      // no room yet
            float* dst = ring + start_off;
            const float* xs = a.x.cores + ic.xo;
            const float* ys = a.y.cores + ic.yo;
            if (boundary) {
                stage_plain(dst, xs, R * I * S, lane);
                stage_plain(dst + ((R * I * S + 3) & ~3), ys, P * I * Q, lane);
            } else {
                const int Fa = vf ? R : P, Fb = vf ? S : Q, Ga = vf ? P : R, Gb = vf ? Q : S;
                if (kTma) {
                    // F as I Fb / 8 boxes of 8 runs of Fa, G as Gb / 8 boxes of 8 runs of Ga I, one box per lane
                    uint64_t* bar = bars + (qh + qn) % kQ;
                    if (lane == 0) tc::mbar_arrive_expect_tx(bar, 4u * (unsigned)tx);
                    __syncwarp();
                    const int nf = part != 2 ? (I * Fb) >> 3 : 0, ng = part != 1 ? Gb >> 3 : 0;
                    // (staging loops are kept rolled: a compact step loop in the instruction caches, +2% on C5)
#pragma unroll 1
                    for (int j = lane; j < nf + ng; j += 32) {
                        const bool isF = j < nf;
                        const int jj = isF ? j : j - nf, L = isF ? Fa : Ga * I;
                        const bool fromX = isF == (vf != 0);
                        const int64_t o = (fromX ? ic.xo : ic.yo) + (int64_t)8 * jj * L;
                        float* d = dst + (isF || part == 2 ? 0 : I * Fb * (Fa + kPad)) + jj * 8 * (L + kPad);
                        tc::fence_proxy_async();   // the slot's previous (generic-proxy) contents are dead
                        tc::tma_3d(d, &maps.m[maps.ix[fromX ? 0 : 1][L >> 2]], 0, 0, (int)(o >> 2), bar);
                    }
                } else {
                    const float* Fs = vf ? xs : ys;
                    const float* Gs = vf ? ys : xs;
                    if (part != 2) stage_padded(dst, Fs, I * Fb, Fa, lane);
                    if (part != 1) stage_padded(part == 2 ? dst : dst + I * Fb * (Fa + kPad), Gs, Gb, Ga * I, lane);
                }
            }
            tc::cp_commit_group();
            int znext = 0;   // the next step's Z orientation (the last step reads [r][p])
            if (n + 1 < N - 1) znext = (vfm[(n + 1) >> 5] >> ((n + 1) & 31)) & 1u;
            if (lane == 0) {
                FStep f;
                f.start = (int)start_off;
                f.b = ic.b; f.n = n; f.R = R; f.P = P; f.S = S; f.Q = Q; f.I = I;
                f.vf = vf;
                f.part = part;
                f.znext = znext;
                f.end = start + need;
                q[(qh + qn) % kQ] = f;
            }
            ++qn;
            head = start + need;
            head_off = start_off + need;
            if (part == 1) {   // the same step's G operand is staged next
                ic.half = true;
                continue;
            }
            ic.half = false;
            ic.xo += (int64_t)R * I * S;
            ic.yo += (int64_t)P * I * Q;
            ic.R = S;
            ic.P = Q;
            if (++ic.n == N) fc_pop(a, w, ic, rk, lane);
        }
        if (qn == 0) break;
        // ---- compute the oldest staged step
        tc::cp_wait_pending(qn - 1);   // boundary steps (cp.async); kTma: interior steps commit empty groups
        __syncwarp();
        const FStep f = q[qh];
        if (kTma && f.n != 0 && f.n != N - 1) {
            tc::mbar_wait(bars + qh, (phase >> qh) & 1u);
            phase ^= 1u << qh;
        }
        float* X = ring + f.start;
        if (f.n == N - 1) {   // last step (also N = 1)
            const float* Y = X + ((f.R * f.I * f.S + 3) & ~3);
            const float v = ff_last(X, Y, f.R, f.P, f.I, f.n == 0, Z, lane);
            if (lane == 0) a.out[f.b] = v;
        } else if (f.n == 0) {
            const float* Y = X + ((f.R * f.I * f.S + 3) & ~3);
            ff_first(X, Y, f.S, f.Q, f.I, f.znext, Z, lane);
        } else {
            const int vf = f.vf;
            const int Fa = vf ? f.R : f.P, Fb = vf ? f.S : f.Q, Ga = vf ? f.P : f.R, Gb = vf ? f.Q : f.S;
            // one call site per GEMM (part 0: both, 1: GEMM-1 on F, 2: GEMM-2 on G staged alone)
            if (f.part != 2) ff_step1(X, Fa, Fb, Ga, f.I, Z, W, lane);
            if (f.part != 1) ff_step2(Fb, f.part == 2 ? X : X + f.I * Fb * (Fa + kPad), Ga, Gb, f.I, Z, W, f.znext != vf, lane);
        }
        __syncwarp();
        tail = f.end;
        qh = (qh + 1) % kQ;
        --qn;
    }
    tc::cp_wait_pending(0);
}

// Floats of the per-warp buffers for a batch whose interior ranks are <= max_rank and dims <= max_dim.
struct FfSizes {
    int64_t step, half, zbuf, wbuf, qf;   // qf: step queue + the staged pair's rank rows
};
FfSizes ffma_sizes(int max_rank, int max_dim, int N) {
    const int64_t r = max_rank, I = max_dim;
    FfSizes z;
    z.step = I * r * (r + kPad) + r * (r * I + kPad) + 64;   // padded F + G regions of the largest step (+ slack)
    z.half = std::max(I * r * (r + kPad), r * (r * I + kPad)) + 64;   // its larger operand (a split step)
    z.zbuf = r * (r + kPad);
    z.wbuf = r * (r * I + kPad);
    z.qf = (kQ * (int64_t)sizeof(FStep) / 4 + 2 * kQ + 2 * (N + 1) + (N + 31) / 32 + 3) & ~int64_t(3);
    return z;
}
constexpr int64_t kSmemPerSM = 228 * 1024, kSmemPerCTA = 227 * 1024, kReservedPerCTA = 1024;

}  // namespace

bool inner_ffma_supported(const InnerArgs& a, int max_rank, bool ranks_mult8) {
    if (!ranks_mult8 || max_rank > 32 || a.N < 1) return false;
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = std::max(max_dim, (int)a.dims[n]);
    if (max_rank * max_dim / 4 > kMagicMax) return false;
    const FfSizes z = ffma_sizes(max_rank, max_dim, a.N);
    // at least 4 warps per SM, each holding one step of the largest shape
    return 4 * (4 * (z.step + z.zbuf + z.wbuf + z.qf) + kReservedPerCTA) <= kSmemPerSM;   // (z.half: split steps)
}

namespace {
// The tensor maps of the TMA staging path: every run length an interior step can stage (F: Fa = a rank <= max_rank
// and a multiple of 8; G: Ga I for the interior dims I), per buffer.  false if a run is too long for one box, the
// table is full, or an encoding fails -- the launch then stages with cp.async.
bool ffma_maps(const InnerArgs& a, int max_rank, int64_t nx, int64_t ny, FfMaps* m) {
    EncodeFn enc = encode_fn();
    if (!enc) return false;
    std::memset(m, 0, sizeof(*m));
    std::memset(m->ix, 0xff, sizeof(m->ix));
    int runs[kMaxMaps], nr = 0;
    auto add = [&](int L) {
        if (L % 4 != 0 || L / 4 > kMaxRunQ) return false;
        for (int i = 0; i < nr; ++i)
            if (runs[i] == L) return true;
        if (2 * (nr + 1) > kMaxMaps) return false;
        runs[nr++] = L;
        return true;
    };
    for (int r = 8; r <= max_rank; r += 8) {
        if (!add(r)) return false;
        for (int n = 1; n + 1 < a.N; ++n)
            if (!add(r * a.dims[n])) return false;
    }
    int k = 0;
    for (int buf = 0; buf < 2; ++buf) {
        const float* base = buf ? a.y.cores : a.x.cores;
        const int64_t n = buf ? ny : nx;
        if (n / 4 < 1 || n / 4 > (int64_t(1) << 31)) return false;
        for (int i = 0; i < nr; ++i, ++k) {
            const int L = runs[i];
            const cuuint64_t dims[3] = {(cuuint64_t)L, 8, (cuuint64_t)(n / 4)};
            const cuuint64_t strides[2] = {(cuuint64_t)4 * L, 16};
            const cuuint32_t box[3] = {(cuuint32_t)L + kPad, 8, 1};
            const cuuint32_t es[3] = {1, 1, 1};
            if (enc(&m->m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return false;
            m->ix[buf][L / 4] = (unsigned char)k;
        }
    }
    return true;
}
}  // namespace

cudaError_t launch_inner_ffma(const InnerArgs& a, int max_rank, bool aligned16, int64_t nx, int64_t ny,
                              cudaStream_t s) {
    int max_dim = 1;
    for (int n = 0; n < a.N; ++n) max_dim = std::max(max_dim, (int)a.dims[n]);
    const FfSizes z = ffma_sizes(max_rank, max_dim, a.N);
    const int64_t fixed = z.zbuf + z.wbuf + z.qf;
    // TMA staging unless TTC_FFMA_TMA=0 (A/B) or the maps cannot be built (TTC_FFMA_TMA=1: that is an error)
    FfMaps maps;          // the kernel parameter (copied at launch)
    const char* tv = std::getenv("TTC_FFMA_TMA");
    const bool want_tma = aligned16 && !(tv && tv[0] == '0');
    const bool tma = want_tma && ffma_maps(a, max_rank, nx, ny, &maps);
    if (tv && tv[0] == '1' && !tma) return cudaErrorNotSupported;
    if (!tma) std::memset(maps.ix, 0xff, sizeof(maps.ix));
    auto kern = tma ? inner_ffma_kernel<true> : inner_ffma_kernel<false>;
    // as many warps per SM as fit with a ring of at least one largest step (at most 16); the ring takes the rest
    // (shared memory is allocated per CTA in 256-byte units, plus 1 KB reserved per CTA)
    auto cta_bytes = [](int64_t floats) { return ((4 * floats + 255) & ~int64_t(255)) + kReservedPerCTA; };
    int per_sm = 16;
    // Steps larger than the ring are staged in two parts (F, then G), so the ring needs only the largest operand;
    // but a split step exposes a DRAM round trip, so the ring keeps at least 3/4 of the largest step (C5: 8 warps
    // per SM with rank-32 steps split, measured +8% over 7 warps holding whole steps; 9 warps: -5%)
    const int64_t ring_min = std::max(z.half, (3 * z.step) / 4);
    while (per_sm > 1 && per_sm * cta_bytes(ring_min + fixed) > kSmemPerSM) --per_sm;
    if (const char* v = std::getenv("TTC_FFMA_PER_SM")) {   // A/B: any count whose ring still holds a split step
        int want = std::max(1, std::atoi(v));
        while (want > 1 && want * cta_bytes(z.half + fixed) > kSmemPerSM) --want;
        per_sm = want;
    }
    int64_t warp_floats = (((kSmemPerSM / per_sm - kReservedPerCTA) & ~int64_t(255)) / 4);
    warp_floats = std::min<int64_t>(warp_floats, kSmemPerCTA / 4);
    FfArgs w;
    w.zbuf = (int)z.zbuf;
    w.wbuf = (int)z.wbuf;
    w.ring = (int)((warp_floats - fixed) & ~int64_t(31));   // 128-byte multiple: TMA destinations stay aligned
    w.warp_floats = (int)(w.ring + fixed);
    const size_t smem = sizeof(float) * (size_t)w.warp_floats;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess)
        return e;
    int dev = 0, sms = 0, occ = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, smem)) != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int grid = std::min(a.B, sms * occ);
    kern<<<grid, 32, smem, s>>>(a, w, maps);
    return cudaGetLastError();
}

}  // namespace ttc
