// contract.cu -- batched ladder tt_contract (ttc.h; Alg. 2 steps 4-6, generalised to K
// disjoint non-crossing mode pairs, readings R7-R10).  One CTA per pair.
//
// Per pair: (1) transfers T_k[(r + R p), (r' + R' p')] = sum_i X_{n_k}[r,i,r'] Y_{m_k}[p,i,p'] (the paper's
// K = A_x^T A_y generalised, Eq. 12) and products of consecutive transfers are formed in shared memory;
// (2) every output core is streamed to HBM in Eq. 2 order.  Free cores are Kronecker products with an
// identity (X_n (x) I_P or I_R (x) Y_m): their zeros are generated in registers, never read, and the
// absorbed transfer is applied structure-aware (sum over the non-identity bond only).  The kernel is
// bound by the output writes (output >> input), so stores are 16-byte streaming stores (st.global.cs).
#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kThreads = 256;

struct PairCtx {
    int32_t rx[kMaxContractOrder + 1], ry[kMaxContractOrder + 1];
    int64_t xo[kMaxContractOrder + 1], yo[kMaxContractOrder + 1];   // core offsets within the train
    int32_t orr[kMaxLadder + 1];                                     // output bond ranks
    int64_t oo[kMaxLadder + 1];                                      // output core offsets within the pair
};

__device__ __forceinline__ void st_cs4(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void st_cs1(float* p, float a) {
    asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}

// T_k (rows = R_{n-1} P_{m-1}, cols = R_n P_m) into dst, column-major.
__device__ void build_transfer(const ContractArgs& a, const PairCtx& c, const float* xc, const float* yc,
                               const LadderEl& el, float* dst) {
    const int n = el.mode, m = el.hold;
    const int R = c.rx[n], Rn = c.rx[n + 1], P = c.ry[m], Pn = c.ry[m + 1], I = a.xdims[n];
    const float* X = xc + c.xo[n];
    const float* Y = yc + c.yo[m];
    const int rows = R * P, total = rows * Rn * Pn;
    if ((R & 3) == 0 && ((reinterpret_cast<uintptr_t>(X) & 15u) == 0) && ((I * R) & 3) == 0) {
        // four consecutive r per thread: X[r..r+3, i, r'] is one 16-byte load
        const int R4 = R >> 2, total4 = total >> 2;
        for (int e = threadIdx.x; e < total4; e += blockDim.x) {
            int q = e;
            const int r4 = q % R4; q /= R4;
            const int p = q % P; q /= P;
            const int rr = q % Rn, pp = q / Rn;
            const float* xp = X + 4 * r4 + R * I * rr;
            const float* yp = Y + p + P * I * pp;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = 0; i < I; ++i) {
                const float4 xv = *reinterpret_cast<const float4*>(xp + R * i);
                const float yv = yp[P * i];
                acc.x = fmaf(xv.x, yv, acc.x); acc.y = fmaf(xv.y, yv, acc.y);
                acc.z = fmaf(xv.z, yv, acc.z); acc.w = fmaf(xv.w, yv, acc.w);
            }
            float* d = dst + 4 * r4 + R * (p + P * (rr + Rn * pp));
            d[0] = acc.x; d[1] = acc.y; d[2] = acc.z; d[3] = acc.w;
        }
        return;
    }
    // (r, p, r', p') of entry e by nested loops: e = r + R (p + P (r' + R' p'))
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        int q = e;
        const int r = q % R; q /= R;
        const int p = q % P; q /= P;
        const int rr = q % Rn, pp = q / Rn;
        const float* xp = X + r + R * I * rr;
        const float* yp = Y + p + P * I * pp;
        float acc = 0.0f;
        for (int i = 0; i < I; ++i) acc = fmaf(xp[R * i], yp[P * i], acc);
        dst[e] = acc;
    }
}

// C (m x n) = A (m x k) * B (k x n), column-major, shared memory.
__device__ void smem_matmul(const float* A, const float* B, float* C, int m, int k, int n) {
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
        const int i = e % m, j = e / m;
        float acc = 0.0f;
        for (int l = 0; l < k; ++l) acc = fmaf(A[i + m * l], B[l + k * j], acc);
        C[e] = acc;
    }
}

// Product of `count` consecutive transfers starting at sequence index `first` into dst; returns rows/cols.
__device__ void build_chain(const ContractArgs& a, const PairCtx& c, const float* xc, const float* yc, int first,
                            int count, float* dst, float* tmp, int* rows_out, int* cols_out) {
    const LadderEl& e0 = a.seq[first];
    const int rows = c.rx[e0.mode] * c.ry[e0.hold];
    int cols = c.rx[e0.mode + 1] * c.ry[e0.hold + 1];
    if (count == 1) {
        build_transfer(a, c, xc, yc, e0, dst);
    } else {
        float* cur = tmp;
        float* nxt = tmp + a.tmp_size;
        float* prod = tmp + 2 * a.tmp_size;
        build_transfer(a, c, xc, yc, e0, cur);
        for (int t = 1; t < count; ++t) {
            const LadderEl& et = a.seq[first + t];
            __syncthreads();
            build_transfer(a, c, xc, yc, et, nxt);
            __syncthreads();
            const int kk = cols;
            const int nn = c.rx[et.mode + 1] * c.ry[et.hold + 1];
            float* target = (t == count - 1) ? dst : prod;
            smem_matmul(cur, nxt, target, rows, kk, nn);
            cols = nn;
            if (t != count - 1) { float* sw = cur; cur = prod; prod = sw; }
        }
    }
    *rows_out = rows;
    *cols_out = cols;
}

// Geometry of one free core before absorption.
struct FreeCore {
    bool xfree;
    const float* G;   // source core values
    int Rb;           // XFREE: R (X left bond);  YFREE: P (Y left bond)
    int Rn;           // XFREE: R' (X right bond); YFREE: P'
    int H;            // carried identity size: XFREE: P_b;  YFREE: R_a
    int I;            // mode size
    int Ain, Bin;     // rows / cols before absorption: XFREE (R H, R' H), YFREE (H P, H P')
};

// Value of the (left-absorbed or plain) core at (alpha, i, gamma); gamma indexes the pre-absorption cols.
__device__ __forceinline__ float cprime(const FreeCore& f, const float* TL, int Aout, bool has_tl, int alpha, int i,
                                        int gamma) {
    if (f.xfree) {   // [r + R p, i, r' + R' p'] = X[r, i, r'] delta_{p p'}
        const int rr = gamma % f.Rn, pp = gamma / f.Rn;
        const float* col = f.G + f.Rb * (i + f.I * rr);
        if (has_tl) {
            float acc = 0.0f;
            for (int r = 0; r < f.Rb; ++r) acc = fmaf(TL[alpha + Aout * (r + f.Rb * pp)], col[r], acc);
            return acc;
        }
        const int r = alpha - f.Rb * pp;
        return (r >= 0 && r < f.Rb) ? col[r] : 0.0f;
    } else {         // [r + H p, j, r' + H p'] = delta_{r r'} Y[p, j, p']
        const int rr = gamma % f.H, pp = gamma / f.H;
        const float* col = f.G + f.Rb * (i + f.I * pp);
        if (has_tl) {
            float acc = 0.0f;
            for (int p = 0; p < f.Rb; ++p) acc = fmaf(TL[alpha + Aout * (rr + f.H * p)], col[p], acc);
            return acc;
        }
        const int d = alpha - rr;
        if (d < 0 || d % f.H) return 0.0f;
        const int p = d / f.H;
        return p < f.Rb ? col[p] : 0.0f;
    }
}

// 4 FMAs of one alpha-quad column against one scalar, packed (FFMA2: two FMAs per issue slot).
__device__ __forceinline__ void quad_fma(float4& v, const float4 t, float g) {
    unsigned long long lo, hi, tlo, thi, gg;
    asm("mov.b64 %0, {%1, %2};" : "=l"(lo) : "f"(v.x), "f"(v.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(hi) : "f"(v.z), "f"(v.w));
    asm("mov.b64 %0, {%1, %2};" : "=l"(tlo) : "f"(t.x), "f"(t.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(thi) : "f"(t.z), "f"(t.w));
    asm("mov.b64 %0, {%1, %1};" : "=l"(gg) : "f"(g));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(lo) : "l"(tlo), "l"(gg));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(hi) : "l"(thi), "l"(gg));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(lo));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.z), "=f"(v.w) : "l"(hi));
}

// Fast emission of one free core (no right absorption): every thread owns one alpha-quad of one mode index i
// and walks the output columns beta = rr + Bs pp in steps of nb = blockDim / Q, writing one 16-byte streaming
// store per column; consecutive threads write consecutive 16-byte chunks.  KIND: 0 X (x) I, 1 TL (X (x) I),
// 2 I (x) Y, 3 TL (I (x) Y).  The free core's column it reads is contiguous along the summed bond.
template <int KIND>
__device__ __forceinline__ void emit_fast(const FreeCore& f, const float* TL, int Aout, int Bout, int Q, int Bs,
                                          float* dst) {
    const int I = f.I, R = f.Rb;
    const int qpa = Aout >> 2, nb = blockDim.x / Q;
    const int t = threadIdx.x;
    if (t >= nb * Q) return;
    const int a0 = 4 * (t % qpa), i = (t / qpa) % I;
    int beta = t / Q;
    int rr = beta % Bs, pp = beta / Bs;
    const int blk = KIND < 2 ? R : f.H;
    const int pblk = a0 / blk, roff = a0 - blk * pblk;   // this quad's rows: roff.. of block pblk
    float* d = dst + a0 + (int64_t)Aout * (i + (int64_t)I * beta);
    const int64_t dstep = (int64_t)Aout * I * nb;
    const int rstep = nb % Bs, pstep = nb / Bs;
    const float* gbase = f.G + R * i;                    // column (i, c) of the free core at gbase + R I c
    const int gstride = R * I;
    const int hs = Aout * f.H;
    for (; beta < Bout; beta += nb, d += dstep) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (KIND == 0) {          // rows r + R pp carry X[r, i, rr]
            if (pp == pblk) v = *reinterpret_cast<const float4*>(gbase + gstride * rr + roff);
        } else if (KIND == 1) {   // sum_r TL[a0.., r + R pp] X[r, i, rr]
            const float* gcol = gbase + gstride * rr;
            const float* tl = TL + a0 + Aout * (R * pp);
            float4 v2 = v;
            for (int r = 0; r < R; r += 4) {
                const float4 g = *reinterpret_cast<const float4*>(gcol + r);
                quad_fma(v, *reinterpret_cast<const float4*>(tl + Aout * r), g.x);
                quad_fma(v2, *reinterpret_cast<const float4*>(tl + Aout * (r + 1)), g.y);
                quad_fma(v, *reinterpret_cast<const float4*>(tl + Aout * (r + 2)), g.z);
                quad_fma(v2, *reinterpret_cast<const float4*>(tl + Aout * (r + 3)), g.w);
            }
            v.x += v2.x; v.y += v2.y; v.z += v2.z; v.w += v2.w;
        } else if (KIND == 2) {   // rows rr + H p carry Y[p, j, pp]: this quad holds row rr + H pblk if any
            const int k = rr - roff;
            if ((unsigned)k < 4u) {
                const float val = gbase[gstride * pp + pblk];
                v.x = k == 0 ? val : 0.f; v.y = k == 1 ? val : 0.f; v.z = k == 2 ? val : 0.f; v.w = k == 3 ? val : 0.f;
            }
        } else {                  // sum_p TL[a0.., rr + H p] Y[p, j, pp]
            const float* gcol = gbase + gstride * pp;
            const float* tl = TL + a0 + Aout * rr;
            float4 v2 = v;
            for (int q = 0; q < R; q += 4) {
                const float4 g = *reinterpret_cast<const float4*>(gcol + q);
                quad_fma(v, *reinterpret_cast<const float4*>(tl + hs * q), g.x);
                quad_fma(v2, *reinterpret_cast<const float4*>(tl + hs * (q + 1)), g.y);
                quad_fma(v, *reinterpret_cast<const float4*>(tl + hs * (q + 2)), g.z);
                quad_fma(v2, *reinterpret_cast<const float4*>(tl + hs * (q + 3)), g.w);
            }
            v.x += v2.x; v.y += v2.y; v.z += v2.z; v.w += v2.w;
        }
        st_cs4(d, v.x, v.y, v.z, v.w);
        rr += rstep;
        pp += pstep;
        if (rr >= Bs) { rr -= Bs; ++pp; }
    }
}

// The same emission when nb divides Bs (every thread's betas share its rr residue): nested loops with the
// absorbed transfer's columns held in registers across the inner loop -- KIND 1 (TL (X (x) I)): TL[a0.., r + R pp]
// depends on pp only, so pp is the outer loop; KIND 3 (TL (I (x) Y)): TL[a0.., rr + H q] depends on rr only, so
// rr is the outer loop.  R = 4 RQ (RQ <= 2: the cached quads stay within the 64-register budget).
template <int KIND, int RQ>
__device__ __forceinline__ void emit_nested(const FreeCore& f, const float* TL, int Aout, int Bout, int Q, int Bs,
                                            float* dst) {
    constexpr int R = 4 * RQ;
    const int I = f.I;
    const int qpa = Aout >> 2, nb = blockDim.x / Q;
    const int t = threadIdx.x;
    if (t >= nb * Q) return;
    const int a0 = 4 * (t % qpa), i = (t / qpa) % I, g0 = t / Q;
    const int blk = KIND < 2 ? R : f.H;
    const int pblk = a0 / blk, roff = a0 - blk * pblk;
    const int np = Bout / Bs;
    const int64_t cstride = (int64_t)Aout * I;   // floats between consecutive output columns beta
    float* d0 = dst + a0 + (int64_t)Aout * i;
    const float* gbase = f.G + R * i;
    const int gstride = R * I;
    const int64_t dcol = cstride * nb, dpp = cstride * Bs;   // output step per thread column / per pp
    if (KIND == 1) {
        for (int pp = 0; pp < np; ++pp) {
            float4 tq[R];
#pragma unroll
            for (int r = 0; r < R; ++r) tq[r] = *reinterpret_cast<const float4*>(TL + a0 + Aout * (r + R * pp));
            const float* gcol = gbase + gstride * g0;
            float* dp = d0 + cstride * (g0 + (int64_t)Bs * pp);
            for (int rr = g0; rr < Bs; rr += nb, gcol += gstride * nb, dp += dcol) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int r = 0; r < R; r += 4) {
                    const float4 g = *reinterpret_cast<const float4*>(gcol + r);
                    quad_fma(v, tq[r], g.x);
                    quad_fma(v, tq[r + 1], g.y);
                    quad_fma(v, tq[r + 2], g.z);
                    quad_fma(v, tq[r + 3], g.w);
                }
                st_cs4(dp, v.x, v.y, v.z, v.w);
            }
        }
    } else if (KIND == 3) {
        const int hs = Aout * f.H;
        for (int rr = g0; rr < Bs; rr += nb) {
            float4 tq[R];
#pragma unroll
            for (int q = 0; q < R; ++q) tq[q] = *reinterpret_cast<const float4*>(TL + a0 + Aout * rr + hs * q);
            const float* gcol = gbase;
            float* dp = d0 + cstride * rr;
            for (int pp = 0; pp < np; ++pp, gcol += gstride, dp += dpp) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int q = 0; q < R; q += 4) {
                    const float4 g = *reinterpret_cast<const float4*>(gcol + q);
                    quad_fma(v, tq[q], g.x);
                    quad_fma(v, tq[q + 1], g.y);
                    quad_fma(v, tq[q + 2], g.z);
                    quad_fma(v, tq[q + 3], g.w);
                }
                st_cs4(dp, v.x, v.y, v.z, v.w);
            }
        }
    } else if (KIND == 0) {   // rows r + R pp carry X[r, i, rr]: only pp == pblk is nonzero
        float* dp = d0 + cstride * g0;
        for (int pp = 0; pp < np; ++pp, dp += dpp) {
            const float* gp = gbase + gstride * g0 + roff;
            float* dq = dp;
            for (int rr = g0; rr < Bs; rr += nb, gp += gstride * nb, dq += dcol) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (pp == pblk) v = *reinterpret_cast<const float4*>(gp);
                st_cs4(dq, v.x, v.y, v.z, v.w);
            }
        }
    } else {                  // rows rr + H p carry Y[p, j, pp]: the quad holds row rr + H pblk iff rr - roff < 4
        for (int rr = g0; rr < Bs; rr += nb) {
            const int k = rr - roff;
            const bool has = (unsigned)k < 4u;   // lanes differ: predicated loads, one store stream per warp
            const float* gp = gbase + pblk;
            float* dp = d0 + cstride * rr;
            for (int pp = 0; pp < np; ++pp, gp += gstride, dp += dpp) {   // selects: exact zeros whatever val is
                const float val = has ? *gp : 0.f;
                st_cs4(dp, k == 0 ? val : 0.f, k == 1 ? val : 0.f, k == 2 ? val : 0.f, k == 3 ? val : 0.f);
            }
        }
    }
}

__device__ void emit_core(const ContractArgs& a, const PairCtx& c, const float* xc, const float* yc, int l,
                          const float* TL, const float* TR, float* out) {
    const OutCore& oc = a.outc[l];
    const LadderEl& el = a.seq[oc.el];
    FreeCore f;
    f.xfree = el.kind == EL_XFREE;
    if (f.xfree) {
        f.G = xc + c.xo[el.mode];
        f.Rb = c.rx[el.mode]; f.Rn = c.rx[el.mode + 1]; f.H = c.ry[el.hold]; f.I = a.xdims[el.mode];
        f.Ain = f.Rb * f.H; f.Bin = f.Rn * f.H;
    } else {
        f.G = yc + c.yo[el.mode];
        f.Rb = c.ry[el.mode]; f.Rn = c.ry[el.mode + 1]; f.H = c.rx[el.hold]; f.I = a.ydims[el.mode];
        f.Ain = f.H * f.Rb; f.Bin = f.H * f.Rn;
    }
    const bool has_tl = oc.lt_count > 0, has_tr = oc.rt_count > 0;
    const int Aout = c.orr[l], Bout = c.orr[l + 1];
    const int I = f.I;
    const int64_t total = (int64_t)Aout * I * Bout;
    float* dst = out + c.oo[l];
    const int qpa = Aout >> 2;                              // alpha-quads per column
    const int Q = qpa * I;                                  // threads per output column group (one beta)
    const int Bs = f.xfree ? f.Rn : f.H;                    // beta = rr + Bs * pp
    const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(f.G)) & 15u) == 0 &&
                         ((reinterpret_cast<uintptr_t>(TL) & 15u) == 0);
    // fast path: every thread owns one alpha-quad of one mode index i and walks beta in steps of nb; the free
    // core's column (i, rr) / (i, pp) it reads is contiguous along the summed bond (16-byte loads)
    const bool fast = !has_tr && (Aout & 3) == 0 && (f.Rb & 3) == 0 && aligned && Q <= (int)blockDim.x &&
                      (f.xfree ? true : (f.H & 3) == 0) && total < (1ll << 31);
    if (fast && Bs % (blockDim.x / Q) == 0 && Bout % Bs == 0 && (f.Rb == 4 || f.Rb == 8)) {
        const int kind = (f.xfree ? 0 : 2) + (has_tl ? 1 : 0);
        if (f.Rb == 8) {
            switch (kind) {
                case 0: emit_nested<0, 2>(f, TL, Aout, Bout, Q, Bs, dst); break;
                case 1: emit_nested<1, 2>(f, TL, Aout, Bout, Q, Bs, dst); break;
                case 2: emit_nested<2, 2>(f, TL, Aout, Bout, Q, Bs, dst); break;
                default: emit_nested<3, 2>(f, TL, Aout, Bout, Q, Bs, dst); break;
            }
        } else {
            switch (kind) {
                case 0: emit_nested<0, 1>(f, TL, Aout, Bout, Q, Bs, dst); break;
                case 1: emit_nested<1, 1>(f, TL, Aout, Bout, Q, Bs, dst); break;
                case 2: emit_nested<2, 1>(f, TL, Aout, Bout, Q, Bs, dst); break;
                default: emit_nested<3, 1>(f, TL, Aout, Bout, Q, Bs, dst); break;
            }
        }
        return;
    }
    if (fast) {
        const int kind = (f.xfree ? 0 : 2) + (has_tl ? 1 : 0);
        switch (kind) {
            case 0: emit_fast<0>(f, TL, Aout, Bout, Q, Bs, dst); break;
            case 1: emit_fast<1>(f, TL, Aout, Bout, Q, Bs, dst); break;
            case 2: emit_fast<2>(f, TL, Aout, Bout, Q, Bs, dst); break;
            default: emit_fast<3>(f, TL, Aout, Bout, Q, Bs, dst); break;
        }
        return;
    }
    // general element path (right absorption, unaligned or odd row counts)
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
        const int alpha = (int)(e % Aout);
        const int64_t col = e / Aout;
        const int i = (int)(col % I), beta = (int)(col / I);
        float v;
        if (has_tr) {
            v = 0.0f;
            for (int g = 0; g < f.Bin; ++g) v = fmaf(cprime(f, TL, Aout, has_tl, alpha, i, g), TR[g + f.Bin * beta], v);
        } else {
            v = cprime(f, TL, Aout, has_tl, alpha, i, beta);
        }
        st_cs1(dst + e, v);
    }
}

__device__ __forceinline__ void cp_async4_(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16_(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
// Contiguous copy of n floats global -> shared with cp.async (16-byte pieces when both ends are aligned); the
// caller waits (cp.async.wait_all) and synchronises.
__device__ __forceinline__ void stage_async(float* dst, const float* src, int n) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u) == 0) {
        for (int e = threadIdx.x; e < (n >> 2); e += blockDim.x) cp_async16_(dst + 4 * e, src + 4 * e);
        for (int e = (n & ~3) + threadIdx.x; e < n; e += blockDim.x) cp_async4_(dst + e, src + e);
    } else {
        for (int e = threadIdx.x; e < n; e += blockDim.x) cp_async4_(dst + e, src + e);
    }
}

__global__ void __launch_bounds__(kThreads, 4) contract_kernel(const ContractArgs a) {
    extern __shared__ float scratch[];
    __shared__ PairCtx c;
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        for (int n = 0; n <= a.N; ++n)
            c.rx[n] = a.x.ranks ? a.x.ranks[(int64_t)b * (a.N + 1) + n] : ((n == 0 || n == a.N) ? 1 : a.x.urank);
        for (int m = 0; m <= a.M; ++m)
            c.ry[m] = a.y.ranks ? a.y.ranks[(int64_t)b * (a.M + 1) + m] : ((m == 0 || m == a.M) ? 1 : a.y.urank);
        c.xo[0] = 0;
        for (int n = 0; n < a.N; ++n) c.xo[n + 1] = c.xo[n] + (int64_t)c.rx[n] * a.xdims[n] * c.rx[n + 1];
        c.yo[0] = 0;
        for (int m = 0; m < a.M; ++m) c.yo[m + 1] = c.yo[m] + (int64_t)c.ry[m] * a.ydims[m] * c.ry[m + 1];
        // output bond ranks: the right bond of each output core; first and last are 1
        c.orr[0] = 1;
        for (int l = 0; l < a.L; ++l) {
            const LadderEl& el = a.seq[a.outc[l].el];
            c.orr[l + 1] = el.kind == EL_XFREE ? c.rx[el.mode + 1] * c.ry[el.hold] : c.rx[el.hold] * c.ry[el.mode + 1];
        }
        c.orr[a.L] = 1;
        c.oo[0] = 0;
        for (int l = 0; l < a.L; ++l) {
            const LadderEl& el = a.seq[a.outc[l].el];
            const int I = el.kind == EL_XFREE ? a.xdims[el.mode] : a.ydims[el.mode];
            c.oo[l + 1] = c.oo[l] + (int64_t)c.orr[l] * I * c.orr[l + 1];
        }
    }
    __syncthreads();
    const float* xg = a.x.cores + (a.x.offsets ? a.x.offsets[b] : (int64_t)b * a.x.train_elems);
    const float* yg = a.y.cores + (a.y.offsets ? a.y.offsets[b] : (int64_t)b * a.y.train_elems);
    float* out = a.out + (a.out_offsets ? a.out_offsets[b] : (int64_t)b * a.out_pair_elems);
    float* TL = scratch + a.tl_off;
    float* TR = scratch + a.tr_off;
    float* tmp = scratch + a.tmp_off;
    // stage both trains in shared memory when they fit (every core value is read many times)
    const float* xc = xg;
    const float* yc = yg;
    const int64_t nx = c.xo[a.N], ny = c.yo[a.M];
    if (a.stage_floats > 0 && nx + ny <= a.stage_floats) {
        float* sx = scratch + a.stage_off;
        float* sy = sx + nx;
        stage_async(sx, xg, (int)nx);   // every load of both trains in flight at once (one round trip)
        stage_async(sy, yg, (int)ny);
        asm volatile("cp.async.wait_all;" ::: "memory");
        xc = sx;
        yc = sy;
    }
    for (int l = 0; l < a.L; ++l) {
        const OutCore& oc = a.outc[l];
        int rows, cols;
        __syncthreads();   // the staged trains (first core) / the previous core's buffers are ready / free
        if (oc.lt_count > 0) build_chain(a, c, xc, yc, oc.lt_first, oc.lt_count, TL, tmp, &rows, &cols);
        if (oc.rt_count > 0) {
            __syncthreads();
            build_chain(a, c, xc, yc, oc.rt_first, oc.rt_count, TR, tmp, &rows, &cols);
        }
        __syncthreads();
        emit_core(a, c, xc, yc, l, TL, TR, out);
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_contract(const ContractArgs& a, size_t smem_bytes, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes);
    if (e != cudaSuccess) return e;
    contract_kernel<<<a.B, kThreads, smem_bytes, s>>>(a);
    return cudaGetLastError();
}

cudaError_t contract_func_attributes(cudaFuncAttributes* fa) { return cudaFuncGetAttributes(fa, contract_kernel); }

}  // namespace ttc
