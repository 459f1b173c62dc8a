// ttsvd_big.cu -- TT-SVD (Alg. 1) of tensors too large for the shared-memory kernels of
// ttsvd.cu (more than 16,384 elements, or an unfolding whose smaller side exceeds 64: Example 2's cases (ii)
// 20 x 20 x 20 x 5 and (iii) 20 x 20 x 20 x 5 x 4, whose middle unfoldings are 400 x 100 and
// 400 x 400), over a caller-owned fp64 workspace (ttc_tt_svd_workspace).
//
// Each step n factors the unfolding Z (m x c, column-major: the Eq. 2 order of the remaining modes) by ONE-SIDED
// Jacobi (Hestenes) on the matrix A whose s = min(m, c) columns are orthogonalised:
//   m <= c:  A = Z^T (c x m).  A V has orthogonal columns  =>  V = U (left singular vectors of Z) and
//            (A V)^T = U^T Z = S V'^T, the next unfolding, directly.
//   m >  c:  A = Z   (m x c).  Z V = U S  =>  U = columns of Z V / sigma, next unfolding S V^T.
// Rotations of column pairs in the parallel round-robin order, until a sweep rotates nothing
// (|a_p . a_q| <= 1e-9 sqrt(|a_p|^2 |a_q|^2), R26); singular values = norms of A V's columns.  The
// delta-truncated rank, the 1e-7 singular-value floor (R25) and the sign convention (R24: the largest-magnitude entry of every
// left singular vector positive, the matching row of S V^T flipped with it) are Alg. 1's as the oracle reads
// them (oracle/ttsvd.py).  Alg. 2 step 1's permutation is folded into the first read.
//
// Parallelism: a GROUP of C co-resident CTAs per tensor (cooperative launch), synchronised by a per-tensor
// counter barrier in the workspace.  The s/2 rotations of a round are independent: one warp per column pair
// when the columns are short, one CTA per pair (block reductions) when they are long (L >= 2048, e.g. the
// 8,000-long columns of case (iii)'s first unfolding).  Every reduction is in a fixed order, so the result does
// not depend on C.  A, V and Z live in L2 / HBM (a 400 x 400 fp64 A is 1.25 MB).
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "ttc_internal.h"

namespace ttc {
namespace {

constexpr int kBigThreads = 512;
constexpr int kBigWarps = kBigThreads / 32;
constexpr double kSigmaFloor = 1e-7;   // R25
constexpr int kMaxSweeps = 60;
constexpr int kMaxGroup = 64;          // CTAs per tensor
constexpr int kSyncInts = 32;          // per tensor: barrier counter, rotation counter (128 bytes apart)
constexpr int kCtaPairL = 2048;        // columns at least this long: one CTA per pair
constexpr int kRegCol = 16;            // warp-per-pair columns up to 32 kRegCol long are held in registers
constexpr int kMaxBlk2 = 32;           // block mode: at most 2 x 16 columns per block pair
constexpr int kLocalSweeps = 1;        // block mode: full local sweeps in a sweep's first block round
constexpr int kDynBytes = 200 * 1024;  // block mode: dynamic shared memory per CTA
static_assert(kBigWarps >= kMaxBlk2 / 2, "block mode: one warp per column pair of a full block round");

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ unsigned ld_acquire(const int* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Barrier of the C CTAs of one tensor: a monotone arrival counter (zeroed by the host before the launch).
__device__ __forceinline__ void group_barrier(int* cnt, unsigned& target, int C) {
    __syncthreads();
    target += (unsigned)C;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1);
        while (ld_acquire(cnt) < target) {
        }
    }
    __syncthreads();
}

// round-robin tournament: the player at position pos in round r (position 0 fixed, the others rotate)
__device__ __forceinline__ int rr_player(int pos, int r, int S) { return pos == 0 ? 0 : ((pos - 1 + r) % (S - 1)) + 1; }

// Jacobi rotation of columns (ap, aq) given their Gram entries; false when already orthogonal
__device__ __forceinline__ bool rotation(double al, double be, double ga, double tol, double& cs, double& sn) {
    if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) return false;
    const double zeta = (be - al) / (2.0 * ga);
    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
    cs = 1.0 / sqrt(1.0 + t * t);
    sn = cs * t;
    return true;
}

__global__ void __launch_bounds__(kBigThreads) ttsvd_big_kernel(const TtsvdArgs a, double* ws, int* sync,
                                                               int64_t ws_per, int C, int b0, int dyn_doubles) {
    __shared__ double sig[kTtsvdBigMaxSide];
    __shared__ int ord[kTtsvdBigMaxSide];
    __shared__ double red[3][kBigWarps];
    __shared__ double bc[4];
    __shared__ int rank_s, rot_any, rot_now, lrot, lrot_any;
    extern __shared__ double dsm[];   // block mode: two column blocks of A and their rotation matrix
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = blockIdx.x / C, cg = blockIdx.x - g * C;   // tensor of the chunk, CTA within its group
    const int b = b0 + g;
    if (b >= a.B) return;   // whole groups only: every CTA of a group takes this branch or none does
    const int N = a.N, elems = a.elems, gmax = a.gmax;
    double* Z = ws + (int64_t)b * ws_per;   // current unfolding, column-major
    double* A = Z + elems;                  // the matrix whose columns are orthogonalised
    double* V = A + elems;                  // accumulated rotations (s x s)
    double* sig_g = V + (int64_t)gmax * gmax;
    double* sgn_g = sig_g + gmax;
    double* part = sgn_g + gmax;            // kMaxGroup partial norms
    int* cnt = sync + (int64_t)b * kSyncInts;
    int* rot = cnt + 16;
    unsigned target = 0;
    const float* src = a.dense + (int64_t)b * elems;
    float* core = a.cores + (int64_t)b * a.train_cap;
    int32_t* rk = a.ranks + (int64_t)b * (N + 1);
    const int gt = cg * kBigThreads + tid, gts = C * kBigThreads;   // thread index / count in the group
    const int gw = cg * kBigWarps + warp, gws = C * kBigWarps;      // warp index / count in the group

    // ---- Z_0 = X^rho (Alg. 2 step 1's permutation folded into the gather), ||X||^2 (fixed-order partials)
    double nrm = 0.0;
    for (int e = gt; e < elems; e += gts) {
        int q = e;
        int64_t off = 0;
        for (int k = 0; k < N; ++k) {
            const int ik = q % a.dims[k];
            q /= a.dims[k];
            off += (int64_t)ik * a.in_stride[k];
        }
        const double v = src[off];
        Z[e] = v;
        nrm += v * v;
    }
    nrm = warp_sum(nrm);
    if (lane == 0) red[0][warp] = nrm;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kBigWarps; ++w) t += red[0][w];
        part[cg] = t;
    }
    group_barrier(cnt, target, C);
    if (tid == 0) {
        double t = 0.0;
        for (int k = 0; k < C; ++k) t += part[k];
        bc[0] = t;
        if (cg == 0) {
            rk[0] = 1;
            rk[N] = 1;
        }
    }
    __syncthreads();
    const double delta2 = a.eps2 * bc[0];   // (eps / sqrt(N - 1))^2 ||X||^2

    int Rp = 1;                 // R_{n-1}
    int64_t cur = elems;        // elements of the current unfolding
    int64_t coff = 0;           // offset of core n in the train
    int rot_seen = 0;           // the rotation counter after the previous sweep (the same in every CTA)
    for (int n = 0; n + 1 < N; ++n) {
        const int m = Rp * a.dims[n];
        const int c = (int)(cur / m);
        const bool wide = m <= c;            // A = Z^T
        const int s = wide ? m : c, L = wide ? c : m;
        // A (L x s, column-major) and V = I (s x s)
        for (int64_t e = gt; e < (int64_t)L * s; e += gts) {
            const int row = (int)(e % L), col = (int)(e / L);
            A[e] = wide ? Z[col + (int64_t)m * row] : Z[e];
        }
        for (int64_t e = gt; e < (int64_t)s * s; e += gts) V[e] = (e % s) == (e / s) ? 1.0 : 0.0;
        group_barrier(cnt, target, C);
        // ---- one-sided Jacobi sweeps
        const int S = s + (s & 1);
        const bool cta_pairs = L >= kCtaPairL;
        // orthogonality tolerance (R26): columns orthogonal to 1e-9 relative, 60x below the unit roundoff
        // of the fp32 cores the factors are stored in (the singular values, the column norms, are then exact to
        // ~1e-18 relative); LAPACK dgesvj's sqrt(L) eps_64 costs extra full sweeps that change no stored bit of
        // consequence (A2ii +6.6%, A2iii +4.2% measured)
        const double tol = fmax(1e-9, sqrt((double)L) * DBL_EPSILON);
        // block mode: columns per block (two blocks of A and their rotation matrix Q -- always 32 x 32, identity
        // past the pair's columns, so the V update can run its fixed 32-term loop -- in shared memory)
        int bs = 16;
        while (bs > 4 && (int64_t)L * 2 * bs + kMaxBlk2 * kMaxBlk2 > dyn_doubles) bs >>= 1;
        const bool block_mode = !cta_pairs && s >= 32 && (int64_t)L * 2 * bs + kMaxBlk2 * kMaxBlk2 <= dyn_doubles;
        if (block_mode) {
            // Block one-sided Jacobi: the s columns in nb blocks of bs, block pairs in the round-robin order (one
            // CTA per block pair, nb - 1 group barriers per sweep instead of s - 1); a block pair is loaded into
            // shared memory and orthogonalised there by local round-robin sweeps (warp per column pair), its
            // rotations accumulated in a 2bs x 2bs matrix Q and applied to V's columns once: V_pair <- V_pair Q.
            const int nb0 = (s + bs - 1) / bs, nb = nb0 + (nb0 & 1);
            const int ldq = kMaxBlk2;
            double* As = dsm;                             // nl columns of L doubles
            double* Qm = dsm + (int64_t)L * 2 * bs;       // 32 x 32, column-major (the pair's nl x nl in the corner)
            for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
                if (tid == 0) rot_any = 0;
                __syncthreads();
                for (int r = 0; r < nb - 1; ++r) {
                    for (int k = cg; k < nb / 2; k += C) {
                        const int P = rr_player(k, r, nb), Qb = rr_player(nb - 1 - k, r, nb);
                        const int p0 = P * bs, np = max(0, min(bs, s - p0));
                        const int q0 = Qb * bs, nq = max(0, min(bs, s - q0));
                        const int nl = np + nq;
                        if (nl < 2) continue;
                        for (int e = tid; e < nl * L; e += kBigThreads) {
                            const int j = e / L, i = e - j * L;
                            As[e] = A[(int64_t)L * (j < np ? p0 + j : q0 + j - np) + i];
                        }
                        for (int e = tid; e < ldq * ldq; e += kBigThreads) Qm[e] = (e % ldq) == (e / ldq) ? 1.0 : 0.0;
                        if (tid == 0) lrot_any = 0;
                        __syncthreads();
                        // the sweep's first block round pairs every block once: a full local sweep there covers
                        // the pairs inside the blocks; later rounds only the np x nq cross pairs (Latin square:
                        // round t pairs local column i with np + (i + t) mod M, M = max(np, nq))
                        const bool full = r == 0;
                        const int S2 = nl + (nl & 1), M = max(np, nq);
                        const int nrl = full ? S2 - 1 : M;
                        if (!full && L <= 32 * kRegCol) {
                            // cross rounds with short columns: warp w keeps its P column (local w) in registers for
                            // all M rounds and only streams the partner Q columns through shared memory
                            if (tid == 0) lrot = 0;
                            __syncthreads();
                            double xr[kRegCol];
                            double* xcol = As + (int64_t)L * warp;
                            if (warp < np) {
#pragma unroll
                                for (int t = 0; t < kRegCol; ++t) {
                                    const int e = lane + 32 * t;
                                    xr[t] = e < L ? xcol[e] : 0.0;
                                }
                            }
                            for (int rl = 0; rl < nrl; ++rl) {
                                if (warp < np) {
                                    const int jq = (warp + rl) % M;
                                    if (jq < nq) {
                                        const int qa = np + jq;
                                        double* y = As + (int64_t)L * qa;
                                        double yr[kRegCol];
                                        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
                                        for (int t = 0; t < kRegCol; ++t) {
                                            const int e = lane + 32 * t;
                                            yr[t] = e < L ? y[e] : 0.0;
                                        }
#pragma unroll
                                        for (int t = 0; t < kRegCol; ++t) {
                                            al = fma(xr[t], xr[t], al);
                                            be = fma(yr[t], yr[t], be);
                                            ga = fma(xr[t], yr[t], ga);
                                        }
                                        al = warp_sum(al);
                                        be = warp_sum(be);
                                        ga = warp_sum(ga);
                                        double cs, sn;
                                        if (rotation(al, be, ga, tol, cs, sn)) {
#pragma unroll
                                            for (int t = 0; t < kRegCol; ++t) {
                                                const int e = lane + 32 * t;
                                                const double xv = xr[t], yv = yr[t];
                                                xr[t] = cs * xv - sn * yv;
                                                if (e < L) y[e] = sn * xv + cs * yv;
                                            }
                                            if (lane < nl) {
                                                const double xv = Qm[lane + ldq * warp], yv = Qm[lane + ldq * qa];
                                                Qm[lane + ldq * warp] = cs * xv - sn * yv;
                                                Qm[lane + ldq * qa] = sn * xv + cs * yv;
                                            }
                                            if (lane == 0) lrot = 1;
                                        }
                                    }
                                }
                                __syncthreads();
                            }
                            if (warp < np) {
#pragma unroll
                                for (int t = 0; t < kRegCol; ++t) {
                                    const int e = lane + 32 * t;
                                    if (e < L) xcol[e] = xr[t];
                                }
                            }
                            if (tid == 0 && lrot) lrot_any = 1;
                            __syncthreads();
                        } else
                        for (int ls = 0; ls < (full ? kLocalSweeps : 1); ++ls) {
                            if (tid == 0) lrot = 0;
                            __syncthreads();
                            for (int rl = 0; rl < nrl; ++rl) {
                                if (warp < (full ? S2 / 2 : np)) {
                                    int pa, qa;
                                    if (full) {
                                        pa = rr_player(warp, rl, S2);
                                        qa = rr_player(S2 - 1 - warp, rl, S2);
                                    } else {
                                        pa = warp;
                                        const int jq = (warp + rl) % M;
                                        qa = jq < nq ? np + jq : nl;   // nl: no partner this round
                                    }
                                    if (pa < nl && qa < nl) {
                                        double* x = As + (int64_t)L * pa;
                                        double* y = As + (int64_t)L * qa;
                                        double al = 0.0, be = 0.0, ga = 0.0;
                                        for (int e = lane; e < L; e += 32) {
                                            const double xv = x[e], yv = y[e];
                                            al = fma(xv, xv, al);
                                            be = fma(yv, yv, be);
                                            ga = fma(xv, yv, ga);
                                        }
                                        al = warp_sum(al);
                                        be = warp_sum(be);
                                        ga = warp_sum(ga);
                                        double cs, sn;
                                        if (rotation(al, be, ga, tol, cs, sn)) {
                                            for (int e = lane; e < L; e += 32) {
                                                const double xv = x[e], yv = y[e];
                                                x[e] = cs * xv - sn * yv;
                                                y[e] = sn * xv + cs * yv;
                                            }
                                            if (lane < nl) {
                                                const double xv = Qm[lane + ldq * pa], yv = Qm[lane + ldq * qa];
                                                Qm[lane + ldq * pa] = cs * xv - sn * yv;
                                                Qm[lane + ldq * qa] = sn * xv + cs * yv;
                                            }
                                            if (lane == 0) lrot = 1;
                                        }
                                    }
                                }
                                __syncthreads();
                            }
                            const int lr = lrot;
                            __syncthreads();   // every thread has read lrot before it is reset
                            if (!lr) break;
                            if (tid == 0) lrot_any = 1;
                        }
                        __syncthreads();
                        if (lrot_any) {   // uniform: write the pair back, V's columns times Q
                            for (int e = tid; e < nl * L; e += kBigThreads) {
                                const int j = e / L, i = e - j * L;
                                A[(int64_t)L * (j < np ? p0 + j : q0 + j - np) + i] = As[e];
                            }
                            for (int e = tid; e < s; e += kBigThreads) {
                                double vr[kMaxBlk2];
#pragma unroll
                                for (int j = 0; j < kMaxBlk2; ++j)
                                    vr[j] = j < nl ? V[e + (int64_t)s * (j < np ? p0 + j : q0 + j - np)] : 0.0;
#pragma unroll 4
                                for (int j = 0; j < nl; ++j) {
                                    double o = 0.0;
#pragma unroll
                                    for (int i = 0; i < kMaxBlk2; ++i) o = fma(vr[i], Qm[i + ldq * j], o);
                                    V[e + (int64_t)s * (j < np ? p0 + j : q0 + j - np)] = o;
                                }
                            }
                            if (tid == 0) rot_any = 1;
                        }
                        __syncthreads();   // shared memory is reused by the next block pair
                    }
                    if (r == nb - 2) {
                        __syncthreads();
                        if (tid == 0 && rot_any) atomicAdd(rot, 1);
                    }
                    group_barrier(cnt, target, C);
                }
                if (tid == 0) rot_now = (int)ld_acquire(rot);
                group_barrier(cnt, target, C);
                const int now = rot_now;
                if (now == rot_seen) break;
                rot_seen = now;
            }
        }
        for (int sweep = 0; sweep < kMaxSweeps && s > 1 && !block_mode; ++sweep) {
            if (tid == 0) rot_any = 0;
            __syncthreads();
            for (int r = 0; r < S - 1; ++r) {
                if (cta_pairs) {
                    for (int k = cg; k < S / 2; k += C) {
                        const int p = rr_player(k, r, S), q = rr_player(S - 1 - k, r, S);
                        if (p >= s || q >= s) continue;
                        double* ap = A + (int64_t)L * p;
                        double* aq = A + (int64_t)L * q;
                        double al = 0.0, be = 0.0, ga = 0.0;
                        for (int e = tid; e < L; e += kBigThreads) {
                            const double x = ap[e], y = aq[e];
                            al = fma(x, x, al);
                            be = fma(y, y, be);
                            ga = fma(x, y, ga);
                        }
                        al = warp_sum(al);
                        be = warp_sum(be);
                        ga = warp_sum(ga);
                        if (lane == 0) { red[0][warp] = al; red[1][warp] = be; red[2][warp] = ga; }
                        __syncthreads();
                        al = be = ga = 0.0;
                        for (int w = 0; w < kBigWarps; ++w) { al += red[0][w]; be += red[1][w]; ga += red[2][w]; }
                        __syncthreads();   // red is reused by the next pair
                        double cs, sn;
                        if (!rotation(al, be, ga, tol, cs, sn)) continue;   // uniform over the CTA
                        for (int e = tid; e < L; e += kBigThreads) {
                            const double x = ap[e], y = aq[e];
                            ap[e] = cs * x - sn * y;
                            aq[e] = sn * x + cs * y;
                        }
                        double* vp = V + (int64_t)s * p;
                        double* vq = V + (int64_t)s * q;
                        for (int e = tid; e < s; e += kBigThreads) {
                            const double x = vp[e], y = vq[e];
                            vp[e] = cs * x - sn * y;
                            vq[e] = sn * x + cs * y;
                        }
                        if (tid == 0) rot_any = 1;
                    }
                } else {
                    for (int k = gw; k < S / 2; k += gws) {
                        const int p = rr_player(k, r, S), q = rr_player(S - 1 - k, r, S);
                        if (p >= s || q >= s) continue;
                        double* ap = A + (int64_t)L * p;
                        double* aq = A + (int64_t)L * q;
                        double al = 0.0, be = 0.0, ga = 0.0;
                        double cs, sn;
                        if (L <= 32 * kRegCol) {   // both columns in registers: one load of each element
                            double xr[kRegCol], yr[kRegCol];
#pragma unroll
                            for (int t = 0; t < kRegCol; ++t) {
                                const int e = lane + 32 * t;
                                xr[t] = e < L ? ap[e] : 0.0;
                                yr[t] = e < L ? aq[e] : 0.0;
                            }
#pragma unroll
                            for (int t = 0; t < kRegCol; ++t) {
                                al = fma(xr[t], xr[t], al);
                                be = fma(yr[t], yr[t], be);
                                ga = fma(xr[t], yr[t], ga);
                            }
                            al = warp_sum(al);
                            be = warp_sum(be);
                            ga = warp_sum(ga);
                            if (!rotation(al, be, ga, tol, cs, sn)) continue;
#pragma unroll
                            for (int t = 0; t < kRegCol; ++t) {
                                const int e = lane + 32 * t;
                                if (e < L) {
                                    ap[e] = cs * xr[t] - sn * yr[t];
                                    aq[e] = sn * xr[t] + cs * yr[t];
                                }
                            }
                        } else {
                            for (int e = lane; e < L; e += 32) {
                                const double x = ap[e], y = aq[e];
                                al = fma(x, x, al);
                                be = fma(y, y, be);
                                ga = fma(x, y, ga);
                            }
                            al = warp_sum(al);
                            be = warp_sum(be);
                            ga = warp_sum(ga);
                            if (!rotation(al, be, ga, tol, cs, sn)) continue;
                            for (int e = lane; e < L; e += 32) {
                                const double x = ap[e], y = aq[e];
                                ap[e] = cs * x - sn * y;
                                aq[e] = sn * x + cs * y;
                            }
                        }
                        double* vp = V + (int64_t)s * p;
                        double* vq = V + (int64_t)s * q;
                        for (int e = lane; e < s; e += 32) {
                            const double x = vp[e], y = vq[e];
                            vp[e] = cs * x - sn * y;
                            vq[e] = sn * x + cs * y;
                        }
                        if (lane == 0) rot_any = 1;
                    }
                }
                if (r == S - 2) {   // count the CTAs that rotated this sweep (monotone counter)
                    __syncthreads();
                    if (tid == 0 && rot_any) atomicAdd(rot, 1);
                }
                group_barrier(cnt, target, C);
            }
            if (tid == 0) rot_now = (int)ld_acquire(rot);
            group_barrier(cnt, target, C);   // every CTA has read the count before the next sweep adds to it
            const int now = rot_now;
            if (now == rot_seen) break;      // a sweep without a rotation: converged
            rot_seen = now;
        }
        // ---- singular values (column norms) -> sig_g; every CTA then sorts them itself (same order everywhere)
        for (int j = gw; j < s; j += gws) {
            const double* aj = A + (int64_t)L * j;
            double v = 0.0;
            for (int e = lane; e < L; e += 32) v = fma(aj[e], aj[e], v);
            v = warp_sum(v);
            if (lane == 0) sig_g[j] = sqrt(v);
        }
        group_barrier(cnt, target, C);
        for (int j = tid; j < s; j += kBigThreads) sig[j] = sig_g[j];
        __syncthreads();
        for (int j = tid; j < s; j += kBigThreads) {
            int pos = 0;
            for (int k = 0; k < s; ++k) pos += (sig[k] > sig[j]) || (sig[k] == sig[j] && k < j);
            ord[pos] = j;
        }
        __syncthreads();
        // ---- delta-truncated rank (R23) with the singular-value floor (R25)
        if (tid == 0) {
            const double s0 = sig[ord[0]];
            int R = 1;
            if (s0 > 0.0) {
                int keep = 0;
                for (int k = 0; k < s; ++k) keep += sig[ord[k]] > kSigmaFloor * s0;
                // tail = sum_{j >= R} s_j^2 over every singular value (the below-floor ones included), shrinking R
                // while the discarded part stays within delta^2 (R23; oracle/ttsvd.py delta_rank)
                double tail = 0.0;
                for (int k = keep; k < s; ++k) tail += sig[ord[k]] * sig[ord[k]];
                R = keep;
                while (R > 1) {
                    const double sr = sig[ord[R - 1]];
                    if (tail + sr * sr > delta2) break;
                    tail += sr * sr;
                    --R;
                }
            }
            rank_s = R;
            if (cg == 0) rk[n + 1] = R;
        }
        __syncthreads();
        const int R = rank_s;
        // ---- core n = U (m x R) with the sign convention: column k is V[:, ord[k]] (wide) or A[:, ord[k]] / sigma
        for (int k = gw; k < R; k += gws) {
            const int j = ord[k];
            const double inv = wide ? 1.0 : (sig[j] > 0.0 ? 1.0 / sig[j] : 0.0);
            const double* u = wide ? V + (int64_t)s * j : A + (int64_t)L * j;
            double best = -1.0;
            int bi = 0;
            for (int e = lane; e < m; e += 32) {
                const double v = fabs(u[e]);
                if (v > best) { best = v; bi = e; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            const double sg = u[bi] < 0.0 ? -1.0 : 1.0;
            if (lane == 0) sgn_g[k] = sg;
            for (int e = lane; e < m; e += 32) core[coff + e + (int64_t)m * k] = (float)(sg * inv * u[e]);
        }
        group_barrier(cnt, target, C);
        // ---- next unfolding Z' = S V^T (R x c, column-major), reshaped to (R I_{n+1}) x rest by the index order
        for (int64_t e = gt; e < (int64_t)R * c; e += gts) {
            const int k = (int)(e % R), col = (int)(e / R);
            const int j = ord[k];
            Z[e] = wide ? sgn_g[k] * A[col + (int64_t)L * j] : sgn_g[k] * sig[j] * V[col + (int64_t)s * j];
        }
        group_barrier(cnt, target, C);
        coff += (int64_t)m * R;
        Rp = R;
        cur = (int64_t)R * c;
    }
    // ---- last core: G^(N) = Z (R_{N-1} x I_N x 1)
    for (int64_t e = gt; e < cur; e += gts) core[coff + e] = (float)Z[e];
}

}  // namespace

int64_t ttsvd_big_ws_bytes(int32_t B, int32_t elems, int32_t gmax) {
    // per tensor: Z, A (elems doubles each), V (gmax^2), sig and signs (gmax each), group partials; plus the
    // per-tensor synchronisation ints (zeroed by every launch)
    const int64_t per = 2 * (int64_t)elems + (int64_t)gmax * gmax + 2 * (int64_t)gmax + kMaxGroup + 16;
    return 8 * (int64_t)B * per + 4 * (int64_t)B * kSyncInts;
}

cudaError_t launch_ttsvd_big(const TtsvdArgs& a, void* workspace, cudaStream_t s) {
    if (a.B <= 0) return cudaSuccess;
    const int64_t per = 2 * (int64_t)a.elems + (int64_t)a.gmax * a.gmax + 2 * (int64_t)a.gmax + kMaxGroup + 16;
    double* ws = static_cast<double*>(workspace);
    int* sync = reinterpret_cast<int*>(ws + (int64_t)a.B * per);
    cudaError_t e = cudaMemsetAsync(sync, 0, 4 * (size_t)a.B * kSyncInts, s);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, occ = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(ttsvd_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynBytes)) !=
        cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ttsvd_big_kernel, kBigThreads, kDynBytes)) !=
        cudaSuccess)
        return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int slots = sms * occ;
    // CTAs per tensor: as many as the co-resident slots allow for the whole batch (at most kMaxGroup); batches
    // larger than the slots run in chunks of whole groups
    const int C = std::max(1, std::min(kMaxGroup, slots / a.B));
    const int per_launch = std::max(1, slots / C);
    for (int b0 = 0; b0 < a.B; b0 += per_launch) {
        const int groups = std::min(per_launch, a.B - b0);
        TtsvdArgs aa = a;
        int64_t wp = per;
        int Cc = C, bb = b0, dd = kDynBytes / 8;
        void* args[] = {&aa, &ws, &sync, &wp, &Cc, &bb, &dd};
        e = cudaLaunchCooperativeKernel((const void*)ttsvd_big_kernel, dim3(groups * C), dim3(kBigThreads), args,
                                        kDynBytes, s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace ttc
