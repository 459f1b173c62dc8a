/*
 * ttc_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the TT contraction hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or helper with
 * paper_2109_00626_b200/ (the CUDA product) and neither side includes the other.
 *
 * Everything is fp64, plain loops in a fixed order, no BLAS, no blocking, no fusion.  Cores follow
 * the paper's little-endian convention (Def. 2 / Eq. 2: first index fastest):
 *   core n is R_{n-1} x I_n x R_n, element [r,i,s] at r + R_{n-1}*(i + I_n*s)   (Def. 7 / Eq. 9).
 *
 * Functions and the passage each follows:
 *   oracle_tt_reconstruct   O1a  Eq. 9 left to right, reading "x_3^1" as "contract
 *                                the running product's trailing rank mode with the next core's leading
 *                                rank mode" (reading R4).
 *   oracle_tcp              O1b  Eq. 8 applied to K disjoint mode pairs; output modes
 *                                in Eq. 8 order (X free ascending, then Y free ascending).  K = N = M is
 *                                the "contraction along all modes" of Fig. 1b.
 *   oracle_tt_inner         O2   full contraction of two TTs core by core: Z_0 = [1],
 *                                W[r,i,q] = sum_p Z[r,p] Y_n[p,i,q];  Z_n[s,q] = sum_{r,i} X_n[r,i,s] W[r,i,q];
 *                                result Z_N (1x1).  Z_1 = A_x^T A_y is Eq. 12.
 *   oracle_tt_inner_transfer O2' same value by explicit transfer matrices
 *                                E_n[(r + R p), (s + R' q)] = sum_i X_n[r,i,s] Y_n[p,i,q];  v <- v E_n.
 *   oracle_tt_contract      O3   partial contraction over K disjoint, non-crossing mode pairs returned as a
 *                                TT (Alg. 2 steps 4-6, generalised by the Kronecker
 *                                "ladder" of SURVEY.md Appendix A; readings R7-R10).  Free cores
 *                                are materialised as dense Kronecker products with identities, transfers
 *                                T_k as dense matrices, and absorbed by plain matrix products.
 *   oracle_tt_splice        O5   single-mode contraction of END modes (n in {1, N}, m in {1, M}) as the paper's
 *                                own TTCP splice (Alg. 2 steps 4-5, Example 1 PAPER.md:313-322):
 *                                K = A_x^T A_y (Eq. 12), then the X cores (reversed with rank modes swapped when
 *                                n = 1), K, then the Y cores (reversed when m = M); K absorbed into the next core
 *                                (readings R6, R10).  Ranks stay R and P (no Kronecker bonds).
 *   oracle_tt_inner_batch / oracle_tt_contract_batch: loops of the above over a batch of pairs
 *                                (OpenMP over pairs) -- the CPU baseline bench.py times.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_ARG 1
#define OR_ERR_SHAPE 2
#define OR_ERR_MODES 3
#define OR_ERR_NOMEM 4

/* ---------------------------------------------------------------- O1a: Eq. 9 dense reconstruction */
int oracle_tt_reconstruct(int N, const int32_t* dims, const int32_t* ranks, const double* cores, double* out)
{
    if (N < 1 || ranks[0] != 1 || ranks[N] != 1) return OR_ERR_ARG;
    /* T holds the running product as a (I_1...I_n) x R_n matrix, rows little-endian */
    int64_t A = 1, maxsz = 1;
    for (int n = 0; n < N; ++n) {
        A *= dims[n];
        if (A * ranks[n + 1] > maxsz) maxsz = A * ranks[n + 1];
    }
    double* T = (double*)malloc(sizeof(double) * maxsz);
    double* U = (double*)malloc(sizeof(double) * maxsz);
    if (!T || !U) { free(T); free(U); return OR_ERR_NOMEM; }
    T[0] = 1.0;                       /* 1 x R_0 = 1 x 1 */
    A = 1;
    const double* core = cores;
    for (int n = 0; n < N; ++n) {
        const int64_t R = ranks[n], I = dims[n], S = ranks[n + 1];
        /* U[a + A*i, s] = sum_r T[a, r] * G[r, i, s] */
        for (int64_t s = 0; s < S; ++s)
            for (int64_t i = 0; i < I; ++i)
                for (int64_t a = 0; a < A; ++a) {
                    double acc = 0.0;
                    for (int64_t r = 0; r < R; ++r)
                        acc += T[a + A * r] * core[r + R * (i + I * s)];
                    U[(a + A * i) + (A * I) * s] = acc;
                }
        core += R * I * S;
        A *= I;
        double* t = T; T = U; U = t;
    }
    memcpy(out, T, sizeof(double) * A);   /* R_N = 1: the dense tensor in Eq. 2 order */
    free(T); free(U);
    return OR_OK;
}

/* ---------------------------------------------------------------- O1b: Eq. 8 dense TCP over K pairs */
/* x_modes / y_modes are 1-based (SPEC.md:158 convention), pairwise disjoint within each operand.
 * z == NULL: count only (the loops run, nothing is read or written). *macs accumulates x*y products. */
int oracle_tcp(int N, const int32_t* xdims, const double* x, int M, const int32_t* ydims, const double* y,
               int K, const int32_t* x_modes, const int32_t* y_modes, double* z, int64_t* macs)
{
    if (N < 1 || M < 1 || K < 0 || K > N || K > M) return OR_ERR_ARG;
    int xc[64] = {0}, yc[64] = {0};          /* contracted flags */
    if (N > 64 || M > 64) return OR_ERR_ARG;
    for (int k = 0; k < K; ++k) {
        int n = x_modes[k] - 1, m = y_modes[k] - 1;
        if (n < 0 || n >= N || m < 0 || m >= M || xc[n] || yc[m]) return OR_ERR_MODES;
        if (xdims[n] != ydims[m]) return OR_ERR_SHAPE;
        xc[n] = k + 1; yc[m] = k + 1;
    }
    /* free-mode lists in Eq. 8 order */
    int fx[64], fy[64], nfx = 0, nfy = 0;
    for (int n = 0; n < N; ++n) if (!xc[n]) fx[nfx++] = n;
    for (int m = 0; m < M; ++m) if (!yc[m]) fy[nfy++] = m;
    int64_t xstr[64], ystr[64];
    xstr[0] = 1; for (int n = 1; n < N; ++n) xstr[n] = xstr[n - 1] * xdims[n - 1];   /* Eq. 2 */
    ystr[0] = 1; for (int m = 1; m < M; ++m) ystr[m] = ystr[m - 1] * ydims[m - 1];
    int64_t nout = 1, ncon = 1;
    for (int a = 0; a < nfx; ++a) nout *= xdims[fx[a]];
    for (int a = 0; a < nfy; ++a) nout *= ydims[fy[a]];
    for (int k = 0; k < K; ++k) ncon *= xdims[x_modes[k] - 1];
    int io[128], ic[64];
    int64_t cnt = 0;
    for (int64_t o = 0; o < nout; ++o) {
        /* multi-index of output position o, first free mode fastest (Eq. 2 applied to Z's shape) */
        int64_t rem = o;
        for (int a = 0; a < nfx; ++a) { io[a] = (int)(rem % xdims[fx[a]]); rem /= xdims[fx[a]]; }
        for (int a = 0; a < nfy; ++a) { io[nfx + a] = (int)(rem % ydims[fy[a]]); rem /= ydims[fy[a]]; }
        int64_t xbase = 0, ybase = 0;
        for (int a = 0; a < nfx; ++a) xbase += io[a] * xstr[fx[a]];
        for (int a = 0; a < nfy; ++a) ybase += io[nfx + a] * ystr[fy[a]];
        double acc = 0.0;
        for (int64_t c = 0; c < ncon; ++c) {
            int64_t r2 = c;
            for (int k = 0; k < K; ++k) { int d = xdims[x_modes[k] - 1]; ic[k] = (int)(r2 % d); r2 /= d; }
            int64_t xi = xbase, yi = ybase;
            for (int k = 0; k < K; ++k) {
                xi += ic[k] * xstr[x_modes[k] - 1];
                yi += ic[k] * ystr[y_modes[k] - 1];
            }
            if (z) acc += x[xi] * y[yi];
            ++cnt;
        }
        if (z) z[o] = acc;
    }
    if (macs) *macs += cnt;
    return OR_OK;
}

/* ---------------------------------------------------------------- O2: the TT sweep */
/* Also returns, if zout != NULL and stop_after in [1,N], the R_n x P_n matrix Z after `stop_after` steps
 * (column-major, Z[r + R_n p]).  Returns <X,Y> (Z_N) when stop_after == N. */
static double sweep(int N, const int32_t* dims, const int32_t* xr, const double* xc, const int32_t* yr,
                    const double* yc, int stop_after, double* zout, int64_t* macs, int* err)
{
    *err = OR_OK;
    if (N < 1 || xr[0] != 1 || xr[N] != 1 || yr[0] != 1 || yr[N] != 1) { *err = OR_ERR_ARG; return 0.0; }
    int64_t maxz = 1, maxw = 1;
    for (int n = 0; n <= N; ++n) if ((int64_t)xr[n] * yr[n] > maxz) maxz = (int64_t)xr[n] * yr[n];
    for (int n = 0; n < N; ++n) {
        int64_t w = (int64_t)xr[n] * dims[n] * yr[n + 1];
        if (w > maxw) maxw = w;
    }
    double* Z = (double*)malloc(sizeof(double) * maxz);
    double* Zn = (double*)malloc(sizeof(double) * maxz);
    double* W = (double*)malloc(sizeof(double) * maxw);
    if (!Z || !Zn || !W) { free(Z); free(Zn); free(W); *err = OR_ERR_NOMEM; return 0.0; }
    Z[0] = 1.0;
    int64_t cnt = 0;
    const double* X = xc; const double* Y = yc;
    for (int n = 0; n < N; ++n) {
        const int64_t R = xr[n], S = xr[n + 1], P = yr[n], Q = yr[n + 1], I = dims[n];
        /* W[r, i, q] = sum_p Z[r, p] Y[p, i, q] */
        for (int64_t q = 0; q < Q; ++q)
            for (int64_t i = 0; i < I; ++i)
                for (int64_t r = 0; r < R; ++r) {
                    double acc = 0.0;
                    for (int64_t p = 0; p < P; ++p) acc += Z[r + R * p] * Y[p + P * (i + I * q)];
                    W[r + R * (i + I * q)] = acc;
                }
        cnt += R * P * I * Q;
        /* Z'[s, q] = sum_{r, i} X[r, i, s] W[r, i, q] */
        for (int64_t q = 0; q < Q; ++q)
            for (int64_t s = 0; s < S; ++s) {
                double acc = 0.0;
                for (int64_t i = 0; i < I; ++i)
                    for (int64_t r = 0; r < R; ++r) acc += X[r + R * (i + I * s)] * W[r + R * (i + I * q)];
                Zn[s + S * q] = acc;
            }
        cnt += R * I * S * Q;
        double* t = Z; Z = Zn; Zn = t;
        X += R * I * S; Y += P * I * Q;
        if (zout && stop_after == n + 1) memcpy(zout, Z, sizeof(double) * S * Q);
    }
    double v = Z[0];
    free(Z); free(Zn); free(W);
    if (macs) *macs += cnt;
    return v;
}

int oracle_tt_inner(int N, const int32_t* dims, const int32_t* xr, const double* xc, const int32_t* yr,
                    const double* yc, double* result, int64_t* macs)
{
    int err;
    *result = sweep(N, dims, xr, xc, yr, yc, N, NULL, macs, &err);
    return err;
}

int oracle_tt_inner_partial(int N, const int32_t* dims, const int32_t* xr, const double* xc, const int32_t* yr,
                            const double* yc, int steps, double* zout)
{
    int err;
    if (steps < 1 || steps > N) return OR_ERR_ARG;
    sweep(N, dims, xr, xc, yr, yc, steps, zout, NULL, &err);
    return err;
}

/* ---------------------------------------------------------------- O2': explicit transfer matrices */
int oracle_tt_inner_transfer(int N, const int32_t* dims, const int32_t* xr, const double* xc, const int32_t* yr,
                             const double* yc, double* result)
{
    if (N < 1 || xr[0] != 1 || xr[N] != 1 || yr[0] != 1 || yr[N] != 1) return OR_ERR_ARG;
    int64_t maxv = 1;
    for (int n = 0; n <= N; ++n) if ((int64_t)xr[n] * yr[n] > maxv) maxv = (int64_t)xr[n] * yr[n];
    double* v = (double*)calloc(maxv, sizeof(double));
    double* vn = (double*)calloc(maxv, sizeof(double));
    if (!v || !vn) { free(v); free(vn); return OR_ERR_NOMEM; }
    v[0] = 1.0;
    const double* X = xc; const double* Y = yc;
    for (int n = 0; n < N; ++n) {
        const int64_t R = xr[n], S = xr[n + 1], P = yr[n], Q = yr[n + 1], I = dims[n];
        const int64_t rows = R * P, cols = S * Q;
        double* E = (double*)malloc(sizeof(double) * rows * cols);
        if (!E) { free(v); free(vn); return OR_ERR_NOMEM; }
        for (int64_t q = 0; q < Q; ++q)
            for (int64_t s = 0; s < S; ++s)
                for (int64_t p = 0; p < P; ++p)
                    for (int64_t r = 0; r < R; ++r) {
                        double acc = 0.0;
                        for (int64_t i = 0; i < I; ++i) acc += X[r + R * (i + I * s)] * Y[p + P * (i + I * q)];
                        E[(r + R * p) + rows * (s + S * q)] = acc;
                    }
        for (int64_t c = 0; c < cols; ++c) {
            double acc = 0.0;
            for (int64_t a = 0; a < rows; ++a) acc += v[a] * E[a + rows * c];
            vn[c] = acc;
        }
        free(E);
        double* t = v; v = vn; vn = t;
        X += R * I * S; Y += P * I * Q;
    }
    *result = v[0];
    free(v); free(vn);
    return OR_OK;
}

/* ---------------------------------------------------------------- O3: the ladder tt_contract */
/* Sequence element kinds */
#define EL_XFREE 1
#define EL_YFREE 2
#define EL_T 3

typedef struct { int kind, mode, hold; } el_t;   /* mode: 0-based source mode (X for XFREE/T, Y for YFREE);
                                                    hold: 0-based bond index of the carried operand,
                                                    for T: the Y mode (0-based) */

/* Builds the ladder sequence S.  Returns number of elements or -1 on error. */
static int ladder(int N, int M, int K, const int32_t* xm, const int32_t* ym, el_t* S)
{
    int ns = 0;
    for (int k = 1; k <= K + 1; ++k) {
        const int nprev = (k == 1) ? 0 : xm[k - 2], mprev = (k == 1) ? 0 : ym[k - 2];
        const int ncur = (k <= K) ? xm[k - 1] : N + 1, mcur = (k <= K) ? ym[k - 1] : M + 1;
        for (int n = nprev + 1; n <= ncur - 1; ++n) { S[ns].kind = EL_XFREE; S[ns].mode = n - 1; S[ns].hold = mprev; ++ns; }
        for (int m = mprev + 1; m <= mcur - 1; ++m) { S[ns].kind = EL_YFREE; S[ns].mode = m - 1; S[ns].hold = ncur - 1; ++ns; }
        if (k <= K) { S[ns].kind = EL_T; S[ns].mode = ncur - 1; S[ns].hold = mcur - 1; ++ns; }
    }
    return ns;
}

/* dense C = A (m x k) * B (k x n), column-major */
static void matmul(int64_t m, int64_t k, int64_t n, const double* A, const double* B, double* C, int64_t* macs)
{
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            double acc = 0.0;
            for (int64_t l = 0; l < k; ++l) acc += A[i + m * l] * B[l + k * j];
            C[i + m * j] = acc;
        }
    if (macs) *macs += m * k * n;
}

/* Metadata + cores of X x_{pairs} Y as a TT.
 *   out_order    : L = N + M - 2K
 *   out_dims[L], out_ranks[L+1], out_src[L] (+n: X mode n, -m: Y mode m, 1-based),
 *   out_perm[L]  : 1-based ladder position of canonical (Eq. 8 order) output mode c
 *   out_elems    : total elements of the output cores
 *   out_cores    : if non-NULL, the cores (concatenated, Eq. 2 order); L == 0 -> one scalar.
 *   t_macs / a_macs: MACs spent forming transfers (the paper's K step) / absorbing them (dense, not
 *                    structure-aware), may be NULL. */
int oracle_tt_contract(int N, const int32_t* xdims, const int32_t* xr, const double* xc,
                       int M, const int32_t* ydims, const int32_t* yr, const double* yc,
                       int K, const int32_t* xm, const int32_t* ym,
                       int32_t* out_order, int32_t* out_dims, int32_t* out_ranks, int32_t* out_src,
                       int32_t* out_perm, int64_t* out_elems, double* out_cores, int64_t* t_macs, int64_t* a_macs)
{
    if (N < 1 || M < 1 || K < 0 || K > N || K > M || N > 256 || M > 256) return OR_ERR_ARG;
    if (xr[0] != 1 || xr[N] != 1 || yr[0] != 1 || yr[M] != 1) return OR_ERR_ARG;
    for (int k = 0; k < K; ++k) {
        if (xm[k] < 1 || xm[k] > N || ym[k] < 1 || ym[k] > M) return OR_ERR_MODES;
        if (k > 0 && (xm[k] <= xm[k - 1] || ym[k] <= ym[k - 1])) return OR_ERR_MODES;
        if (xdims[xm[k] - 1] != ydims[ym[k] - 1]) return OR_ERR_SHAPE;
    }
    el_t S[600];
    const int ns = ladder(N, M, K, xm, ym, S);
    /* core offsets of the inputs */
    int64_t xoff[257], yoff[257];
    xoff[0] = 0; for (int n = 0; n < N; ++n) xoff[n + 1] = xoff[n] + (int64_t)xr[n] * xdims[n] * xr[n + 1];
    yoff[0] = 0; for (int m = 0; m < M; ++m) yoff[m + 1] = yoff[m] + (int64_t)yr[m] * ydims[m] * yr[m + 1];

    /* metadata: cores of S in order, ranks from the bonds they connect */
    const int L = N + M - 2 * K;
    *out_order = L;
    int l = 0;
    out_ranks[0] = 1;
    for (int e = 0; e < ns; ++e) {
        if (S[e].kind == EL_XFREE) {
            const int n = S[e].mode, b = S[e].hold;     /* Y bond P_b carried */
            out_dims[l] = xdims[n];
            out_src[l] = n + 1;
            out_ranks[l + 1] = xr[n + 1] * yr[b];
            ++l;
        } else if (S[e].kind == EL_YFREE) {
            const int m = S[e].mode, a = S[e].hold;     /* X bond R_a carried */
            out_dims[l] = ydims[m];
            out_src[l] = -(m + 1);
            out_ranks[l + 1] = xr[a] * yr[m + 1];
            ++l;
        }
    }
    out_ranks[L] = 1;   /* the last bond is (R_N, P_M) = (1, 1); a trailing transfer is absorbed from the right */
    /* canonical order: X free ascending then Y free ascending (Eq. 8) */
    {
        int c = 0;
        for (int n = 1; n <= N; ++n)
            for (int p = 0; p < L; ++p) if (out_src[p] == n) out_perm[c++] = p + 1;
        for (int m = 1; m <= M; ++m)
            for (int p = 0; p < L; ++p) if (out_src[p] == -m) out_perm[c++] = p + 1;
    }
    int64_t total = 0;
    for (int p = 0; p < L; ++p) total += (int64_t)out_ranks[p] * out_dims[p] * out_ranks[p + 1];
    *out_elems = (L == 0) ? 1 : total;
    if (!out_cores) return OR_OK;

    /* numeric part: dense Kronecker cores, dense transfers, plain matmul absorption */
    double* pend = NULL;           /* pending product of consecutive transfers, rows x cols */
    int64_t prow = 0, pcol = 0;
    double* prev_core = NULL;      /* last emitted core (for absorption from the right at the end) */
    int64_t prev_a = 0, prev_i = 0, prev_b = 0;
    double* outp = out_cores;
    l = 0;
    for (int e = 0; e < ns; ++e) {
        if (S[e].kind == EL_T) {
            const int n = S[e].mode, m = S[e].hold;
            const int64_t R = xr[n], Rn = xr[n + 1], P = yr[m], Pn = yr[m + 1], I = xdims[n];
            const int64_t rows = R * P, cols = Rn * Pn;
            double* T = (double*)malloc(sizeof(double) * rows * cols);
            const double* X = xc + xoff[n]; const double* Y = yc + yoff[m];
            for (int64_t pp = 0; pp < Pn; ++pp)
                for (int64_t rr = 0; rr < Rn; ++rr)
                    for (int64_t p = 0; p < P; ++p)
                        for (int64_t r = 0; r < R; ++r) {
                            double acc = 0.0;
                            for (int64_t i = 0; i < I; ++i) acc += X[r + R * (i + I * rr)] * Y[p + P * (i + I * pp)];
                            T[(r + R * p) + rows * (rr + Rn * pp)] = acc;
                        }
            if (t_macs) *t_macs += rows * cols * I;
            if (!pend) { pend = T; prow = rows; pcol = cols; }
            else {
                double* Pm = (double*)malloc(sizeof(double) * prow * cols);
                matmul(prow, pcol, cols, pend, T, Pm, a_macs);
                free(pend); free(T);
                pend = Pm; pcol = cols;
            }
            continue;
        }
        /* a free core: dense Kronecker expansion */
        int64_t A, I, Bc;
        double* C;
        if (S[e].kind == EL_XFREE) {
            const int n = S[e].mode; const int64_t R = xr[n], Rn = xr[n + 1], Pb = yr[S[e].hold];
            I = xdims[n]; A = R * Pb; Bc = Rn * Pb;
            C = (double*)calloc(A * I * Bc, sizeof(double));
            const double* X = xc + xoff[n];
            for (int64_t p = 0; p < Pb; ++p)            /* [r + R p, i, r' + Rn p] = X[r,i,r'] */
                for (int64_t rr = 0; rr < Rn; ++rr)
                    for (int64_t i = 0; i < I; ++i)
                        for (int64_t r = 0; r < R; ++r)
                            C[(r + R * p) + A * (i + I * (rr + Rn * p))] = X[r + R * (i + I * rr)];
        } else {
            const int m = S[e].mode; const int64_t P = yr[m], Pn = yr[m + 1], Ra = xr[S[e].hold];
            I = ydims[m]; A = Ra * P; Bc = Ra * Pn;
            C = (double*)calloc(A * I * Bc, sizeof(double));
            const double* Y = yc + yoff[m];
            for (int64_t pp = 0; pp < Pn; ++pp)         /* [r + Ra p, j, r + Ra p'] = Y[p,j,p'] */
                for (int64_t j = 0; j < I; ++j)
                    for (int64_t p = 0; p < P; ++p)
                        for (int64_t r = 0; r < Ra; ++r)
                            C[(r + Ra * p) + A * (j + I * (r + Ra * pp))] = Y[p + P * (j + I * pp)];
        }
        if (pend) {   /* absorb the pending transfer product from the left: C'[a,i,b] = sum_g T[a,g] C[g,i,b] */
            double* Cn = (double*)malloc(sizeof(double) * prow * I * Bc);
            matmul(prow, A, I * Bc, pend, C, Cn, a_macs);
            free(C); free(pend); pend = NULL;
            C = Cn; A = prow;
        }
        /* flush the previous core, keep this one (it may receive a right absorption) */
        if (prev_core) {
            memcpy(outp, prev_core, sizeof(double) * prev_a * prev_i * prev_b);
            outp += prev_a * prev_i * prev_b;
            free(prev_core);
        }
        prev_core = C; prev_a = A; prev_i = I; prev_b = Bc;
        ++l;
    }
    if (pend) {
        if (prev_core) {   /* no core follows: absorb from the right, C'[a,i,b] = sum_g C[a,i,g] T[g,b] */
            double* Cn = (double*)malloc(sizeof(double) * prev_a * prev_i * pcol);
            matmul(prev_a * prev_i, prev_b, pcol, prev_core, pend, Cn, a_macs);
            free(prev_core);
            prev_core = Cn; prev_b = pcol;
        } else {           /* no cores at all: the result is the 1x1 product (= tt_inner) */
            out_cores[0] = pend[0];
        }
        free(pend);
    }
    if (prev_core) {
        memcpy(outp, prev_core, sizeof(double) * prev_a * prev_i * prev_b);
        free(prev_core);
    }
    return OR_OK;
}

/* ---------------------------------------------------------------- O5: TTCP splice of end modes */
/* Z = X x_n^m Y for n in {1, N}, m in {1, M} (1-based), as a TT in the order of Alg. 2 step 5
 * (PAPER.md:363-374): the X free cores -- reversed, N..2, each core transposed in its rank modes, when n = 1
 * (the B_x x_2^1 G_x^(N-1) ... G_x^(2) chain of step 5); in order 1..N-1 when n = N -- then
 * K = A_x^T A_y (step 4, Eq. 12), then the Y free cores (2..M when m = 1; reversed M-1..1, transposed, when
 * m = M).  A_x is the contracted X core read as I x R (its one non-unit bond), A_y likewise.  K is absorbed
 * into the next core of the chain by a plain matrix product (reading R10), else into the previous one; with no
 * free core at all the result is the scalar K.  Same outputs as oracle_tt_contract (src, perm: canonical Eq. 8
 * order, X free ascending then Y free ascending). */
int oracle_tt_splice(int N, const int32_t* xdims, const int32_t* xr, const double* xc,
                     int M, const int32_t* ydims, const int32_t* yr, const double* yc, int n, int m,
                     int32_t* out_order, int32_t* out_dims, int32_t* out_ranks, int32_t* out_src,
                     int32_t* out_perm, int64_t* out_elems, double* out_cores)
{
    if (N < 1 || M < 1 || N > 256 || M > 256) return OR_ERR_ARG;
    if (xr[0] != 1 || xr[N] != 1 || yr[0] != 1 || yr[M] != 1) return OR_ERR_ARG;
    if ((n != 1 && n != N) || (m != 1 && m != M)) return OR_ERR_MODES;
    if (xdims[n - 1] != ydims[m - 1]) return OR_ERR_SHAPE;
    int64_t xoff[257], yoff[257];
    xoff[0] = 0; for (int k = 0; k < N; ++k) xoff[k + 1] = xoff[k] + (int64_t)xr[k] * xdims[k] * xr[k + 1];
    yoff[0] = 0; for (int k = 0; k < M; ++k) yoff[k + 1] = yoff[k] + (int64_t)yr[k] * ydims[k] * yr[k + 1];
    /* the chain of free cores: source (+x / -y, 0-based mode), reversed? */
    int src[512], rev[512], L = 0;
    if (n == 1) for (int k = N - 1; k >= 1; --k) { src[L] = k + 1; rev[L] = 1; ++L; }
    else        for (int k = 0; k < N - 1; ++k) { src[L] = k + 1; rev[L] = 0; ++L; }
    const int nx = L;   /* K sits between chain positions nx - 1 and nx */
    if (m == 1) for (int k = 1; k < M; ++k) { src[L] = -(k + 1); rev[L] = 0; ++L; }
    else        for (int k = M - 2; k >= 0; --k) { src[L] = -(k + 1); rev[L] = 1; ++L; }
    /* K = A_x^T A_y: A_x[i, r] is X_1[0, i, r] (n = 1) or X_N[r, i, 0] (n = N) */
    const int I = xdims[n - 1];
    const int Rk = (n == 1) ? xr[1] : xr[N - 1], Pk = (m == 1) ? yr[1] : yr[M - 1];
    const double* Ax = xc + xoff[n - 1];
    const double* Ay = yc + yoff[m - 1];
    double* Km = (double*)malloc(sizeof(double) * Rk * Pk);   /* Km[r + Rk p] */
    for (int p = 0; p < Pk; ++p)
        for (int r = 0; r < Rk; ++r) {
            double acc = 0.0;
            for (int i = 0; i < I; ++i) {
                const double a = (n == 1) ? Ax[i + I * r] : Ax[r + Rk * i];
                const double b = (m == 1) ? Ay[i + I * p] : Ay[p + Pk * i];
                acc += a * b;
            }
            Km[r + Rk * p] = acc;
        }
    /* metadata */
    *out_order = L;
    out_ranks[0] = 1;
    for (int l = 0; l < L; ++l) {
        const int s = src[l] > 0 ? src[l] - 1 : -src[l] - 1;
        const int32_t* rr = src[l] > 0 ? xr : yr;
        out_dims[l] = src[l] > 0 ? xdims[s] : ydims[s];
        out_src[l] = src[l];
        out_ranks[l + 1] = rev[l] ? rr[s] : rr[s + 1];
    }
    if (L > 0) {
        /* the bond at K: the left core's right rank is Rk, the right core's left rank Pk; K's rows (cols) replace
           it on the side it is absorbed into */
        if (nx < L) out_ranks[nx] = (nx == 0) ? 1 : Rk;   /* absorbed into chain core nx: its left bond becomes Rk */
        out_ranks[L] = 1;
    }
    {
        int c = 0;
        for (int k = 1; k <= N; ++k) for (int q = 0; q < L; ++q) if (out_src[q] == k) out_perm[c++] = q + 1;
        for (int k = 1; k <= M; ++k) for (int q = 0; q < L; ++q) if (out_src[q] == -k) out_perm[c++] = q + 1;
    }
    int64_t total = 0;
    for (int l = 0; l < L; ++l) total += (int64_t)out_ranks[l] * out_dims[l] * out_ranks[l + 1];
    *out_elems = (L == 0) ? 1 : total;
    if (!out_cores) { free(Km); return OR_OK; }
    if (L == 0) { out_cores[0] = Km[0]; free(Km); return OR_OK; }
    /* numeric: each chain core as a dense (A x I x B) array, K absorbed by a plain matrix product */
    double* outp = out_cores;
    for (int l = 0; l < L; ++l) {
        const int s = src[l] > 0 ? src[l] - 1 : -src[l] - 1;
        const int32_t* rr = src[l] > 0 ? xr : yr;
        const double* G = (src[l] > 0 ? xc + xoff[s] : yc + yoff[s]);
        const int64_t a0 = rr[s], Id = src[l] > 0 ? xdims[s] : ydims[s], b0 = rr[s + 1];
        const int64_t A = rev[l] ? b0 : a0, B = rev[l] ? a0 : b0;
        double* C = (double*)malloc(sizeof(double) * A * Id * B);   /* C[u, i, v] at u + A (i + Id v) */
        for (int64_t v = 0; v < B; ++v)
            for (int64_t i = 0; i < Id; ++i)
                for (int64_t u = 0; u < A; ++u)
                    C[u + A * (i + Id * v)] = rev[l] ? G[v + a0 * (i + Id * u)] : G[u + a0 * (i + Id * v)];
        if (l == nx) {               /* left absorption: C'[r, i, v] = sum_p K[r, p] C[p, i, v] */
            double* Cn = (double*)malloc(sizeof(double) * Rk * Id * B);
            matmul(Rk, A, Id * B, Km, C, Cn, NULL);
            free(C); C = Cn;
            memcpy(outp, C, sizeof(double) * Rk * Id * B);
            outp += Rk * Id * B;
        } else if (l == L - 1 && nx == L) {   /* no core after K: right absorption C'[u, i, p] = sum_r C[u, i, r] K[r, p] */
            double* Cn = (double*)malloc(sizeof(double) * A * Id * Pk);
            matmul(A * Id, B, Pk, C, Km, Cn, NULL);
            memcpy(outp, Cn, sizeof(double) * A * Id * Pk);
            outp += A * Id * Pk;
            free(Cn);
        } else {
            memcpy(outp, C, sizeof(double) * A * Id * B);
            outp += A * Id * B;
        }
        free(C);
    }
    free(Km);
    return OR_OK;
}

/* ---------------------------------------------------------------- batches (CPU baseline) */
/* Trains of fp32 values (the product's storage) are widened exactly to fp64 before the sweep. */
static double* widen(const float* src, int64_t n)
{
    double* d = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    for (int64_t k = 0; k < n; ++k) d[k] = (double)src[k];
    return d;
}

int oracle_tt_inner_batch(int B, int N, const int32_t* dims,
                          const int32_t* xranks, const int64_t* xoff, const float* xcores,
                          const int32_t* yranks, const int64_t* yoff, const float* ycores,
                          double* out, int nthreads)
{
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
#endif
    for (int b = 0; b < B; ++b) {
        const int32_t* xr = xranks + (int64_t)b * (N + 1);
        const int32_t* yr = yranks + (int64_t)b * (N + 1);
        int64_t nx = 0, ny = 0;
        for (int n = 0; n < N; ++n) { nx += (int64_t)xr[n] * dims[n] * xr[n + 1]; ny += (int64_t)yr[n] * dims[n] * yr[n + 1]; }
        double* X = widen(xcores + xoff[b], nx);
        double* Y = widen(ycores + yoff[b], ny);
        double v = 0.0;
        if (oracle_tt_inner(N, dims, xr, X, yr, Y, &v, NULL) != OR_OK) bad |= 1;
        out[b] = v;
        free(X); free(Y);
    }
    return bad ? OR_ERR_ARG : OR_OK;
}

int oracle_tt_contract_batch(int B, int N, const int32_t* xdims, const int32_t* xranks, const int64_t* xoff,
                             const float* xcores, int M, const int32_t* ydims, const int32_t* yranks,
                             const int64_t* yoff, const float* ycores, int K, const int32_t* xm, const int32_t* ym,
                             const int64_t* out_off, double* out_cores, int nthreads)
{
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
#endif
    for (int b = 0; b < B; ++b) {
        const int32_t* xr = xranks + (int64_t)b * (N + 1);
        const int32_t* yr = yranks + (int64_t)b * (M + 1);
        int64_t nx = 0, ny = 0;
        for (int n = 0; n < N; ++n) nx += (int64_t)xr[n] * xdims[n] * xr[n + 1];
        for (int m = 0; m < M; ++m) ny += (int64_t)yr[m] * ydims[m] * yr[m + 1];
        double* X = widen(xcores + xoff[b], nx);
        double* Y = widen(ycores + yoff[b], ny);
        int32_t L, od[512], ork[513], os[512], op[512];
        int64_t ne;
        if (oracle_tt_contract(N, xdims, xr, X, M, ydims, yr, Y, K, xm, ym, &L, od, ork, os, op, &ne,
                               out_cores + out_off[b], NULL, NULL) != OR_OK) bad |= 1;
        free(X); free(Y);
    }
    return bad ? OR_ERR_ARG : OR_OK;
}

int oracle_tt_splice_batch(int B, int N, const int32_t* xdims, const int32_t* xranks, const int64_t* xoff,
                           const float* xcores, int M, const int32_t* ydims, const int32_t* yranks,
                           const int64_t* yoff, const float* ycores, int n, int m,
                           const int64_t* out_off, double* out_cores, int nthreads)
{
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
#endif
    for (int b = 0; b < B; ++b) {
        const int32_t* xr = xranks + (int64_t)b * (N + 1);
        const int32_t* yr = yranks + (int64_t)b * (M + 1);
        int64_t nx = 0, ny = 0;
        for (int k = 0; k < N; ++k) nx += (int64_t)xr[k] * xdims[k] * xr[k + 1];
        for (int k = 0; k < M; ++k) ny += (int64_t)yr[k] * ydims[k] * yr[k + 1];
        double* X = widen(xcores + xoff[b], nx);
        double* Y = widen(ycores + yoff[b], ny);
        int32_t L, od[512], ork[513], os[512], op[512];
        int64_t ne;
        if (oracle_tt_splice(N, xdims, xr, X, M, ydims, yr, Y, n, m, &L, od, ork, os, op, &ne,
                             out_cores + out_off[b]) != OR_OK) bad |= 1;
        free(X); free(Y);
    }
    return bad ? OR_ERR_ARG : OR_OK;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
