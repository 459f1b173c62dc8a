/*
 * ttc.h -- C ABI of libttc.so: batched Tensor-Train contraction on B200 (sm_100a).
 *
 * Method: Kisil et al., "Reducing Computational Complexity of Tensor Contractions via Tensor-Train
 * Networks" (arXiv 2109.00626), text in PAPER.md.  Citations are PAPER.md line numbers.
 *
 * DATA MODEL
 *   A tensor X in R^{I_1 x ... x I_N} held in TT format (Def. 7 / Eq. 9) is N cores
 *   G^(n) in R^{R_{n-1} x I_n x R_n} with boundary ranks R_0 = R_N = 1.
 *   Core storage is the paper's little-endian linear order (Def. 2 / Eq. 2; first index
 *   fastest): element [r, i, s] of core n is at r + R_{n-1} * (i + I_n * s).  A train is its N cores
 *   concatenated in core order ("TTD1" layout); train b of a batch starts at element
 *   offsets[b] of `cores` (offsets NULL: trains packed back to back, train b right after train b-1).
 *   Mode numbers at this API are 1-based.
 *
 * OWNERSHIP AND STREAMS
 *   The caller owns every device buffer (e.g. torch tensors); the library never allocates or frees device
 *   memory.  Contraction plans are host-only objects owned by the library until ttc_contract_plan_destroy.
 *   Compute calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *   stream) on the caller's current device.  All functions are re-entrant.
 *
 * ERRORS
 *   Every argument check runs on the host before anything is enqueued.  On error nothing is launched,
 *   the call returns a non-zero ttc_status, and ttc_last_error() (thread-local) names the offending
 *   quantity, e.g. "pair 17: X mode 4 (I=8) vs Y mode 3 (J=4)".  Launch failures return TTC_ERR_CUDA;
 *   asynchronous device faults surface at the caller's next synchronisation.  There is no CPU fallback:
 *   without a usable CUDA device a valid call returns TTC_ERR_CUDA.  Finiteness of core values and the
 *   TT-SVD rank bound are NOT validated (reading R15, R19).
 *
 * NUMERICS
 *   IEEE fp32 storage and arithmetic, fp32 accumulation, no fast-math, no atomics in any reduction: a
 *   call is bitwise deterministic run to run and independent of the batch split across GPUs.
 */
#ifndef TTC_H_
#define TTC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTC_VERSION_MAJOR 0
#define TTC_VERSION_MINOR 1
#define TTC_MAX_ORDER 256   /* ttc_inner: N <= 256 */
#define TTC_MAX_CONTRACT_ORDER 64  /* ttc_contract: N, M <= 64 */
#define TTC_MAX_RANK 128    /* every bond rank <= 128 (larger: TTC_ERR_UNSUPPORTED) */
#define TTC_MAX_SPLICE_RANK 1024   /* ttc_splice_plan_create / its ttc_contract / ttc_reconstruct: ranks <= 1024
                                      (the TT-SVD of Example 2's order-5 tensor has R_2 = 400) */

typedef enum {
    TTC_OK = 0,
    TTC_ERR_NULL = 1,        /* a required pointer is NULL */
    TTC_ERR_SHAPE = 2,       /* order / mode-size mismatch (e.g. I_n != J_m), batch mismatch, dims < 1 */
    TTC_ERR_RANK = 3,        /* R_0 != 1 or R_N != 1, a rank < 1 */
    TTC_ERR_MODES = 4,       /* contraction modes out of range, repeated or not strictly increasing */
    TTC_ERR_ALIGN = 5,       /* a core or output buffer not 4-byte aligned */
    TTC_ERR_OVERFLOW = 6,    /* a size or offset overflows int64, or a train runs past n_elems */
    TTC_ERR_UNSUPPORTED = 7, /* a rank > TTC_MAX_RANK, order > TTC_MAX_ORDER, ... */
    TTC_ERR_CUDA = 8,        /* CUDA runtime error (no device, launch failure) */
    TTC_ERR_ARG = 9          /* any other invalid argument (negative batch, k < 1, ...) */
} ttc_status;

/* A batch of B tensor trains of a common order N and common mode sizes dims[0..N-1]. */
typedef struct {
    int32_t        batch;         /* B >= 0; B = 0 makes every compute call a no-op returning TTC_OK      */
    int32_t        order;         /* N >= 1                                                              */
    const int32_t* dims;          /* host [N], I_n >= 1                                                  */
    const int32_t* ranks_host;    /* host [B*(N+1)], row b = R_0..R_N of train b; NULL => uniform ranks  */
    const int32_t* ranks_dev;     /* device copy of ranks_host (required iff ranks_host != NULL)         */
    int32_t        uniform_rank;  /* with ranks_host == NULL: ranks (1, R, ..., R, 1), R >= 1           */
    const int64_t* offsets_host;  /* host [B] element offset of train b; NULL => packed                  */
    const int64_t* offsets_dev;   /* device copy of offsets_host (required iff offsets_host != NULL)     */
    const float*   cores;         /* device fp32 core values (see DATA MODEL)                           */
    int64_t        n_elems;       /* number of floats addressable at `cores` (>= 1 when batch > 0, else
                                     TTC_ERR_ARG); every train must fit in [0, n_elems)                 */
} ttc_tt_batch;

/* ---------------------------------------------------------------------------------------------------
 * ttc_inner: out[b] = <X_b, Y_b>, the contraction of two equal-shape tensors "along all modes"
 * (Fig. 1b) evaluated on their TT cores, never on the dense tensors:
 *     Z_0 = [1];  Z_n = sum_{i=1..I_n} X_n[:, i, :]^T  Z_{n-1}  Y_n[:, i, :]   (R_n x P_n);  out[b] = Z_N.
 * Z_1 = A_x^T A_y is the paper's K (Eq. 12); the sweep is the all-modes case of
 * Alg. 2 step 4 applied mode after mode.  Cost sum_n I_n min(R_{n-1}P_n(P_{n-1}+R_n), R_nP_{n-1}(R_{n-1}+P_n))
 * MACs instead of the dense prod_n I_n.
 *   x, y    : batches with x->batch == y->batch, equal order and dims (else TTC_ERR_SHAPE); ranks of X and
 *             Y may differ (R_n vs P_n).
 *   out_dev : device fp32 [B], written once per pair, in pair order.
 * ------------------------------------------------------------------------------------------------- */
ttc_status ttc_inner(const ttc_tt_batch* x, const ttc_tt_batch* y, float* out_dev, void* stream);

/* ttc_inner with a processing order (a cost-descending work list, so that the batch's
 * most expensive pairs start first and heterogeneous-rank batches such as C5 end with a short tail).  The
 * results are identical (bitwise) to ttc_inner's: out_dev[b] is still pair b's value.
 *   order_host: host int32 [B], a permutation of 0..B-1 (validated: else TTC_ERR_ARG); order_dev: its device
 *   copy (caller-owned, read by the kernels).  ttc_pair_cost gives the cost to sort by. */
ttc_status ttc_inner_ordered(const ttc_tt_batch* x, const ttc_tt_batch* y, const int32_t* order_host,
                             const int32_t* order_dev, float* out_dev, void* stream);

/* ---------------------------------------------------------------------------------------------------
 * Partial contraction (TTCP, Alg. 2) of pair b: Z_b = X_b x_{(n_1,m_1),...,(n_K,m_K)} Y_b
 * (Eq. 8, applied to each of K disjoint mode pairs), returned in TT format
 * ("automatically given in the TT-format").  For K >= 1 the pairs must be strictly
 * increasing in both operands (1 <= n_1 < ... < n_K <= N, 1 <= m_1 < ... < m_K <= M) and I_{n_k} = J_{m_k}.
 *
 * Output train ("ladder", readings R7-R10): L = N + M - 2K cores.  Between consecutive contracted
 * pairs the free X cores come first (carrying the Y bond: X_n (x) I), then the free Y cores (carrying the X
 * bond: I (x) Y_m); contracted pairs become transfer matrices
 *     T_k[(r + R p), (r' + R' p')] = sum_i X_{n_k}[r, i, r'] Y_{m_k}[p, i, p']      (T_1 = K of Eq. 12 when
 * n_1 = m_1 = 1), products of consecutive transfers are absorbed into the next core (or the previous one at
 * the end).  Bond index (r, p) -> r + R*p (X fastest).  The canonical Eq. 8 mode order is recovered by the
 * permutation out_perm (Alg. 2 step 6) which this library returns as metadata.
 * K = N = M: L = 0 and the result is a single scalar equal to ttc_inner.
 * ------------------------------------------------------------------------------------------------- */
typedef struct ttc_contract_plan ttc_contract_plan;   /* opaque, host-only, immutable once created */

/* Validates x, y and the modes (all host data; no CUDA call) and builds the plan.  x_modes / y_modes are
 * host int32 [npairs] (may be NULL when npairs == 0).  *plan receives a new object on TTC_OK. */
ttc_status ttc_contract_plan_create(const ttc_tt_batch* x, const ttc_tt_batch* y, int32_t npairs,
                                    const int32_t* x_modes, const int32_t* y_modes, ttc_contract_plan** plan);

/* ---------------------------------------------------------------------------------------------------
 * ttc_splice_plan_create: the paper's own TTCP construction for one pair of END modes (Alg. 2 steps 4-5,
 * PAPER.md:358-374; Example 1), for operands already in TT format: with x_mode in {1, N} and
 * y_mode in {1, M} (1-based, I_{x_mode} = J_{y_mode}) the result Z = X x_n^m Y is the chain
 *     [X free cores]  K = A_x^T A_y (Eq. 12)  [Y free cores]
 * where the X free cores run N..2 with their rank modes swapped (core [s, i, r] = X_n[r, i, s]) when x_mode = 1
 * and 1..N-1 unchanged when x_mode = N; the Y free cores run 2..M when y_mode = 1 and M-1..1 swapped when
 * y_mode = M; A_x is the contracted X core read as I x R (its non-unit bond), A_y likewise.  K is absorbed into
 * the first Y free core (from the left), else into the last X free core (from the right); N = M = 1 gives the
 * scalar.  Output bonds are the operands' own ranks (no R*P Kronecker bonds as in the ladder), L = N + M - 2.
 * The returned plan is used exactly like a contraction plan (query, layout, ttc_contract, destroy): out_src /
 * out_perm give the chain order and the permutation to Eq. 8's order (Alg. 2 step 6).  Errors as
 * ttc_contract_plan_create; an interior mode gives TTC_ERR_MODES (use ttc_contract_plan_create).
 * ------------------------------------------------------------------------------------------------- */
ttc_status ttc_splice_plan_create(const ttc_tt_batch* x, const ttc_tt_batch* y, int32_t x_mode, int32_t y_mode,
                                  ttc_contract_plan** plan);

/* Structural metadata (identical for every pair of the batch).  Any output pointer may be NULL.
 *   out_order : L;  out_dims[L] : mode sizes in ladder order;
 *   out_src[L] : +n (X mode n) or -m (Y mode m), 1-based;
 *   out_perm[L]: 1-based ladder position of canonical (Eq. 8 order) output mode c;
 *   total_elems: floats of all output trains (layout of ttc_contract_plan_layout), >= 1 per pair;
 *   max_rank   : largest output bond rank over the batch. */
ttc_status ttc_contract_plan_query(const ttc_contract_plan* plan, int32_t* out_order, int32_t* out_dims,
                                   int32_t* out_src, int32_t* out_perm, int64_t* total_elems, int32_t* max_rank);

/* Per-pair output layout: out_ranks_host [B*(L+1)] (row b = bond ranks of output train b, each a product
 * R_a * P_b of operand bonds) and out_offsets_host [B] (packed element offsets).  Either may be NULL. */
ttc_status ttc_contract_plan_layout(const ttc_contract_plan* plan, int32_t* out_ranks_host,
                                    int64_t* out_offsets_host);

/* Computes the output cores of every pair into out_cores_dev (device fp32, total_elems floats) at the
 * offsets out_offsets_dev (device int64 [B], a copy of plan_layout's offsets; may be NULL when every pair
 * has the same ranks, in which case pair b starts at b * (total_elems / B)).  x and y must describe the
 * same shapes and ranks the plan was created with (else TTC_ERR_SHAPE). */
ttc_status ttc_contract(const ttc_contract_plan* plan, const ttc_tt_batch* x, const ttc_tt_batch* y,
                        float* out_cores_dev, const int64_t* out_offsets_dev, void* stream);

void ttc_contract_plan_destroy(ttc_contract_plan* plan);

/* ---------------------------------------------------------------------------------------------------
 * ttc_reconstruct: the dense tensor of every train of a batch (Eq. 9: the cores contracted
 * over consecutive rank modes), written in Eq. 2 order (first index fastest) after an optional
 * mode permutation -- Alg. 2 steps 5-6 ("obtain reconstructed version of Z^rho", then permute
 * Z^rho -> Z).  perm: host int32 [N], 1-based, output mode c is the train's mode perm[c] (pass a contraction
 * plan's out_perm to obtain Eq. 8's order), NULL = identity.  out_dev: device fp32, prod_n I_n floats per train
 * at out_offsets_dev[b] (device int64 [B]; NULL = packed, train b at b * prod_n I_n).
 * The kernel splits every train into a left and a right block of modes whose partial products fit in shared
 * memory together (prod_{n<=k} I_n R_k + R_k prod_{n>k} I_n <= 48K floats for some k) and multiplies them in one
 * launch (one CTA per train).  Trains with no such split (Example 2's outputs) need
 * ttc_reconstruct_ws: ttc_reconstruct returns TTC_ERR_ARG for them, naming the workspace size.  Errors as
 * ttc_inner (TTC_ERR_MODES for a perm that is not a permutation of 1..N).
 * ttc_reconstruct_workspace: bytes of device workspace ttc_reconstruct_ws needs for this batch and perm (0: the
 *   shared-memory kernel runs; else B x the two partial-product chains' ping-pong buffers).  Host only.
 * ttc_reconstruct_ws: ttc_reconstruct with a caller-owned device workspace (16-byte aligned, >= that size; NULL /
 *   0 when it is 0).  The large path is a chain of tiled FP32 GEMM launches on `stream` -- Left = X_1..X_k and
 *   Right = X_{k+1}..X_N built in the workspace, k minimising the multiply-adds -- with the output tile stored
 *   through the permuted Eq. 2 strides.  Same result as the one-launch kernel to fp32 rounding.
 * ------------------------------------------------------------------------------------------------- */
ttc_status ttc_reconstruct(const ttc_tt_batch* t, const int32_t* perm, float* out_dev, const int64_t* out_offsets_dev,
                           void* stream);
ttc_status ttc_reconstruct_workspace(const ttc_tt_batch* t, const int32_t* perm, int64_t* workspace_bytes);
ttc_status ttc_reconstruct_ws(const ttc_tt_batch* t, const int32_t* perm, float* out_dev, const int64_t* out_offsets_dev,
                              void* workspace_dev, int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------------
 * ttc_tt_svd: TT decomposition of a batch of dense tensors (Alg. 1, TT-SVD), optionally of the
 * permuted tensors X^rho (Alg. 2 step 1): the decomposed tensor's mode k is the input's mode
 * perm[k] (1-based; NULL = identity).  delta = eps / sqrt(N - 1) ||X||_F; each delta-truncated SVD keeps the
 * smallest rank with sum of discarded s_j^2 <= delta^2 (R23), singular values below 1e-7 of the largest
 * count as zero (R25), every left singular vector has its largest-magnitude entry positive (R24); then
 * ||X - TT(X)||_F <= eps ||X||_F.
 *   order, dims (host [N]): the INPUT tensor's shape; dense_dev: B tensors of prod(dims) floats, Eq. 2 order,
 *   packed.  Output: train b is packed (TTD1 layout) from cores_dev + b * train_cap, where train_cap comes from
 *   ttc_tt_svd_capacity (the floats of the largest possible ranks R_n <= min(prod_{k<=n} I_k, prod_{k>n} I_k));
 *   ranks_dev: device int32 [B, N + 1], the ranks found (read them back before describing the trains in a
 *   ttc_tt_batch with offsets b * train_cap).
 *   workspace_dev / workspace_bytes: caller-owned device scratch (16-byte aligned) of at least the size
 *   ttc_tt_svd_workspace returns.  With it, and every unfolding's smaller side <= 32, the decomposition runs as
 *   a pipeline of 1 + 2 (N - 1) launches (one warp per eigenproblem); with NULL / too small a workspace, or
 *   larger sides, as one fused launch (one CTA per tensor).  Both give the same ranks and cores to fp32
 *   rounding.  The library allocates nothing.
 * Tensors of prod(dims) <= 16384 with every unfolding's smaller side <= 64 are held in shared memory (the two
 * paths above).  Larger ones (Example 2's 20 x 20 x 20 x 5 and 20 x 20 x 20 x 5 x 4) take a
 * one-sided Jacobi kernel over the workspace, which is then REQUIRED (8 (2 prod(dims) + gmax^2 + 2 gmax + 80)
 * + 128 bytes per tensor, gmax the largest smaller side; NULL / too small: TTC_ERR_ARG naming the size); a group
 * of co-resident CTAs per tensor (cooperative launches, chunked when the batch exceeds the resident CTAs); limits
 * prod(dims) <= 2^27 and gmax <= 1024 (else TTC_ERR_UNSUPPORTED).  eps < 0: TTC_ERR_ARG.
 * ------------------------------------------------------------------------------------------------- */
ttc_status ttc_tt_svd_capacity(int32_t order, const int32_t* dims, const int32_t* perm, int64_t* train_cap);
ttc_status ttc_tt_svd_workspace(int32_t batch, int32_t order, const int32_t* dims, const int32_t* perm,
                                int64_t* workspace_bytes);   /* 0 when the fused launch is used anyway */
ttc_status ttc_tt_svd(int32_t batch, int32_t order, const int32_t* dims, const float* dense_dev, const int32_t* perm,
                      double eps, float* cores_dev, int32_t* ranks_dev, void* workspace_dev, int64_t workspace_bytes,
                      void* stream);

/* ---------------------------------------------------------------------------------------------------
 * Host cost model and batch partitioner (multi-GPU sharding).
 * ttc_pair_cost: per pair b of ttc_inner, mac[b] = sweep MACs (cheaper association per step) and
 *                bytes[b] = algorithmic HBM bytes (every core read once + 4-byte result).  Host only.
 * ttc_partition: splits B pairs into k contiguous ranges [bounds[j], bounds[j+1]) with bounds[0] = 0,
 *                bounds[k] = B, minimising the largest range cost (cost[b] >= 0, host [B]).  Host only.
 * ------------------------------------------------------------------------------------------------- */
ttc_status ttc_pair_cost(const ttc_tt_batch* x, const ttc_tt_batch* y, double* mac, double* bytes);
ttc_status ttc_partition(const double* cost, int32_t B, int32_t k, int32_t* bounds);

/* Static strings; ttc_last_error is the detail of the calling thread's last failed call. */
const char* ttc_status_string(ttc_status s);
const char* ttc_last_error(void);
int32_t     ttc_version(void);   /* TTC_VERSION_MAJOR * 100 + TTC_VERSION_MINOR */

#ifdef __cplusplus
}
#endif
#endif /* TTC_H_ */
