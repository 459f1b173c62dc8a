// ttc_internal.h -- internal (non-ABI) structures shared by the host library and the kernels.
// Nothing here crosses the C ABI; include/ttc.h is the boundary.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../include/ttc.h"

namespace ttc {

// One operand batch as the kernels see it.  ranks == nullptr: uniform (1, urank, ..., urank, 1);
// offsets == nullptr: packed, train b at b * train_elems (uniform ranks only).
struct TrainDev {
    const float*   cores;
    const int32_t* ranks;
    const int64_t* offsets;
    int32_t        urank;
    int64_t        train_elems;
};

struct InnerArgs {
    int32_t  B, N;
    int32_t  dims[TTC_MAX_ORDER];
    TrainDev x, y;
    float*   out;
    const int32_t* order;   // optional device work list (pair indices, e.g. cost-descending); nullptr = identity
    int32_t  zmax;          // max_n R_n * P_n over the batch (floats)
    int32_t  wbuf;          // floats of the W chunk buffer (generic kernel)
};

// Launchers (inner_generic.cu, inner_fast.cu, contract.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_inner_generic(const InnerArgs& a, cudaStream_t s);
bool        inner_fast_supported(const InnerArgs& a, int max_rank, bool uniform);
cudaError_t launch_inner_fast(const InnerArgs& a, int max_rank, bool uniform, cudaStream_t s);
bool        inner_r16_supported(const InnerArgs& a, bool uniform_r16);
cudaError_t launch_inner_r16(const InnerArgs& a, cudaStream_t s);
bool        inner_r64_supported(const InnerArgs& a, bool uniform_r64);
cudaError_t launch_inner_r64(const InnerArgs& a, cudaStream_t s);
// uniform rank 64, I_n = 4, packed trains: tcgen05 / TMEM / TMA kernel (inner_r64tc.cu)
bool        inner_r64tc_supported(const InnerArgs& a, bool uniform_r64);
cudaError_t launch_inner_r64tc(const InnerArgs& a, cudaStream_t s);
// tiny batches (inner_small.cu): both trains of a pair in SMEM at once; floats of each region
struct SmallLayout {
    int32_t xmax, ymax, wmax, zmax;
};
cudaError_t launch_inner_small(const InnerArgs& a, const SmallLayout& L, cudaStream_t s);
bool        inner_ffma_supported(const InnerArgs& a, int max_rank, bool ranks_mult8);
// aligned16: both core buffers 16-byte aligned and every train offset a multiple of 4 floats (the TMA staging
// path; otherwise 16-byte cp.async); nx / ny: floats at X / Y cores (the tensor maps' extent)
cudaError_t launch_inner_ffma(const InnerArgs& a, int max_rank, bool aligned16, int64_t nx, int64_t ny,
                              cudaStream_t s);
// cuTensorMapEncodeTiled through the runtime's driver entry point (nullptr if unavailable)
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn();

// ---- tt_contract (ladder) ------------------------------------------------------------------------
enum ElKind : int32_t { EL_XFREE = 1, EL_YFREE = 2, EL_T = 3 };

struct LadderEl {
    int32_t kind;  // ElKind
    int32_t mode;  // 0-based: X mode (XFREE, T), Y mode (YFREE)
    int32_t hold;  // XFREE: Y bond index b carried (P_b); YFREE: X bond index a carried (R_a); T: 0-based Y mode
};

// One output core of the ladder: the free core it comes from plus the transfers absorbed into it
// (consecutive transfers multiplied left to right; lt = from the left, rt = from the right).
struct OutCore {
    int32_t el;        // index into the ladder sequence of the free core
    int32_t lt_first;  // first left transfer (index into the sequence), lt_count of them
    int32_t lt_count;
    int32_t rt_first;  // trailing transfers absorbed from the right (last core only)
    int32_t rt_count;
};

constexpr int kMaxContractOrder = 64;            // N, M <= 64 for ttc_contract (kernel-parameter budget)
constexpr int kMaxLadder = 2 * kMaxContractOrder + 4;

struct ContractArgs {
    int32_t  B, N, M, K, L, nseq;
    int32_t  xdims[kMaxContractOrder];
    int32_t  ydims[kMaxContractOrder];
    LadderEl seq[kMaxLadder];
    OutCore  outc[kMaxLadder];
    TrainDev x, y;
    float*   out;
    const int64_t* out_offsets;   // device [B] or nullptr (uniform: b * out_pair_elems)
    int64_t  out_pair_elems;
    int32_t  tl_off, tr_off;      // shared-scratch offsets (floats) of the left / right transfer products
    int32_t  tmp_off, tmp_size;   // three temporaries of tmp_size floats for chains of >= 2 transfers
    int32_t  stage_off, stage_floats;   // shared copy of the pair's two trains (0: read from global)
};

cudaError_t launch_contract(const ContractArgs& a, size_t smem_bytes, cudaStream_t s);
cudaError_t contract_func_attributes(cudaFuncAttributes* fa);   // static shared memory of the contract kernel

// ---- TTCP splice of end modes (splice.cu) ------------------------------------------------------------
struct SpliceArgs {
    int32_t  B, N, M, L;
    int32_t  n, m;                      // contracted modes, 1-based, n in {1, N}, m in {1, M}
    int32_t  nx;                        // chain position of the core absorbing K from the left (L: none, right)
    int32_t  xdims[kMaxContractOrder];
    int32_t  ydims[kMaxContractOrder];
    int32_t  src[kMaxLadder];           // +(mode + 1) X, -(mode + 1) Y (0-based mode inside)
    int32_t  rev[kMaxLadder];           // 1: rank modes swapped
    TrainDev x, y;
    float*   out;
    const int64_t* out_offsets;         // device [B] or nullptr (uniform)
    int64_t  out_pair_elems;
    int32_t  k4;                        // floats of SMEM for K (rounded up to 4)
    int32_t  stage_x, stage_y;          // floats of SMEM for the whole X / Y train (0: cores read from global)
};
cudaError_t launch_splice(const SpliceArgs& a, size_t smem_bytes, cudaStream_t s);

// ---- dense reconstruction (reconstruct.cu) -------------------------------------------------------------
struct ReconArgs {
    int32_t  B, N, k;                   // split: left block = modes 1..k, right block = k+1..N (1 <= k < N)
    int32_t  rows, cols;                // prod_{n<=k} I_n, prod_{n>k} I_n
    int32_t  lbuf, t1, rbuf, t2;        // floats of: Left (+ same-parity partials), its temporary, Right, its temporary
    int32_t  tm;                        // output tile 64 x 16 tm (tm = 4 or 5)
    int32_t  ldl;                       // row stride of Left^T (rows rounded up to a multiple of 4)
    int32_t  ld[TTC_MAX_ORDER];         // row stride of the left partial P_{j+1}^T (= ldl for j = k - 1)
    int32_t  lrev;                      // 1: Left's rows enumerate modes k..1 fastest-first (big-endian)
    int32_t  dims[TTC_MAX_ORDER];
    int64_t  ostride[TTC_MAX_ORDER];    // output stride of train mode n (permuted Eq. 2 order)
    TrainDev t;
    float*   out;
    const int64_t* out_offsets;         // device [B] or nullptr (packed)
    int64_t  pair_elems;                // prod_n I_n
};
cudaError_t launch_reconstruct(const ReconArgs& a, size_t smem_bytes, cudaStream_t s);

// trains whose partial products exceed shared memory (reconstruct_big.cu): a chain of tiled GEMM launches over a
// caller-owned workspace (0-based modes; pre[j] = prod_{n<j} I_n, suf[j] = prod_{n>=j} I_n)
struct ReconBigArgs {
    int32_t  B, N, k;                   // split: Left = cores 0..k-1, Right = cores k..N-1 (1 <= k < N)
    int32_t  row_fast;                  // 1: the output's stride-1 mode is one of Left's (store along rows)
    int32_t  dims[TTC_MAX_ORDER];
    int64_t  pre[TTC_MAX_ORDER + 1], suf[TTC_MAX_ORDER + 1];
    int64_t  ostride[TTC_MAX_ORDER];
    int64_t  tiles_left[TTC_MAX_ORDER], tiles_right[TTC_MAX_ORDER], tiles_final;   // 64 x 64 tiles per launch
    TrainDev t;
    float*   out;
    const int64_t* out_offsets;
    int64_t  pair_elems;
    float*   ws;                        // B x (2 ws_left + 2 ws_right) floats
    int64_t  ws_left, ws_right;         // floats of one Left / Right ping-pong buffer
};
cudaError_t launch_reconstruct_big(const ReconBigArgs& a, cudaStream_t s);

// ---- batched TT-SVD (ttsvd.cu) -------------------------------------------------------------------------
struct TtsvdArgs {
    int32_t  B, N, elems, gmax;         // tensors, order, prod dims (<= shared memory), largest Gram side
    int32_t  dims[TTC_MAX_ORDER];       // dims of the decomposed tensor X^rho
    int64_t  in_stride[TTC_MAX_ORDER];  // source stride of X^rho's mode k (Alg. 2 step 1's permutation)
    const float* dense;                 // B tensors, elems floats each, Eq. 2 order of X
    double   eps2;                      // eps^2 / (N - 1)
    float*   cores;                     // B * train_cap floats
    int64_t  train_cap;
    int32_t* ranks;                     // device [B, N + 1]
};
cudaError_t launch_ttsvd(const TtsvdArgs& a, size_t smem_bytes, cudaStream_t s);
// workspace of the multi-kernel TT-SVD (Gram sides <= 32): Z_n, the Gram matrix, its eigen-decomposition
struct TtsvdWs {
    float*   z;                         // B x elems
    double*  g;                         // B x gmax^2
    double*  v;                         // B x gmax^2
    double*  lam;                       // B x gmax
    int32_t* ord;                       // B x gmax
    double*  nrm;                       // B
};
cudaError_t launch_ttsvd_pipeline(const TtsvdArgs& a, const TtsvdWs& w, cudaStream_t s);
// tensors beyond the shared-memory kernels (ttsvd_big.cu): one CTA per tensor over an fp64 workspace of
// ttsvd_big_ws_per(elems, gmax) doubles per tensor; every unfolding's smaller side <= kTtsvdBigMaxSide
constexpr int kTtsvdBigMaxSide = 1024;
int64_t     ttsvd_big_ws_bytes(int32_t B, int32_t elems, int32_t gmax);
cudaError_t launch_ttsvd_big(const TtsvdArgs& a, void* workspace, cudaStream_t s);

}  // namespace ttc
