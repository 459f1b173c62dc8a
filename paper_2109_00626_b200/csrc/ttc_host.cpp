// ttc_host.cpp -- the C ABI of libttc.so (include/ttc.h): host-side validation, planning, cost model,
// partitioner and kernel dispatch.  Host data only until the final launch; no device allocation.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ttc_internal.h"

namespace {

thread_local std::string g_last_error;

ttc_status fail(ttc_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

bool mul_ok(int64_t a, int64_t b, int64_t* out) { return !__builtin_mul_overflow(a, b, out); }
bool add_ok(int64_t a, int64_t b, int64_t* out) { return !__builtin_add_overflow(a, b, out); }

// Host view of one validated operand batch.
struct HostTrain {
    const ttc_tt_batch* t = nullptr;
    int B = 0, N = 0;
    bool uniform = true;
    int urank = 1;
    int max_rank = 1;
    bool mult8 = true;                 // every interior rank is a multiple of 8
    int64_t train_elems_uniform = 0;   // uniform ranks: elements per train
    std::vector<int64_t> sizes;        // heterogeneous ranks: elements of train b (valid ranks only)

    int rank(int b, int n) const {
        if (!uniform) return t->ranks_host[(int64_t)b * (N + 1) + n];
        return (n == 0 || n == N) ? 1 : urank;
    }
};

// A1: validate one operand batch; `name` is "X" or "Y".
ttc_status check_batch(const ttc_tt_batch* t, const char* name, int max_order, HostTrain* h,
                       int max_rank = TTC_MAX_RANK) {
    if (!t) return fail(TTC_ERR_NULL, "%s: batch descriptor is NULL", name);
    if (t->batch < 0) return fail(TTC_ERR_ARG, "%s: batch = %d < 0", name, t->batch);
    if (t->order < 1) return fail(TTC_ERR_SHAPE, "%s: order N = %d < 1", name, t->order);
    if (t->order > max_order)
        return fail(TTC_ERR_UNSUPPORTED, "%s: order N = %d > %d supported", name, t->order, max_order);
    if (!t->dims) return fail(TTC_ERR_NULL, "%s: dims is NULL", name);
    h->t = t;
    h->B = t->batch;
    h->N = t->order;
    for (int n = 0; n < t->order; ++n)
        if (t->dims[n] < 1) return fail(TTC_ERR_SHAPE, "%s: mode %d has I = %d < 1", name, n + 1, t->dims[n]);
    h->uniform = (t->ranks_host == nullptr);
    if (h->uniform) {
        if (t->ranks_dev)
            return fail(TTC_ERR_ARG, "%s: ranks_dev given without ranks_host", name);
        if (t->order > 1) {
            if (t->uniform_rank < 1) return fail(TTC_ERR_RANK, "%s: uniform_rank = %d < 1", name, t->uniform_rank);
            if (t->uniform_rank > max_rank)
                return fail(TTC_ERR_UNSUPPORTED, "%s: uniform_rank = %d > %d", name, t->uniform_rank, max_rank);
            h->urank = t->uniform_rank;
            h->mult8 = (h->urank & 7) == 0;
        }
        h->max_rank = t->order > 1 ? h->urank : 1;
    } else {
        if (t->batch > 0 && !t->ranks_dev) return fail(TTC_ERR_NULL, "%s: ranks_host given but ranks_dev is NULL", name);
        // one branch-light pass over the interior ranks (this runs on every call: O(B N), e.g. 1M ranks for
        // C5); the slow loop below only runs to name the first offending rank
        int mr = 1, bad = 0;
        unsigned or8 = 0;
        const int N = t->order;
        const int32_t* rh = t->ranks_host;
        // the train sizes come out of the same pass (h->sizes): sizes and bounds are checked below
        h->sizes.resize(t->batch);
        for (int b = 0; b < t->batch; ++b) {
            const int32_t* r = rh + (int64_t)b * (N + 1);
            bad |= (r[0] != 1) | (r[N] != 1);
            int64_t elems = (int64_t)t->dims[0] * r[1];
            for (int n = 1; n < N; ++n) {
                const int v = r[n];
                bad |= (v < 1) | (v > max_rank);
                mr = v > mr ? v : mr;
                or8 |= (unsigned)v;
                elems += (int64_t)v * t->dims[n] * r[n + 1];
            }
            h->sizes[b] = elems;
        }
        if (bad) {
            for (int b = 0; b < t->batch; ++b) {
                const int32_t* r = rh + (int64_t)b * (N + 1);
                if (r[0] != 1 || r[N] != 1)
                    return fail(TTC_ERR_RANK, "%s pair %d: boundary ranks R_0 = %d, R_N = %d (must be 1)", name, b,
                                r[0], r[N]);
                for (int n = 1; n < N; ++n) {
                    if (r[n] < 1) return fail(TTC_ERR_RANK, "%s pair %d: rank R_%d = %d < 1", name, b, n, r[n]);
                    if (r[n] > max_rank)
                        return fail(TTC_ERR_UNSUPPORTED, "%s pair %d: rank R_%d = %d > %d", name, b, n, r[n], max_rank);
                }
            }
        }
        h->mult8 = (or8 & 7u) == 0;   // every interior rank is a multiple of 8
        h->max_rank = N > 1 ? mr : 1;
    }
    if (t->offsets_host && t->batch > 0 && !t->offsets_dev)
        return fail(TTC_ERR_NULL, "%s: offsets_host given but offsets_dev is NULL", name);
    if (!t->offsets_host && t->offsets_dev) return fail(TTC_ERR_ARG, "%s: offsets_dev given without offsets_host", name);
    if (!t->offsets_host && !h->uniform && t->batch > 1)
        return fail(TTC_ERR_ARG, "%s: heterogeneous ranks need explicit offsets", name);
    if (t->batch > 0 && !t->cores) return fail(TTC_ERR_NULL, "%s: cores is NULL", name);
    if (t->batch > 0 && t->n_elems < 1)
        return fail(TTC_ERR_ARG, "%s: n_elems = %lld: the number of floats at cores is required (>= 1)", name,
                    (long long)t->n_elems);
    if (t->cores && (reinterpret_cast<uintptr_t>(t->cores) & 3u))
        return fail(TTC_ERR_ALIGN, "%s: cores pointer not 4-byte aligned", name);
    // sizes and bounds, overflow-checked.  A train has at most TTC_MAX_ORDER cores of at most
    // TTC_MAX_SPLICE_RANK^2 * (2^31 - 1) elements, < 2^52: its size cannot overflow; offset + size can.
    const int N = t->order;
    if (h->uniform) {
        int64_t elems = 0;
        for (int n = 0; n < N; ++n) elems += (int64_t)h->rank(0, n) * t->dims[n] * h->rank(0, n + 1);
        h->train_elems_uniform = elems;
    }
    int64_t packed_end = 0;
    if (!t->offsets_host && h->uniform && t->batch > 0) {   // packed uniform: the last train bounds everything
        int64_t last;
        if (!mul_ok(h->train_elems_uniform, t->batch, &last)) return fail(TTC_ERR_OVERFLOW, "%s: batch size overflows", name);
        if (last > t->n_elems)
            return fail(TTC_ERR_OVERFLOW, "%s: %d packed trains of %lld floats exceed n_elems = %lld", name,
                        t->batch, (long long)h->train_elems_uniform, (long long)t->n_elems);
        return TTC_OK;
    }
    for (int b = 0; b < t->batch; ++b) {
        const int64_t elems = h->uniform ? h->train_elems_uniform : h->sizes[b];
        int64_t start = t->offsets_host ? t->offsets_host[b] : packed_end, end;
        if (start < 0) return fail(TTC_ERR_OVERFLOW, "%s pair %d: offset %lld < 0", name, b, (long long)start);
        if (!add_ok(start, elems, &end)) return fail(TTC_ERR_OVERFLOW, "%s pair %d: offset + size overflows", name, b);
        if (end > t->n_elems)
            return fail(TTC_ERR_OVERFLOW, "%s pair %d: train [%lld, %lld) runs past n_elems = %lld", name, b,
                        (long long)start, (long long)end, (long long)t->n_elems);
        packed_end = end;
    }
    return TTC_OK;
}

ttc::TrainDev to_dev(const HostTrain& h) {
    ttc::TrainDev d;
    d.cores = h.t->cores;
    d.ranks = h.uniform ? nullptr : h.t->ranks_dev;
    d.offsets = h.t->offsets_host ? h.t->offsets_dev : nullptr;
    d.urank = h.urank;
    d.train_elems = h.train_elems_uniform;
    return d;
}

ttc_status cuda_fail(cudaError_t e, const char* what) {
    return fail(TTC_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

}  // namespace

// ================================================================================================ C ABI
extern "C" {

const char* ttc_status_string(ttc_status s) {
    switch (s) {
        case TTC_OK: return "TTC_OK";
        case TTC_ERR_NULL: return "TTC_ERR_NULL";
        case TTC_ERR_SHAPE: return "TTC_ERR_SHAPE";
        case TTC_ERR_RANK: return "TTC_ERR_RANK";
        case TTC_ERR_MODES: return "TTC_ERR_MODES";
        case TTC_ERR_ALIGN: return "TTC_ERR_ALIGN";
        case TTC_ERR_OVERFLOW: return "TTC_ERR_OVERFLOW";
        case TTC_ERR_UNSUPPORTED: return "TTC_ERR_UNSUPPORTED";
        case TTC_ERR_CUDA: return "TTC_ERR_CUDA";
        case TTC_ERR_ARG: return "TTC_ERR_ARG";
    }
    return "TTC_ERR_UNKNOWN";
}

const char* ttc_last_error(void) { return g_last_error.c_str(); }

int32_t ttc_version(void) { return TTC_VERSION_MAJOR * 100 + TTC_VERSION_MINOR; }

namespace {
ttc_status inner_impl(const ttc_tt_batch* x, const ttc_tt_batch* y, const int32_t* order_dev, float* out_dev,
                      void* stream);
}  // namespace

ttc_status ttc_inner(const ttc_tt_batch* x, const ttc_tt_batch* y, float* out_dev, void* stream) {
    g_last_error.clear();
    return inner_impl(x, y, nullptr, out_dev, stream);
}

ttc_status ttc_inner_ordered(const ttc_tt_batch* x, const ttc_tt_batch* y, const int32_t* order_host,
                             const int32_t* order_dev, float* out_dev, void* stream) {
    g_last_error.clear();
    if (!x || !y) return fail(TTC_ERR_NULL, "X / Y batch descriptor is NULL");
    const int B = x->batch;
    if (B > 0) {
        if (!order_host || !order_dev) return fail(TTC_ERR_NULL, "order_host / order_dev is NULL");
        std::vector<char> seen((size_t)B, 0);
        for (int k = 0; k < B; ++k) {
            const int32_t v = order_host[k];
            if (v < 0 || v >= B || seen[(size_t)v])
                return fail(TTC_ERR_ARG, "order[%d] = %d: order must be a permutation of 0..%d", k, v, B - 1);
            seen[(size_t)v] = 1;
        }
    }
    return inner_impl(x, y, order_dev, out_dev, stream);
}

namespace {
ttc_status inner_impl(const ttc_tt_batch* x, const ttc_tt_batch* y, const int32_t* order_dev, float* out_dev,
                      void* stream) {
    HostTrain hx, hy;
    ttc_status st;
    if ((st = check_batch(x, "X", TTC_MAX_ORDER, &hx)) != TTC_OK) return st;
    if ((st = check_batch(y, "Y", TTC_MAX_ORDER, &hy)) != TTC_OK) return st;
    if (x->batch != y->batch) return fail(TTC_ERR_SHAPE, "batch mismatch: X has %d trains, Y has %d", x->batch, y->batch);
    if (x->order != y->order) return fail(TTC_ERR_SHAPE, "order mismatch: X N = %d, Y N = %d", x->order, y->order);
    for (int n = 0; n < x->order; ++n)
        if (x->dims[n] != y->dims[n])
            return fail(TTC_ERR_SHAPE, "X mode %d (I=%d) vs Y mode %d (J=%d)", n + 1, x->dims[n], n + 1, y->dims[n]);
    const int B = x->batch;
    if (B == 0) return TTC_OK;
    if (!out_dev) return fail(TTC_ERR_NULL, "out_dev is NULL");
    if (reinterpret_cast<uintptr_t>(out_dev) & 3u) return fail(TTC_ERR_ALIGN, "out_dev not 4-byte aligned");

    ttc::InnerArgs a;
    std::memset(&a, 0, sizeof(a));
    a.B = B;
    a.N = x->order;
    for (int n = 0; n < a.N; ++n) a.dims[n] = x->dims[n];
    a.x = to_dev(hx);
    a.y = to_dev(hy);
    a.out = out_dev;
    a.order = order_dev;   // nullptr: natural order
    const int mr = std::max(hx.max_rank, hy.max_rank);
    a.zmax = mr * mr;
    a.wbuf = std::max(mr * mr, 8192);
    const bool uniform = hx.uniform && hy.uniform && hx.urank == hy.urank;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    // TTC_KERNEL=generic|fast|small|ffma|mmasync forces the general-shape / CTA-per-pair tensor-core / tiny-batch /
    // warp-per-pair FP32 / legacy mma.sync rank-64 kernel (cross-checks and A/B measurements)
    const char* kv = std::getenv("TTC_KERNEL");
    const bool force_generic = kv && std::strcmp(kv, "generic") == 0;
    // uniform rank-16 trains with 16-byte aligned cores and trains: the specialised rank-16 kernel
    bool aligned16 = ((reinterpret_cast<uintptr_t>(x->cores) | reinterpret_cast<uintptr_t>(y->cores)) & 15u) == 0;
    for (int b = 0; aligned16 && b < B; ++b) {
        if (x->offsets_host && (x->offsets_host[b] & 3)) aligned16 = false;
        if (y->offsets_host && (y->offsets_host[b] & 3)) aligned16 = false;
    }
    const bool uniform_r16 = uniform && hx.urank == 16 && aligned16 && (hx.train_elems_uniform & 3) == 0;
    const bool force_fast = kv && std::strcmp(kv, "fast") == 0;
    const bool force_ffma = kv && std::strcmp(kv, "ffma") == 0;
    const bool force_mma_sync = kv && std::strcmp(kv, "mmasync") == 0;   // rank 64: the mma.sync kernel
    const bool uniform_r64 = uniform && hx.urank == 64 && aligned16 && (hx.train_elems_uniform & 3) == 0;
    // tiny batches are latency-bound: both trains of a pair staged at once, one DRAM round trip per pair
    // (TTC_KERNEL=small forces it for any batch that fits, for cross-checks)
    const bool force_small = kv && std::strcmp(kv, "small") == 0;
    if ((B <= 4 && !kv) || force_small) {
        ttc::SmallLayout L{0, 0, 1, 1};
        for (int b = 0; b < B; ++b) {
            int64_t xe = 0, ye = 0;
            for (int n = 0; n < a.N; ++n) {
                const int64_t R = hx.rank(b, n), S = hx.rank(b, n + 1), P = hy.rank(b, n), Q = hy.rank(b, n + 1);
                xe += R * a.dims[n] * S;
                ye += P * a.dims[n] * Q;
                L.wmax = (int32_t)std::max<int64_t>(L.wmax, R * a.dims[n] * Q);
                L.zmax = (int32_t)std::max<int64_t>(L.zmax, S * Q);
            }
            L.xmax = (int32_t)std::max<int64_t>(L.xmax, (xe + 3) & ~int64_t(3));
            L.ymax = (int32_t)std::max<int64_t>(L.ymax, (ye + 3) & ~int64_t(3));
        }
        L.wmax = (L.wmax + 3) & ~3;
        L.zmax = (L.zmax + 3) & ~3;
        const int64_t bytes = 4 * ((int64_t)L.xmax + L.ymax + L.wmax + 2 * (int64_t)L.zmax);
        if (bytes <= 200 * 1024) {
            e = ttc::launch_inner_small(a, L, s);
            if (e != cudaSuccess) return cuda_fail(e, "ttc_inner launch");
            return TTC_OK;
        }
    }
    // every core starts on 16 bytes (the FP32 kernel stages with 16-byte copies): aligned buffers, and offsets
    // (given, or b * train_elems) multiples of 4 floats
    const bool cores16 = aligned16 && (x->offsets_host || (hx.train_elems_uniform & 3) == 0) &&
                         (y->offsets_host || (hy.train_elems_uniform & 3) == 0);
    const bool ffma_ok = cores16 && ttc::inner_ffma_supported(a, mr, hx.mult8 && hy.mult8);
    if (force_ffma && ffma_ok)
        e = ttc::launch_inner_ffma(a, mr, cores16, x->n_elems, y->n_elems, s);
    else if (!force_generic && !force_fast && ttc::inner_r16_supported(a, uniform_r16))
        e = ttc::launch_inner_r16(a, s);
    else if (!force_generic && !force_mma_sync && ttc::inner_r64tc_supported(a, uniform_r64))
        e = ttc::launch_inner_r64tc(a, s);     // tcgen05.mma kind::tf32, TMEM accumulators, TMA operands
    else if (!force_generic && ttc::inner_r64_supported(a, uniform_r64))
        e = ttc::launch_inner_r64(a, s);       // legacy mma.sync 3xTF32 (any I_n, offsets allowed)
    else if (!force_generic && !force_fast && ffma_ok)
        e = ttc::launch_inner_ffma(a, mr, cores16, x->n_elems, y->n_elems, s);   // warp per pair on the FP32 pipe (ranks multiple of 8, <= 32)
    else if (!force_generic && ttc::inner_fast_supported(a, mr, uniform))
        e = ttc::launch_inner_fast(a, mr, uniform, s);
    else
        e = ttc::launch_inner_generic(a, s);
    if (e != cudaSuccess) return cuda_fail(e, "ttc_inner launch");
    return TTC_OK;
}
}  // namespace

namespace {

// The large path (reconstruct_big.cu): the split k minimising the batch's multiply-adds (chain steps + the final
// product), the tiles of every launch, and the ping-pong buffers' floats (each rounded to 16 bytes).
ttc_status recon_big_plan(const HostTrain& h, const ttc_tt_batch* t, ttc::ReconBigArgs* a) {
    const int N = t->order, B = t->batch;
    a->B = B; a->N = N;
    a->pre[0] = 1;
    for (int n = 0; n < N; ++n) a->pre[n + 1] = a->pre[n] * t->dims[n];
    a->suf[N] = 1;
    for (int n = N - 1; n >= 0; --n) a->suf[n] = a->suf[n + 1] * t->dims[n];
    for (int n = 0; n < N; ++n) a->dims[n] = t->dims[n];
    auto tiles = [](int64_t m, int64_t n) { return ((m + 63) / 64) * ((n + 63) / 64); };
    double best = -1.0;
    for (int k = 1; k < N; ++k) {
        double mac = 0.0;
        for (int b = 0; b < B; ++b) {
            for (int j = 1; j < k; ++j) mac += (double)a->pre[j] * h.rank(b, j) * t->dims[j] * h.rank(b, j + 1);
            for (int j = k; j < N - 1; ++j)
                mac += (double)h.rank(b, j) * t->dims[j] * h.rank(b, j + 1) * a->suf[j + 1];
            mac += (double)a->pre[k] * h.rank(b, k) * a->suf[k];
        }
        if (best < 0.0 || mac < best) { best = mac; a->k = k; }
    }
    const int k = a->k;
    int64_t wl = 0, wr = 0;
    for (int j = 0; j < TTC_MAX_ORDER; ++j) a->tiles_left[j] = a->tiles_right[j] = 0;
    a->tiles_final = 0;
    for (int b = 0; b < B; ++b) {
        for (int j = 1; j < k; ++j) {
            wl = std::max(wl, a->pre[j + 1] * h.rank(b, j + 1));
            a->tiles_left[j] = std::max(a->tiles_left[j], tiles(a->pre[j], (int64_t)t->dims[j] * h.rank(b, j + 1)));
        }
        for (int j = k; j < N - 1; ++j) {
            wr = std::max(wr, (int64_t)h.rank(b, j) * a->suf[j]);
            a->tiles_right[j] = std::max(a->tiles_right[j], tiles((int64_t)h.rank(b, j) * t->dims[j], a->suf[j + 1]));
        }
        a->tiles_final = std::max(a->tiles_final, tiles(a->pre[k], a->suf[k]));
    }
    a->ws_left = (wl + 3) & ~int64_t(3);
    a->ws_right = (wr + 3) & ~int64_t(3);
    if (a->tiles_final > 0x7fffffffLL) return fail(TTC_ERR_UNSUPPORTED, "output of %lld x %lld per train too large",
                                                    (long long)a->pre[k], (long long)a->suf[k]);
    return TTC_OK;
}

// ttc_reconstruct_ws, or (query != NULL) only the workspace it needs
ttc_status reconstruct_impl(const ttc_tt_batch* t, const int32_t* perm, float* out_dev, const int64_t* out_offsets_dev,
                            void* workspace_dev, int64_t workspace_bytes, void* stream, int64_t* query) {
    g_last_error.clear();
    if (query) *query = 0;
    HostTrain h;
    ttc_status st;
    if ((st = check_batch(t, "T", TTC_MAX_ORDER, &h, TTC_MAX_SPLICE_RANK)) != TTC_OK) return st;
    const int N = t->order, B = t->batch;
    // output strides of the train's modes: output mode c is train mode perm[c] (1-based)
    std::vector<int64_t> ostride(N, 0);
    {
        std::vector<int> seen(N, 0);
        int64_t stride = 1;
        for (int c = 0; c < N; ++c) {
            const int m = perm ? perm[c] : c + 1;
            if (m < 1 || m > N || seen[m - 1])
                return fail(TTC_ERR_MODES, "perm[%d] = %d: perm must be a permutation of 1..%d", c, m, N);
            seen[m - 1] = 1;
            ostride[m - 1] = stride;
            if (!mul_ok(stride, t->dims[m - 1], &stride)) return fail(TTC_ERR_OVERFLOW, "dense size overflows int64");
        }
        if (stride >= (int64_t(1) << 31))
            return fail(TTC_ERR_UNSUPPORTED, "dense tensor of %lld elements per train (>= 2^31)", (long long)stride);
    }
    int64_t pair_elems = 1;
    for (int n = 0; n < N; ++n) pair_elems *= t->dims[n];
    if (B == 0) return TTC_OK;
    if (!query) {
        if (!out_dev) return fail(TTC_ERR_NULL, "out_dev is NULL");
        if (reinterpret_cast<uintptr_t>(out_dev) & 3u) return fail(TTC_ERR_ALIGN, "out_dev not 4-byte aligned");
    }
    // the split k: left block modes 1..k, right block k+1..N; shared memory = both blocks + build temporaries +
    // the row / column offset tables, the batch maximum over pairs, minimised over k
    const int64_t kSmemMax = 220 * 1024;
    int best_k = -1;
    int64_t best = 0, bl = 0, bt1 = 0, br = 0, bt2 = 0;
    std::vector<int64_t> pre(N + 1, 1), suf(N + 1, 1);
    for (int n = 0; n < N; ++n) pre[n + 1] = pre[n] * t->dims[n];
    for (int n = N - 1; n >= 0; --n) suf[n] = suf[n + 1] * t->dims[n];
    auto ldl = [](int64_t rows) { return (rows + 3) & ~int64_t(3); };   // 16-byte rows (tile over-reads of the
                                                                         // last row land in the next buffer)
    for (int k = 1; k <= (N == 1 ? 1 : N - 1); ++k) {
        // the left chain's partial products P_j (pre[j] x R_j, j = 1..k) alternate between Left and its
        // temporary so that P_k lands in Left; the right chain's Q_j (R_j x suf[j], j = N-1..k) likewise
        // plus the staged core of a build step (cores 2..N-1 as stored)
        int64_t lb = 0, t1 = 0, rb = N == 1 ? 1 : 0, t2 = 0, xs = 0;
        for (int b = 0; b < B; ++b) {
            for (int j = 1; j <= k; ++j) {   // P_j^T: R_j rows of ldl(pre[j]) floats
                const int64_t v = ldl(pre[j]) * h.rank(b, j);
                if ((k - j) % 2 == 0) lb = std::max(lb, v); else t1 = std::max(t1, v);
            }
            for (int j = k; j < N; ++j) {
                const int64_t v = suf[j] * h.rank(b, j);
                if ((j - k) % 2 == 0) rb = std::max(rb, v); else t2 = std::max(t2, v);
            }
            for (int j = 1; j < N - 1; ++j)
                xs = std::max(xs, (int64_t)t->dims[j] * h.rank(b, j) * h.rank(b, j + 1));
        }
        xs += 512 + 4;   // tile over-reads past the last buffer (4 rows x 128 threads) + 16-byte alignment
        auto r4 = [](int64_t v) { return (v + 3) & ~int64_t(3); };   // keep every buffer 16-byte aligned
        lb = r4(lb); t1 = r4(t1); rb = r4(rb); t2 = r4(t2);
        const int64_t bytes = 4 * (lb + t1 + rb + t2 + pre[k] + suf[k] + xs);
        if (bytes <= kSmemMax && (best_k < 0 || bytes < best)) {
            best_k = k; best = bytes; bl = lb; bt1 = t1; br = rb; bt2 = t2;
        }
    }
    // TTC_RECON_BIG=1 forces the workspace path (tests compare it with the shared-memory kernel)
    if (N == 1 && best_k < 0)
        return fail(TTC_ERR_UNSUPPORTED, "order-1 train of %d entries exceeds shared memory", t->dims[0]);
    if (best_k < 0 || (N > 1 && std::getenv("TTC_RECON_BIG"))) {
        ttc::ReconBigArgs a;
        std::memset(&a, 0, sizeof(a));
        ttc_status st2;
        if ((st2 = recon_big_plan(h, t, &a)) != TTC_OK) return st2;
        const int64_t need = 4 * (int64_t)B * (2 * a.ws_left + 2 * a.ws_right);
        if (query) {
            *query = need;
            return TTC_OK;
        }
        if (need > 0 && (!workspace_dev || workspace_bytes < need))
            return fail(TTC_ERR_ARG, "no split of the %d modes fits shared memory: the workspace path needs %lld bytes "
                        "(ttc_reconstruct_workspace), got %lld", N, (long long)need, (long long)workspace_bytes);
        if (reinterpret_cast<uintptr_t>(workspace_dev) & 15u) return fail(TTC_ERR_ALIGN, "workspace_dev not 16-byte aligned");
        a.row_fast = 0;
        for (int n = 0; n < a.k; ++n) a.row_fast |= ostride[n] == 1;
        for (int n = 0; n < N; ++n) a.ostride[n] = ostride[n];
        a.t = to_dev(h);
        a.out = out_dev;
        a.out_offsets = out_offsets_dev;
        a.pair_elems = pair_elems;
        a.ws = static_cast<float*>(workspace_dev);
        const cudaError_t e = ttc::launch_reconstruct_big(a, reinterpret_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return cuda_fail(e, "ttc_reconstruct launch");
        return TTC_OK;
    }
    if (query) return TTC_OK;
    ttc::ReconArgs a;
    std::memset(&a, 0, sizeof(a));
    a.B = B; a.N = N; a.k = best_k;
    a.rows = (int32_t)pre[best_k];
    a.cols = (int32_t)suf[best_k];
    a.lbuf = (int32_t)bl; a.t1 = (int32_t)bt1; a.rbuf = (int32_t)br; a.t2 = (int32_t)bt2;
    a.ldl = (int32_t)ldl(a.rows);
    // 16-byte output stores need the output's stride-1 mode to be the fastest row index: mode 1 as enumerated,
    // or the left block's last mode k with the rows enumerated big-endian
    {
        const int m1 = (perm ? perm[0] : 1) - 1;   // train mode with output stride 1
        a.lrev = (m1 != 0 && m1 == best_k - 1) ? 1 : 0;
    }
    for (int j = 0; j < best_k; ++j) a.ld[j] = (int32_t)ldl(pre[j + 1]);
    a.tm = (a.cols + 79) / 80 * 80 < (a.cols + 63) / 64 * 64 ? 5 : 4;   // 80 columns when that pads less
    for (int n = 0; n < N; ++n) { a.dims[n] = t->dims[n]; a.ostride[n] = ostride[n]; }
    a.t = to_dev(h);
    a.out = out_dev;
    a.out_offsets = out_offsets_dev;
    a.pair_elems = pair_elems;
    const cudaError_t e = ttc::launch_reconstruct(a, (size_t)best, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "ttc_reconstruct launch");
    return TTC_OK;
}

}  // namespace

ttc_status ttc_reconstruct(const ttc_tt_batch* t, const int32_t* perm, float* out_dev, const int64_t* out_offsets_dev,
                           void* stream) {
    return reconstruct_impl(t, perm, out_dev, out_offsets_dev, nullptr, 0, stream, nullptr);
}

ttc_status ttc_reconstruct_workspace(const ttc_tt_batch* t, const int32_t* perm, int64_t* workspace_bytes) {
    if (!workspace_bytes) return fail(TTC_ERR_NULL, "workspace_bytes is NULL");
    return reconstruct_impl(t, perm, nullptr, nullptr, nullptr, 0, nullptr, workspace_bytes);
}

ttc_status ttc_reconstruct_ws(const ttc_tt_batch* t, const int32_t* perm, float* out_dev, const int64_t* out_offsets_dev,
                              void* workspace_dev, int64_t workspace_bytes, void* stream) {
    return reconstruct_impl(t, perm, out_dev, out_offsets_dev, workspace_dev, workspace_bytes, stream, nullptr);
}

namespace {

// dims of X^rho and the source strides of its modes; the rank bounds and the capacity of one train
ttc_status ttsvd_shape(int32_t order, const int32_t* dims, const int32_t* perm, std::vector<int32_t>* rd,
                       std::vector<int64_t>* stride, int64_t* cap, int32_t* gmax) {
    if (order < 1 || order > TTC_MAX_ORDER) return fail(TTC_ERR_SHAPE, "order N = %d outside [1, %d]", order, TTC_MAX_ORDER);
    if (!dims) return fail(TTC_ERR_NULL, "dims is NULL");
    std::vector<int64_t> xs(order, 1);
    for (int n = 0; n < order; ++n) {
        if (dims[n] < 1) return fail(TTC_ERR_SHAPE, "mode %d has I = %d < 1", n + 1, dims[n]);
        if (n > 0) xs[n] = xs[n - 1] * dims[n - 1];
        if (xs[n] > (int64_t(1) << 40)) return fail(TTC_ERR_OVERFLOW, "dense size overflows");
    }
    rd->assign(order, 0);
    stride->assign(order, 0);
    std::vector<int> seen(order, 0);
    for (int k = 0; k < order; ++k) {
        const int m = perm ? perm[k] : k + 1;
        if (m < 1 || m > order || seen[m - 1])
            return fail(TTC_ERR_MODES, "perm[%d] = %d: perm must be a permutation of 1..%d", k, m, order);
        seen[m - 1] = 1;
        (*rd)[k] = dims[m - 1];
        (*stride)[k] = xs[m - 1];
    }
    int64_t total = 1;
    for (int k = 0; k < order; ++k)
        if (!mul_ok(total, (*rd)[k], &total) || total > (int64_t(1) << 40))
            return fail(TTC_ERR_OVERFLOW, "dense size overflows");
    // capacity: R_n <= min(prod_{k<=n} I_k, prod_{k>n} I_k); the Gram side of step n <= min(R_{n-1} I_n, rest)
    int64_t c = 0, left = 1, g = 1;
    int64_t Rprev = 1;
    for (int n = 0; n < order; ++n) {
        left *= (*rd)[n];
        const int64_t right = total / left;
        const int64_t Rn = n == order - 1 ? 1 : std::min(left, right);
        c += Rprev * (*rd)[n] * Rn;
        if (n < order - 1) g = std::max(g, std::min(Rprev * (*rd)[n], right));
        Rprev = Rn;
    }
    *cap = c;
    *gmax = (int32_t)g;
    // beyond the shared-memory kernels (16,384 elements, Gram side 64) the workspace-based one-sided Jacobi kernel
    // (ttsvd_big.cu) takes over, up to a side of kTtsvdBigMaxSide and 2^27 elements
    if (total > (int64_t(1) << 27))
        return fail(TTC_ERR_UNSUPPORTED, "tensor of %lld elements (> 2^27)", (long long)total);
    if (g > ttc::kTtsvdBigMaxSide)
        return fail(TTC_ERR_UNSUPPORTED, "an unfolding's smaller side is %lld > %d", (long long)g, ttc::kTtsvdBigMaxSide);
    return TTC_OK;
}

// TTC_TTSVD_BIG=1 forces the workspace kernel for every size (tests compare it with the shared-memory kernels)
bool ttsvd_needs_big(int64_t total, int32_t gmax) {
    return total > 16384 || gmax > 64 || std::getenv("TTC_TTSVD_BIG") != nullptr;
}

}  // namespace

ttc_status ttc_tt_svd_capacity(int32_t order, const int32_t* dims, const int32_t* perm, int64_t* train_cap) {
    g_last_error.clear();
    if (!train_cap) return fail(TTC_ERR_NULL, "train_cap is NULL");
    std::vector<int32_t> rd;
    std::vector<int64_t> st;
    int32_t g;
    return ttsvd_shape(order, dims, perm, &rd, &st, train_cap, &g);
}

namespace {
// Byte layout of the TT-SVD pipeline's workspace (ttsvd.cu TtsvdWs): Z_n, Gram, eigenvectors, eigenvalues, order,
// norms, each 256-byte aligned.  Returns the total.
int64_t ttsvd_ws_layout(int64_t B, int64_t elems, int64_t g, int64_t* off) {
    auto al = [](int64_t v) { return (v + 255) & ~int64_t(255); };
    const int64_t sz[6] = {4 * B * elems, 8 * B * g * g, 8 * B * g * g, 8 * B * g, 4 * B * g, 8 * B};
    int64_t o = 0;
    for (int k = 0; k < 6; ++k) { off[k] = o; o += al(sz[k]); }
    return o;
}
}  // namespace

ttc_status ttc_tt_svd_workspace(int32_t batch, int32_t order, const int32_t* dims, const int32_t* perm,
                                int64_t* workspace_bytes) {
    g_last_error.clear();
    if (!workspace_bytes) return fail(TTC_ERR_NULL, "workspace_bytes is NULL");
    if (batch < 0) return fail(TTC_ERR_ARG, "batch = %d < 0", batch);
    std::vector<int32_t> rd;
    std::vector<int64_t> st;
    int64_t cap;
    int32_t gmax;
    ttc_status s;
    if ((s = ttsvd_shape(order, dims, perm, &rd, &st, &cap, &gmax)) != TTC_OK) return s;
    int64_t total = 1, off[6];
    for (int n = 0; n < order; ++n) total *= rd[n];
    if (ttsvd_needs_big(total, gmax)) {
        *workspace_bytes = ttc::ttsvd_big_ws_bytes(batch, (int32_t)total, gmax);
        return TTC_OK;
    }
    *workspace_bytes = (order >= 2 && gmax <= 32) ? ttsvd_ws_layout(batch, total, gmax, off) : 0;
    return TTC_OK;
}

ttc_status ttc_tt_svd(int32_t batch, int32_t order, const int32_t* dims, const float* dense_dev, const int32_t* perm,
                      double eps, float* cores_dev, int32_t* ranks_dev, void* workspace_dev, int64_t workspace_bytes,
                      void* stream) {
    g_last_error.clear();
    if (batch < 0) return fail(TTC_ERR_ARG, "batch = %d < 0", batch);
    if (!(eps >= 0.0)) return fail(TTC_ERR_ARG, "eps = %g must be >= 0", eps);
    std::vector<int32_t> rd;
    std::vector<int64_t> st;
    int64_t cap;
    int32_t gmax;
    ttc_status s;
    if ((s = ttsvd_shape(order, dims, perm, &rd, &st, &cap, &gmax)) != TTC_OK) return s;
    if (batch == 0) return TTC_OK;
    if (!dense_dev || !cores_dev || !ranks_dev) return fail(TTC_ERR_NULL, "dense_dev / cores_dev / ranks_dev is NULL");
    if ((reinterpret_cast<uintptr_t>(dense_dev) | reinterpret_cast<uintptr_t>(cores_dev)) & 3u)
        return fail(TTC_ERR_ALIGN, "dense_dev / cores_dev not 4-byte aligned");
    if (reinterpret_cast<uintptr_t>(workspace_dev) & 15u) return fail(TTC_ERR_ALIGN, "workspace_dev not 16-byte aligned");
    ttc::TtsvdArgs a;
    std::memset(&a, 0, sizeof(a));
    a.B = batch; a.N = order; a.gmax = gmax;
    int64_t total = 1;
    for (int n = 0; n < order; ++n) { a.dims[n] = rd[n]; a.in_stride[n] = st[n]; total *= rd[n]; }
    a.elems = (int32_t)total;
    a.dense = dense_dev;
    a.eps2 = order > 1 ? eps * eps / (order - 1) : 0.0;
    a.cores = cores_dev;
    a.train_cap = cap;
    a.ranks = ranks_dev;
    const int64_t g = gmax;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (ttsvd_needs_big(total, gmax)) {   // one-sided Jacobi over the caller's fp64 workspace (ttsvd_big.cu)
        const int64_t need = ttc::ttsvd_big_ws_bytes(batch, (int32_t)total, gmax);
        if (!workspace_dev || workspace_bytes < need)
            return fail(TTC_ERR_ARG, "tensors of %lld elements (largest unfolding side %d) need a workspace of %lld bytes "
                        "(ttc_tt_svd_workspace), got %lld", (long long)total, gmax, (long long)need,
                        (long long)workspace_bytes);
        if (reinterpret_cast<uintptr_t>(workspace_dev) & 7u) return fail(TTC_ERR_ALIGN, "workspace_dev not 8-byte aligned");
        const cudaError_t e = ttc::launch_ttsvd_big(a, workspace_dev, cs);
        if (e != cudaSuccess) return cuda_fail(e, "ttc_tt_svd launch");
        return TTC_OK;
    }
    int64_t off[6];
    const int64_t need = (order >= 2 && gmax <= 32) ? ttsvd_ws_layout(batch, total, g, off) : 0;
    if (need > 0 && workspace_dev && workspace_bytes >= need && !std::getenv("TTC_TTSVD_FUSED")) {
        // warp-per-eigenproblem pipeline over the caller's workspace
        char* p = static_cast<char*>(workspace_dev);
        ttc::TtsvdWs w;
        w.z = reinterpret_cast<float*>(p + off[0]);
        w.g = reinterpret_cast<double*>(p + off[1]);
        w.v = reinterpret_cast<double*>(p + off[2]);
        w.lam = reinterpret_cast<double*>(p + off[3]);
        w.ord = reinterpret_cast<int32_t*>(p + off[4]);
        w.nrm = reinterpret_cast<double*>(p + off[5]);
        const cudaError_t e = ttc::launch_ttsvd_pipeline(a, w, cs);
        if (e != cudaSuccess) return cuda_fail(e, "ttc_tt_svd launch");
        return TTC_OK;
    }
    const size_t smem = sizeof(double) * (size_t)(2 * g * g + g + 2 * (g / 2 + 1) + 32) +
                        sizeof(int) * (size_t)(g + 2 * (g / 2 + 1) + 4) + 16 + sizeof(float) * 2 * (size_t)total;
    const cudaError_t e = ttc::launch_ttsvd(a, smem, cs);
    if (e != cudaSuccess) return cuda_fail(e, "ttc_tt_svd launch");
    return TTC_OK;
}

ttc_status ttc_pair_cost(const ttc_tt_batch* x, const ttc_tt_batch* y, double* mac, double* bytes) {
    g_last_error.clear();
    HostTrain hx, hy;
    ttc_status st;
    if ((st = check_batch(x, "X", TTC_MAX_ORDER, &hx)) != TTC_OK) return st;
    if ((st = check_batch(y, "Y", TTC_MAX_ORDER, &hy)) != TTC_OK) return st;
    if (x->batch != y->batch || x->order != y->order)
        return fail(TTC_ERR_SHAPE, "X (B=%d, N=%d) and Y (B=%d, N=%d) differ", x->batch, x->order, y->batch, y->order);
    for (int n = 0; n < x->order; ++n)
        if (x->dims[n] != y->dims[n])
            return fail(TTC_ERR_SHAPE, "X mode %d (I=%d) vs Y mode %d (J=%d)", n + 1, x->dims[n], n + 1, y->dims[n]);
    for (int b = 0; b < x->batch; ++b) {
        double m = 0.0, by = 4.0;
        for (int n = 0; n < x->order; ++n) {
            const double R = hx.rank(b, n), S = hx.rank(b, n + 1), P = hy.rank(b, n), Q = hy.rank(b, n + 1);
            const double I = x->dims[n];
            m += I * std::min(R * P * Q + R * S * Q, R * P * S + P * S * Q);
            by += 4.0 * I * (R * S + P * Q);
        }
        if (mac) mac[b] = m;
        if (bytes) bytes[b] = by;
    }
    return TTC_OK;
}

// Contiguous k-way split minimising the largest part: binary search on the bottleneck over prefix sums,
// then greedy fill (each part takes as many pairs as fit under the bottleneck).
ttc_status ttc_partition(const double* cost, int32_t B, int32_t k, int32_t* bounds) {
    g_last_error.clear();
    if (!bounds) return fail(TTC_ERR_NULL, "bounds is NULL");
    if (B < 0) return fail(TTC_ERR_ARG, "B = %d < 0", B);
    if (k < 1) return fail(TTC_ERR_ARG, "k = %d < 1", k);
    if (B > 0 && !cost) return fail(TTC_ERR_NULL, "cost is NULL");
    double total = 0.0, mx = 0.0;
    for (int b = 0; b < B; ++b) {
        if (!(cost[b] >= 0.0)) return fail(TTC_ERR_ARG, "cost[%d] = %g is negative or NaN", b, cost[b]);
        total += cost[b];
        mx = std::max(mx, cost[b]);
    }
    auto fill = [&](double cap, int32_t* out) -> bool {  // true if B pairs fit in k parts of <= cap
        int part = 0;
        double acc = 0.0;
        if (out) out[0] = 0;
        for (int b = 0; b < B; ++b) {
            if (acc + cost[b] > cap && acc > 0.0) {
                ++part;
                if (part >= k) return false;
                if (out) out[part] = b;
                acc = 0.0;
            }
            acc += cost[b];
        }
        if (out)
            for (int j = part + 1; j <= k; ++j) out[j] = B;
        return true;
    };
    if (B == 0 || total == 0.0) {   // equal counts
        for (int j = 0; j <= k; ++j) bounds[j] = (int32_t)(((int64_t)B * j) / k);
        return TTC_OK;
    }
    double lo = std::max(mx, total / k), hi = total;
    for (int it = 0; it < 100 && hi - lo > 1e-12 * total; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (fill(mid, nullptr)) hi = mid; else lo = mid;
    }
    fill(hi, bounds);
    // keep every part non-empty when B >= k (bounds strictly increasing)
    if (B >= k) {
        for (int j = k - 1; j >= 1; --j) bounds[j] = std::min(bounds[j], bounds[j + 1] - 1);
        for (int j = 1; j < k; ++j) bounds[j] = std::max(bounds[j], bounds[j - 1] + 1);
    }
    return TTC_OK;
}

}  // extern "C"

// ================================================================================================ contract
// Host-only plan for the ladder tt_contract (ttc.h; readings R7-R10).
struct ttc_contract_plan {
    int B = 0, N = 0, M = 0, K = 0, L = 0;
    std::vector<int32_t> xdims, ydims, xmodes, ymodes;
    std::vector<ttc::LadderEl> seq;
    std::vector<ttc::OutCore> outc;
    std::vector<int32_t> out_dims, out_src, out_perm;
    std::vector<int32_t> xranks, yranks;      // host copies [B*(N+1)], [B*(M+1)]
    std::vector<int32_t> out_ranks;           // [B*(L+1)]
    std::vector<int64_t> out_offsets;         // [B]
    int64_t total = 0;
    int32_t max_rank = 1;
    bool uniform_out = true;                  // every pair has the same output ranks
    int64_t scratch_floats = 0;               // per-CTA shared scratch for transfers: TL + TR + 3 tmp
    int64_t tl_floats = 0, tr_floats = 0, tmp_floats = 0;
    // TTCP splice of end modes (ttc_splice_plan_create): chain sources / reversal, K's absorption position
    bool splice = false;
    int sn = 0, sm = 0, nx = 0;
    std::vector<int32_t> sp_src, sp_rev;
    int64_t k_floats = 1;                     // largest K (Rk x Pk) over the batch
    bool rows_equal_x = true, rows_equal_y = true;   // every pair has the same rank row (per operand)
};

extern "C" {

ttc_status ttc_contract_plan_create(const ttc_tt_batch* x, const ttc_tt_batch* y, int32_t npairs,
                                    const int32_t* x_modes, const int32_t* y_modes, ttc_contract_plan** plan) {
    g_last_error.clear();
    if (!plan) return fail(TTC_ERR_NULL, "plan output pointer is NULL");
    *plan = nullptr;
    HostTrain hx, hy;
    ttc_status st;
    if ((st = check_batch(x, "X", ttc::kMaxContractOrder, &hx)) != TTC_OK) return st;
    if ((st = check_batch(y, "Y", ttc::kMaxContractOrder, &hy)) != TTC_OK) return st;
    if (x->batch != y->batch) return fail(TTC_ERR_SHAPE, "batch mismatch: X has %d trains, Y has %d", x->batch, y->batch);
    const int N = x->order, M = y->order, K = npairs;
    if (K < 0 || K > std::min(N, M)) return fail(TTC_ERR_MODES, "npairs = %d outside [0, min(N, M) = %d]", K, std::min(N, M));
    if (K > 0 && (!x_modes || !y_modes)) return fail(TTC_ERR_NULL, "x_modes / y_modes is NULL");
    for (int k = 0; k < K; ++k) {
        if (x_modes[k] < 1 || x_modes[k] > N) return fail(TTC_ERR_MODES, "pair %d: X mode %d outside [1, %d]", k + 1, x_modes[k], N);
        if (y_modes[k] < 1 || y_modes[k] > M) return fail(TTC_ERR_MODES, "pair %d: Y mode %d outside [1, %d]", k + 1, y_modes[k], M);
        if (k > 0 && (x_modes[k] <= x_modes[k - 1] || y_modes[k] <= y_modes[k - 1]))
            return fail(TTC_ERR_MODES, "pairs %d, %d: modes must be strictly increasing in both operands "
                        "(got X %d, %d and Y %d, %d)", k, k + 1, x_modes[k - 1], x_modes[k], y_modes[k - 1], y_modes[k]);
        if (x->dims[x_modes[k] - 1] != y->dims[y_modes[k] - 1])
            return fail(TTC_ERR_SHAPE, "X mode %d (I=%d) vs Y mode %d (J=%d)", x_modes[k], x->dims[x_modes[k] - 1],
                        y_modes[k], y->dims[y_modes[k] - 1]);
    }
    std::unique_ptr<ttc_contract_plan> p(new ttc_contract_plan());
    p->B = x->batch; p->N = N; p->M = M; p->K = K; p->L = N + M - 2 * K;
    p->xdims.assign(x->dims, x->dims + N);
    p->ydims.assign(y->dims, y->dims + M);
    p->xmodes.assign(x_modes, x_modes + K);
    p->ymodes.assign(y_modes, y_modes + K);
    // ladder sequence S (R7): per gap k, X free cores, then Y free cores, then transfer T_k
    for (int k = 1; k <= K + 1; ++k) {
        const int nprev = k == 1 ? 0 : x_modes[k - 2], mprev = k == 1 ? 0 : y_modes[k - 2];
        const int ncur = k <= K ? x_modes[k - 1] : N + 1, mcur = k <= K ? y_modes[k - 1] : M + 1;
        for (int n = nprev + 1; n < ncur; ++n) p->seq.push_back({ttc::EL_XFREE, n - 1, mprev});
        for (int m = mprev + 1; m < mcur; ++m) p->seq.push_back({ttc::EL_YFREE, m - 1, ncur - 1});
        if (k <= K) p->seq.push_back({ttc::EL_T, ncur - 1, mcur - 1});
    }
    // output cores with their absorbed transfers (R10: into the next core; trailing ones into the last core)
    int pend_first = -1, pend_count = 0;
    for (int e = 0; e < (int)p->seq.size(); ++e) {
        const auto& el = p->seq[e];
        if (el.kind == ttc::EL_T) {
            if (pend_count == 0) pend_first = e;
            ++pend_count;
            continue;
        }
        ttc::OutCore oc{e, pend_count ? pend_first : -1, pend_count, -1, 0};
        p->outc.push_back(oc);
        pend_first = -1; pend_count = 0;
        if (el.kind == ttc::EL_XFREE) { p->out_dims.push_back(x->dims[el.mode]); p->out_src.push_back(el.mode + 1); }
        else { p->out_dims.push_back(y->dims[el.mode]); p->out_src.push_back(-(el.mode + 1)); }
    }
    if (pend_count && !p->outc.empty()) { p->outc.back().rt_first = pend_first; p->outc.back().rt_count = pend_count; }
    // canonical order (Eq. 8): X free ascending, then Y free ascending -> ladder positions
    for (int n = 1; n <= N; ++n)
        for (int l = 0; l < p->L; ++l) if (p->out_src[l] == n) p->out_perm.push_back(l + 1);
    for (int m = 1; m <= M; ++m)
        for (int l = 0; l < p->L; ++l) if (p->out_src[l] == -m) p->out_perm.push_back(l + 1);
    // per-pair ranks, offsets, scratch
    const int B = p->B, L = p->L;
    p->xranks.resize((size_t)B * (N + 1));
    p->yranks.resize((size_t)B * (M + 1));
    for (int b = 0; b < B; ++b) {
        for (int n = 0; n <= N; ++n) p->xranks[(size_t)b * (N + 1) + n] = hx.rank(b, n);
        for (int m = 0; m <= M; ++m) p->yranks[(size_t)b * (M + 1) + m] = hy.rank(b, m);
    }
    p->out_ranks.assign((size_t)B * (L + 1), 1);
    p->out_offsets.assign(B, 0);
    int64_t off = 0;
    for (int b = 0; b < B; ++b) {
        const int32_t* xr = p->xranks.data() + (size_t)b * (N + 1);
        const int32_t* yr = p->yranks.data() + (size_t)b * (M + 1);
        int32_t* orr = p->out_ranks.data() + (size_t)b * (L + 1);
        for (int l = 0; l < L; ++l) {
            const auto& el = p->seq[p->outc[l].el];
            int64_t right = el.kind == ttc::EL_XFREE ? (int64_t)xr[el.mode + 1] * yr[el.hold]
                                                      : (int64_t)xr[el.hold] * yr[el.mode + 1];
            orr[l + 1] = (int32_t)right;
        }
        orr[L] = 1;
        if (L > 0) orr[0] = 1;
        int64_t pair_elems = 0;
        for (int l = 0; l < L; ++l) {
            int64_t c;
            if (!mul_ok((int64_t)orr[l] * p->out_dims[l], orr[l + 1], &c) || !add_ok(pair_elems, c, &pair_elems))
                return fail(TTC_ERR_OVERFLOW, "pair %d: output train size overflows int64", b);
            p->max_rank = std::max(p->max_rank, orr[l + 1]);
        }
        if (L == 0) pair_elems = 1;
        p->out_offsets[b] = off;
        if (!add_ok(off, pair_elems, &off)) return fail(TTC_ERR_OVERFLOW, "total output size overflows int64");
        // scratch: every transfer and chain product of this pair (rows*cols), two temporaries + TL + TR
        int64_t tmax = 0;
        for (const auto& el : p->seq)
            if (el.kind == ttc::EL_T) {
                const int64_t rows = (int64_t)xr[el.mode] * yr[el.hold], cols = (int64_t)xr[el.mode + 1] * yr[el.hold + 1];
                tmax = std::max(tmax, rows * cols);
            }
        // chain products have the rows of the first transfer and the cols of the current one
        for (const auto& oc : p->outc)
            for (int side = 0; side < 2; ++side) {
                const int f = side ? oc.rt_first : oc.lt_first, c = side ? oc.rt_count : oc.lt_count;
                if (c <= 0) continue;
                const auto& e0 = p->seq[f];
                const int64_t rows = (int64_t)xr[e0.mode] * yr[e0.hold];
                int64_t cm = 0;
                for (int t = 0; t < c; ++t) {
                    const auto& et = p->seq[f + t];
                    cm = std::max(cm, rows * (int64_t)xr[et.mode + 1] * yr[et.hold + 1]);
                }
                int64_t& dst = side ? p->tr_floats : p->tl_floats;
                dst = std::max(dst, cm);
                if (c > 1) p->tmp_floats = std::max(p->tmp_floats, std::max(tmax, cm));
            }
    }
    p->total = off;
    p->scratch_floats = p->tl_floats + p->tr_floats + 3 * p->tmp_floats;
    const int64_t scratch = p->scratch_floats;
    for (int b = 1; b < B && p->uniform_out; ++b)
        for (int l = 0; l <= L; ++l)
            if (p->out_ranks[(size_t)b * (L + 1) + l] != p->out_ranks[l]) { p->uniform_out = false; break; }
    if (L > 0 && scratch * (int64_t)sizeof(float) > 200 * 1024)
        return fail(TTC_ERR_UNSUPPORTED, "transfer scratch of %lld floats exceeds shared memory (ranks too large)",
                    (long long)scratch);
    for (int b = 1; b < p->B && p->rows_equal_x; ++b)
        p->rows_equal_x = std::equal(p->xranks.begin(), p->xranks.begin() + (p->N + 1), p->xranks.begin() + (size_t)b * (p->N + 1));
    for (int b = 1; b < p->B && p->rows_equal_y; ++b)
        p->rows_equal_y = std::equal(p->yranks.begin(), p->yranks.begin() + (p->M + 1), p->yranks.begin() + (size_t)b * (p->M + 1));
    *plan = p.release();
    return TTC_OK;
}

ttc_status ttc_splice_plan_create(const ttc_tt_batch* x, const ttc_tt_batch* y, int32_t x_mode, int32_t y_mode,
                                  ttc_contract_plan** plan) {
    g_last_error.clear();
    if (!plan) return fail(TTC_ERR_NULL, "plan output pointer is NULL");
    *plan = nullptr;
    HostTrain hx, hy;
    ttc_status st;
    if ((st = check_batch(x, "X", ttc::kMaxContractOrder, &hx, TTC_MAX_SPLICE_RANK)) != TTC_OK) return st;
    if ((st = check_batch(y, "Y", ttc::kMaxContractOrder, &hy, TTC_MAX_SPLICE_RANK)) != TTC_OK) return st;
    if (x->batch != y->batch) return fail(TTC_ERR_SHAPE, "batch mismatch: X has %d trains, Y has %d", x->batch, y->batch);
    const int N = x->order, M = y->order;
    if (x_mode != 1 && x_mode != N)
        return fail(TTC_ERR_MODES, "X mode %d is not an end mode (1 or %d): use ttc_contract_plan_create", x_mode, N);
    if (y_mode != 1 && y_mode != M)
        return fail(TTC_ERR_MODES, "Y mode %d is not an end mode (1 or %d): use ttc_contract_plan_create", y_mode, M);
    if (x->dims[x_mode - 1] != y->dims[y_mode - 1])
        return fail(TTC_ERR_SHAPE, "X mode %d (I=%d) vs Y mode %d (J=%d)", x_mode, x->dims[x_mode - 1], y_mode,
                    y->dims[y_mode - 1]);
    std::unique_ptr<ttc_contract_plan> p(new ttc_contract_plan());
    p->splice = true;
    p->sn = x_mode; p->sm = y_mode;
    p->B = x->batch; p->N = N; p->M = M; p->K = 1; p->L = N + M - 2;
    p->xdims.assign(x->dims, x->dims + N);
    p->ydims.assign(y->dims, y->dims + M);
    p->xmodes.assign(1, x_mode);
    p->ymodes.assign(1, y_mode);
    // chain (Alg. 2 step 5): X free cores (N..2 reversed when n = 1, else 1..N-1), then Y free cores
    if (x_mode == 1) for (int k = N; k >= 2; --k) { p->sp_src.push_back(k); p->sp_rev.push_back(1); }
    else for (int k = 1; k <= N - 1; ++k) { p->sp_src.push_back(k); p->sp_rev.push_back(0); }
    p->nx = (int)p->sp_src.size();
    if (y_mode == 1) for (int k = 2; k <= M; ++k) { p->sp_src.push_back(-k); p->sp_rev.push_back(0); }
    else for (int k = M - 1; k >= 1; --k) { p->sp_src.push_back(-k); p->sp_rev.push_back(1); }
    const int L = p->L;
    for (int l = 0; l < L; ++l) {
        const int sidx = p->sp_src[l];
        p->out_src.push_back(sidx);
        p->out_dims.push_back(sidx > 0 ? x->dims[sidx - 1] : y->dims[-sidx - 1]);
    }
    for (int n = 1; n <= N; ++n)
        for (int l = 0; l < L; ++l) if (p->out_src[l] == n) p->out_perm.push_back(l + 1);
    for (int m = 1; m <= M; ++m)
        for (int l = 0; l < L; ++l) if (p->out_src[l] == -m) p->out_perm.push_back(l + 1);
    const int B = p->B;
    p->xranks.resize((size_t)B * (N + 1));
    p->yranks.resize((size_t)B * (M + 1));
    p->out_ranks.assign((size_t)B * (L + 1), 1);
    p->out_offsets.assign(B, 0);
    int64_t off = 0;
    for (int b = 0; b < B; ++b) {
        for (int n = 0; n <= N; ++n) p->xranks[(size_t)b * (N + 1) + n] = hx.rank(b, n);
        for (int m = 0; m <= M; ++m) p->yranks[(size_t)b * (M + 1) + m] = hy.rank(b, m);
        const int32_t* xr = p->xranks.data() + (size_t)b * (N + 1);
        const int32_t* yr = p->yranks.data() + (size_t)b * (M + 1);
        const int64_t Rk = x_mode == 1 ? xr[1] : xr[N - 1], Pk = y_mode == 1 ? yr[1] : yr[M - 1];
        p->k_floats = std::max(p->k_floats, Rk * Pk);
        int32_t* orr = p->out_ranks.data() + (size_t)b * (L + 1);
        for (int l = 0; l < L; ++l) {   // right bond of chain core l (its left bond is the previous right bond)
            const int sidx = p->sp_src[l];
            const int32_t* rr = sidx > 0 ? xr : yr;
            const int k = (sidx > 0 ? sidx : -sidx) - 1;
            orr[l + 1] = p->sp_rev[l] ? rr[k] : rr[k + 1];
        }
        orr[0] = 1;
        if (L > 0) orr[L] = 1;
        int64_t pair_elems = 0;
        for (int l = 0; l < L; ++l) {
            int64_t cl;
            if (!mul_ok((int64_t)orr[l] * p->out_dims[l], orr[l + 1], &cl) || !add_ok(pair_elems, cl, &pair_elems))
                return fail(TTC_ERR_OVERFLOW, "pair %d: output train size overflows int64", b);
            p->max_rank = std::max(p->max_rank, orr[l + 1]);
        }
        if (L == 0) pair_elems = 1;
        p->out_offsets[b] = off;
        if (!add_ok(off, pair_elems, &off)) return fail(TTC_ERR_OVERFLOW, "total output size overflows int64");
    }
    p->total = off;
    for (int b = 1; b < B && p->uniform_out; ++b)
        for (int l = 0; l <= L; ++l)
            if (p->out_ranks[(size_t)b * (L + 1) + l] != p->out_ranks[l]) { p->uniform_out = false; break; }
    if (p->k_floats * (int64_t)sizeof(float) > 200 * 1024)
        return fail(TTC_ERR_UNSUPPORTED, "K of %lld floats exceeds shared memory (ranks too large)",
                    (long long)p->k_floats);
    for (int b = 0; b < B; ++b)   // the splice kernel indexes a core with 32-bit magic-number divisions
        for (int l = 0; l < L; ++l) {
            const int32_t* orr = p->out_ranks.data() + (size_t)b * (L + 1);
            if ((int64_t)orr[l] * p->out_dims[l] * orr[l + 1] >= (1 << 20) || p->out_dims[l] > 4096)
                return fail(TTC_ERR_UNSUPPORTED, "pair %d: output core %d of %lld elements (or I = %d) too large "
                            "for the splice kernel (< 2^20 elements, I <= 4096)", b, l + 1,
                            (long long)orr[l] * p->out_dims[l] * orr[l + 1], p->out_dims[l]);
        }
    for (int b = 1; b < p->B && p->rows_equal_x; ++b)
        p->rows_equal_x = std::equal(p->xranks.begin(), p->xranks.begin() + (p->N + 1), p->xranks.begin() + (size_t)b * (p->N + 1));
    for (int b = 1; b < p->B && p->rows_equal_y; ++b)
        p->rows_equal_y = std::equal(p->yranks.begin(), p->yranks.begin() + (p->M + 1), p->yranks.begin() + (size_t)b * (p->M + 1));
    *plan = p.release();
    return TTC_OK;
}

ttc_status ttc_contract_plan_query(const ttc_contract_plan* p, int32_t* out_order, int32_t* out_dims, int32_t* out_src,
                                   int32_t* out_perm, int64_t* total_elems, int32_t* max_rank) {
    g_last_error.clear();
    if (!p) return fail(TTC_ERR_NULL, "plan is NULL");
    if (out_order) *out_order = p->L;
    if (out_dims) std::copy(p->out_dims.begin(), p->out_dims.end(), out_dims);
    if (out_src) std::copy(p->out_src.begin(), p->out_src.end(), out_src);
    if (out_perm) std::copy(p->out_perm.begin(), p->out_perm.end(), out_perm);
    if (total_elems) *total_elems = p->total;
    if (max_rank) *max_rank = p->max_rank;
    return TTC_OK;
}

ttc_status ttc_contract_plan_layout(const ttc_contract_plan* p, int32_t* out_ranks_host, int64_t* out_offsets_host) {
    g_last_error.clear();
    if (!p) return fail(TTC_ERR_NULL, "plan is NULL");
    if (out_ranks_host) std::copy(p->out_ranks.begin(), p->out_ranks.end(), out_ranks_host);
    if (out_offsets_host) std::copy(p->out_offsets.begin(), p->out_offsets.end(), out_offsets_host);
    return TTC_OK;
}

void ttc_contract_plan_destroy(ttc_contract_plan* p) { delete p; }

ttc_status ttc_contract(const ttc_contract_plan* p, const ttc_tt_batch* x, const ttc_tt_batch* y, float* out_cores_dev,
                        const int64_t* out_offsets_dev, void* stream) {
    g_last_error.clear();
    if (!p) return fail(TTC_ERR_NULL, "plan is NULL");
    HostTrain hx, hy;
    ttc_status st;
    if ((st = check_batch(x, "X", ttc::kMaxContractOrder, &hx, p->splice ? TTC_MAX_SPLICE_RANK : TTC_MAX_RANK)) != TTC_OK) return st;
    if ((st = check_batch(y, "Y", ttc::kMaxContractOrder, &hy, p->splice ? TTC_MAX_SPLICE_RANK : TTC_MAX_RANK)) != TTC_OK) return st;
    if (x->batch != p->B || y->batch != p->B || x->order != p->N || y->order != p->M)
        return fail(TTC_ERR_SHAPE, "operands (B=%d/%d, N=%d, M=%d) differ from the plan (B=%d, N=%d, M=%d)", x->batch,
                    y->batch, x->order, y->order, p->B, p->N, p->M);
    for (int n = 0; n < p->N; ++n)
        if (x->dims[n] != p->xdims[n]) return fail(TTC_ERR_SHAPE, "X mode %d: I=%d differs from the plan (%d)", n + 1, x->dims[n], p->xdims[n]);
    for (int m = 0; m < p->M; ++m)
        if (y->dims[m] != p->ydims[m]) return fail(TTC_ERR_SHAPE, "Y mode %d: J=%d differs from the plan (%d)", m + 1, y->dims[m], p->ydims[m]);
    // the operands' ranks must be the plan's (uniform descriptors: compare the rank rows of one pair against
    // every stored row only when the plan saw different rows; explicit ranks: compare the arrays)
    auto same_ranks = [&](const HostTrain& h, const std::vector<int32_t>& pr, int n1, const char* nm) -> ttc_status {
        if (h.uniform) {
            const bool eq = (nm[0] == 'X') ? p->rows_equal_x : p->rows_equal_y;
            if (eq && p->B > 0) {   // the plan's rows are all equal: compare one row
                for (int n = 0; n < n1; ++n)
                    if (pr[n] != h.rank(0, n)) return fail(TTC_ERR_SHAPE, "%s: rank %d differs from the plan", nm, n);
                return TTC_OK;
            }
            for (int b = 0; b < p->B; ++b)
                for (int n = 0; n < n1; ++n)
                    if (pr[(size_t)b * n1 + n] != h.rank(0, n))
                        return fail(TTC_ERR_SHAPE, "%s pair %d: rank %d differs from the plan", nm, b, n);
            return TTC_OK;
        }
        if (std::memcmp(h.t->ranks_host, pr.data(), sizeof(int32_t) * pr.size()) != 0)
            for (int b = 0; b < p->B; ++b)
                for (int n = 0; n < n1; ++n)
                    if (h.t->ranks_host[(size_t)b * n1 + n] != pr[(size_t)b * n1 + n])
                        return fail(TTC_ERR_SHAPE, "%s pair %d: rank %d differs from the plan", nm, b, n);
        return TTC_OK;
    };
    if ((st = same_ranks(hx, p->xranks, p->N + 1, "X")) != TTC_OK) return st;
    if ((st = same_ranks(hy, p->yranks, p->M + 1, "Y")) != TTC_OK) return st;
    if (p->B == 0) return TTC_OK;
    if (!out_cores_dev) return fail(TTC_ERR_NULL, "out_cores_dev is NULL");
    if (reinterpret_cast<uintptr_t>(out_cores_dev) & 3u) return fail(TTC_ERR_ALIGN, "out_cores_dev not 4-byte aligned");
    if (!out_offsets_dev && !p->uniform_out)
        return fail(TTC_ERR_NULL, "pairs have different output ranks: out_offsets_dev is required");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (p->splice) {   // the paper's TTCP splice of end modes (splice.cu)
        ttc::SpliceArgs sa;
        std::memset(&sa, 0, sizeof(sa));
        sa.B = p->B; sa.N = p->N; sa.M = p->M; sa.L = p->L; sa.n = p->sn; sa.m = p->sm; sa.nx = p->nx;
        for (int n = 0; n < p->N; ++n) sa.xdims[n] = p->xdims[n];
        for (int m = 0; m < p->M; ++m) sa.ydims[m] = p->ydims[m];
        for (int l = 0; l < p->L; ++l) { sa.src[l] = p->sp_src[l]; sa.rev[l] = p->sp_rev[l]; }
        sa.x = to_dev(hx);
        sa.y = to_dev(hy);
        sa.out = out_cores_dev;
        sa.out_offsets = out_offsets_dev;
        sa.out_pair_elems = p->B ? p->total / p->B : 0;
        // whole trains staged in shared memory (one round trip for all of a pair's loads) when they fit
        auto max_elems = [](const HostTrain& h) {
            if (h.uniform) return h.train_elems_uniform;
            int64_t m = 0;
            for (const int64_t v : h.sizes) m = std::max(m, v);
            return m;
        };
        const int64_t sx = (max_elems(hx) + 3) & ~int64_t(3), sy = (max_elems(hy) + 3) & ~int64_t(3);
        sa.k4 = (int32_t)((p->k_floats + 3) & ~int64_t(3));
        size_t smem = sizeof(float) * (size_t)sa.k4;
        if (4 * (sx + sy) + smem <= 110 * 1024) {   // (2 CTAs per SM at the limit)
            sa.stage_x = (int32_t)sx;
            sa.stage_y = (int32_t)sy;
            smem += 4 * (size_t)(sx + sy);
        }
        e = ttc::launch_splice(sa, smem, s);
        if (e != cudaSuccess) return cuda_fail(e, "ttc_contract (splice) launch");
        return TTC_OK;
    }
    if (p->L == 0) {   // every mode contracted: the scalar <X_b, Y_b>, one float per pair (packed)
        const ttc_status r = ttc_inner(x, y, out_cores_dev, stream);
        return r;
    }
    ttc::ContractArgs a;
    std::memset(&a, 0, sizeof(a));
    a.B = p->B; a.N = p->N; a.M = p->M; a.K = p->K; a.L = p->L; a.nseq = (int)p->seq.size();
    for (int n = 0; n < p->N; ++n) a.xdims[n] = p->xdims[n];
    for (int m = 0; m < p->M; ++m) a.ydims[m] = p->ydims[m];
    for (int i = 0; i < a.nseq; ++i) a.seq[i] = p->seq[i];
    for (int l = 0; l < p->L; ++l) a.outc[l] = p->outc[l];
    a.x = to_dev(hx);
    a.y = to_dev(hy);
    a.out = out_cores_dev;
    a.out_offsets = out_offsets_dev;
    a.out_pair_elems = p->B ? p->total / p->B : 0;
    a.tl_off = 0;
    a.tr_off = (int32_t)p->tl_floats;
    a.tmp_off = (int32_t)(p->tl_floats + p->tr_floats);
    a.tmp_size = (int32_t)p->tmp_floats;
    // stage both trains of a pair in shared memory when the largest pair fits 40 KB
    int64_t max_train = 0;
    for (int b = 0; b < p->B; ++b) {
        int64_t tx = 0, ty = 0;
        for (int n = 0; n < p->N; ++n) tx += (int64_t)p->xranks[(size_t)b * (p->N + 1) + n] * p->xdims[n] * p->xranks[(size_t)b * (p->N + 1) + n + 1];
        for (int m = 0; m < p->M; ++m) ty += (int64_t)p->yranks[(size_t)b * (p->M + 1) + m] * p->ydims[m] * p->yranks[(size_t)b * (p->M + 1) + m + 1];
        max_train = std::max(max_train, tx + ty);
    }
    a.stage_off = (int32_t)p->scratch_floats;
    a.stage_floats = max_train <= 10240 ? (int32_t)max_train : 0;
    {   // stage only when transfer scratch + staged trains + the kernel's static shared memory fit one block
        int dev = 0, optin = 0;
        cudaFuncAttributes fa;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
        if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess)
            return cuda_fail(e, "cudaDeviceGetAttribute");
        if ((e = ttc::contract_func_attributes(&fa)) != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes");
        const int64_t need = 4 * (p->scratch_floats + a.stage_floats) + (int64_t)fa.sharedSizeBytes;
        if (need > optin) a.stage_floats = 0;
    }
    e = ttc::launch_contract(a, sizeof(float) * ((size_t)p->scratch_floats + (size_t)a.stage_floats), s);
    if (e != cudaSuccess) return cuda_fail(e, "ttc_contract launch");
    return TTC_OK;
}

}  // extern "C"
