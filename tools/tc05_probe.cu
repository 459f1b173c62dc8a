// tc05_probe.cu -- on-box probe of tcgen05.mma kind::tf32 (SURVEY.md:132 / 282-285: "picked by on-box
// microbenchmark"): (1) operand layout / descriptor / TMEM-layout check and how fp32 inputs are reduced to tf32
// (truncation vs round-to-nearest), (2) precision of long accumulation chains in TMEM, (3) issue throughput of
// M64/M128 x N64/N256 x K8 MMAs from shared memory, (4) the same for legacy mma.sync m16n8k8 tf32.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc05_probe tools/tc05_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major SWIZZLE_128B tile of `rows` x 32 fp32 (one 128-byte swizzle atom column); element (r, k) byte offset
__host__ __device__ __forceinline__ uint32_t sw128_off(int r, int k) {
    return (uint32_t)(r * 128 + ((((k >> 2) ^ (r & 7)) & 7) << 4) + ((k & 3) << 2));
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B (8-row groups), version 1 (sm_100)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);
    d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major), 16 B
    d |= (uint64_t)(1024 >> 4) << 32;             // SBO
    d |= (uint64_t)1 << 46;                       // version
    d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
    return d;
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
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}\n"
                 :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// D[m][n] = sum over `chain` repetitions of sum_k A[m][k] B[n][k] (A: 64 or 128 rows x 32 K, B: N rows x 32 K,
// both K-major SW128), 4 MMAs (K = 8 each) per repetition, all accumulated in one TMEM tile.  D to global
// [M][N] fp32.  Also times `timed` extra MMAs (clock64 between the first issue and the commit's arrival).
template <int M, int N>
__global__ void probe_kernel(const float* A, const float* B, float* D, int chain, int timed, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    unsigned char* sa = base;
    unsigned char* sb = base + M * 128;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int e = tid; e < M * 32; e += blockDim.x) *(float*)(sa + sw128_off(e / 32, e % 32)) = A[e];
    for (int e = tid; e < N * 32; e += blockDim.x) *(float*)(sb + sw128_off(e / 32, e % 32)) = B[e];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t dt = tbase;
    const uint32_t idesc = idesc_tf32(M, N);
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        const uint64_t ad = desc_sw128(smem_u32(sa)), bd = desc_sw128(smem_u32(sb));
        for (int c = 0; c < chain; ++c)
            for (int k = 0; k < 4; ++k) mma_tf32(dt, ad + 2 * k, bd + 2 * k, idesc, (c | k) ? 1u : 0u);   // +32 B
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        if (timed > 0) {
            t0 = clock64();
            for (int c = 0; c < timed; ++c) mma_tf32(dt + 256, ad + 2 * (c & 3), bd + 2 * (c & 3), idesc, 1u);
            mma_commit(&bar);
            mbar_wait(&bar, 1);
            t1 = clock64();
            cycles[0] = t1 - t0;
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // D: M = 128 -> row m at lane m; M = 64 -> row m at lane (m % 16) + 32 (m / 16)
    const int lane_base = 32 * (warp & 3);
    const int t = tid & 31;
    int row = -1;
    if (M == 128) row = lane_base + t;
    else if (t < 16) row = 16 * (warp & 3) + t;
    if (warp < 4) {
        for (int c0 = 0; c0 < N; c0 += 16) {
            float v[16];
            tmem_ld16(dt + ((uint32_t)lane_base << 16) + c0, v);
            if (row >= 0)
                for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(dt), "r"(512));
}

// legacy mma.sync m16n8k8 tf32 issue throughput: one warp, `n` independent-accumulator MMAs
__global__ void hmma_kernel(int n, float* sink, long long* cycles) {
    float d[4][4] = {};
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u}, b0 = threadIdx.x, b1 = 5u;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x * 8 + threadIdx.x / 32] = t1 - t0;
    float s = 0;
    for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }
static float rn_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }

template <int M, int N>
void run(int chain, int timed, bool exact_inputs, unsigned seed) {
    std::vector<float> A(M * 32), B(N * 32), D(M * N);
    srand(seed);
    for (auto& x : A) { float v = (rand() / (float)RAND_MAX - 0.5f) * powf(2.f, (float)(rand() % 9 - 4)); x = exact_inputs ? trunc_tf32(v) : v; }
    for (auto& x : B) { float v = (rand() / (float)RAND_MAX - 0.5f) * powf(2.f, (float)(rand() % 9 - 4)); x = exact_inputs ? trunc_tf32(v) : v; }
    float *dA, *dB, *dD; long long* dc;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 64));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const size_t smem = 1024 + (M + N) * 128;
    CK(cudaFuncSetAttribute(probe_kernel<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    probe_kernel<M, N><<<1, 128, smem>>>(dA, dB, dD, chain, timed, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    long long cyc = 0;
    if (timed) CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    // references: exact (double) of truncated inputs, of RN inputs, and fp32 sequential RN accumulation
    double e_tr = 0, e_rn = 0, e_f32 = 0, mx = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double st = 0, sr = 0; float sf = 0.f;
            for (int c = 0; c < chain; ++c)
                for (int k = 0; k < 32; ++k) {
                    st += (double)trunc_tf32(A[m * 32 + k]) * trunc_tf32(B[n * 32 + k]);
                    sr += (double)rn_tf32(A[m * 32 + k]) * rn_tf32(B[n * 32 + k]);
                    sf = fmaf(trunc_tf32(A[m * 32 + k]), trunc_tf32(B[n * 32 + k]), sf);
                }
            const double g = D[m * N + n];
            e_tr = fmax(e_tr, fabs(g - st)); e_rn = fmax(e_rn, fabs(g - sr)); e_f32 = fmax(e_f32, fabs((double)sf - st));
            mx = fmax(mx, fabs(st));
        }
    printf("M=%d N=%d chain=%d (%d MMAs/output) exact_in=%d: max|D-ref_trunc|=%.3e  max|D-ref_rn|=%.3e  "
           "(fp32 RN sequential accumulation error %.3e; max|ref| %.3e)", M, N, chain, 4 * chain, (int)exact_inputs,
           e_tr, e_rn, e_f32, mx);
    if (timed) printf("  timed %d MMAs: %lld cycles = %.1f cyc/MMA", timed, cyc, (double)cyc / timed);
    printf("\n");
    CK(cudaFree(dA)); CK(cudaFree(dB)); CK(cudaFree(dD)); CK(cudaFree(dc));
}

// accumulation rounding mode: all-positive tf32-exact inputs (no cancellation), mean signed relative error of D
// against the exact sum, next to fp32 models of the chain (K = 8 partial sums added with RN or with RZ)
static float rz_add(float a, double b) {   // a + b truncated toward zero to fp32
    double s = (double)a + b;
    float f = (float)s;
    if (fabs((double)f) > fabs(s)) f = nextafterf(f, 0.f);
    return f;
}
template <int M, int N>
void bias(int chain) {
    std::vector<float> A(M * 32), B(N * 32), D(M * N);
    srand(77 + chain);
    for (auto& x : A) x = trunc_tf32(0.5f + 0.5f * rand() / (float)RAND_MAX);
    for (auto& x : B) x = trunc_tf32(0.5f + 0.5f * rand() / (float)RAND_MAX);
    float *dA, *dB, *dD; long long* dc;
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 64));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const size_t smem = 1024 + (M + N) * 128;
    CK(cudaFuncSetAttribute(probe_kernel<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    probe_kernel<M, N><<<1, 128, smem>>>(dA, dB, dD, chain, 0, dc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double mg = 0, mrn = 0, mrz = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double ex = 0; float rn = 0.f, rz = 0.f;
            for (int c = 0; c < chain; ++c)
                for (int kb = 0; kb < 4; ++kb) {
                    double part = 0;
                    for (int k = 8 * kb; k < 8 * kb + 8; ++k) part += (double)A[m * 32 + k] * B[n * 32 + k];
                    ex += part;
                    rn = (float)((double)rn + part);
                    rz = rz_add(rz, part);
                }
            mg += (D[m * N + n] - ex) / ex; mrn += (rn - ex) / ex; mrz += (rz - ex) / ex;
        }
    const double cnt = (double)M * N;
    printf("bias M=%d N=%d %4d accumulations: mean rel err GPU %+.3e | model RN %+.3e | model RZ %+.3e\n", M, N, 4 * chain,
           mg / cnt, mrn / cnt, mrz / cnt);
    CK(cudaFree(dA)); CK(cudaFree(dB)); CK(cudaFree(dD)); CK(cudaFree(dc));
}

int main() {
    for (int ch : {1, 4, 16, 64}) bias<64, 64>(ch);
    bias<128, 64>(16);
    // (1) layout + input reduction (one chain of 4 MMAs, K = 32)
    run<64, 64>(1, 0, false, 1);
    run<128, 64>(1, 0, false, 2);
    run<64, 256>(1, 0, false, 3);
    run<128, 256>(1, 0, false, 4);
    // (2) accumulation precision: tf32-exact inputs, long chains in one TMEM accumulator
    run<64, 64>(1, 0, true, 5);
    run<64, 64>(8, 0, true, 6);
    run<64, 64>(24, 0, true, 7);
    run<128, 64>(24, 0, true, 8);
    // (3) issue throughput
    run<64, 64>(1, 1024, false, 9);
    run<128, 64>(1, 1024, false, 10);
    run<64, 128>(1, 1024, false, 11);
    run<128, 128>(1, 1024, false, 12);
    run<64, 256>(1, 1024, false, 13);
    run<128, 256>(1, 1024, false, 14);
    // (4) legacy mma.sync tf32: 4 warps x 4 independent accumulators
    {
        float* sink; long long* c;
        CK(cudaMalloc(&sink, 148 * 128 * 4)); CK(cudaMalloc(&c, 148 * 8 * 8));
        hmma_kernel<<<1, 128>>>(4096, sink, c);
        CK(cudaDeviceSynchronize());
        long long cyc; CK(cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost));
        printf("mma.sync m16n8k8 tf32: 4 warps x %d MMAs: %lld cycles per warp -> %.2f cyc per warp-MMA (%.0f MAC/cyc/SM)\n",
               4 * 4096, cyc, cyc / (4.0 * 4096), 4 * 4 * 4096 * 1024.0 / cyc);
    }
    return 0;
}
