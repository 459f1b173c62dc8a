// tc_common.cuh -- PTX helpers shared by the tensor-core tt_inner kernels (inner_fast.cu, inner_r16.cu):
// mbarriers, TMA bulk copies, and the 3xTF32 split / mma.sync m16n8k8 building blocks.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ttc {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// TMA tensor copies (cp.async.bulk.tensor, tile mode) into this CTA's shared memory, completing on `bar`;
// m: the CUtensorMap (__grid_constant__ parameter, constant or global memory)
__device__ __forceinline__ void tma_2d(void* dst, const void* m, int c0, int c1, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const void* m, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most `pending` of this thread's newest cp.async groups are still in flight
__device__ __forceinline__ void cp_wait_pending(int pending) {
    switch (pending) {
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
    }
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// 3xTF32 split without the (emulated) cvt.rna.tf32: hi = x rounded to nearest at mantissa bit 13 by an
// integer add + mask (finite inputs), lo = x - hi exactly in fp32; the tensor core reads only the top 19
// bits of lo (truncation), which keeps |x - hi - lo_tf32| <= 2^-22 |x|.
__device__ __forceinline__ uint32_t hi_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xffffe000u; }
__device__ __forceinline__ uint32_t lo_bits(float x, uint32_t hi) { return __float_as_uint(x - __uint_as_float(hi)); }

__device__ __forceinline__ void mma_acc(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_zero(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};\n"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.0f));
}

struct AFrag {
    uint32_t hi[4], lo[4];
};
struct BFrag {
    uint32_t hi[2], lo[2];
};
__device__ __forceinline__ AFrag split_a(const float (&a)[4]) {
    AFrag f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f.hi[k] = hi_bits(a[k]);
        f.lo[k] = lo_bits(a[k], f.hi[k]);
    }
    return f;
}
__device__ __forceinline__ BFrag split_b(float b0, float b1) {
    BFrag f;
    f.hi[0] = hi_bits(b0);
    f.lo[0] = lo_bits(b0, f.hi[0]);
    f.hi[1] = hi_bits(b1);
    f.lo[1] = lo_bits(b1, f.hi[1]);
    return f;
}
// d += A * B in 3xTF32 (A_lo B_hi + A_hi B_lo + A_hi B_hi): the group starts from zero in the tensor core
// and is added to d with a round-to-nearest FADD, so the truncating internal accumulation never spans
// more than one group.
__device__ __forceinline__ void mma3_add(float (&d)[4], const AFrag& A, const BFrag& B) {
    float tmp[4];
    mma_zero(tmp, A.lo, B.hi[0], B.hi[1]);
    mma_acc(tmp, A.hi, B.lo[0], B.lo[1]);
    mma_acc(tmp, A.hi, B.hi[0], B.hi[1]);
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] += tmp[k];
}


// A operand split by truncation (its fp32 bits are the hi part as the tensor core reads them):
// hi = top 19 bits of x, lo = x - hi (exact), |x - hi - lo_tf32| <= 2^-20 |x|.  2 instructions per element.
__device__ __forceinline__ AFrag split_a_trunc(const float (&a)[4]) {
    AFrag f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f.hi[k] = __float_as_uint(a[k]);
        f.lo[k] = __float_as_uint(a[k] - __uint_as_float(f.hi[k] & 0xffffe000u));
    }
    return f;
}
// d (=) or (+=) A * B, 3xTF32 inside the tensor core (A_lo B_hi + A_hi B_lo + A_hi B_hi)
template <bool FIRST>
__device__ __forceinline__ void mma3(float (&d)[4], const AFrag& A, const BFrag& B) {
    if (FIRST) mma_zero(d, A.lo, B.hi[0], B.hi[1]);
    else mma_acc(d, A.lo, B.hi[0], B.hi[1]);
    mma_acc(d, A.hi, B.lo[0], B.lo[1]);
    mma_acc(d, A.hi, B.hi[0], B.hi[1]);
}

// d (=) A0 B0 + A1 B1 over two k8 blocks, 3xTF32, ordered so the four small cross terms accumulate first
// and the two large hi*hi products last: the tensor core's truncating accumulation then loses at most two
// large-magnitude roundings per group.
template <bool FIRST>
__device__ __forceinline__ void mma6(float (&d)[4], const AFrag& A0, const BFrag& B0, const AFrag& A1, const BFrag& B1) {
    if (FIRST) mma_zero(d, A0.lo, B0.hi[0], B0.hi[1]);
    else mma_acc(d, A0.lo, B0.hi[0], B0.hi[1]);
    mma_acc(d, A0.hi, B0.lo[0], B0.lo[1]);
    mma_acc(d, A1.lo, B1.hi[0], B1.hi[1]);
    mma_acc(d, A1.hi, B1.lo[0], B1.lo[1]);
    mma_acc(d, A0.hi, B0.hi[0], B0.hi[1]);
    mma_acc(d, A1.hi, B1.hi[0], B1.hi[1]);
}

__host__ __device__ __forceinline__ int plane_stride(int floats) {   // >= floats, multiple of 4, = 8 mod 32
    int ps = (floats + 3) & ~3;
    ps += (8 - (ps & 31) + 32) & 31;
    return ps;
}

__device__ __forceinline__ void bar_named(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace tc
}  // namespace ttc
