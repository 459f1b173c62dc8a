// LDS.128 / LDS.64 wavefronts per instruction for lane -> address patterns (profile with ncu:
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum / smsp__inst_executed_op_shared_ld.sum).
// Usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_bench tools/lds_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT, int VEC>
__global__ void lds_kernel(float* out, int iters) {
    __shared__ __align__(16) float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (float)i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int idx;   // 16-byte slot index
    switch (PAT) {
        case 0: idx = lane; break;                 // 32 distinct, consecutive
        case 1: idx = lane >> 2; break;            // 8 distinct, 4 consecutive lanes share (2 per quarter)
        case 2: idx = lane & 3; break;             // 4 distinct, quarters identical
        case 3: idx = lane & 7; break;             // 8 distinct, quarters identical
        case 4: idx = lane >> 3; break;            // 4 distinct, one per quarter
        case 5: idx = 0; break;                    // broadcast
        case 6: idx = (lane & 7) + 8 * (lane >> 4); break;   // 16 distinct, half-warps differ
        case 7: idx = (lane >> 3) * 9; break;      // 4 distinct, one per quarter, spread banks
        case 8: idx = (lane >> 1) & 7; break;      // 8 distinct, pairs of lanes share
        case 9: idx = (lane & 1) + 2 * (lane >> 4); break;   // 4 distinct: 2 alternating per half
        case 10: idx = lane & 1; break;            // 2 distinct, alternating
        case 11: idx = lane >> 1; break;           // 16 distinct, pairs share
        case 12: idx = (lane & 3) + 4 * (lane >> 4); break;  // 8 distinct: 4 strided per half
        case 13: idx = (lane >> 2) & 3; break;     // 4 distinct, 4 consecutive share, halves identical
        case 14: idx = (lane & 1) | ((lane >> 3) << 1); break;   // 8 distinct: alternating pairs per quarter
        case 15: idx = (lane >> 1) & 3; break;     // 4 distinct, pairs share, quarters identical
        case 16: idx = 2 * lane; break;            // 32 distinct, 32-byte stride
        default: idx = (lane & 1) | ((lane >> 2) << 1); break;   // 16 distinct: alternating, quad steps
    }
    float acc = 0.f;
    const float* p = s + 4 * idx;
    for (int it = 0; it < iters; ++it) {
        const unsigned a = (unsigned)__cvta_generic_to_shared(p + (it & 1) * 256);
        if (VEC == 4) {
            float x, y, z, w;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
            acc += x + y + z + w;
        } else {
            float x, y;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
            acc += x + y;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 256 * sizeof(float));
#define RUN(P, V) lds_kernel<P, V><<<148, 256>>>(out, 1000);
    RUN(0, 4) RUN(1, 4) RUN(2, 4) RUN(3, 4) RUN(4, 4) RUN(5, 4) RUN(6, 4) RUN(7, 4)
    RUN(8, 4) RUN(9, 4) RUN(10, 4) RUN(11, 4) RUN(12, 4) RUN(13, 4) RUN(14, 4) RUN(15, 4) RUN(16, 4) RUN(17, 4)
    RUN(0, 2) RUN(1, 2) RUN(2, 2) RUN(3, 2) RUN(4, 2) RUN(5, 2) RUN(6, 2) RUN(7, 2)
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
