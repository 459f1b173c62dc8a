// tf32_probe.cu -- how mma.sync tf32 reads a raw fp32 register: truncation or rounding of the low 13 bits?
#include <cstdio>
#include <cstdint>
#include <cstring>
__global__ void k(const float* x, float* out) {
    // A (16x8) row g: a0 = A[g][t] = x[g*4+t] for row g<8, zeros elsewhere; B = identity-ish: B[k][n] = (k == n)
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    float a0 = x[g * 4 + t], a1 = 0.f, a2 = 0.f, a3 = 0.f;
    float b0 = (t == g) ? 1.f : 0.f, b1 = 0.f;
    float d[4] = {0, 0, 0, 0};
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(__float_as_uint(a0)), "r"(__float_as_uint(a1)), "r"(__float_as_uint(a2)), "r"(__float_as_uint(a3)),
                   "r"(__float_as_uint(b0)), "r"(__float_as_uint(b1)));
    // C[g][2t], C[g][2t+1] = sum_k A[g][k] B[k][n] = A[g][n] for n < 4
    out[g * 8 + 2 * t] = d[0];
    out[g * 8 + 2 * t + 1] = d[1];
}
int main() {
    float hx[32], *dx, *dout, hout[64];
    for (int i = 0; i < 32; ++i) {
        uint32_t u = 0x3f800000u | (uint32_t)(0x1000 + 0x0fff * (i & 1) + 0x400 * (i % 5));  // low bits near / above half
        memcpy(&hx[i], &u, 4);
    }
    cudaMalloc(&dx, sizeof hx); cudaMalloc(&dout, sizeof hout);
    cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dx, dout);
    cudaMemcpy(hout, dout, sizeof hout, cudaMemcpyDeviceToHost);
    int trunc_ok = 0, rn_ok = 0, n = 0;
    for (int g = 0; g < 8; ++g)
        for (int c = 0; c < 4; ++c) {
            float x = hx[g * 4 + c], y = hout[g * 8 + c];
            uint32_t u; memcpy(&u, &x, 4);
            uint32_t tr = u & 0xffffe000u, rn = (u + 0x1000u) & 0xffffe000u;
            float ft, fr; memcpy(&ft, &tr, 4); memcpy(&fr, &rn, 4);
            trunc_ok += (y == ft); rn_ok += (y == fr); ++n;
        }
    printf("{\"samples\": %d, \"matches_truncation\": %d, \"matches_round_nearest\": %d}\n", n, trunc_ok, rn_ok);
    return 0;
}
