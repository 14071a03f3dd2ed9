// Check packed fp32x2 add/sub/mul/fma against the scalar .rn ops on random bit patterns.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }
__device__ float rf(uint32_t s, int mode) {
  uint32_t b = hsh(s);
  if (mode == 0) { // normal range around 1e-3..1e4
    float f = __uint_as_float((b & 0x807FFFFFu) | ((uint32_t)(117 + (hsh(s ^ 0x9e37) % 24)) << 23));
    return f;
  }
  return __uint_as_float(b);  // any pattern (incl. subnormal, inf, nan)
}
__global__ void k(unsigned long long n, int mode, unsigned long long* bad, unsigned* ex) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
    const float a0 = rf(4 * i, mode), a1 = rf(4 * i + 1, mode), b0 = rf(4 * i + 2, mode), b1 = rf(4 * i + 3, mode);
    const float c0 = rf(7 * i + 5, mode), c1 = rf(7 * i + 6, mode);
    unsigned long long A, B, C, R;
    asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b0), "f"(b1));
    asm("mov.b64 %0, {%1,%2};" : "=l"(C) : "f"(c0), "f"(c1));
    float r0, r1;
    // add
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r0), "=f"(r1) : "l"(R));
    float s0 = __fadd_rn(a0, b0), s1 = __fadd_rn(a1, b1);
    if ((__float_as_uint(r0) != __float_as_uint(s0) && !(isnan(r0) && isnan(s0))) || (__float_as_uint(r1) != __float_as_uint(s1) && !(isnan(r1) && isnan(s1)))) { if (atomicAdd(&bad[0], 1) < 4) { ex[0] = __float_as_uint(a0); ex[1] = __float_as_uint(b0); ex[2] = __float_as_uint(r0); ex[3] = __float_as_uint(s0);} }
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r0), "=f"(r1) : "l"(R));
    s0 = __fsub_rn(a0, b0); s1 = __fsub_rn(a1, b1);
    if ((__float_as_uint(r0) != __float_as_uint(s0) && !(isnan(r0) && isnan(s0))) || (__float_as_uint(r1) != __float_as_uint(s1) && !(isnan(r1) && isnan(s1)))) { if (atomicAdd(&bad[1], 1) < 4) { ex[4] = __float_as_uint(a0); ex[5] = __float_as_uint(b0); ex[6] = __float_as_uint(r0); ex[7] = __float_as_uint(s0);} }
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r0), "=f"(r1) : "l"(R));
    s0 = __fmul_rn(a0, b0); s1 = __fmul_rn(a1, b1);
    if ((__float_as_uint(r0) != __float_as_uint(s0) && !(isnan(r0) && isnan(s0))) || (__float_as_uint(r1) != __float_as_uint(s1) && !(isnan(r1) && isnan(s1)))) { if (atomicAdd(&bad[2], 1) < 4) { ex[8] = __float_as_uint(a0); ex[9] = __float_as_uint(b0); ex[10] = __float_as_uint(r0); ex[11] = __float_as_uint(s0);} }
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(R) : "l"(A), "l"(B), "l"(C));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r0), "=f"(r1) : "l"(R));
    s0 = __fmaf_rn(a0, b0, c0); s1 = __fmaf_rn(a1, b1, c1);
    if ((__float_as_uint(r0) != __float_as_uint(s0) && !(isnan(r0) && isnan(s0))) || (__float_as_uint(r1) != __float_as_uint(s1) && !(isnan(r1) && isnan(s1)))) { if (atomicAdd(&bad[3], 1) < 4) { ex[12] = __float_as_uint(a0); ex[13] = __float_as_uint(b0); ex[14] = __float_as_uint(r0); ex[15] = __float_as_uint(s0);} }
  }
}
int main() {
  unsigned long long* bad; unsigned* ex;
  cudaMallocManaged(&bad, 64); cudaMallocManaged(&ex, 64 * 4);
  for (int mode = 0; mode < 2; ++mode) {
    for (int q = 0; q < 8; ++q) bad[q] = 0;
    for (int q = 0; q < 16; ++q) ex[q] = 0;
    k<<<148 * 8, 256>>>(1ull << 30, mode, bad, ex);
    cudaDeviceSynchronize();
    printf("mode %d (%s): mismatches add %llu sub %llu mul %llu fma %llu of 2^31 each\n", mode, mode ? "any bits" : "normal", bad[0], bad[1], bad[2], bad[3]);
    for (int q = 0; q < 4; ++q) if (bad[q]) printf("  op %d example a=%08x b=%08x packed=%08x scalar=%08x\n", q, ex[4*q], ex[4*q+1], ex[4*q+2], ex[4*q+3]);
  }
  return 0;
}
