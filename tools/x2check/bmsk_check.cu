#include <cstdio>
__device__ __forceinline__ unsigned bmsk32(int pos, int len) { unsigned r; asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(r) : "r"(pos), "r"(len)); return r; }
__global__ void k(int* bad) {
  for (int a = 0; a < 64; ++a) for (int b = a; b < 64; ++b) {
    const int len = b - a + 1;
    const unsigned long long bits = ((len >= 64) ? ~0ull : ((1ull << len) - 1ull)) << a;
    const unsigned lo = bmsk32(a, b - a + 1);
    const unsigned hi = b >= 32 ? bmsk32(max(a - 32, 0), b - max(a, 32) + 1) : 0u;
    if (lo != (unsigned)bits || hi != (unsigned)(bits >> 32)) { atomicAdd(bad, 1); if (*bad < 3) printf("a %d b %d lo %08x hi %08x want %016llx\n", a, b, lo, hi, bits); }
  }
}
int main() { int* bad; cudaMallocManaged(&bad, 4); *bad = 0; k<<<1,1>>>(bad); cudaDeviceSynchronize(); printf("bmsk mismatches: %d of 2080\n", *bad); return 0; }
