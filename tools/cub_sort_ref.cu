// Yardstick only (not on the product path): CUB DeviceRadixSort::SortPairs on
// (u32 tile key, u32 payload) pairs of the config-C tile-sort size, 15 key bits.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
__global__ void fill(unsigned* k, unsigned* v, long long n, unsigned ntiles) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    // runs of ~8 consecutive tiles per record, like the emission order
    unsigned rec = (unsigned)((h >> 8) % ntiles);
    k[i] = (rec + (unsigned)(i & 7)) % ntiles; v[i] = (unsigned)i;
  }
}
int main(int argc, char** argv) {
  long long n = argc > 1 ? atoll(argv[1]) : 212674810LL;
  unsigned ntiles = 32400;
  unsigned *k0, *k1, *v0, *v1; void* tmp = nullptr; size_t tb = 0;
  cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
  fill<<<148 * 8, 256>>>(k0, v0, n, ntiles);
  cub::DoubleBuffer<unsigned> dk(k0, k1), dv(v0, v1);
  cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)n, 0, 15);
  cudaMalloc(&tmp, tb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int it = 0; it < 8; ++it) {
    fill<<<148 * 8, 256>>>(dk.Current(), dv.Current(), n, ntiles);
    cudaEventRecord(a);
    cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)n, 0, 15);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cub SortPairs n=%lld bits=15: %.3f ms (%.1f GB/s moved, 2 passes)\n", n, ms, 2 * 16.0 * n / ms / 1e6);
  }
  return 0;
}
