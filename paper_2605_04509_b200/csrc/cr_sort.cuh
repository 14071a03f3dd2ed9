// cr_sort.cuh — device-wide exclusive scan and a CUB-free, stable LSD radix
// sort (8-bit digits) of (u32 key, u32 value) pairs.  Used for
//   * visible-record compaction (scan of cnt > 0),
//   * the depth presort of records by (k, depth) (4 depth passes + 1 k pass),
//   * the pair offsets (scan of per-record tile counts),
//   * the final stable tile sort of pairs (2 passes at 4K, 3 at 8K).
// Memory-bound: per pass the upsweep reads the digit source (4 B) and the
// downsweep reads key+value and writes key+value (16 B) -> 20 B/element.
#pragma once
#include "cr_device.cuh"

namespace cr {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

// block-wide exclusive scan of one u32 per thread; returns the block total.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t& excl,
                                                         uint32_t* s_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = lane < NT / 32 ? s_warp[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    if (lane < NT / 32) s_warp[lane] = xi - x;
    if (lane == 31) s_warp[32] = xi;
  }
  __syncthreads();
  excl = s_warp[w] + incl - v;
  const uint32_t total = s_warp[32];
  __syncthreads();
  return total;
}

// Phase 1: per-block sums of in(i).
template <class In>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(In in, long long n,
                                                              uint32_t* __restrict__ bsum) {
  __shared__ uint32_t s_warp[33];
  const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t v = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q)
    if (base + q < n) v += in(base + q);
  uint32_t ex;
  const uint32_t tot = block_exclusive_scan<kScanThreads>(v, ex, s_warp);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// Phase 2: exclusive scan of the block sums in place (one block); total out.
// Overflow beyond 2^32-1 sets *overflow.
__global__ void __launch_bounds__(1024) k_scan_bsums(uint32_t* __restrict__ bsum, int nb,
                                                     uint32_t* __restrict__ total,
                                                     int* __restrict__ overflow) {
  __shared__ uint32_t s_warp[33];
  __shared__ unsigned long long s_big;
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  unsigned long long v = 0;
  for (int q = 0; q < per; ++q)
    if (b0 + q < nb) v += bsum[b0 + q];
  if (threadIdx.x == 0) s_big = 0;
  __syncthreads();
  atomicAdd(&s_big, v);
  uint32_t ex;
  block_exclusive_scan<1024>((uint32_t)v, ex, s_warp);
  uint32_t run = ex;
  for (int q = 0; q < per; ++q)
    if (b0 + q < nb) {
      const uint32_t x = bsum[b0 + q];
      bsum[b0 + q] = run;
      run += x;
    }
  if (threadIdx.x == 0) {
    *total = (uint32_t)s_big;
    if (s_big > 0xFFFFFFFFull && overflow) *overflow = 1;
  }
}

// Phase 3: out(i, exclusive prefix, value).
template <class In, class Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(In in, Out out, long long n,
                                                            const uint32_t* __restrict__ bsum) {
  __shared__ uint32_t s_warp[33];
  const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t vals[kScanItems], v = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    vals[q] = (base + q < n) ? in(base + q) : 0u;
    v += vals[q];
  }
  uint32_t ex;
  block_exclusive_scan<kScanThreads>(v, ex, s_warp);
  uint32_t run = bsum[blockIdx.x] + ex;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q)
    if (base + q < n) {
      out(base + q, run, vals[q]);
      run += vals[q];
    }
}

// ----------------------------------------------------------------- radix
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 elements per block
constexpr int kSortWarps = kSortThreads / 32;

// DIGIT_FROM_VAL: digit = val / div (cluster id of record index r = k*M+i);
// otherwise digit = (key >> shift) & 255.
template <bool DIGIT_FROM_VAL>
__device__ __forceinline__ uint32_t sort_digit(const uint32_t* __restrict__ keys,
                                               const uint32_t* __restrict__ vals, long long e,
                                               int shift, unsigned long long div) {
  if (DIGIT_FROM_VAL) return (uint32_t)((unsigned long long)vals[e] / div) & 255u;
  return (keys[e] >> shift) & 255u;
}

template <bool DIGIT_FROM_VAL>
__global__ void __launch_bounds__(kSortThreads) k_radix_upsweep(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, long long n, int shift,
    unsigned long long div, uint32_t* __restrict__ hist /* [256][nb] */, int nb) {
  __shared__ uint32_t s_h[kSortWarps][256];
  const int w = threadIdx.x >> 5;
  for (int q = threadIdx.x; q < kSortWarps * 256; q += kSortThreads) (&s_h[0][0])[q] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int q = 0; q < kSortItems; ++q) {
    const long long e = base + q * kSortThreads + threadIdx.x;
    if (e < n) atomicAdd(&s_h[w][sort_digit<DIGIT_FROM_VAL>(keys, vals, e, shift, div)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += kSortThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) s += s_h[ww][d];
    hist[(long long)d * nb + blockIdx.x] = s;
  }
}

// Stable scatter.  Elements of a block are processed in kSortItems rounds of
// kSortThreads consecutive elements; within a round, ranks come from
// __match_any_sync per warp and an exclusive prefix over warps per digit.
template <bool DIGIT_FROM_VAL, bool MOVE_KEYS>
__global__ void __launch_bounds__(kSortThreads) k_radix_downsweep(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, long long n, int shift,
    unsigned long long div, const uint32_t* __restrict__ hist_scanned, int nb) {
  __shared__ uint32_t s_base[256];            // global base + running count, per digit
  __shared__ uint32_t s_wc[kSortWarps][256];  // per-warp counts -> per-warp prefixes
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int d = threadIdx.x; d < 256; d += kSortThreads)
    s_base[d] = hist_scanned[(long long)d * nb + blockIdx.x];
  for (int q = threadIdx.x; q < kSortWarps * 256; q += kSortThreads) (&s_wc[0][0])[q] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kSortTile;
  for (int q = 0; q < kSortItems; ++q) {
    const long long e = base + q * kSortThreads + threadIdx.x;
    const bool valid = e < n;
    uint32_t k = 0, v = 0, d = 256;
    if (valid) {
      v = vals[e];
      if (MOVE_KEYS || !DIGIT_FROM_VAL) k = keys[e];
      d = DIGIT_FROM_VAL ? ((uint32_t)((unsigned long long)v / div) & 255u) : ((k >> shift) & 255u);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) s_wc[w][d] = __popc(peers);
    __syncthreads();
    // per digit: exclusive prefix over warps, advance the running base
    for (int dd = threadIdx.x; dd < 256; dd += kSortThreads) {
      uint32_t acc = s_base[dd];
#pragma unroll
      for (int ww = 0; ww < kSortWarps; ++ww) {
        const uint32_t c = s_wc[ww][dd];
        s_wc[ww][dd] = acc;
        acc += c;
      }
      s_base[dd] = acc;
    }
    __syncthreads();
    if (valid) {
      const uint32_t pos = s_wc[w][d] + rank;
      vals_out[pos] = v;
      if (MOVE_KEYS) keys_out[pos] = k;
    }
    __syncthreads();
    for (int qq = threadIdx.x; qq < kSortWarps * 256; qq += kSortThreads) (&s_wc[0][0])[qq] = 0;
    __syncthreads();
  }
}

}  // namespace cr
