// cr_sort.cuh — device-wide single-pass exclusive scan and a CUB-free,
// stable LSD radix sort (8-bit digits, onesweep) of (u32 key, u32 value)
// pairs.  Used for
//   * visible-record compaction straight to presort keys (scan of vis),
//   * the depth presort of records by (k, depth) (compressed keys, <= 4 passes),
//   * the pair offsets (scan of per-record tile counts),
//   * the final stable tile sort of pairs (2 passes at 4K, 3 at 8K).
// Per onesweep pass: read key+value, write key+value (16 B/element) plus one
// digit histogram pass per sort.
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

// Single-pass exclusive scan (decoupled look-back): CTA tiles in the order of
// an atomic ticket; each publishes its aggregate, looks back over the
// predecessors' status words for its exclusive prefix, publishes the
// inclusive prefix and writes out(i, prefix, value).  One read of in, one
// write of out (the 3-kernel scan reads in twice).  Status word (u64): hi =
// epoch << 2 | flag (1 aggregate, 2 inclusive), lo = count; the epoch changes
// every launch, so the buffer is never cleared.  *total = the sum; a sum
// beyond 2^32-1 sets *overflow.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Decoupled look-back over the predecessors' status words at p, p - stride,
// p - 2*stride, ... (tile b-1, b-2, ...): four independent loads per round,
// consumed in order (a not-yet-published word is re-polled), so the walk
// over aggregate-only predecessors costs a quarter of the dependent L2 round
// trips.  Returns the exclusive prefix; tile 0 always publishes inclusive.
__device__ __forceinline__ uint32_t lookback4(const unsigned long long* p, long long avail,
                                              long long stride, uint32_t epoch) {
  uint32_t excl = 0;
  for (;;) {
    unsigned long long sv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[q] = q < avail ? ld_status(p - q * stride) : 0ull;
    int q = 0;
    for (; q < 4 && q < avail; ++q) {
      const unsigned long long s = sv[q];
      if ((uint32_t)(s >> 34) != epoch || ((s >> 32) & 3u) == 0u) break;  // not ready: re-poll
      excl += (uint32_t)s;
      if (((s >> 32) & 3u) == 2u) return excl;
    }
    p -= q * stride;
    avail -= q;
  }
}


// inputs that can load 8 consecutive elements at once (vectorized)
template <class T, class = void>
struct HasLoad8 { static constexpr bool value = false; };
template <class T>
struct HasLoad8<T, decltype(void(&T::load8))> { static constexpr bool value = true; };

// outputs that compact flagged elements to (u32, u32) pairs: staged in shared
// memory by block-local rank and written out coalesced (stage(i) -> pair,
// put(global position, pair))
template <class T, class = void>
struct HasStage { static constexpr bool value = false; };
template <class T>
struct HasStage<T, decltype(void(&T::stage))> { static constexpr bool value = true; };
// outputs that store the 8 exclusive prefixes of a thread at once
template <class T, class = void>
struct HasStore8 { static constexpr bool value = false; };
template <class T>
struct HasStore8<T, decltype(void(&T::store8))> { static constexpr bool value = true; };

template <class In, class Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_onepass(
    In in, Out out, long long n, unsigned long long* __restrict__ look,
    uint32_t* __restrict__ ticket, uint32_t epoch, uint32_t* __restrict__ total,
    int* __restrict__ overflow) {
  __shared__ uint32_t s_warp[33];
  __shared__ uint32_t s_bid, s_pre;
  if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t bid = s_bid;
  const long long nb = (n + kScanTile - 1) / kScanTile;
  const long long base = (long long)bid * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t vals[kScanItems], v = 0;
  if constexpr (HasLoad8<In>::value) {
    static_assert(kScanItems == 8, "load8 reads 8 elements");
    if (base + kScanItems <= n) {
      in.load8(base, vals);
    } else {
#pragma unroll
      for (int q = 0; q < kScanItems; ++q) vals[q] = (base + q < n) ? in(base + q) : 0u;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) vals[q] = (base + q < n) ? in(base + q) : 0u;
  }
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) v += vals[q];
  uint32_t ex;
  const uint32_t T = block_exclusive_scan<kScanThreads>(v, ex, s_warp);
  const unsigned long long hiA = (unsigned long long)((epoch << 2) | 1u) << 32;
  const unsigned long long hiP = (unsigned long long)((epoch << 2) | 2u) << 32;
  if (threadIdx.x == 0) st_relaxed_u64(look + bid, (bid == 0 ? hiP : hiA) | T);
  __shared__ uint2 s_kv[HasStage<Out>::value ? kScanTile : 1];
  if constexpr (HasStage<Out>::value) {  // stage before the look-back: overlaps its wait
    uint32_t loc = ex;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q)
      if (base + q < n && vals[q]) s_kv[loc++] = out.stage(base + q);
  }
  if (threadIdx.x == 0) {
    uint32_t excl = 0;
    if (bid > 0) {
      excl = lookback4(look + (bid - 1), (long long)bid, 1, epoch);
      st_relaxed_u64(look + bid, hiP | (excl + T));
    }
    if (excl + T < excl && overflow) *overflow = 1;
    if ((long long)bid == nb - 1) *total = excl + T;
    s_pre = excl;
  }
  __syncthreads();
  if constexpr (HasStage<Out>::value) {  // flags -> compacted pairs, coalesced writes
    const uint32_t pre = s_pre;
    for (uint32_t p = threadIdx.x; p < T; p += kScanThreads) out.put(pre + p, s_kv[p]);
  } else if constexpr (HasStore8<Out>::value) {
    uint32_t run = s_pre + ex, ex8[kScanItems];
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
      ex8[q] = run;
      run += vals[q];
    }
    if (base + kScanItems <= n) {
      out.store8(base, ex8);
    } else {
#pragma unroll
      for (int q = 0; q < kScanItems; ++q)
        if (base + q < n) out(base + q, ex8[q], vals[q]);
    }
  } else {
    uint32_t run = s_pre + ex;
#pragma unroll
    for (int q = 0; q < kScanItems; ++q)
      if (base + q < n) {
        out(base + q, run, vals[q]);
        run += vals[q];
      }
  }
}

// ----------------------------------------------------------------- radix
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 elements per block
constexpr int kSortWarps = kSortThreads / 32;

// DIGIT_FROM_VAL: digit = val / M (cluster id of record index r = k*M+i, via c_fp.divM);
// otherwise digit = (key >> shift) & 255.
template <bool DIGIT_FROM_VAL>
__device__ __forceinline__ uint32_t sort_digit(const uint32_t* __restrict__ keys,
                                               const uint32_t* __restrict__ vals, long long e,
                                               int shift, unsigned long long div) {
  if (DIGIT_FROM_VAL) return fdiv(vals[e], c_fp.divM) & 255u;
  return (keys[e] >> shift) & 255u;
}

template <bool DIGIT_FROM_VAL, bool AGG>
__global__ void __launch_bounds__(kSortThreads) k_radix_upsweep(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, long long n, int shift,
    unsigned long long div, uint32_t* __restrict__ hist /* [256][nb] */, int nb) {
  // per-warp digit counts.  AGG: equal digits within a round are aggregated
  // by an 8-ballot multisplit so skewed digit distributions (the few tile
  // rows of a band in the high tile digit) do not serialise on shared
  // atomics; otherwise one shared atomic per element (cheaper when spread)
  __shared__ uint32_t s_h[kSortWarps][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < kSortWarps * 256; q += kSortThreads) (&s_h[0][0])[q] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int q = 0; q < kSortItems; ++q) {
    const long long e = base + q * kSortThreads + threadIdx.x;
    const uint32_t d = (e < n) ? sort_digit<DIGIT_FROM_VAL>(keys, vals, e, shift, div) : 256u;
    if (!AGG) {
      if (d < 256) atomicAdd(&s_h[w][d], 1u);
      continue;
    }
    unsigned peers = __ballot_sync(0xffffffffu, d < 256);
#pragma unroll
    for (int bit = 0; bit < 8; ++bit) {
      const unsigned bal = __ballot_sync(0xffffffffu, (d >> bit) & 1u);
      peers &= ((d >> bit) & 1u) ? bal : ~bal;
    }
    if (d < 256 && (__ffs(peers) - 1) == lane) atomicAdd(&s_h[w][d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += kSortThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) s += s_h[ww][d];
    hist[(long long)d * nb + blockIdx.x] = s;
  }
}

// Stable scatter, three phases per block of kSortTile elements (kSortWarps
// contiguous warp sub-tiles of kSortItems*32, each walked in order):
//  1. per round of 32: digit peers by 8-bit ballot multisplit (no MATCH),
//     the group leader's shared atomicAdd returns the same-digit count of the
//     warp's earlier rounds -> rank within the warp (kept packed in a register)
//  2. per digit: exclusive prefix over warps -> block-local offsets; elements
//     are written digit-sorted into shared memory
//  3. the block streams shared memory out in order: each digit's run lands
//     contiguously at its global base (coalesced stores).
template <bool DIGIT_FROM_VAL, bool MOVE_KEYS>
__global__ void __launch_bounds__(kSortThreads, 3) k_radix_downsweep(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, long long n, int shift,
    unsigned long long div, const uint32_t* __restrict__ hist_scanned, int nb) {
  __shared__ uint32_t s_cnt[kSortWarps][256];  // counts -> block-local warp offsets
  __shared__ uint32_t s_loff[256];             // block-local digit offsets
  __shared__ uint32_t s_gbase[256];            // global digit bases of this block
  __shared__ uint32_t s_k[MOVE_KEYS ? kSortTile : 1];
  __shared__ uint32_t s_v[kSortTile];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int q = threadIdx.x; q < kSortWarps * 256; q += kSortThreads) (&s_cnt[0][0])[q] = 0;
  __syncthreads();
  const long long bbase = (long long)blockIdx.x * kSortTile;
  const long long wbase = bbase + (long long)w * (kSortItems * 32);
  uint32_t kr[kSortItems], vr[kSortItems], dl[kSortItems];  // dl = digit | rank << 9
#pragma unroll
  for (int q = 0; q < kSortItems; ++q) {
    const long long e = wbase + q * 32 + lane;
    uint32_t k = 0, v = 0, d = 256;
    if (e < n) {
      v = vals[e];
      if (MOVE_KEYS || !DIGIT_FROM_VAL) k = keys[e];
      d = DIGIT_FROM_VAL ? (fdiv(v, c_fp.divM) & 255u) : ((k >> shift) & 255u);
    }
    kr[q] = k;
    vr[q] = v;
    unsigned peers = __ballot_sync(0xffffffffu, d < 256);
#pragma unroll
    for (int bit = 0; bit < 8; ++bit) {
      const unsigned bal = __ballot_sync(0xffffffffu, (d >> bit) & 1u);
      peers &= ((d >> bit) & 1u) ? bal : ~bal;
    }
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (d < 256 && lane == leader) old = atomicAdd(&s_cnt[w][d], (uint32_t)__popc(peers));
    old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
    dl[q] = d | ((old + __popc(peers & lt)) << 9);
  }
  __syncthreads();
  // per digit: warp prefix (block-local), block-local digit offsets, global base
  {
    const int d = threadIdx.x;  // kSortThreads == 256
    uint32_t acc = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = s_cnt[ww][d];
      s_cnt[ww][d] = acc;
      acc += c;
    }
    // exclusive scan of the 256 digit totals across the block
    uint32_t incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __shared__ uint32_t s_ws[kSortWarps];
    if (lane == 31) s_ws[w] = incl;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) wpre += (ww < w) ? s_ws[ww] : 0u;
    const uint32_t loff = wpre + incl - acc;
    s_loff[d] = loff;
    s_gbase[d] = hist_scanned[(long long)d * nb + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) s_cnt[ww][d] += loff;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSortItems; ++q) {
    const uint32_t d = dl[q] & 511u;
    if (d < 256) {
      const uint32_t p = s_cnt[w][d] + (dl[q] >> 9);
      s_v[p] = vr[q];
      if (MOVE_KEYS) s_k[p] = kr[q];
    }
  }
  __syncthreads();
  const int cnt = (int)min((long long)kSortTile, n - bbase);
  for (int p = threadIdx.x; p < cnt; p += kSortThreads) {
    const uint32_t v = s_v[p];
    uint32_t k = 0, d;
    if (MOVE_KEYS) k = s_k[p];
    if (DIGIT_FROM_VAL) d = fdiv(v, c_fp.divM) & 255u;
    else d = (k >> shift) & 255u;
    const uint32_t gp = s_gbase[d] + ((uint32_t)p - s_loff[d]);
    vals_out[gp] = v;
    if (MOVE_KEYS) keys_out[gp] = k;
  }
}

// ------------------------------------------------------ onesweep radix
// Single-pass-per-digit variant (decoupled look-back): one histogram kernel
// reads the keys once for all digit positions, then each pass is ONE kernel
// whose blocks take their tile index from an atomic counter, rank their
// elements (warp multisplit), publish their per-digit counts, look back over
// the preceding tiles' published counts for their global per-digit base and
// scatter through shared memory.  Per pass: 16 B/element (+~6 B per 4096
// elements of look-back status, L2-resident) instead of 20 B plus a device
// scan of the 256 x blocks histogram.
//
// Look-back status word (u64): hi = epoch << 2 | flag (1 aggregate,
// 2 inclusive prefix), lo = count.  The epoch changes every pass, so the
// buffer is never cleared between passes.

// lanes holding the same 8-bit digit as this lane (valid lanes only)
__device__ __forceinline__ unsigned warp_peers8(uint32_t d, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    unsigned m;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
        "@!p not.b32 %0, %0;\n\t}"
        : "=r"(m)
        : "r"(d), "r"(1u << b));
    peers &= m;
  }
  return peers;
}

// lanes holding the same 9-bit digit as this lane (valid lanes only)
__device__ __forceinline__ unsigned warp_peers9(uint32_t d, bool valid) {
  unsigned peers = warp_peers8(d, valid);
  unsigned m;
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
      "and.b32 t, %1, 256;\n\t"
      "setp.ne.u32 p, t, 0;\n\t"
      "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
      "@!p not.b32 %0, %0;\n\t}"
      : "=r"(m)
      : "r"(d));
  return peers & m;
}

constexpr int kHistThreads = 256;
constexpr int kHistBins = 512;  // per pass in ghist: 256 bins, or 512 for a 9-bit first digit
// global histograms of NPASS consecutive digits (the first bits0 = 8 or 9
// bits wide at shift0, then 8-bit digits) into ghist[pass][kHistBins]
// (zeroed by the caller).  aggmask bit p: digit p is skewed (few distinct
// values) -> warp-aggregated counts.
__device__ __forceinline__ int digit_shift(int shift0, int bits0, int p) {
  return p == 0 ? shift0 : shift0 + bits0 + 8 * (p - 1);
}
__global__ void __launch_bounds__(kHistThreads) k_radix_hist(const uint32_t* __restrict__ keys,
                                                             long long n, int shift0, int npass,
                                                             unsigned aggmask,
                                                             uint32_t* __restrict__ ghist,
                                                             int bits0 = 8) {
  __shared__ uint32_t s_h[4][kHistBins];
  for (int q = threadIdx.x; q < 4 * kHistBins; q += kHistThreads) (&s_h[0][0])[q] = 0;
  __syncthreads();
  const long long n4 = n >> 2;
  const uint4* k4 = reinterpret_cast<const uint4*>(keys);
  const long long stride = (long long)gridDim.x * kHistThreads;
  // whole-warp trip count so the aggregated (ballot) path stays converged
  const long long nround = (n4 + stride - 1) / stride;
  for (long long it = 0; it < nround; ++it) {
    const long long e = it * stride + (long long)blockIdx.x * kHistThreads + threadIdx.x;
    const bool ok = e < n4;
    const uint4 v = ok ? k4[e] : make_uint4(0, 0, 0, 0);
    for (int p = 0; p < npass; ++p) {
      const int sh = digit_shift(shift0, bits0, p);
      const uint32_t dm = (p == 0 && bits0 == 9) ? 511u : 255u;
      const uint32_t d0 = (v.x >> sh) & dm, d1 = (v.y >> sh) & dm;
      const uint32_t d2 = (v.z >> sh) & dm, d3 = (v.w >> sh) & dm;
      if ((aggmask >> p) & 1u) {
        // run-aggregate the 4 keys, then across the warp
        const bool same = ok && d0 == d1 && d0 == d2 && d0 == d3;
        if (ok && !same) {
          atomicAdd(&s_h[p][d0], 1u);
          atomicAdd(&s_h[p][d1], 1u);
          atomicAdd(&s_h[p][d2], 1u);
          atomicAdd(&s_h[p][d3], 1u);
        }
        const unsigned peers = dm == 511u ? warp_peers9(d0, same) : warp_peers8(d0, same);
        if (same && (__ffs(peers) - 1) == (int)(threadIdx.x & 31))
          atomicAdd(&s_h[p][d0], 4u * (uint32_t)__popc(peers));
      } else if (ok) {
        atomicAdd(&s_h[p][d0], 1u);
        atomicAdd(&s_h[p][d1], 1u);
        atomicAdd(&s_h[p][d2], 1u);
        atomicAdd(&s_h[p][d3], 1u);
      }
    }
  }
  // tail (n % 4) in block 0
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const uint32_t k = keys[(n4 << 2) + threadIdx.x];
    for (int p = 0; p < npass; ++p)
      atomicAdd(&s_h[p][(k >> digit_shift(shift0, bits0, p)) & ((p == 0 && bits0 == 9) ? 511u : 255u)], 1u);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < npass * kHistBins; q += kHistThreads) {
    const uint32_t c = (&s_h[0][0])[q];
    if (c) atomicAdd(&ghist[q], c);
  }
}

// one stable pass on digit (key >> shift) & 255; ghist = this digit's global
// histogram; look = [tiles][256] status words; ctr = tile counter (zeroed).
// slotK != 0 (last tile-sort pass only): write the (t, k) range slot
// t*K + k (k = val / M) instead of the key t, so k_ranges reads keys only.
// Ranks by 8-ballot multisplit peers (measured faster than match.any.sync on
// B200: 4.37 vs 4.88 ms for the frame's 6 passes; 16 items/thread beat 12).
// VAR bit 0: full tiles skip the bounds checks; bit 1: scatter into shared
// memory before the look-back (the wait overlaps the local scatter); bit 2:
// values loaded at the scatter, not held in registers through the ranking.
// Shipped: VAR = 7, 18 items at 4 CTAs/SM (measured at config C, sort stage
// with 16 items: 4.26 ms for VAR = 0 at 3 CTAs/SM; 3.94 bit 0; 4.11 bit 1;
// 3.64 bits 0+1; 3.55 bits 0+1 at 4 CTAs/SM; 3.40 VAR = 7 at 5 CTAs/SM; 18
// items at 4 CTAs/SM 3.25; 12 items at 6 CTAs/SM and keys re-read at the
// scatter were slower).
template <int ITEMS, bool FULL, bool VALS>
__device__ __forceinline__ void onesweep_rank(const uint32_t* __restrict__ keys,
                                              const uint32_t* __restrict__ vals, long long n,
                                              long long wbase, int shift, int lane, unsigned lt,
                                              uint32_t* s_cw, uint32_t* kr, uint32_t* vr,
                                              uint32_t* dl) {
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const long long e = wbase + q * 32 + lane;
    const bool ok = FULL || e < n;
    kr[q] = ok ? keys[e] : 0u;
    if (VALS) vr[q] = ok ? vals[e] : 0u;
  }
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const bool ok = FULL || wbase + q * 32 + lane < n;
    const uint32_t d = ok ? ((kr[q] >> shift) & 255u) : 256u;
    const unsigned peers = FULL ? warp_peers8(d, true) : warp_peers8(d, ok);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (ok && lane == leader) old = atomicAdd(&s_cw[d], (uint32_t)__popc(peers));
    old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
    dl[q] = d | ((old + __popc(peers & lt)) << 9);
  }
}

template <int ITEMS, int VAR, int MINB = 3>
__global__ void __launch_bounds__(kSortThreads, MINB) k_radix_onesweep(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, long long n, int shift,
    const uint32_t* __restrict__ ghist, unsigned long long* __restrict__ look,
    uint32_t* __restrict__ ctr, uint32_t epoch, uint32_t slotK) {
  constexpr int TILE = kSortThreads * ITEMS;
  constexpr bool LATE = (VAR & 2) != 0;
  __shared__ uint32_t s_cnt[kSortWarps][256];  // counts -> block-local warp offsets
  __shared__ uint32_t s_off[256];              // global base - block-local offset
  __shared__ uint32_t s_k[TILE];
  __shared__ uint32_t s_v[TILE];
  __shared__ uint32_t s_ws[2][kSortWarps];
  __shared__ uint32_t s_bid;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x == 0) s_bid = atomicAdd(ctr, 1u);
  for (int q = threadIdx.x; q < kSortWarps * 256; q += kSortThreads) (&s_cnt[0][0])[q] = 0;
  __syncthreads();
  const uint32_t bid = s_bid;
  const long long bbase = (long long)bid * TILE;
  const long long wbase = bbase + (long long)w * (ITEMS * 32);
  uint32_t kr[ITEMS], vr[ITEMS], dl[ITEMS];  // dl = digit | rank << 9
  constexpr bool VALS = (VAR & 4) == 0;  // bit 2: values loaded at the scatter
  if ((VAR & 1) && bbase + TILE <= n)
    onesweep_rank<ITEMS, true, VALS>(keys, vals, n, wbase, shift, lane, lt, s_cnt[w], kr, vr, dl);
  else
    onesweep_rank<ITEMS, false, VALS>(keys, vals, n, wbase, shift, lane, lt, s_cnt[w], kr, vr, dl);
  __syncthreads();
  const int d = threadIdx.x;  // kSortThreads == 256: one digit per thread
  uint32_t acc = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const uint32_t c = s_cnt[ww][d];
    s_cnt[ww][d] = acc;
    acc += c;
  }
  // publish this tile's count of digit d as early as possible
  unsigned long long* my = look + (size_t)bid * 256 + d;
  const unsigned long long hiA = (unsigned long long)((epoch << 2) | 1u) << 32;
  const unsigned long long hiP = (unsigned long long)((epoch << 2) | 2u) << 32;
  st_status(my, (bid == 0 ? hiP : hiA) | acc);
  // block-local digit offsets and global digit starts (two 256-wide scans)
  const uint32_t gh = ghist[d];
  uint32_t i1 = acc, i2 = gh;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y1 = __shfl_up_sync(0xffffffffu, i1, o);
    const uint32_t y2 = __shfl_up_sync(0xffffffffu, i2, o);
    if (lane >= o) { i1 += y1; i2 += y2; }
  }
  if (lane == 31) { s_ws[0][w] = i1; s_ws[1][w] = i2; }
  // look back for the exclusive prefix of digit d over the preceding tiles
  uint32_t excl = 0;
  if (!LATE && bid > 0) {
    excl = lookback4(look + (size_t)(bid - 1) * 256 + d, (long long)bid, 256, epoch);
    st_status(my, hiP | (excl + acc));
  }
  __syncthreads();
  uint32_t p1 = 0, p2 = 0;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww)
    if (ww < w) { p1 += s_ws[0][ww]; p2 += s_ws[1][ww]; }
  const uint32_t loff = p1 + i1 - acc;
  if (!LATE) s_off[d] = (p2 + i2 - gh) + excl - loff;
#pragma unroll
  for (int ww = 0; ww < kSortWarps; ++ww) s_cnt[ww][d] += loff;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const uint32_t dq = dl[q] & 511u;
    if (dq < 256) {
      const uint32_t p = s_cnt[w][dq] + (dl[q] >> 9);
      s_v[p] = VALS ? vr[q] : vals[wbase + q * 32 + lane];
      s_k[p] = kr[q];
    }
  }
  if (LATE) {
    if (bid > 0) {
      excl = lookback4(look + (size_t)(bid - 1) * 256 + d, (long long)bid, 256, epoch);
      st_status(my, hiP | (excl + acc));
    }
    s_off[d] = (p2 + i2 - gh) + excl - loff;
  }
  __syncthreads();
  const int cnt = (int)min((long long)TILE, n - bbase);
  for (int p = threadIdx.x; p < cnt; p += kSortThreads) {
    const uint32_t k = s_k[p], v = s_v[p];
    const uint32_t gp = s_off[(k >> shift) & 255u] + (uint32_t)p;
    vals_out[gp] = v;
    keys_out[gp] = slotK ? k * slotK + fdiv(v, c_fp.divM) : k;
  }
}

template <int ITEMS, bool FULL, bool VALS, int NDIG>
__device__ __forceinline__ void onesweep_rank_n(const uint32_t* __restrict__ keys,
                                              const uint32_t* __restrict__ vals, long long n,
                                              long long wbase, int shift, int lane, unsigned lt,
                                              uint32_t* s_cw, uint32_t* kr, uint32_t* vr,
                                              uint32_t* dl) {
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const long long e = wbase + q * 32 + lane;
    const bool ok = FULL || e < n;
    kr[q] = ok ? keys[e] : 0u;
    if (VALS) vr[q] = ok ? vals[e] : 0u;
  }
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const bool ok = FULL || wbase + q * 32 + lane < n;
    const uint32_t d = ok ? ((kr[q] >> shift) & (uint32_t)(NDIG - 1)) : (uint32_t)NDIG;
    unsigned peers;
    if (NDIG == 512) peers = FULL ? warp_peers9(d, true) : warp_peers9(d, ok);
    else peers = FULL ? warp_peers8(d, true) : warp_peers8(d, ok);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (ok && lane == leader) old = atomicAdd(&s_cw[d], (uint32_t)__popc(peers));
    old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
    dl[q] = d | ((old + __popc(peers & lt)) << 10);
  }
}

// The same pass for NDIG = 512 (a 9-bit digit: the first pass of a 17-bit
// 8K tile sort, which then takes 2 passes instead of 3), each thread owning
// NDIG / 256 digits; key / value staging in dynamic shared memory.  (Kept
// apart from the 8-bit kernel above, which the generic form slows by 1 %.)
template <int ITEMS>
constexpr int onesweep_dyn_smem() { return 2 * kSortThreads * ITEMS * 4; }
template <int ITEMS, int VAR, int MINB = 3, int NDIG = 256>
__global__ void __launch_bounds__(kSortThreads, MINB) k_radix_onesweep_n(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, long long n, int shift,
    const uint32_t* __restrict__ ghist, unsigned long long* __restrict__ look,
    uint32_t* __restrict__ ctr, uint32_t epoch, uint32_t slotK) {
  constexpr int TILE = kSortThreads * ITEMS;
  constexpr bool LATE = (VAR & 2) != 0;
  constexpr int DPT = NDIG / kSortThreads;  // digits per thread
  constexpr uint32_t DM = NDIG - 1;
  __shared__ uint32_t s_cnt[kSortWarps][NDIG];  // counts -> block-local warp offsets
  __shared__ uint32_t s_off[NDIG];              // global base - block-local offset
  __shared__ uint32_t s_kv_st[NDIG == 256 ? 2 * TILE : 1];
  extern __shared__ uint32_t s_kv_dyn[];
  uint32_t* s_k = NDIG == 256 ? s_kv_st : s_kv_dyn;
  uint32_t* s_v = s_k + TILE;
  __shared__ uint32_t s_ws[2][kSortWarps];
  __shared__ uint32_t s_bid;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (threadIdx.x == 0) s_bid = atomicAdd(ctr, 1u);
  for (int q = threadIdx.x; q < kSortWarps * NDIG; q += kSortThreads) (&s_cnt[0][0])[q] = 0;
  __syncthreads();
  const uint32_t bid = s_bid;
  const long long bbase = (long long)bid * TILE;
  const long long wbase = bbase + (long long)w * (ITEMS * 32);
  uint32_t kr[ITEMS], vr[ITEMS], dl[ITEMS];  // dl = digit | rank << 10
  constexpr bool VALS = (VAR & 4) == 0;  // bit 2: values loaded at the scatter
  if ((VAR & 1) && bbase + TILE <= n)
    onesweep_rank_n<ITEMS, true, VALS, NDIG>(keys, vals, n, wbase, shift, lane, lt, s_cnt[w], kr, vr, dl);
  else
    onesweep_rank_n<ITEMS, false, VALS, NDIG>(keys, vals, n, wbase, shift, lane, lt, s_cnt[w], kr, vr, dl);
  __syncthreads();
  const unsigned long long hiA = (unsigned long long)((epoch << 2) | 1u) << 32;
  const unsigned long long hiP = (unsigned long long)((epoch << 2) | 2u) << 32;
  uint32_t acc[DPT], gh[DPT], loff[DPT], goff[DPT];
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * kSortThreads + threadIdx.x;
    uint32_t a = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const uint32_t c = s_cnt[ww][d];
      s_cnt[ww][d] = a;
      a += c;
    }
    acc[h] = a;
    // publish this tile's count of digit d as early as possible
    st_status(look + (size_t)bid * NDIG + d, (bid == 0 ? hiP : hiA) | a);
    gh[h] = ghist[d];
  }
  // block-local digit offsets and global digit starts (two NDIG-wide scans)
  uint32_t c1 = 0, c2 = 0;
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    uint32_t i1 = acc[h], i2 = gh[h];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y1 = __shfl_up_sync(0xffffffffu, i1, o);
      const uint32_t y2 = __shfl_up_sync(0xffffffffu, i2, o);
      if (lane >= o) { i1 += y1; i2 += y2; }
    }
    if (lane == 31) { s_ws[0][w] = i1; s_ws[1][w] = i2; }
    __syncthreads();
    uint32_t p1 = 0, p2 = 0, t1 = 0, t2 = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      if (ww < w) { p1 += s_ws[0][ww]; p2 += s_ws[1][ww]; }
      t1 += s_ws[0][ww];
      t2 += s_ws[1][ww];
    }
    loff[h] = c1 + p1 + i1 - acc[h];
    goff[h] = c2 + p2 + i2 - gh[h];
    c1 += t1;
    c2 += t2;
    if (DPT > 1) __syncthreads();  // s_ws is reused by the next digit group
  }
  // look back for the exclusive prefix of digit d over the preceding tiles
  uint32_t excl[DPT];
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * kSortThreads + threadIdx.x;
    excl[h] = 0;
    if (!LATE && bid > 0) {
      excl[h] = lookback4(look + (size_t)(bid - 1) * NDIG + d, (long long)bid, NDIG, epoch);
      st_status(look + (size_t)bid * NDIG + d, hiP | (excl[h] + acc[h]));
    }
    if (!LATE) s_off[d] = goff[h] + excl[h] - loff[h];
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) s_cnt[ww][d] += loff[h];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const uint32_t dq = dl[q] & 1023u;
    if (dq < (uint32_t)NDIG) {
      const uint32_t p = s_cnt[w][dq] + (dl[q] >> 10);
      s_v[p] = VALS ? vr[q] : vals[wbase + q * 32 + lane];
      s_k[p] = kr[q];
    }
  }
  if (LATE) {
#pragma unroll
    for (int h = 0; h < DPT; ++h) {
      const int d = h * kSortThreads + threadIdx.x;
      if (bid > 0) {
        excl[h] = lookback4(look + (size_t)(bid - 1) * NDIG + d, (long long)bid, NDIG, epoch);
        st_status(look + (size_t)bid * NDIG + d, hiP | (excl[h] + acc[h]));
      }
      s_off[d] = goff[h] + excl[h] - loff[h];
    }
  }
  __syncthreads();
  const int cnt = (int)min((long long)TILE, n - bbase);
  for (int p = threadIdx.x; p < cnt; p += kSortThreads) {
    const uint32_t k = s_k[p], v = s_v[p];
    const uint32_t gp = s_off[(k >> shift) & DM] + (uint32_t)p;
    vals_out[gp] = v;
    keys_out[gp] = slotK ? k * slotK + fdiv(v, c_fp.divM) : k;
  }
}

}  // namespace cr
