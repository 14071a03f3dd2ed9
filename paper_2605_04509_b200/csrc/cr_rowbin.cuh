// cr_rowbin.cuh — a6 emission + a7 tile sort + a8 ranges by tile ROWS first
// (MSD), without materialising unsorted (tile, record) pairs.
//
// The lists the composite reads are the Eq.11 key order: tile t,
// then cluster k, then depth, then i (Alg.2 GenerateKeys P:791-808, sort
// P:760-761, ranges P:377).  The binning produces, per record of the
// (k, depth, i)-sorted list (position g), its cluster tile union as ROW
// ENTRIES: one entry per union tile row = (record r, tile row, column of
// bit 0, 64-bit column mask).  Then:
//   B  k_rowbin     stable counting sort of the entries by tile row
//                   (onesweep: block-local multisplit ranks + decoupled
//                   look-back per row digit), 16-byte entries
//   C0 k_rowscan    exclusive scan of the entries' pair counts (row-major
//                   pair offsets) + the per-tile pair histogram + the map
//                   from column-sort tiles to their first entry
//   C1 k_tile_bases per band tile: start of its list (row base + prefix over
//                   the row's columns)
//   C  k_colsort    per tile row, stable counting sort of the row's pairs by
//                   tile column, pairs generated from the entries' masks in
//                   shared memory (onesweep within the row, tiles never span
//                   two rows); writes the record index r only
//   R  k_ranges_rb  [S, E) of (t, k): binary search on k = r / M inside the
//                   tile's list (lists are k-sorted)
// Stability: entries leave B in list order within a row, pairs leave C in
// entry order within a tile, so each (t, k) list is in (depth, i) order —
// the same permutation as the LSD sort of the emitted pairs (bit-identical
// S, E and payloads; introspection rebuilds the keys from S, E).
// Traffic per pair ~ (16 B entry write + read)/3.7 + 4 B payload, against
// 8 B emitted + 2 x 16 B sorted + 8 B ranges for emission + 2-pass LSD.
// Used when the band has <= 512 tile rows and the frame <= 512 tile columns
// (8K: 270 x 480); larger panels take the emission + LSD path.
#pragma once
#include "cr_sort.cuh"

namespace cr {

constexpr int kRbThreads = 256;
constexpr int kRbEPT = 8;                     // entries per thread in k_rowbin
constexpr int kRbTE = kRbThreads * kRbEPT;    // entries per k_rowbin tile
constexpr int kRbIPT = 16;                    // pairs per thread in k_colsort
constexpr int kRbTP = kRbThreads * kRbIPT;    // pairs per k_colsort tile
constexpr int kRbDynSmem = 32768;             // dynamic shared memory of k_rowbin / k_colsort
constexpr int kRbRecCap = 1024;               // records of a k_rowbin tile staged in shared memory
constexpr int kCsEntCap = 1536;               // entries of a k_colsort tile staged in shared memory
constexpr int kCsDynSmem = 2 * kRbTP * 4 + kCsEntCap * 20;  // k_colsort dynamic shared memory
constexpr uint32_t kSlotBigEnt = 0x40000000u;  // big record: entries in the big store

// entry: x = r, y = (tile row << 16) | (u16) column of bit 0 (>= -1), z/w = mask
__device__ __forceinline__ int ent_row(const uint4& e) { return (int)(e.y >> 16); }
__device__ __forceinline__ int ent_col(const uint4& e) { return (int)(int16_t)(e.y & 0xFFFFu); }

// lanes holding the same NB-bit digit as this lane (valid lanes only)
template <int NB>
__device__ __forceinline__ unsigned warp_peers(uint32_t d, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const unsigned bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? bal : ~bal;
  }
  return peers;
}

// exclusive scan of one u32 per thread over an NT-thread block (s_w: NT/32
// words); total = the block sum
template <int NT>
__device__ __forceinline__ uint32_t scan_block(uint32_t v, uint32_t* s_w, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  uint32_t pre = 0, tot = 0;
#pragma unroll
  for (int ww = 0; ww < NT / 32; ++ww) {
    const uint32_t x = s_w[ww];
    pre += ww < w ? x : 0u;
    tot += x;
  }
  __syncthreads();
  total = tot;
  return pre + incl - v;
}

// Per-row prefix tables of the band from the row histograms (nb <= NDIG <=
// 512 rows; every thread of the NT-thread block must call):
//   rowE[ro]  first entry of row ro in the row-bucketed entry array
//   rowP[ro]  first pair of row ro (row-major)
//   rowT[ro]  first k_colsort tile of row ro (ceil(pairs / kRbTP) per row)
// for ro in [0, nb]; index nb = the totals.
template <int NDIG, int NT>
__device__ void row_tables(const uint32_t* __restrict__ rowhist, int nb, uint32_t* s_rowE,
                           uint32_t* s_rowP, uint32_t* s_rowT, uint32_t* s_w) {
  uint32_t cE = 0, cP = 0, cT = 0;
  for (int h = 0; h < (NDIG + NT - 1) / NT; ++h) {
    const int ro = h * NT + threadIdx.x;
    const uint32_t e = ro < nb ? rowhist[ro] : 0u;
    const uint32_t p = ro < nb ? rowhist[kRbMaxRows + ro] : 0u;
    const uint32_t t = (p + kRbTP - 1) / kRbTP;
    uint32_t tE, tP, tT;
    const uint32_t xE = scan_block<NT>(e, s_w, tE);
    const uint32_t xP = scan_block<NT>(p, s_w, tP);
    const uint32_t xT = scan_block<NT>(t, s_w, tT);
    if (ro <= nb) {
      if (s_rowE) s_rowE[ro] = cE + xE;
      if (s_rowP) s_rowP[ro] = cP + xP;
      if (s_rowT) s_rowT[ro] = cT + xT;
    }
    cE += tE;
    cP += tP;
    cT += tT;
  }
  if (threadIdx.x == 0 && nb % NT == 0) {  // the totals, when row nb starts a new chunk
    if (s_rowE) s_rowE[nb] = cE;
    if (s_rowP) s_rowP[nb] = cP;
    if (s_rowT) s_rowT[nb] = cT;
  }
  __syncthreads();
}

// The band's row tables once per frame into global memory:
// rowtab[0][ro] = rowE, rowtab[1][ro] = rowP, rowtab[2][ro] = rowT (ro <= nb).
constexpr int kRowTab = kRbMaxRows + 1;
template <int NDIG>
__global__ void __launch_bounds__(kRbThreads) k_row_tables(const uint32_t* __restrict__ rowhist,
                                                           uint32_t* __restrict__ rowtab) {
  __shared__ uint32_t s_t[3][NDIG + 1];
  __shared__ uint32_t s_w[16];
  const int nb = c_fp.row1 - c_fp.row0;
  row_tables<NDIG, kRbThreads>(rowhist, nb, s_t[0], s_t[1], s_t[2], s_w);
  for (int q = threadIdx.x; q <= nb; q += kRbThreads) {
    rowtab[q] = s_t[0][q];
    rowtab[kRowTab + q] = s_t[1][q];
    rowtab[2 * kRowTab + q] = s_t[2][q];
  }
}

// Decoupled look-back as lookback4, with a short back-off while a
// predecessor has not published (keeps polling warps off the issue slots).
__device__ __forceinline__ uint32_t lookback4_backoff(const unsigned long long* p, long long avail,
                                                      long long stride, uint32_t epoch) {
  uint32_t excl = 0;
  for (;;) {
    unsigned long long sv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[q] = q < avail ? ld_status(p - q * stride) : 0ull;
    int q = 0;
    for (; q < 4 && q < avail; ++q) {
      const unsigned long long st = sv[q];
      if ((uint32_t)(st >> 34) != epoch || ((st >> 32) & 3u) == 0u) break;
      excl += (uint32_t)st;
      if (((st >> 32) & 3u) == 2u) return excl;
    }
    if (q == 0) __nanosleep(64);
    p -= q * stride;
    avail -= q;
  }
}

// ---------------------------------------------------------------------------
// Big records (footprint beyond a 64-byte slot): their entries in a store of
// nrows x nw entries per record (all union rows x the 64-column windows of a
// conservative column range), written by k_count_big_rb; the slot header is
// {kSlotOverflow | kSlotBigEnt, store base, nrows, nw}.
// ---------------------------------------------------------------------------
struct BigEnt {
  uint4* e;
  uint32_t* ctr;   // entries allocated (atomic)
  uint32_t cap;
  uint32_t* err;   // [0] store capacity exceeded, [1] a tile outside the window range
};

template <int G>
__global__ void __launch_bounds__(kBinThreads) k_count_big_rb(
    const uint32_t* __restrict__ big, const uint32_t* __restrict__ recs,
    const uint32_t* __restrict__ n_ptr, const float4* __restrict__ mean4,
    const float4* __restrict__ geom, uint32_t* __restrict__ cnt, uint4* __restrict__ slots,
    BigEnt be, uint32_t* __restrict__ rowhist) {
  extern __shared__ float s_cam[];  // c_fp.N cameras x kCamStride (dynamic)
  __shared__ uint32_t s_rh[2 * kRbMaxRows];
  for (int q = threadIdx.x; q < 2 * kRbMaxRows; q += blockDim.x) s_rh[q] = 0u;
  stage_cams(s_cam);
  __syncthreads();
  const uint32_t n = *n_ptr;
  constexpr int GPW = 32 / G;
  const int s = c_fp.s, N = c_fp.N, TX = c_fp.TX, TY = c_fp.TY;
  const int row0 = c_fp.row0, row1 = c_fp.row1;
  const int lane = threadIdx.x & 31, v = lane & (G - 1), gi = lane / G;
  const bool lead = v == 0;
  const uint32_t nwarps = gridDim.x * kBinWarps;
  for (uint32_t g = (blockIdx.x * kBinThreads + threadIdx.x) / 32; g < n; g += nwarps) {
    const uint32_t o = big[g];
    const uint32_t r = recs[o];
    const int k = (int)fdiv(r, c_fp.divM);
    const float4 m = mean4[(long long)r - (long long)k * c_fp.M];
    const EllRec el = ell_load(geom[2ull * r], geom[2ull * r + 1]);
    // lane v of each group: view j = k*s + v (exact mean, Eq.5; AccuTile rows, O7)
    const int j = k * s + v;
    bool vis = false;
    float mx = 0.f, my = 0.f;
    int ty0 = 0x7fffffff, ty1 = -1, cl = 0x7fffffff, ch = -0x7fffffff;
    if (v < s && j < N) {
      const CamDev cam = load_cam(s_cam, j);
      const F3 p = cam_point_exact(cam, m.x, m.y, m.z);
      if (p.z >= c_fp.znear) {
        mean2d_exact(cam, p, mx, my);
        view_rows(el, my, TY, ty0, ty1);
        vis = true;
        // conservative column range of the view's footprint (bounding box + 1 tile)
        cl = (int)fminf(fmaxf(floorf((mx - el.ex - 15.5f) * 0.0625f) - 1.0f, -1.0f), (float)TX);
        ch = (int)fmaxf(fminf(ceilf((mx + el.ex - 0.5f) * 0.0625f) + 1.0f, (float)TX), -1.0f);
      }
    }
    const int rmin = max(gmin<G>(vis ? ty0 : 0x7fffffff), row0);
    const int rmax = min(gmax<G>(vis ? ty1 : -1), row1 - 1);
    const int nrows = rmax >= rmin ? rmax - rmin + 1 : 0;
    const int glo = gmin<G>(vis ? cl : 0x7fffffff);
    const int ghi = gmax<G>(vis ? ch : -0x7fffffff);
    const int nw = (nrows > 0 && ghi >= glo) ? ((ghi - glo) >> 6) + 1 : 0;
    const uint32_t ne = (uint32_t)(nrows * nw);
    uint32_t base = 0;
    if (lane == 0 && ne) base = atomicAdd(be.ctr, ne);
    base = __shfl_sync(0xffffffffu, base, 0);
    const bool fits = (unsigned long long)base + ne <= be.cap;
    if (lane == 0 && !fits) atomicExch(&be.err[0], 1u);
    const int it_max = (nrows + GPW - 1) / GPW;  // warp-uniform (the record is shared)
    for (int ii = 0; ii < it_max; ++ii) {
      const int it = gi + ii * GPW;
      const bool rowok = it < nrows;
      const int ty = rmin + it;
      int tx0 = 0x7fffffff, tx1 = -1;
      if (rowok && vis && ty >= ty0 && ty <= ty1) {
        int q0, q1;
        if (view_row_cols(el, mx, my, ty, TX, q0, q1) && q0 <= q1) {
          tx0 = q0;
          tx1 = q1;
        }
      }
      if (tx1 >= tx0 && (tx0 < glo || tx1 > glo + 64 * nw - 1)) atomicExch(&be.err[1], 1u);
      for (int wi = 0; wi < nw; ++wi) {
        const int wlo = glo + 64 * wi;
        unsigned long long mask = 0ull;
        if (tx1 >= tx0) {
          const int a0 = max(tx0, wlo), a1 = min(tx1, wlo + 63);
          if (a0 <= a1) {
            const int len = a1 - a0 + 1;
            mask = ((len >= 64) ? ~0ull : ((1ull << len) - 1ull)) << (a0 - wlo);
          }
        }
        mask = gor64<G>(mask);
        if (lead && rowok && fits) {
          be.e[base + (uint32_t)(it * nw + wi)] =
              make_uint4(r, ((uint32_t)ty << 16) | ((uint32_t)wlo & 0xFFFFu), (uint32_t)mask,
                         (uint32_t)(mask >> 32));
          const uint32_t pc = (uint32_t)__popcll(mask);
          if (pc) atomicAdd(&s_rh[kRbMaxRows + ty - row0], pc);
        }
      }
      if (lead && rowok && fits) atomicAdd(&s_rh[ty - row0], (uint32_t)nw);
    }
    if (lane == 0) {
      cnt[o] = fits ? ne : 0u;
      slots[4ull * o] = make_uint4(kSlotOverflow | kSlotBigEnt, base, (uint32_t)nrows, (uint32_t)nw);
    }
    __syncwarp();
  }
  __syncthreads();
  const int nb = row1 - row0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    if (s_rh[q]) atomicAdd(&rowhist[q], s_rh[q]);
    if (s_rh[kRbMaxRows + q]) atomicAdd(&rowhist[kRbMaxRows + q], s_rh[kRbMaxRows + q]);
  }
}

// Scan output of the per-record entry counts: eoff[g] and, for every k_rowbin
// tile whose first entry lies in record g, tfirst[tile] = g.
struct OutEoff {
  uint32_t* eoff;
  uint32_t* tfirst;
  __device__ __forceinline__ void operator()(long long i, uint32_t x, uint32_t v) const {
    eoff[i] = x;
    for (uint32_t c = (x + kRbTE - 1) / kRbTE; v && c * (uint32_t)kRbTE < x + v; ++c)
      tfirst[c] = (uint32_t)i;
  }
};

// ---------------------------------------------------------------------------
// B: stable counting sort of the row entries by tile row (digit = row - row0,
// NDIG = 256 or 512 digits).  Tile = kRbTE consecutive entries of the list
// order; entry -> record by the records' start marks and a running max.
// ---------------------------------------------------------------------------
template <int NDIG>
__global__ void __launch_bounds__(kRbThreads, 3) k_rowbin(
    const uint32_t* __restrict__ rec_sorted, const uint4* __restrict__ slots,
    const uint32_t* __restrict__ eoff, uint32_t nrec, uint32_t NE,
    const uint32_t* __restrict__ tfirst, const uint4* __restrict__ bigent,
    const uint32_t* __restrict__ rowtab, uint4* __restrict__ out,
    unsigned long long* __restrict__ look, uint32_t* __restrict__ ctr, uint32_t epoch) {
  constexpr int NB = NDIG == 512 ? 9 : 8;
  constexpr int DPT = NDIG / 256;
  __shared__ uint32_t s_cnt[kRbThreads / 32][NDIG];  // per-warp digit counts -> offsets
  extern __shared__ uint4 s_e[];                     // [kRbTE] entries (dynamic, 32 KB)
  // until the entries are ranked, the same 32 KB hold per position the record
  // (relative to g0) and per record of the tile its first entry, r and slot header
  uint32_t* s_g = reinterpret_cast<uint32_t*>(s_e);           // [kRbTE]
  uint4* s_h = s_e + kRbTE / 4;                               // [kRbRecCap]
  uint32_t* s_x = reinterpret_cast<uint32_t*>(s_h + kRbRecCap);  // [kRbRecCap]
  uint32_t* s_r = s_x + kRbRecCap;                            // [kRbRecCap]
  __shared__ uint32_t s_off[NDIG];
  __shared__ uint32_t s_rowE[NDIG + 1];
  __shared__ uint32_t s_w[16];
  __shared__ uint32_t s_bid;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int nb = c_fp.row1 - c_fp.row0;
  if (threadIdx.x == 0) s_bid = atomicAdd(ctr, 1u);
  for (int q = threadIdx.x; q < (kRbThreads / 32) * NDIG; q += kRbThreads) (&s_cnt[0][0])[q] = 0;
  for (int q = threadIdx.x; q < kRbTE; q += kRbThreads) s_g[q] = 0;
  for (int q = threadIdx.x; q < nb; q += kRbThreads) s_rowE[q] = rowtab[q];
  __syncthreads();
  const uint32_t bid = s_bid;
  const uint32_t ntile = (NE + kRbTE - 1) / kRbTE;
  const uint32_t J0 = bid * (uint32_t)kRbTE;
  const int nh = (int)min((uint32_t)kRbTE, NE - J0);
  // ---- the tile's records [g0, g1]: first entries (-> start marks), and, when
  // they fit, r and slot headers staged in shared memory (coalesced loads)
  const uint32_t g0 = tfirst[bid];
  const uint32_t g1 = bid + 1 < ntile ? tfirst[bid + 1] : nrec - 1;
  const bool staged = g1 - g0 < (uint32_t)kRbRecCap;
  for (uint32_t g = g0 + threadIdx.x; g <= g1; g += kRbThreads) {
    const uint32_t x = eoff[g];
    if (staged) {
      s_x[g - g0] = x;
      s_r[g - g0] = rec_sorted[g];
      s_h[g - g0] = slots[4ull * g];
    }
    if (g == g0) continue;
    const uint32_t xe = g + 1 < nrec ? eoff[g + 1] : NE;
    if (xe > x && x < J0 + (uint32_t)nh) s_g[x - J0] = g - g0;
  }
  __syncthreads();
  {  // running max over positions (blocked: 8 per thread), block exclusive max-scan
    uint32_t mloc = 0;
#pragma unroll
    for (int q = 0; q < kRbEPT; ++q) mloc = max(mloc, s_g[threadIdx.x * kRbEPT + q]);
    uint32_t incl = mloc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) incl = max(incl, __shfl_up_sync(0xffffffffu, incl, o) & (lane >= o ? ~0u : 0u));
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    uint32_t carry = 0;
    for (int ww = 0; ww < w; ++ww) carry = max(carry, s_w[ww]);
    const uint32_t ex = __shfl_up_sync(0xffffffffu, incl, 1);
    carry = max(carry, lane > 0 ? ex : 0u);
#pragma unroll
    for (int q = 0; q < kRbEPT; ++q) {
      carry = max(carry, s_g[threadIdx.x * kRbEPT + q]);
      s_g[threadIdx.x * kRbEPT + q] = carry;
    }
  }
  __syncthreads();
  // ---- decode (warp-striped: warp w owns positions [w*256, w*256+256)): all
  // global loads of the thread's entries first, then the ranking
  uint4 ent[kRbEPT];
#pragma unroll
  for (int q = 0; q < kRbEPT; ++q) {
    const int p = w * 32 * kRbEPT + q * 32 + lane;
    ent[q] = make_uint4(0u, 0xFFFF0000u, 0u, 0u);  // row field 0xFFFF: no entry
    if (p < nh) {
      const uint32_t gl = s_g[p];
      const uint32_t g = g0 + gl;
      uint32_t x, r;
      uint4 h;
      if (staged) {
        x = s_x[gl];
        r = s_r[gl];
        h = s_h[gl];
      } else {
        x = eoff[g];
        r = rec_sorted[g];
        h = slots[4ull * g];
      }
      const uint32_t sub = J0 + (uint32_t)p - x;
      if (h.x & kSlotOverflow) {
        ent[q] = bigent[h.y + sub];
        ent[q].x = r;
      } else {
        const uint2 mk = reinterpret_cast<const uint2*>(slots + 4ull * g + 1)[sub];
        const uint32_t row = (h.x & 0xFFFFu) + sub;
        ent[q] = make_uint4(r, (row << 16) | (h.y & 0xFFFFu), mk.x, mk.y);
      }
    }
  }
  uint32_t dl[kRbEPT];  // digit | rank << 10
#pragma unroll
  for (int q = 0; q < kRbEPT; ++q) {
    const bool ok = (ent[q].y >> 16) != 0xFFFFu;
    const uint32_t d = ok ? (uint32_t)(ent_row(ent[q]) - c_fp.row0) : 0u;
    const unsigned peers = warp_peers<NB>(d, ok);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (ok && lane == leader) old = atomicAdd(&s_cnt[w][d], (uint32_t)__popc(peers));
    old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
    dl[q] = ok ? (d | ((old + __popc(peers & lt)) << 10)) : 0xFFFFFFFFu;
  }
  __syncthreads();
  // ---- per digit: warp offsets, publish, block-local offsets, look-back
  const unsigned long long hiA = (unsigned long long)((epoch << 2) | 1u) << 32;
  const unsigned long long hiP = (unsigned long long)((epoch << 2) | 2u) << 32;
  uint32_t acc[DPT], loff[DPT];
  uint32_t carryL = 0;
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * 256 + threadIdx.x;
    uint32_t a = 0;
#pragma unroll
    for (int ww = 0; ww < kRbThreads / 32; ++ww) {
      const uint32_t c = s_cnt[ww][d];
      s_cnt[ww][d] = a;
      a += c;
    }
    acc[h] = a;
    st_status(look + (size_t)bid * NDIG + d, (bid == 0 ? hiP : hiA) | a);
  }
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    uint32_t tot;
    loff[h] = carryL + scan_block<kRbThreads>(acc[h], s_w, tot);
    carryL += tot;
  }
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * 256 + threadIdx.x;
#pragma unroll
    for (int ww = 0; ww < kRbThreads / 32; ++ww) s_cnt[ww][d] += loff[h];
  }
  __syncthreads();
  // block-local scatter first, so the look-back wait overlaps it
#pragma unroll
  for (int q = 0; q < kRbEPT; ++q)
    if (dl[q] != 0xFFFFFFFFu) s_e[s_cnt[w][dl[q] & 1023u] + (dl[q] >> 10)] = ent[q];
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * 256 + threadIdx.x;
    uint32_t excl = 0;
    if (bid > 0 && d < nb) {
      excl = lookback4_backoff(look + (size_t)(bid - 1) * NDIG + d, (long long)bid, NDIG, epoch);
      st_status(look + (size_t)bid * NDIG + d, hiP | (excl + acc[h]));
    }
    s_off[d] = (d < nb ? s_rowE[d] : 0u) + excl - loff[h];
  }
  __syncthreads();
  for (int p = threadIdx.x; p < nh; p += kRbThreads) {
    const uint4 e = s_e[p];
    out[s_off[ent_row(e) - c_fp.row0] + (uint32_t)p] = e;
  }
}

// ---------------------------------------------------------------------------
// C0: exclusive scan of the row-bucketed entries' pair counts -> poff (the
// row-major pair index of each entry's first pair), per band tile pair counts
// hist[(row - row0) * TX + col] and cmap[colsort tile] = its first entry.
// 512 threads x 8 entries per CTA, decoupled look-back (as k_scan_onepass).
// ---------------------------------------------------------------------------
constexpr int kRsSpan = 4;  // tile rows of a scan tile counted in shared memory
template <int NDIG>
__global__ void __launch_bounds__(kScanThreads) k_rowscan(
    const uint4* __restrict__ ent, uint32_t NE, const uint32_t* __restrict__ rowtab,
    uint32_t* __restrict__ poff, uint32_t* __restrict__ hist, uint32_t* __restrict__ cmap,
    unsigned long long* __restrict__ look, uint32_t* __restrict__ ticket, uint32_t epoch) {
  __shared__ uint32_t s_warp[33];
  __shared__ uint32_t s_bid, s_pre;
  __shared__ uint32_t s_h[kRsSpan * kRbMaxRows];
  const int TX = c_fp.TX, row0 = c_fp.row0;
  if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
  for (int q = threadIdx.x; q < kRsSpan * kRbMaxRows; q += blockDim.x) s_h[q] = 0u;
  __syncthreads();
  const uint32_t bid = s_bid;
  const long long base = (long long)bid * kScanTile + (long long)threadIdx.x * kScanItems;
  const int rowA = (int)(ent[(long long)bid * kScanTile].y >> 16);
  uint4 e[kScanItems];
  uint32_t vals[kScanItems], v = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    e[q] = (base + q < NE) ? ent[base + q] : make_uint4(0u, 0u, 0u, 0u);
    vals[q] = (uint32_t)__popc(e[q].z) + (uint32_t)__popc(e[q].w);
    v += vals[q];
  }
  uint32_t ex;
  const uint32_t T = block_exclusive_scan<kScanThreads>(v, ex, s_warp);
  const unsigned long long hiA = (unsigned long long)((epoch << 2) | 1u) << 32;
  const unsigned long long hiP = (unsigned long long)((epoch << 2) | 2u) << 32;
  if (threadIdx.x == 0) st_relaxed_u64(look + bid, (bid == 0 ? hiP : hiA) | T);
  // per-tile pair counts in shared memory for the first kRsSpan rows of the
  // scan tile (a contiguous mask, the usual union row: column by column; a
  // mask with holes bit by bit); further rows straight to global memory
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    if (!vals[q]) continue;
    const int ro = ent_row(e[q]), c0 = ent_col(e[q]);
    const int rr = ro - rowA;
    uint32_t* hrow = rr < kRsSpan ? s_h + rr * kRbMaxRows + c0 : hist + (ro - row0) * TX + c0;
    const int lo = __ffsll(((long long)e[q].w << 32) | e[q].z) - 1;
    const int hi = 63 - __clzll(((long long)e[q].w << 32) | e[q].z);
    if ((int)vals[q] == hi - lo + 1) {
      for (int b = lo; b <= hi; ++b) atomicAdd(hrow + b, 1u);
    } else {
      unsigned long long m = ((unsigned long long)e[q].w << 32) | e[q].z;
      while (m) {
        const int b = __ffsll((long long)m) - 1;
        m &= m - 1;
        atomicAdd(hrow + b, 1u);
      }
    }
  }
  if (threadIdx.x == 0) {
    uint32_t excl = 0;
    if (bid > 0) {
      excl = lookback4(look + (bid - 1), (long long)bid, 1, epoch);
      st_relaxed_u64(look + bid, hiP | (excl + T));
    }
    s_pre = excl;
  }
  __syncthreads();
  uint32_t run = s_pre + ex;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    if (base + q < NE) {
      poff[base + q] = run;
      if (vals[q]) {  // colsort tiles of this row that start inside the entry
        const int ro = ent_row(e[q]) - row0;
        const uint32_t rp = rowtab[kRowTab + ro];
        for (uint32_t jt = (run - rp + kRbTP - 1) / kRbTP; rp + jt * kRbTP < run + vals[q]; ++jt)
          cmap[rowtab[2 * kRowTab + ro] + jt] = (uint32_t)(base + q);
      }
    }
    run += vals[q];
  }
  for (int q = threadIdx.x; q < kRsSpan * kRbMaxRows; q += blockDim.x) {
    const int rr = q / kRbMaxRows, col = q % kRbMaxRows;
    const uint32_t c = s_h[q];
    if (c && col < TX) atomicAdd(&hist[(rowA + rr - row0) * TX + col], c);
  }
}

// C1: per band row, tb[t] = row pair base + exclusive prefix over the row's
// columns (512 threads, one column each).
template <int NDIG>
__global__ void __launch_bounds__(512) k_tile_bases(const uint32_t* __restrict__ rowhist,
                                                    const uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ tb) {
  __shared__ uint32_t s_warp[33];
  __shared__ uint32_t s_rowP;
  const int TX = c_fp.TX, ro = blockIdx.x;
  if (threadIdx.x < 32) {  // pair base of row ro: sum of the earlier rows' pair counts
    uint32_t a = 0;
    for (int q = threadIdx.x; q < ro; q += 32) a += rowhist[kRbMaxRows + q];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x == 0) s_rowP = a;
  }
  const uint32_t c = threadIdx.x < TX ? hist[ro * TX + threadIdx.x] : 0u;
  uint32_t ex;
  block_exclusive_scan<512>(c, ex, s_warp);
  if (threadIdx.x < TX) tb[ro * TX + threadIdx.x] = s_rowP + ex;
}

// ---------------------------------------------------------------------------
// C: per tile row, stable counting sort of the row's pairs by tile column.
// Tile = kRbTP consecutive pairs of ONE row; pairs are generated from the
// entries' masks straight into shared memory, ranked by column (NB-bit warp
// multisplit), and placed by a decoupled look-back over the row's earlier
// tiles (the row's first tile publishes its counts as inclusive).
// ---------------------------------------------------------------------------
template <int NDIG>
__global__ void __launch_bounds__(kRbThreads, 3) k_colsort(
    const uint4* __restrict__ ent, const uint32_t* __restrict__ poff, uint32_t NE,
    const uint32_t* __restrict__ rowtab, const uint32_t* __restrict__ cmap,
    const uint32_t* __restrict__ tb, uint32_t* __restrict__ out,
    unsigned long long* __restrict__ look, uint32_t* __restrict__ ctr, uint32_t epoch) {
  constexpr int NB = NDIG == 512 ? 9 : 8;
  constexpr int DPT = NDIG / 256;
  __shared__ uint32_t s_cnt[kRbThreads / 32][NDIG];
  extern __shared__ uint32_t s_kv[];  // [2][kRbTP] column, record; then the staged entries
  uint32_t* s_k = s_kv;
  uint32_t* s_v = s_kv + kRbTP;
  uint4* s_ent = reinterpret_cast<uint4*>(s_kv + 2 * kRbTP);          // [kCsEntCap]
  uint32_t* s_px = s_kv + 2 * kRbTP + 4 * kCsEntCap;                   // [kCsEntCap]
  __shared__ uint32_t s_off[NDIG];
  __shared__ uint32_t s_rowP[NDIG + 1], s_rowT[NDIG + 1];
  __shared__ uint32_t s_w[16];
  __shared__ uint32_t s_bid;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int TX = c_fp.TX, nb = c_fp.row1 - c_fp.row0;
  if (threadIdx.x == 0) s_bid = atomicAdd(ctr, 1u);
  for (int q = threadIdx.x; q < (kRbThreads / 32) * NDIG; q += kRbThreads) (&s_cnt[0][0])[q] = 0;
  for (int q = threadIdx.x; q <= nb; q += kRbThreads) {
    s_rowP[q] = rowtab[kRowTab + q];
    s_rowT[q] = rowtab[2 * kRowTab + q];
  }
  __syncthreads();
  const uint32_t bid = s_bid;
  // the tile's row: last ro with rowT[ro] <= bid (rows without pairs own no tile)
  int lo = 0, hi = nb;  // invariant rowT[lo] <= bid < rowT[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (s_rowT[mid] <= bid) lo = mid; else hi = mid;
  }
  const int ro = lo;
  const uint32_t jt = bid - s_rowT[ro];
  const uint32_t q0 = s_rowP[ro] + jt * kRbTP;
  const uint32_t q1 = min(q0 + (uint32_t)kRbTP, s_rowP[ro + 1]);
  const int nh = (int)(q1 - q0);
  // ---- the tile's pairs (column, r), pairs [q0, q1) of row ro, generated from
  // its entries [e0, e1] (e1 = the next tile's first entry; entries of other
  // rows add nothing).  Staged path (<= kCsEntCap entries): entries in shared
  // memory, each pair position -> its entry by the entries' start marks and a
  // running max, pair = the (offset)-th set bit of the entry's mask (a
  // contiguous mask: first bit + offset).  Otherwise every thread expands its
  // entries into shared memory and the ranking reads them back.
  const uint32_t e0 = cmap[bid];
  const uint32_t e1 = bid + 1 < gridDim.x ? min(cmap[bid + 1], NE - 1) : NE - 1;
  const uint32_t ne = e1 - e0 + 1;
  uint32_t vr[kRbIPT], dl[kRbIPT];
  if (ne <= (uint32_t)kCsEntCap) {
    uint32_t* s_m = s_k;  // pair position -> entry (until the sorted scatter)
    for (int q = threadIdx.x; q < kRbTP; q += kRbThreads) s_m[q] = 0u;
    for (uint32_t i = threadIdx.x; i < ne; i += kRbThreads) {
      s_ent[i] = ent[e0 + i];
      s_px[i] = poff[e0 + i];
    }
    __syncthreads();
    for (uint32_t i = 1 + threadIdx.x; i < ne; i += kRbThreads) {
      const uint32_t x = s_px[i];
      const uint4 en = s_ent[i];
      if ((en.z | en.w) && x < q1) s_m[x - q0] = i;  // x > q0 for every entry after e0
    }
    __syncthreads();
    {  // running max over positions (blocked: kRbIPT per thread)
      uint32_t mloc = 0;
#pragma unroll
      for (int q = 0; q < kRbIPT; ++q) mloc = max(mloc, s_m[threadIdx.x * kRbIPT + q]);
      uint32_t incl = mloc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1)
        incl = max(incl, __shfl_up_sync(0xffffffffu, incl, o) & (lane >= o ? ~0u : 0u));
      if (lane == 31) s_w[w] = incl;
      __syncthreads();
      uint32_t carry = 0;
      for (int ww = 0; ww < w; ++ww) carry = max(carry, s_w[ww]);
      const uint32_t ex = __shfl_up_sync(0xffffffffu, incl, 1);
      carry = max(carry, lane > 0 ? ex : 0u);
#pragma unroll
      for (int q = 0; q < kRbIPT; ++q) {
        carry = max(carry, s_m[threadIdx.x * kRbIPT + q]);
        s_m[threadIdx.x * kRbIPT + q] = carry;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kRbIPT; ++q) {
      const int p = w * 32 * kRbIPT + q * 32 + lane;
      const bool ok = p < nh;
      uint32_t d = 0;
      vr[q] = 0u;
      if (ok) {
        const uint32_t i = s_m[p];
        const uint4 en = s_ent[i];
        const uint32_t kin = q0 + (uint32_t)p - s_px[i];  // pair offset within the entry
        const unsigned long long m = ((unsigned long long)en.w << 32) | en.z;
        const int lo = __ffsll((long long)m) - 1;
        int bit;
        if (((m >> lo) & (((m >> lo) + 1ull))) == 0ull) {  // contiguous run of bits
          bit = lo + (int)kin;
        } else {
          const int pl = __popc(en.z);
          bit = (int)kin < pl ? nth_set_bit(en.z, (int)kin) : 32 + nth_set_bit(en.w, (int)kin - pl);
        }
        d = (uint32_t)(ent_col(en) + bit);
        vr[q] = en.x;
      }
      const unsigned peers = warp_peers<NB>(d, ok);
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (ok && lane == leader) old = atomicAdd(&s_cnt[w][d], (uint32_t)__popc(peers));
      old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
      dl[q] = ok ? (d | ((old + __popc(peers & lt)) << 10)) : 0xFFFFFFFFu;
    }
  } else {
    for (uint32_t eb = e0; eb <= e1; eb += 8 * kRbThreads) {
      uint4 en[8];
      uint32_t xs[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t e = eb + (uint32_t)(i * kRbThreads) + threadIdx.x;
        xs[i] = 0xFFFFFFFFu;
        if (e <= e1) {
          xs[i] = poff[e];
          en[i] = ent[e];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t x = xs[i];
        if (x == 0xFFFFFFFFu || x >= q1) continue;
        const uint32_t pv = (uint32_t)__popc(en[i].z) + (uint32_t)__popc(en[i].w);
        if (x + pv <= q0) continue;
        unsigned long long m = ((unsigned long long)en[i].w << 32) | en[i].z;
        const int c0 = ent_col(en[i]);
        uint32_t pos = x;
        while (pos < q0) {  // an entry split across tiles: skip its earlier pairs
          m &= m - 1;
          ++pos;
        }
        while (m && pos < q1) {
          const int b = __ffsll((long long)m) - 1;
          m &= m - 1;
          s_k[pos - q0] = (uint32_t)(c0 + b);
          s_v[pos - q0] = en[i].x;
          ++pos;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kRbIPT; ++q) {
      const int p = w * 32 * kRbIPT + q * 32 + lane;
      const bool ok = p < nh;
      const uint32_t d = ok ? s_k[p] : 0u;
      vr[q] = ok ? s_v[p] : 0u;
      const unsigned peers = warp_peers<NB>(d, ok);
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (ok && lane == leader) old = atomicAdd(&s_cnt[w][d], (uint32_t)__popc(peers));
      old = __shfl_sync(0xffffffffu, old, leader < 0 ? 0 : leader);
      dl[q] = ok ? (d | ((old + __popc(peers & lt)) << 10)) : 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  const unsigned long long hiA = (unsigned long long)((epoch << 2) | 1u) << 32;
  const unsigned long long hiP = (unsigned long long)((epoch << 2) | 2u) << 32;
  uint32_t acc[DPT], loff[DPT];
  uint32_t carryL = 0;
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * 256 + threadIdx.x;
    uint32_t a = 0;
#pragma unroll
    for (int ww = 0; ww < kRbThreads / 32; ++ww) {
      const uint32_t c = s_cnt[ww][d];
      s_cnt[ww][d] = a;
      a += c;
    }
    acc[h] = a;
    st_status(look + (size_t)bid * NDIG + d, (jt == 0 ? hiP : hiA) | a);
  }
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    uint32_t tot;
    loff[h] = carryL + scan_block<kRbThreads>(acc[h], s_w, tot);
    carryL += tot;
  }
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * 256 + threadIdx.x;
#pragma unroll
    for (int ww = 0; ww < kRbThreads / 32; ++ww) s_cnt[ww][d] += loff[h];
  }
  __syncthreads();
  // block-local scatter first, so the look-back wait overlaps it
#pragma unroll
  for (int q = 0; q < kRbIPT; ++q)
    if (dl[q] != 0xFFFFFFFFu) {
      const uint32_t d = dl[q] & 1023u, pp = s_cnt[w][d] + (dl[q] >> 10);
      s_v[pp] = vr[q];
      s_k[pp] = d;
    }
#pragma unroll
  for (int h = 0; h < DPT; ++h) {
    const int d = h * 256 + threadIdx.x;
    uint32_t excl = 0;
    if (jt > 0 && d < TX) {
      excl = lookback4_backoff(look + (size_t)(bid - 1) * NDIG + d, (long long)jt, NDIG, epoch);
      st_status(look + (size_t)bid * NDIG + d, hiP | (excl + acc[h]));
    }
    s_off[d] = (d < TX ? tb[ro * TX + d] : 0u) + excl - loff[h];
  }
  __syncthreads();
  for (int p = threadIdx.x; p < nh; p += kRbThreads) out[s_off[s_k[p]] + (uint32_t)p] = s_v[p];
}

// R: [S, E) of every (band tile, k): lists are k-sorted, so binary search on
// k(r) = r / M (one thread per (tile, k)).
__global__ void k_ranges_rb(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ tb,
                            const uint32_t* __restrict__ hist, uint32_t* __restrict__ S,
                            uint32_t* __restrict__ E) {
  const int TX = c_fp.TX, K = c_fp.K;
  const long long n = (long long)(c_fp.row1 - c_fp.row0) * TX * K;
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int tl = (int)(q / K), k = (int)(q % K);
  const uint32_t b = tb[tl], e = b + hist[tl];
  auto lower = [&](uint32_t key) {  // first position in [b, e) with k(r) >= key
    uint32_t lo = b, hi = e;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (fdiv(vals[mid], c_fp.divM) < key) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const long long t = (long long)c_fp.row0 * TX + tl;
  const uint32_t s0 = lower((uint32_t)k), s1 = lower((uint32_t)k + 1);
  S[t * K + k] = s1 > s0 ? s0 : 0u;  // an empty list is [0, 0)
  E[t * K + k] = s1 > s0 ? s1 : 0u;
}

// Introspection: the (t, k) slot of every sorted pair (the key the LSD path's
// last pass writes), from the ranges.
__global__ void k_fill_slots(const uint32_t* __restrict__ S, const uint32_t* __restrict__ E,
                             uint32_t* __restrict__ slot) {
  const int TX = c_fp.TX, K = c_fp.K;
  const long long n = (long long)(c_fp.row1 - c_fp.row0) * TX * K;
  for (long long q = blockIdx.x; q < n; q += gridDim.x) {
    const long long t = (long long)c_fp.row0 * TX + q / K;
    const uint32_t sk = (uint32_t)(t * K + q % K);
    for (uint32_t e = S[sk] + threadIdx.x; e < E[sk]; e += blockDim.x) slot[e] = sk;
  }
}

}  // namespace cr
