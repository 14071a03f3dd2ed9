// cr_kernels.cuh — display (view map, Ψ, composite work items), upload,
// preprocess, tile-union count, emission and range kernels of the
// CoherentRaster B200 path.  See DESIGN.md §5 for the
// roofline of each kernel and its algorithmic bytes per unit.
#pragma once
#include <cuda_fp16.h>

#include "cr_device.cuh"

namespace cr {

// ===========================================================================
// a1 — View-number map (Eqs.1-3), fp64 with explicit rounding.
// One thread per subpixel, u8 [H][W][3].
// ===========================================================================
__global__ void k_viewmap(uint8_t* __restrict__ V, int W, int H, int N, double Lx, double tA,
                          double Koff) {
  const long long n = (long long)W * H * 3;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int u = (int)(g % 3);
    const long long p = g / 3;
    const int x = (int)(p % W), y = (int)(p / W);
    const double s = (double)(3 * x + u);
    const double t1 = __dmul_rn((double)(3 * y), tA);
    const double d = __dsub_rn(__dadd_rn(s, t1), Koff);   // Eq.1
    const double q = floor(__ddiv_rn(d, Lx));
    double xo = __dsub_rn(d, __dmul_rn(q, Lx));           // Eq.2
    if (xo < 0) xo = __dadd_rn(xo, Lx);
    if (xo >= Lx) xo = __dsub_rn(xo, Lx);
    int j = (int)floor(__ddiv_rn(__dmul_rn((double)N, xo), Lx));  // Eq.3
    j = j < 0 ? 0 : (j > N - 1 ? N - 1 : j);
    V[g] = (uint8_t)j;
  }
}

// ===========================================================================
// a2 — View-coherent Remapping table Psi (Eq.8): per tile, stable
// counting sort of the local subpixel indices l = (ly*16+lx)*3+u by V.
// One warp per tile; ties keep row-major order (match_any ranks, chunk order).
// ===========================================================================
__global__ void k_remap_build(const uint8_t* __restrict__ V, uint16_t* __restrict__ psi, int W,
                              int H, int TX, int TY) {
  __shared__ unsigned s_hist[8][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + w;
  unsigned* hist = s_hist[w];
  for (int b = lane; b < 256; b += 32) hist[b] = 0;
  __syncwarp();
  if (t >= TX * TY) return;
  const int tx = t % TX, ty = t / TX;
  auto val = [&](int l) -> int {
    const int ly = l / 48, rem = l % 48, lx = rem / 3, u = rem % 3;
    const int x = tx * 16 + lx, y = ty * 16 + ly;
    if (x >= W || y >= H) return 256;  // not in the panel
    return V[((long long)y * W + x) * 3 + u];
  };
  for (int c = 0; c < 24; ++c) {
    const int v = val(c * 32 + lane);
    if (v < 256) atomicAdd(&hist[v], 1u);
  }
  __syncwarp();
  // exclusive scan of 256 bins: 8 consecutive bins per lane
  unsigned loc[8], sum = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) { loc[q] = hist[lane * 8 + q]; sum += loc[q]; }
  unsigned incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const unsigned nvalid = __shfl_sync(0xffffffffu, incl, 31);
  unsigned run = incl - sum;
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 8; ++q) { hist[lane * 8 + q] = run; run += loc[q]; }
  __syncwarp();
  uint16_t* out = psi + (long long)t * kTileSub;
  const unsigned lt = (1u << lane) - 1u;
  for (int c = 0; c < 24; ++c) {
    const int l = c * 32 + lane;
    const int v = val(l);
    const unsigned peers = __match_any_sync(0xffffffffu, v);
    const unsigned rank = __popc(peers & lt);
    unsigned base = 0;
    if (v < 256) base = hist[v];
    __syncwarp();
    if (v < 256) {
      out[base + rank] = (uint16_t)l;
      if (rank == 0) hist[v] = base + __popc(peers);
    }
    __syncwarp();
  }
  for (int r = nvalid + lane; r < kTileSub; r += 32) out[r] = 0xFFFF;
}

// Composite work items: per tile, "cluster-aligned chunks" of <= kChunkMax
// consecutive Psi ranks that share one cluster k (DESIGN.md §5 composite).
// Packed as start | (len-1) << 10 | k << 16.  One thread per tile.
constexpr int kChunkMax = 32;
__global__ void k_chunks_build(const uint8_t* __restrict__ V, const uint16_t* __restrict__ psi,
                               uint32_t* __restrict__ chunks, uint32_t* __restrict__ nchunks,
                               int stride, int W, int TX, int TY, int s) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= TX * TY) return;
  const int tx = t % TX, ty = t / TX;
  const uint16_t* ps = psi + (long long)t * kTileSub;
  uint32_t* out = chunks + (long long)t * stride;
  int n = 0, seg_k = -1, seg_start = 0;
  for (int r = 0; r < kTileSub; ++r) {
    const int l = ps[r];
    if (l == 0xFFFF) break;
    const int ly = l / 48, rem = l % 48, lx = rem / 3, u = rem % 3;
    const int j = V[((long long)(ty * 16 + ly) * W + tx * 16 + lx) * 3 + u];
    const int k = j / s;
    if (k != seg_k || r - seg_start == kChunkMax) {
      if (seg_k >= 0) out[n++] = (uint32_t)seg_start | ((uint32_t)(r - seg_start - 1) << 10) |
                                 ((uint32_t)seg_k << 16);
      seg_k = k;
      seg_start = r;
    }
    if (r == kTileSub - 1 || ps[r + 1] == 0xFFFF) {
      out[n++] = (uint32_t)seg_start | ((uint32_t)(r - seg_start) << 10) | ((uint32_t)seg_k << 16);
    }
  }
  nchunks[t] = n;
}

// Paired work items for the two-subpixels-per-lane composite: per tile, the
// Psi order with every view run padded to an even length (hole 0xFFFF), so
// slot pairs (2i, 2i+1) always hold two subpixels of ONE view (or one and a
// hole); psi2 [T][kPairSlots] u16 (<= 768 subpixels + one hole per run).
// Each cluster segment is cut into ceil(len/64) equal even-length chunks
// (greedy: 64-slot chunks and the remainder),
// packed as start_slot | (lanes-1) << 10 | k << 16 (a lane takes one pair).
__global__ void k_pairs_build(const uint8_t* __restrict__ V, const uint16_t* __restrict__ psi,
                              uint16_t* __restrict__ psi2, uint32_t* __restrict__ chunks,
                              uint32_t* __restrict__ nchunks, int stride, int W, int TX, int TY,
                              int s, int greedy) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= TX * TY) return;
  const int tx = t % TX, ty = t / TX;
  const uint16_t* ps = psi + (long long)t * kTileSub;
  uint16_t* o2 = psi2 + (long long)t * kPairSlots;
  uint32_t* out = chunks + (long long)t * stride;
  int n = 0, nc = 0, cur_j = -1, cur_k = -1, seg = 0, run = 0;
  auto close_seg = [&](int end) {  // cut [seg, end) into equal even chunks of <= 64 slots
    const int len = end - seg;
    if (len <= 0 || cur_k < 0) return;
    const int np = (len + 63) / 64;
    const int per = greedy ? 64 : 2 * ((len / 2 + np - 1) / np);  // full warps first, or equal
    for (int a = seg; a < end; a += per) {
      const int ln = min(per, end - a);
      out[nc++] = (uint32_t)a | ((uint32_t)(ln / 2 - 1) << 10) | ((uint32_t)cur_k << 16);
    }
  };
  for (int r = 0; r < kTileSub; ++r) {
    const int l = ps[r];
    if (l == 0xFFFF) break;
    const int ly = l / 48, rem = l % 48, lx = rem / 3, u = rem % 3;
    const int j = V[((long long)(ty * 16 + ly) * W + tx * 16 + lx) * 3 + u];
    if (j != cur_j) {
      if (run & 1) o2[n++] = 0xFFFF;
      run = 0;
      const int k = j / s;
      if (k != cur_k) {
        close_seg(n);
        seg = n;
        cur_k = k;
      }
      cur_j = j;
    }
    o2[n++] = (uint16_t)l;
    ++run;
  }
  if (run & 1) o2[n++] = 0xFFFF;
  close_seg(n);
  nchunks[t] = nc;
}

// ===========================================================================
// Upload (O4): Sigma3D = R S S^T R^T in fp64 with explicit rounding (same
// order as written in DESIGN.md O4), SH transposed to coefficient-major SoA.
// mean4 = (mu, tau), cov8 = {S00,S01,S02,S11},{S12,S22,o,0}.
// ===========================================================================
// Validation pass over the staged inputs: any NaN/Inf sets *nonfinite.
// Runs before the scene buffers are touched, so a rejected upload leaves the
// previous scene intact (header: "on error the context keeps its state").
__global__ void k_validate(long long n, const float* __restrict__ x, int* __restrict__ nonfinite) {
  bool bad = false;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(x[q]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

__global__ void k_upload(long long M, int nc3, const float* __restrict__ means,
                         const float* __restrict__ quats, const float* __restrict__ scales,
                         const float* __restrict__ opac, const float* __restrict__ tau,
                         const float* __restrict__ sh, float4* __restrict__ mean4,
                         float4* __restrict__ cov8, float* __restrict__ shsoa) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= M) return;
  float q4[4], s3[3], m3[3];
#pragma unroll
  for (int a = 0; a < 4; ++a) q4[a] = quats[4 * i + a];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    s3[a] = scales[3 * i + a];
    m3[a] = means[3 * i + a];
  }
  const float o = opac[i];
  double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
  const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w, w), __dmul_rn(x, x)),
                                                  __dmul_rn(y, y)),
                                        __dmul_rn(z, z)));
  w = __ddiv_rn(w, n); x = __ddiv_rn(x, n); y = __ddiv_rn(y, n); z = __ddiv_rn(z, n);
  double R[3][3];
  R[0][0] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, y), __dmul_rn(z, z))));
  R[0][1] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
  R[0][2] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
  R[1][0] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
  R[1][1] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(z, z))));
  R[1][2] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
  R[2][0] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
  R[2][1] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
  R[2][2] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y))));
  const double ss[3] = {__dmul_rn((double)s3[0], (double)s3[0]),
                        __dmul_rn((double)s3[1], (double)s3[1]),
                        __dmul_rn((double)s3[2], (double)s3[2])};
  const int IA[6] = {0, 0, 0, 1, 1, 2}, IB[6] = {0, 1, 2, 1, 2, 2};
  float c6[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const int a = IA[e], b = IB[e];
    const double v = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(R[a][0], ss[0]), R[b][0]),
                                         __dmul_rn(__dmul_rn(R[a][1], ss[1]), R[b][1])),
                               __dmul_rn(__dmul_rn(R[a][2], ss[2]), R[b][2]));
    c6[e] = __double2float_rn(v);
  }
  mean4[i] = make_float4(m3[0], m3[1], m3[2], tau[i]);
  cov8[2 * i] = make_float4(c6[0], c6[1], c6[2], c6[3]);
  cov8[2 * i + 1] = make_float4(c6[4], c6[5], o, 0.0f);
  for (int q = 0; q < nc3; ++q) shsoa[(long long)q * M + i] = sh[(long long)i * nc3 + q];
}

// ===========================================================================
// Cameras staged in shared memory with an 80-byte stride (20 floats): the 8
// consecutive cameras a G=8 lane group reads hit 8 distinct 16-byte bank
// groups, and each camera is 4 x LDS.128.
// ===========================================================================
constexpr int kCamStride = 20;
__device__ __forceinline__ void stage_cams(float* s_cam) {
  const int N = c_fp.N;
  for (int q = threadIdx.x; q < N * 16; q += blockDim.x) {
    const int j = q >> 4, f = q & 15;
    s_cam[j * kCamStride + f] = (&c_cams[j].R[0])[f];
  }
}
__device__ __forceinline__ CamDev load_cam(const float* s_cam, int j) {
  const float4* q4 = reinterpret_cast<const float4*>(s_cam + j * kCamStride);
  const float4 c0 = q4[0], c1 = q4[1], c2 = q4[2], c3 = q4[3];
  CamDev c;
  c.R[0] = c0.x; c.R[1] = c0.y; c.R[2] = c0.z; c.R[3] = c0.w;
  c.R[4] = c1.x; c.R[5] = c1.y; c.R[6] = c1.z; c.R[7] = c1.w;
  c.R[8] = c2.x; c.t[0] = c2.y; c.t[1] = c2.z; c.t[2] = c2.w;
  c.fx = c3.x; c.fy = c3.y; c.cx = c3.z; c.cy = c3.w;
  return c;
}

// Group-of-G-lane reductions (G a power of two, groups aligned in the warp).
// Every caller keeps the WHOLE warp converged (warp-uniform loops), so the
// shuffles use the full mask and stay inside the group via offsets < G.
template <int G>
__device__ __forceinline__ int gmin(int v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ int gmax(int v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int G>
__device__ __forceinline__ unsigned long long gor64(unsigned long long v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// len set bits from bit pos (pos < 32, len >= 1; bits past 31 dropped): one BMSK
__device__ __forceinline__ unsigned bmsk32(int pos, int len) {
  unsigned r;
  asm("bmsk.clamp.b32 %0, %1, %2;" : "=r"(r) : "r"(pos), "r"(len));
  return r;
}

// Position of the n-th (0-based) set bit of x (n < popc(x)): popcount
// bisection over halves, bytes, nibbles, pairs — branch-free, ~20 ALU ops
// (the __fns intrinsic is a much longer software sequence).
__device__ __forceinline__ int nth_set_bit(unsigned x, int n) {
  int pos = 0;
  int c = __popc(x & 0xFFFFu);
  if (n >= c) { n -= c; x >>= 16; pos += 16; }
  c = __popc(x & 0xFFu);
  if (n >= c) { n -= c; x >>= 8; pos += 8; }
  c = __popc(x & 0xFu);
  if (n >= c) { n -= c; x >>= 4; pos += 4; }
  c = __popc(x & 0x3u);
  if (n >= c) { n -= c; x >>= 2; pos += 2; }
  return pos + ((n >= (int)(x & 1u)) ? 1 : 0);
}

// ===========================================================================
// O8 — cluster tile union (Alg.2 GenerateKeys) restricted to the
// band rows, computed by a GROUP of G lanes: lane v of the group owns view
// j = k*s + v of cluster k (exact per-view mean, Eq.5, and AccuTile rows /
// per-row columns, O7); per tile row the views' column intervals are merged
// by shuffles into 64-bit masks over 64-column windows.  MODE 0 counts; MODE 2 also writes the tile ids (rows ascending,
// columns ascending) + payload r.  This is the GENERAL path (any footprint);
// k_count's fast path handles records of <= kSlotRows rows and < 64 columns
// and produces the same set (same exactly-rounded per-(view,row) code).
// Must be called by all 32 lanes of the warp (inactive groups: active=false).
// ===========================================================================
constexpr int kSlotRows = 6;               // rows of a 64-byte union slot
constexpr uint32_t kSlotOverflow = 0x80000000u;

template <int MODE, int G>
__device__ uint32_t group_union(const float* s_cam, bool active, int k, int v, float mux,
                                float muy, float muz, const EllRec& el, int it0, int istep,
                                uint32_t* __restrict__ row_cnt, const uint32_t* __restrict__ row_off,
                                uint32_t* __restrict__ out_t, uint32_t* __restrict__ out_v,
                                uint32_t payload, unsigned long long* __restrict__ row_mask = nullptr,
                                int* __restrict__ row_wlo = nullptr, int* __restrict__ wide = nullptr,
                                int row_cap = 1 << 30, int* __restrict__ nrows_out = nullptr,
                                int wbeg = 0, int wend = 1 << 30) {
  // MODE 0: count the group's rows; MODE 3: also store per-row counts in
  // row_cnt[it - wbeg] (and, with row_mask, the row's 64-column window mask and
  // the tile id of its bit 0; *wide = 1 if a row needs more than one window);
  // MODE 2: write the tiles of row it at row_off[it - wbeg] + rank.
  // The group handles union rows it = it0, it0 + istep, ... restricted to the
  // row window [wbeg, wend) (callers with bounded per-row arrays walk a tall
  // union window by window); stores need it - wbeg < row_cap.
  const int s = c_fp.s, N = c_fp.N, TX = c_fp.TX, TY = c_fp.TY;
  const int j = k * s + v;
  bool vis = false;
  float mx = 0.f, my = 0.f;
  int ty0 = 0x7fffffff, ty1 = -1;
  if (active && v < s && j < N) {
    const CamDev cam = load_cam(s_cam, j);
    const F3 p = cam_point_exact(cam, mux, muy, muz);
    if (p.z >= c_fp.znear) {  // Z12: a view that cannot see i contributes no tiles
      mean2d_exact(cam, p, mx, my);
      view_rows(el, my, TY, ty0, ty1);
      vis = true;
    }
  }
  const int rmin = max(gmin<G>(vis ? ty0 : 0x7fffffff), c_fp.row0);
  const int rmax = min(gmax<G>(vis ? ty1 : -1), c_fp.row1 - 1);
  const int nrows = (active && rmax >= rmin) ? rmax - rmin + 1 : 0;
  if (MODE == 3 && nrows_out && (threadIdx.x & 31) == 0) *nrows_out = nrows;
  const int rend = min(nrows, wend);
  const int mine = rend > it0 ? (rend - it0 + istep - 1) / istep : 0;
  const int ii_lo = wbeg > it0 ? (wbeg - it0 + istep - 1) / istep : 0;
  const int it_max = __reduce_max_sync(0xffffffffu, mine);
  const int ii_min = __reduce_min_sync(0xffffffffu, (unsigned)ii_lo);
  const bool lead = (threadIdx.x & (G - 1)) == 0;
  uint32_t n = 0;
  for (int ii = ii_min; ii < it_max; ++ii) {
    const int it = it0 + ii * istep;
    const int ty = rmin + it;
    const int il = it - wbeg;  // index into the window's per-row arrays
    const bool rowok = ii < mine && ii >= ii_lo;
    int tx0 = 0x7fffffff, tx1 = -1;
    if (rowok && vis && ty >= ty0 && ty <= ty1) {
      int q0, q1;
      if (view_row_cols(el, mx, my, ty, TX, q0, q1) && q0 <= q1) {
        tx0 = q0;
        tx1 = q1;
      }
    }
    const int lo = gmin<G>(tx0), hi = gmax<G>(tx1);
    const bool any = rowok && hi >= lo;
    const uint32_t rowbase = (uint32_t)ty * (uint32_t)TX;
    uint32_t rowpos = (MODE == 2 && rowok) ? row_off[il] : 0u;
    uint32_t rown = 0;
    // merge the views' intervals in 64-column windows (one window unless the
    // row spans >= 64 tiles), warp-uniform window count
    const int nwin = any ? ((hi - lo) >> 6) + 1 : 0;
    const int wmax = __reduce_max_sync(0xffffffffu, nwin);
    for (int wi = 0; wi < wmax; ++wi) {
      const int wlo = lo + (wi << 6);
      unsigned long long mask = 0ull;
      if (wi < nwin && tx1 >= tx0) {
        const int a0 = max(tx0, wlo), a1 = min(tx1, wlo + 63);
        if (a0 <= a1) {
          const int len = a1 - a0 + 1;
          mask = ((len >= 64) ? ~0ull : ((1ull << len) - 1ull)) << (a0 - wlo);
        }
      }
      mask = gor64<G>(mask);
      if (wi < nwin) {
        const int pc = __popcll(mask);
        if (MODE == 2) {  // the group's lanes write ranks v, v+G, ... (ascending tiles)
          const unsigned lo32 = (unsigned)mask, hi32 = (unsigned)(mask >> 32);
          const int pl = __popc(lo32);
          for (int q = (int)(threadIdx.x & (G - 1)); q < pc; q += G) {
            const int bit = q < pl ? nth_set_bit(lo32, q) : 32 + nth_set_bit(hi32, q - pl);
            out_t[rowpos + q] = rowbase + (uint32_t)(wlo + bit);
            out_v[rowpos + q] = payload;
          }
          rowpos += (uint32_t)pc;
        }
        rown += (uint32_t)pc;
        if (MODE == 3 && row_mask && lead && rowok && wi == 0 && il < row_cap) {
          row_mask[il] = mask;
          row_wlo[il] = (int)(rowbase + (uint32_t)wlo);  // tile id of the mask's bit 0
        }
      }
    }
    if (MODE == 3 && row_mask && lead && rowok && nwin > 1) *wide = 1;
    if (MODE == 3 && lead && rowok && il < row_cap) row_cnt[il] = rown;
    n += rown;
  }
  return n;
}

// ===========================================================================
// a4 — Preprocess + SH (Cross-view Coherent Attribute Reuse, Eq.6).
// One thread per Gaussian, looping over the K clusters so the SH
// coefficients are read once and evaluated K times.  Per (k,i), r = k*M + i:
//   rec[2r]   = (A', B', C', log2 o)  conic prescaled by -log2(e)/2, -log2(e)
//   rec[2r+1] = (r, g, b, ext)        colour at v'_k; ext = half2 (ex, ey) extents
//   (one 32-byte aligned record: a composite gather touches one DRAM sector)
//   geom[2r..2r+1] = exact AccuTile constants (ex, ey, dyR, tc), (1/c, b, det)
//   dkey[r] = bits(d_{i,k}),  vis[r] = 1 if (i,k) survives culling, else 0
// ===========================================================================
constexpr float kLog2e = 1.4426950408889634f;

// Per-view variant of the pre-cull (clusters spanning wide camera motions,
// where the rigid-motion bound below is loose): with
// fast FMA math and a rigorous padding for its rounding (|p_fast - p_exact| <=
// ~1e-6 (|mu|_1 + |t|_1) per coordinate), decide whether ANY view of cluster
// k could give the record a tile in the band rows x frame columns.  When this
// returns false the exact union (O8) is empty, so skipping the record changes
// no result; when in doubt (near-znear depths) it returns true.
__device__ __forceinline__ bool may_touch_band_views(int k, float mx, float my, float mz, float exw,
                                               float eyw) {
  const int s = c_fp.s, N = c_fp.N;
  const int j0 = k * s, j1 = min(j0 + s, N);
  const float S = fabsf(mx) + fabsf(my) + fabsf(mz);
  const float ylo = 16.0f * (float)c_fp.row0 - 16.0f, yhi = 16.0f * (float)c_fp.row1 + 16.0f;
  const float xlo = -16.0f, xhi = 16.0f * (float)c_fp.TX + 16.0f;
  bool hit = false;
  for (int j = j0; j < j1; ++j) {  // j is warp-uniform (one k per launch-wide loop step)
    const CamDev& c = c_cams[j];
    const float px = fmaf(c.R[0], mx, fmaf(c.R[1], my, fmaf(c.R[2], mz, c.t[0])));
    const float py = fmaf(c.R[3], mx, fmaf(c.R[4], my, fmaf(c.R[5], mz, c.t[1])));
    const float pz = fmaf(c.R[6], mx, fmaf(c.R[7], my, fmaf(c.R[8], mz, c.t[2])));
    const float err = 4e-6f * (S + fabsf(c.t[0]) + fabsf(c.t[1]) + fabsf(c.t[2]) + 1.0f);
    if (pz + err < c_fp.znear) continue;        // certainly invisible from view j
    if (pz < 2.0f * c_fp.znear + err) {         // too close to call
      hit = true;
      continue;
    }
    const float iz = __fdividef(1.0f, pz);  // approximate: covered by the padding
    const float u = px * iz, v = py * iz;
    const float ex = c.fx * u + c.cx, ey = c.fy * v + c.cy;
    const float mgx = c.fx * err * iz * (1.0f + fabsf(u)) * 2.0f + 1e-5f * fabsf(ex) + 1.0f;
    const float mgy = c.fy * err * iz * (1.0f + fabsf(v)) * 2.0f + 1e-5f * fabsf(ey) + 1.0f;
    const bool in = ey + eyw + mgy >= ylo && ey - eyw - mgy <= yhi && ex + exw + mgx >= xlo &&
                    ex - exw - mgx <= xhi;
    hit |= in;  // no early exit: the warp stays converged over the cluster's views
  }
  return hit;
}

// Conservative band / frame pre-cull of an (i,k) record (exactness-safe).
// Only the representative view is projected, from the record's exact
// camera-space point p: every view j of cluster k sees p_j = A_j p + b_j, and
// |p_j - p| <= D = dA |p - c| + db (c_clb: rigid-motion bound of the cluster
// about its least-squares fixed point c, fp64 on the host, rounded up), so
// view j's image x lies within fx (D_x + |p.x/p.z| D_z) / (p.z - D_z) of the
// rep's (same for y), with per-axis bounds D_a (c_clax / c_clbx).  When even the box grown by that shift (and by pads for fp32
// rounding: 1 %, 2e-5 relative, 3 px) misses the band rows x frame columns, no
// view can give the record a tile there: the exact union (O8) is empty and
// skipping the record changes no result.  Near-znear depths return true.
// Used when every cluster's rotation bound dA < kMotionBoundMax (narrow
// clusters, e.g. config C: preprocess 1.78 -> 1.02 ms for 5 % more surviving
// records, all with empty unions); wider clusters (B, E, P2K, P4K) keep the
// per-view test, where the bound would let through up to 27 % more records.
constexpr float kMotionBoundMax = 0.08f;
__device__ __forceinline__ bool may_touch_band(int k, int jr, const F3& p, float exw,
                                               float eyw) {
  const float ylo = 16.0f * (float)c_fp.row0 - 16.0f, yhi = 16.0f * (float)c_fp.row1 + 16.0f;
  const float xlo = -16.0f, xhi = 16.0f * (float)c_fp.TX + 16.0f;
  const CamDev& c = c_cams[jr];
  const float4 cl = c_clb[k], ax = c_clax[k], bx = c_clbx[k];
  const float dx = p.x - cl.x, dy = p.y - cl.y, dz = p.z - cl.z;
  const float dist = sqrtf(dx * dx + dy * dy + dz * dz);
  const float pad = 1e-5f * (fabsf(p.x) + fabsf(p.y) + fabsf(p.z));
  // per-axis displacement bounds (each also <= the isotropic one)
  const float Dx = (ax.x * dist + bx.x) * 1.001f + pad;
  const float Dy = (ax.y * dist + bx.y) * 1.001f + pad;
  const float Dz = (ax.z * dist + bx.z) * 1.001f + pad;
  const float zlo = p.z - Dz;
  if (zlo < 2.0f * c_fp.znear) return true;  // too close to call
  const float iz = 1.0f / p.z, izl = 1.0f / zlo;
  const float u = p.x * iz, v = p.y * iz;
  const float ex = c.fx * u + c.cx, ey = c.fy * v + c.cy;
  // x_j - x = fx (e_x - u e_z) / (p.z + e_z), |e_a| <= D_a (same for y)
  const float sx = c.fx * (Dx + fabsf(u) * Dz) * izl * 1.01f + 2e-5f * fabsf(ex) + 3.0f;
  const float sy = c.fy * (Dy + fabsf(v) * Dz) * izl * 1.01f + 2e-5f * fabsf(ey) + 3.0f;
  return ey + eyw + sy >= ylo && ey - eyw - sy <= yhi && ex + exw + sx >= xlo &&
         ex - exw - sx <= xhi;
}

// 116 registers, 4 CTAs/SM (measured at config C: capping at 96 / 80
// registers for 5 / 6 CTAs/SM gives 1.14 / 1.38 ms against 1.13 ms)
// SH colour (O11) of one Gaussian at two unit view directions (packed halves),
// the scalar evaluation's operations in the same order per half.
template <int DEG>
__device__ __forceinline__ void sh_colour_x2(const float (*sh)[3], f32x2 dx, f32x2 dy, f32x2 dz,
                                             float2* col) {
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    f32x2 v = mul2(bc2(0.28209479177387814f), bc2(sh[0][ch]));
    if (DEG >= 1) {
      // v += -C1 dy s1 + C1 dz s2 - C1 dx s3, as ((a + b) - c) + v, a = -C1 dy s1
      const f32x2 t1 = mul2(mul2(bc2(-0.4886025119029199f), dy), bc2(sh[1][ch]));
      const f32x2 t2 = mul2(mul2(bc2(0.4886025119029199f), dz), bc2(sh[2][ch]));
      const f32x2 t3 = mul2(mul2(bc2(0.4886025119029199f), dx), bc2(sh[3][ch]));
      v = add2(v, sub2(add2(t1, t2), t3));
    }
    col[ch] = upk2(v);
  }
}

template <int DEG, bool MB>
__global__ void __launch_bounds__(128) k_preprocess(
    const float4* __restrict__ mean4, const float4* __restrict__ cov8,
    const float* __restrict__ shsoa, float4* __restrict__ rec0, float4* __restrict__ rec1,
    float4* __restrict__ geom, uint32_t* __restrict__ dkey, uint32_t* __restrict__ vis,
    unsigned long long* __restrict__ counters /* near, degenerate, opacity */,
    uint32_t* __restrict__ drange /* [min, max] depth bits of kept records */) {
  constexpr int NC = (DEG + 1) * (DEG + 1);
  const long long M = c_fp.M;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned n_near = 0, n_deg = 0, n_op = 0;
  uint32_t dmn = 0xFFFFFFFFu, dmx = 0u;
  if (i < M) {
    const float4 m = mean4[i];
    const float tau = m.w;
    const float4 ca = cov8[2 * i], cb = cov8[2 * i + 1];
    const float S6[6] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y};
    const float o = cb.z;
    const float lo2 = log2f(o);
    const int K = c_fp.K;
    if (!(tau > 0.0f)) {
      n_op = 1;
      for (int k = 0; k < K; ++k) vis[(long long)k * M + i] = 0;
    } else {
      float sh[NC][3];
#pragma unroll
      for (int q = 0; q < NC; ++q)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) sh[q][ch] = shsoa[(long long)(q * 3 + ch) * M + i];
      // the record (i,k) after its exact projection and EWA (a, b, c, det)
      auto tail = [&](int k, long long r, int jr, const F3& p, float a, float b, float c,
                      float det) {
        dkey[r] = __float_as_uint(p.z);
        {  // exact per-record AccuTile constants (O7), used by count and emit
          const EllRec el = ell_rec(a, b, c, det, tau);
          if (MB ? !may_touch_band(k, jr, p, el.ex * 1.001f + 1.0f, el.ey * 1.001f + 1.0f)
                 : !may_touch_band_views(k, m.x, m.y, m.z, el.ex * 1.001f + 1.0f,
                                         el.ey * 1.001f + 1.0f)) {
            vis[r] = 0;  // no view can reach the band / frame: empty union
            return;
          }
          vis[r] = 1;
          dmn = min(dmn, __float_as_uint(p.z));
          dmx = max(dmx, __float_as_uint(p.z));
          geom[2 * r] = make_float4(el.ex, el.ey, el.dyR, el.tc);
          geom[2 * r + 1] = make_float4(el.ic, el.b, el.det, 0.0f);
        }
        // conic (tolerance path): one correctly rounded reciprocal of det, three products
        const float idet = __frcp_rn(det);
        const float A = c * idet, B = -b * idet, C = a * idet;
        rec0[2 * r] = make_float4(-0.5f * kLog2e * A, -kLog2e * B, -0.5f * kLog2e * C, lo2);
        // SH colour at the representative camera centre (O11)
        const CamConstDev& cc = c_ccon[jr];
        float dx = m.x - cc.C[0], dy = m.y - cc.C[1], dz = m.z - cc.C[2];
        const float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
        dx *= inv; dy *= inv; dz *= inv;
        float col[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          float v = 0.28209479177387814f * sh[0][ch];
          if (DEG >= 1) {
            v += -0.4886025119029199f * dy * sh[1][ch] + 0.4886025119029199f * dz * sh[2][ch] -
                 0.4886025119029199f * dx * sh[3][ch];
          }
          if (DEG >= 2) {
            const float xx = dx * dx, yy = dy * dy, zz = dz * dz;
            v += 1.0925484305920792f * dx * dy * sh[4][ch] +
                 -1.0925484305920792f * dy * dz * sh[5][ch] +
                 0.31539156525252005f * (2.f * zz - xx - yy) * sh[6][ch] +
                 -1.0925484305920792f * dx * dz * sh[7][ch] +
                 0.5462742152960396f * (xx - yy) * sh[8][ch];
            if (DEG >= 3) {
              v += -0.5900435899266435f * dy * (3.f * xx - yy) * sh[9][ch] +
                   2.890611442640554f * dx * dy * dz * sh[10][ch] +
                   -0.4570457994644658f * dy * (4.f * zz - xx - yy) * sh[11][ch] +
                   0.3731763325901154f * dz * (2.f * zz - 3.f * xx - 3.f * yy) * sh[12][ch] +
                   -0.4570457994644658f * dx * (4.f * zz - xx - yy) * sh[13][ch] +
                   1.445305721320277f * dz * (xx - yy) * sh[14][ch] +
                   -0.5900435899266435f * dx * (xx - 3.f * yy) * sh[15][ch];
            }
          }
          col[ch] = fmaxf(v + 0.5f, 0.0f);
        }
        // conservative half extents of the alpha >= 1/255 ellipse (+0.5 px, +0.1%):
        // the composite uses them to cull (entry, view) pairs that cannot reach a
        // subpixel (superfluous cluster-union pairs)
        const float ex = fmaf(sqrtf(tau * a), 1.001f, 0.5f), ey = fmaf(sqrtf(tau * c), 1.001f, 0.5f);
        const __half2 ext = __halves2half2(__float2half_ru(ex), __float2half_ru(ey));
        rec0[2 * r + 1] = make_float4(col[0], col[1], col[2], *reinterpret_cast<const float*>(&ext));
      };
      for (int k = 0; k < K; ++k) {
        const long long r = (long long)k * M + i;
        const int jr = c_rep[k];
        const CamDev& rc = c_cams[jr];
        const F3 p = cam_point_exact(rc, m.x, m.y, m.z);
        if (p.z < c_fp.znear) { vis[r] = 0; ++n_near; continue; }
        float a, b, c, det;
        if (!cov2d_exact(rc, c_ccon[jr], p, S6, a, b, c, det)) { vis[r] = 0; ++n_deg; continue; }
        tail(k, r, jr, p, a, b, c, det);
      }
    }
  }
  // block-aggregated culling counters
  __shared__ unsigned s_c[3];
  if (threadIdx.x < 3) s_c[threadIdx.x] = 0;
  __syncthreads();
  if (n_near) atomicAdd(&s_c[0], n_near);
  if (n_deg) atomicAdd(&s_c[1], n_deg);
  if (n_op) atomicAdd(&s_c[2], n_op);
  __syncthreads();
  if (threadIdx.x < 3 && s_c[threadIdx.x]) atomicAdd(&counters[threadIdx.x], s_c[threadIdx.x]);
  // depth-bit range of the kept records (the presort compresses its keys to it)
  dmn = __reduce_min_sync(0xffffffffu, dmn);
  dmx = __reduce_max_sync(0xffffffffu, dmx);
  if ((threadIdx.x & 31) == 0 && dmx >= dmn) {
    atomicMin(&drange[0], dmn);
    atomicMax(&drange[1], dmx);
  }
}

// ===========================================================================
// a6 count — per warp, 32/G records (one G-lane group each; every lane owns
// VPL consecutive views of its record).  Fast path (footprint <= kSlotRows
// rows, < 64 columns from a conservative reference column lo_ref): the
// (view, row) items of all the warp's records are redistributed evenly over
// the 32 lanes (segment-start marks + clz source lookup, source data staged
// in shared memory), each item computes its exact AccuTile interval (O7) and
// ORs it into the record's per-row 64-bit mask in shared memory; the group's
// lanes write the record's 64-byte union slot (header, lo_ref, up to
// kSlotRows masks) at its depth-sorted list position g for the emit pass.
// Records outside the fast path are flagged in their slot and listed for
// k_count_big.  recs is the depth-sorted record list; every output is indexed
// by the list position (cnt[g], slot g, big list of positions), so the offsets
// scan and the emission read them sequentially.  Grid-stride, warp-uniform
// loop; cameras in shared memory.
// ===========================================================================
constexpr int kBinThreads = 256;
constexpr int kBinWarps = kBinThreads / 32;

// VPL = 2 (s >= 8): a G-lane group covers 2G views and a warp takes twice the
// records per step, halving the per-record share of loads, group reductions,
// the item prefix scan and the slot write (measured: binning 7.56 -> 6.58 ms
// at config C; VPL = 4: 6.54 ms, not worth its 77 registers).
template <int G, int VPL, int NTH = kBinThreads>
__global__ void __launch_bounds__(NTH) k_countv(const uint32_t* __restrict__ recs,
                                                        uint32_t n,
                                                        const float4* __restrict__ mean4,
                                                        const float4* __restrict__ geom,
                                                        uint32_t* __restrict__ cnt,
                                                        uint4* __restrict__ slots,
                                                        uint8_t* __restrict__ rows8,
                                                        uint32_t* __restrict__ big,
                                                        uint32_t* __restrict__ n_big) {
  constexpr int kBW = NTH / 32;  // warps per block
  extern __shared__ float s_cam[];  // c_fp.N cameras x kCamStride (dynamic)
  __shared__ unsigned long long s_mask[kBW][32][kSlotRows];  // [warp][group][row]
  __shared__ int s_flag[kBW][32];
  __shared__ int s_src[kBW][32];
  __shared__ int s_seg[kBW][32];            // per lane: first item of its segment
  __shared__ float4 s_lv[kBW][VPL][32];     // per lane, view u: mx, my, first, items before u
  __shared__ float4 s_gv[kBW][32][2];       // per group: ellipse constants, rmin
  stage_cams(s_cam);
  __syncthreads();
  constexpr int GPW = 32 / G;
  const int s = c_fp.s, N = c_fp.N, TX = c_fp.TX, TY = c_fp.TY;
  const int lane = threadIdx.x & 31, v = lane & (G - 1), gi = lane / G, w = threadIdx.x >> 5;
  const bool lead = v == 0;
  const unsigned long long nwarps = (unsigned long long)gridDim.x * kBW;
  for (unsigned long long wb = (blockIdx.x * (unsigned long long)NTH + threadIdx.x) / 32 * GPW;
       wb < n; wb += nwarps * GPW) {  // warp-uniform loop
    const unsigned long long g = wb + gi;
    const bool active = g < n;
    uint32_t r = 0;
    float4 m = make_float4(0.f, 0.f, 0.f, 1.f);
    float4 q0 = make_float4(1.f, 1.f, 0.f, 1.f), q1 = make_float4(1.f, 0.f, 1.f, 0.f);
    int k = 0;
    if (active) {
      r = recs[g];
      k = (int)fdiv(r, c_fp.divM);
      m = mean4[(long long)r - (long long)k * c_fp.M];
      q0 = geom[2ull * r];
      q1 = geom[2ull * r + 1];
    }
    const EllRec el = ell_load(q0, q1);
    // ---- the lane's views: exact means (Eq.5) and AccuTile rows (O7)
    float mx[VPL], my[VPL];
    int ty0[VPL], ty1[VPL];
    bool vis[VPL];
    int tmin = 0x7fffffff, tmax = -1, kl = 0x7f800000;
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      mx[u] = 0.f; my[u] = 0.f; ty0[u] = 0x7fffffff; ty1[u] = -1; vis[u] = false;
      const int vv = VPL * v + u;
      const int j = k * s + vv;
      if (active && vv < s && j < N) {
        const CamDev cam = load_cam(s_cam, j);
        const F3 p = cam_point_exact(cam, m.x, m.y, m.z);
        if (p.z >= c_fp.znear) {
          mean2d_exact(cam, p, mx[u], my[u]);
          view_rows(el, my[u], TY, ty0[u], ty1[u]);
          vis[u] = true;
          tmin = min(tmin, ty0[u]);
          tmax = max(tmax, ty1[u]);
          const int xk = __float_as_int(mx[u]);
          kl = min(kl, xk ^ ((xk >> 31) & 0x7fffffff));
        }
      }
    }
    const int rmin = max(gmin<G>(tmin), c_fp.row0);
    const int rmax = min(gmax<G>(tmax), c_fp.row1 - 1);
    const int nrows = (active && rmax >= rmin) ? rmax - rmin + 1 : 0;
    const int kmin = gmin<G>(kl);
    const float mxlo = __int_as_float(kmin ^ ((kmin >> 31) & 0x7fffffff));
    const int lo_ref = (int)fmaxf(floorf((mxlo - el.ex - 15.5f) * 0.0625f) - 1.0f, -1.0f);
    const bool fast = nrows > 0 && nrows <= kSlotRows;
    int ni = 0;
#pragma unroll
    for (int u = 0; u < VPL; ++u) {
      int f = 0, c = 0;
      if (fast && vis[u]) {
        f = max(ty0[u], rmin);
        c = max(0, min(ty1[u], rmax) - f + 1);
      }
      s_lv[w][u][lane] = make_float4(mx[u], my[u], __int_as_float(f), __int_as_float(ni));
      ni += c;
    }
    if (lead) {
      s_flag[w][gi] = 0;
#pragma unroll
      for (int t = 0; t < kSlotRows; ++t) s_mask[w][gi][t] = 0ull;
    }
    int pre = ni;  // warp inclusive prefix of (view,row) items
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    const int total = __shfl_sync(0xffffffffu, pre, 31);
    const int seg0 = pre - ni;
    s_seg[w][lane] = seg0;
    if (lead) {
      s_gv[w][gi][0] = make_float4(el.ex, el.ey, el.dyR, el.tc);
      s_gv[w][gi][1] = make_float4(el.ic, el.b, el.det, __int_as_float(rmin));
    }
    __syncwarp();
    for (int base = 0; base < total; base += 32) {
      const bool inter = ni > 0 && pre > base && seg0 < base + 32;
      const int spos = max(seg0, base) - base;
      if (inter) s_src[w][spos] = lane;
      const unsigned marks = __reduce_or_sync(0xffffffffu, inter ? (1u << spos) : 0u);
      const int idx = base + lane;
      const unsigned upto = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
      const unsigned mk = marks & upto;
      __syncwarp();
      const int src = (idx < total && mk) ? s_src[w][31 - __clz(mk)] : 0;
      const int loc = idx - s_seg[w][src];  // item index within the source lane
      // the source view: the last u whose items start at or before loc
      float4 lv = s_lv[w][0][src];
#pragma unroll
      for (int u = 1; u < VPL; ++u) {
        const float4 lu = s_lv[w][u][src];
        if (loc >= __float_as_int(lu.w)) lv = lu;
      }
      const float smx = lv.x, smy = lv.y;
      const int row = __float_as_int(lv.z) + (loc - __float_as_int(lv.w));
      const float4 g0 = s_gv[w][src / G][0], g1 = s_gv[w][src / G][1];
      const int srmin = __float_as_int(g1.w);
      const int slo = __shfl_sync(0xffffffffu, lo_ref, src);
      EllRec e;
      e.ex = g0.x; e.ey = g0.y; e.dyR = g0.z; e.tc = g0.w;
      e.ic = g1.x; e.b = g1.y; e.det = g1.z;
      if (idx < total) {
        const int gs = src / G;
        int tx0, tx1;
        if (view_row_cols(e, smx, smy, row, TX, tx0, tx1) && tx0 <= tx1) {
          if (tx0 < slo || tx1 - slo >= 64) {
            atomicOr(&s_flag[w][gs], 1);
          } else {
            // bits [a, b] of the 64-column window as two 32-bit words (BMSK)
            const int a = tx0 - slo, b = tx1 - slo;
            const unsigned lo = bmsk32(a, b - a + 1);
            const unsigned hi = b >= 32 ? bmsk32(max(a - 32, 0), b - max(a, 32) + 1) : 0u;
            unsigned* mw = reinterpret_cast<unsigned*>(&s_mask[w][gs][row - srmin]);
            if (lo) atomicOr(mw, lo);
            if (hi) atomicOr(mw + 1, hi);
          }
        }
      }
    }
    __syncwarp();
    // ---- finalize: the group's lanes write the slot; general path for the rest
    const bool slow = active && nrows > 0 && (!fast || s_flag[w][gi] != 0);
    uint32_t c = 0;
    const unsigned long long o = g;
    {
      const bool wr = active && fast && !slow;
      uint32_t pc = 0;
      if (wr)
        for (int t = v; t < kSlotRows; t += G) pc += (uint32_t)__popcll(s_mask[w][gi][t]);
#pragma unroll
      for (int q = 1; q < G; q <<= 1) pc += __shfl_xor_sync(0xffffffffu, pc, q);
      if (wr) c = pc;
      // masks of rows >= nrows are never read (k_emit_rows loads by rows8)
      for (int q = v; wr && q < 4 && 2 * q - 1 <= nrows; q += G) {
        uint4 val;
        if (q == 0) {
          val = make_uint4((uint32_t)(rmin & 0xFFFF) | ((uint32_t)nrows << 16), (uint32_t)lo_ref, c, 0u);
        } else {
          val = *reinterpret_cast<const uint4*>(&s_mask[w][gi][2 * (q - 1)]);
        }
        slots[4ull * o + q] = val;
      }
    }
    if (slow && lead) {  // footprint beyond the fast path: k_count_big
      slots[4ull * o] = make_uint4(kSlotOverflow, 0u, 0u, 0u);
      big[atomicAdd(n_big, 1u)] = (uint32_t)o;
    }
    if (active && lead) {
      cnt[o] = c;
      rows8[o] = (uint8_t)(slow ? 7 : (fast ? nrows : 0));  // 7: overflow (header only)
    }
    __syncwarp();
  }
}

// ===========================================================================
// a6 emit, fast path over the depth-sorted, position-indexed slots (k_countv):
// each warp takes 32 consecutive records, stages their union rows (64-bit
// mask, output start, tile of bit 0) in shared memory, spreads the ~2 rows per
// record evenly over its lanes (segment-start marks + clz, as in the count)
// and every lane writes its row's tiles (consecutive outputs) into the warp's
// shared-memory window over its records' output range [O, f1), copied out
// coalesced (WB = window size in pairs; a range that does not fit, or WB = 0,
// is written directly).
// Records flagged overflow have no rows here: k_emit_big writes their pairs,
// concurrently on a forked stream.  Grid-stride over record blocks.
// (Measured against a lane-per-record decode through a shared window: 0.15 ms
// less at config C; a run table + max-scan and a pair-flat binary-search
// decode were both slower.)
// ===========================================================================
// Per-block inputs of the emission: the records' output offsets, the slot
// (header + six row masks) and payload r of lane e = b*32 + lane.
struct EmitIn {
  uint32_t o, f1, r, rows;
  uint4 h, s1, s2, s3;
};
__device__ __forceinline__ void emit_load_offs(const uint32_t* __restrict__ offs,
                                               const uint8_t* __restrict__ rows8, uint32_t n,
                                               uint32_t P, uint32_t nblk, uint32_t b, int lane,
                                               EmitIn& in) {
  const uint32_t e = b * 32u + (uint32_t)lane;
  in.o = (b < nblk && e < n) ? offs[e] : P;
  in.rows = (b < nblk && e < n) ? rows8[e] : 0u;
  in.f1 = (b < nblk && b * 32u + 32u < n) ? offs[b * 32u + 32u] : P;
}
__device__ __forceinline__ void emit_load_slots(const uint32_t* __restrict__ rec_sorted,
                                                const uint4* __restrict__ slots, uint32_t n,
                                                uint32_t nblk, uint32_t b, int lane, EmitIn& in) {
  const uint32_t e = b * 32u + (uint32_t)lane;
  uint32_t o1 = __shfl_down_sync(0xffffffffu, in.o, 1);  // next record's offset
  if (lane == 31) o1 = in.f1;
  const bool ok = b < nblk && e < n;
  in.h = make_uint4(kSlotOverflow, 0u, 0u, 0u);
  in.s1 = make_uint4(0u, 0u, 0u, 0u);
  in.s2 = in.s1;
  in.s3 = in.s1;
  in.r = ok ? rec_sorted[e] : 0u;
  if (ok && o1 > in.o) {  // the slot of a record without tiles is never written
    // only the masks of the record's rows (rows8: 1..6, 7 = overflow, header only)
    const uint4* sl = slots + 4ull * e;
    in.h = sl[0];
    if (in.rows != 7u) in.s1 = sl[1];
    if (in.rows > 2u && in.rows != 7u) in.s2 = sl[2];
    if (in.rows > 4u && in.rows != 7u) in.s3 = sl[3];
  }
}

// PF: software pipeline over the warp's blocks (slots + payloads of the next
// block and offsets of the one after are in flight while a block is written)
template <int WB, bool PF = false>
__global__ void __launch_bounds__(256) k_emit_rows(const uint32_t* __restrict__ rec_sorted,
                                                   const uint32_t* __restrict__ offs, uint32_t n,
                                                   uint32_t P, const uint4* __restrict__ slots,
                                                   const uint8_t* __restrict__ rows8,
                                                   uint32_t* __restrict__ out_t,
                                                   uint32_t* __restrict__ out_v) {
  extern __shared__ uint32_t s_obuf[];  // WB > 0: [8 warps][2][WB] staged (tile, payload)
  __shared__ unsigned long long s_m[8][32][kSlotRows];  // per record lane: row masks
  __shared__ uint32_t s_q[8][32][kSlotRows];            // per record lane: row output start
  __shared__ uint32_t s_rb[8][32];                      // per record lane: tile of (row0, bit 0)
  __shared__ uint32_t s_r[8][32];                       // per record lane: payload r
  __shared__ int s_seg[8][32];                          // per record lane: first item
  __shared__ int s_src[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t TX = (uint32_t)c_fp.TX;
  const uint32_t nblk = (n + 31) / 32;
  uint32_t* s_ot = s_obuf + w * 2 * WB;
  uint32_t* s_ov = s_ot + WB;
  if (WB > 0)
    for (int i = lane; i < WB; i += 32) s_ot[i] = 0xFFFFFFFFu;  // sentinel: not ours
  const uint32_t bstep = gridDim.x * 8u;
  EmitIn cur, nx;
  if (PF) {
    const uint32_t b0 = blockIdx.x * 8u + (uint32_t)w;
    emit_load_offs(offs, rows8, n, P, nblk, b0, lane, cur);
    emit_load_slots(rec_sorted, slots, n, nblk, b0, lane, cur);
    emit_load_offs(offs, rows8, n, P, nblk, b0 + bstep, lane, nx);
  }
  for (uint32_t b = blockIdx.x * 8u + (uint32_t)w; b < nblk; b += bstep) {
    const uint32_t e = b * 32u + (uint32_t)lane;
    const bool ok = e < n;
    if (PF) {  // issue the next block's slots and the offsets after it
      emit_load_slots(rec_sorted, slots, n, nblk, b + bstep, lane, nx);
    } else {
      emit_load_offs(offs, rows8, n, P, nblk, b, lane, cur);
      emit_load_slots(rec_sorted, slots, n, nblk, b, lane, cur);
    }
    EmitIn nn;
    if (PF) emit_load_offs(offs, rows8, n, P, nblk, b + 2 * bstep, lane, nn);
    const uint32_t o = cur.o, f1 = cur.f1;
    const uint4 h = cur.h, s1 = cur.s1, s2 = cur.s2, s3 = cur.s3;
    const bool dec = !(h.x & kSlotOverflow);  // fast record (big ones: k_emit_big)
    const int nrows = dec ? (int)((h.x >> 16) & 0xFFu) : 0;
    {  // stage the rows
      const unsigned long long mr[kSlotRows] = {
          (unsigned long long)s1.x | ((unsigned long long)s1.y << 32),
          (unsigned long long)s1.z | ((unsigned long long)s1.w << 32),
          (unsigned long long)s2.x | ((unsigned long long)s2.y << 32),
          (unsigned long long)s2.z | ((unsigned long long)s2.w << 32),
          (unsigned long long)s3.x | ((unsigned long long)s3.y << 32),
          (unsigned long long)s3.z | ((unsigned long long)s3.w << 32)};
      uint32_t q = o;
#pragma unroll
      for (int t = 0; t < kSlotRows; ++t) {
        s_m[w][lane][t] = mr[t];
        s_q[w][lane][t] = q;
        q += (uint32_t)__popcll(mr[t]);
      }
      s_rb[w][lane] = (h.x & 0xFFFFu) * TX + h.y;
      s_r[w][lane] = ok ? cur.r : 0u;
    }
    int pre = nrows;  // warp inclusive prefix of row items
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, pre, d);
      if (lane >= d) pre += y;
    }
    const int total = __shfl_sync(0xffffffffu, pre, 31);
    const int seg0 = pre - nrows;
    s_seg[w][lane] = seg0;
    // the warp's 32 records own the contiguous outputs [O, f1) (minus the
    // overflow records', written by k_emit_big): stage them when they fit
    const uint32_t O = __shfl_sync(0xffffffffu, o, 0);
    const bool stage = WB > 0 && f1 - O <= (uint32_t)WB;
    __syncwarp();
    for (int base = 0; base < total; base += 32) {
      const bool inter = nrows > 0 && pre > base && seg0 < base + 32;
      const int spos = max(seg0, base) - base;
      if (inter) s_src[w][spos] = lane;
      const unsigned marks = __reduce_or_sync(0xffffffffu, inter ? (1u << spos) : 0u);
      const int idx = base + lane;
      const unsigned upto = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
      const unsigned mk = marks & upto;
      __syncwarp();
      if (idx < total && mk) {
        const int src = s_src[w][31 - __clz(mk)];
        const int t = idx - s_seg[w][src];
        unsigned long long m = s_m[w][src][t];
        uint32_t q = s_q[w][src][t];
        const uint32_t rb = s_rb[w][src] + (uint32_t)t * TX;
        const uint32_t r = s_r[w][src];
        if (stage) {
          q -= O;
          while (m) {
            const int bit = __ffsll((long long)m) - 1;
            m &= m - 1;
            s_ot[q] = rb + (uint32_t)bit;
            s_ov[q] = r;
            ++q;
          }
        } else {
          while (m) {
            const int bit = __ffsll((long long)m) - 1;
            m &= m - 1;
            out_t[q] = rb + (uint32_t)bit;
            out_v[q] = r;
            ++q;
          }
        }
      }
      __syncwarp();
    }
    if (stage) {  // coalesced copy-out of the staged range, sentinel reset
      const int np = (int)(f1 - O);
      for (int i = lane; i < np; i += 32) {
        const uint32_t tv = s_ot[i];
        if (tv != 0xFFFFFFFFu) {
          out_t[O + i] = tv;
          out_v[O + i] = s_ov[i];
          s_ot[i] = 0xFFFFFFFFu;
        }
      }
      __syncwarp();
    }
    if (PF) {
      cur = nx;
      nx.o = nn.o;
      nx.f1 = nn.f1;
      nx.rows = nn.rows;
    }
  }
}

// ===========================================================================
// Records whose union exceeds the fast path (> kSlotRows rows or >= 64
// columns): one WARP per record; its 32/G groups each compute all views and
// take interleaved union rows (it = g, g + 32/G, ...).
// ===========================================================================
// Union rows of the first cap big records, kept by k_count_big for k_emit_big
// (record g: rows [g*kStoreRows, (g+1)*kStoreRows) relative to its first union
// row; info[g] = number of union rows, or -1 when a row needs more than one
// 64-column window or the union has more than kStoreRows rows: recompute).
constexpr int kStoreRows = 64;
struct BigRows {
  uint32_t* cnt;
  unsigned long long* mask;
  int* wlo;
  int* info;
  uint32_t cap;
};

template <int G>
__global__ void __launch_bounds__(kBinThreads) k_count_big(const uint32_t* __restrict__ big,
                                                           const uint32_t* __restrict__ recs,
                                                           const uint32_t* __restrict__ n_ptr,
                                                           const float4* __restrict__ mean4,
                                                           const float4* __restrict__ geom,
                                                           uint32_t* __restrict__ cnt,
                                                           BigRows st) {
  extern __shared__ float s_cam[];  // c_fp.N cameras x kCamStride (dynamic: N * 68 B)
  __shared__ int s_nr[kBinWarps];
  stage_cams(s_cam);
  __syncthreads();
  const uint32_t n = *n_ptr;
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31, v = lane & (G - 1), gi = lane / G, w = threadIdx.x >> 5;
  const uint32_t nwarps = gridDim.x * kBinWarps;
  for (uint32_t g = (blockIdx.x * kBinThreads + threadIdx.x) / 32; g < n; g += nwarps) {
    const uint32_t o = big[g];
    const uint32_t r = recs[o];
    const int k = (int)fdiv(r, c_fp.divM);
    const float4 m = mean4[(long long)r - (long long)k * c_fp.M];
    const EllRec el = ell_load(geom[2ull * r], geom[2ull * r + 1]);
    uint32_t c;
    if (g < st.cap) {  // also keep the union's rows (counts, window masks) for k_emit_big
      const size_t b = (size_t)g * kStoreRows;
      if (lane == 0) st.info[g] = 0;  // the wide flag until the end
      __syncwarp();
      c = group_union<3, G>(s_cam, true, k, v, m.x, m.y, m.z, el, gi, GPW, st.cnt + b, nullptr,
                            nullptr, nullptr, 0, st.mask + b, st.wlo + b, &st.info[g], kStoreRows,
                            &s_nr[w]);
      __syncwarp();
      if (lane == 0) {
        const int nr = s_nr[w];
        st.info[g] = (st.info[g] != 0 || nr > kStoreRows) ? -1 : nr;  // -1: recompute
      }
    } else {
      c = group_union<0, G>(s_cam, true, k, v, m.x, m.y, m.z, el, gi, GPW, nullptr, nullptr,
                            nullptr, nullptr, 0);
    }
    const uint32_t tot = __reduce_add_sync(0xffffffffu, v == 0 ? c : 0u);
    if (lane == 0) cnt[o] = tot;
    __syncwarp();
  }
}

// Per-warp row arrays hold kMaxRows union rows; a taller union (panels over
// 16 * kMaxRows px, tall bands) is written window by window.
constexpr int kMaxRows = 288;
template <int G>
__global__ void __launch_bounds__(kBinThreads) k_emit_big(
    const uint32_t* __restrict__ rec_sorted, const uint32_t* __restrict__ offs,
    const uint32_t* __restrict__ elist, const uint32_t* __restrict__ n_ptr,
    const float4* __restrict__ mean4, const float4* __restrict__ geom,
    uint32_t* __restrict__ out_t, uint32_t* __restrict__ out_v, BigRows st) {
  extern __shared__ float s_cam[];  // c_fp.N cameras x kCamStride (dynamic)
  __shared__ uint32_t s_rows[kBinWarps][kMaxRows];
  __shared__ unsigned long long s_rmask[kBinWarps][kMaxRows];  // per row: window mask
  __shared__ int s_rwlo[kBinWarps][kMaxRows];                  // per row: window column
  __shared__ int s_wide[kBinWarps];
  __shared__ int s_nr[kBinWarps];
  stage_cams(s_cam);
  __syncthreads();
  const uint32_t n = *n_ptr;
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31, v = lane & (G - 1), gi = lane / G, w = threadIdx.x >> 5;
  uint32_t* rows = s_rows[w];
  const uint32_t nwarps = gridDim.x * kBinWarps;
  for (uint32_t g = (blockIdx.x * kBinThreads + threadIdx.x) / 32; g < n; g += nwarps) {
    const uint32_t e = elist[g];
    const uint32_t r = rec_sorted[e];
    const int k = (int)fdiv(r, c_fp.divM);
    const float4 m = mean4[(long long)r - (long long)k * c_fp.M];
    const EllRec el = ell_load(geom[2ull * r], geom[2ull * r + 1]);
    // per-row counts and window masks (rows relative to the union's first row):
    // stored by k_count_big (<= kStoreRows rows), else recomputed per window
    const int info = g < st.cap ? st.info[g] : -1;
    uint32_t carry = offs[e];
    for (int wb = 0;; wb += kMaxRows) {
      for (int q = lane; q < kMaxRows; q += 32) rows[q] = 0;
      if (lane == 0) { s_wide[w] = 0; s_nr[w] = 0; }
      __syncwarp();
      if (info >= 0) {
        const size_t b = (size_t)g * kStoreRows;
        for (int q = lane; q < info; q += 32) {
          const uint32_t cq = st.cnt[b + q];
          rows[q] = cq;
          if (cq) {
            s_rmask[w][q] = st.mask[b + q];
            s_rwlo[w][q] = st.wlo[b + q];
          }
        }
        if (lane == 0) s_nr[w] = info;
      } else {
        group_union<3, G>(s_cam, true, k, v, m.x, m.y, m.z, el, gi, GPW, rows, nullptr, nullptr,
                          nullptr, 0, s_rmask[w], s_rwlo[w], &s_wide[w], kMaxRows, &s_nr[w], wb,
                          wb + kMaxRows);
      }
      __syncwarp();
      const int nr_all = s_nr[w];
      // exclusive scan of the window's per-row counts -> row offsets (in place)
      int nrows = 0;
      for (int b0 = 0; b0 < kMaxRows; b0 += 32) {
        const uint32_t x = rows[b0 + lane];
        uint32_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        rows[b0 + lane] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
        nrows = max(nrows, __reduce_max_sync(0xffffffffu, x ? b0 + lane + 1 : 0));
      }
      __syncwarp();
      if (s_wide[w]) {  // a row wider than one 64-column window: recompute and write
        group_union<2, G>(s_cam, true, k, v, m.x, m.y, m.z, el, gi, GPW, nullptr, rows, out_t,
                          out_v, r, nullptr, nullptr, nullptr, kMaxRows, nullptr, wb,
                          wb + kMaxRows);
      } else {  // every row from its stored window mask (no second union): lane per row
        for (int it = lane; it < nrows; it += 32) {
          uint32_t pos = rows[it];
          const uint32_t end = it + 1 < nrows ? rows[it + 1] : carry;
          if (end == pos) continue;  // empty row (its mask slot was not written)
          unsigned long long mk = s_rmask[w][it];
          const uint32_t tb = (uint32_t)s_rwlo[w][it];
          while (mk) {
            const int bit = __ffsll((long long)mk) - 1;
            mk &= mk - 1;
            out_t[pos] = tb + (uint32_t)bit;
            out_v[pos] = r;
            ++pos;
          }
        }
      }
      __syncwarp();
      if (info >= 0 || wb + kMaxRows >= nr_all) break;
    }
  }
}

// Introspection (cr_get_counts): per-(i,k) tile counts |T_{i,k}| recovered from
// the emitted pairs (each pair carries its record r).
__global__ void k_pair_counts(const uint32_t* __restrict__ val, uint32_t P,
                              uint32_t* __restrict__ cnt) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < P) atomicAdd(&cnt[val[e]], 1u);
}

// ===========================================================================
// a8 — ranges [S_{t,k}, E_{t,k}) from the (t, k)-sorted pairs.
// slot[e] = t*K + k, written by the tile sort's last pass (k_radix_onesweep
// with slotK = K), so only the keys are read.
// ===========================================================================
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ slot, uint32_t P,
                                                uint32_t* __restrict__ S, uint32_t* __restrict__ E) {
  // 4 consecutive pairs per thread (16-byte loads), grid-stride over quads;
  // neighbour slots via shuffles, lanes 0/31 load their outer neighbour once.
  // Buffers are padded, so a partial last quad is safe.
  const int lane = threadIdx.x & 31;
  const uint32_t nq = (P + 3) / 4;
  for (uint32_t q0 = blockIdx.x * blockDim.x; q0 < nq; q0 += gridDim.x * blockDim.x) {
    const uint32_t q = q0 + threadIdx.x;
    const uint32_t e = 4 * q;
    uint32_t key[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
    if (q < nq) {
      const uint4 tt = reinterpret_cast<const uint4*>(slot)[q];
      const uint32_t ta[4] = {tt.x, tt.y, tt.z, tt.w};
#pragma unroll
      for (int h = 0; h < 4; ++h)
        if (e + h < P) key[h] = ta[h];
    }
    uint32_t prev = __shfl_up_sync(0xffffffffu, key[3], 1);
    uint32_t next = __shfl_down_sync(0xffffffffu, key[0], 1);
    if (lane == 0) prev = (q < nq && e > 0) ? slot[e - 1] : 0xFFFFFFFEu;
    if (lane == 31) next = (q < nq && e + 4 < P) ? slot[e + 4] : 0xFFFFFFFEu;
    if (q >= nq) continue;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint32_t eh = e + h;
      if (eh >= P) break;
      const uint32_t pk = h == 0 ? prev : key[h - 1];
      const uint32_t nk = (h == 3 || eh + 1 >= P) ? (h == 3 ? next : 0xFFFFFFFEu) : key[h + 1];
      if (eh == 0 || pk != key[h]) S[key[h]] = eh;
      if (eh == P - 1 || nk != key[h]) E[key[h]] = eh + 1;
    }
  }
}

// Introspection: 64-bit keys of Eq.11 and payload i.
// slot[e] = t*K + k (the tile sort's output, see k_ranges).
__global__ void k_make_keys(const uint32_t* __restrict__ slot, const uint32_t* __restrict__ val,
                            const uint32_t* __restrict__ dkey, uint32_t P,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ pay) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P) return;
  const unsigned long long M = (unsigned long long)c_fp.M;
  const uint32_t r = val[e];
  const unsigned long long k = fdiv(r, c_fp.divM);
  const unsigned long long t = slot[e] / (uint32_t)c_fp.K;
  keys[e] = (t << (32 + c_fp.bitK)) | (k << 32) |
            (unsigned long long)dkey[r];
  pay[e] = (uint32_t)(r - k * M);
}

}  // namespace cr
