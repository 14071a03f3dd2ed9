// cr_composite.cuh — a9 subpixel compositing (Eqs.9-10; Alg.2
// Alpha-Blend).
//
// k_composite_pairs (default) is the design below with two subpixels of one
// view per lane and packed fp32x2 blend arithmetic (see its comment);
// k_composite_staged (round 2's kernel, CR_EXP bit 6) is kept for A/B:
//   CTA per 16x16 tile, 8 warps pulling "cluster-aligned warp chunks" (<= 32
//   consecutive Psi ranks of one cluster k) from a shared-memory queue.  Per
//   chunk the warp streams list (t,k) in 32-entry batches: lane l gathers
//   entry l's record and world mean once, projects the mean for each of the
//   <= 8 distinct views present in the chunk (per-view mu2D_{i,j}, Eq.5),
//   stages everything in shared memory and ballots, per view, which entries
//   can reach that view's subpixels at all (alpha >= 1/255 box test: the
//   cluster tile union holds many entries a given view never touches,
//   P:379-382, and skipping them is exact).  Every lane then walks only its
//   view's surviving entries from shared memory (broadcast reads).  A warp
//   ballot ends the list as soon as every lane has saturated.  Results go to
//   a smem tile and leave in 16-byte vector row stores (store_tile).
// k_composite_thread (the paper's design): one thread per subpixel rank r,
//   x = Psi(r) (remap=1) or raster order (remap=0), private list traversal
//   with direct gathers and a direct scattered store.
#pragma once
#include <cuda_fp16.h>

#include "cr_device.cuh"

namespace cr {

#ifndef CR_COMP_MINB
#define CR_COMP_MINB 10  // measured: 48 regs, 11.04 vs 11.17 ms at config C
#endif
constexpr int kCompWarps = 4;
constexpr int kMaxChunks = kMaxViews + 24;  // k_chunks_build emits <= K + 24 per tile
constexpr int kSlots = 8;  // distinct views staged per pass of a chunk

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Tolerance-path per-view mean (fast FMA / approximate reciprocal); far away
// when the view cannot see the Gaussian (Z12) so that alpha underflows to 0.
// The camera comes as 4 float4 {R0..R3}, {R4..R7}, {R8,t0,t1,t2}, {fx,fy,cx,cy}.
// position of the most significant set bit (x != 0): one FLO
__device__ __forceinline__ int msb_pos(unsigned x) {
  int p;
  asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(x));
  return p;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 mean2d_fast4(const float4 a, const float4 b, const float4 c,
                                               const float4 d, float mx, float my, float mz) {
  const float px = fmaf(a.x, mx, fmaf(a.y, my, fmaf(a.z, mz, c.y)));
  const float py = fmaf(a.w, mx, fmaf(b.x, my, fmaf(b.y, mz, c.z)));
  const float pz = fmaf(b.z, mx, fmaf(b.w, my, fmaf(c.x, mz, c.w)));
  if (!(pz >= c_fp.znear)) return make_float2(1e18f, 1e18f);
  const float iz = rcp_approx(pz);
  return make_float2(fmaf(d.x, px * iz, d.z), fmaf(d.y, py * iz, d.w));
}
__device__ __forceinline__ float2 mean2d_fast(const CamDev& c, float mx, float my, float mz) {
  const float4* q = reinterpret_cast<const float4*>(&c);
  return mean2d_fast4(q[0], q[1], q[2], q[3], mx, my, mz);
}

// One blend step (Eq.10 alpha, Eq.9 accumulation; 0.99 clamp, 1/255 skip,
// stop before blending when T(1-alpha) < 1e-4 — Z9), tolerance-path math
// shared by every composite kernel (so they agree bit for bit):
//   g = (A', B', C', log2 o) with the conic prescaled by -log2(e)/2, -log2(e),
//   -log2(e)/2, so q = power * log2(e) = A' dx^2 + B' dx dy + C' dy^2 (5 ops);
//   the 1/255 skip is decided in the log domain before the exponential
//   (t = q + log2 o >= log2(1/255)), so skipped entries never reach the MUFU;
//   w = alpha T, T' = T - w, C += c w.
constexpr float kLog2MinAlpha = -7.99435343685886f;  // log2(1/255)
__device__ __forceinline__ void blend_step(const float4 g, const float2 m, const float col,
                                           const float px, const float py, float& T, float& C,
                                           bool& done) {
  const float dx = m.x - px, dy = m.y - py;
  const float q = fmaf(dx, fmaf(g.x, dx, g.y * dy), (g.z * dy) * dy);
  const float t = q + g.w;
  if (t >= kLog2MinAlpha && q <= 0.0f) {  // power > 0 or alpha < 1/255: skip
    const float alpha = fminf(0.99f, ex2_approx(t));
    const float wgt = alpha * T;
    const float Tn = T - wgt;
    if (Tn < 1e-4f) {
      done = true;
    } else {
      C = fmaf(col, wgt, C);
      T = Tn;
    }
  }
}

// RGB8 quantisation: floor(min(max(v,0),1) * 255 + 1/2), fp32
__device__ __forceinline__ uint32_t quant_u8(float v) {
  const float cl = fminf(fmaxf(v, 0.0f), 1.0f);
  return (uint32_t)floorf(__fadd_rn(__fmul_rn(cl, 255.0f), 0.5f));
}

// Interlaced tile out of shared memory.  A full 16-pixel-wide tile row is
// 48 bytes (RGB8) or 192 bytes (float) starting at a multiple of 48 / 192
// bytes within its image row, so when the image row pitch W*3 (bytes, RGB8)
// is a multiple of 16 every tile row leaves in 16-byte vector stores: 3 x
// uint4 of 16 quantised subpixels (RGB8) or 12 x float4 (float) per row.
// Partial tiles (right frame edge), unaligned pitches or buffers store
// subpixel by subpixel.
template <int FMT>
__device__ __forceinline__ void store_tile(const float* s_out, void* out, int tx, int ty, int W,
                                           int H, int y_band0) {
  const int nx = min(16, W - tx * 16), ny = min(16, H - ty * 16);
  if (nx == 16 && (W * 3) % 16 == 0 && ((uintptr_t)out & 15) == 0) {
    constexpr int kVecRow = FMT == 0 ? 3 : 12;  // 16-byte vectors per tile row
    for (int q = threadIdx.x; q < ny * kVecRow; q += blockDim.x) {
      const int ly = q / kVecRow, part = q % kVecRow;
      const long long row = (long long)(ty * 16 + ly - y_band0) * W + tx * 16;
      if (FMT == 0) {
        const float4* src = reinterpret_cast<const float4*>(s_out + ly * 48 + part * 16);
        uint32_t wd[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float4 f = src[v];
          wd[v] = quant_u8(f.x) | (quant_u8(f.y) << 8) | (quant_u8(f.z) << 16) |
                  (quant_u8(f.w) << 24);
        }
        reinterpret_cast<uint4*>((uint8_t*)out + row * 3)[part] =
            make_uint4(wd[0], wd[1], wd[2], wd[3]);
      } else {
        reinterpret_cast<float4*>((float*)out + row * 3)[part] =
            reinterpret_cast<const float4*>(s_out + ly * 48)[part];
      }
    }
    return;
  }
  if (FMT == 0) {
    uint8_t* o = (uint8_t*)out;
    const int rowb = nx * 3;
    for (int q = threadIdx.x; q < ny * rowb; q += blockDim.x) {
      const int ly = q / rowb, b = q % rowb;
      o[((long long)(ty * 16 + ly - y_band0) * W + tx * 16) * 3 + b] =
          (uint8_t)quant_u8(s_out[ly * 48 + b]);
    }
  } else {
    float* o = (float*)out;
    const int rowb = nx * 3;
    for (int q = threadIdx.x; q < ny * rowb; q += blockDim.x) {
      const int ly = q / rowb, b = q % rowb;
      o[((long long)(ty * 16 + ly - y_band0) * W + tx * 16) * 3 + b] = s_out[ly * 48 + b];
    }
  }
}

// Instrumentation (CR_FLAG_COUNT_EVALS): add this thread's evaluation count.
__device__ __forceinline__ void add_evals(unsigned long long* evals, unsigned long long n) {
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(evals, n);
}

struct Staged {  // one list entry as gathered by one lane
  float4 m, r0, r1;
  bool valid;
};
__device__ __forceinline__ Staged gather_entry(const float4* __restrict__ rec0,
                                               const float4* __restrict__ rec1,
                                               const float4* __restrict__ mean4, uint32_t r,
                                               bool valid, long long kM) {
  Staged st;
  st.valid = valid;
  if (valid) {
    st.m = mean4[(long long)r - kM];
    st.r0 = rec0[2ull * r];
    st.r1 = rec0[2ull * r + 1];
  } else {
    st.m = make_float4(0.f, 0.f, 0.f, 0.f);
    st.r0 = st.m;
    st.r1 = st.m;
  }
  return st;
}

// NW warps per CTA; VAR bit 0: schedule the tile's chunks longest list first
// (measured at config C: NW=4 without sorting is fastest, 11.4 ms vs 12.1 ms
// for NW=8; colour selects instead of indexed smem loads were slower).
template <int FMT, bool COUNT, int NW, int VAR>
__global__ void __launch_bounds__(NW * 32, CR_COMP_MINB) k_composite_staged(
    const uint8_t* __restrict__ V, const uint16_t* __restrict__ psi,
    const uint32_t* __restrict__ chunks, const uint32_t* __restrict__ nchunks, int stride,
    const uint32_t* __restrict__ S, const uint32_t* __restrict__ E,
    const uint32_t* __restrict__ vals, const float4* __restrict__ rec0,
    const float4* __restrict__ rec1, const float4* __restrict__ mean4, void* __restrict__ out,
    unsigned long long* __restrict__ evals, int tsplit) {
  __shared__ float4 s_rec[NW][32];  // v1: register pipeline
  __shared__ float4 s_col[NW][32];
  // per staged view, per entry slot: mu2D; rows padded to 33 entries so lanes
  // of different views reading the same slot hit different banks (measured:
  // 9.88 -> 9.87 ms at config C)
  constexpr int kMuStride = 33;
  __shared__ float2 s_mu_[NW][kSlots * kMuStride];
  __shared__ float4 s_box[NW][kSlots];  // per staged view: pixel box centre, half size
  __shared__ float4 s_cam4[NW][kSlots][4];  // per staged view: camera (4 float4)
  __shared__ __align__(16) float s_out[kTileSub];
  __shared__ int s_next;
  const int W = c_fp.W, H = c_fp.H, TX = c_fp.TX, K = c_fp.K;
  const long long M = c_fp.M;
  // tsplit > 1 (grids under ~3 waves, e.g. narrow row bands): tsplit CTAs share
  // one tile, CTA `part` taking chunks part, part + tsplit, ... and storing its
  // subpixels directly, so the densest tiles no longer set the band's time
  const int t = c_fp.row0 * TX + (int)(blockIdx.x / (unsigned)tsplit);
  const int part = (int)(blockIdx.x % (unsigned)tsplit);
  const int tx = t % TX, ty = t / TX;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ uint32_t s_ch[kMaxChunks];
  __shared__ uint32_t s_len[kMaxChunks];
  if (threadIdx.x == 0) s_next = 0;
  const int nch = min((int)nchunks[t], kMaxChunks);
  const uint32_t* ch_t0 = chunks + (long long)t * stride;
  if (VAR & 1) {
    for (int q = threadIdx.x; q < nch; q += blockDim.x) {
      const int kq = ch_t0[q] >> 16;
      s_len[q] = E[t * K + kq] - S[t * K + kq];
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nch; q += blockDim.x) {
      const uint32_t lq = s_len[q];
      int rank = 0;
      for (int p = 0; p < nch; ++p) {
        const uint32_t lp = s_len[p];
        rank += (lp > lq) || (lp == lq && p < q);
      }
      s_ch[rank] = ch_t0[q];
    }
  }
  __syncthreads();
  const uint32_t* ch_t = (VAR & 1) ? s_ch : ch_t0;
  const uint16_t* ps = psi + (long long)t * kTileSub;
  unsigned long long nev = 0;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&s_next, 1) * tsplit + part;
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= nch) break;
    const uint32_t ch = ch_t[c];
    const int start = ch & 1023, len = ((ch >> 10) & 63) + 1, k = ch >> 16;
    // this lane's subpixel
    int l = 0, u = 0, j = 0, x = 0, y = 0;
    const bool mine = lane < len;
    if (mine) {
      l = ps[start + lane];
      const int ly = l / 48, rem = l % 48, lx = rem / 3;
      u = rem % 3;
      x = tx * 16 + lx;
      y = ty * 16 + ly;
      j = V[((long long)y * W + x) * 3 + u];
    }
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;
    const int jlo = __shfl_sync(0xffffffffu, j, 0);
    const int jhi = __shfl_sync(0xffffffffu, j, len - 1);
    const int nsl = jhi - jlo + 1;
    const int slot = j - jlo;
    const uint32_t e0 = S[t * K + k], e1 = E[t * K + k];
    const long long kM = (long long)k * M;
    for (int g0 = 0; g0 < nsl; g0 += kSlots) {
      const bool active = mine && slot >= g0 && slot < g0 + kSlots;
      if (!__any_sync(0xffffffffu, active)) continue;
      const int ns = min(kSlots, nsl - g0);
      const int sl = slot - g0;
      // pixel-centre box of each staged view's subpixels (for the per-view cull)
      for (int v = 0; v < ns; ++v) {
        const bool in = active && sl == v;
        const int x0 = __reduce_min_sync(0xffffffffu, in ? x : 0x7fffffff);
        const int x1 = __reduce_max_sync(0xffffffffu, in ? x : -0x7fffffff);
        const int y0 = __reduce_min_sync(0xffffffffu, in ? y : 0x7fffffff);
        const int y1 = __reduce_max_sync(0xffffffffu, in ? y : -0x7fffffff);
        if (lane == 0)
          s_box[w][v] = make_float4(0.5f * (float)(x0 + x1) + 0.5f, 0.5f * (float)(y0 + y1) + 0.5f,
                                    0.5f * (float)(x1 - x0), 0.5f * (float)(y1 - y0));
      }
      if (lane < 4 * ns)
        s_cam4[w][lane >> 2][lane & 3] =
            reinterpret_cast<const float4*>(&c_cams[jlo + g0 + (lane >> 2)])[lane & 3];
      __syncwarp();
      float T = 1.0f, C = 0.0f;
      bool done = !active;
      // two-stage software pipeline: records of batch b+32 and indices of
      // batch b+64 are in flight while batch b is blended
      uint32_t r_nxt = (e0 + 32 + lane < e1) ? vals[e0 + 32 + lane] : 0u;
      Staged cur = gather_entry(rec0, rec1, mean4, (e0 + lane < e1) ? vals[e0 + lane] : 0u,
                                e0 + lane < e1, kM);
      for (uint32_t b = e0; b < e1; b += 32) {
        const Staged nxt = gather_entry(rec0, rec1, mean4, r_nxt, b + 32 + lane < e1, kM);
        r_nxt = (b + 64 + lane < e1) ? vals[b + 64 + lane] : 0u;
        // entry of lane l is staged at slot 31 - l and the masks are bit-reversed,
        // so the front-most remaining entry is the highest set bit (one FLO)
        const int slot = 31 - lane;
        float hx = -1.f, hy = -1.f;
        if (cur.valid) {
          s_rec[w][slot] = cur.r0;
          s_col[w][slot] = cur.r1;
          const __half2 ext = *reinterpret_cast<const __half2*>(&cur.r1.w);
          hx = __low2float(ext);
          hy = __high2float(ext);
        }
        unsigned mymask = 0u;
        for (int v = 0; v < ns; ++v) {
          const float2 mu = mean2d_fast4(s_cam4[w][v][0], s_cam4[w][v][1], s_cam4[w][v][2],
                                         s_cam4[w][v][3], cur.m.x, cur.m.y, cur.m.z);
          s_mu_[w][v * kMuStride + slot] = mu;
          const float4 bx = s_box[w][v];
          const bool pass = cur.valid && fabsf(mu.x - bx.x) <= bx.z + hx &&
                            fabsf(mu.y - bx.y) <= bx.w + hy;
          const unsigned bits = __ballot_sync(0xffffffffu, pass);
          if (sl == v) mymask = bits;
        }
        __syncwarp();
        const int n = min(32u, e1 - b);
        if (!done) {
          unsigned mm = __brev(mymask);
          int qstop = -1;
          const float2* mu_v = &s_mu_[w][sl * kMuStride];
          // colour of channel u: 32-bit shared address kept in a register and
          // loaded on every visit (cheaper than the address the compiler would
          // otherwise rebuild inside the contributing branch)
          const uint32_t col_a = (uint32_t)__cvta_generic_to_shared(&s_col[w][0].x + u);
          while (mm) {
            const int q = msb_pos(mm);
            mm ^= 1u << q;
            float col;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(col) : "r"(col_a + 16u * (uint32_t)q));
            bool stop = false;
            blend_step(s_rec[w][q], mu_v[q], col, px, py, T, C, stop);
            if (stop) {
              done = true;
              qstop = 31 - q;
              mm = 0u;
            }
          }
          if (COUNT) nev += (qstop >= 0) ? (unsigned)(qstop + 1) : (unsigned)n;
        }
        if (__all_sync(0xffffffffu, done)) break;
        __syncwarp();
        cur = nxt;
      }
      __syncwarp();
      if (active) {
        const float v = C + c_fp.bg[u] * T;
        if (tsplit == 1) {
          s_out[l] = v;
        } else {
          const long long o = ((long long)(y - c_fp.row0 * 16) * W + x) * 3 + u;
          if (FMT == 0) ((uint8_t*)out)[o] = (uint8_t)quant_u8(v);
          else ((float*)out)[o] = v;
        }
      }
    }
  }
  if (COUNT) add_evals(evals, nev);
  if (tsplit == 1) {
    __syncthreads();
    store_tile<FMT>(s_out, out, tx, ty, W, H, c_fp.row0 * 16);
  }
}

// ===========================================================================
// k_composite_pairs — the staged design with TWO subpixels of one view per
// lane (k_pairs_build: view runs padded to even length, chunks of <= 32 slot
// pairs), so one staged batch, one per-view cull mask and one walk serve twice
// the subpixels, and the blend arithmetic of the two runs as packed fp32x2
// instructions (FADD2 / FMUL2 / FFMA2, sm_100a), each half rounding exactly
// like blend_step's scalar op (same operations, same order: frames are bit
// identical to k_composite_staged).  A subpixel that saturates stops blending
// (its weight is selected to 0 and T kept); the lane leaves the walk when both
// have.
// ===========================================================================

__device__ __forceinline__ unsigned bit_at(int q) {  // 1u << q in one BMSK
  unsigned r;
  asm("bmsk.clamp.b32 %0, %1, 1;" : "=r"(r) : "r"(q));
  return r;
}

#ifndef CR_COMP2_MINB
#define CR_COMP2_MINB 10  // 48 registers, 10 CTAs x 4 warps per SM (measured at C: 9 -> 8.63 ms, 10 -> 8.36, 11 -> 10.9)
#endif
// mean2d_fast4 with the (x, y) rows packed: the camera staged as
// q0 = (R0, R3, R1, R4), q1 = (R2, R5, t0, t1), q2 = (R6, R7, R8, t2),
// q3 = (fx, fy, cx, cy), so each (x, y) operand pair is one register pair
// (same operations per half as mean2d_fast4: bit-identical)
__device__ __forceinline__ void cam_pairs(const CamDev& c, float4* q) {
  q[0] = make_float4(c.R[0], c.R[3], c.R[1], c.R[4]);
  q[1] = make_float4(c.R[2], c.R[5], c.t[0], c.t[1]);
  q[2] = make_float4(c.R[6], c.R[7], c.R[8], c.t[2]);
  q[3] = make_float4(c.fx, c.fy, c.cx, c.cy);
}
__device__ __forceinline__ float2 mean2d_fast_pairs(const float4 q0, const float4 q1,
                                                    const float4 q2, const float4 q3, float mx,
                                                    float my, float mz) {
  const f32x2 pxy = fma2(pk2(q0.x, q0.y), bc2(mx),
                         fma2(pk2(q0.z, q0.w), bc2(my), fma2(pk2(q1.x, q1.y), bc2(mz), pk2(q1.z, q1.w))));
  const float pz = fmaf(q2.x, mx, fmaf(q2.y, my, fmaf(q2.z, mz, q2.w)));
  if (!(pz >= c_fp.znear)) return make_float2(1e18f, 1e18f);
  const float iz = rcp_approx(pz);
  return upk2(fma2(pk2(q3.x, q3.y), mul2(pxy, bc2(iz)), pk2(q3.z, q3.w)));
}

template <int NW>
struct PairStage {  // one warp's staging area (rec / col share the entry offset 16 q)
  float4 rec[32];
  float4 col[32];          // (r, g, b, extents): a lane's colour is at rec + 512 + 4 u
  float2 mu[kSlots * 33];  // per staged view, rows padded to 33 entries
  float4 box[kSlots];
  float4 cam[kSlots][4];
};
template <int FMT, bool COUNT, int NW>
__global__ void __launch_bounds__(NW * 32, CR_COMP2_MINB) k_composite_pairs(
    const uint8_t* __restrict__ V, const uint16_t* __restrict__ psi2,
    const uint32_t* __restrict__ chunks, const uint32_t* __restrict__ nchunks, int stride,
    const uint32_t* __restrict__ S, const uint32_t* __restrict__ E,
    const uint32_t* __restrict__ vals, const float4* __restrict__ rec0,
    const float4* __restrict__ mean4, void* __restrict__ out, unsigned long long* __restrict__ evals,
    int tsplit) {
  __shared__ PairStage<NW> s_ws[NW];
  __shared__ __align__(16) float s_out[kTileSub];
  __shared__ int s_next;
  const int W = c_fp.W, H = c_fp.H, TX = c_fp.TX, K = c_fp.K;
  const long long M = c_fp.M;
  const int t = c_fp.row0 * TX + (int)(blockIdx.x / (unsigned)tsplit);
  const int part = (int)(blockIdx.x % (unsigned)tsplit);
  const int tx = t % TX, ty = t / TX;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  PairStage<NW>& ws = s_ws[w];
  if (threadIdx.x == 0) s_next = 0;
  const int nch = (int)nchunks[t];
  const uint32_t* ch_t = chunks + (long long)t * stride;
  const uint32_t* ps2 = reinterpret_cast<const uint32_t*>(psi2 + (long long)t * kPairSlots);
  __syncthreads();
  const float kNaN = __int_as_float(0x7fc00000);
  unsigned long long nev = 0;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&s_next, 1) * tsplit + part;
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= nch) break;
    const uint32_t ch = ch_t[c];
    const int start = ch & 1023, nl = ((ch >> 10) & 31) + 1, k = ch >> 16;
    // this lane's two subpixels, local indices la | lb << 16 (lb = 0xFFFF: a
    // hole); decoded where needed so that few registers live across the walk
    const bool mine = lane < nl;
    const uint32_t pr = mine ? ps2[(start >> 1) + lane] : 0u;
    auto decode = [&](uint32_t w, int& x, int& y, int& u) {
      const int l = (int)(w & 0xFFFFu), ly = l / 48, rem = l - 48 * ly;
      u = rem % 3;
      x = tx * 16 + rem / 3;
      y = ty * 16 + ly;
    };
    int j = 0;
    if (mine) {
      int x, y, u;
      decode(pr, x, y, u);
      j = V[((long long)y * W + x) * 3 + u];
    }
    const int jlo = __shfl_sync(0xffffffffu, j, 0);
    const int jhi = __shfl_sync(0xffffffffu, j, nl - 1);
    const int nsl = jhi - jlo + 1;
    const int slot = j - jlo;
    const uint32_t e0 = S[t * K + k], e1 = E[t * K + k];
    const long long kM = (long long)k * M;
    for (int g0 = 0; g0 < nsl; g0 += kSlots) {
      const bool active = mine && slot >= g0 && slot < g0 + kSlots;
      if (!__any_sync(0xffffffffu, active)) continue;
      const int ns = min(kSlots, nsl - g0);
      const int sl = slot - g0;
      const bool hasb = (pr >> 16) != 0xFFFFu;
      int xa, ya, ua, xb, yb, ub;
      decode(pr, xa, ya, ua);
      if (hasb) decode(pr >> 16, xb, yb, ub); else { xb = xa; yb = ya; ub = ua; }
      const int bxlo = min(xa, xb), bxhi = max(xa, xb), bylo = min(ya, yb), byhi = max(ya, yb);
      for (int v = 0; v < ns; ++v) {
        const bool in = active && sl == v;
        const int x0 = __reduce_min_sync(0xffffffffu, in ? bxlo : 0x7fffffff);
        const int x1 = __reduce_max_sync(0xffffffffu, in ? bxhi : -0x7fffffff);
        const int y0 = __reduce_min_sync(0xffffffffu, in ? bylo : 0x7fffffff);
        const int y1 = __reduce_max_sync(0xffffffffu, in ? byhi : -0x7fffffff);
        if (lane == 0)
          ws.box[v] = make_float4(0.5f * (float)(x0 + x1) + 0.5f, 0.5f * (float)(y0 + y1) + 0.5f,
                                  0.5f * (float)(x1 - x0), 0.5f * (float)(y1 - y0));
      }
      if (lane < ns) cam_pairs(c_cams[jlo + g0 + lane], ws.cam[lane]);
      __syncwarp();
      // a saturated (or absent) subpixel gets a NaN position: every later
      // quadratic form is NaN and fails the blend test, so it never blends again
      // done flags: bit 0 subpixel a, bit 1 subpixel b (saturated or absent)
      uint32_t dd = (active ? 0u : 3u) | (hasb ? 0u : 2u);
      const bool da0 = (dd & 1u) != 0u, db0 = (dd & 2u) != 0u;
      f32x2 PX = pk2(da0 ? kNaN : (float)xa + 0.5f, db0 ? kNaN : (float)xb + 0.5f);
      const f32x2 PY = pk2((float)ya + 0.5f, (float)yb + 0.5f);
      f32x2 T2 = pk2(1.0f, 1.0f), C2 = pk2(0.0f, 0.0f);
      // batch b's records are gathered at its start, only the next batch's
      // indices are prefetched: holding the next records in registers (as
      // k_composite_staged does) costs the occupancy that hides this latency
      // (measured at C: 10.19 ms with the register prefetch at 48 registers,
      // 9.67 ms without)
      uint32_t r_nxt = (e0 + lane < e1) ? vals[e0 + lane] : 0u;
      for (uint32_t b = e0; b < e1; b += 32) {
        const Staged cur = gather_entry(rec0, rec0, mean4, r_nxt, b + lane < e1, kM);
        r_nxt = (b + 32 + lane < e1) ? vals[b + 32 + lane] : 0u;
        const int slot = 31 - lane;
        float hx = -1.f, hy = -1.f;
        if (cur.valid) {
          ws.rec[slot] = cur.r0;
          ws.col[slot] = cur.r1;
          const __half2 ext = *reinterpret_cast<const __half2*>(&cur.r1.w);
          hx = __low2float(ext);
          hy = __high2float(ext);
        }
        unsigned mymask = 0u;
        for (int v = 0; v < ns; ++v) {
          const float2 mu = mean2d_fast_pairs(ws.cam[v][0], ws.cam[v][1], ws.cam[v][2],
                                              ws.cam[v][3], cur.m.x, cur.m.y, cur.m.z);
          ws.mu[v * 33 + slot] = mu;
          const float4 bx = ws.box[v];
          const float2 dd = upk2(sub2(pk2(mu.x, mu.y), pk2(bx.x, bx.y)));
          const float2 lim = upk2(add2(pk2(bx.z, bx.w), pk2(hx, hy)));
          const bool pass = cur.valid && fabsf(dd.x) <= lim.x && fabsf(dd.y) <= lim.y;
          const unsigned bits = __ballot_sync(0xffffffffu, pass);
          if (sl == v) mymask = bits;
        }
        __syncwarp();
        const int n = min(32u, e1 - b);
        if (dd != 3u) {
          unsigned mm = __brev(mymask);
          int qa = -1, qb = -1;
          const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&ws.mu[sl * 33]);
          // one base register: entry q's record at rb + 16 q, its colours at
          // rb + 16 q + 512 + 4 u (u = the subpixel's channel)
          const uint32_t rb = (uint32_t)__cvta_generic_to_shared(&ws.rec[0]);
          const uint32_t oa = 512u + 4u * (uint32_t)ua, ob = 512u + 4u * (uint32_t)ub;
          while (mm) {
            const int q = msb_pos(mm);
            mm ^= bit_at(q);
            const uint32_t ra = rb + 16u * (uint32_t)q;
            float4 g;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(g.x), "=f"(g.y), "=f"(g.z), "=f"(g.w) : "r"(ra));
            float2 m;
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(m.x), "=f"(m.y) : "r"(mb + 8u * (uint32_t)q));
            const f32x2 dx = sub2(bc2(m.x), PX), dy = sub2(bc2(m.y), PY);
            const f32x2 q2 = fma2(dx, fma2(bc2(g.x), dx, mul2(bc2(g.y), dy)),
                                  mul2(mul2(bc2(g.z), dy), dy));
            const f32x2 t2 = add2(q2, bc2(g.w));
            const float2 qq = upk2(q2), tt = upk2(t2);
            const bool oka = tt.x >= kLog2MinAlpha && qq.x <= 0.0f;
            const bool okb = tt.y >= kLog2MinAlpha && qq.y <= 0.0f;
            if (oka || okb) {
              const float aa = oka ? fminf(0.99f, ex2_approx(tt.x)) : 0.0f;
              const float ab = okb ? fminf(0.99f, ex2_approx(tt.y)) : 0.0f;
              const f32x2 w2 = mul2(pk2(aa, ab), T2);
              const f32x2 n2 = sub2(T2, w2);
              const float2 ww = upk2(w2), tn = upk2(n2), to = upk2(T2);
              const bool sa = tn.x < 1e-4f, sb = tn.y < 1e-4f;
              T2 = pk2(sa ? to.x : tn.x, sb ? to.y : tn.y);
              float ca, cb;
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(ca) : "r"(ra + oa));
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(cb) : "r"(ra + ob));
              C2 = fma2(pk2(ca, cb), pk2(sa ? 0.0f : ww.x, sb ? 0.0f : ww.y), C2);
              if (sa || sb) {  // a subpixel saturated (Z9): it stops here
                const float2 px = upk2(PX);
                PX = pk2(sa ? kNaN : px.x, sb ? kNaN : px.y);
                if (COUNT) {
                  if (sa) qa = 31 - q;
                  if (sb) qb = 31 - q;
                }
                dd |= (sa ? 1u : 0u) | (sb ? 2u : 0u);
                if (dd == 3u) mm = 0u;
              }
            }
          }
          if (COUNT) {
            if (active) nev += (qa >= 0) ? (unsigned)(qa + 1) : ((dd & 1u) ? 0u : (unsigned)n);
            if (active && hasb) nev += (qb >= 0) ? (unsigned)(qb + 1) : ((dd & 2u) ? 0u : (unsigned)n);
          }
        }
        if (__all_sync(0xffffffffu, dd == 3u)) break;
        __syncwarp();
      }
      __syncwarp();
      if (active) {
        uint32_t pq;  // re-decode after the walk (nothing of it stays live across)
        asm volatile("mov.b32 %0, %1;" : "=r"(pq) : "r"(pr));
        const int la = (int)(pq & 0xFFFFu), lb = (int)(pq >> 16);
        decode(pq, xa, ya, ua);
        if (hasb) decode(pq >> 16, xb, yb, ub);
        const float2 cc = upk2(C2), tt = upk2(T2);
        const float va = cc.x + c_fp.bg[ua] * tt.x;
        const float vb = cc.y + c_fp.bg[ub] * tt.y;
        if (tsplit == 1) {
          s_out[la] = va;
          if (hasb) s_out[lb] = vb;
        } else {
          const long long oa = ((long long)(ya - c_fp.row0 * 16) * W + xa) * 3 + ua;
          const long long ob = ((long long)(yb - c_fp.row0 * 16) * W + xb) * 3 + ub;
          if (FMT == 0) {
            ((uint8_t*)out)[oa] = (uint8_t)quant_u8(va);
            if (hasb) ((uint8_t*)out)[ob] = (uint8_t)quant_u8(vb);
          } else {
            ((float*)out)[oa] = va;
            if (hasb) ((float*)out)[ob] = vb;
          }
        }
      }
    }
  }
  if (COUNT) add_evals(evals, nev);
  if (tsplit == 1) {
    __syncthreads();
    store_tile<FMT>(s_out, out, tx, ty, W, H, c_fp.row0 * 16);
  }
}

// ===========================================================================
// Full-frame render of every view, then interlace.
// CTA = (tile, view j): 256 threads = the tile's pixels, RGB per thread; list
// (t, k(j)) of the binning at cluster size s (s = 1: the traditional N1
// baseline, each view with its own attributes; s > 1: the per-view images of
// Cross-view Coherent Attribute Reuse that the paper evaluates);
// entries staged in shared memory 256 at a time with their view-j mean; a
// CTA-wide count ends the list when all pixels saturate.  Each channel uses
// exactly the staged kernel's blend arithmetic, so interlacing the frames
// reproduces the subpixel render at the same s bit for bit.
// ===========================================================================
template <int FMT>
__global__ void __launch_bounds__(256) k_fullframe(const uint32_t* __restrict__ S,
                                                   const uint32_t* __restrict__ E,
                                                   const uint32_t* __restrict__ vals,
                                                   const float4* __restrict__ rec,
                                                   const float4* __restrict__ mean4,
                                                   void* __restrict__ frames) {
  __shared__ float4 s_g[256];
  __shared__ float4 s_c[256];
  __shared__ float2 s_m[256];
  const int W = c_fp.W, H = c_fp.H, TX = c_fp.TX, K = c_fp.K;
  const long long M = c_fp.M;
  const int t = c_fp.row0 * TX + (int)(blockIdx.x % (unsigned)((c_fp.row1 - c_fp.row0) * TX));
  const int j = (int)(blockIdx.x / (unsigned)((c_fp.row1 - c_fp.row0) * TX));
  const int tx = t % TX, ty = t / TX;
  const int x = tx * 16 + (threadIdx.x & 15), y = ty * 16 + (threadIdx.x >> 4);
  const bool inside = x < W && y < H;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  const int k = j / c_fp.s;  // GetClusterID(j)
  const uint32_t e0 = S[t * K + k], e1 = E[t * K + k];
  const long long kM = (long long)k * M;
  const CamDev& cam = c_cams[j];
  float T[3] = {1.f, 1.f, 1.f}, C[3] = {0.f, 0.f, 0.f};
  bool done[3] = {!inside, !inside, !inside};
  for (uint32_t b = e0; b < e1; b += 256) {
    __syncthreads();
    const uint32_t e = b + threadIdx.x;
    if (e < e1) {
      const uint32_t r = vals[e];
      const float4 m = mean4[(long long)r - kM];
      s_g[threadIdx.x] = rec[2ull * r];
      s_c[threadIdx.x] = rec[2ull * r + 1];
      s_m[threadIdx.x] = mean2d_fast(cam, m.x, m.y, m.z);
    }
    __syncthreads();
    const int n = (int)min(256u, e1 - b);
    for (int q = 0; q < n && !(done[0] && done[1] && done[2]); ++q) {
      const float4 g = s_g[q];
      const float2 mu = s_m[q];
      const float4 cl = s_c[q];
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (!done[u]) blend_step(g, mu, (&cl.x)[u], px, py, T[u], C[u], done[u]);
    }
    if (__syncthreads_count(done[0] && done[1] && done[2]) == 256) break;
  }
  if (!inside) return;
  const long long o = ((((long long)j * (c_fp.row1 - c_fp.row0) * 16 + (y - c_fp.row0 * 16)) * W) + x) * 3;
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const float v = C[u] + c_fp.bg[u] * T[u];
    if (FMT == 0) {
      const float cl = fminf(fmaxf(v, 0.0f), 1.0f);
      ((uint8_t*)frames)[o + u] = (uint8_t)floorf(__fadd_rn(__fmul_rn(cl, 255.0f), 0.5f));
    } else {
      ((float*)frames)[o + u] = v;
    }
  }
}

// interlace: out[y][x][u] = F_{V[y][x][u]}[y][x][u] for the band
template <int FMT>
__global__ void k_interlace(const uint8_t* __restrict__ V, const void* __restrict__ frames,
                            void* __restrict__ out, int rows_px) {
  const long long n = (long long)rows_px * c_fp.W * 3;
  const long long plane = n;
  const long long base = (long long)c_fp.row0 * 16 * c_fp.W * 3;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = V[base + q];
    if (FMT == 0) ((uint8_t*)out)[q] = ((const uint8_t*)frames)[(long long)j * plane + q];
    else ((float*)out)[q] = ((const float*)frames)[(long long)j * plane + q];
  }
}

template <int FMT, bool COUNT>
__global__ void __launch_bounds__(kTileSub) k_composite_thread(
    const uint8_t* __restrict__ V, const uint16_t* __restrict__ psi,
    const uint32_t* __restrict__ S, const uint32_t* __restrict__ E,
    const uint32_t* __restrict__ vals, const float4* __restrict__ rec0,
    const float4* __restrict__ rec1, const float4* __restrict__ mean4, void* __restrict__ out,
    unsigned long long* __restrict__ evals) {
  const int W = c_fp.W, H = c_fp.H, TX = c_fp.TX, K = c_fp.K, s = c_fp.s;
  const long long M = c_fp.M;
  const int t = c_fp.row0 * TX + blockIdx.x;
  const int tx = t % TX, ty = t / TX;
  const int r = threadIdx.x;
  int l = r;
  if (c_fp.remap) l = psi[(long long)t * kTileSub + r];  // x^ = Psi(r)
  const int ly = l / 48, rem = l % 48, lx = rem / 3, u = rem % 3;
  const int x = tx * 16 + lx, y = ty * 16 + ly;
  const bool in_panel = l != 0xFFFF && x < W && y < H;
  if (!in_panel) return;
  const int j = V[((long long)y * W + x) * 3 + u];  // j = V[x^]
  const int k = j / s;                                // k = GetClusterID(j)
  const uint32_t e0 = S[t * K + k], e1 = E[t * K + k];
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  const CamDev& cam = c_cams[j];
  const long long kM = (long long)k * M;
  float T = 1.0f, C = 0.0f;
  bool done = false;
  unsigned long long nev = 0;
  for (uint32_t e = e0; e < e1 && !done; ++e) {
    if (COUNT) ++nev;
    const uint32_t rr = vals[e];
    const float4 m = mean4[(long long)rr - kM];
    const float2 mu = mean2d_fast(cam, m.x, m.y, m.z);
    const float4 g = rec0[2ull * rr];
    const float4 cl = rec0[2ull * rr + 1];
    blend_step(g, mu, (&cl.x)[u], px, py, T, C, done);
  }
  if (COUNT) atomicAdd(evals, nev);
  const float v = C + c_fp.bg[u] * T;
  const long long o = ((long long)(y - c_fp.row0 * 16) * W + x) * 3 + u;
  if (FMT == 0) {
    const float cl = fminf(fmaxf(v, 0.0f), 1.0f);
    ((uint8_t*)out)[o] = (uint8_t)floorf(__fadd_rn(__fmul_rn(cl, 255.0f), 0.5f));
  } else {
    ((float*)out)[o] = v;
  }
}

}  // namespace cr
