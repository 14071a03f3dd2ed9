// cr_kernels.cuh — display, upload, preprocess (+tile-union count), emit and
// range kernels of the CoherentRaster B200 path.  See DESIGN.md §5 for the
// roofline of each kernel and its algorithmic bytes per unit.
#pragma once
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

// Composite work items: per tile, "cluster-aligned warp chunks" of <= 32
// consecutive Psi ranks that share one cluster k (DESIGN.md §5 composite).
// Packed as start | (len-1) << 10 | k << 16.  One thread per tile.
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
    if (k != seg_k || r - seg_start == 32) {
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

// ===========================================================================
// Upload (O4): Sigma3D = R S S^T R^T in fp64 with explicit rounding (same
// order as written in DESIGN.md O4), SH transposed to coefficient-major SoA.
// mean4 = (mu, tau), cov8 = {S00,S01,S02,S11},{S12,S22,o,0}.
// ===========================================================================
__global__ void k_upload(long long M, int nc3, const float* __restrict__ means,
                         const float* __restrict__ quats, const float* __restrict__ scales,
                         const float* __restrict__ opac, const float* __restrict__ tau,
                         const float* __restrict__ sh, float4* __restrict__ mean4,
                         float4* __restrict__ cov8, float* __restrict__ shsoa,
                         int* __restrict__ nonfinite) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= M) return;
  bool bad = false;
  float q4[4], s3[3], m3[3];
#pragma unroll
  for (int a = 0; a < 4; ++a) { q4[a] = quats[4 * i + a]; bad |= !isfinite(q4[a]); }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    s3[a] = scales[3 * i + a];
    m3[a] = means[3 * i + a];
    bad |= !isfinite(s3[a]) || !isfinite(m3[a]);
  }
  const float o = opac[i];
  bad |= !isfinite(o);
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
  for (int q = 0; q < nc3; ++q) {
    const float v = sh[(long long)i * nc3 + q];
    bad |= !isfinite(v);
    shsoa[(long long)q * M + i] = v;
  }
  if (bad) atomicOr(nonfinite, 1);
}

// ===========================================================================
// O8 — cluster tile union (Alg.2 GenerateKeys) restricted to the
// band rows.  EMIT=false counts; EMIT=true writes tile ids (ascending within
// each row, rows ascending) + payload r.  Identical set on both passes: the
// same inputs go through the same exactly-rounded code.
// ===========================================================================
template <bool EMIT>
__device__ uint32_t tile_union(int k, float mux, float muy, float muz, float a, float b, float c,
                               float det, float tau, uint32_t* __restrict__ out_t,
                               uint32_t* __restrict__ out_v, uint32_t payload) {
  const int s = c_fp.s, N = c_fp.N, TX = c_fp.TX, TY = c_fp.TY;
  const int j0 = k * s;
  const int nv = min(j0 + s, N) - j0;
  float vmx[kMaxCluster], vmy[kMaxCluster];
  int vrow[kMaxCluster];  // ty0 | ty1 << 16 as 16-bit fields; ty0 = -1 marks an invisible view
  float ex = 0.f, ey = 0.f;
  int rmin = TY, rmax = -1;
  for (int l = 0; l < nv; ++l) {
    const CamDev& cam = c_cams[j0 + l];
    const F3 p = cam_point_exact(cam, mux, muy, muz);
    if (!(p.z >= c_fp.znear)) {  // Z12: this view contributes no tiles
      vrow[l] = 0x0000FFFF;      // ty0 = -1 (never produced for a visible view)
      continue;
    }
    float mx, my;
    mean2d_exact(cam, p, mx, my);
    const ViewRows vr = view_rows(mx, my, a, c, tau, TY);
    ex = vr.ex;
    ey = vr.ey;
    vmx[l] = mx;
    vmy[l] = my;
    vrow[l] = (vr.ty0 & 0xFFFF) | ((vr.ty1 & 0xFFFF) << 16);
    rmin = min(rmin, vr.ty0);
    rmax = max(rmax, vr.ty1);
  }
  rmin = max(rmin, c_fp.row0);
  rmax = min(rmax, c_fp.row1 - 1);
  uint32_t n = 0;
  int iv[kMaxCluster];
  for (int ty = rmin; ty <= rmax; ++ty) {
    int lo = 0x7fffffff, hi = -1, ni = 0;
    for (int l = 0; l < nv; ++l) {
      const int ty0 = (int)(short)(vrow[l] & 0xFFFF), ty1 = (int)(short)(vrow[l] >> 16);
      if (ty0 < 0 || ty < ty0 || ty > ty1) continue;  // invisible view or row outside
      ViewRows vr;
      vr.mx = vmx[l]; vr.my = vmy[l]; vr.ex = ex; vr.ey = ey;
      int tx0, tx1;
      if (!view_row_cols(vr, a, b, c, det, tau, ty, TX, tx0, tx1)) continue;
      if (tx0 > tx1) continue;
      iv[ni++] = tx0 | (tx1 << 16);
      lo = min(lo, tx0);
      hi = max(hi, tx1);
    }
    if (ni == 0) continue;
    const uint32_t rowbase = (uint32_t)ty * (uint32_t)TX;
    if (hi - lo < 64) {
      unsigned long long mask = 0ull;
      for (int q = 0; q < ni; ++q) {
        const int s0 = iv[q] & 0xFFFF, s1 = iv[q] >> 16;
        const int len = s1 - s0 + 1;
        const unsigned long long bits = (len >= 64) ? ~0ull : ((1ull << len) - 1ull);
        mask |= bits << (s0 - lo);
      }
      if (EMIT) {
        unsigned long long m = mask;
        uint32_t q = n;
        while (m) {
          const int bit = __ffsll((long long)m) - 1;
          m &= m - 1;
          out_t[q] = rowbase + (uint32_t)(lo + bit);
          out_v[q] = payload;
          ++q;
        }
      }
      n += (uint32_t)__popcll(mask);
    } else {
      for (int tx = lo; tx <= hi; ++tx) {
        bool hit = false;
        for (int q = 0; q < ni; ++q) hit |= ((iv[q] & 0xFFFF) <= tx && tx <= (iv[q] >> 16));
        if (hit) {
          if (EMIT) {
            out_t[n] = rowbase + (uint32_t)tx;
            out_v[n] = payload;
          }
          ++n;
        }
      }
    }
  }
  return n;
}

// ===========================================================================
// a4 — Preprocess + SH (Cross-view Coherent Attribute Reuse, Eq.6)
// fused with the tile-union count (a6).  One thread per Gaussian, looping
// over the K clusters so the SH coefficients are read once and evaluated K
// times.  Writes per (k,i) (index r = k*M + i, k-major):
//   rec0[r] = (A', B', C', log2 o)  conic prescaled by -log2(e)/2, -log2(e)
//   rec1[r] = (r, g, b, depth)      colour at v'_k, depth d_{i,k}
//   cnt[r]  = |T_{i,k}| in the band (0 if culled)
//   dkey[r] = bits(d_{i,k})
// ===========================================================================
constexpr float kLog2e = 1.4426950408889634f;

template <int DEG>
__global__ void __launch_bounds__(128) k_preprocess(
    const float4* __restrict__ mean4, const float4* __restrict__ cov8,
    const float* __restrict__ shsoa, float4* __restrict__ rec0, float4* __restrict__ rec1,
    uint32_t* __restrict__ cnt, uint32_t* __restrict__ dkey,
    unsigned long long* __restrict__ counters /* near, degenerate, opacity */) {
  constexpr int NC = (DEG + 1) * (DEG + 1);
  const long long M = c_fp.M;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned n_near = 0, n_deg = 0, n_op = 0;
  if (i < M) {
    const float4 m = mean4[i];
    const float tau = m.w;
    const float4 ca = cov8[2 * i], cb = cov8[2 * i + 1];
    const float S6[6] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y};
    const float o = cb.z;
    float sh[NC][3];
#pragma unroll
    for (int q = 0; q < NC; ++q)
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) sh[q][ch] = shsoa[(long long)(q * 3 + ch) * M + i];
    const float lo2 = log2f(o);
    const int K = c_fp.K;
    if (!(tau > 0.0f)) n_op = 1;
    for (int k = 0; k < K; ++k) {
      const long long r = (long long)k * M + i;
      if (!(tau > 0.0f)) { cnt[r] = 0; continue; }
      const int jr = c_rep[k];
      const CamDev& rc = c_cams[jr];
      const F3 p = cam_point_exact(rc, m.x, m.y, m.z);
      if (p.z < c_fp.znear) { cnt[r] = 0; ++n_near; continue; }
      float a, b, c, det;
      if (!cov2d_exact(rc, c_ccon[jr], p, S6, a, b, c, det)) { cnt[r] = 0; ++n_deg; continue; }
      // conic (tolerance path), prescaled for exp2
      const float A = c / det, B = -b / det, C = a / det;
      rec0[r] = make_float4(-0.5f * kLog2e * A, -kLog2e * B, -0.5f * kLog2e * C, lo2);
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
      rec1[r] = make_float4(col[0], col[1], col[2], p.z);
      dkey[r] = __float_as_uint(p.z);
      cnt[r] = tile_union<false>(k, m.x, m.y, m.z, a, b, c, det, tau, nullptr, nullptr, 0);
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
}

// ===========================================================================
// a6 emit — one thread per depth-sorted visible record e: recompute Sigma2D
// at v'_k and the cluster tile union, write <tile, r> at offs[e].
// ===========================================================================
__global__ void __launch_bounds__(128) k_emit(const uint32_t* __restrict__ rec_sorted,
                                              const uint32_t* __restrict__ offs, uint32_t nrec,
                                              const float4* __restrict__ mean4,
                                              const float4* __restrict__ cov8,
                                              uint32_t* __restrict__ out_t,
                                              uint32_t* __restrict__ out_v) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nrec) return;
  const uint32_t r = rec_sorted[e];
  const long long M = c_fp.M;
  const int k = (int)(r / (unsigned long long)M);
  const long long i = (long long)r - (long long)k * M;
  const float4 m = mean4[i];
  const float4 ca = cov8[2 * i], cb = cov8[2 * i + 1];
  const float S6[6] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y};
  const int jr = c_rep[k];
  const F3 p = cam_point_exact(c_cams[jr], m.x, m.y, m.z);
  float a, b, c, det;
  cov2d_exact(c_cams[jr], c_ccon[jr], p, S6, a, b, c, det);
  const uint32_t o = offs[e];
  tile_union<true>(k, m.x, m.y, m.z, a, b, c, det, m.w, out_t + o, out_v + o, r);
}

// ===========================================================================
// a8 — ranges [S_{t,k}, E_{t,k}) from the (t, k)-sorted pairs.
// ===========================================================================
__global__ void k_ranges(const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ val,
                         uint32_t P, uint32_t* __restrict__ S, uint32_t* __restrict__ E) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P) return;
  const unsigned long long M = (unsigned long long)c_fp.M;
  const int K = c_fp.K;
  const uint32_t t = tkey[e];
  const uint32_t k = (uint32_t)(val[e] / M);
  const uint32_t slot = t * K + k;
  if (e == 0 || tkey[e - 1] != t || (uint32_t)(val[e - 1] / M) != k) S[slot] = e;
  if (e == P - 1 || tkey[e + 1] != t || (uint32_t)(val[e + 1] / M) != k) E[slot] = e + 1;
}

// Introspection: 64-bit keys of Eq.11 and payload i.
__global__ void k_make_keys(const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ val,
                            const uint32_t* __restrict__ dkey, uint32_t P,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ pay) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P) return;
  const unsigned long long M = (unsigned long long)c_fp.M;
  const uint32_t r = val[e];
  const unsigned long long k = r / M;
  keys[e] = ((unsigned long long)tkey[e] << (32 + c_fp.bitK)) | (k << 32) |
            (unsigned long long)dkey[r];
  pay[e] = (uint32_t)(r - k * M);
}

}  // namespace cr
