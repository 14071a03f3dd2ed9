// cr_device.cuh — device-side state and exact-arithmetic helpers of the
// CoherentRaster B200 path.  Included once by cr_api.cu (unity build, so the
// __constant__ rig is visible to every kernel without -rdc).
//
// Exactness rule (DESIGN.md §3 "exact path"): everything that decides a view
// index, a sort key or a tile list is computed with explicitly rounded IEEE
// intrinsics (__fadd_rn/__fmul_rn/__fdiv_rn/__fsqrt_rn; fp64 __d*_rn for the
// view map and Sigma3D), so ptxas can neither contract to FMA nor
// approximate, and min/max are plain compares.  Colours, conics and alpha are
// "tolerance path" values and use fast FMA / MUFU math.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cr {

constexpr int kTile = 16;
constexpr int kTileSub = kTile * kTile * 3;  // 768 subpixels per tile
constexpr int kMaxViews = 255;
constexpr int kMaxCluster = 32;
constexpr int kPairSlots = 1024;  // paired composite slots per tile (k_pairs_build)

struct __align__(16) CamDev {
  float R[9], t[3], fx, fy, cx, cy;  // 64 B
};
struct CamConstDev {
  float limxp, limxn, limyp, limyn;  // EWA frustum clamp (O6)
  float C[3];                        // camera centre -R^T t (O11)
  float pad;
};
// n / d for 32-bit n by a runtime divisor (Granlund-Montgomery round-up
// method): q = umulhi(n, m); (q + ((n - q) >> 1)) >> sh; d == 1 special.
struct FastDiv {
  uint32_t d, m, sh;
};
__host__ __device__ inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0u, 0u};
  if (d <= 1) return f;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
  f.sh = l - 1;
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  if (f.d <= 1) return n;
  const uint32_t q = __umulhi(n, f.m);
  return (q + ((n - q) >> 1)) >> f.sh;
}

struct FrameParams {
  int W, H, TX, TY, N, s, K, bitK;
  int row0, row1;  // tile-row band [row0, row1)
  int deg;
  int remap;
  long long M;
  FastDiv divM;  // record r = k*M + i  ->  k = fdiv(r, divM)
  float znear;
  float bg[3];
  int exp;  // CR_EXP developer A/B switches (0 = shipped path)
};

__constant__ CamDev c_cams[kMaxViews];
__constant__ CamConstDev c_ccon[kMaxViews];
__constant__ int c_rep[kMaxViews];
// Per cluster k: bound of the camera-space displacement between the
// representative view and any view j of the cluster.  With p_j = A_j p + b_j
// (p in rep camera space) and a centre c (least-squares fixed point of the
// cluster's rigid motions): |p_j - p| <= dA |p - c| + db, dA = max_j ||A_j - I||_F,
// db = max_j |(A_j - I) c + b_j|.  c_clb[k] = (c.x, c.y, c.z, dA), c_cldb[k] = db.
__constant__ float4 c_clb[kMaxViews];
__constant__ float c_cldb[kMaxViews];
// Per camera-space axis a: |p_j,a - p_a| <= dA_a |p - c| + db_a with dA_a = max_j
// ||row a of (A_j - I)||, db_a = max_j |((A_j - I) c + b_j)_a| (a row band only
// needs the y shift, which a horizontal camera motion keeps small).
__constant__ float4 c_clax[kMaxViews];  // (dA_x, dA_y, dA_z, 0)
__constant__ float4 c_clbx[kMaxViews];  // (db_x, db_y, db_z, 0)
__constant__ FrameParams c_fp;

// ---------------------------------------------------------------- exact ops
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float xsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float xdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float xsqrt(float a) { return __fsqrt_rn(a); }
// sqrt of a value already clamped to >= +0: +0 skips __fsqrt_rn, whose range
// check sends zero to its slow-path subroutine (same result, +0)
__device__ __forceinline__ float xsqrt_nn(float a) { return a > 0.0f ? __fsqrt_rn(a) : a; }
__device__ __forceinline__ float xmin(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ float xmax(float a, float b) { return (a < b) ? b : a; }
__device__ __forceinline__ int clamp_to_int(float v, float lo, float hi) {
  if (!(v >= lo)) v = lo;
  if (v > hi) v = hi;
  return (int)v;
}

// Packed fp32x2 (sm_100a FADD2 / FMUL2 / FFMA2): each half is the correctly
// rounded IEEE result of the scalar op (.rn, no FTZ), so packing two
// independent exact-path operations changes no bit.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(f32x2 r) {
  float2 f;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(r));
  return f;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// CAUTION: ptxas contracts a packed mul feeding a packed add / sub into one
// FFMA2 (single rounding) whatever the .rn qualifier or -fmad=false (also
// fma(a, b, -0) + c), so on the exact path a packed product may only feed a
// multiply, a compare or a SCALAR add (__fadd_rn is never contracted).
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 bc2(float a) { return pk2(a, a); }

struct F3 {
  float x, y, z;
};

// O5: camera-space point, each product/sum rounded in the written order.
__device__ __forceinline__ F3 cam_point_exact(const CamDev& c, float mx, float my, float mz) {
  F3 p;
  p.x = xadd(xadd(xadd(xmul(c.R[0], mx), xmul(c.R[1], my)), xmul(c.R[2], mz)), c.t[0]);
  p.y = xadd(xadd(xadd(xmul(c.R[3], mx), xmul(c.R[4], my)), xmul(c.R[5], mz)), c.t[1]);
  p.z = xadd(xadd(xadd(xmul(c.R[6], mx), xmul(c.R[7], my)), xmul(c.R[8], mz)), c.t[2]);
  return p;
}
// Eq.5: mu2D = (fx * (px/pz) + cx, fy * (py/pz) + cy)
__device__ __forceinline__ void mean2d_exact(const CamDev& c, const F3& p, float& ox, float& oy) {
  ox = xadd(xmul(c.fx, xdiv(p.x, p.z)), c.cx);
  oy = xadd(xmul(c.fy, xdiv(p.y, p.z)), c.cy);
}

// O6: EWA Sigma2D at camera c (gsplat classic: +0.3, no compensation).
// S6 = {00, 01, 02, 11, 12, 22}.  Returns det > 0.
__device__ __forceinline__ bool cov2d_exact(const CamDev& c, const CamConstDev& k, const F3& p,
                                            const float* S6, float& a, float& b, float& cc,
                                            float& det) {
  const float txz = xdiv(p.x, p.z), tyz = xdiv(p.y, p.z);
  const float tx = xmul(p.z, xmin(k.limxp, xmax(-k.limxn, txz)));
  const float ty = xmul(p.z, xmin(k.limyp, xmax(-k.limyn, tyz)));
  const float zz = xmul(p.z, p.z);
  const float J00 = xdiv(c.fx, p.z), J02 = -xdiv(xmul(c.fx, tx), zz);
  const float J11 = xdiv(c.fy, p.z), J12 = -xdiv(xmul(c.fy, ty), zz);
  float T0[3], T1[3];
#pragma unroll
  for (int col = 0; col < 3; ++col) {
    T0[col] = xadd(xmul(J00, c.R[col]), xmul(J02, c.R[6 + col]));
    T1[col] = xadd(xmul(J11, c.R[3 + col]), xmul(J12, c.R[6 + col]));
  }
  const float S[3][3] = {{S6[0], S6[1], S6[2]}, {S6[1], S6[3], S6[4]}, {S6[2], S6[4], S6[5]}};
  float U0[3], U1[3];
#pragma unroll
  for (int col = 0; col < 3; ++col) {
    U0[col] = xadd(xadd(xmul(T0[0], S[0][col]), xmul(T0[1], S[1][col])), xmul(T0[2], S[2][col]));
    U1[col] = xadd(xadd(xmul(T1[0], S[0][col]), xmul(T1[1], S[1][col])), xmul(T1[2], S[2][col]));
  }
  a = xadd(xadd(xmul(U0[0], T0[0]), xmul(U0[1], T0[1])), xmul(U0[2], T0[2]));
  b = xadd(xadd(xmul(U0[0], T1[0]), xmul(U0[1], T1[1])), xmul(U0[2], T1[2]));
  cc = xadd(xadd(xmul(U1[0], T1[0]), xmul(U1[1], T1[1])), xmul(U1[2], T1[2]));
  a = xadd(a, 0.3f);
  cc = xadd(cc, 0.3f);
  det = xsub(xmul(a, cc), xmul(b, b));
  return det > 0.0f;
}

// O7 (AccuTile reading): tiles whose pixel-centre rectangle meets the ellipse
// {d^T Sigma^-1 d <= tau}.  Per-record constants (view independent: the
// cluster shares Sigma2D, Eq.6) are evaluated once; x/16 is evaluated as
// x*0.0625 (both are the correctly rounded x*2^-4: bit-identical).
struct EllRec {
  float a, b, c, det, tau;
  float ex, ey;  // sqrt(tau a), sqrt(tau c): x / y half extents
  float dyR;     // (b ex)/a: dy of the rightmost point
  float tc;      // tau c
  float ic;      // 1/c (rounded once)
};
__device__ __forceinline__ EllRec ell_rec(float a, float b, float c, float det, float tau) {
  EllRec e;
  e.a = a; e.b = b; e.c = c; e.det = det; e.tau = tau;
  e.ex = xsqrt(xmul(tau, a));
  e.ey = xsqrt(xmul(tau, c));
  e.dyR = xdiv(xmul(b, e.ex), a);
  e.tc = xmul(tau, c);
  e.ic = xdiv(1.0f, c);
  return e;
}
// the stored form: g0 = (ex, ey, dyR, tc), g1 = (ic, b, det, 0)
__device__ __forceinline__ EllRec ell_load(const float4& g0, const float4& g1) {
  EllRec e;
  e.a = 0.f; e.c = 0.f; e.tau = 0.f;
  e.ex = g0.x; e.ey = g0.y; e.dyR = g0.z; e.tc = g0.w;
  e.ic = g1.x; e.b = g1.y; e.det = g1.z;
  return e;
}
// row range [ty0, ty1] of one view (mean my)
__device__ __forceinline__ void view_rows(const EllRec& e, float my, int TY, int& ty0, int& ty1) {
  ty0 = clamp_to_int(ceilf(xmul(xsub(xsub(my, e.ey), 15.5f), 0.0625f)), 0.0f, (float)TY);
  ty1 = clamp_to_int(floorf(xmul(xsub(xadd(my, e.ey), 0.5f), 0.0625f)), -1.0f, (float)(TY - 1));
}
// Tile columns [tx0, tx1] of row ty for one view (mean mx, my); false when
// the row band misses the ellipse.
__device__ __forceinline__ bool view_row_cols(const EllRec& e, float mx, float my, int ty, int TX,
                                              int& tx0, int& tx1) {
  // the row's band ends (dlo, dhi) and, below, the slice ends / column
  // arguments of both sides as packed pairs: the same rounded operations as
  // the scalar reading of O7, two per instruction
  const float2 d = upk2(sub2(add2(bc2(xmul(16.0f, (float)ty)), pk2(0.5f, 15.5f)), bc2(my)));
  const float dlo = xmax(d.x, -e.ey);
  const float dhi = xmin(d.y, e.ey);
  if (dlo > dhi) return false;
  const float dyR = e.dyR, dyL = -e.dyR;
  const bool rin = dlo <= dyR && dyR <= dhi, lin = dlo <= dyL && dyL <= dhi;
  float right = e.ex, left = -e.ex;
  if (!(rin && lin)) {  // the band misses an x-extreme: evaluate the slice ends
    // products packed, the sums after them scalar (see mul2)
    const f32x2 D = pk2(dlo, dhi);
    const float2 dd = upk2(mul2(D, D));
    const float2 hh = upk2(mul2(bc2(e.det), pk2(xsub(e.tc, dd.x), xsub(e.tc, dd.y))));
    const float hlo = xsqrt_nn(xmax(0.0f, hh.x)), hhi = xsqrt_nn(xmax(0.0f, hh.y));
    const float2 bb = upk2(mul2(bc2(e.b), D));  // (bl, bh)
    const float2 r = upk2(mul2(pk2(xadd(bb.x, hlo), xadd(bb.y, hhi)), bc2(e.ic)));
    const float2 l = upk2(mul2(pk2(xsub(bb.x, hlo), xsub(bb.y, hhi)), bc2(e.ic)));
    if (!rin) right = xmax(r.x, r.y);
    if (!lin) left = xmin(l.x, l.y);
  }
  const float2 a = upk2(mul2(sub2(add2(bc2(mx), pk2(left, right)), pk2(15.5f, 0.5f)), bc2(0.0625f)));
  tx0 = clamp_to_int(ceilf(a.x), 0.0f, (float)TX);
  tx1 = clamp_to_int(floorf(a.y), -1.0f, (float)(TX - 1));
  return true;
}

}  // namespace cr
