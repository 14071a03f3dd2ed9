#include <cstdio>
#include "../../paper_2605_04509_b200/csrc/cr_device.cuh"
using namespace cr;
__global__ void k(float a, float b, float c, float det, float tau, float mx, float my, int ty) {
  EllRec e = ell_rec(a, b, c, det, tau);
  printf("ex %.9g ey %.9g dyR %.9g tc %.9g ic %.9g\n", e.ex, e.ey, e.dyR, e.tc, e.ic);
  // scalar
  const float dlo = xmax(xsub(xadd(xmul(16.0f, (float)ty), 0.5f), my), -e.ey);
  const float dhi = xmin(xsub(xadd(xmul(16.0f, (float)ty), 15.5f), my), e.ey);
  const float dyR = e.dyR, dyL = -e.dyR;
  const bool rin = dlo <= dyR && dyR <= dhi, lin = dlo <= dyL && dyL <= dhi;
  const float m1 = xmul(dlo, dlo), s1 = xsub(e.tc, m1), p1 = xmul(e.det, s1);
  const float m2 = xmul(dhi, dhi), s2 = xsub(e.tc, m2), p2 = xmul(e.det, s2);
  const float hlo = xsqrt(xmax(0.0f, p1)), hhi = xsqrt(xmax(0.0f, p2));
  const float bl = xmul(e.b, dlo), bh = xmul(e.b, dhi);
  const float r1 = xmul(xadd(bl, hlo), e.ic), r2 = xmul(xadd(bh, hhi), e.ic);
  printf("S dlo %.9g dhi %.9g rin %d lin %d m %.9g %.9g s %.9g %.9g p %.9g %.9g h %.9g %.9g bl %.9g %.9g r %.9g %.9g\n",
         dlo, dhi, rin, lin, m1, m2, s1, s2, p1, p2, hlo, hhi, bl, bh, r1, r2);
  const f32x2 D = pk2(dlo, dhi);
  const float2 mm = upk2(mul2(D, D));
  const float2 ss = upk2(sub2(bc2(e.tc), mul2(D, D)));
  const float2 hh = upk2(mul2(bc2(e.det), sub2(bc2(e.tc), mul2(D, D))));
  const f32x2 Hs = pk2(xsqrt(xmax(0.0f, hh.x)), xsqrt(xmax(0.0f, hh.y)));
  const f32x2 B = mul2(bc2(e.b), D);
  const float2 r = upk2(mul2(add2(B, Hs), bc2(e.ic)));
  const float2 bb = upk2(B), hs = upk2(Hs);
  printf("P m %.9g %.9g s %.9g %.9g p %.9g %.9g h %.9g %.9g bl %.9g %.9g r %.9g %.9g\n",
         mm.x, mm.y, ss.x, ss.y, hh.x, hh.y, hs.x, hs.y, bb.x, bb.y, r.x, r.y);
  int t0, t1; view_row_cols(e, mx, my, ty, 480, t0, t1);
  printf("packed fn: %d %d\n", t0, t1);
}
int main() { k<<<1, 1>>>(664428.188f, 76552.1484f, 288068.562f, 1.85540641e+11f, 10.7184601f, 1669.90112f, -507.790924f, 25); cudaDeviceSynchronize(); return 0; }
