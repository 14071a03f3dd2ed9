// Compare the packed view_row_cols (cr_device.cuh) with the scalar reading on
// random inputs, including huge footprints.
#include <cstdio>
#include "../../paper_2605_04509_b200/csrc/cr_device.cuh"
using namespace cr;
__device__ bool vrc_ref(const EllRec& e, float mx, float my, int ty, int TX, int& tx0, int& tx1) {
  const float dlo = xmax(xsub(xadd(xmul(16.0f, (float)ty), 0.5f), my), -e.ey);
  const float dhi = xmin(xsub(xadd(xmul(16.0f, (float)ty), 15.5f), my), e.ey);
  if (dlo > dhi) return false;
  const float dyR = e.dyR, dyL = -e.dyR;
  const bool rin = dlo <= dyR && dyR <= dhi, lin = dlo <= dyL && dyL <= dhi;
  float right = e.ex, left = -e.ex;
  if (!(rin && lin)) {
    const float hlo = xsqrt(xmax(0.0f, xmul(e.det, xsub(e.tc, xmul(dlo, dlo)))));
    const float hhi = xsqrt(xmax(0.0f, xmul(e.det, xsub(e.tc, xmul(dhi, dhi)))));
    const float bl = xmul(e.b, dlo), bh = xmul(e.b, dhi);
    if (!rin) right = xmax(xmul(xadd(bl, hlo), e.ic), xmul(xadd(bh, hhi), e.ic));
    if (!lin) left = xmin(xmul(xsub(bl, hlo), e.ic), xmul(xsub(bh, hhi), e.ic));
  }
  tx0 = clamp_to_int(ceilf(xmul(xsub(xadd(mx, left), 15.5f), 0.0625f)), 0.0f, (float)TX);
  tx1 = clamp_to_int(floorf(xmul(xsub(xadd(mx, right), 0.5f), 0.0625f)), -1.0f, (float)(TX - 1));
  return true;
}
__device__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }
__device__ float u01(uint32_t s) { return (hsh(s) >> 8) * (1.0f / 16777216.0f); }
__global__ void k(unsigned long long n, unsigned long long* bad, float* ex) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n; i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i * 16);
    // random ellipse: sigma 0.3 .. 3000 px, correlation, tau
    const float sx = exp2f(-2.f + 14.f * u01(s)), sy = exp2f(-2.f + 14.f * u01(s + 1));
    const float rho = 0.999f * (2.f * u01(s + 2) - 1.f);
    const float a = __fadd_rn(__fmul_rn(sx, sx), 0.3f), c = __fadd_rn(__fmul_rn(sy, sy), 0.3f);
    const float b = __fmul_rn(__fmul_rn(rho, sx), sy);
    const float det = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, b));
    if (!(det > 0.f)) continue;
    const float tau = 2.f * logf(255.f * (0.01f + u01(s + 3)));
    if (!(tau > 0.f)) continue;
    EllRec e = ell_rec(a, b, c, det, tau);
    const float mx = -3000.f + 10000.f * u01(s + 4), my = -3000.f + 10000.f * u01(s + 5);
    const int ty = (int)(u01(s + 6) * 300.f);
    int p0, p1, q0, q1;
    const bool rp = view_row_cols(e, mx, my, ty, 480, p0, p1);
    const bool rq = vrc_ref(e, mx, my, ty, 480, q0, q1);
    if (rp != rq || (rp && (p0 != q0 || p1 != q1))) {
      if (atomicAdd(bad, 1) < 1) {
        ex[0] = a; ex[1] = b; ex[2] = c; ex[3] = det; ex[4] = tau; ex[5] = mx; ex[6] = my; ex[7] = ty;
        ex[8] = rp; ex[9] = p0; ex[10] = p1; ex[11] = rq; ex[12] = q0; ex[13] = q1;
      }
    }
  }
}
int main() {
  unsigned long long* bad; float* ex;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&ex, 64 * 4);
  *bad = 0;
  k<<<148 * 8, 256>>>(1ull << 31, bad, ex);
  cudaDeviceSynchronize();
  printf("view_row_cols packed vs scalar: %llu mismatches of 2^31\n", *bad);
  if (*bad) for (int q = 0; q < 14; ++q) printf("  ex[%d] = %.9g\n", q, ex[q]);
  return 0;
}
