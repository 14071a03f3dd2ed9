// CoherentRaster CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Plain, slow, obviously-correct CPU implementation of what the subpixel
// light-field rasterizer of arXiv 2605.04509 ("CoherentRaster") computes.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  The product path
// (paper_2605_04509_b200/) never links, imports or executes it, and this file
// shares no code, header, table or constant generator with the CUDA path.
//
// Citations: "P:n" = /root/reference/PAPER.md line n (section / equation /
// algorithm named beside it); "S:n" = SPEC.md line n; "O1".."O12" = the
// readings in DESIGN.md §3 for everything the paper
// leaves to gsplat.
//
// Precision (reading R-prec): the paper's rasterizer is gsplat's
// fp32 rasterizer, so every quantity that decides a view index, a sort
// key, a tile list or a blend decision is evaluated in IEEE fp32 (fp64 for the
// view map) with each + - * / sqrt rounded separately in the order
// written below.  Compile with -O2 -ffp-contract=off and no fast-math.
// SH colour is evaluated in fp64 and rounded to fp32 once.
//
// Parity pins: every function is pinned by a `-m "not gpu"` test in
// tests/test_oracle_*.py (worked examples, closed forms, invariants, brute
// force).  The reuse approximation itself (Eq.6) is "parity unpinned" by
// design; its error is reported against the exact s=1 render instead.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// Small helpers.  min/max are written as plain comparisons so that their NaN
// behaviour is fully specified (returns the first operand if a compare fails).
// ---------------------------------------------------------------------------
inline float mnf(float a, float b) { return (b < a) ? b : a; }
inline float mxf(float a, float b) { return (a < b) ? b : a; }
// clamp in the float domain before any float->int conversion (O7 "Float->int")
inline int clamp_to_int(float v, float lo, float hi) {
    if (!(v >= lo)) v = lo;  // also maps NaN to lo
    if (v > hi) v = hi;
    return (int)v;
}

int hw_threads(int req) {
    if (req > 0) return req;
    unsigned h = std::thread::hardware_concurrency();
    return h ? (int)h : 1;
}

template <class F>
void parallel_for(int64_t n, int nthreads, F f) {
    if (n <= 0) return;
    if (nthreads <= 1 || n < 2) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<int64_t> next(0);
    const int64_t chunk = std::max<int64_t>(1, n / (int64_t(nthreads) * 16));
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t)
        th.emplace_back([&]() {
            for (;;) {
                int64_t b = next.fetch_add(chunk);
                if (b >= n) break;
                int64_t e = std::min(n, b + chunk);
                for (int64_t i = b; i < e; ++i) f(i);
            }
        });
    for (auto& x : th) x.join();
}

// ---------------------------------------------------------------------------
// O1 — viewpoint index, Eqs.1–3 (§3.1).  fp64, floor-mod
// into [0, Lx), j clamped into [0, N-1].
// ---------------------------------------------------------------------------
int view_index(int x, int y, int u, int N, double Lx, double tA, double Koff) {
    double s = (double)(3 * x + u);
    double t1 = (double)(3 * y) * tA;
    double d = (s + t1) - Koff;                 // Eq.1 d_offset
    double q = std::floor(d / Lx);
    double xo = d - q * Lx;                     // Eq.2 x_offset = d mod Lx
    if (xo < 0) xo += Lx;
    if (xo >= Lx) xo -= Lx;
    int j = (int)std::floor(((double)N * xo) / Lx);  // Eq.3
    if (j < 0) j = 0;
    if (j > N - 1) j = N - 1;
    return j;
}

// ---------------------------------------------------------------------------
// O4 — upload-time per-Gaussian constants (fp64 -> fp32 once).
// Sigma = R S S^T R^T (3DGS factorisation), tau = 2 ln(255 o).
// ---------------------------------------------------------------------------
void gaussian_constants(const float* q4, const float* s3, float o, float* cov6, float* tau) {
    double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    double n = std::sqrt(((w * w + x * x) + y * y) + z * z);
    w = w / n; x = x / n; y = y / n; z = z / n;
    double R[3][3] = {
        {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)},
        {2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)},
        {2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)}};
    double ss[3] = {(double)s3[0] * (double)s3[0], (double)s3[1] * (double)s3[1],
                    (double)s3[2] * (double)s3[2]};
    const int A[6] = {0, 0, 0, 1, 1, 2}, B[6] = {0, 1, 2, 1, 2, 2};
    for (int e = 0; e < 6; ++e) {
        int a = A[e], b = B[e];
        double v = ((R[a][0] * ss[0]) * R[b][0] + (R[a][1] * ss[1]) * R[b][1]) +
                   (R[a][2] * ss[2]) * R[b][2];
        cov6[e] = (float)v;
    }
    *tau = (float)(2.0 * std::log(255.0 * (double)o));
}

// ---------------------------------------------------------------------------
// Cameras.  World->camera rotation R (row-major), translation t, pinhole
// intrinsics (OpenCV axes).  Per-camera host constants in fp64 -> fp32 (O6).
// ---------------------------------------------------------------------------
struct Cam {
    float R[9], t[3], fx, fy, cx, cy;
};
struct CamConst {
    float limxp, limxn, limyp, limyn;  // O6 frustum clamp limits
    float C[3];                        // camera centre -R^T t (O11)
};
CamConst cam_const(const Cam& c, int W, int H) {
    CamConst k;
    double tanfx = 0.5 * (double)W / (double)c.fx;
    double tanfy = 0.5 * (double)H / (double)c.fy;
    k.limxp = (float)(((double)W - (double)c.cx) / (double)c.fx + 0.3 * tanfx);
    k.limxn = (float)((double)c.cx / (double)c.fx + 0.3 * tanfx);
    k.limyp = (float)(((double)H - (double)c.cy) / (double)c.fy + 0.3 * tanfy);
    k.limyn = (float)((double)c.cy / (double)c.fy + 0.3 * tanfy);
    for (int a = 0; a < 3; ++a) {
        double v = 0.0;
        for (int r = 0; r < 3; ++r) v += (double)c.R[r * 3 + a] * (double)c.t[r];
        k.C[a] = (float)(-v);
    }
    return k;
}

// O5 — camera-space point and per-view mean, Eq.5.
struct P3 { float x, y, z; };
P3 cam_point(const Cam& c, const float* mu) {
    P3 p;
    p.x = ((c.R[0] * mu[0] + c.R[1] * mu[1]) + c.R[2] * mu[2]) + c.t[0];
    p.y = ((c.R[3] * mu[0] + c.R[4] * mu[1]) + c.R[5] * mu[2]) + c.t[1];
    p.z = ((c.R[6] * mu[0] + c.R[7] * mu[1]) + c.R[8] * mu[2]) + c.t[2];
    return p;
}
void mean2d(const Cam& c, const P3& p, float* mx, float* my) {
    *mx = (c.fx * (p.x / p.z)) + c.cx;
    *my = (c.fy * (p.y / p.z)) + c.cy;
}

// O6 — EWA 2D covariance at a camera (Pi_cov of Eq.6; gsplat classic).
// Returns false when det <= 0 (degenerate).
bool cov2d(const Cam& c, const CamConst& k, const P3& p, const float* S6, float* a_, float* b_,
           float* c_, float* det_) {
    float txz = p.x / p.z, tyz = p.y / p.z;
    float tx = p.z * mnf(k.limxp, mxf(-k.limxn, txz));
    float ty = p.z * mnf(k.limyp, mxf(-k.limyn, tyz));
    float zz = p.z * p.z;
    float J00 = c.fx / p.z, J02 = -((c.fx * tx) / zz);
    float J11 = c.fy / p.z, J12 = -((c.fy * ty) / zz);
    const float* R = c.R;
    float T[2][3];
    for (int col = 0; col < 3; ++col) {
        T[0][col] = J00 * R[0 * 3 + col] + J02 * R[2 * 3 + col];
        T[1][col] = J11 * R[1 * 3 + col] + J12 * R[2 * 3 + col];
    }
    float S[3][3] = {{S6[0], S6[1], S6[2]}, {S6[1], S6[3], S6[4]}, {S6[2], S6[4], S6[5]}};
    float U[2][3];
    for (int r = 0; r < 2; ++r)
        for (int col = 0; col < 3; ++col)
            U[r][col] = (T[r][0] * S[0][col] + T[r][1] * S[1][col]) + T[r][2] * S[2][col];
    float a = (U[0][0] * T[0][0] + U[0][1] * T[0][1]) + U[0][2] * T[0][2];
    float b = (U[0][0] * T[1][0] + U[0][1] * T[1][1]) + U[0][2] * T[1][2];
    float cc = (U[1][0] * T[1][0] + U[1][1] * T[1][1]) + U[1][2] * T[1][2];
    a = a + 0.3f;
    cc = cc + 0.3f;
    float det = a * cc - b * b;
    *a_ = a; *b_ = b; *c_ = cc; *det_ = det;
    return det > 0.0f;
}

// O7 — AccuTile reading: tiles whose pixel-centre rectangle
// meets the ellipse {m + d : d^T Sigma^-1 d <= tau}.  Row range of one view.
struct RowRange { int ty0, ty1; float ex, ey; };
// `pad` (test knob, default 0) grows every tile rectangle by pad pixels on each
// side: the superfluous-keys check of S:392 / P:379-382.  With pad = 0 every
// expression below is bit-identical to the unpadded reading (x - 0 = x).
RowRange row_range(float mx, float my, float a, float c, float tau, int TY, float pad = 0.0f) {
    RowRange r;
    r.ex = std::sqrt(tau * a);
    r.ey = std::sqrt(tau * c);
    r.ty0 = clamp_to_int(std::ceil((((my - r.ey) - 15.5f) - pad) / 16.0f), 0.0f, (float)TY);
    r.ty1 = clamp_to_int(std::floor((((my + r.ey) - 0.5f) + pad) / 16.0f), -1.0f, (float)(TY - 1));
    return r;
}
// Tile columns [tx0, tx1] hit in row ty (empty if tx0 > tx1).  Returns false
// if the row band misses the ellipse.
bool row_cols(float mx, float my, float a, float b, float c, float det, float tau,
              const RowRange& rr, int ty, int TX, int* tx0, int* tx1, float pad = 0.0f) {
    float ex = rr.ex, ey = rr.ey;
    float dlo = mxf(((16.0f * (float)ty + 0.5f) - pad) - my, -ey);
    float dhi = mnf(((16.0f * (float)ty + 15.5f) + pad) - my, ey);
    if (dlo > dhi) return false;
    float dyR = (b * ex) / a;
    float dyL = -dyR;
    float tc = tau * c;
    float ic = 1.0f / c;  // reading O7: one rounded reciprocal, then products
    auto h = [&](float dy) { return std::sqrt(mxf(0.0f, det * (tc - dy * dy))); };
    auto xr = [&](float dy) { return ((b * dy) + h(dy)) * ic; };
    auto xl = [&](float dy) { return ((b * dy) - h(dy)) * ic; };
    float right = mx + ((dlo <= dyR && dyR <= dhi) ? ex : mxf(xr(dlo), xr(dhi)));
    float left = mx + ((dlo <= dyL && dyL <= dhi) ? -ex : mnf(xl(dlo), xl(dhi)));
    *tx0 = clamp_to_int(std::ceil(((left - 15.5f) - pad) / 16.0f), 0.0f, (float)TX);
    *tx1 = clamp_to_int(std::floor(((right - 0.5f) + pad) / 16.0f), -1.0f, (float)(TX - 1));
    return true;
}

// O11 — 3DGS real SH colour (Pi_SH of Eq.6; constants S:77,S:91).
// sh: (deg+1)^2 coefficients x 3 channels, coefficient-major channel-minor.
const double SH_C0 = 0.28209479177387814;
const double SH_C1 = 0.4886025119029199;
const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                         -1.0925484305920792, 0.5462742152960396};
const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};
void sh_basis(int deg, double x, double y, double z, double* B) {
    B[0] = SH_C0;
    if (deg < 1) return;
    B[1] = -SH_C1 * y;
    B[2] = SH_C1 * z;
    B[3] = -SH_C1 * x;
    if (deg < 2) return;
    double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    B[4] = SH_C2[0] * xy;
    B[5] = SH_C2[1] * yz;
    B[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    B[7] = SH_C2[3] * xz;
    B[8] = SH_C2[4] * (xx - yy);
    if (deg < 3) return;
    B[9] = SH_C3[0] * y * (3.0 * xx - yy);
    B[10] = SH_C3[1] * xy * z;
    B[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
    B[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    B[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
    B[14] = SH_C3[5] * z * (xx - yy);
    B[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}
// Unclamped SH value + 0.5 (clamp applied by the caller, O11 / Z10).
void eval_sh_raw(int deg, const float* sh, const double* dir, double* rgb) {
    double B[16];
    sh_basis(deg, dir[0], dir[1], dir[2], B);
    int nc = (deg + 1) * (deg + 1);
    for (int ch = 0; ch < 3; ++ch) {
        double v = 0.0;
        for (int m = 0; m < nc; ++m) v += B[m] * (double)sh[m * 3 + ch];
        rgb[ch] = v + 0.5;
    }
}

// O12 — front-to-back compositing of one subpixel, Eqs.9–10.
struct Splat { float mx, my, A, B, C, o, col; };
float blend(const Splat* L, int n, float px, float py, float bg, int* n_eval) {
    float T = 1.0f, Cacc = 0.0f;
    int ev = 0;
    for (int e = 0; e < n; ++e) {
        const Splat& g = L[e];
        ++ev;
        float dx = g.mx - px, dy = g.my - py;
        float power = -0.5f * (g.A * dx * dx + g.C * dy * dy) - g.B * dx * dy;
        if (power > 0.0f) continue;
        float alpha = mnf(0.99f, g.o * std::exp(power));
        if (alpha < 1.0f / 255.0f) continue;
        float Tn = T * (1.0f - alpha);
        if (Tn < 1e-4f) break;  // saturation: this splat is not blended
        Cacc = Cacc + g.col * alpha * T;
        T = Tn;
    }
    if (n_eval) *n_eval = ev;
    return Cacc + bg * T;
}

}  // namespace

// ===========================================================================
// Oracle context: one scene + display + rig; render() runs O3..O12.
// ===========================================================================
struct cro_ctx {
    // scene (D1)
    int64_t M = 0;
    int deg = 0;
    std::vector<float> means, quats, scales, opac, sh, cov6, tau;
    // display (D2, D9)
    int W = 0, H = 0, N = 0, TX = 0, TY = 0;
    double Lx = 0, tanA = 0, Koff = 0;
    std::vector<uint8_t> V;
    // rig (D3)
    std::vector<Cam> cams;
    std::vector<CamConst> cconst;
    float znear = 0.01f;
    // per-frame state
    int s = 1, K = 0, bitK = 1;
    std::vector<int> rep;
    int row0 = 0, row1 = 0;
    float bg[3] = {0, 0, 0};
    // per (k, i) records, index k*M + i (D5)
    std::vector<uint8_t> state;  // 0 visible, 1 culled opacity, 2 near, 3 degenerate
    std::vector<float> depth, ca, cb, cc, cdet, conA, conB, conC, col;  // col: 3 per record
    std::vector<uint32_t> count;
    // pairs (D6/D7): key, payload i
    std::vector<uint64_t> keys;
    std::vector<uint32_t> pay;
    std::vector<uint32_t> S, E;  // (D8) [TX*TY*K]
    std::vector<float> img;      // band image [rows*16 clipped][W][3]
    int64_t n_evals = 0;
    int nthreads = 0;
    float tile_pad = 0.0f;  // test knob: grow tile rectangles by this many pixels
};

extern "C" {

// ---- unit entry points (pinned individually by tests) ---------------------
int cro_view_index(int x, int y, int u, int N, double Lx, double tan_alpha, double Koff) {
    return view_index(x, y, u, N, Lx, tan_alpha, Koff);
}

void cro_gaussian_constants(int64_t M, const float* quats, const float* scales, const float* opac,
                            float* cov6, float* tau) {
    for (int64_t i = 0; i < M; ++i)
        gaussian_constants(quats + 4 * i, scales + 3 * i, opac[i], cov6 + 6 * i, tau + i);
}

// cam: 16 floats (R[9], t[3], fx, fy, cx, cy)
int cro_project_mean(const float* cam, const float* mu, float znear, float* out2, float* depth) {
    Cam c;
    std::memcpy(&c, cam, sizeof(Cam));
    P3 p = cam_point(c, mu);
    *depth = p.z;
    mean2d(c, p, &out2[0], &out2[1]);
    return p.z >= znear ? 1 : 0;
}

// out4 = a, b, c, det (after +0.3 dilation); returns 1 if det > 0
int cro_cov2d(const float* cam, int W, int H, const float* mu, const float* cov6, float* out4) {
    Cam c;
    std::memcpy(&c, cam, sizeof(Cam));
    CamConst k = cam_const(c, W, H);
    P3 p = cam_point(c, mu);
    return cov2d(c, k, p, cov6, &out4[0], &out4[1], &out4[2], &out4[3]) ? 1 : 0;
}

// Tiles of one view (O7) into tiles_out (row-major ids, ascending); returns
// the count (or -needed if cap is too small).
int64_t cro_tileset(float mx, float my, float a, float b, float c, float det, float tau, int TX,
                    int TY, int32_t* tiles_out, int64_t cap) {
    RowRange rr = row_range(mx, my, a, c, tau, TY);
    int64_t n = 0;
    for (int ty = rr.ty0; ty <= rr.ty1; ++ty) {
        int tx0, tx1;
        if (!row_cols(mx, my, a, b, c, det, tau, rr, ty, TX, &tx0, &tx1)) continue;
        for (int tx = tx0; tx <= tx1; ++tx) {
            if (n < cap) tiles_out[n] = ty * TX + tx;
            ++n;
        }
    }
    return n <= cap ? n : -n;
}

void cro_sh_basis(int deg, const double* dir, double* out16) {
    for (int m = 0; m < 16; ++m) out16[m] = 0.0;
    sh_basis(deg, dir[0], dir[1], dir[2], out16);
}
void cro_eval_sh(int deg, const float* sh, const double* dir, double* rgb) {
    eval_sh_raw(deg, sh, dir, rgb);
}

// splats: n x 7 floats (mx, my, A, B, C, o, colour)
float cro_blend(const float* splats, int n, float px, float py, float bg) {
    std::vector<Splat> L(n);
    for (int e = 0; e < n; ++e) {
        const float* s = splats + 7 * e;
        L[e] = Splat{s[0], s[1], s[2], s[3], s[4], s[5], s[6]};
    }
    return blend(L.data(), n, px, py, bg, nullptr);
}

// ---- context --------------------------------------------------------------
cro_ctx* cro_create(int nthreads) {
    cro_ctx* c = new cro_ctx();
    c->nthreads = hw_threads(nthreads);
    return c;
}
void cro_destroy(cro_ctx* c) { delete c; }
int cro_threads(const cro_ctx* c) { return c->nthreads; }
// Superfluous-keys check: grow every tile's pixel-centre
// rectangle by pad pixels in the tile test (O7).  0 = the reading itself.
void cro_set_tile_pad(cro_ctx* c, float pad) { c->tile_pad = pad; }

// D1: Gaussians, SoA fp32, quats (w,x,y,z), linear scales, post-sigmoid
// opacity, sh[M][(deg+1)^2][3].  O4 constants computed here.
int cro_set_scene(cro_ctx* c, int64_t M, int deg, const float* means, const float* quats,
                  const float* scales, const float* opac, const float* sh) {
    if (M < 0 || deg < 0 || deg > 3) return 1;
    int nc = (deg + 1) * (deg + 1);
    c->M = M;
    c->deg = deg;
    c->means.assign(means, means + 3 * M);
    c->quats.assign(quats, quats + 4 * M);
    c->scales.assign(scales, scales + 3 * M);
    c->opac.assign(opac, opac + M);
    c->sh.assign(sh, sh + (int64_t)nc * 3 * M);
    c->cov6.resize(6 * M);
    c->tau.resize(M);
    parallel_for(M, c->nthreads, [&](int64_t i) {
        gaussian_constants(&c->quats[4 * i], &c->scales[3 * i], c->opac[i], &c->cov6[6 * i],
                           &c->tau[i]);
    });
    return 0;
}
void cro_get_constants(const cro_ctx* c, float* cov6, float* tau) {
    std::memcpy(cov6, c->cov6.data(), sizeof(float) * 6 * c->M);
    std::memcpy(tau, c->tau.data(), sizeof(float) * c->M);
}

// D2: viewpoint index matrix V (O1).  tan_alpha given directly.
int cro_set_display_tan(cro_ctx* c, int W, int H, int N, double Lx, double tan_alpha,
                        double Koff) {
    if (W < 1 || H < 1 || N < 1 || N > 255 || !(Lx > 0)) return 2;
    c->W = W; c->H = H; c->N = N; c->Lx = Lx; c->tanA = tan_alpha; c->Koff = Koff;
    c->TX = (W + 15) / 16;
    c->TY = (H + 15) / 16;
    c->V.resize((size_t)W * H * 3);
    parallel_for(H, c->nthreads, [&](int64_t y) {
        for (int x = 0; x < W; ++x)
            for (int u = 0; u < 3; ++u)
                c->V[((size_t)y * W + x) * 3 + u] =
                    (uint8_t)view_index(x, (int)y, u, N, Lx, tan_alpha, Koff);
    });
    return 0;
}
// slant alpha in radians; tan evaluated once on the host in fp64 (Z2)
int cro_set_display(cro_ctx* c, int W, int H, int N, double Lx, double slant, double Koff) {
    return cro_set_display_tan(c, W, H, N, Lx, std::tan(slant), Koff);
}
void cro_get_view_map(const cro_ctx* c, uint8_t* dst) {
    std::memcpy(dst, c->V.data(), c->V.size());
}

// O2 — View-coherent Remapping table Psi (Eq.8): per tile the local
// subpixel indices l = (ly*16+lx)*3+u of in-panel subpixels in increasing l,
// stably sorted by V.  Layout [TY*TX][768]; unused slots of clipped tiles 0xFFFF.
void cro_get_remap(const cro_ctx* c, int remap, uint16_t* dst) {
    const int TX = c->TX, TY = c->TY, W = c->W, H = c->H;
    for (int t = 0; t < TX * TY; ++t) {
        int tx = t % TX, ty = t / TX;
        std::vector<std::pair<int, int>> items;  // (V, l)
        for (int ly = 0; ly < 16; ++ly)
            for (int lx = 0; lx < 16; ++lx) {
                int x = tx * 16 + lx, y = ty * 16 + ly;
                if (x >= W || y >= H) continue;
                for (int u = 0; u < 3; ++u)
                    items.push_back({c->V[((size_t)y * W + x) * 3 + u], (ly * 16 + lx) * 3 + u});
            }
        if (remap)
            std::stable_sort(items.begin(), items.end(),
                             [](const std::pair<int, int>& p, const std::pair<int, int>& q) {
                                 return p.first < q.first;
                             });
        uint16_t* o = dst + (size_t)t * 768;
        for (int r = 0; r < 768; ++r) o[r] = 0xFFFF;
        for (size_t r = 0; r < items.size(); ++r) o[r] = (uint16_t)items[r].second;
    }
}

// D3: rig of N cameras (16 floats each) + znear.
int cro_set_rig(cro_ctx* c, int N, const float* cams16, float znear) {
    if (N != c->N) return 3;  // CONFIG_MISMATCH
    c->cams.resize(N);
    c->cconst.resize(N);
    for (int j = 0; j < N; ++j) {
        std::memcpy(&c->cams[j], cams16 + 16 * j, sizeof(Cam));
        c->cconst[j] = cam_const(c->cams[j], c->W, c->H);
    }
    c->znear = znear;
    return 0;
}

// O3 — contiguous clusters, median-index representative, padding by
// duplicating v_{N-1} (P:336, P:695 Supp. A.1); Bit_K.
int cro_clusters(int N, int s, int* K, int* bitK, int* rep_out) {
    if (N < 1 || s < 1) return 1;
    int k = (N + s - 1) / s;
    int b = 0;
    while ((1 << b) < k) ++b;
    if (b < 1) b = 1;
    *K = k;
    *bitK = b;
    if (rep_out)
        for (int q = 0; q < k; ++q) rep_out[q] = std::min(q * s + s / 2, N - 1);
    return 0;
}

// Full pipeline O3..O12 for tile rows [row0, row1) (0,0 = all).  If
// tile_filter is non-null only pairs in the listed tiles are kept and only
// those tiles are composited (sampled parity at full size).
int cro_render(cro_ctx* c, int s, int row0, int row1, const float* bg,
               const int32_t* tile_filter, int64_t n_filter, int do_composite) {
    if (c->N < 1 || (int)c->cams.size() != c->N) return 6;
    if (s < 1 || s > 32) return 2;
    const int64_t M = c->M;
    const int N = c->N, TX = c->TX, TY = c->TY, W = c->W, H = c->H;
    if (row0 == 0 && row1 == 0) row1 = TY;
    if (row0 < 0 || row1 > TY || row0 >= row1) return 1;
    c->s = s;
    c->row0 = row0;
    c->row1 = row1;
    for (int u = 0; u < 3; ++u) c->bg[u] = bg ? bg[u] : 0.0f;
    cro_clusters(N, s, &c->K, &c->bitK, nullptr);
    const int K = c->K;
    if ((int64_t)TX * TY >= ((int64_t)1 << (32 - c->bitK))) return 4;  // TILE_ID_OVERFLOW
    c->rep.resize(K);
    cro_clusters(N, s, &c->K, &c->bitK, c->rep.data());

    std::vector<uint8_t> in_filter;
    if (tile_filter) {
        in_filter.assign((size_t)TX * TY, 0);
        for (int64_t q = 0; q < n_filter; ++q) in_filter[tile_filter[q]] = 1;
    }

    const int64_t R = (int64_t)K * M;
    c->state.assign(R, 0);
    c->depth.assign(R, 0); c->ca.assign(R, 0); c->cb.assign(R, 0); c->cc.assign(R, 0);
    c->cdet.assign(R, 0); c->conA.assign(R, 0); c->conB.assign(R, 0); c->conC.assign(R, 0);
    c->col.assign(3 * R, 0);
    c->count.assign(R, 0);
    const int nc = (c->deg + 1) * (c->deg + 1);

    // Stage 1 (Alg.1): per (i,k) shared attributes at v'_k (Eq.6).
    // Stage 2 (Alg.2 GenerateKeys P:791-808): tile union over the cluster.
    const int nchunks = 256;
    std::vector<std::vector<std::pair<uint64_t, uint32_t>>> chunk_pairs(nchunks);
    const int64_t per = (M + nchunks - 1) / nchunks;
    parallel_for(nchunks, c->nthreads, [&](int64_t ch) {
        std::vector<std::pair<uint64_t, uint32_t>>& out = chunk_pairs[ch];
        std::vector<float> vmx(s), vmy(s);
        std::vector<RowRange> vrr(s);
        std::vector<int> vok(s);
        std::vector<std::pair<int, int>> iv;
        for (int64_t i = ch * per; i < std::min(M, (ch + 1) * per); ++i) {
            const float* mu = &c->means[3 * i];
            for (int k = 0; k < K; ++k) {
                const int64_t r = (int64_t)k * M + i;
                if (!(c->tau[i] > 0.0f)) { c->state[r] = 1; continue; }
                const Cam& rc = c->cams[c->rep[k]];
                const CamConst& rk = c->cconst[c->rep[k]];
                P3 p = cam_point(rc, mu);
                if (p.z < c->znear) { c->state[r] = 2; continue; }
                float a, b, cc, det;
                if (!cov2d(rc, rk, p, &c->cov6[6 * i], &a, &b, &cc, &det)) {
                    c->state[r] = 3;
                    continue;
                }
                c->depth[r] = p.z;
                c->ca[r] = a; c->cb[r] = b; c->cc[r] = cc; c->cdet[r] = det;
                c->conA[r] = cc / det; c->conB[r] = -b / det; c->conC[r] = a / det;
                // SH colour at the representative camera centre (O11)
                double dir[3], nrm = 0.0;
                for (int q = 0; q < 3; ++q) {
                    dir[q] = (double)mu[q] - (double)rk.C[q];
                    nrm += dir[q] * dir[q];
                }
                nrm = std::sqrt(nrm);
                for (int q = 0; q < 3; ++q) dir[q] /= nrm;
                double rgb[3];
                eval_sh_raw(c->deg, &c->sh[(size_t)i * nc * 3], dir, rgb);
                for (int q = 0; q < 3; ++q) c->col[3 * r + q] = (float)std::max(rgb[q], 0.0);
                // O8: union over the cluster's real views of the per-view tile sets
                const int j0 = k * s, j1 = std::min(k * s + s, N);
                int rmin = TY, rmax = -1;
                for (int j = j0; j < j1; ++j) {
                    int l = j - j0;
                    P3 pj = cam_point(c->cams[j], mu);
                    vok[l] = pj.z >= c->znear;
                    if (!vok[l]) continue;
                    mean2d(c->cams[j], pj, &vmx[l], &vmy[l]);
                    vrr[l] = row_range(vmx[l], vmy[l], a, cc, c->tau[i], TY, c->tile_pad);
                    rmin = std::min(rmin, vrr[l].ty0);
                    rmax = std::max(rmax, vrr[l].ty1);
                }
                rmin = std::max(rmin, row0);
                rmax = std::min(rmax, row1 - 1);
                uint32_t cnt = 0;
                for (int ty = rmin; ty <= rmax; ++ty) {
                    iv.clear();
                    for (int j = j0; j < j1; ++j) {
                        int l = j - j0;
                        if (!vok[l] || ty < vrr[l].ty0 || ty > vrr[l].ty1) continue;
                        int tx0, tx1;
                        if (!row_cols(vmx[l], vmy[l], a, b, cc, det, c->tau[i], vrr[l], ty, TX,
                                      &tx0, &tx1, c->tile_pad))
                            continue;
                        if (tx0 <= tx1) iv.push_back({tx0, tx1});
                    }
                    std::sort(iv.begin(), iv.end());
                    int cur = -1;  // last tile emitted in this row
                    for (auto& q : iv) {
                        for (int tx = std::max(q.first, cur + 1); tx <= q.second; ++tx) {
                            ++cnt;
                            uint32_t t = (uint32_t)(ty * TX + tx);
                            if (tile_filter && !in_filter[t]) continue;
                            // Eq.11 key: t << (32+Bit_K) | k << 32 | bits(d)
                            uint32_t dbits;
                            std::memcpy(&dbits, &p.z, 4);
                            uint64_t key = ((uint64_t)t << (32 + c->bitK)) |
                                           ((uint64_t)k << 32) | (uint64_t)dbits;
                            out.push_back({key, (uint32_t)i});
                        }
                        cur = std::max(cur, q.second);
                    }
                }
                c->count[r] = cnt;
            }
        }
    });
    // Stage 3 (Alg.1): sort by (key, i) — a total order (O9/Z13).
    size_t P = 0;
    for (auto& v : chunk_pairs) P += v.size();
    std::vector<std::pair<uint64_t, uint32_t>> all;
    all.reserve(P);
    for (auto& v : chunk_pairs) {
        all.insert(all.end(), v.begin(), v.end());
        std::vector<std::pair<uint64_t, uint32_t>>().swap(v);
    }
    std::sort(all.begin(), all.end());
    c->keys.resize(P);
    c->pay.resize(P);
    for (size_t e = 0; e < P; ++e) { c->keys[e] = all[e].first; c->pay[e] = all[e].second; }
    std::vector<std::pair<uint64_t, uint32_t>>().swap(all);
    // O10 ranges [S,E) per (t,k); absent -> S=E=0.
    c->S.assign((size_t)TX * TY * K, 0);
    c->E.assign((size_t)TX * TY * K, 0);
    const uint64_t kmask = ((uint64_t)1 << c->bitK) - 1;
    for (size_t e = 0; e < P; ++e) {
        uint64_t t = c->keys[e] >> (32 + c->bitK);
        uint64_t k = (c->keys[e] >> 32) & kmask;
        size_t slot = (size_t)t * K + k;
        if (e == 0 || (c->keys[e - 1] >> 32) != (c->keys[e] >> 32)) c->S[slot] = (uint32_t)e;
        c->E[slot] = (uint32_t)(e + 1);
    }
    if (!do_composite) return 0;

    // Stage 4 (Alg.2 Alpha-Blend P:810-824): per subpixel, raster order (Psi
    // only permutes independent writes, O12).
    const int y0 = row0 * 16, y1 = std::min(H, row1 * 16);
    c->img.assign((size_t)(y1 - y0) * W * 3, 0.0f);
    std::atomic<int64_t> evals(0);
    parallel_for(y1 - y0, c->nthreads, [&](int64_t yy) {
        int y = y0 + (int)yy;
        int ty = y / 16;
        std::vector<Splat> L;
        int64_t ev_local = 0;
        for (int x = 0; x < W; ++x) {
            int tx = x / 16;
            uint32_t t = (uint32_t)(ty * TX + tx);
            if (tile_filter && !in_filter[t]) continue;
            for (int u = 0; u < 3; ++u) {
                int j = c->V[((size_t)y * W + x) * 3 + u];
                int k = j / s;
                size_t slot = (size_t)t * K + k;
                L.clear();
                for (uint32_t e = c->S[slot]; e < c->E[slot]; ++e) {
                    uint32_t i = c->pay[e];
                    int64_t r = (int64_t)k * M + i;
                    P3 pj = cam_point(c->cams[j], &c->means[3 * i]);
                    if (pj.z < c->znear) continue;  // Z12: view j cannot see i
                    Splat g;
                    mean2d(c->cams[j], pj, &g.mx, &g.my);
                    g.A = c->conA[r]; g.B = c->conB[r]; g.C = c->conC[r];
                    g.o = c->opac[i];
                    g.col = c->col[3 * r + u];
                    L.push_back(g);
                }
                int ev = 0;
                float v = blend(L.data(), (int)L.size(), (float)x + 0.5f, (float)y + 0.5f,
                                c->bg[u], &ev);
                ev_local += ev;
                c->img[((size_t)yy * W + x) * 3 + u] = v;
            }
        }
        evals += ev_local;
    });
    c->n_evals = evals.load();
    return 0;
}

int cro_num_clusters(const cro_ctx* c) { return c->K; }
int cro_bit_k(const cro_ctx* c) { return c->bitK; }
int64_t cro_num_pairs(const cro_ctx* c) { return (int64_t)c->keys.size(); }
int64_t cro_num_evals(const cro_ctx* c) { return c->n_evals; }
void cro_get_pairs(const cro_ctx* c, uint64_t* keys, uint32_t* pay) {
    std::memcpy(keys, c->keys.data(), 8 * c->keys.size());
    std::memcpy(pay, c->pay.data(), 4 * c->pay.size());
}
void cro_get_ranges(const cro_ctx* c, uint32_t* S, uint32_t* E) {
    std::memcpy(S, c->S.data(), 4 * c->S.size());
    std::memcpy(E, c->E.data(), 4 * c->E.size());
}
// image of the last render's band: [(y1-y0)][W][3] float
void cro_get_image(const cro_ctx* c, float* dst) {
    std::memcpy(dst, c->img.data(), 4 * c->img.size());
}
// per-(k,i) records: state, depth, a, b, c, det, conic A,B,C, colour[3], count
void cro_get_records(const cro_ctx* c, uint8_t* state, float* depth, float* cov2d4,
                     float* conic3, float* col3, uint32_t* count) {
    const int64_t R = (int64_t)c->K * c->M;
    for (int64_t r = 0; r < R; ++r) {
        if (state) state[r] = c->state[r];
        if (depth) depth[r] = c->depth[r];
        if (cov2d4) {
            cov2d4[4 * r] = c->ca[r]; cov2d4[4 * r + 1] = c->cb[r];
            cov2d4[4 * r + 2] = c->cc[r]; cov2d4[4 * r + 3] = c->cdet[r];
        }
        if (conic3) {
            conic3[3 * r] = c->conA[r]; conic3[3 * r + 1] = c->conB[r];
            conic3[3 * r + 2] = c->conC[r];
        }
        if (col3)
            for (int q = 0; q < 3; ++q) col3[3 * r + q] = c->col[3 * r + q];
        if (count) count[r] = c->count[r];
    }
}

// Per-view frames of the last cro_render(s): every view j rendered full frame
// (all pixels, all three channels) from its cluster's (t, k(j)) lists, per-view
// means mu2D_{i,j} and the cluster's shared attributes — O12 applied to every
// (j, x, y, u) instead of only u's view V[y][x][u] (the per-view images the
// paper evaluates; Eq.4 then picks one view per subpixel).
// dst: [N][H][W][3] float.  Requires a full-frame (row0 = 0, row1 = TY) render.
int cro_render_views(cro_ctx* c, float* dst) {
    const int64_t M = c->M;
    const int N = c->N, W = c->W, H = c->H, s = c->s, TX = c->TX, K = c->K;
    if (c->row0 != 0 || c->row1 != c->TY) return 1;
    parallel_for((int64_t)N * H, c->nthreads, [&](int64_t jy) {
        const int j = (int)(jy / H), y = (int)(jy % H);
        const int k = j / s;
        std::vector<Splat> L;
        for (int x = 0; x < W; ++x) {
            const size_t slot = (size_t)((y / 16) * TX + x / 16) * K + k;
            for (int u = 0; u < 3; ++u) {
                L.clear();
                for (uint32_t e = c->S[slot]; e < c->E[slot]; ++e) {
                    uint32_t i = c->pay[e];
                    int64_t r = (int64_t)k * M + i;
                    P3 pj = cam_point(c->cams[j], &c->means[3 * i]);
                    if (pj.z < c->znear) continue;  // Z12
                    Splat g;
                    mean2d(c->cams[j], pj, &g.mx, &g.my);
                    g.A = c->conA[r]; g.B = c->conB[r]; g.C = c->conC[r];
                    g.o = c->opac[i];
                    g.col = c->col[3 * r + u];
                    L.push_back(g);
                }
                dst[(((size_t)j * H + y) * W + x) * 3 + u] =
                    blend(L.data(), (int)L.size(), (float)x + 0.5f, (float)y + 0.5f, c->bg[u],
                          nullptr);
            }
        }
    });
    return 0;
}

// Brute force (north_star check): render every view full frame with no
// tiles — per pixel all Gaussians with (i, k(j)) not culled and visible from
// v_j, ordered by (d_{i,k(j)}, i) — then interlace by V.
// Requires a prior cro_render(s, ...) for the per-(i,k) records.
int cro_render_bruteforce(cro_ctx* c, float* dst) {
    const int64_t M = c->M;
    const int N = c->N, W = c->W, H = c->H, s = c->s;
    std::vector<float> frames((size_t)N * H * W * 3);
    parallel_for(N, c->nthreads, [&](int64_t j) {
        int k = (int)j / s;
        std::vector<std::pair<std::pair<float, uint32_t>, uint32_t>> order;
        for (int64_t i = 0; i < M; ++i) {
            int64_t r = (int64_t)k * M + i;
            if (c->state[r] != 0) continue;
            P3 pj = cam_point(c->cams[j], &c->means[3 * i]);
            if (pj.z < c->znear) continue;
            order.push_back({{c->depth[r], (uint32_t)i}, (uint32_t)i});
        }
        std::sort(order.begin(), order.end());
        std::vector<Splat> L[3];
        for (int u = 0; u < 3; ++u) L[u].reserve(order.size());
        for (auto& o : order) {
            uint32_t i = o.second;
            int64_t r = (int64_t)k * M + i;
            Splat g;
            P3 pj = cam_point(c->cams[j], &c->means[3 * i]);
            mean2d(c->cams[j], pj, &g.mx, &g.my);
            g.A = c->conA[r]; g.B = c->conB[r]; g.C = c->conC[r];
            g.o = c->opac[i];
            for (int u = 0; u < 3; ++u) { g.col = c->col[3 * r + u]; L[u].push_back(g); }
        }
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                for (int u = 0; u < 3; ++u)
                    frames[(((size_t)j * H + y) * W + x) * 3 + u] =
                        blend(L[u].data(), (int)L[u].size(), (float)x + 0.5f, (float)y + 0.5f,
                              c->bg[u], nullptr);
    });
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int u = 0; u < 3; ++u) {
                size_t o = ((size_t)y * W + x) * 3 + u;
                int j = c->V[o];
                dst[o] = frames[(((size_t)j * H + y) * W + x) * 3 + u];
            }
    return 0;
}

}  // extern "C"
