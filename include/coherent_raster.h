/*
 * coherent_raster.h — C ABI of libcoherent_raster.so, the B200 (sm_100a)
 * subpixel-level light-field 3DGS rasterizer of arXiv 2605.04509
 * ("CoherentRaster: Efficient 3D Gaussian Splatting for Light Field Displays").
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * O1..O12 and Z1..Z19 = the readings listed in DESIGN.md §3.
 *
 * Problem statement (§4): given 3D Gaussians G = {G_i} and a
 * display setup (target views V = {v_j}, j < N, and the viewpoint index
 * matrix V in Z^{W x H x 3}), synthesise the interlaced light-field image
 * I_LF in R^{W x H x 3}.  Every pixel-space stage runs in this library's
 * CUDA kernels; the host code only validates, sizes buffers and launches.
 *
 * Conventions
 *  - Every call returns a cr_status; no C++ exception crosses the ABI.
 *  - A context is bound to one CUDA device and one stream and is NOT
 *    thread-safe; use one context per device (one process per GPU).
 *  - Inputs are COPIED; the library never frees or retains caller memory.
 *  - Images are row-major, y = 0 at the top row, channel-minor
 *    ([rows][W][3]); tiles are 16x16 pixels, row-major ids t = ty*TX + tx
 *    (global ids, also for bands) (Z15).
 *  - All work is ordered on the context's stream.  cr_render_interlaced
 *    returns after the frame is complete when the output is on the host or
 *    stats are requested; otherwise the image is ready when the stream is.
 *  - On error the context keeps its previous state; cr_last_error() has
 *    a one-line diagnostic.
 */
#ifndef COHERENT_RASTER_H
#define COHERENT_RASTER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cr_ctx cr_ctx; /* opaque; owns all its device memory */

typedef enum {
  CR_OK = 0,
  CR_ERR_INVALID_ARG = 1,      /* NULL pointer, size mismatch, bad enum      */
  CR_ERR_INVALID_CONFIG = 2,   /* W,H,N >= 1, N <= 255, Lx > 0, tile 16,
                                  1 <= s <= 32                */
  CR_ERR_CONFIG_MISMATCH = 3,  /* rig views != display N            */
  CR_ERR_TILE_ID_OVERFLOW = 4, /* tiles >= 2^(32 - Bit_K)    */
  CR_ERR_NONFINITE = 5,        /* NaN/Inf in uploaded data           */
  CR_ERR_NOT_READY = 6,        /* render before upload/display/rig          */
  CR_ERR_OUT_OF_MEMORY = 7,    /* device allocation failed                   */
  CR_ERR_CUDA = 8,             /* any other CUDA runtime error               */
  CR_ERR_CAPACITY = 9          /* pair count exceeds 2^32 - 1               */
} cr_status;

/* Create a context on `cuda_device`.  `cuda_stream` is a cudaStream_t (may be
 * NULL = the legacy default stream); PyTorch callers pass
 * torch.cuda.current_stream().cuda_stream.  *out receives the context. */
cr_status cr_create(int cuda_device, void* cuda_stream, cr_ctx** out);
void cr_destroy(cr_ctx* ctx);
/* Re-bind the stream used by subsequent calls. */
cr_status cr_set_stream(cr_ctx* ctx, void* cuda_stream);
/* Wait until every frame this context has rendered is complete, including
 * the host copies of CR_FLAG_ASYNC_OUT renders (their host buffers may be
 * read after this returns). */
cr_status cr_synchronize(cr_ctx* ctx);
/* Context-owned diagnostic of the last failing call (valid until the next call). */
const char* cr_last_error(const cr_ctx* ctx);
const char* cr_status_string(cr_status s);
/* Library build tag, e.g. "coherent_raster sm_100a <git>". */
const char* cr_version(void);

/* ---------------------------------------------------------------------
 * Scene upload (D1): Gaussians G_i = (mu_i, Sigma_i, o_i, h_i).
 *   means[M*3]      world positions
 *   quats[M*4]      rotation (w,x,y,z); renormalised here
 *   scales[M*3]     per-axis standard deviations, linear, > 0
 *   opacities[M]    post-sigmoid, in [0,1]
 *   sh[M*(d+1)^2*3] SH coefficients, coefficient-major, channel-minor
 *                   (gsplat layout [M][(d+1)^2][3]), d = sh_degree in 0..3
 * Pointers are device pointers if ptrs_on_device != 0, else host pointers.
 * Data are copied.  Sigma = R S S^T R^T is built on the device in fp64 (O4);
 * tau_i = 2 ln(255 o_i), the alpha >= 1/255 threshold used by AccuTile (O7),
 * is evaluated on the host in fp64.  Returns CR_ERR_NONFINITE on NaN/Inf.
 * M = 0 is a valid (empty) scene.
 * ------------------------------------------------------------------- */
cr_status cr_upload_gaussians(cr_ctx* ctx, int64_t M, int sh_degree, const float* means,
                              const float* quats, const float* scales, const float* opacities,
                              const float* sh, int ptrs_on_device);

/* ---------------------------------------------------------------------
 * Display (§3.1).  Builds on the device, once per call:
 *   V   u8 [H][W][3]: j = floor(N * ((3x+u+3y tan(alpha) - K_offset) mod Lx) / Lx)
 *       (Eqs.1-3; fp64, floor-mod, O1/Z1/Z2)
 *   Psi u16 [TY*TX][768]: per tile, local subpixel index l = (ly*16+lx)*3+u
 *       stably sorted by V (View-coherent Remapping, Eq.8); unused
 *       slots of clipped edge tiles are 0xFFFF (O2).
 * ------------------------------------------------------------------- */
typedef struct {
  int32_t width, height; /* W, H panel pixels                            */
  int32_t num_views;     /* N, 1..255                                    */
  double lens_pitch;     /* L_x: grating line count in subpixel units    */
  double slant;          /* alpha: grating tilt angle, radians           */
  double center_offset;  /* K_offset: lens-to-panel offset, subpixels    */
  double view_cone;      /* total angular range of the N views, degrees; */
                         /* informational, used by cr_make_orbit_rig             */
  int32_t tile_size;     /* must be 16; 0 means 16                       */
} cr_display;
cr_status cr_set_display(cr_ctx* ctx, const cr_display* display);

/* ---------------------------------------------------------------------
 * Camera rig: the N target views v_j, world->camera rotation
 * R (row-major, OpenCV axes: x right, y down, z forward), translation t,
 * pinhole intrinsics in pixels.  znear culls means with camera z < znear
 * (default 0.01).  num_views must equal the display's N.
 * ------------------------------------------------------------------- */
typedef struct {
  float R[9];
  float t[3];
  float fx, fy, cx, cy;
} cr_camera;
cr_status cr_set_camera_rig(cr_ctx* ctx, int32_t num_views, const cr_camera* views, float znear);

/* Host helper: N inward-looking cameras on a horizontal arc of
 * display->view_cone degrees around look_at (orbit trajectories),
 * view 0 at -cone/2, fy = fx = H / (2 tan(fov_y/2)), principal point at the
 * image centre.  Writes display->num_views cameras to out_views. */
cr_status cr_make_orbit_rig(const cr_display* display, const float look_at[3], const float up[3],
                            float radius, float height, float yaw_deg, float pitch_deg,
                            float fov_y_deg, cr_camera* out_views);

/* ---------------------------------------------------------------------
 * Render one interlaced frame (Alg.1):
 *   Stage 1  per (Gaussian i, cluster k) attributes at the representative
 *            view v'_k: depth, EWA Sigma2D (+0.3), conic, SH colour (Eq.6,
 *            Cross-view Coherent Attribute Reuse), and the size
 *            of the cluster tile union (Alg.2 GenerateKeys)
 *   Stage 2  keys <t, k, depth> (Eq.7/Eq.11) for every tile of the union
 *   Stage 3  stable sort by (t, k, depth, i) + ranges [S,E)
 *   Stage 4  per subpixel, via Psi: front-to-back blend of list (t, k(j))
 *            with per-view means mu2D_{i,j} (Eqs.9-10)
 * Options:
 *   cluster_size   s = |V_k| (1..32; default 8); s = 1 is "w/o reuse"
 *   remap          1 = View-coherent Remapping (default), 0 = raster order
 *   kernel         0 = B200 staged composite (warp per cluster chunk of up to
 *                  32 lanes x two subpixels of one view, shared-memory
 *                  batches, per-view cull ballots, early exit) [requires
 *                  remap = 1];
 *                  1 = thread-per-subpixel composite (the paper's design,
 *                  Alg.2 Alpha-Blend), used for remap = 0 and for ablations
 *   background     colour added with the remaining transmittance (Z18)
 *   output_format  0 = RGB8 (floor(clamp(C,0,1)*255+0.5)), 1 = float32
 *   tile_row_begin/end  render only tile rows [begin, end) (row band for
 *                  multi-GPU sharding); 0,0 = full frame
 *   flags          CR_FLAG_COUNT_EVALS counts (subpixel, splat) evaluations;
 *                  CR_FLAG_FULLFRAME renders the traditional baseline instead
 *                  (SURVEY N1): every one of the N views at full
 *                  resolution with its own attributes (cluster_size 1), one
 *                  RGB pixel per thread, into an internal [N][rows][W][3]
 *                  buffer, then interlaced by V.  Equal, subpixel
 *                  by subpixel, to the s=1 subpixel path.
 *                  CR_FLAG_FULLFRAME with cluster_size s > 1 renders every view
 *                  full frame with the attributes of its cluster (the per-view
 *                  images of Cross-view Coherent Attribute Reuse the paper
 *                  evaluates); interlaced it equals the subpixel path.
 *                  CR_FLAG_VIEW_FRAMES (implies the full-frame render) returns
 *                  those per-view frames instead of interlacing them: out is
 *                  [N][rows][W][3], out_bytes >= N times the band size.
 *                  CR_FLAG_ASYNC_OUT (host `out` only, interlaced frame): the
 *                  frame is copied to `out` on the context's copy stream after
 *                  the composite (two device staging buffers, so the copy of
 *                  frame n overlaps the rendering of frame n+1) and the call
 *                  returns without waiting; `out` must stay valid and unread
 *                  until cr_synchronize (pinned memory makes the copy
 *                  asynchronous).  Ignored with stats (they synchronise).
 *   view_batch     full-frame render only: views per pass (the paper's
 *                  "3DGS (batch=B)" baseline, T2 P:520; 1 = plain
 *                  per-view 3DGS): the N views are rendered B at a time, each
 *                  pass running preprocess, binning, sort and the full-frame
 *                  composite for its views only, then the frames are
 *                  interlaced once.  Must be a multiple of cluster_size;
 *                  0 (or >= N) = all N views in one pass.  Ignored otherwise.
 * out: caller-owned, [rows][W][3] of the band (rows = clipped band height),
 * out_bytes must be >= rows*W*3*(1 or 4).  out_on_device selects a device
 * pointer (written on the stream) or a host pointer (copied back, the call
 * then synchronises).  stats may be NULL; when given the call synchronises
 * and fills it.
 * ------------------------------------------------------------------- */
#define CR_FLAG_COUNT_EVALS 1
#define CR_FLAG_FULLFRAME 2
#define CR_FLAG_VIEW_FRAMES 4
#define CR_FLAG_ASYNC_OUT 8
typedef struct {
  int32_t cluster_size;
  int32_t remap;
  int32_t kernel;
  float background[3];
  int32_t output_format;
  int32_t tile_row_begin, tile_row_end;
  int32_t flags;         /* bit 0: count blend evaluations into cr_stats.evals
                            (instrumented composite; slower, for rooflines)   */
  int32_t view_batch;    /* full-frame baseline: views per pass (0 = all)    */
} cr_render_opts;

typedef struct {
  int64_t pairs;             /* Gaussian-tile-cluster pairs P (T5/T6 "#Pairs")       */
  int64_t visible_ik;        /* (i,k) records with >= 1 tile in the band             */
  int64_t culled_near;       /* (i,k) with camera z < znear at v'_k                  */
  int64_t culled_degenerate; /* (i,k) with det(Sigma2D) <= 0                 */
  int64_t culled_opacity;    /* Gaussians with o <= 1/255 (tau <= 0), counted once  */
  int32_t num_clusters;      /* K                                                   */
  int32_t bit_k;             /* Bit_K                                               */
  int32_t launches;          /* kernels launched by this call                       */
  int32_t emit_fallback;     /* records whose tile union did not fit a 32-B slot     */
  float ms_preprocess, ms_bin, ms_sort, ms_composite, ms_total; /* CUDA-event times   */
  int64_t device_bytes;      /* device memory held by the context                   */
  int64_t evals;             /* blend evaluations (only with CR_FLAG_COUNT_EVALS)   */
} cr_stats;

cr_status cr_render_interlaced(cr_ctx* ctx, const cr_render_opts* opts, void* out,
                               size_t out_bytes, int out_on_device, cr_stats* stats);

/* ---------------------------------------------------------------------
 * Introspection for bit-exact parity tests (host destination pointers).
 * Call with dst = NULL to query the element count in *n; otherwise *n is
 * the capacity of dst in elements and is set to the count written.
 * ------------------------------------------------------------------- */
cr_status cr_get_view_map(cr_ctx* ctx, uint8_t* dst, size_t* n);   /* [H][W][3]            */
cr_status cr_get_remap(cr_ctx* ctx, uint16_t* dst, size_t* n);     /* [TY*TX][768]         */
/* last frame: 64-bit keys t<<(32+Bit_K) | k<<32 | bits(d_{i,k}) (Eq.11)
 * and payloads i, in sorted order. */
cr_status cr_get_sorted_pairs(cr_ctx* ctx, uint64_t* keys, uint32_t* payloads, size_t* n);
/* last frame: S_{t,k}, E_{t,k} over all global tiles, index t*K + k */
cr_status cr_get_ranges(cr_ctx* ctx, uint32_t* S, uint32_t* E, size_t* n);
/* last frame: per (k,i) depth d_{i,k} (index k*M + i); undefined for culled records */
cr_status cr_get_depths(cr_ctx* ctx, float* dst, size_t* n);
/* last frame: per (k,i) tile-union count |T_{i,k}| (index k*M + i)   */
cr_status cr_get_counts(cr_ctx* ctx, uint32_t* dst, size_t* n);

#ifdef __cplusplus
}
#endif
#endif /* COHERENT_RASTER_H */
