// cr_api.cu — C ABI (include/coherent_raster.h) and stage orchestration of
// the CoherentRaster B200 path.  Unity build: includes every kernel header so
// the __constant__ rig is shared without relocatable device code.
//
// Per-frame launch sequence (one stream):
//   preprocess<DEG>             a4 per-(i,k) records + exact band pre-cull   HBM/ALU
//   scan(vis) -> (key, r)       visible records, compressed presort keys     HBM
//   onesweep x4 (k, depth)      a7 depth presort of the records              HBM/issue
//   count + count_big           a6 cluster tile unions, list-position order  ALU
//   scan(counts)                pair offsets, P                              HBM
//   emit_rows + emit_big        a6 <tile, r> pairs in (k, depth, i) order    HBM
//   hist + onesweep x2..3       a7 stable tile sort                          HBM/issue
//   ranges                      a8                                           HBM
//   composite                   a9                                           ALU/MUFU
// Host<->device: two small reads (visible records + depth range, P) size the sorts.
#include <cuda_runtime.h>
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/coherent_raster.h"
#include "cr_composite.cuh"
#include "cr_device.cuh"
#include "cr_kernels.cuh"
#include "cr_sort.cuh"

#ifndef CR_GIT_TAG
#define CR_GIT_TAG "dev"
#endif

namespace {

using namespace cr;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Scan {  // functors for the generic device scan
  struct OutCompactVis {  // visible record r -> presort (key, r), same key as OutCompactList
    const uint32_t* dkey;
    uint32_t* ko;
    uint32_t* vo;
    const uint32_t* drange;
    int kbits;
    __device__ uint2 stage(long long i) const {  // flagged element i -> (key, r)
      const uint32_t r = (uint32_t)i;
      const uint32_t d = dkey[r], lo = drange[0], span = drange[1] - lo;
      const int B = span ? 32 - __clz(span) : 1;
      uint32_t key = d;
      if (B + kbits <= 32) {
        key = d - lo;
        if (kbits) key |= fdiv(r, c_fp.divM) << B;
      }
      return make_uint2(key, r);
    }
    __device__ void put(uint32_t pos, uint2 kv) const {
      ko[pos] = kv.x;
      vo[pos] = kv.y;
    }
  };
  struct InArr {
    const uint32_t* a;
    __device__ uint32_t operator()(long long i) const { return a[i]; }
    // 8 consecutive elements from i (i % 8 == 0, i + 8 <= n): two 16-byte loads
    __device__ void load8(long long i, uint32_t* v) const {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(a + i));
      const uint4 y = __ldg(reinterpret_cast<const uint4*>(a + i) + 1);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
      v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    }
  };
  struct OutStore {
    uint32_t* o;
    __device__ void operator()(long long i, uint32_t ex, uint32_t) const { o[i] = ex; }
    __device__ void store8(long long i, const uint32_t* ex) const {  // i % 8 == 0
      uint4* p = reinterpret_cast<uint4*>(o + i);
      p[0] = make_uint4(ex[0], ex[1], ex[2], ex[3]);
      p[1] = make_uint4(ex[4], ex[5], ex[6], ex[7]);
    }
  };
};

}  // namespace

struct cr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // scene
  bool has_scene = false;
  long long M = 0;
  int deg = 0;
  DevBuf mean4, cov8, shsoa;
  // display
  bool has_display = false;
  cr_display disp{};
  int TX = 0, TY = 0;
  DevBuf V, psi;
  int chunks_s = -1, chunk_stride = 0, chunks_pairs = -1;
  DevBuf chunks, nchunks, psi2;  // composite work items (psi2: paired-subpixel order)
  // rig
  bool has_rig = false;
  std::vector<CamDev> cams;
  std::vector<CamConstDev> ccon;
  float znear = 0.01f;
  // frame buffers
  DevBuf rec0, rec1, geom, vis, cnt, dkey, offs, slots, rows8, biglist;
  DevBuf bigcnt, bigmask, bigwlo, biginfo;  // union rows of big records (k_count_big)
  DevBuf ka, va, kb, vb;           // record sort ping-pong
  DevBuf pta, pva, ptb, pvb;       // pair sort ping-pong
  DevBuf hist, scalars, S, E, stage_out, frames;
  DevBuf look;                     // onesweep look-back status words
  DevBuf slook;                    // single-pass scan look-back status words + ticket
  uint32_t sepoch = 0;
  uint32_t epoch = 0;              // look-back tag of the last radix pass
  DevBuf tmp;                      // upload staging
  uint32_t* h_pinned = nullptr;    // small pinned readback
  // last frame
  int K = 0, bitK = 1;
  uint32_t P = 0, nvis = 0;
  const uint32_t* final_t = nullptr;
  const uint32_t* final_v = nullptr;
  bool has_frame = false;
  int launches = 0;
  cudaEvent_t ev[6] = {};
  cudaStream_t side = nullptr;     // forked stream for concurrent big-record emission
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_batch[2] = {};    // around a batched full-frame render
  // CR_FLAG_ASYNC_OUT: double-buffered device staging, copies on their own stream
  DevBuf astage[2];
  int aslot = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_comp[2] = {}, ev_copy[2] = {};
  long long device_bytes = 0;
  bool debug = false;  // CR_DEBUG=1: synchronise + trace after every stage
  int exp = 0;         // CR_EXP (read once at cr_create): developer A/B switches, 0 = shipped path
  bool motion_bound = false;  // pre-cull by the cluster motion bound (narrow clusters)
};

namespace {

cr_status fail(cr_ctx* c, cr_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

#define CR_CUDA(c, call)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail((c), e_ == cudaErrorMemoryAllocation ? CR_ERR_OUT_OF_MEMORY : CR_ERR_CUDA, \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);     \
  } while (0)

#define CR_LAUNCHED(c)                                                                     \
  do {                                                                                     \
    ++(c)->launches;                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                   \
    if (e_ != cudaSuccess)                                                                 \
      return fail((c), CR_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_),   \
                  __FILE__, __LINE__);                                                     \
  } while (0)

// CR_DEBUG tracing: synchronise the stream and report the stage + CUDA state.
#define CR_TRACE(c, what)                                                                   \
  do {                                                                                      \
    if ((c)->debug) {                                                                       \
      cudaError_t e_ = cudaStreamSynchronize((c)->stream);                                  \
      fprintf(stderr, "[cr] %-28s %s\n", what, cudaGetErrorString(e_));                    \
      fflush(stderr);                                                                       \
      if (e_ != cudaSuccess) return fail((c), CR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e_)); \
    }                                                                                       \
  } while (0)

void segv_handler(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  fprintf(stderr, "[cr] fatal signal %d, native backtrace:\n", sig);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}

#define CR_TRY(x)                 \
  do {                            \
    cr_status s_ = (x);           \
    if (s_ != CR_OK) return s_;   \
  } while (0)

cr_status ensure(cr_ctx* c, DevBuf& b, size_t bytes) {
  if (bytes <= b.bytes && b.p) return CR_OK;
  if (b.p) {
    cudaFree(b.p);
    c->device_bytes -= (long long)b.bytes;
    b.p = nullptr;
    b.bytes = 0;
  }
  size_t want = std::max<size_t>(bytes + bytes / 8, 256);
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    b.p = nullptr;
    return fail(c, CR_ERR_OUT_OF_MEMORY, "cudaMalloc(%zu): %s", want, cudaGetErrorString(e));
  }
  b.bytes = want;
  c->device_bytes += (long long)want;
  return CR_OK;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

template <class T>
T* P_(DevBuf& b) { return (T*)b.p; }

unsigned grid_for(long long n, int block) { return (unsigned)((n + block - 1) / block); }

// Kernels whose cameras are staged in dynamic shared memory (N x 80 B, up to
// 20 KB at N = 255) on top of their static arrays: allow the opt-in maximum
// of dynamic shared memory per block once per kernel (the default caps static
// + dynamic at 48 KB).
template <auto kernel>  // one instantiation (and one flag) per kernel
void allow_dyn_smem() {
  static bool done = false;
  if (done) return;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess && optin > (int)fa.sharedSizeBytes)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)fa.sharedSizeBytes);
  done = true;
}

// device exclusive scan: out(i, excl, in(i)); *d_total = sum
template <class In, class Out>
cr_status dev_scan(cr_ctx* c, In in, Out out, long long n, uint32_t* d_total) {
  if (n <= 0) {
    CR_CUDA(c, cudaMemsetAsync(d_total, 0, 4, c->stream));
    return CR_OK;
  }
  const long long nb = (n + kScanTile - 1) / kScanTile;
  const size_t lbytes = (size_t)nb * 8 + 64;  // the ticket counter + status words
  if (lbytes > c->slook.bytes || !c->slook.p) {
    CR_TRY(ensure(c, c->slook, lbytes));
    CR_CUDA(c, cudaMemsetAsync(c->slook.p, 0, c->slook.bytes, c->stream));
    c->sepoch = 0;
  }
  if (++c->sepoch >= (1u << 30)) {
    CR_CUDA(c, cudaMemsetAsync(c->slook.p, 0, c->slook.bytes, c->stream));
    c->sepoch = 1;
  }
  uint32_t* ticket = P_<uint32_t>(c->slook);  // first 64 bytes: ticket; then status words
  unsigned long long* look = (unsigned long long*)((char*)c->slook.p + 64);
  CR_CUDA(c, cudaMemsetAsync(ticket, 0, 4, c->stream));
  int* ovf = P_<int>(c->scalars) + 3;
  k_scan_onepass<In, Out><<<(unsigned)nb, kScanThreads, 0, c->stream>>>(in, out, n, look, ticket,
                                                                         c->sepoch, d_total, ovf);
  CR_LAUNCHED(c);
  return CR_OK;
}

// one stable LSD pass
cr_status radix_pass(cr_ctx* c, const uint32_t* kin, const uint32_t* vin, uint32_t* kout,
                     uint32_t* vout, long long n, int shift, bool from_val,
                     unsigned long long div, bool move_keys, bool agg = false) {
  if (n <= 0) return CR_OK;
  const long long nb = (n + kSortTile - 1) / kSortTile;
  CR_TRY(ensure(c, c->hist, (size_t)nb * 256 * 4));
  uint32_t* h = P_<uint32_t>(c->hist);
  if (from_val)
    k_radix_upsweep<true, false><<<(unsigned)nb, kSortThreads, 0, c->stream>>>(kin, vin, n, shift,
                                                                               div, h, (int)nb);
  else if (agg)
    k_radix_upsweep<false, true><<<(unsigned)nb, kSortThreads, 0, c->stream>>>(kin, vin, n, shift,
                                                                               div, h, (int)nb);
  else
    k_radix_upsweep<false, false><<<(unsigned)nb, kSortThreads, 0, c->stream>>>(kin, vin, n, shift,
                                                                                div, h, (int)nb);
  CR_LAUNCHED(c);
  uint32_t* tot = P_<uint32_t>(c->scalars) + 2;
  CR_TRY(dev_scan(c, Scan::InArr{h}, Scan::OutStore{h}, nb * 256, tot));
  if (from_val && move_keys)
    k_radix_downsweep<true, true><<<(unsigned)nb, kSortThreads, 0, c->stream>>>(
        kin, vin, kout, vout, n, shift, div, h, (int)nb);
  else if (from_val)
    k_radix_downsweep<true, false><<<(unsigned)nb, kSortThreads, 0, c->stream>>>(
        kin, vin, kout, vout, n, shift, div, h, (int)nb);
  else
    k_radix_downsweep<false, true><<<(unsigned)nb, kSortThreads, 0, c->stream>>>(
        kin, vin, kout, vout, n, shift, div, h, (int)nb);
  CR_LAUNCHED(c);
  return CR_OK;
}

// Stable LSD sort of (key, value) pairs on key bits [shift0, shift0 + 8*npass)
// by onesweep passes (one histogram kernel + one kernel per digit).  The
// result lands in (kA, vA) after the swaps (the pointers are swapped here).
// aggmask bit p: digit p is skewed (band mode), aggregate its histogram.
// 18 items per thread at 4 CTAs/SM (measured: sort stage 3.39 -> 3.25 ms at
// config C and 21.2 -> 20.3 ms at D against 16 items at 5 CTAs/SM; 12 items
// at 6 CTAs/SM 3.70 ms; 20 items exceed the 48 KB static shared memory)
constexpr int kOneItems = 18;
// bits0 = 9: the first digit is 9 bits wide (512 buckets), so a 17-bit 8K
// tile id takes 2 passes instead of 3.
cr_status radix_sort(cr_ctx* c, uint32_t*& kA, uint32_t*& vA, uint32_t*& kB, uint32_t*& vB,
                     long long n, int shift0, int npass, unsigned aggmask = 0,
                     bool hist_ready = false, uint32_t slotK = 0, int bits0 = 8) {
  if (n <= 0 || npass <= 0) return CR_OK;
  if (npass > 4) return fail(c, CR_ERR_CAPACITY, "radix_sort: npass %d > 4", npass);
  constexpr long long kTile = (long long)kSortThreads * kOneItems;
  const long long nb = (n + kTile - 1) / kTile;
  CR_TRY(ensure(c, c->hist, (size_t)(4 * kHistBins + 16) * 4));
  const size_t lbytes = (size_t)nb * (bits0 == 9 ? 512 : 256) * 8;
  if (lbytes > c->look.bytes || !c->look.p) {
    CR_TRY(ensure(c, c->look, lbytes));
    CR_CUDA(c, cudaMemsetAsync(c->look.p, 0, c->look.bytes, c->stream));
    c->epoch = 0;
  }
  uint32_t* gh = P_<uint32_t>(c->hist);
  uint32_t* ctr = gh + 4 * kHistBins;
  if (hist_ready) {  // histograms already in c->hist (k_bin): zero only the tile counters
    CR_CUDA(c, cudaMemsetAsync(ctr, 0, 16 * 4, c->stream));
  } else {
    CR_CUDA(c, cudaMemsetAsync(gh, 0, (4 * kHistBins + 16) * 4, c->stream));
  }
  const unsigned hgrid = (unsigned)std::max<long long>(
      1, std::min<long long>((n / 4 + kHistThreads - 1) / kHistThreads, 148 * 8));
  if (!hist_ready) {
    k_radix_hist<<<hgrid, kHistThreads, 0, c->stream>>>(kA, n, shift0, npass, aggmask, gh, bits0);
    CR_LAUNCHED(c);
  }
  for (int p = 0; p < npass; ++p) {
    if (++c->epoch >= (1u << 30)) {  // never in practice; keep the tags unambiguous
      CR_CUDA(c, cudaMemsetAsync(c->look.p, 0, c->look.bytes, c->stream));
      c->epoch = 1;
    }
    const int sh = p == 0 ? shift0 : shift0 + bits0 + 8 * (p - 1);
    if (p == 0 && bits0 == 9) {
      constexpr int dyn = onesweep_dyn_smem<kOneItems>();
      cudaFuncSetAttribute(k_radix_onesweep_n<kOneItems, 7, 3, 512>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
      k_radix_onesweep_n<kOneItems, 7, 3, 512><<<(unsigned)nb, kSortThreads, dyn, c->stream>>>(
          kA, vA, kB, vB, n, sh, gh + kHistBins * p, P_<unsigned long long>(c->look), ctr + p,
          c->epoch, p == npass - 1 ? slotK : 0u);
    } else {
      k_radix_onesweep<kOneItems, 7, 4><<<(unsigned)nb, kSortThreads, 0, c->stream>>>(
          kA, vA, kB, vB, n, sh, gh + kHistBins * p, P_<unsigned long long>(c->look), ctr + p,
          c->epoch, p == npass - 1 ? slotK : 0u);
    }
    CR_LAUNCHED(c);
    std::swap(kA, kB);
    std::swap(vA, vB);
  }
  return CR_OK;
}

cr_status read_words(cr_ctx* c, const uint32_t* d, uint32_t* h, int n) {
  CR_CUDA(c, cudaMemcpyAsync(c->h_pinned, d, 4 * n, cudaMemcpyDeviceToHost, c->stream));
  CR_CUDA(c, cudaStreamSynchronize(c->stream));
  std::memcpy(h, c->h_pinned, 4 * n);
  return CR_OK;
}

cr_status read_u32(cr_ctx* c, const uint32_t* d, uint32_t* h) {
  CR_CUDA(c, cudaMemcpyAsync(c->h_pinned, d, 4, cudaMemcpyDeviceToHost, c->stream));
  CR_CUDA(c, cudaStreamSynchronize(c->stream));
  *h = c->h_pinned[0];
  return CR_OK;
}

void cam_consts_host(const cr_camera& in, int W, int H, CamDev* d, CamConstDev* k) {
  std::memcpy(d->R, in.R, sizeof(float) * 9);
  std::memcpy(d->t, in.t, sizeof(float) * 3);
  d->fx = in.fx; d->fy = in.fy; d->cx = in.cx; d->cy = in.cy;
  // O6 frustum clamp constants and O11 camera centre, fp64 -> fp32
  const double tfx = 0.5 * (double)W / (double)in.fx;
  const double tfy = 0.5 * (double)H / (double)in.fy;
  k->limxp = (float)(((double)W - (double)in.cx) / (double)in.fx + 0.3 * tfx);
  k->limxn = (float)((double)in.cx / (double)in.fx + 0.3 * tfx);
  k->limyp = (float)(((double)H - (double)in.cy) / (double)in.fy + 0.3 * tfy);
  k->limyn = (float)((double)in.cy / (double)in.fy + 0.3 * tfy);
  for (int a = 0; a < 3; ++a) {
    double v = 0.0;
    for (int r = 0; r < 3; ++r) v += (double)in.R[r * 3 + a] * (double)in.t[r];
    k->C[a] = (float)(-v);
  }
  k->pad = 0.f;
}

bool finite_all(const float* p, long long n) {
  for (long long q = 0; q < n; ++q)
    if (!std::isfinite(p[q])) return false;
  return true;
}

}  // namespace

extern "C" {

const char* cr_version(void) { return "coherent_raster sm_100a " CR_GIT_TAG; }

const char* cr_status_string(cr_status s) {
  switch (s) {
    case CR_OK: return "CR_OK";
    case CR_ERR_INVALID_ARG: return "CR_ERR_INVALID_ARG";
    case CR_ERR_INVALID_CONFIG: return "CR_ERR_INVALID_CONFIG";
    case CR_ERR_CONFIG_MISMATCH: return "CR_ERR_CONFIG_MISMATCH";
    case CR_ERR_TILE_ID_OVERFLOW: return "CR_ERR_TILE_ID_OVERFLOW";
    case CR_ERR_NONFINITE: return "CR_ERR_NONFINITE";
    case CR_ERR_NOT_READY: return "CR_ERR_NOT_READY";
    case CR_ERR_OUT_OF_MEMORY: return "CR_ERR_OUT_OF_MEMORY";
    case CR_ERR_CUDA: return "CR_ERR_CUDA";
    case CR_ERR_CAPACITY: return "CR_ERR_CAPACITY";
  }
  return "CR_ERR_UNKNOWN";
}

cr_status cr_create(int cuda_device, void* cuda_stream, cr_ctx** out) {
  if (!out) return CR_ERR_INVALID_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device < 0 || cuda_device >= n) {
    cudaGetLastError();
    return CR_ERR_CUDA;
  }
  cr_ctx* c = new cr_ctx();
  c->device = cuda_device;
  const char* dbg = getenv("CR_DEBUG");
  c->debug = dbg && dbg[0] && dbg[0] != '0';
  const char* ex = getenv("CR_EXP");
  c->exp = ex ? atoi(ex) : 0;
  if (c->debug) {
    signal(SIGSEGV, segv_handler);
    signal(SIGBUS, segv_handler);
  }
  c->stream = (cudaStream_t)cuda_stream;
  if (cudaSetDevice(cuda_device) != cudaSuccess || cudaMallocHost(&c->h_pinned, 256) != cudaSuccess) {
    delete c;
    return CR_ERR_CUDA;
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  for (auto& e : c->ev_batch) cudaEventCreate(&e);
  for (int q = 0; q < 2; ++q) {
    cudaEventCreateWithFlags(&c->ev_comp[q], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_copy[q], cudaEventDisableTiming);
  }
  cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (ensure(c, c->scalars, 64) != CR_OK) {
    delete c;
    return CR_ERR_OUT_OF_MEMORY;
  }
  *out = c;
  return CR_OK;
}

void cr_destroy(cr_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  DevBuf* all[] = {&c->mean4, &c->cov8, &c->shsoa, &c->V, &c->psi, &c->chunks, &c->nchunks, &c->psi2,
                   &c->rec0, &c->rec1, &c->geom, &c->vis, &c->slots, &c->rows8, &c->biglist, &c->bigcnt,
                   &c->bigmask, &c->bigwlo, &c->biginfo, &c->cnt, &c->dkey, &c->offs, &c->ka, &c->va, &c->kb,
                   &c->vb, &c->pta, &c->pva, &c->ptb, &c->pvb, &c->hist, &c->look, &c->slook,
                   &c->scalars, &c->S, &c->E, &c->stage_out, &c->frames, &c->tmp};
  for (DevBuf* b : all) release(*b);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_batch)
    if (e) cudaEventDestroy(e);
  if (c->copy) {
    cudaStreamSynchronize(c->copy);
    cudaStreamDestroy(c->copy);
  }
  for (int q = 0; q < 2; ++q) {
    if (c->ev_comp[q]) cudaEventDestroy(c->ev_comp[q]);
    if (c->ev_copy[q]) cudaEventDestroy(c->ev_copy[q]);
    release(c->astage[q]);
  }
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  delete c;
}

cr_status cr_synchronize(cr_ctx* c) {
  if (!c) return CR_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  CR_CUDA(c, cudaStreamSynchronize(c->stream));
  CR_CUDA(c, cudaStreamSynchronize(c->copy));
  return CR_OK;
}

cr_status cr_set_stream(cr_ctx* c, void* s) {
  if (!c) return CR_ERR_INVALID_ARG;
  c->stream = (cudaStream_t)s;
  return CR_OK;
}

const char* cr_last_error(const cr_ctx* c) { return c ? c->err.c_str() : "null context"; }

cr_status cr_upload_gaussians(cr_ctx* c, int64_t M, int deg, const float* means,
                              const float* quats, const float* scales, const float* opac,
                              const float* sh, int on_dev) {
  if (!c) return CR_ERR_INVALID_ARG;
  if (M < 0 || deg < 0 || deg > 3) return fail(c, CR_ERR_INVALID_ARG, "M=%lld deg=%d", (long long)M, deg);
  if (M > 0 && (!means || !quats || !scales || !opac || !sh))
    return fail(c, CR_ERR_INVALID_ARG, "null Gaussian pointer");
  if (M > (1LL << 30)) return fail(c, CR_ERR_INVALID_ARG, "M too large");
  cudaSetDevice(c->device);
  const int nc3 = (deg + 1) * (deg + 1) * 3;
  c->has_frame = false;
  if (M == 0) {
    c->M = 0;
    c->deg = deg;
    c->has_scene = true;
    return CR_OK;
  }
  // tau_i = 2 ln(255 o_i) on the host in fp64 (O4); opacities needed on the host
  std::vector<float> h_op((size_t)M), h_tau((size_t)M);
  if (on_dev) {
    CR_CUDA(c, cudaMemcpyAsync(h_op.data(), opac, 4 * M, cudaMemcpyDeviceToHost, c->stream));
    CR_CUDA(c, cudaStreamSynchronize(c->stream));
  } else {
    std::memcpy(h_op.data(), opac, 4 * M);
  }
  for (long long i = 0; i < M; ++i) {
    if (!std::isfinite(h_op[i])) return fail(c, CR_ERR_NONFINITE, "opacity %lld not finite", i);
    if (!(h_op[i] >= 0.0f && h_op[i] <= 1.0f))
      return fail(c, CR_ERR_INVALID_ARG, "opacity %lld = %g outside [0,1]", i, (double)h_op[i]);
    h_tau[i] = (float)(2.0 * std::log(255.0 * (double)h_op[i]));  // o = 0: -inf, culled (O4)
  }
  const size_t nin = (size_t)M * (3 + 4 + 3 + 1 + 1 + nc3);
  CR_TRY(ensure(c, c->tmp, nin * 4));
  float* t = P_<float>(c->tmp);
  float *d_means = t, *d_quats = d_means + 3 * M, *d_scales = d_quats + 4 * M,
        *d_op = d_scales + 3 * M, *d_tau = d_op + M, *d_sh = d_tau + M;
  const cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CR_CUDA(c, cudaMemcpyAsync(d_means, means, 12 * M, kind, c->stream));
  CR_CUDA(c, cudaMemcpyAsync(d_quats, quats, 16 * M, kind, c->stream));
  CR_CUDA(c, cudaMemcpyAsync(d_scales, scales, 12 * M, kind, c->stream));
  CR_CUDA(c, cudaMemcpyAsync(d_op, h_op.data(), 4 * M, cudaMemcpyHostToDevice, c->stream));
  CR_CUDA(c, cudaMemcpyAsync(d_tau, h_tau.data(), 4 * M, cudaMemcpyHostToDevice, c->stream));
  CR_CUDA(c, cudaMemcpyAsync(d_sh, sh, 4 * (size_t)M * nc3, kind, c->stream));
  // validate the staged copy first: a rejected upload keeps the previous scene
  int* flag = P_<int>(c->scalars) + 7;
  CR_CUDA(c, cudaMemsetAsync(flag, 0, 4, c->stream));
  k_validate<<<148 * 8, 256, 0, c->stream>>>((long long)(d_op - d_means), d_means, flag);
  CR_LAUNCHED(c);
  k_validate<<<148 * 8, 256, 0, c->stream>>>((long long)M * nc3, d_sh, flag);
  CR_LAUNCHED(c);
  uint32_t bad = 0;
  CR_TRY(read_u32(c, (const uint32_t*)flag, &bad));
  if (bad) return fail(c, CR_ERR_NONFINITE, "NaN/Inf in uploaded Gaussians");
  c->has_scene = false;  // the scene buffers may be reallocated from here on
  CR_TRY(ensure(c, c->mean4, 16 * (size_t)M));
  CR_TRY(ensure(c, c->cov8, 32 * (size_t)M));
  CR_TRY(ensure(c, c->shsoa, 4 * (size_t)M * nc3));
  k_upload<<<grid_for(M, 256), 256, 0, c->stream>>>(M, nc3, d_means, d_quats, d_scales, d_op,
                                                     d_tau, d_sh, P_<float4>(c->mean4),
                                                     P_<float4>(c->cov8), P_<float>(c->shsoa));
  CR_LAUNCHED(c);
  c->M = M;
  c->deg = deg;
  c->has_scene = true;
  return CR_OK;
}

cr_status cr_set_display(cr_ctx* c, const cr_display* d) {
  if (!c || !d) return CR_ERR_INVALID_ARG;
  const int ts = d->tile_size == 0 ? 16 : d->tile_size;
  if (d->width < 1 || d->height < 1 || d->num_views < 1 || d->num_views > kMaxViews ||
      !(d->lens_pitch > 0) || !std::isfinite(d->lens_pitch) || !std::isfinite(d->slant) ||
      !std::isfinite(d->center_offset) || ts != 16 || d->width > 65535 || d->height > 65535)
    return fail(c, CR_ERR_INVALID_CONFIG, "invalid display (W=%d H=%d N=%d Lx=%g tile=%d)",
                d->width, d->height, d->num_views, d->lens_pitch, ts);
  cudaSetDevice(c->device);
  const int W = d->width, H = d->height;
  const int TX = (W + 15) / 16, TY = (H + 15) / 16;
  CR_TRY(ensure(c, c->V, (size_t)W * H * 3));
  CR_TRY(ensure(c, c->psi, (size_t)TX * TY * kTileSub * 2));
  const double tA = std::tan(d->slant);  // Z2: tan on the host in fp64
  const long long nsub = (long long)W * H * 3;
  k_viewmap<<<(unsigned)std::min<long long>(grid_for(nsub, 256), 148 * 64), 256, 0, c->stream>>>(
      P_<uint8_t>(c->V), W, H, d->num_views, d->lens_pitch, tA, d->center_offset);
  CR_LAUNCHED(c);
  k_remap_build<<<grid_for((long long)TX * TY, 8), 256, 0, c->stream>>>(
      P_<uint8_t>(c->V), P_<uint16_t>(c->psi), W, H, TX, TY);
  CR_LAUNCHED(c);
  c->disp = *d;
  c->disp.tile_size = 16;
  c->TX = TX;
  c->TY = TY;
  c->chunks_s = -1;
  c->has_frame = false;
  c->has_display = true;
  if (c->has_rig && (int)c->cams.size() != d->num_views) c->has_rig = false;
  return CR_OK;
}

cr_status cr_set_camera_rig(cr_ctx* c, int32_t n, const cr_camera* views, float znear) {
  if (!c || !views || n < 1) return CR_ERR_INVALID_ARG;
  if (!c->has_display) return fail(c, CR_ERR_NOT_READY, "set the display before the rig");
  if (n != c->disp.num_views)
    return fail(c, CR_ERR_CONFIG_MISMATCH, "rig has %d views, display has %d", n,
                c->disp.num_views);
  if (!(znear > 0) || !std::isfinite(znear)) return fail(c, CR_ERR_INVALID_ARG, "znear");
  for (int j = 0; j < n; ++j)
    if (!finite_all((const float*)&views[j], 16) || !(views[j].fx > 0) || !(views[j].fy > 0))
      return fail(c, CR_ERR_NONFINITE, "camera %d not finite / non-positive focal", j);
  c->cams.resize(n);
  c->ccon.resize(n);
  for (int j = 0; j < n; ++j)
    cam_consts_host(views[j], c->disp.width, c->disp.height, &c->cams[j], &c->ccon[j]);
  c->znear = znear;
  c->has_rig = true;
  c->has_frame = false;
  return CR_OK;
}

cr_status cr_make_orbit_rig(const cr_display* d, const float look_at[3], const float up[3],
                            float radius, float height, float yaw_deg, float pitch_deg,
                            float fov_y_deg, cr_camera* out) {
  if (!d || !look_at || !up || !out || d->num_views < 1 || d->height < 1) return CR_ERR_INVALID_ARG;
  const int N = d->num_views;
  const double pi = 3.14159265358979323846;
  const double fy = d->height / (2.0 * std::tan(fov_y_deg * pi / 360.0));
  for (int j = 0; j < N; ++j) {
    const double a = N > 1 ? (-d->view_cone / 2.0 + d->view_cone * j / (N - 1)) : 0.0;
    const double th = (yaw_deg + a) * pi / 180.0, ph = pitch_deg * pi / 180.0;
    const double C[3] = {look_at[0] + radius * std::sin(th) * std::cos(ph),
                         look_at[1] + height + radius * std::sin(ph),
                         look_at[2] + radius * std::cos(th) * std::cos(ph)};
    double f[3] = {look_at[0] - C[0], look_at[1] - C[1], look_at[2] - C[2]};
    double fn = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
    for (double& v : f) v /= fn;
    double x[3] = {f[1] * up[2] - f[2] * up[1], f[2] * up[0] - f[0] * up[2],
                   f[0] * up[1] - f[1] * up[0]};
    double xn = std::sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
    for (double& v : x) v /= xn;
    const double y[3] = {f[1] * x[2] - f[2] * x[1], f[2] * x[0] - f[0] * x[2],
                         f[0] * x[1] - f[1] * x[0]};
    const double* rows[3] = {x, y, f};
    cr_camera& cam = out[j];
    for (int r = 0; r < 3; ++r) {
      for (int q = 0; q < 3; ++q) cam.R[r * 3 + q] = (float)rows[r][q];
      cam.t[r] = (float)(-(rows[r][0] * C[0] + rows[r][1] * C[1] + rows[r][2] * C[2]));
    }
    cam.fx = cam.fy = (float)fy;
    cam.cx = (float)(d->width / 2.0);
    cam.cy = (float)(d->height / 2.0);
  }
  return CR_OK;
}

// The full-frame baseline B views per pass (the paper's "3DGS (batch=B)",
// P:520): each pass renders views [v0, v0 + B) as a B-view frame with
// CR_FLAG_VIEW_FRAMES straight into its slice of the [N][rows][W][3] frame
// buffer (its own preprocess, binning, sort and full-frame composite), then
// the N frames are interlaced by V once.
static cr_status render_view_batches(cr_ctx* c, const cr_render_opts* o, void* out,
                                     size_t out_bytes, int out_on_device, cr_stats* st) {
  const int N = c->disp.num_views, W = c->disp.width, H = c->disp.height;
  const int B = o->view_batch;
  if (B % o->cluster_size != 0)
    return fail(c, CR_ERR_INVALID_ARG, "view_batch %d is not a multiple of cluster_size %d", B,
                o->cluster_size);
  int row0 = o->tile_row_begin, row1 = o->tile_row_end;
  if (row0 == 0 && row1 == 0) row1 = c->TY;
  if (row0 < 0 || row1 > c->TY || row0 >= row1)
    return fail(c, CR_ERR_INVALID_ARG, "tile rows [%d,%d) outside [0,%d)", row0, row1, c->TY);
  const int rows_px = std::min(H, row1 * 16) - row0 * 16;
  const bool view_frames = (o->flags & CR_FLAG_VIEW_FRAMES) != 0;
  const size_t plane = (size_t)rows_px * W * 3 * (o->output_format ? 4 : 1);
  const size_t obytes = view_frames ? (size_t)N * plane : plane;
  if (out_bytes < obytes) return fail(c, CR_ERR_INVALID_ARG, "out_bytes %zu < %zu", out_bytes, obytes);
  cudaSetDevice(c->device);
  void* fr = out;
  if (!(view_frames && out_on_device)) {
    CR_TRY(ensure(c, c->frames, (size_t)N * plane));
    fr = c->frames.p;
  }
  CR_CUDA(c, cudaEventRecord(c->ev_batch[0], c->stream));
  const std::vector<CamDev> cams = c->cams;
  const std::vector<CamConstDev> ccon = c->ccon;
  cr_render_opts oi = *o;
  oi.flags = (o->flags & CR_FLAG_COUNT_EVALS) | CR_FLAG_VIEW_FRAMES;
  oi.view_batch = 0;
  cr_stats acc{};
  int launches = 0;
  cr_status r = CR_OK;
  for (int v0 = 0; v0 < N && r == CR_OK; v0 += B) {
    const int nb = std::min(B, N - v0);
    c->cams.assign(cams.begin() + v0, cams.begin() + v0 + nb);
    c->ccon.assign(ccon.begin() + v0, ccon.begin() + v0 + nb);
    c->disp.num_views = nb;
    cr_stats sb{};
    r = cr_render_interlaced(c, &oi, (char*)fr + (size_t)v0 * plane, (size_t)nb * plane, 1,
                             st ? &sb : nullptr);
    launches += c->launches;
    acc.pairs += sb.pairs;
    acc.visible_ik += sb.visible_ik;
    acc.culled_near += sb.culled_near;
    acc.culled_degenerate += sb.culled_degenerate;
    acc.culled_opacity += sb.culled_opacity;
    acc.evals += sb.evals;
    acc.num_clusters += sb.num_clusters;
    acc.emit_fallback += sb.emit_fallback;
  }
  c->cams = cams;
  c->ccon = ccon;
  c->disp.num_views = N;
  if (r != CR_OK) return r;
  c->has_frame = false;  // introspection would describe the last pass only
  cudaStream_t str = c->stream;
  if (!view_frames) {
    void* dst = out;
    if (!out_on_device) {
      CR_TRY(ensure(c, c->stage_out, plane));
      dst = c->stage_out.p;
    }
    const long long nsub = (long long)rows_px * W * 3;
    const unsigned gi = (unsigned)std::min<long long>(grid_for(nsub, 256), 148 * 32);
    if (o->output_format == 0) k_interlace<0><<<gi, 256, 0, str>>>(P_<uint8_t>(c->V), fr, dst, rows_px);
    else k_interlace<1><<<gi, 256, 0, str>>>(P_<uint8_t>(c->V), fr, dst, rows_px);
    c->launches = launches;
    CR_LAUNCHED(c);
    launches = c->launches;
    if (!out_on_device) CR_CUDA(c, cudaMemcpyAsync(out, dst, plane, cudaMemcpyDeviceToHost, str));
  } else if (!out_on_device) {
    CR_CUDA(c, cudaMemcpyAsync(out, fr, (size_t)N * plane, cudaMemcpyDeviceToHost, str));
  }
  CR_CUDA(c, cudaEventRecord(c->ev_batch[1], str));
  c->launches = launches;
  if (!out_on_device || st) CR_CUDA(c, cudaStreamSynchronize(str));
  if (st) {
    *st = acc;
    st->bit_k = 0;
    st->launches = launches;
    cudaEventElapsedTime(&st->ms_total, c->ev_batch[0], c->ev_batch[1]);
    st->device_bytes = c->device_bytes;
  }
  return CR_OK;
}

cr_status cr_render_interlaced(cr_ctx* c, const cr_render_opts* o, void* out, size_t out_bytes,
                               int out_on_device, cr_stats* st) {
  if (!c || !o || !out) return CR_ERR_INVALID_ARG;
  if (!c->has_scene || !c->has_display || !c->has_rig)
    return fail(c, CR_ERR_NOT_READY, "upload Gaussians, set display and rig first");
  const int N = c->disp.num_views, W = c->disp.width, H = c->disp.height;
  const int TX = c->TX, TY = c->TY;
  const int s = o->cluster_size;
  if (s < 1 || s > kMaxCluster) return fail(c, CR_ERR_INVALID_CONFIG, "cluster_size %d not in 1..32", s);
  if (o->remap != 0 && o->remap != 1) return fail(c, CR_ERR_INVALID_ARG, "remap must be 0/1");
  if (o->kernel != 0 && o->kernel != 1) return fail(c, CR_ERR_INVALID_ARG, "kernel must be 0/1");
  if (o->kernel == 0 && o->remap == 0)
    return fail(c, CR_ERR_INVALID_ARG, "the staged composite needs remap=1 (use kernel=1)");
  if (o->output_format != 0 && o->output_format != 1) return fail(c, CR_ERR_INVALID_ARG, "format");
  const bool view_frames = (o->flags & CR_FLAG_VIEW_FRAMES) != 0;
  const bool fullframe = view_frames || (o->flags & CR_FLAG_FULLFRAME) != 0;
  if (o->view_batch < 0) return fail(c, CR_ERR_INVALID_ARG, "view_batch %d < 0", o->view_batch);
  if (fullframe && o->view_batch > 0 && o->view_batch < N)
    return render_view_batches(c, o, out, out_bytes, out_on_device, st);
  for (int u = 0; u < 3; ++u)
    if (!std::isfinite(o->background[u])) return fail(c, CR_ERR_NONFINITE, "background");
  int row0 = o->tile_row_begin, row1 = o->tile_row_end;
  if (row0 == 0 && row1 == 0) row1 = TY;
  if (row0 < 0 || row1 > TY || row0 >= row1)
    return fail(c, CR_ERR_INVALID_ARG, "tile rows [%d,%d) outside [0,%d)", row0, row1, TY);
  const int y0 = row0 * 16, y1 = std::min(H, row1 * 16);
  const size_t obytes =
      (size_t)(y1 - y0) * W * 3 * (o->output_format ? 4 : 1) * (view_frames ? (size_t)N : 1);
  if (out_bytes < obytes) return fail(c, CR_ERR_INVALID_ARG, "out_bytes %zu < %zu", out_bytes, obytes);
  // O3 clusters
  const int K = (N + s - 1) / s;
  int bitK = 0;
  while ((1 << bitK) < K) ++bitK;
  bitK = std::max(bitK, 1);
  if ((long long)TX * TY >= (1LL << (32 - bitK)))
    return fail(c, CR_ERR_TILE_ID_OVERFLOW, "%d tiles need more than %d bits", TX * TY, 32 - bitK);
  const long long M = c->M;
  const long long R = (long long)K * M;
  if (R > 0xFFFFFFFFLL) return fail(c, CR_ERR_CAPACITY, "K*M = %lld exceeds 2^32", R);
  cudaSetDevice(c->device);
  c->launches = 0;
  c->has_frame = false;
  cudaStream_t str = c->stream;

  // ---- constants: rig, representatives, frame parameters
  FrameParams fp{};
  fp.W = W; fp.H = H; fp.TX = TX; fp.TY = TY; fp.N = N; fp.s = s; fp.K = K; fp.bitK = bitK;
  fp.row0 = row0; fp.row1 = row1; fp.deg = c->deg; fp.remap = o->remap; fp.M = M;
  fp.divM = make_fastdiv((uint32_t)std::max<long long>(M, 1));
  fp.exp = c->exp;
  fp.znear = c->znear;
  for (int u = 0; u < 3; ++u) fp.bg[u] = o->background[u];
  std::vector<int> rep(K);
  for (int k = 0; k < K; ++k) rep[k] = std::min(k * s + s / 2, N - 1);
  CR_CUDA(c, cudaMemcpyToSymbolAsync(c_cams, c->cams.data(), sizeof(CamDev) * N, 0,
                                     cudaMemcpyHostToDevice, str));
  CR_CUDA(c, cudaMemcpyToSymbolAsync(c_ccon, c->ccon.data(), sizeof(CamConstDev) * N, 0,
                                     cudaMemcpyHostToDevice, str));
  CR_CUDA(c, cudaMemcpyToSymbolAsync(c_rep, rep.data(), sizeof(int) * K, 0,
                                     cudaMemcpyHostToDevice, str));
  {  // cluster motion bounds for the band / frame pre-cull (fp64, rounded up)
    std::vector<float4> clb(K), clax(K), clbx(K);
    std::vector<float> cldb(K);
    double maxdA = 0.0;
    for (int k = 0; k < K; ++k) {
      const CamDev& cr = c->cams[rep[k]];
      std::vector<std::array<double, 12>> mv;  // (A - I) row-major, then b
      for (int j = k * s; j < std::min(k * s + s, N); ++j) {
        const CamDev& cj = c->cams[j];
        std::array<double, 12> q{};
        for (int a = 0; a < 3; ++a)
          for (int bb = 0; bb < 3; ++bb) {  // A = R_j R_rep^T
            double v = 0.0;
            for (int z = 0; z < 3; ++z) v += (double)cj.R[a * 3 + z] * (double)cr.R[bb * 3 + z];
            q[a * 3 + bb] = v;
          }
        for (int a = 0; a < 3; ++a) {  // b = t_j - A t_rep
          double v = (double)cj.t[a];
          for (int z = 0; z < 3; ++z) v -= q[a * 3 + z] * (double)cr.t[z];
          q[9 + a] = v;
        }
        for (int a = 0; a < 3; ++a) q[a * 3 + a] -= 1.0;
        mv.push_back(q);
      }
      // centre: argmin_c sum_j |(A_j - I) c + b_j|^2, lightly regularised (Cramer)
      double Mm[9] = {0}, rhs[3] = {0};
      for (const auto& q : mv)
        for (int a = 0; a < 3; ++a) {
          for (int bb = 0; bb < 3; ++bb)
            for (int z = 0; z < 3; ++z) Mm[a * 3 + bb] += q[z * 3 + a] * q[z * 3 + bb];
          for (int z = 0; z < 3; ++z) rhs[a] -= q[z * 3 + a] * q[9 + z];
        }
      const double tr = Mm[0] + Mm[4] + Mm[8];
      for (int a = 0; a < 3; ++a) Mm[a * 3 + a] += 1e-9 * tr + 1e-300;
      auto det3 = [](const double* m) {
        return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
               m[2] * (m[3] * m[7] - m[4] * m[6]);
      };
      double cc[3] = {0, 0, 0};
      const double dM = det3(Mm);
      if (std::isfinite(dM) && dM != 0.0)
        for (int a = 0; a < 3; ++a) {
          double t3[9];
          std::memcpy(t3, Mm, sizeof(t3));
          for (int z = 0; z < 3; ++z) t3[z * 3 + a] = rhs[z];
          cc[a] = det3(t3) / dM;
          if (!std::isfinite(cc[a])) cc[a] = 0.0;
        }
      double dA = 0.0, db = 0.0;  // the bound holds for ANY c; the centre only tightens it
      double dAa[3] = {0, 0, 0}, dba[3] = {0, 0, 0};  // per camera-space axis
      for (const auto& q : mv) {
        double fro = 0.0, b2 = 0.0;
        for (int a = 0; a < 9; ++a) fro += q[a] * q[a];
        for (int a = 0; a < 3; ++a) {
          double v = q[9 + a];
          for (int z = 0; z < 3; ++z) v += q[a * 3 + z] * cc[z];
          b2 += v * v;
          const double rn = std::sqrt(q[a * 3] * q[a * 3] + q[a * 3 + 1] * q[a * 3 + 1] +
                                      q[a * 3 + 2] * q[a * 3 + 2]);
          dAa[a] = std::max(dAa[a], rn);
          dba[a] = std::max(dba[a], std::fabs(v));
        }
        dA = std::max(dA, std::sqrt(fro));
        db = std::max(db, std::sqrt(b2));
      }
      clb[k] = make_float4((float)cc[0], (float)cc[1], (float)cc[2], (float)(dA * 1.0001 + 1e-7));
      maxdA = std::max(maxdA, dA);
      cldb[k] = (float)(db * 1.0001 + 1e-6);
      clax[k] = make_float4((float)(dAa[0] * 1.0001 + 1e-7), (float)(dAa[1] * 1.0001 + 1e-7),
                            (float)(dAa[2] * 1.0001 + 1e-7), 0.f);
      clbx[k] = make_float4((float)(dba[0] * 1.0001 + 1e-6), (float)(dba[1] * 1.0001 + 1e-6),
                            (float)(dba[2] * 1.0001 + 1e-6), 0.f);
    }
    CR_CUDA(c, cudaMemcpyToSymbolAsync(c_clb, clb.data(), sizeof(float4) * K, 0,
                                       cudaMemcpyHostToDevice, str));
    CR_CUDA(c, cudaMemcpyToSymbolAsync(c_cldb, cldb.data(), sizeof(float) * K, 0,
                                       cudaMemcpyHostToDevice, str));
    CR_CUDA(c, cudaMemcpyToSymbolAsync(c_clax, clax.data(), sizeof(float4) * K, 0,
                                       cudaMemcpyHostToDevice, str));
    CR_CUDA(c, cudaMemcpyToSymbolAsync(c_clbx, clbx.data(), sizeof(float4) * K, 0,
                                       cudaMemcpyHostToDevice, str));
    c->motion_bound = maxdA < (double)kMotionBoundMax;  // narrow clusters: one projection
  }
  CR_CUDA(c, cudaMemcpyToSymbolAsync(c_fp, &fp, sizeof(fp), 0, cudaMemcpyHostToDevice, str));

  // ---- composite work items (static per display and s)
  // two subpixels of one view per lane (k_composite_pairs, the default); CR_EXP
  // bit 6: one subpixel per lane (k_composite_staged, round 2's kernel)
  const int pairs = (c->exp & 64) ? 0 : 1;
  if (o->kernel == 0 && !fullframe && (c->chunks_s != s || c->chunks_pairs != pairs)) {
    const int stride = K + 24;
    CR_TRY(ensure(c, c->chunks, (size_t)TX * TY * stride * 4));
    CR_TRY(ensure(c, c->nchunks, (size_t)TX * TY * 4));
    if (pairs) {
      CR_TRY(ensure(c, c->psi2, (size_t)TX * TY * kPairSlots * 2));
      k_pairs_build<<<grid_for((long long)TX * TY, 128), 128, 0, str>>>(
          P_<uint8_t>(c->V), P_<uint16_t>(c->psi), P_<uint16_t>(c->psi2), P_<uint32_t>(c->chunks),
          P_<uint32_t>(c->nchunks), stride, W, TX, TY, s, (c->exp & 2048) ? 0 : 1);
    } else {
      k_chunks_build<<<grid_for((long long)TX * TY, 128), 128, 0, str>>>(
          P_<uint8_t>(c->V), P_<uint16_t>(c->psi), P_<uint32_t>(c->chunks),
          P_<uint32_t>(c->nchunks), stride, W, TX, TY, s);
    }
    CR_LAUNCHED(c);
    c->chunks_s = s;
    c->chunks_pairs = pairs;
    c->chunk_stride = stride;
  }

  uint32_t* sc = P_<uint32_t>(c->scalars);  // [0] nvis [1] P [2] tmp [3] overflow [4] nvis0
  // counters: [0] near [1] degenerate [2] opacity [3] evals (u64 at byte 32)
  unsigned long long* counters = (unsigned long long*)(sc + 8);
  CR_CUDA(c, cudaMemsetAsync(sc, 0, 64, str));
  CR_CUDA(c, cudaMemsetAsync(sc + 16, 0xFF, 4, str));  // depth-bit range [min, max]
  CR_CUDA(c, cudaMemsetAsync(sc + 17, 0, 4, str));
  CR_TRACE(c, "constants+chunks");
  CR_CUDA(c, cudaEventRecord(c->ev[0], str));

  // ---- a4 preprocess + SH, a6 count, compaction of records with >= 1 tile
  const size_t Rz = (size_t)std::max<long long>(R, 1);
  CR_TRY(ensure(c, c->rec0, Rz * 32));  // AoS 32-byte records (rec1 unused)
  CR_TRY(ensure(c, c->geom, Rz * 32));
  CR_TRY(ensure(c, c->vis, Rz * 4));
  CR_TRY(ensure(c, c->cnt, Rz * 4));
  CR_TRY(ensure(c, c->dkey, Rz * 4));
  CR_TRY(ensure(c, c->ka, Rz * 4));
  CR_TRY(ensure(c, c->va, Rz * 4));
  CR_TRY(ensure(c, c->kb, Rz * 4));
  CR_TRY(ensure(c, c->vb, Rz * 4));
  CR_TRY(ensure(c, c->offs, Rz * 4));
  CR_TRY(ensure(c, c->slots, Rz * 64));
  CR_TRY(ensure(c, c->rows8, Rz));
  CR_TRY(ensure(c, c->biglist, Rz * 4));
  // stored union rows for up to 1/64 of the records (0.66 % are big at config C)
  const size_t bcap = std::max<size_t>(4096, Rz / 64);
  CR_TRY(ensure(c, c->bigcnt, bcap * kStoreRows * 4));
  CR_TRY(ensure(c, c->bigmask, bcap * kStoreRows * 8));
  CR_TRY(ensure(c, c->bigwlo, bcap * kStoreRows * 4));
  CR_TRY(ensure(c, c->biginfo, bcap * 4));
  const BigRows bigrows{P_<uint32_t>(c->bigcnt), P_<unsigned long long>(c->bigmask),
                        P_<int>(c->bigwlo), P_<int>(c->biginfo), (uint32_t)bcap};
  int G = 1;
  while (G < s) G <<= 1;
  const unsigned bin_grid = (unsigned)(148 * 8);
  const size_t cam_smem = (size_t)N * kCamStride * sizeof(float);  // cameras staged per CTA
  uint32_t nvis = 0;
  uint32_t drange_h[2] = {0u, 0u};
  int kbits = 0;  // bits of the cluster id in the compressed presort key
  while ((1 << kbits) < K) ++kbits;
  if (M > 0) {
    const unsigned g = grid_for(M, 128);
#define CR_PRE(D)                                                                               \
  if (c->motion_bound) CR_PRE2(D, true); else CR_PRE2(D, false)
#define CR_PRE2(D, MBV)                                                                         \
  k_preprocess<D, MBV><<<g, 128, 0, str>>>(P_<float4>(c->mean4), P_<float4>(c->cov8),               \
                                      P_<float>(c->shsoa), P_<float4>(c->rec0),                 \
                                      P_<float4>(c->rec0) + 1, P_<float4>(c->geom),                 \
                                      P_<uint32_t>(c->dkey), P_<uint32_t>(c->vis), counters, sc + 16)
    switch (c->deg) {
      case 0: CR_PRE(0); break;
      case 1: CR_PRE(1); break;
      case 2: CR_PRE(2); break;
      default: CR_PRE(3); break;
    }
#undef CR_PRE
#undef CR_PRE2
    CR_LAUNCHED(c);
    CR_TRACE(c, "preprocess");
    // visible (i,k) records straight to presort (key, r) pairs, (k, i) order
    CR_TRY(dev_scan(c, Scan::InArr{P_<uint32_t>(c->vis)},
                    Scan::OutCompactVis{P_<uint32_t>(c->dkey), P_<uint32_t>(c->ka),
                                        P_<uint32_t>(c->va), sc + 16, kbits},
                    R, sc + 0));
    uint32_t hw[18];
    CR_TRY(read_words(c, sc, hw, 18));  // nvis and the depth-bit range in one read
    nvis = hw[0];
    drange_h[0] = hw[16];
    drange_h[1] = hw[17];
    CR_TRACE(c, "compaction");
  }
  CR_CUDA(c, cudaEventRecord(c->ev[1], str));

  // ---- a7 depth presort: stable by depth bits (4 passes), then by k (1 pass)
  uint32_t *kA = P_<uint32_t>(c->ka), *vA = P_<uint32_t>(c->va);
  uint32_t *kB = P_<uint32_t>(c->kb), *vB = P_<uint32_t>(c->vb);
  int key_bits = 32;
  bool compressed = false;
  if (nvis > 0) {
    const uint32_t span = drange_h[1] - drange_h[0];
    int B = 1;
    while (B < 32 && (span >> B)) ++B;
    if (B + kbits <= 32) { compressed = true; key_bits = B + kbits; }
  }
  CR_TRY(radix_sort(c, kA, vA, kB, vB, nvis, 0, (key_bits + 7) / 8));
  if (!compressed && K > 1) {  // key did not fit: stable cluster pass on top
    CR_TRY(radix_pass(c, kA, vA, kB, vB, nvis, 0, true, (unsigned long long)M, false));
    std::swap(vA, vB);
  }
  const uint32_t* rec_sorted = vA;  // (k, depth, i)-ordered record indices r
  CR_TRACE(c, "depth presort");
  CR_CUDA(c, cudaEventRecord(c->ev[2], str));

  // ---- a6 offsets + emit
  uint32_t P = 0;
  int tbits = 1;
  while ((1LL << tbits) < (long long)TX * TY) ++tbits;
  const int tpass = (tbits + 7) / 8;
  if (nvis > 0) {
    // count in (k, depth, i) order: position-indexed counts and union slots
    // k_countv: 16 blocks per resident slot, so the grid-stride tail is short
    // (measured at config C: binning 6.38 ms at 148 x 8 blocks, 6.27 at x16,
    // 6.20 at x32, 6.14 at x64, 6.18 at x128); small frames: no more blocks
    // than 64-record blocks of work
    const unsigned count_grid =
        (unsigned)std::min<long long>(148 * 64, std::max<long long>(148, ((long long)nvis + 63) / 64));
#define CR_COUNTL(GL, VL)                                                                      \
  do {                                                                                          \
    allow_dyn_smem<k_countv<GL, VL>>();                                                         \
    k_countv<GL, VL><<<count_grid, kBinThreads, cam_smem, str>>>(                               \
        rec_sorted, nvis, P_<float4>(c->mean4), P_<float4>(c->geom), P_<uint32_t>(c->cnt),      \
        P_<uint4>(c->slots), P_<uint8_t>(c->rows8), P_<uint32_t>(c->biglist), sc + 6);          \
  } while (0)
  // lanes per record x views per lane (measured at C, s = 8: 4 x 2 -> 2 x 4 lanes/views
  // took binning 5.65 -> 5.28 ms, s = 4: 4 x 1 -> 2 x 2 7.29 -> 6.21 ms, s = 2: 2 x 1 ->
  // 1 x 2 9.46 -> 8.70 ms; P2K s = 16:
  // 4 x 4 no faster than 8 x 2; P4K s = 18: 8 x 3 instead of 16 x 2, 9.2 -> 8.3 ms)
#define CR_COUNTS(GG)                                                                         \
  if (GG == 32 && s <= 24) CR_COUNTL(8, 3);                                                   \
  else if (GG == 8) CR_COUNTL(2, 4);                                                          \
  else if (GG == 4) CR_COUNTL(2, 2);                                                          \
  else if (GG == 2) CR_COUNTL(1, 2);                                                          \
  else if (GG >= 8) CR_COUNTL((GG >= 8 ? GG / 2 : 1), 2);                                     \
  else CR_COUNTL(GG, 1);                                                                      \
  CR_LAUNCHED(c);                                                                             \
  allow_dyn_smem<k_count_big<GG>>();                                                          \
  k_count_big<GG><<<bin_grid, kBinThreads, cam_smem, str>>>(                                   \
      P_<uint32_t>(c->biglist), rec_sorted, sc + 6, P_<float4>(c->mean4), P_<float4>(c->geom), \
      P_<uint32_t>(c->cnt), bigrows)
    switch (G) {
      case 1: CR_COUNTS(1); break;
      case 2: CR_COUNTS(2); break;
      case 4: CR_COUNTS(4); break;
      case 8: CR_COUNTS(8); break;
      case 16: CR_COUNTS(16); break;
      default: CR_COUNTS(32); break;
    }
#undef CR_COUNTS
#undef CR_COUNTL
    CR_LAUNCHED(c);
    CR_TRACE(c, "count");
    CR_TRY(dev_scan(c, Scan::InArr{P_<uint32_t>(c->cnt)}, Scan::OutStore{P_<uint32_t>(c->offs)},
                    nvis, sc + 1));
    uint32_t hw[4];
    CR_TRY(read_words(c, sc, hw, 4));
    P = hw[1];
    if (hw[3]) return fail(c, CR_ERR_CAPACITY, "pair count exceeds 2^32-1");
  }
  const size_t Pz = std::max<size_t>(P, 1);
  CR_TRY(ensure(c, c->pta, Pz * 4));
  CR_TRY(ensure(c, c->pva, Pz * 4));
  CR_TRY(ensure(c, c->ptb, Pz * 4));
  CR_TRY(ensure(c, c->pvb, Pz * 4));
  uint32_t *tA = P_<uint32_t>(c->pta), *pA = P_<uint32_t>(c->pva);
  uint32_t *tB = P_<uint32_t>(c->ptb), *pB = P_<uint32_t>(c->pvb);
  if (P > 0) {
    // big-footprint records are emitted on a forked stream, concurrently with
    // k_emit_rows (disjoint output positions); joined before the tile sort.
    // (Launch errors of both are caught by the CR_LAUNCHED below.)
    CR_CUDA(c, cudaEventRecord(c->ev_fork, str));
    CR_CUDA(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    auto launch_rows = [&]() {
      // outputs staged per warp in shared memory, 256 pairs (measured at config
      // C: emission 0.12 ms less than direct per-lane stores; 128 / 384 / 512
      // pairs: 0.07 / 0.11 / 0.09 ms less)
      constexpr int kWB = 256;
      const unsigned eg = (unsigned)std::min<long long>((nvis + 255) / 256, 148 * 16);
      const int sm = 8 * 2 * kWB * 4;
      // software-pipelined block inputs (measured at config C: binning 6.09 ->
      // 5.94 ms; P4K unchanged)
      cudaFuncSetAttribute(k_emit_rows<kWB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      k_emit_rows<kWB, true><<<eg, 256, sm, str>>>(rec_sorted, P_<uint32_t>(c->offs), nvis, P,
                                                   P_<uint4>(c->slots), P_<uint8_t>(c->rows8), tA, pA);
    };
    auto launch_big = [&]() {
#define CR_EMITB(GG)                                                                        \
  allow_dyn_smem<k_emit_big<GG>>();                                                          \
  k_emit_big<GG><<<bin_grid, kBinThreads, cam_smem, c->side>>>(                              \
      rec_sorted, P_<uint32_t>(c->offs), P_<uint32_t>(c->biglist), sc + 6, P_<float4>(c->mean4), \
      P_<float4>(c->geom), tA, pA, bigrows)
      switch (G) {
        case 1: CR_EMITB(1); break;
        case 2: CR_EMITB(2); break;
        case 4: CR_EMITB(4); break;
        case 8: CR_EMITB(8); break;
        case 16: CR_EMITB(16); break;
        default: CR_EMITB(32); break;
      }
#undef CR_EMITB
    };
    // the latency-bound big-record emission first, so its CTAs are resident
    // while k_emit_rows fills the remaining slots (measured: binning 6.53 ->
    // 6.49 ms at config C, 9.87 -> 9.13 ms at P4K, 1.60 -> 1.46 ms at B)
    launch_big();
    launch_rows();
    CR_LAUNCHED(c);
    CR_CUDA(c, cudaEventRecord(c->ev_join, c->side));
    CR_CUDA(c, cudaStreamWaitEvent(str, c->ev_join, 0));
  }
  CR_TRACE(c, "offsets+emit");
  CR_CUDA(c, cudaEventRecord(c->ev[3], str));

  // ---- a7 stable tile sort + a8 ranges
  {
    // digits that span only the band's few tile rows: aggregate their histograms
    unsigned agg = 0;
    for (int sh = 8, q = 1; sh < tbits; sh += 8, ++q)
      if (((long long)(row1 - row0) * TX >> sh) < 64) agg |= 1u << q;
    // 17-bit (8K) tile ids: a 9-bit first digit makes it 2 passes (CR_EXP bit 3: 8-bit digits)
    const int b0 = (tbits == 17 && !(c->exp & 8)) ? 9 : 8;
    const int np = b0 == 9 ? 2 : tpass;
    unsigned agg2 = 0;
    for (int q = 1, sh = b0; sh < tbits; sh += 8, ++q)
      if (((long long)(row1 - row0) * TX >> sh) < 64) agg2 |= 1u << q;
    CR_TRY(radix_sort(c, tA, pA, tB, pB, P, 0, np, b0 == 9 ? agg2 : agg, false, (uint32_t)K, b0));
  }
  const size_t nSE = (size_t)TX * TY * K;
  CR_TRY(ensure(c, c->S, nSE * 4));
  CR_TRY(ensure(c, c->E, nSE * 4));
  CR_CUDA(c, cudaMemsetAsync(c->S.p, 0, nSE * 4, str));
  CR_CUDA(c, cudaMemsetAsync(c->E.p, 0, nSE * 4, str));
  if (P > 0) {
    k_ranges<<<(unsigned)std::min<long long>(grid_for((P + 3) / 4, 256), 148 * 8), 256, 0, str>>>(
        tA, P, P_<uint32_t>(c->S), P_<uint32_t>(c->E));
    CR_LAUNCHED(c);
  }
  CR_TRACE(c, "tile sort+ranges");
  CR_CUDA(c, cudaEventRecord(c->ev[4], str));

  // ---- a9 composite
  void* dst = out;
  const bool async_out = !out_on_device && !st && !fullframe && (o->flags & CR_FLAG_ASYNC_OUT);
  const int aslot = c->aslot;
  if (async_out) {  // this slot's previous host copy must be done before it is rewritten
    CR_TRY(ensure(c, c->astage[aslot], obytes));
    CR_CUDA(c, cudaStreamWaitEvent(str, c->ev_copy[aslot], 0));
    dst = c->astage[aslot].p;
  } else if (!out_on_device) {
    CR_TRY(ensure(c, c->stage_out, obytes));
    dst = c->stage_out.p;
  }
  const unsigned ntile = (unsigned)((row1 - row0) * TX);
  const float4* m4 = P_<float4>(c->mean4);
  const bool count = (o->flags & CR_FLAG_COUNT_EVALS) != 0;
  unsigned long long* evals = counters + 3;
  // grids under ~3 waves of 148 x 10 resident CTAs (narrow row bands): split
  // each tile's chunks over up to 4 CTAs (measured: see DESIGN.md §7)
  // (CR_EXP bit 5: never split, so tests cover both store paths on small frames)
  const int tsplit = (c->exp & 32) ? 1 : (int)std::min<long long>(
      4, std::max<long long>(1, (3LL * 148 * CR_COMP_MINB + ntile - 1) / std::max(1u, ntile)));
#define CR_STAGED1(F, CNT, VAR)                                                                \
  k_composite_staged<F, CNT, kCompWarps, VAR><<<ntile * tsplit, kCompWarps * 32, 0, str>>>(  \
      P_<uint8_t>(c->V), P_<uint16_t>(c->psi), P_<uint32_t>(c->chunks),                       \
      P_<uint32_t>(c->nchunks), c->chunk_stride, P_<uint32_t>(c->S), P_<uint32_t>(c->E), pA, \
      P_<float4>(c->rec0), P_<float4>(c->rec0) + 1, m4, dst, evals, tsplit)
#define CR_PAIRS(F, CNT)                                                                      \
  k_composite_pairs<F, CNT, kCompWarps><<<ntile * tsplit, kCompWarps * 32, 0, str>>>(          \
      P_<uint8_t>(c->V), P_<uint16_t>(c->psi2), P_<uint32_t>(c->chunks),                      \
      P_<uint32_t>(c->nchunks), c->chunk_stride, P_<uint32_t>(c->S), P_<uint32_t>(c->E), pA, \
      P_<float4>(c->rec0), m4, dst, evals, tsplit)
#define CR_STAGED(F, CNT) do { if (pairs) CR_PAIRS(F, CNT); else CR_STAGED1(F, CNT, 0); } while (0)
#define CR_THREAD(F, CNT)                                                                     \
  k_composite_thread<F, CNT><<<ntile, kTileSub, 0, str>>>(                                    \
      P_<uint8_t>(c->V), P_<uint16_t>(c->psi), P_<uint32_t>(c->S), P_<uint32_t>(c->E), pA,    \
      P_<float4>(c->rec0), P_<float4>(c->rec0) + 1, m4, dst, evals)
  const int fmt = o->output_format;
  if (fullframe) {
    // per-view frames [N][rows][W][3]: straight into the caller's buffer for
    // CR_FLAG_VIEW_FRAMES (no interlace), else into the context's buffer
    void* fr = dst;
    if (!view_frames) {
      const size_t fb = (size_t)N * (y1 - y0) * W * 3 * (fmt ? 4 : 1);
      CR_TRY(ensure(c, c->frames, fb));
      fr = c->frames.p;
    }
    const unsigned nb = ntile * (unsigned)N;
    if (fmt == 0)
      k_fullframe<0><<<nb, 256, 0, str>>>(P_<uint32_t>(c->S), P_<uint32_t>(c->E), pA,
                                          P_<float4>(c->rec0), m4, fr);
    else
      k_fullframe<1><<<nb, 256, 0, str>>>(P_<uint32_t>(c->S), P_<uint32_t>(c->E), pA,
                                          P_<float4>(c->rec0), m4, fr);
    if (!view_frames) {
      const long long nsub = (long long)(y1 - y0) * W * 3;
      const unsigned gi = (unsigned)std::min<long long>(grid_for(nsub, 256), 148 * 32);
      if (fmt == 0) k_interlace<0><<<gi, 256, 0, str>>>(P_<uint8_t>(c->V), c->frames.p, dst, y1 - y0);
      else k_interlace<1><<<gi, 256, 0, str>>>(P_<uint8_t>(c->V), c->frames.p, dst, y1 - y0);
    }
  } else if (o->kernel == 0) {
    if (fmt == 0) { if (count) CR_STAGED(0, true); else CR_STAGED(0, false); }
    else          { if (count) CR_STAGED(1, true); else CR_STAGED(1, false); }
  } else {
    if (fmt == 0) { if (count) CR_THREAD(0, true); else CR_THREAD(0, false); }
    else          { if (count) CR_THREAD(1, true); else CR_THREAD(1, false); }
  }
#undef CR_STAGED
#undef CR_PAIRS
#undef CR_STAGED1
#undef CR_THREAD
  CR_LAUNCHED(c);
  CR_TRACE(c, "composite");
  CR_CUDA(c, cudaEventRecord(c->ev[5], str));
  if (async_out) {  // D2H on the copy stream, overlapping the next frame's kernels
    CR_CUDA(c, cudaEventRecord(c->ev_comp[aslot], str));
    CR_CUDA(c, cudaStreamWaitEvent(c->copy, c->ev_comp[aslot], 0));
    CR_CUDA(c, cudaMemcpyAsync(out, dst, obytes, cudaMemcpyDeviceToHost, c->copy));
    CR_CUDA(c, cudaEventRecord(c->ev_copy[aslot], c->copy));
    c->aslot = aslot ^ 1;
  } else if (!out_on_device) {
    CR_CUDA(c, cudaMemcpyAsync(out, dst, obytes, cudaMemcpyDeviceToHost, str));
    CR_CUDA(c, cudaStreamSynchronize(str));
  }
  c->K = K;
  c->bitK = bitK;
  c->P = P;
  c->nvis = nvis;
  c->final_t = tA;
  c->final_v = pA;
  c->has_frame = true;
  if (st) {
    CR_CUDA(c, cudaStreamSynchronize(str));
    std::memset(st, 0, sizeof(*st));
    unsigned long long cnts[4] = {0, 0, 0, 0};
    CR_CUDA(c, cudaMemcpy(cnts, counters, sizeof(cnts), cudaMemcpyDeviceToHost));
    st->pairs = P;
    st->visible_ik = nvis;
    st->culled_near = (int64_t)cnts[0];
    st->culled_degenerate = (int64_t)cnts[1];
    st->culled_opacity = (int64_t)cnts[2];
    st->evals = (int64_t)cnts[3];
    uint32_t nfb = 0;
    CR_CUDA(c, cudaMemcpy(&nfb, sc + 6, 4, cudaMemcpyDeviceToHost));
    st->emit_fallback = (int32_t)nfb;
    st->num_clusters = K;
    st->bit_k = bitK;
    st->launches = c->launches;
    float ms[5];
    for (int q = 0; q < 5; ++q) cudaEventElapsedTime(&ms[q], c->ev[q], c->ev[q + 1]);
    st->ms_preprocess = ms[0];
    st->ms_sort = ms[1] + ms[3];
    st->ms_bin = ms[2];
    st->ms_composite = ms[4];
    cudaEventElapsedTime(&st->ms_total, c->ev[0], c->ev[5]);
    st->device_bytes = c->device_bytes;
  }
  return CR_OK;
}

// ---------------------------------------------------------------- introspection
static cr_status copy_out(cr_ctx* c, void* dst, const void* src, size_t count, size_t elt,
                          size_t* n) {
  if (!n) return CR_ERR_INVALID_ARG;
  if (!dst) { *n = count; return CR_OK; }
  if (*n < count) return fail(c, CR_ERR_INVALID_ARG, "capacity %zu < %zu", *n, count);
  if (count) {
    CR_CUDA(c, cudaStreamSynchronize(c->stream));
    CR_CUDA(c, cudaMemcpy(dst, src, count * elt, cudaMemcpyDeviceToHost));
  }
  *n = count;
  return CR_OK;
}

cr_status cr_get_view_map(cr_ctx* c, uint8_t* dst, size_t* n) {
  if (!c) return CR_ERR_INVALID_ARG;
  if (!c->has_display) return fail(c, CR_ERR_NOT_READY, "no display");
  cudaSetDevice(c->device);
  return copy_out(c, dst, c->V.p, (size_t)c->disp.width * c->disp.height * 3, 1, n);
}

cr_status cr_get_remap(cr_ctx* c, uint16_t* dst, size_t* n) {
  if (!c) return CR_ERR_INVALID_ARG;
  if (!c->has_display) return fail(c, CR_ERR_NOT_READY, "no display");
  cudaSetDevice(c->device);
  return copy_out(c, dst, c->psi.p, (size_t)c->TX * c->TY * kTileSub, 2, n);
}

cr_status cr_get_sorted_pairs(cr_ctx* c, uint64_t* keys, uint32_t* pay, size_t* n) {
  if (!c || !n) return CR_ERR_INVALID_ARG;
  if (!c->has_frame) return fail(c, CR_ERR_NOT_READY, "no frame rendered");
  if (!keys || !pay) { *n = c->P; return CR_OK; }
  if (*n < c->P) return fail(c, CR_ERR_INVALID_ARG, "capacity");
  cudaSetDevice(c->device);
  if (c->P) {
    DevBuf kb, pb;
    CR_TRY(ensure(c, kb, (size_t)c->P * 8));
    cr_status s = ensure(c, pb, (size_t)c->P * 4);
    if (s != CR_OK) { release(kb); return s; }
    k_make_keys<<<grid_for(c->P, 256), 256, 0, c->stream>>>(
        c->final_t, c->final_v, P_<uint32_t>(c->dkey), c->P, P_<unsigned long long>(kb),
        P_<uint32_t>(pb));
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = cudaMemcpy(keys, kb.p, (size_t)c->P * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(pay, pb.p, (size_t)c->P * 4, cudaMemcpyDeviceToHost);
    c->device_bytes -= (long long)(kb.bytes + pb.bytes);
    release(kb);
    release(pb);
    if (e != cudaSuccess) return fail(c, CR_ERR_CUDA, "get_sorted_pairs: %s", cudaGetErrorString(e));
  }
  *n = c->P;
  return CR_OK;
}

cr_status cr_get_ranges(cr_ctx* c, uint32_t* S, uint32_t* E, size_t* n) {
  if (!c || !n) return CR_ERR_INVALID_ARG;
  if (!c->has_frame) return fail(c, CR_ERR_NOT_READY, "no frame rendered");
  const size_t cnt = (size_t)c->TX * c->TY * c->K;
  if (!S || !E) { *n = cnt; return CR_OK; }
  size_t cap = *n;
  CR_TRY(copy_out(c, S, c->S.p, cnt, 4, n));
  *n = cap;
  return copy_out(c, E, c->E.p, cnt, 4, n);
}

cr_status cr_get_depths(cr_ctx* c, float* dst, size_t* n) {
  if (!c) return CR_ERR_INVALID_ARG;
  if (!c->has_frame) return fail(c, CR_ERR_NOT_READY, "no frame rendered");
  cudaSetDevice(c->device);
  return copy_out(c, dst, c->dkey.p, (size_t)c->K * c->M, 4, n);
}

cr_status cr_get_counts(cr_ctx* c, uint32_t* dst, size_t* n) {
  if (!c) return CR_ERR_INVALID_ARG;
  if (!c->has_frame) return fail(c, CR_ERR_NOT_READY, "no frame rendered");
  cudaSetDevice(c->device);
  if (dst) {  // |T_{i,k}| recovered from the emitted pairs (payload r); cnt is per list position
    const size_t R = (size_t)c->K * c->M;
    CR_TRY(ensure(c, c->cnt, std::max<size_t>(R, 1) * 4));
    CR_CUDA(c, cudaMemsetAsync(c->cnt.p, 0, R * 4, c->stream));
    if (c->P > 0) {
      k_pair_counts<<<grid_for(c->P, 256), 256, 0, c->stream>>>(c->final_v, c->P,
                                                               P_<uint32_t>(c->cnt));
      CR_LAUNCHED(c);
    }
  }
  return copy_out(c, dst, c->cnt.p, (size_t)c->K * c->M, 4, n);
}

}  // extern "C"
