// dts_lib.cu -- libdts.so: C ABI (include/dts.h), EDA table build, the
// persistent render kernel and the debug kernel for sm_100a.
//
// Design: one lane per path, persistent CTAs (one per SM
// while the 16-bit EDA table is resident in shared memory), warp-level lane
// refill from a warp-private chunk of a global work counter, per-path
// accumulation in a register and ONE fp32 RED per path into the caller's
// histogram (PAPER.md:373 per-bin dedicated paths: a path only ever lands in
// its own cell).  No tensor cores: nothing on this path is a dense contraction.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dts.h"
#include "dts_device.cuh"
#include "fastdiv.h"

using namespace dts;

// ============================================================== error handling
static thread_local std::string g_last_error;
static thread_local int g_last_launches = 0, g_last_grid = 0, g_last_block = 0, g_last_smem = 0;

static dts_status fail(dts_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return fail(DTS_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kHostBands = 4;  // dts_render_host row bands for large histograms

// ============================================================== device buffer pool
// The large library-owned buffers (hand-off records, dts_render_host's device
// histogram: gigabytes for config 5) are returned here when a scene is destroyed
// and handed to the next scene of the same device that needs as much, so an
// application that creates a scene per frame (bench.py's e2e leg) does not pay
// a cudaMalloc / cudaFree of tens of GB per frame.  Pooled bytes per device are
// capped (kPoolCap); the rest is freed.
namespace {
struct PoolBuf {
  int dev;
  void* p;
  size_t bytes;
};
std::mutex g_pool_mu;
std::vector<PoolBuf> g_pool;
constexpr size_t kPoolCap = (size_t)96 << 30;

// a buffer of >= bytes on device dev (the smallest pooled one that fits, else cudaMalloc)
cudaError_t pool_get(int dev, size_t bytes, void** out, size_t* got) {
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    int best = -1;
    for (int i = 0; i < (int)g_pool.size(); ++i)
      if (g_pool[i].dev == dev && g_pool[i].bytes >= bytes && (best < 0 || g_pool[i].bytes < g_pool[best].bytes))
        best = i;
    if (best >= 0) {
      *out = g_pool[best].p;
      *got = g_pool[best].bytes;
      g_pool.erase(g_pool.begin() + best);
      return cudaSuccess;
    }
  }
  *got = bytes;
  return cudaMalloc(out, bytes);
}

// returns a buffer to the pool (the caller has synchronised its last use)
void pool_put(int dev, void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  size_t held = 0;
  for (const PoolBuf& b : g_pool)
    if (b.dev == dev) held += b.bytes;
  if (held + bytes > kPoolCap) {
    cudaFree(p);
    return;
  }
  g_pool.push_back(PoolBuf{dev, p, bytes});
}
}  // namespace

struct dts_scene {
  dts_scene_desc desc;
  DevScene S;
  uint16_t* d_table = nullptr;
  size_t table_n = 0;
  double* d_table_f = nullptr;     // table build scratch: fp64 bin integrals (table_f_kernel)
  size_t table_f_n = 0;
  // the table build runs on its own stream, forked from the caller's; table
  // readers (render, debug) wait for tab_ready (table_wait)
  cudaStream_t tab_stream = nullptr;
  cudaEvent_t tab_fork = nullptr, tab_ready = nullptr;
  bool tab_async = false;
  unsigned long long* d_work = nullptr;  // global work counter
  float* d_hist_host = nullptr;          // dts_render_host scratch
  size_t d_hist_host_n = 0;              // its capacity in floats
  uint64_t* d_ctr_host = nullptr;
  uint32_t* d_resp_cdf = nullptr;  // R31 bin CDF (n_bins + 1)
  float* d_resp_wgt = nullptr;     // W_b / pi_b
  float* d_resp_w = nullptr;       // W_b
  uint16_t* d_zero_cell = nullptr; // debug kernel table for vanilla scenes
  float* d_qover = nullptr;        // deferred-connection queue overflow slots
  size_t qover_n = 0;
  cudaStream_t band_stream[2] = {nullptr, nullptr};  // dts_render_host row bands
  cudaEvent_t band_ev[kHostBands + 1] = {};
  unsigned long long* d_work_band = nullptr;
  // two-stage render: hand-off buffer and 3 counters (walk work, connect work,
  // slots) per launch slot: 0 = dts_render, 1 + band = row-band launches
  // (dts_render's slot 0 holds two halves: consecutive chunks alternate between
  // them and between the caller's stream and wf_stream, so each chunk's connect-
  // stage tail overlaps the next chunk's walk stage)
  struct HandOff* d_ho[1 + kHostBands] = {};
  size_t ho_cap[1 + kHostBands] = {};
  unsigned long long* d_wf = nullptr;
  cudaStream_t wf_stream = nullptr;
  cudaEvent_t wf_ev[2] = {};
  float4* d_bvh = nullptr;         // mesh BVH nodes (R32)
  float4* d_tri4 = nullptr;        // mesh triangles in leaf order
  int32_t* d_tri_map = nullptr;    // caller -> leaf order, then leaf -> caller order (2 n_tris)
  int num_sms = 0;
  int device = 0;
  int live[4] = {0, 0, 0, 0};  // pixels [x0, x1) x [y0, y1) outside which every camera ray misses (live_rect)
};

// a stream about to run a kernel that reads the EDA table waits for its build
static cudaError_t table_wait(dts_scene* s, cudaStream_t st) {
  return s->tab_async ? cudaStreamWaitEvent(st, s->tab_ready, 0) : cudaSuccess;
}

// ============================================================== EDA table build (fp64, R9/R10)
__constant__ double kGLx8[8] = {-0.9602898564975362, -0.7966664774136267, -0.525532409916329, -0.18343464249564978,
                                0.18343464249564978, 0.525532409916329,   0.7966664774136267, 0.9602898564975362};
__constant__ double kGLw8[8] = {0.10122853629037706, 0.22238103445337443, 0.3137066458778869, 0.36268378337836166,
                                0.36268378337836166, 0.3137066458778869,  0.22238103445337443, 0.10122853629037706};

struct TableParams {
  double sigma_s, sigma_a, sigma_t, D, norm;
  double smin, smax;
  int nr, ns;
};

// E17 for one cos(theta): sigma_s * int_0^{t_M} e^{-sigma_t t} Phi(x + w t, S - t) dt
// (emitter at the far focus, distance C), cut at 40/sigma_t, split at the
// closest approach t = C cos, 4 panels x 8-point Gauss-Legendre per part.
__device__ double e17_integrand(const TableParams& P, double C, double S, double cth) {
  const double tM = (S - C) * (S + C) / (2.0 * (S - C * cth));
  const double tend = fmin(tM, 40.0 / P.sigma_t);
  const double tc = C * cth;
  double cuts[3];
  int nc = 0;
  cuts[nc++] = 0.0;
  if (tc > 0.0 && tc < tend) cuts[nc++] = tc;
  cuts[nc++] = tend;
  const double k = 1.0 / (4.0 * P.D);
  double total = 0.0;
  for (int part = 0; part + 1 < nc; ++part) {
    const double a = cuts[part], h = (cuts[part + 1] - a) * 0.25;
    double sum = 0.0;
    for (int panel = 0; panel < 4; ++panel) {
      const double pa = a + panel * h;
      for (int i = 0; i < 8; ++i) {
        const double t = pa + 0.5 * h * (1.0 + kGLx8[i]);
        const double r2 = t * t - 2.0 * t * C * cth + C * C;
        const double dt = S - t;
        // e^{-sigma_t t} Phi(r, dt) / norm: one exp of the summed exponents, one
        // division and one rsqrt (dt^{-3/2} = (1/dt) dt^{-1/2})
        if (dt > 0.0) {
          const double idt = 1.0 / dt;
          sum += kGLw8[i] * exp(-P.sigma_t * t - r2 * k * idt - P.sigma_a * dt) * idt * rsqrt(dt);
        }
      }
    }
    total += 0.5 * h * sum;
  }
  return P.sigma_s * P.norm * total;  // norm = (4 pi D)^{-3/2}
}

// Two kernels.  table_f_kernel: grid = 4 x cells, block = 256 (a quarter of a
// cell's 64 cos bins per CTA): four threads per cos bin, two of its eight
// cos-direction Gauss-Legendre nodes each, summed by two shuffles -> F (fp64,
// global scratch).  Small CTAs spread the fp64 work evenly over the SMs (one
// 1024-thread CTA per cell left some SMs with two cells and others with one;
// DESIGN.md 5.3).  table_cdf_kernel: grid = cells, block = 256: the cell's
// quantised CDF (serial sums in bin order, as the oracle) and its guide row.
constexpr int kTableThreads = 256;
__global__ void __launch_bounds__(kTableThreads) table_f_kernel(TableParams P, double* __restrict__ F) {
  const int cell = blockIdx.x >> 2;
  const int ir = cell / P.ns, is = cell % P.ns;
  const double ratio = (ir + 0.5) / P.nr;
  const double S = P.smin * pow(P.smax / P.smin, (is + 0.5) / P.ns);
  const double C = ratio * S;
  const int bin = (blockIdx.x & 3) * 64 + (threadIdx.x >> 2), part = threadIdx.x & 3;
  const double dc = 2.0 / 256.0;
  const double c0 = -1.0 + bin * dc;
  double acc = 0.0;
  for (int n = 2 * part; n < 2 * part + 2; ++n)
    acc += 0.5 * dc * kGLw8[n] * e17_integrand(P, C, S, c0 + 0.5 * dc * (1.0 + kGLx8[n]));
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  if (part == 0) F[(size_t)cell * 256 + bin] = acc;
}
__global__ void __launch_bounds__(256) table_cdf_kernel(const double* __restrict__ Fg, uint16_t* __restrict__ q,
                                                        size_t n_total) {
  __shared__ double F[256], Cd[256];
  __shared__ double s_total;
  __shared__ uint16_t Q[256];
  const int cell = blockIdx.x;
  const int j = threadIdx.x;
  F[j] = Fg[(size_t)cell * 256 + j];
  __syncthreads();
  // the oracle's operations in its order (total, then cdf_i = sum_{k<i} F_k / total
  // accumulated in bin order); only the divisions, which are independent, and the
  // quantisation run on all 256 threads (the serial chains are fp64 adds only)
  if (j == 0) {
    double total = 0.0;
    for (int i = 0; i < 256; ++i) total += F[i];
    s_total = total;
  }
  __syncthreads();
  const double pj = F[j] / s_total;
  __syncthreads();
  F[j] = pj;
  __syncthreads();
  if (j == 0) {
    double cdf = 0.0;
    for (int i = 0; i < 256; ++i) {
      Cd[i] = cdf;
      cdf += F[i];
    }
  }
  __syncthreads();
  {
    double qv = floor(65536.0 * Cd[j] + 0.5);
    if (qv > 65535.0) qv = 65535.0;
    Q[j] = (uint16_t)qv;
  }
  __syncthreads();
  q[(size_t)cell * 256 + j] = Q[j];
  // guide row (acceleration structure of the same inverse transform):
  // guide[g] = largest i with Q[i] <= 256 g
  int lo = 0, hi = 255;
  const uint32_t key = 256u * (uint32_t)j;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((uint32_t)Q[mid] <= key) lo = mid; else hi = mid - 1;
  }
  reinterpret_cast<uint8_t*>(q + n_total)[(size_t)cell * 256 + j] = (uint8_t)lo;
}

// ============================================================== debug kernel
template <int SH, int FL>
__global__ void debug_kernel(DevScene S, const uint16_t* __restrict__ tab, int n, const dts_debug_in* __restrict__ in,
                             dts_debug_out* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dts_debug_out o;
  memset(&o, 0, sizeof(o));
  o.istar = -1;
  const dts_debug_in rec = in[i];
  if ((FL & FL_MESH) && rec.kind == KIND_SURF && (uint32_t)rec.face >= (uint32_t)S.n_tris) {
    o.terminate = 1;
    out[i] = o;
    return;
  }
  PathState ps;
  ps.x = mk(rec.x[0], rec.x[1], rec.x[2]);
  ps.w = mk(rec.w[0], rec.w[1], rec.w[2]);
  ps.beta = rec.beta;
  ps.kind = rec.kind;
  ps.face = ((FL & FL_MESH) && rec.kind == KIND_SURF) ? S.tri_leaf[rec.face] : rec.face;
  ps.e = rec.emitter;
  const double RM = S.t0 + (double)(rec.bin + 1) * S.dt - (double)S.em_t[rec.emitter];
  ps.resM = RM - rec.E;
  uint32_t r[8];
  for (int k = 0; k < 8; ++k) r[k] = rec.r[k];
  float c;
  bool cn, wn;
  int reason;
  darts_vertex<true, false, SH, FL>(S, tab, ps, r, c, &o, cn, wn, reason);
  if ((FL & FL_MESH) && o.hit == HIT_SURF) o.face_hit = S.tri_orig[o.face_hit];
  o.E_next = RM - ps.resM;
  out[i] = o;
}

// ============================================================== render kernel
struct RenderParams {
  DevScene S;
  const uint16_t* tab;
  float* hist;
  float* hist_sq;
  unsigned long long* counters;
  unsigned long long* work;
  uint64_t total;    // work items of this launch
  uint64_t s_begin;  // first sample index
  uint64_t n_s;      // samples per cell/pixel in this launch
  uint64_t spp;      // samples per cell (PER_CELL) or per pixel
  uint32_t npix;     // pixels of the launch's live rectangle (S.crop[0..1]: its origin; live_rect)
  uint32_t cw;       // its width
  uint32_t hw;       // histogram rows' width in pixels (the launch's crop / band)
  uint32_t ph_base;  // histogram pixel of the live rectangle's first pixel
  uint32_t table_u4; // table size in 16-byte words
  uint32_t spp_div_b, spp_mod_b;  // SPP_PER_PIXEL cell counts (R21)
  const uint32_t* resp_cdf;       // SPP_RESPONSE: bin CDF c_0..c_B (R31)
  const float* resp_wgt;          // SPP_RESPONSE: W_b / pi_b
  const float* resp_w;            // W_b (vanilla weighting; null = rectangle)
  uint32_t priv_cells;            // > 0: the CTA privatises the whole histogram in shared memory
  uint32_t defer;                 // 1: connections are queued per warp and evaluated in batches
  uint32_t flush_at;              // queue length that triggers a batch
  uint32_t flush1_at;             // stage-1 queue length that triggers a batch (SPLIT)
  float* qover;                   // DEFER: global overflow queue slots, kQueue x (kJobWords + kJob1Words) per warp
  uint32_t refill_k;              // idle lane-iterations that trigger a refill
  uint32_t chunk;                 // work items a warp takes from the global counter at a time (32..kChunk)
  uint32_t one_cell_warps;        // 1: per-cell order with >= 32 samples per cell (splat fast path)
  uint32_t splat_plain;           // 2: one RED per retiring lane (default); 0 / 1: in-warp aggregation (-DDTS_SPLAT_AGG=1 builds)
  uint32_t div32;                 // 1: work indices, sample indices + B fit 32 bits (fast divisions)
  uint32_t cells;                 // histogram cells of this launch (< 2^32; bounds checks of the check build)
  uint32_t van_rows;              // vanilla: 1 = pixel-major batches splat into per-warp shared-memory rows
  uint64_t w_base;                // first work index of this launch (two-stage render: the chunk's)
  struct HandOff* ho;             // two-stage render: the chunk's hand-off records
  unsigned long long* ho_count;   // two-stage render: hand-off slots allocated (the connect stage's work count)
  uint64_t ho_cap;                // two-stage render: hand-off slots of the chunk's buffer (bounds checks)
  struct HandOff* ho_in;          // three-stage render (SPLIT): the start stage's records the walk stage continues
  unsigned long long* ho_in_count;  // their count
  FastDiv fd_ns, fd_npix, fd_cw, fd_b;  // division by n_s, npix, cw, n_bins (fastdiv.h)
};

#ifndef DTS_BLOCK
#define DTS_BLOCK 768
#endif
constexpr int kBlock = DTS_BLOCK;  // deferred-connection kernels: the queues take the shared memory
#ifndef DTS_BLOCK_IMM
#define DTS_BLOCK_IMM 896
#endif
// immediate-connection kernels: 28 warps at <= 72 registers (A/B in profiles/README.md)
constexpr int kBlockImm = DTS_BLOCK_IMM;
// mesh kernels (BVH traversal state: more live values) run 768 threads at <= 80 registers
// (A/B: +2 % / +3.5 % on config 6 with 336 / 81936 triangles against 640)
#ifndef DTS_BLOCK_MESH
#define DTS_BLOCK_MESH 768
#endif
constexpr int kBlockMesh = DTS_BLOCK_MESH;
// connect stage of a REUSE scene's start-stage render (no camera vertices):
// 32 warps at <= 64 registers (A/B against 896: config 2 +0.7 %, config 4 +0.8 %,
// profiles/ab_r02v_nocam_block.log)
#ifndef DTS_BLOCK_RESUME_REUSE
#define DTS_BLOCK_RESUME_REUSE 1024
#endif
constexpr int kBlockResReuse = DTS_BLOCK_RESUME_REUSE;
__host__ __device__ constexpr int render_block(bool defer, bool mesh = false, bool resume_reuse = false) {
  return mesh ? kBlockMesh : (defer ? kBlock : (resume_reuse ? kBlockResReuse : kBlockImm));
}
constexpr uint32_t kChunk = 128;  // work items per global-counter grab (P.chunk: 32..kChunk)
#ifndef DTS_RIS_WARP
#define DTS_RIS_WARP 0
#endif
// RIS layout: A = lane per path, 8 candidates in registers
// (default); B = warp-collective 8-lane groups with shuffle scan/selection.
constexpr bool kRisWarp = DTS_RIS_WARP != 0;
#ifndef DTS_INNER
#define DTS_INNER 1
#endif
constexpr int kInner = DTS_INNER;  // vertices per lane between refill checks
constexpr size_t kPrivMaxCells = 4096;  // histograms up to 16 KiB are privatised per CTA

struct PathCtx {
  PathState ps;
  uint32_t id_lo, id_hi;
  uint32_t k;
  uint32_t cell;  // histogram cell (crop-local)
  float inv_n;
  float acc;
};

// decode a work index into a path (returns false if the path retires at start)
template <int SH, int FL>
__device__ __forceinline__ bool start_path(const RenderParams& P, uint64_t widx, PathCtx& pc,
                                           uint32_t* s_ctr) {
  const DevScene& S = P.S;
  const uint32_t B = (uint32_t)S.n_bins;
  uint64_t s;
  uint32_t pl, b;
  uint64_t id;
  const uint64_t Npix = (uint64_t)S.width * (uint64_t)S.height;
  float inv_n;
  uint32_t cx, cy;
  if (S.spp_mode == DTS_SPP_PER_CELL) {
    // issue order (b descending, pixel, s): long late-bin walks first
    uint64_t sl, rest;
    if (P.div32) {  // 32-bit divisions by launch invariants when the launch allows
      uint32_t sl32, pl32;
      const uint32_t rest32 = fastdiv_divmod((uint32_t)widx, P.fd_ns, sl32);
      b = B - 1u - fastdiv_divmod(rest32, P.fd_npix, pl32);
      sl = sl32;
      pl = pl32;
    } else {
      sl = widx % P.n_s;
      rest = widx / P.n_s;
      pl = (uint32_t)(rest % P.npix);
      b = B - 1u - (uint32_t)(rest / P.npix);
    }
    s = P.s_begin + sl;
    inv_n = 1.0f / (float)P.spp;
  } else {
    if (P.div32) {
      s = P.s_begin + fastdiv_divmod((uint32_t)widx, P.fd_npix, pl);
    } else {
      pl = (uint32_t)(widx % P.npix);
      s = P.s_begin + widx / P.npix;
    }
  }
  cy = fastdiv_divmod(pl, P.fd_cw, cx);
  const uint32_t px = (uint32_t)S.crop[0] + cx, py = (uint32_t)S.crop[1] + cy;
  const uint64_t p = (uint64_t)py * (uint64_t)S.width + px;
  pl = P.ph_base + cy * P.hw + cx;  // the histogram's pixel
  float scale = 1.0f;
  if (S.spp_mode == DTS_SPP_PER_CELL) {
    id = (s * Npix + p) * (uint64_t)B + b;
  } else if (S.spp_mode == DTS_SPP_RESPONSE) {
    // R31: bin b with c_b <= m < c_{b+1} (m = 23 bits of the path-start draw's
    // 4th word), weight W_b / pi_b; every path of the pixel samples each cell
    id = s * Npix + p;
    const u4 a0 = philox_rk((uint32_t)id, (uint32_t)(id >> 32), 0xFFFFFFFFu, 0u, S.rk);
    const uint32_t m = a0.d >> 9;
    int lo = 0, hi = (int)B - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      DTS_CHECK(mid > 0 && mid <= (int)B);
      if (__ldg(P.resp_cdf + mid) <= m) lo = mid; else hi = mid - 1;
    }
    b = (uint32_t)lo;
    scale = __ldg(P.resp_wgt + b);
    inv_n = 1.0f / (float)P.spp;
  } else {
    // R21: bin = (s + o_p) mod B with a per-pixel Philox offset
    const u4 o = philox_rk((uint32_t)p, (uint32_t)(p >> 32), 0xFFFFFFFEu, 0u, S.rk);
    const uint32_t op = unif_index(B, o.a);
    // b = (s + op) mod B; the cell's rank rel = (b - op) mod B = s mod B
    uint32_t rel;
    if (P.div32) fastdiv_divmod((uint32_t)s, P.fd_b, rel);
    else rel = (uint32_t)(s % B);
    b = rel + op >= B ? rel + op - B : rel + op;
    const uint32_t n_pb = P.spp_div_b + (rel < P.spp_mod_b ? 1u : 0u);
    inv_n = 1.0f / (float)n_pb;
    id = s * Npix + p;
  }
  pc.id_lo = (uint32_t)id;
  pc.id_hi = (uint32_t)(id >> 32);
  pc.k = 0;
  pc.cell = pl * B + b;
  pc.inv_n = inv_n;
  pc.acc = 0.0f;
  const u4 a = philox_rk(pc.id_lo, pc.id_hi, 0xFFFFFFFFu, 0u, S.rk);
  const int e = (FL & FL_MULTI_E) ? (int)unif_index((uint32_t)S.n_emitters, a.c) : 0;
  PathState& ps = pc.ps;
  ps.e = e;
  if (S.camera_kind == DTS_CAMERA_PINHOLE) {
    const float sx = (__fdividef(2.0f * ((float)px + unif(a.a)), (float)S.width) - 1.0f) * S.tan_half * S.aspect;
    const float sy = (1.0f - __fdividef(2.0f * ((float)py + unif(a.b)), (float)S.height)) * S.tan_half;
    f3 w = mk(S.fwd[0] + sx * S.right[0] + sy * S.upc[0], S.fwd[1] + sx * S.right[1] + sy * S.upc[1],
              S.fwd[2] + sx * S.right[2] + sy * S.upc[2]);
    ps.w = w * rsqrtf(dot(w, w));
    ps.x = ld3(S.cam_pos);
    ps.beta = 1.0f;
  } else {
    const u4 bb = philox_rk(pc.id_lo, pc.id_hi, 0xFFFFFFFFu, 1u, S.rk);
    const u4 cc = philox_rk(pc.id_lo, pc.id_hi, 0xFFFFFFFFu, 2u, S.rk);
    const float rad = S.det_radius * cbrtf(unif(bb.a));
    const float z = 1.0f - 2.0f * unif(bb.b);
    const float sz = sqrtf(fmaxf(0.0f, 1.0f - z * z));
    float sp, cp;
    __sincosf(2.0f * kPi * unif(bb.c), &sp, &cp);
    ps.x = mk(S.cam_pos[0] + rad * sz * cp, S.cam_pos[1] + rad * sz * sp, S.cam_pos[2] + rad * z);
    const float z2 = 1.0f - 2.0f * unif(bb.d);
    const float s2 = sqrtf(fmaxf(0.0f, 1.0f - z2 * z2));
    __sincosf(2.0f * kPi * unif(cc.a), &sp, &cp);
    ps.w = mk(s2 * cp, s2 * sp, z2);
    ps.beta = 4.0f * kPi;
  }
  ps.beta *= scale;
  ps.kind = KIND_CAMERA;
  ps.face = -1;
  ps.resM = S.t0 + (double)(b + 1) * S.dt - (double)S.em_t[e];  // R_M - E with E = 0
  float lo, hi;
  int f;
  if (intersect<SH, (FL & FL_WALLS) != 0>(S, ps.x, ps.w, lo, hi, f) == HIT_MISS) {
    atomicAdd(s_ctr + DTS_CTR_CAMERA_MISS, 1u);
    return false;
  }
  if (S.warped || S.camera_kind == DTS_CAMERA_SPHERE_DETECTOR) {
    const f3 dv = ps.x - ld3(S.em_pos[e]);
    if (sqrtf(dot(dv, dv)) >= d2f(ps.resM)) {
      atomicAdd(s_ctr + DTS_CTR_EARLY_EXIT, 1u);
      return false;
    }
  }
  return true;
}

// ---------------------------------------------------------------- persistent work distribution
// Hands the lanes of `need` (warp-uniform mask) consecutive work items from the
// warp's private queue [wn, we), refilled with `chunk` (>= 32) items from the
// global counter `work` (one atomicAdd per chunk); returns this lane's item, ~0
// if it gets none (then `exhausted` is set: the global range is used up).
// (hand-off prefetch on grabs: measured -0.35 % on config 5, within +-0.3 % on
// configs 2, 3, 4 -- the refill loads were not what stalls the connect stage;
// off by default: profiles/ab_r02x_ho_prefetch.log)
#ifndef DTS_HO_PREFETCH
#define DTS_HO_PREFETCH 0
#endif
// L2 prefetch of a byte range by the TMA unit (no registers, no completion to wait for)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// (pf: the hand-off records when the work items are hand-off slots (64 bytes
// each): a grab prefetches its records into L2, so the later refills from the
// chunk load them from L2 instead of HBM)
__device__ __forceinline__ uint64_t take_work(unsigned need, int lane, unsigned lt_mask, uint64_t& wn, uint64_t& we,
                                              bool& exhausted, unsigned long long* work, uint64_t ntotal,
                                              uint32_t chunk, const char* pf = nullptr) {
  const uint32_t nidle = __popc(need);
  const uint32_t rank = __popc(need & lt_mask);
  const uint64_t avail = we - wn;
  uint64_t my = ~0ull;
  if (avail >= nidle) {
    my = wn + rank;
    wn += nidle;
  } else {
    unsigned long long nb = 0;
    if (lane == 0) nb = atomicAdd(work, (unsigned long long)chunk);
    nb = __shfl_sync(0xffffffffu, nb, 0);
    uint64_t ne = nb + chunk < ntotal ? nb + chunk : ntotal;
    if (nb >= ntotal) {
      exhausted = true;
      ne = nb;
    }
    if (rank < avail) {
      my = wn + rank;
    } else {
      const uint64_t cand = nb + (rank - avail);
      my = cand < ne ? cand : ~0ull;
    }
    const uint64_t nq = nb + (nidle - avail);
    wn = nq < ne ? nq : ne;
    we = ne;
    if (DTS_HO_PREFETCH && pf && lane == 0 && ne > nb) prefetch_l2_bulk(pf + nb * 64u, (uint32_t)((ne - nb) * 64u));
  }
  return ((need >> lane) & 1u) ? my : ~0ull;
}
#ifndef DTS_START_TRIES
#define DTS_START_TRIES 1
#endif
// start attempts per refill for a lane whose path retires at its start: 1 (A/B,
// profiles/ab_r02_start_tries.log: 8 tries cost 0.5-5 % on configs 1, 2, 4, 6)
constexpr int kStartTries = DTS_START_TRIES;

// ---------------------------------------------------------------- TMA 1-D bulk staging
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Copies `bytes` (multiple of 16, both addresses 16-byte aligned) from global
// to shared memory with cp.async.bulk (the TMA unit's non-tensor mode), one
// elected thread issuing, completion tracked by an mbarrier transaction count;
// every thread of the CTA returns once the data has landed.
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    constexpr uint32_t kPiece = 32768;
    for (uint32_t off = 0; off < bytes; off += kPiece) {
      const uint32_t n = bytes - off < kPiece ? bytes - off : kPiece;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(static_cast<char*>(dst) + off)),
                   "l"(static_cast<const char*>(src) + off), "r"(n), "r"(b)
                   : "memory");
    }
  }
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(b)
      : "memory");
}

// ---------------------------------------------------------------- histogram splat (step 4)
// Per-bin dedicated paths: a retiring path adds its whole
// contribution to its own cell by a RED (splat_retired below): to a shared-
// memory copy of the histogram when the CTA privatises it (small histograms,
// flushed once at kernel end), else to HBM/L2.  The in-warp aggregation that
// follows is the DTS_SPLAT_AGG=1 build option (and the deferred-connection
// kernels' flush): lanes that retire in the same iteration on the same cell are
// combined first (__match_any_sync + shuffles, one RED per distinct cell and warp).
// Every retiring lane of the warp on one cell (per-cell issue order with >= 32
// samples per cell: a warp's paths are mostly consecutive samples of one cell):
// a 5-step butterfly and one RED.  Called by all 32 lanes of a converged warp;
// returns false (nothing done) when the lanes are on several cells.
// (ncells: the launch's histogram cells, for the bounds checks of the check build)
__device__ __forceinline__ bool splat_one_cell(unsigned dmask, bool done, uint32_t cell, float v, float v2,
                                               float* g_hist, float* g_sq, float* s_hist, float* s_sq, int lane,
                                               uint32_t ncells) {
  const int first = __ffs(dmask) - 1;
  const uint32_t c0 = __shfl_sync(0xffffffffu, cell, first);
  if (!__all_sync(0xffffffffu, !done || cell == c0)) return false;
  const bool sq = (s_hist ? s_sq : g_sq) != nullptr;
  float a = done ? v : 0.0f, a2 = done ? v2 : 0.0f;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    if (sq) a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (lane != first || a == 0.0f) return true;
  DTS_CHECK(c0 < ncells);
  if (s_hist) {
    atomicAdd(s_hist + c0, a);
    if (s_sq) atomicAdd(s_sq + c0, a2);
  } else {
    atomicAdd(g_hist + c0, a);
    if (g_sq) atomicAdd(g_sq + c0, a2);
  }
  return true;
}
__device__ __forceinline__ void splat(unsigned dmask, bool done, uint32_t cell, float v, float v2, float* g_hist,
                                      float* g_sq, float* s_hist, float* s_sq, int lane, uint32_t ncells) {
  if (!done) return;
  const unsigned peers = __match_any_sync(dmask, cell);
  const int leader = __ffs(peers) - 1;
  const int n = __popc(peers);
  const int nmax = __reduce_max_sync(dmask, n);
  unsigned m = peers & (peers - 1u);  // peers above the leader, consumed one per step
  for (int i = 1; i < nmax; ++i) {
    const int src = (lane == leader && m) ? __ffs(m) - 1 : lane;
    const float o = __shfl_sync(dmask, v, src);
    const float o2 = __shfl_sync(dmask, v2, src);
    if (lane == leader && m) {
      v += o;
      v2 += o2;
      m &= m - 1u;
    }
  }
  if (lane != leader || v == 0.0f) return;
  DTS_CHECK(cell < ncells);
  if (s_hist) {
    atomicAdd(s_hist + cell, v);
    if (s_sq) atomicAdd(s_sq + cell, v2);
  } else {
    atomicAdd(g_hist + cell, v);
    if (g_sq) atomicAdd(g_sq + cell, v2);
  }
}

// splat of the lanes retiring in this iteration (dmask): one RED per retiring
// lane with a non-zero contribution, to the CTA's private histogram or to L2.
// Plain REDs beat the in-warp aggregation (one-cell butterfly, then
// __match_any_sync + shuffles, one RED per distinct cell) on every config:
// config 4 +4.9 %, config 2 +4.1 %, config 6 +1.3 %, config 3 +0.9 %, config 5
// +0.2 %, config 1 even (profiles/ab_r02z_splat.log) -- the aggregation cost
// ~1.9 warp-instructions per vertex at SIMT 11 in config 4's connect stage,
// while the L2 absorbs same-address REDs of paths that retire at different
// times.  -DDTS_SPLAT_AGG=1 builds keep the aggregation, selected per launch
// by DTS_SPLAT_PLAIN=0 (aggregate) / 1 (butterfly, else plain) / 2 (plain).
// (A two-cell butterfly variant measured 5 % slower than the aggregation on
// config 4: profiles/ab_r02_start_knobs.log)
#ifndef DTS_SPLAT_AGG
#define DTS_SPLAT_AGG 0
#endif
__device__ __forceinline__ void splat_retired(const RenderParams& P, unsigned dmask, bool done, uint32_t cell, float v,
                                              float v2, float* s_hist, float* s_sq, int lane) {
  if (DTS_SPLAT_AGG && P.splat_plain < 2u) {
    if (P.one_cell_warps && splat_one_cell(dmask, done, cell, v, v2, P.hist, P.hist_sq, s_hist, s_sq, lane, P.cells))
      return;
    if (P.splat_plain == 0u) {
      splat(dmask, done, cell, v, v2, P.hist, P.hist_sq, s_hist, s_sq, lane, P.cells);
      return;
    }
  }
  if (done && v != 0.0f) {
    DTS_CHECK(cell < P.cells);
    if (s_hist) {  // (one branch per address space: a selected pointer compiles to generic atomics)
      atomicAdd(s_hist + cell, v);
      if (s_sq) atomicAdd(s_sq + cell, v2);
    } else {
      atomicAdd(P.hist + cell, v);
      if (P.hist_sq) atomicAdd(P.hist_sq + cell, v2);
    }
  }
}

#ifndef DTS_MINB
#define DTS_MINB 1
#endif
#ifndef DTS_TABLE_SMEM
#define DTS_TABLE_SMEM 1
#endif
// ---------------------------------------------------------------- two-stage render (SPLIT scenes)
// In SPLIT scenes (R29) the walk direction does not depend on the connection,
// so while a path's connections provably cannot reach its bin (conn_margin >
// 0: R_m - E exceeds every S a connection could have) its vertices need only
// the walk.  For config 5 that holds for ~70 % of all vertices, for config 3
// for ~78 %.  The walk stage (walk_kernel) runs those vertices with the walk-
// only darts_vertex<WALK> -- every lane of a warp in the same, cheaper code --
// and hands each surviving path over, at the first vertex that might connect,
// through a 64-byte record in HBM; the connect stage (render_darts_kernel
// <RESUME>) continues the path with full vertices.  Same path ids, same random
// numbers, same vertices: the histogram equals the one-stage render's.
struct __align__(16) HandOff {
  float x[3], beta;
  float w[3];
  uint32_t k;                // next bounce index; 0xFFFFFFFF marks an unused slot
  double resM;
  uint32_t id_lo, id_hi;
  uint32_t cell;
  float inv_n;
  int32_t kind_face_e;       // kind | (face + 1) << 8 | e << 16
  float acc;                 // contribution so far (the start stage's camera vertex; 0 after walk-only vertices)
};
static_assert(sizeof(HandOff) == 64, "hand-off records are 64 bytes");
constexpr uint32_t kHoEmpty = 0xFFFFFFFFu;
constexpr uint32_t kHoBlock = 32;  // hand-off slots a warp reserves at a time

// Lower bound of (R_m - E) - max S of any connection from x: every point y of a
// chord from x satisfies S = |y - x| + |y - x_e| <= (farthest medium point from
// x) + (farthest medium point from any emitter) (may_connect_bound).  A
// connection lands in the bin only if S >= R_m - E, so a positive margin means
// it cannot (nor can the wall NEE: C <= that bound).  fp32 safety: 1e-4
// relative + 1e-3 absolute.  (In a box the exact maximum of S is at a corner;
// that bound moved 0.2 % of config 5's vertices into the walk stage and cost
// more than it saved: profiles/ab_r02_margin_corners.log.)
template <int SH>
__device__ __forceinline__ float conn_margin(const DevScene& S, f3 x, double resM) {
  const float resm = d2f(resM - S.dt);
  float far_x;
  if (SH == DTS_MEDIUM_BOX) {
    const float fx = fmaxf(x.x - S.bmin[0], S.bmax[0] - x.x);
    const float fy = fmaxf(x.y - S.bmin[1], S.bmax[1] - x.y);
    const float fz = fmaxf(x.z - S.bmin[2], S.bmax[2] - x.z);
    far_x = sqrtf(fmaf(fx, fx, fmaf(fy, fy, fz * fz)));
  } else {
    const f3 d = x - ld3(S.center);
    far_x = sqrtf(dot(d, d)) + sqrtf(S.radius2);
  }
  return resm - fmaf(far_x + S.far_e, 1.0001f, 1e-3f);
}

__device__ __forceinline__ void store_handoff(HandOff* ho, const PathCtx& pc) {
  const PathState& ps = pc.ps;
  uint4* d = reinterpret_cast<uint4*>(ho);
  d[0] = make_uint4(__float_as_uint(ps.x.x), __float_as_uint(ps.x.y), __float_as_uint(ps.x.z), __float_as_uint(ps.beta));
  d[1] = make_uint4(__float_as_uint(ps.w.x), __float_as_uint(ps.w.y), __float_as_uint(ps.w.z), pc.k);
  d[2] = make_uint4((uint32_t)__double2loint(ps.resM), (uint32_t)__double2hiint(ps.resM), pc.id_lo, pc.id_hi);
  d[3] = make_uint4(pc.cell, __float_as_uint(pc.inv_n), (uint32_t)(ps.kind | ((ps.face + 1) << 8) | (ps.e << 16)),
                   __float_as_uint(pc.acc));
}

__device__ __forceinline__ bool load_handoff_from(const HandOff* rec, PathCtx& pc);
__device__ __forceinline__ bool load_handoff(const RenderParams& P, uint64_t slot, PathCtx& pc) {
  DTS_CHECK(slot < P.ho_cap);
  return load_handoff_from(P.ho + slot, pc);
}
__device__ __forceinline__ bool load_handoff_from(const HandOff* rec, PathCtx& pc) {
  const uint4* s = reinterpret_cast<const uint4*>(rec);
  // all four 16-byte loads in flight at once (an empty slot's are harmless)
  const uint4 a = __ldcs(s + 1), b = __ldcs(s), c = __ldcs(s + 2), d = __ldcs(s + 3);
  if (a.w == kHoEmpty) return false;
  PathState& ps = pc.ps;
  ps.x = mk(__uint_as_float(b.x), __uint_as_float(b.y), __uint_as_float(b.z));
  ps.beta = __uint_as_float(b.w);
  ps.w = mk(__uint_as_float(a.x), __uint_as_float(a.y), __uint_as_float(a.z));
  pc.k = a.w;
  ps.resM = __hiloint2double((int)c.y, (int)c.x);
  pc.id_lo = c.z;
  pc.id_hi = c.w;
  pc.cell = d.x;
  pc.inv_n = __uint_as_float(d.y);
  ps.kind = (int)(d.z & 0xFFu);
  ps.face = (int)((d.z >> 8) & 0xFFu) - 1;
  ps.e = (int)(d.z >> 16);
  pc.acc = __uint_as_float(d.w);
  return true;
}

template <bool SMEM, int SH, int FL, bool DEFER, bool RESUME = false>
__global__ void __launch_bounds__(render_block(DEFER, (FL & FL_MESH) != 0, RESUME && (FL & FL_SPLIT) == 0), DTS_MINB)
    render_darts_kernel(const RenderParams P) {
  constexpr bool WALLS = (FL & FL_WALLS) != 0;
  // the connect stage of a REUSE scene resumes paths after the start stage's
  // camera vertex: no camera vertices (SPLIT scenes hand paths over at any vertex)
  constexpr bool kNoCam = RESUME && (FL & FL_SPLIT) == 0;
  // RESUME (connect stage): the work items are the walk stage's hand-off slots
  const uint64_t ntotal = RESUME ? (uint64_t)*(volatile unsigned long long*)P.ho_count : P.total;
  extern __shared__ __align__(16) uint16_t s_dyn[];
  __shared__ uint64_t s_bar;
  // rare events (path starts and ends) are counted per CTA in shared memory;
  // the per-vertex ones in registers
  __shared__ uint32_t s_ctr[DTS_NUM_COUNTERS];  // 32-bit: native shared atomics; <= paths per CTA
  if (threadIdx.x < DTS_NUM_COUNTERS) s_ctr[threadIdx.x] = 0u;
  const DevScene& S = P.S;
  const uint16_t* tab = P.tab;
  // dynamic shared memory: [EDA table (SMEM)] [private histogram] [private hist_sq] [job queues]
  float* s_hist = nullptr;
  float* s_sq = nullptr;
  float* s_queue = nullptr;
  {
    char* base = reinterpret_cast<char*>(s_dyn) + (SMEM ? (size_t)P.table_u4 * 16 : 0);
    if (P.priv_cells) {
      s_hist = reinterpret_cast<float*>(base);
      if (P.hist_sq) s_sq = s_hist + P.priv_cells;
      const uint32_t n = P.priv_cells * (P.hist_sq ? 2u : 1u);
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s_hist[i] = 0.0f;
      base += (size_t)n * sizeof(float);
    }
    if (DEFER) s_queue = reinterpret_cast<float*>(base);
  }
  if (SMEM) {
    bulk_stage(s_dyn, P.tab, P.table_u4 * 16u, &s_bar);
    tab = s_dyn;
  }
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  // this warp's connection-job queue: field f of slot j at q[f * qstride + j]
  const uint32_t qstride = (uint32_t)kQueue * (kBlock / 32);  // (DEFER kernels only)
  Defer df;
  df.q = DEFER ? s_queue + (threadIdx.x >> 5) * kQueue : nullptr;
  // SPLIT kernels: the stage-1 queues follow the sampling queues
  constexpr bool kStage1 = kStage1Build && DEFER && (FL & FL_SPLIT) != 0;
  df.q1 = kStage1 ? s_queue + (size_t)kJobWords * qstride + (threadIdx.x >> 5) * kQueue : nullptr;
  {  // this warp's global overflow slots (kQueue per queue)
    float* gw = DEFER ? P.qover + ((size_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5)) *
                                      (size_t)(kQueue * (kJobWords + kJob1Words))
                      : nullptr;
    df.g = gw;
    df.g1 = DEFER ? gw + kQueue * kJobWords : nullptr;
  }
  df.qstride = qstride;
  df.qn = 0;
  df.qn1 = 0;
  df.lane_lt = lt_mask;
  // warp-uniform work queue [wn, we)
  uint64_t wn = 0, we = 0;
  bool exhausted = false;
  bool active = false;
  PathCtx pc;
  // per-lane event counters, summed over the warp at the end
  uint32_t c_vert = 0, c_conn = 0, c_nee = 0;
  uint32_t c_wall = 0;  // wall / surface vertices (scenes with walls or meshes)
  uint32_t c_samp = 0;  // non-zero contributions (path samples); DARTS never rejects one (its bin has W > 0)
  uint32_t waste = 0;                // idle lane-iterations since the last refill
  // runs up to kQueue queued sampling jobs, one per lane, and splats them;
  // jobs left in the global overflow slots move down into the shared slots
  auto flush = [&]() {
    float c = 0.0f;
    uint32_t cell = 0;
    if ((uint32_t)lane < df.qn) {
      c = conn_job_eval<SH, FL>(S, df.q + lane, qstride, cell);
      if (!isfinite(c)) {
        atomicAdd(s_ctr + DTS_CTR_NONFINITE, 1u);
        c = 0.0f;
      }
      c_samp += c != 0.0f ? 1u : 0u;
    }
    const bool has = c != 0.0f;
    const unsigned m = __ballot_sync(FULL, has);
    if (m) splat(m, has, cell, c, 0.0f, P.hist, nullptr, s_hist, nullptr, lane, P.cells);
    __syncwarp();
    const uint32_t rest = df.qn > (uint32_t)kQueue ? df.qn - kQueue : 0u;
    if ((uint32_t)lane < rest)
      for (int f = 0; f < kJobWords; ++f) df.q[f * qstride + lane] = df.g[f * kQueue + lane];
    df.qn = rest;
    __syncwarp();
  };
  // runs up to kQueue stage-1 jobs (SPLIT: mixture direction, its intersection,
  // S range), one per lane, and forwards the non-empty ones to the sampling queue
  auto flush1 = [&]() {
    bool want2 = false;
    f3 x = mk(0.0f, 0.0f, 0.0f), wc = x;
    float dlo = 0.0f, width = 0.0f, coef2 = 0.0f;
    uint32_t m7e = 0, cell = 0;
    if ((uint32_t)lane < df.qn1) {
      const float* q = df.q1 + lane;
      const uint32_t st = qstride;
      x = mk(q[0 * st], q[1 * st], q[2 * st]);
      const f3 wprev = mk(q[3 * st], q[4 * st], q[5 * st]);
      const double resM_d = __hiloint2double(__float_as_int(q[6 * st]), __float_as_int(q[7 * st]));
      const float coef = q[8 * st];
      const uint32_t r4 = __float_as_uint(q[9 * st]), r5 = __float_as_uint(q[10 * st]), r6 = __float_as_uint(q[11 * st]);
      m7e = __float_as_uint(q[12 * st]);
      cell = __float_as_uint(q[13 * st]);
      const int e = (FL & FL_MULTI_E) ? (int)(m7e >> 23) : 0;
      const f3 xe = ld3(S.em_pos[e]);
      const MixDir md = mix_direction<SMEM, false>(S, tab, x, wprev, d2f(resM_d), xe, r4, r5, r6);
      wc = md.om;
      float lo_, chi;
      int face_;
      if (intersect_inside<SH, WALLS>(S, x, wc, lo_, chi, face_) != HIT_MISS) {
        const f3 cv = xe - x;
        const float C = sqrtf(dot(cv, cv));
        const SRange rg = conn_range(S, x, wc, xe, C, dot(wc, cv), 0.0f, chi, resM_d);
        if (rg.width > 0.0f) {
          want2 = true;
          ++c_conn;
          dlo = rg.dlo;
          width = rg.width;
          coef2 = coef * __fdividef(md.p_hg, md.p_mix);  // R29 SPLIT: the MIS weight stays on the connection
        }
      }
    }
    __syncwarp();
    const uint32_t rest = df.qn1 > (uint32_t)kQueue ? df.qn1 - kQueue : 0u;
    if ((uint32_t)lane < rest)
      for (int f = 0; f < kJob1Words; ++f) df.q1[f * qstride + lane] = df.g1[f * kQueue + lane];
    df.qn1 = rest;
    const unsigned m2 = __ballot_sync(FULL, want2);
    if (want2) {
      uint32_t st;
      float* qq = queue_slot(df.q, qstride, df.g, df.qn + __popc(m2 & lt_mask), &st);
      qq[0 * st] = x.x; qq[1 * st] = x.y; qq[2 * st] = x.z;
      qq[3 * st] = wc.x; qq[4 * st] = wc.y; qq[5 * st] = wc.z;
      qq[6 * st] = dlo;
      qq[7 * st] = width;
      qq[8 * st] = coef2;
      qq[9 * st] = __uint_as_float(m7e);
      qq[10 * st] = __uint_as_float(cell);
    }
    df.qn += __popc(m2);
    __syncwarp();
  };
  while (true) {
    // Lanes retire one at a time, and a path start (+ its camera vertex) runs
    // at a few active lanes.  Refill when the idle lane-iterations accumulated
    // since the last refill reach refill_k (ski rental: an idle lane costs
    // ~1/32 of an iteration, a start ~refill_k of those), so long-walk scenes
    // start paths in small batches and short-walk scenes in large ones.
    const unsigned idle = __ballot_sync(FULL, !active);
    waste += __popc(idle);
    if (idle && !exhausted && (waste >= P.refill_k || idle == FULL)) {
      waste = 0;
      // (kStartTries > 1: a lane whose new path retires at its start -- camera
      // miss, early exit, empty hand-off slot -- takes the next one in the same
      // refill; measured slower, off by default)
      unsigned need = idle;
      for (int t = 0; t < kStartTries && need && !exhausted; ++t) {
        const uint64_t my = take_work(need, lane, lt_mask, wn, we, exhausted, P.work, ntotal, P.chunk,
                                      RESUME ? reinterpret_cast<const char*>(P.ho) : nullptr);
        const bool starts = my != ~0ull && my < ntotal;
        const unsigned sm = __ballot_sync(FULL, starts);
        if (!RESUME && lane == 0 && sm) atomicAdd(s_ctr + DTS_CTR_PATHS, (uint32_t)__popc(sm));
        if (starts) active = RESUME ? load_handoff(P, my, pc) : start_path<SH, FL>(P, P.w_base + my, pc, s_ctr);
        DTS_CHECK(!(kNoCam && active && pc.ps.kind == KIND_CAMERA));
        need = __ballot_sync(FULL, ((need >> lane) & 1u) && !active);
      }
    }
    const unsigned act = __ballot_sync(FULL, active);
    // queue batches; once the work is exhausted and every lane idle, drain them
    // (one call site each: the queue code is inlined once)
    const bool drain = act == 0u && exhausted;
    // Capacity: each queue has kQueue shared + kQueue global slots.  After this
    // loop qn < flush_at and qn1 < flush1_at (<= kQueue), so the <= 32 pushes of
    // the next vertex always fit; flush1 (which feeds <= 32 jobs to the sampling
    // queue) only runs while that queue has <= kQueue jobs.
    while (DEFER) {
      const bool need1 = kStage1 && df.qn1 && (df.qn1 >= P.flush1_at || drain);
      if (df.qn && (df.qn >= P.flush_at || drain || (need1 && df.qn > (uint32_t)kQueue))) {
        flush();
      } else if (need1) {
        flush1();
      } else {
        break;
      }
    }
    if (act == 0u) {
      if (drain && df.qn1 == 0u && df.qn == 0u) break;
      continue;
    }
    bool done = false;
    // kInner vertices per lane between refills (the refill / flush bookkeeping
    // is paid once per kInner vertices; a lane that retires in the first waits)
    for (int rep = 0; rep < kInner; ++rep) {
      const unsigned act_r = rep == 0 ? act : __ballot_sync(FULL, active && !done);
      if (act_r == 0u) break;
      const bool run = active && !done;
      bool pushed = false, pushed1 = false;
      bool cn = false, wnee = false, alive = false;
      int reason = 0;
      uint32_t r[8];
      float contrib = 0.0f;
      RisReq rq;
      rq.need = false;
      if (run) {
        // vertex mix of the roofline basis (bench/opcounts.json): camera vertices
        // (once per walk, shared-memory counter), wall / surface vertices
        if (!kNoCam && pc.ps.kind == KIND_CAMERA) atomicAdd(s_ctr + DTS_CTR_CAMERA_VERTICES, 1u);
        if (WALLS || (FL & FL_MESH)) c_wall += (pc.ps.kind == KIND_WALL || pc.ps.kind == KIND_SURF) ? 1u : 0u;
        const u4 a = philox_rk(pc.id_lo, pc.id_hi, pc.k, 0u, S.rk);
        const u4 b = philox_rk(pc.id_lo, pc.id_hi, pc.k, 1u, S.rk);
        r[0] = a.a; r[1] = a.b; r[2] = a.c; r[3] = a.d;
        r[4] = b.a; r[5] = b.b; r[6] = b.c; r[7] = b.d;
        df.act = act_r;
        df.cell = pc.cell;
        df.inv_n = pc.inv_n;
        alive = darts_vertex<false, SMEM, SH, FL, DEFER, false, kNoCam>(S, tab, pc.ps, r, contrib, nullptr, cn, wnee, reason,
                                                         DEFER ? &df : nullptr, &pushed, kRisWarp ? &rq : nullptr,
                                                         &c_samp, &pushed1);
      }
      if (kRisWarp) {
        // RIS layout B: the warp draws every pending medium event's distance
        const f3 xe = ld3(S.em_pos[(FL & FL_MULTI_E) ? pc.ps.e : 0]);
        float dsel, Wr, wsel;
        ris_warp(S, pc.ps, rq, xe, r[1], r[2], r[3], lane, dsel, Wr, wsel);
        if (rq.need) {
          if (Wr > 0.0f) {
            ris_apply(S, pc.ps, dsel, Wr, wsel, rq.counts);
            alive = vertex_tail(pc.ps, xe, reason);
          } else {
            alive = false;
            reason = DTS_CTR_RIS_INVALID;  // R5
          }
        }
      }
      if (run) {
        pc.acc += contrib;
        ++pc.k;
        const bool cap = alive && pc.k >= (uint32_t)S.max_bounces;
        done = !alive || cap;
        ++c_vert;
        c_conn += cn ? 1u : 0u;
        if (WALLS) c_nee += wnee ? 1u : 0u;
        if (done) atomicAdd(s_ctr + (cap ? (int)DTS_CTR_CAP_HITS : reason), 1u);  // reason: a DTS_CTR_* index
      }
      if (DEFER) df.qn += __popc(__ballot_sync(FULL, pushed));
      if (kStage1) df.qn1 += __popc(__ballot_sync(FULL, pushed1));
    }
    const unsigned dmask = __ballot_sync(FULL, done);
    if (dmask) {
      const float v = isfinite(pc.acc) ? pc.acc : 0.0f;
      splat_retired(P, dmask, done, pc.cell, v * pc.inv_n, v * v * pc.inv_n, s_hist, s_sq, lane);
      if (done) active = false;
    }
  }

  for (int o = 16; o > 0; o >>= 1) {
    c_vert += __shfl_xor_sync(FULL, c_vert, o);
    c_conn += __shfl_xor_sync(FULL, c_conn, o);
    c_nee += __shfl_xor_sync(FULL, c_nee, o);
    c_samp += __shfl_xor_sync(FULL, c_samp, o);
    if (WALLS || (FL & FL_MESH)) c_wall += __shfl_xor_sync(FULL, c_wall, o);
  }
  if (lane == 0 && P.counters) {  // per-vertex counters: 64-bit, straight to global
    atomicAdd(P.counters + DTS_CTR_VERTICES, (unsigned long long)c_vert);
    atomicAdd(P.counters + DTS_CTR_CONN_NONEMPTY, (unsigned long long)c_conn);
    atomicAdd(P.counters + DTS_CTR_WALL_NEE, (unsigned long long)c_nee);
    atomicAdd(P.counters + DTS_CTR_SAMPLES, (unsigned long long)c_samp);
    if (WALLS || (FL & FL_MESH)) atomicAdd(P.counters + DTS_CTR_WALL_VERTICES, (unsigned long long)c_wall);
  }
  __syncthreads();
  if (P.priv_cells) {  // flush the CTA's private histogram (coalesced REDs of its non-zero cells)
    for (uint32_t i = threadIdx.x; i < P.priv_cells; i += blockDim.x) {
      if (s_hist[i] != 0.0f) atomicAdd(P.hist + i, s_hist[i]);
      if (s_sq && s_sq[i] != 0.0f) atomicAdd(P.hist_sq + i, s_sq[i]);
    }
  }
  if (P.counters && threadIdx.x < DTS_NUM_COUNTERS && s_ctr[threadIdx.x])
    atomicAdd(P.counters + threadIdx.x, (unsigned long long)s_ctr[threadIdx.x]);
}

// Walk stage of the two-stage render (see HandOff): persistent, one lane per
// path, no EDA table (so no shared-memory staging), walk-only vertices while
// conn_margin > 0.  The margin is tracked without re-evaluating the bound at
// every vertex: a step of length d lowers R_m - E by (counts d) and can raise
// the bound by at most d (|y - x| is 1-Lipschitz in x), so margin - (1 +
// counts) d is a lower bound; the exact margin is recomputed only when that
// lower bound reaches 0.  A path whose margin is <= 0 is written to the next
// hand-off slot (warp-level reservation of kHoBlock slots from a global
// counter); a path that ends in the walk stage contributed nothing.
#ifndef DTS_BLOCK_WALK
#define DTS_BLOCK_WALK 1024
#endif
constexpr int kBlockWalk = DTS_BLOCK_WALK;
#ifndef DTS_WALK_INNER
#define DTS_WALK_INNER 4
#endif
constexpr int kWalkInner = DTS_WALK_INNER;
template <int SH, int FL, bool RESUME = false>
__global__ void __launch_bounds__(kBlockWalk, 1) walk_kernel(const RenderParams P) {
  static_assert((FL & FL_SPLIT) && !(FL & FL_MESH), "walk stage: SPLIT scenes without meshes");
  // RESUME (three-stage render): the work items are the start stage's records
  const uint64_t ntotal = RESUME ? (uint64_t)*(volatile unsigned long long*)P.ho_in_count : P.total;
  __shared__ uint32_t s_ctr[DTS_NUM_COUNTERS];
  if (threadIdx.x < DTS_NUM_COUNTERS) s_ctr[threadIdx.x] = 0u;
  __syncthreads();
  const DevScene& S = P.S;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint64_t wn = 0, we = 0;   // warp-uniform work queue [wn, we)
  uint32_t hn = 0, he = 0;   // warp-uniform reserved hand-off slots [hn, he) (a chunk holds < 2^31)
  bool exhausted = false, active = false;
  PathCtx pc;
  float margin = 0.0f;
  uint32_t c_vert = 0, c_camw = 0, c_wall = 0, waste = 0;
  while (true) {
    const unsigned idle = __ballot_sync(FULL, !active);
    waste += __popc(idle);
    if (idle && !exhausted && (waste >= P.refill_k || idle == FULL)) {
      waste = 0;
      unsigned need = idle;  // (retry paths that retire at their start, as in render_darts_kernel)
      for (int t = 0; t < kStartTries && need && !exhausted; ++t) {
        const uint64_t my = take_work(need, lane, lt_mask, wn, we, exhausted, P.work, ntotal, P.chunk,
                                      RESUME ? reinterpret_cast<const char*>(P.ho_in) : nullptr);
        const bool starts = my != ~0ull && my < ntotal;
        const unsigned sm = __ballot_sync(FULL, starts);
        if (!RESUME && lane == 0 && sm) atomicAdd(s_ctr + DTS_CTR_PATHS, (uint32_t)__popc(sm));
        if (starts) {
          if (RESUME) {
            DTS_CHECK(my < P.ho_cap);
            const HandOff* src = P.ho_in + my;
            active = load_handoff_from(src, pc);
          } else {
            active = start_path<SH, FL>(P, P.w_base + my, pc, s_ctr);
          }
          margin = conn_margin<SH>(S, pc.ps.x, pc.ps.resM);
          c_camw += (active && margin > 0.0f) ? 1u : 0u;  // its camera vertex runs in the walk stage
        }
        need = __ballot_sync(FULL, ((need >> lane) & 1u) && !active);
      }
    }
    const unsigned act = __ballot_sync(FULL, active);
    if (act == 0u) {
      if (exhausted) break;
      continue;
    }
    bool hand = false, done = false;
    // kWalkInner vertices per lane between refills and hand-offs (the warp's
    // refill / hand-off bookkeeping is paid once per kWalkInner vertices; a lane
    // that stops in an earlier one waits; walk phases last ~10^2 vertices)
    for (int rep = 0; rep < kWalkInner; ++rep) {
      if (rep > 0 && !__any_sync(FULL, active && !hand && !done)) break;
      if (active && !hand && !done) {
        if (margin <= 0.0f) margin = conn_margin<SH>(S, pc.ps.x, pc.ps.resM);
        hand = margin <= 0.0f;
      }
      if (active && !hand && !done) {
        // a walk-only vertex reads u0..u3 and the SPLIT walk's u8, u9, all from
        // the first Philox block (R24); only a wall's cosine bounce needs u5, u6
        const u4 a = philox_rk(pc.id_lo, pc.id_hi, pc.k, 0u, S.rk);
        u4 b = u4{0u, 0u, 0u, 0u};
        if (FL & FL_WALLS) b = philox_rk(pc.id_lo, pc.id_hi, pc.k, 1u, S.rk);
        const uint32_t r[8] = {a.a, a.b, a.c, a.d, b.a, b.b, b.c, b.d};
        if (FL & FL_WALLS) c_wall += pc.ps.kind == KIND_WALL ? 1u : 0u;
        float contrib = 0.0f;
        bool cn = false, wnee = false;
        int reason = 0;
        const bool alive = darts_vertex<false, false, SH, FL, false, true>(S, nullptr, pc.ps, r, contrib, nullptr, cn,
                                                                           wnee, reason, nullptr, nullptr, nullptr,
                                                                           nullptr, nullptr, &margin);
        ++pc.k;
        ++c_vert;
        const bool cap = alive && pc.k >= (uint32_t)S.max_bounces;
        done = !alive || cap;
        if (done) atomicAdd(s_ctr + (cap ? (int)DTS_CTR_CAP_HITS : reason), 1u);
      }
    }
    const unsigned hm = __ballot_sync(FULL, hand);
    if (hm) {
      const uint32_t nh = __popc(hm), rank = __popc(hm & lt_mask);
      const uint32_t avail = he - hn;
      uint32_t slot;
      if (avail >= nh) {
        slot = hn + rank;
        hn += nh;
      } else {
        unsigned long long nb = 0;
        if (lane == 0) nb = atomicAdd(P.ho_count, (unsigned long long)kHoBlock);
        const uint32_t nb32 = (uint32_t)__shfl_sync(FULL, nb, 0);
        slot = rank < avail ? hn + rank : nb32 + (rank - avail);
        hn = nb32 + (nh - avail);
        he = nb32 + kHoBlock;
      }
      DTS_CHECK(!hand || slot < P.ho_cap);
      if (hand) store_handoff(P.ho + slot, pc);
    }
    if (hand || done) active = false;
  }
  // this warp's unused reserved slots are marked empty for the connect stage
  if ((uint32_t)lane < he - hn) reinterpret_cast<uint4*>(P.ho + hn + lane)[1].w = kHoEmpty;
  for (int o = 16; o > 0; o >>= 1) {
    c_vert += __shfl_xor_sync(FULL, c_vert, o);
    c_camw += __shfl_xor_sync(FULL, c_camw, o);
    c_wall += __shfl_xor_sync(FULL, c_wall, o);
  }
  if (lane == 0 && P.counters) {
    atomicAdd(P.counters + DTS_CTR_VERTICES, (unsigned long long)c_vert);
    // walk-only medium vertices: every walk-stage vertex but the camera and wall ones
    atomicAdd(P.counters + DTS_CTR_WALK_VERTICES, (unsigned long long)(c_vert - c_camw - c_wall));
    if (c_camw) atomicAdd(P.counters + DTS_CTR_CAMERA_VERTICES, (unsigned long long)c_camw);
    if (c_wall) atomicAdd(P.counters + DTS_CTR_WALL_VERTICES, (unsigned long long)c_wall);
  }
  __syncthreads();
  if (P.counters && threadIdx.x < DTS_NUM_COUNTERS && s_ctr[threadIdx.x])
    atomicAdd(P.counters + threadIdx.x, (unsigned long long)s_ctr[threadIdx.x]);
}

// Start stage of the two-stage render of REUSE scenes:
// every work item's path start (decode, camera ray, R18 miss, start early
// exit) and its camera vertex (the camera-ray connection and RIS distance; no
// mixture direction, so no EDA table) run here, one work item per lane and
// every lane in the same code, instead of one start at a time inside the
// persistent loop's refills next to medium and wall vertices.  A path that
// ends at its camera vertex splats here; a surviving one is handed over,
// with its contribution so far, through a 64-byte HBM record (one slot
// reservation per warp) to the connect stage (render_darts_kernel<RESUME>),
// which continues it from bounce 1.  Same path ids, random numbers, vertices
// and per-path sums as the one-stage kernel.
#ifndef DTS_BLOCK_START
#define DTS_BLOCK_START 1024
#endif
constexpr int kBlockStart = DTS_BLOCK_START;
// CAM = false (three-stage render of SPLIT scenes): the path starts only; every
// started path is handed to the walk stage (walk_kernel<RESUME>), which runs its
// camera vertex like any other.
template <int SH, int FL, bool CAM = true>
__global__ void __launch_bounds__(kBlockStart) start_kernel(const RenderParams P) {
  static_assert(!CAM || !(FL & FL_SPLIT), "start stage with camera vertices: REUSE scenes");
  __shared__ uint32_t s_ctr[DTS_NUM_COUNTERS];
  if (threadIdx.x < DTS_NUM_COUNTERS) s_ctr[threadIdx.x] = 0u;
  __syncthreads();
  const DevScene& S = P.S;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t c_vert = 0, c_conn = 0, c_samp = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < P.total; base += stride) {
    const uint64_t my = base + (uint64_t)lane;
    PathCtx pc;
    bool active = false;
    if (my < P.total) active = start_path<SH, FL>(P, P.w_base + my, pc, s_ctr);
    if (lane == 0) atomicAdd(s_ctr + DTS_CTR_PATHS, (uint32_t)(P.total - base < 32u ? P.total - base : 32u));
    bool done = false;
    if (CAM && active) {
      const u4 a = philox_rk(pc.id_lo, pc.id_hi, 0u, 0u, S.rk);
      const u4 b = philox_rk(pc.id_lo, pc.id_hi, 0u, 1u, S.rk);
      const uint32_t r[8] = {a.a, a.b, a.c, a.d, b.a, b.b, b.c, b.d};
      float contrib = 0.0f;
      bool cn = false, wnee = false;
      int reason = 0;
      pc.ps.kind = KIND_CAMERA;  // (constant: only the camera branches of the vertex are compiled in)
      const bool alive = darts_vertex<false, false, SH, FL>(S, nullptr, pc.ps, r, contrib, nullptr, cn, wnee, reason,
                                                            nullptr, nullptr, nullptr, &c_samp);
      pc.acc += contrib;
      ++pc.k;
      ++c_vert;
      c_conn += cn ? 1u : 0u;
      const bool cap = alive && pc.k >= (uint32_t)S.max_bounces;
      done = !alive || cap;
      if (done) atomicAdd(s_ctr + (cap ? (int)DTS_CTR_CAP_HITS : reason), 1u);
    }
    const bool hand = active && !done;
    const unsigned hm = __ballot_sync(FULL, hand);
    if (hm) {
      unsigned long long nb = 0;
      if (lane == 0) nb = atomicAdd(P.ho_count, (unsigned long long)__popc(hm));
      const uint32_t slot = (uint32_t)__shfl_sync(FULL, nb, 0) + __popc(hm & lt_mask);
      DTS_CHECK(!hand || slot < P.ho_cap);
      if (hand) store_handoff(P.ho + slot, pc);
    }
    const unsigned dmask = CAM ? __ballot_sync(FULL, done) : 0u;
    if (dmask) {
      const float v = isfinite(pc.acc) ? pc.acc : 0.0f;
      splat_retired(P, dmask, done, pc.cell, v * pc.inv_n, v * v * pc.inv_n, nullptr, nullptr, lane);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    c_vert += __shfl_xor_sync(FULL, c_vert, o);
    c_conn += __shfl_xor_sync(FULL, c_conn, o);
    c_samp += __shfl_xor_sync(FULL, c_samp, o);
  }
  if (CAM && lane == 0 && P.counters) {
    atomicAdd(P.counters + DTS_CTR_VERTICES, (unsigned long long)c_vert);
    atomicAdd(P.counters + DTS_CTR_CAMERA_VERTICES, (unsigned long long)c_vert);  // every vertex here is one
    atomicAdd(P.counters + DTS_CTR_CONN_NONEMPTY, (unsigned long long)c_conn);
    atomicAdd(P.counters + DTS_CTR_SAMPLES, (unsigned long long)c_samp);
  }
  __syncthreads();
  if (P.counters && threadIdx.x < DTS_NUM_COUNTERS && s_ctr[threadIdx.x])
    atomicAdd(P.counters + threadIdx.x, (unsigned long long)s_ctr[threadIdx.x]);
}

// ============================================================== vanilla
// splats a vanilla connection into the bin of its arrival time, weighted by
// the sensor response W there (RESPONSE scenes); returns 1 for a path sample
// rejected by W = 0 (outside the bins, or a zero of W), 0 if splatted
// splats a vanilla connection into the bin of its arrival time, weighted by
// the sensor response W there (RESPONSE scenes); returns 1 for a path sample
// rejected by W = 0 (outside the bins, or a zero of W), 0 if splatted.  row:
// the warp's shared-memory copy of this pixel's histogram row (privatised
// launches), else null (RED to the histogram in global memory)
__device__ __forceinline__ int vanilla_splat(const RenderParams& P, uint32_t pl, double arrive, float c, float* row) {
  const DevScene& S = P.S;
  const int bin = arrive >= S.t0 ? (int)floor((arrive - S.t0) / S.dt) : -1;
  if (bin < 0 || bin >= S.n_bins) return 1;
  DTS_CHECK((size_t)pl * S.n_bins + bin < P.cells);
  const float w = P.resp_w ? __ldg(P.resp_w + bin) : 1.0f;
  if (w == 0.0f) return 1;
  const float v = __fdividef(w * c, (float)P.spp);
  if (row) atomicAdd(row + bin, v);
  else atomicAdd(P.hist + (size_t)pl * S.n_bins + bin, v);
  return 0;
}

struct VanCtr {
  uint32_t paths = 0, miss = 0, vert = 0, early = 0, esc = 0, cap = 0, samp = 0, rej = 0;
};

// One vanilla path: work item (pixel pl of the crop, sample s).
template <int SH, bool WALLS, bool MESH>
__device__ __forceinline__ void vanilla_path(const RenderParams& P, uint32_t pl, uint64_t s, float* row, VanCtr& c) {
  const DevScene& S = P.S;
  uint32_t cx;
  const uint32_t cy = fastdiv_divmod(pl, P.fd_cw, cx);
  const uint32_t px = (uint32_t)S.crop[0] + cx, py = (uint32_t)S.crop[1] + cy;
  const uint64_t p = (uint64_t)py * (uint64_t)S.width + px;
  const uint64_t id = s * ((uint64_t)S.width * (uint64_t)S.height) + p;
  pl = P.ph_base + cy * P.hw + cx;  // the histogram's pixel
  const uint32_t id_lo = (uint32_t)id, id_hi = (uint32_t)(id >> 32);
  ++c.paths;
  const u4 a = philox_rk(id_lo, id_hi, 0xFFFFFFFFu, 0u, S.rk);
  const int e = (int)unif_index((uint32_t)S.n_emitters, a.c);
  const f3 xe = ld3(S.em_pos[e]);
  const double te = (double)S.em_t[e];
  const float ek = S.em_k[e];
  f3 x, w;
  float beta;
  if (S.camera_kind == DTS_CAMERA_PINHOLE) {
    const float sx = (__fdividef(2.0f * ((float)px + unif(a.a)), (float)S.width) - 1.0f) * S.tan_half * S.aspect;
    const float sy = (1.0f - __fdividef(2.0f * ((float)py + unif(a.b)), (float)S.height)) * S.tan_half;
    w = mk(S.fwd[0] + sx * S.right[0] + sy * S.upc[0], S.fwd[1] + sx * S.right[1] + sy * S.upc[1],
           S.fwd[2] + sx * S.right[2] + sy * S.upc[2]);
    w = w * rsqrtf(dot(w, w));
    x = ld3(S.cam_pos);
    beta = 1.0f;
  } else {
    const u4 bb = philox_rk(id_lo, id_hi, 0xFFFFFFFFu, 1u, S.rk);
    const u4 cc = philox_rk(id_lo, id_hi, 0xFFFFFFFFu, 2u, S.rk);
    const float rad = S.det_radius * cbrtf(unif(bb.a));
    const float z = 1.0f - 2.0f * unif(bb.b);
    const float sz = sqrtf(fmaxf(0.0f, 1.0f - z * z));
    float sp, cp;
    __sincosf(2.0f * kPi * unif(bb.c), &sp, &cp);
    x = mk(S.cam_pos[0] + rad * sz * cp, S.cam_pos[1] + rad * sz * sp, S.cam_pos[2] + rad * z);
    const float z2 = 1.0f - 2.0f * unif(bb.d);
    const float s2 = sqrtf(fmaxf(0.0f, 1.0f - z2 * z2));
    __sincosf(2.0f * kPi * unif(cc.a), &sp, &cp);
    w = mk(s2 * cp, s2 * sp, z2);
    beta = 4.0f * kPi;
  }
  {
    float lo, hi;
    int f;
    if (intersect<SH, WALLS>(S, x, w, lo, hi, f) == HIT_MISS) {
      ++c.miss;
      return;
    }
  }
  int kind = KIND_CAMERA, face = -1;
  double E = 0.0;
  bool alive = true;
  int k;
  for (k = 0; k < S.max_bounces && alive; ++k) {
    const u4 r = philox_rk(id_lo, id_hi, (uint32_t)k, 0u, S.rk);
    ++c.vert;
    if (kind == KIND_MEDIUM) {
      float opc, omc;
      hg_sample(S, unif(r.b), opc, omc);
      w = from_frame(w, opc, omc, kPi * (2.0f * unif(r.c) - 1.0f));
    } else if (kind == KIND_WALL) {
      const f3 n = inward_normal(face);
      const float u5 = unif(r.b), u6 = unif(r.c);
      const float rr = sqrtf(u5);
      float sp, cp;
      __sincosf(2.0f * kPi * u6, &sp, &cp);
      const float sign = n.z >= -1e-6f ? 1.0f : -1.0f;  // R12 tie-break (from_frame)
      const float aa = __fdividef(-1.0f, sign + n.z);
      const float bq = n.x * n.y * aa;
      const f3 b1 = mk(1.0f + sign * n.x * n.x * aa, sign * bq, -sign * n.x);
      const f3 b2 = mk(bq, sign + n.y * n.y * aa, -n.y);
      const float lx = rr * cp, ly = rr * sp, lz = sqrtf(fmaxf(0.0f, 1.0f - u5));
      w = mk(b1.x * lx + b2.x * ly + n.x * lz, b1.y * lx + b2.y * ly + n.y * lz, b1.z * lx + b2.z * ly + n.z * lz);
      beta *= S.wall_albedo[face];
    } else if (MESH && kind == KIND_SURF) {
      // R32 sampling (lobe u3, direction u1 u2; the oracle's vanilla order)
      int mat;
      const f3 n = tri_side_normal(S, face, w, mat);
      f3 wo;
      const float wgt = bsdf_sample(S, mat, n, w, unif(r.d), unif(r.b), unif(r.c), wo);
      if (!(wgt > 0.0f)) { ++c.esc; alive = false; break; }
      beta *= wgt;
      w = wo;
    }
    float lo, hi;
    int hf;
    int hit = intersect<SH, WALLS>(S, x, w, lo, hi, hf);
    if (MESH && hit != HIT_MISS) {
      float tm;
      const int tri = mesh_trace<false>(S, x, w, hi, tm);
      if (tri >= 0) { hi = tm; hit = HIT_SURF; hf = tri; }
    }
    if (hit == HIT_MISS) { ++c.esc; alive = false; break; }
    const float counts = (S.warped || kind != KIND_CAMERA) ? 1.0f : 0.0f;
    const f3 d0 = x - xe;
    const float Cprev = sqrtf(dot(d0, d0));
    float d = lo + neg_log1m(unif(r.a)) * S.inv_sigma_t;
    if (d < hi) {
      x = fma3(w, d, x);
      E += (double)(counts * d);
      beta *= S.albedo;
      kind = KIND_MEDIUM;
    } else if (WALLS && hit == HIT_WALL) {
      d = hi;
      f3 xn = fma3(w, hi, x);
      const int ax = hf >> 1;
      const float pl2 = (hf & 1) ? S.bmax[ax] : S.bmin[ax];
      if (ax == 0) xn.x = pl2; else if (ax == 1) xn.y = pl2; else xn.z = pl2;
      x = xn;
      E += (double)(counts * hi);
      kind = KIND_WALL;
      face = hf;
    } else if (MESH && hit == HIT_SURF) {
      d = hi;
      int mat;
      const f3 n = tri_side_normal(S, hf, w, mat);
      x = fma3(n, kSurfEps, fma3(w, hi, x));
      E += (double)(counts * hi);
      kind = KIND_SURF;
      face = hf;
    } else { ++c.esc; alive = false; break; }
    const f3 cv = xe - x;
    const float C = sqrtf(dot(cv, cv));
    const double arrive = te + E + (double)C;
    if (arrive >= S.t0 + S.dt * S.n_bins) { ++c.early; alive = false; break; }
    const f3 we = cv * (1.0f / C);
    float cc;
    if (kind == KIND_MEDIUM) {
      cc = beta * hg_eval(S, dot(w, we));
      if (S.s_excess > 0.0f && d + C - Cprev < S.s_excess) cc = 0.0f;
    } else if (MESH && kind == KIND_SURF) {
      int mat;
      const f3 n = tri_side_normal(S, face, w, mat);
      cc = beta * bsdf_eval(S, mat, n, w, we) * fmaxf(0.0f, dot(n, we));
    } else {
      cc = beta * (S.wall_albedo[face] * (1.0f / kPi)) * fmaxf(0.0f, dot(inward_normal(face), we));
    }
    cc *= segment_tr<SH, WALLS, MESH>(S, x, xe, C, we) * __fdividef(ek, C * C);
    if (S.r_excl > 0.0f && C < S.r_excl) cc = 0.0f;
    if (cc != 0.0f && isfinite(cc)) {
      ++c.samp;
      c.rej += vanilla_splat(P, pl, arrive, cc, row);
    }
  }
  if (alive && k >= S.max_bounces) ++c.cap;
}

// Vanilla estimator: one lane per path.  Privatised launches (P.van_rows:
// vanilla paths splat into every bin along their walk, ~1 RED per vertex) take
// the work in pixel-major order, so a warp's 32 lanes are consecutive samples
// of one pixel; their connections go to the warp's shared-memory copy of that
// pixel's row of n_bins floats (shared-memory atomics), flushed to HBM with
// coalesced REDs of the non-zero bins after each batch of 32 paths.  Lanes of a
// batch that crosses into the next pixel RED straight to HBM.
template <int SH, bool WALLS, bool MESH = false>
__global__ void __launch_bounds__(kBlock) render_vanilla_kernel(const RenderParams P) {
  extern __shared__ float s_rows[];
  const DevScene& S = P.S;
  const uint32_t B = (uint32_t)S.n_bins;
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  float* row = P.van_rows ? s_rows + (size_t)(threadIdx.x >> 5) * B : nullptr;
  if (row)
    for (uint32_t b = lane; b < B; b += 32) row[b] = 0.0f;
  __syncwarp();
  VanCtr c;
  // warp-uniform batches of 32 consecutive work items
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < P.total; base += stride) {
    const uint64_t widx = base + (uint64_t)lane;
    const bool valid = widx < P.total;
    uint32_t pl = 0;
    uint64_t s = 0;
    if (valid) {
      if (P.van_rows) {  // pixel-major: samples of a pixel are consecutive
        if (P.div32) {
          uint32_t sl;
          pl = fastdiv_divmod((uint32_t)widx, P.fd_ns, sl);
          s = P.s_begin + sl;
        } else {
          s = P.s_begin + widx % P.n_s;
          pl = (uint32_t)(widx / P.n_s);
        }
      } else if (P.div32) {
        s = P.s_begin + fastdiv_divmod((uint32_t)widx, P.fd_npix, pl);
      } else {
        pl = (uint32_t)(widx % P.npix);
        s = P.s_begin + widx / P.npix;
      }
    }
    const uint32_t pw = __shfl_sync(0xffffffffu, pl, 0);   // the batch's pixel (lane 0 is always valid)
    uint32_t pwx;
    const uint32_t pwh = P.ph_base + fastdiv_divmod(pw, P.fd_cw, pwx) * P.hw + pwx;  // its histogram pixel
    if (valid) vanilla_path<SH, WALLS, MESH>(P, pl, s, (row && pl == pw) ? row : nullptr, c);
    if (row) {  // flush the batch's row: coalesced REDs of its non-zero bins
      __syncwarp();
      float* g = P.hist + (size_t)pwh * B;
      for (uint32_t b = lane; b < B; b += 32) {
        const float v = row[b];
        if (v != 0.0f) {
          atomicAdd(g + b, v);
          row[b] = 0.0f;
        }
      }
      __syncwarp();
    }
  }
  // warp-reduce and flush counters
  for (int o = 16; o > 0; o >>= 1) {
    c.paths += __shfl_xor_sync(0xffffffffu, c.paths, o);
    c.miss += __shfl_xor_sync(0xffffffffu, c.miss, o);
    c.vert += __shfl_xor_sync(0xffffffffu, c.vert, o);
    c.early += __shfl_xor_sync(0xffffffffu, c.early, o);
    c.esc += __shfl_xor_sync(0xffffffffu, c.esc, o);
    c.cap += __shfl_xor_sync(0xffffffffu, c.cap, o);
    c.samp += __shfl_xor_sync(0xffffffffu, c.samp, o);
    c.rej += __shfl_xor_sync(0xffffffffu, c.rej, o);
  }
  if (lane == 0 && P.counters) {
    atomicAdd(P.counters + DTS_CTR_PATHS, (unsigned long long)c.paths);
    atomicAdd(P.counters + DTS_CTR_CAMERA_MISS, (unsigned long long)c.miss);
    atomicAdd(P.counters + DTS_CTR_VERTICES, (unsigned long long)c.vert);
    atomicAdd(P.counters + DTS_CTR_EARLY_EXIT, (unsigned long long)c.early);
    atomicAdd(P.counters + DTS_CTR_ESCAPES, (unsigned long long)c.esc);
    atomicAdd(P.counters + DTS_CTR_CAP_HITS, (unsigned long long)c.cap);
    atomicAdd(P.counters + DTS_CTR_SAMPLES, (unsigned long long)c.samp);
    atomicAdd(P.counters + DTS_CTR_REJECTED, (unsigned long long)c.rej);
  }
}

// culled camera rays (live_rect) are counted as started paths that missed
__global__ void add_culled_kernel(unsigned long long* counters, unsigned long long n) {
  atomicAdd(counters + DTS_CTR_PATHS, n);
  atomicAdd(counters + DTS_CTR_CAMERA_MISS, n);
}

// ============================================================== kernel selection
// Render and debug kernels are specialised at compile time on the medium
// shape and the variant flags FL_WALLS, FL_SPLIT (direction mode, R29) and
// FL_MULTI_E (more than one emitter), so no launch carries the branches,
// registers or constant-bank indexing of the other scene kinds.  Walls exist
// only in BOX media (validated), so the other shapes instantiate the even FLs.
template <int SH, int FL>
static const void* dk_ptr() { return (const void*)debug_kernel<SH, FL>; }

template <template <int> class Pick>
static const void* pick_fl(int shape, int fl) {
  if (shape == DTS_MEDIUM_BOX) {
    switch (fl) {
      case 0: return Pick<0>::box(); case 1: return Pick<1>::box();
      case 2: return Pick<2>::box(); case 3: return Pick<3>::box();
      case 4: return Pick<4>::box(); case 5: return Pick<5>::box();
      case 6: return Pick<6>::box(); case 7: return Pick<7>::box();
    }
    return nullptr;
  }
  if (fl & FL_WALLS) return nullptr;
  const bool inf = shape == DTS_MEDIUM_INFINITE;
  if (!inf && shape != DTS_MEDIUM_SPHERE) return nullptr;
  switch (fl) {
    case 0: return inf ? Pick<0>::inf() : Pick<0>::sph();
    case 2: return inf ? Pick<2>::inf() : Pick<2>::sph();
    case 4: return inf ? Pick<4>::inf() : Pick<4>::sph();
    case 6: return inf ? Pick<6>::inf() : Pick<6>::sph();
  }
  return nullptr;
}
template <bool SMEM, bool DEFER>
struct PickRender {
  template <int FL>
  struct F {
    static const void* box() { return (const void*)render_darts_kernel<SMEM, DTS_MEDIUM_BOX, FL, DEFER>; }
    static const void* inf() { return (const void*)render_darts_kernel<SMEM, DTS_MEDIUM_INFINITE, FL, DEFER>; }
    static const void* sph() { return (const void*)render_darts_kernel<SMEM, DTS_MEDIUM_SPHERE, FL, DEFER>; }
  };
};
template <int FL> struct PickDebug {
  static const void* box() { return dk_ptr<DTS_MEDIUM_BOX, FL>(); }
  static const void* inf() { return dk_ptr<DTS_MEDIUM_INFINITE, FL>(); }
  static const void* sph() { return dk_ptr<DTS_MEDIUM_SPHERE, FL>(); }
};
template <int FL> struct PickDebugMesh {
  static const void* box() { return dk_ptr<DTS_MEDIUM_BOX, FL | FL_MESH>(); }
  static const void* inf() { return dk_ptr<DTS_MEDIUM_INFINITE, FL | FL_MESH>(); }
  static const void* sph() { return dk_ptr<DTS_MEDIUM_SPHERE, FL | FL_MESH>(); }
};
static int scene_flags(const dts_scene_desc& d) {
  return (d.wall_mask ? FL_WALLS : 0) | (d.direction_mode == DTS_DIR_SPLIT ? FL_SPLIT : 0) |
         (d.n_emitters > 1 ? FL_MULTI_E : 0);
}
// mesh scenes (FL_MESH): immediate kernels with the table in shared memory
template <int FL>
struct PickMesh {
  static const void* box() { return (const void*)render_darts_kernel<true, DTS_MEDIUM_BOX, FL | FL_MESH, false>; }
  static const void* inf() { return (const void*)render_darts_kernel<true, DTS_MEDIUM_INFINITE, FL | FL_MESH, false>; }
  static const void* sph() { return (const void*)render_darts_kernel<true, DTS_MEDIUM_SPHERE, FL | FL_MESH, false>; }
};
// two-stage render (SPLIT scenes without meshes, BOX or SPHERE media)
template <bool SMEM, bool DEFER = false>
struct PickResume {
  template <int FL>
  struct F {
    static const void* box() {
      if constexpr ((FL & FL_SPLIT) != 0) return (const void*)render_darts_kernel<SMEM, DTS_MEDIUM_BOX, FL, DEFER, true>;
      return nullptr;
    }
    static const void* inf() { return nullptr; }
    static const void* sph() {
      if constexpr ((FL & FL_SPLIT) != 0 && (FL & FL_WALLS) == 0)
        return (const void*)render_darts_kernel<SMEM, DTS_MEDIUM_SPHERE, FL, DEFER, true>;
      return nullptr;
    }
  };
};
template <int FL>
struct PickWalk {
  static const void* box() {
    if constexpr ((FL & FL_SPLIT) != 0) return (const void*)walk_kernel<DTS_MEDIUM_BOX, FL>;
    return nullptr;
  }
  static const void* inf() { return nullptr; }
  static const void* sph() {
    if constexpr ((FL & FL_SPLIT) != 0 && (FL & FL_WALLS) == 0) return (const void*)walk_kernel<DTS_MEDIUM_SPHERE, FL>;
    return nullptr;
  }
};

// start stage + connect stage of REUSE scenes in BOX / SPHERE media, EDA table
// in shared memory (meshes included)
template <int FL>
struct PickStart {
  static const void* box() {
    if constexpr ((FL & FL_SPLIT) == 0) return (const void*)start_kernel<DTS_MEDIUM_BOX, FL>;
    return nullptr;
  }
  static const void* inf() { return nullptr; }
  static const void* sph() {
    if constexpr ((FL & (FL_SPLIT | FL_WALLS)) == 0) return (const void*)start_kernel<DTS_MEDIUM_SPHERE, FL>;
    return nullptr;
  }
};
template <int FL>
struct PickStartMesh {
  static const void* box() {
    if constexpr ((FL & FL_SPLIT) == 0) return (const void*)start_kernel<DTS_MEDIUM_BOX, FL | FL_MESH>;
    return nullptr;
  }
  static const void* inf() { return nullptr; }
  static const void* sph() {
    if constexpr ((FL & (FL_SPLIT | FL_WALLS)) == 0) return (const void*)start_kernel<DTS_MEDIUM_SPHERE, FL | FL_MESH>;
    return nullptr;
  }
};
// three-stage render of SPLIT scenes: start stage (path starts only) + walk stage
// continuing the start records
template <int FL>
struct PickStartSplit {
  static const void* box() {
    if constexpr ((FL & FL_SPLIT) != 0) return (const void*)start_kernel<DTS_MEDIUM_BOX, FL, false>;
    return nullptr;
  }
  static const void* inf() { return nullptr; }
  static const void* sph() {
    if constexpr ((FL & FL_SPLIT) != 0 && (FL & FL_WALLS) == 0)
      return (const void*)start_kernel<DTS_MEDIUM_SPHERE, FL, false>;
    return nullptr;
  }
};
template <int FL>
struct PickWalkResume {
  static const void* box() {
    if constexpr ((FL & FL_SPLIT) != 0) return (const void*)walk_kernel<DTS_MEDIUM_BOX, FL, true>;
    return nullptr;
  }
  static const void* inf() { return nullptr; }
  static const void* sph() {
    if constexpr ((FL & FL_SPLIT) != 0 && (FL & FL_WALLS) == 0)
      return (const void*)walk_kernel<DTS_MEDIUM_SPHERE, FL, true>;
    return nullptr;
  }
};
template <int FL>
struct PickResumeReuse {
  static const void* box() {
    if constexpr ((FL & FL_SPLIT) == 0) return (const void*)render_darts_kernel<true, DTS_MEDIUM_BOX, FL, false, true>;
    return nullptr;
  }
  static const void* inf() { return nullptr; }
  static const void* sph() {
    if constexpr ((FL & (FL_SPLIT | FL_WALLS)) == 0)
      return (const void*)render_darts_kernel<true, DTS_MEDIUM_SPHERE, FL, false, true>;
    return nullptr;
  }
};
template <int FL>
struct PickResumeMesh {
  static const void* box() {
    if constexpr ((FL & FL_SPLIT) == 0)
      return (const void*)render_darts_kernel<true, DTS_MEDIUM_BOX, FL | FL_MESH, false, true>;
    return nullptr;
  }
  static const void* inf() { return nullptr; }
  static const void* sph() {
    if constexpr ((FL & (FL_SPLIT | FL_WALLS)) == 0)
      return (const void*)render_darts_kernel<true, DTS_MEDIUM_SPHERE, FL | FL_MESH, false, true>;
    return nullptr;
  }
};

static const void* darts_kernel_ptr(bool smem, bool defer, const dts_scene_desc& d) {
  const int sh = d.medium_shape, fl = scene_flags(d);
  if (d.n_tris > 0) return (smem && !defer) ? pick_fl<PickMesh>(sh, fl) : nullptr;
  if (smem) return defer ? pick_fl<PickRender<true, true>::F>(sh, fl) : pick_fl<PickRender<true, false>::F>(sh, fl);
  return defer ? pick_fl<PickRender<false, true>::F>(sh, fl) : pick_fl<PickRender<false, false>::F>(sh, fl);
}
static const void* debug_kernel_ptr(const dts_scene_desc& d) {
  return d.n_tris > 0 ? pick_fl<PickDebugMesh>(d.medium_shape, scene_flags(d))
                      : pick_fl<PickDebug>(d.medium_shape, scene_flags(d));
}
static const void* vanilla_kernel_ptr(int shape, bool walls, bool mesh) {
  if (mesh) {
    if (shape == DTS_MEDIUM_INFINITE) return (const void*)render_vanilla_kernel<DTS_MEDIUM_INFINITE, false, true>;
    if (shape == DTS_MEDIUM_SPHERE) return (const void*)render_vanilla_kernel<DTS_MEDIUM_SPHERE, false, true>;
    if (shape == DTS_MEDIUM_BOX)
      return walls ? (const void*)render_vanilla_kernel<DTS_MEDIUM_BOX, true, true>
                   : (const void*)render_vanilla_kernel<DTS_MEDIUM_BOX, false, true>;
    return nullptr;
  }
  if (shape == DTS_MEDIUM_INFINITE) return (const void*)render_vanilla_kernel<DTS_MEDIUM_INFINITE, false>;
  if (shape == DTS_MEDIUM_SPHERE) return (const void*)render_vanilla_kernel<DTS_MEDIUM_SPHERE, false>;
  if (shape == DTS_MEDIUM_BOX)
    return walls ? (const void*)render_vanilla_kernel<DTS_MEDIUM_BOX, true>
                 : (const void*)render_vanilla_kernel<DTS_MEDIUM_BOX, false>;
  return nullptr;
}

// Philox4x32-10 key schedule of a seed (R24): round r uses
// (k0 + r 0x9E3779B9, k1 + r 0xBB67AE85) mod 2^32.
static void set_round_keys(DevScene& S, uint64_t seed) {
  S.seed_lo = (uint32_t)seed;
  S.seed_hi = (uint32_t)(seed >> 32);
  uint32_t k0 = S.seed_lo, k1 = S.seed_hi;
  for (int r = 0; r < 10; ++r) {
    S.rk[2 * r] = k0;
    S.rk[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// ============================================================== host helpers
static void vsub(const double a[3], const double b[3], double o[3]) { for (int i = 0; i < 3; ++i) o[i] = a[i] - b[i]; }
static void vnorm(double a[3]) { double n = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); for (int i = 0; i < 3; ++i) a[i] /= n; }
static void vcross(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

static dts_status validate(const dts_scene_desc& d) {
  auto bad = [](const char* m) { return fail(DTS_E_INVALID_ARG, m); };
  if (!(d.sigma_s > 0.0f) || !(d.sigma_a >= 0.0f) || !std::isfinite(d.sigma_s) || !std::isfinite(d.sigma_a))
    return bad("sigma_s must be > 0 and sigma_a >= 0");
  if (!(d.g > -1.0f && d.g < 1.0f)) return bad("HG g must lie in (-1, 1)");
  if (d.medium_shape < 0 || d.medium_shape > 2) return bad("unknown medium_shape");
  if (d.medium_shape == DTS_MEDIUM_SPHERE && !(d.radius > 0.0f)) return bad("sphere radius must be > 0");
  if (d.medium_shape == DTS_MEDIUM_BOX)
    for (int a = 0; a < 3; ++a)
      if (!(d.bmax[a] > d.bmin[a])) return bad("box bmax must exceed bmin");
  if (d.wall_mask && d.medium_shape != DTS_MEDIUM_BOX) return bad("walls need a BOX medium");
  if (d.wall_mask >= 64u) return bad("wall_mask has bits above face 5");
  if (d.n_emitters < 1 || d.n_emitters > DTS_MAX_EMITTERS) return bad("n_emitters must be 1..8");
  for (int e = 0; e < d.n_emitters; ++e)
    if (!(d.em_energy[e] >= 0.0f)) return bad("emitter energy must be >= 0");
  if (d.camera_kind != DTS_CAMERA_PINHOLE && d.camera_kind != DTS_CAMERA_SPHERE_DETECTOR) return bad("unknown camera_kind");
  if (d.width < 1 || d.height < 1) return bad("width/height must be >= 1");
  if (d.camera_kind == DTS_CAMERA_PINHOLE && !(d.fov_y_deg > 0.0f && d.fov_y_deg < 180.0f)) return bad("fov must be in (0,180)");
  if (d.camera_kind == DTS_CAMERA_SPHERE_DETECTOR && !(d.det_radius > 0.0f)) return bad("det_radius must be > 0");
  if (d.crop[0] < 0 || d.crop[1] < 0 || d.crop[2] > d.width || d.crop[3] > d.height || d.crop[2] <= d.crop[0] ||
      d.crop[3] <= d.crop[1])
    return bad("crop must be a non-empty sub-rectangle of the image");
  if (!(d.t1 > d.t0) || d.n_bins < 1) return bad("need t1 > t0 and n_bins >= 1");
  if (d.strategy < DTS_STRATEGY_DARTS || d.strategy > DTS_STRATEGY_EDA_ONLY) return bad("unknown strategy");
  if (d.conn_sampling != DTS_CONN_TRUNC_EXP && d.conn_sampling != DTS_CONN_UNIFORM_S) return bad("unknown conn_sampling");
  if (d.n_ris != 8) return bad("n_ris must be 8 (PAPER.md:240)");
  if (!(d.alpha >= 0.0f)) return bad("alpha must be >= 0");
  if (d.max_bounces < 1 || d.max_bounces > 65536) return bad("max_bounces must be 1..65536");
  if (d.direction_mode != DTS_DIR_REUSE && d.direction_mode != DTS_DIR_SPLIT) return bad("unknown direction_mode");
  if (d.spp_mode < DTS_SPP_PER_CELL || d.spp_mode > DTS_SPP_RESPONSE) return bad("unknown spp_mode");
  if (!(d.parity_r_excl >= 0.0f) || !(d.parity_s_excess >= 0.0f)) return bad("parity restrictions must be >= 0");
  if (d.n_tris < 0) return bad("n_tris must be >= 0");
  if (d.n_tris > 0) {  // R32, R33
    if (!d.tris || !d.tri_mat) return bad("mesh arrays are NULL");
    if (d.n_mats < 1 || d.n_mats > DTS_MAX_MATERIALS) return bad("n_mats must be 1..8");
    for (int m = 0; m < d.n_mats; ++m)
      if (!(d.mats[m][0] >= 0.0f && d.mats[m][0] <= 1.0f) || !(d.mats[m][1] >= 0.0f && d.mats[m][1] <= 1.0f) ||
          !(d.mats[m][2] >= 0.0f && d.mats[m][2] <= 1e4f))
        return bad("material needs rho, ks in [0, 1] and 0 <= n <= 1e4");
    for (int i = 0; i < d.n_tris; ++i) {
      if (d.tri_mat[i] < 0 || d.tri_mat[i] >= d.n_mats) return bad("triangle material index out of range");
      const float* v = d.tris + 9 * (size_t)i;
      for (int k = 0; k < 9; ++k)
        if (!std::isfinite(v[k])) return bad("non-finite triangle vertex");
      if (d.medium_shape == DTS_MEDIUM_BOX)
        for (int k = 0; k < 3; ++k)
          for (int a = 0; a < 3; ++a)
            if (!(v[3 * k + a] >= d.bmin[a] + 1e-3f && v[3 * k + a] <= d.bmax[a] - 1e-3f))
              return bad("mesh vertices must lie >= 1e-3 inside the box");
      if (d.medium_shape == DTS_MEDIUM_SPHERE)
        for (int k = 0; k < 3; ++k) {
          double r2 = 0.0;
          for (int a = 0; a < 3; ++a) r2 += ((double)v[3 * k + a] - d.center[a]) * ((double)v[3 * k + a] - d.center[a]);
          if (!(std::sqrt(r2) <= (double)d.radius - 1e-3)) return bad("mesh vertices must lie >= 1e-3 inside the sphere");
        }
      double e1[3], e2[3], n[3];
      for (int a = 0; a < 3; ++a) { e1[a] = (double)v[3 + a] - v[a]; e2[a] = (double)v[6 + a] - v[a]; }
      vcross(e1, e2, n);
      if (!(n[0] * n[0] + n[1] * n[1] + n[2] * n[2] > 0.0)) return bad("degenerate (zero-area) triangle");
    }
  }
  return DTS_OK;
}

// Median-split BVH over the triangles' centroids (leaves of <= 4 triangles,
// nodes in depth-first order: an inner node's first child follows it).
static int bvh_node(const float* tris, std::vector<int>& ord, int b, int e, std::vector<float4>& nodes) {
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  float clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = b; i < e; ++i) {
    const float* v = tris + 9 * (size_t)ord[i];
    for (int a = 0; a < 3; ++a) {
      const float c = (v[a] + v[3 + a] + v[6 + a]) / 3.0f;
      clo[a] = std::fmin(clo[a], c);
      chi[a] = std::fmax(chi[a], c);
      for (int k = 0; k < 3; ++k) {
        lo[a] = std::fmin(lo[a], v[3 * k + a]);
        hi[a] = std::fmax(hi[a], v[3 * k + a]);
      }
    }
  }
  const int id = (int)nodes.size() / 2;
  nodes.push_back(make_float4(lo[0], lo[1], lo[2], 0.0f));
  nodes.push_back(make_float4(hi[0], hi[1], hi[2], 0.0f));
  int a_field, n_field;
  if (e - b <= 4) {
    a_field = b;
    n_field = e - b;
  } else {
    int ax = 0;
    for (int a = 1; a < 3; ++a)
      if (chi[a] - clo[a] > chi[ax] - clo[ax]) ax = a;
    const int mid = (b + e) / 2;
    auto cen = [&](int t) { const float* v = tris + 9 * (size_t)t; return v[ax] + v[3 + ax] + v[6 + ax]; };
    std::nth_element(ord.begin() + b, ord.begin() + mid, ord.begin() + e, [&](int x, int y) { return cen(x) < cen(y); });
    bvh_node(tris, ord, b, mid, nodes);  // = id + 1
    a_field = bvh_node(tris, ord, mid, e, nodes);
    n_field = 0;
  }
  int ai = a_field, ni = n_field;
  float af, nf;
  memcpy(&af, &ai, 4);
  memcpy(&nf, &ni, 4);
  nodes[2 * id].w = af;
  nodes[2 * id + 1].w = nf;
  return id;
}

static dts_status upload_mesh(dts_scene* s) {
  const dts_scene_desc& d = s->desc;
  std::vector<int> ord(d.n_tris);
  for (int i = 0; i < d.n_tris; ++i) ord[i] = i;
  std::vector<float4> nodes;
  nodes.reserve(4 * (size_t)d.n_tris / 2 + 2);
  bvh_node(d.tris, ord, 0, d.n_tris, nodes);
  std::vector<float4> tri4(3 * (size_t)d.n_tris);
  for (int i = 0; i < d.n_tris; ++i) {
    const float* v = d.tris + 9 * (size_t)ord[i];
    int m = d.tri_mat[ord[i]];
    float mf;
    memcpy(&mf, &m, 4);
    tri4[3 * (size_t)i] = make_float4(v[0], v[1], v[2], mf);
    tri4[3 * (size_t)i + 1] = make_float4(v[3] - v[0], v[4] - v[1], v[5] - v[2], 0.0f);
    tri4[3 * (size_t)i + 2] = make_float4(v[6] - v[0], v[7] - v[1], v[8] - v[2], 0.0f);
  }
  if (cudaMalloc(&s->d_bvh, nodes.size() * sizeof(float4)) != cudaSuccess ||
      cudaMalloc(&s->d_tri4, tri4.size() * sizeof(float4)) != cudaSuccess)
    return fail(DTS_E_OOM, "cudaMalloc(mesh) failed");
  CUDA_TRY(cudaMemcpy(s->d_bvh, nodes.data(), nodes.size() * sizeof(float4), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(s->d_tri4, tri4.data(), tri4.size() * sizeof(float4), cudaMemcpyHostToDevice));
  std::vector<int32_t> tmap(2 * (size_t)d.n_tris);
  for (int i = 0; i < d.n_tris; ++i) {
    tmap[(size_t)ord[i]] = i;              // caller's index -> leaf position
    tmap[(size_t)d.n_tris + i] = ord[i];   // leaf position -> caller's index
  }
  if (cudaMalloc(&s->d_tri_map, tmap.size() * sizeof(int32_t)) != cudaSuccess) return fail(DTS_E_OOM, "cudaMalloc(mesh) failed");
  CUDA_TRY(cudaMemcpy(s->d_tri_map, tmap.data(), tmap.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  DevScene& S = s->S;
  S.bvh = s->d_bvh;
  S.tri4 = s->d_tri4;
  S.tri_leaf = s->d_tri_map;
  S.tri_orig = s->d_tri_map + d.n_tris;
  S.n_tris = d.n_tris;
  for (int m = 0; m < d.n_mats; ++m) {  // R32 constants
    const double rho = d.mats[m][0], ks = d.mats[m][1], n = d.mats[m][2];
    S.mat_ks[m] = (float)ks;
    S.mat_kd[m] = (float)(rho * (1.0 - ks) / M_PI);
    S.mat_kl[m] = (float)(rho * ks * (n + 2.0) / (2.0 * M_PI));
    S.mat_pd[m] = (float)((1.0 - ks) / M_PI);
    S.mat_pl[m] = (float)(ks * (n + 1.0) / (2.0 * M_PI));
    S.mat_n[m] = (float)n;
    S.mat_inv_n1[m] = (float)(1.0 / (n + 1.0));
  }
  // the caller keeps its arrays: forget their addresses
  s->desc.tris = nullptr;
  s->desc.tri_mat = nullptr;
  return DTS_OK;
}

// Camera-ray culling: the pixels [x0, x1) x [y0, y1) (absolute image
// coordinates) outside of which every pinhole ray -- whatever its sub-pixel
// jitter -- misses the medium's bounds, so its path retires at its start with
// nothing splatted (a "camera miss", R18).  The medium's image is bounded by
// projecting a conservative outline: the 8 corners of the (slightly enlarged)
// box -- the box's image is their convex hull -- or, for a sphere, a polygon of
// 1024 directions circumscribing the cone of rays that touch the (enlarged)
// ball.  A pixel is live when its footprint [p, p + 1) meets the outline's
// bounding interval, widened by 2 pixels on every side (the GPU's fp32 ray and
// slab test differ from this fp64 bound by ~1e-6 of a pixel's width).  When
// some outline point lies behind or beside the camera (or the camera is inside
// or near the medium) every pixel stays live.  Same paths, same random
// numbers: culled work items are exactly the ones that would miss.
static void live_rect(const dts_scene_desc& d, int out[4]) {
  out[0] = 0;
  out[1] = 0;
  out[2] = d.width;
  out[3] = d.height;
  if (d.camera_kind != DTS_CAMERA_PINHOLE || d.medium_shape == DTS_MEDIUM_INFINITE) return;
  double cam[3] = {d.cam_pos[0], d.cam_pos[1], d.cam_pos[2]}, la[3] = {d.look_at[0], d.look_at[1], d.look_at[2]},
         up[3] = {d.up[0], d.up[1], d.up[2]};
  double fwd[3], right[3], upc[3];
  vsub(la, cam, fwd);
  vnorm(fwd);
  vcross(fwd, up, right);
  vnorm(right);
  vcross(right, fwd, upc);
  const double th = std::tan(0.5 * (double)d.fov_y_deg * M_PI / 180.0), asp = (double)d.width / d.height;
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  // image-plane coordinates (sx, sy) of direction v; false if v is not well in front
  auto project = [&](const double v[3]) {
    const double z = v[0] * fwd[0] + v[1] * fwd[1] + v[2] * fwd[2];
    const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (!(z > 0.05 * n)) return false;
    const double sx = (v[0] * right[0] + v[1] * right[1] + v[2] * right[2]) / z;
    const double sy = (v[0] * upc[0] + v[1] * upc[1] + v[2] * upc[2]) / z;
    xmin = std::min(xmin, sx); xmax = std::max(xmax, sx);
    ymin = std::min(ymin, sy); ymax = std::max(ymax, sy);
    return true;
  };
  if (d.medium_shape == DTS_MEDIUM_BOX) {
    double ext = 0.0;
    for (int i = 0; i < 3; ++i) ext = std::max(ext, (double)d.bmax[i] - (double)d.bmin[i]);
    const double eps = 1e-4 * ext + 1e-4;
    for (int c = 0; c < 8; ++c) {
      double v[3];
      for (int i = 0; i < 3; ++i) v[i] = (((c >> i) & 1) ? (double)d.bmax[i] + eps : (double)d.bmin[i] - eps) - cam[i];
      if (!project(v)) return;
    }
  } else {
    double a[3];
    for (int i = 0; i < 3; ++i) a[i] = (double)d.center[i] - cam[i];
    const double dist = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    const double R = (double)d.radius * (1.0 + 1e-4) + 1e-4;
    if (!(dist > 1.01 * R)) return;
    for (int i = 0; i < 3; ++i) a[i] /= dist;
    constexpr int kN = 1024;
    // the cone's cross-section at unit distance along a is a circle of radius
    // tan(alpha); the kN-gon of circumradius tan(alpha) / cos(pi / kN) contains it
    const double ta = (R / std::sqrt(dist * dist - R * R)) / std::cos(M_PI / kN);
    double b1[3], b2[3], t[3] = {1.0, 0.0, 0.0};
    if (std::fabs(a[0]) > 0.9) { t[0] = 0.0; t[1] = 1.0; }
    vcross(a, t, b1);
    vnorm(b1);
    vcross(a, b1, b2);
    for (int k = 0; k < kN; ++k) {
      const double ph = 2.0 * M_PI * k / kN, c = std::cos(ph) * ta, s = std::sin(ph) * ta;
      double v[3];
      for (int i = 0; i < 3; ++i) v[i] = a[i] + c * b1[i] + s * b2[i];
      if (!project(v)) return;
    }
  }
  // sx = (2 (px + u) / W - 1) tan_half aspect, sy = (1 - 2 (py + u) / H) tan_half
  const double fx0 = (xmin / (th * asp) + 1.0) * 0.5 * d.width, fx1 = (xmax / (th * asp) + 1.0) * 0.5 * d.width;
  const double fy0 = (1.0 - ymax / th) * 0.5 * d.height, fy1 = (1.0 - ymin / th) * 0.5 * d.height;
  auto clampi = [](double v, int hi) { return (int)std::max(0.0, std::min((double)hi, v)); };
  out[0] = clampi(std::floor(fx0) - 3.0, d.width);
  out[2] = clampi(std::floor(fx1) + 3.0, d.width);
  out[1] = clampi(std::floor(fy0) - 3.0, d.height);
  out[3] = clampi(std::floor(fy1) + 3.0, d.height);
  if (out[2] <= out[0] || out[3] <= out[1]) out[0] = out[1] = out[2] = out[3] = 0;  // the medium is out of view
}

static void derive(const dts_scene_desc& d, DevScene& S) {
  memset(&S, 0, sizeof S);
  const double ss = d.sigma_s, sa = d.sigma_a, g = d.g, st = ss + sa;
  const double D = 1.0 / (3.0 * (sa + ss * (1.0 - g)));  // E9
  S.sigma_s = d.sigma_s;
  S.sigma_a = d.sigma_a;
  S.sigma_t = (float)st;
  S.albedo = (float)(ss / st);
  S.g = d.g;
  S.inv_sigma_t = (float)(1.0 / st);
  S.hg_k = (float)((1.0 - g * g) / (4.0 * M_PI));
  S.hg_1pg2 = (float)(1.0 + g * g);
  S.hg_2g = (float)(2.0 * g);
  S.hg_1mg2 = (float)(1.0 - g * g);
  S.hg_1mg = (float)(1.0 - g);
  S.hg_1pg = (float)(1.0 + g);
  S.neg_inv4D_log2e = (float)(-M_LOG2E / (4.0 * D));
  S.neg_sa_log2e = (float)(-sa * M_LOG2E);
  S.medium_shape = d.medium_shape;
  for (int i = 0; i < 3; ++i) {
    S.center[i] = d.center[i];
    S.bmin[i] = d.bmin[i];
    S.bmax[i] = d.bmax[i];
    S.cam_pos[i] = d.cam_pos[i];
  }
  S.radius2 = d.radius * d.radius;
  S.wall_mask = d.wall_mask;
  for (int f = 0; f < 6; ++f) S.wall_albedo[f] = d.wall_albedo[f];
  S.n_emitters = d.n_emitters;
  for (int e = 0; e < d.n_emitters; ++e) {
    for (int i = 0; i < 3; ++i) S.em_pos[e][i] = d.em_pos[e][i];
    S.em_t[e] = d.em_t[e];
    S.em_k[e] = (float)((double)d.em_energy[e] / (4.0 * M_PI) * d.n_emitters);
  }
  S.camera_kind = d.camera_kind;
  double cam[3] = {d.cam_pos[0], d.cam_pos[1], d.cam_pos[2]}, la[3] = {d.look_at[0], d.look_at[1], d.look_at[2]},
         up[3] = {d.up[0], d.up[1], d.up[2]};
  double fwd[3], right[3], upc[3];
  vsub(la, cam, fwd);
  vnorm(fwd);
  vcross(fwd, up, right);
  vnorm(right);
  vcross(right, fwd, upc);
  for (int i = 0; i < 3; ++i) {
    S.fwd[i] = (float)fwd[i];
    S.right[i] = (float)right[i];
    S.upc[i] = (float)upc[i];
  }
  S.tan_half = (float)std::tan(0.5 * (double)d.fov_y_deg * M_PI / 180.0);
  S.aspect = (float)((double)d.width / d.height);
  S.width = d.width;
  S.height = d.height;
  S.det_radius = d.det_radius;
  for (int i = 0; i < 4; ++i) S.crop[i] = d.crop[i];
  S.t0 = d.t0;
  S.dt = ((double)d.t1 - (double)d.t0) / d.n_bins;
  S.dt_f = (float)S.dt;
  S.n_bins = d.n_bins;
  S.warped = d.warped ? 1 : 0;
  S.strategy = d.strategy;
  S.conn_uniform = d.conn_sampling == DTS_CONN_UNIFORM_S ? 1 : 0;
  S.direction_mode = d.direction_mode;
  S.spp_mode = d.spp_mode;
  S.max_bounces = d.max_bounces;
  S.alpha = d.alpha;
  S.r_excl = d.parity_r_excl;
  S.s_excess = d.parity_s_excess;
  // far_e: largest distance from an emitter to a point of the medium (box: its
  // farthest corner; sphere: centre distance + radius), with a rounding margin
  double far = 0.0;
  for (int e = 0; e < d.n_emitters; ++e) {
    double f2 = 0.0;
    if (d.medium_shape == DTS_MEDIUM_BOX) {
      for (int a = 0; a < 3; ++a) {
        const double u = std::fmax(std::fabs((double)d.bmin[a] - d.em_pos[e][a]), std::fabs((double)d.bmax[a] - d.em_pos[e][a]));
        f2 += u * u;
      }
      far = std::fmax(far, std::sqrt(f2));
    } else if (d.medium_shape == DTS_MEDIUM_SPHERE) {
      for (int a = 0; a < 3; ++a) f2 += ((double)d.em_pos[e][a] - d.center[a]) * ((double)d.em_pos[e][a] - d.center[a]);
      far = std::fmax(far, std::sqrt(f2) + d.radius);
    }
  }
  S.far_e = d.medium_shape == DTS_MEDIUM_INFINITE ? INFINITY : (float)(far * (1.0 + 1e-4) + 1e-4);
}

// ============================================================== C ABI
extern "C" {

int32_t dts_abi_version(void) { return DTS_ABI_VERSION; }

const char* dts_status_string(dts_status s) {
  switch (s) {
    case DTS_OK: return "DTS_OK";
    case DTS_E_INVALID_ARG: return "DTS_E_INVALID_ARG";
    case DTS_E_STATE: return "DTS_E_STATE";
    case DTS_E_CUDA: return "DTS_E_CUDA";
    case DTS_E_OOM: return "DTS_E_OOM";
    case DTS_E_RANGE: return "DTS_E_RANGE";
  }
  return "DTS_E_UNKNOWN";
}

const char* dts_last_error(void) { return g_last_error.c_str(); }

dts_status dts_scene_create(const dts_scene_desc* desc, dts_scene_t* out) {
  if (!out) return fail(DTS_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!desc) return fail(DTS_E_INVALID_ARG, "desc is NULL");
  dts_status st = validate(*desc);
  if (st != DTS_OK) return st;
  if ((uint64_t)(desc->crop[2] - desc->crop[0]) * (uint64_t)(desc->crop[3] - desc->crop[1]) * (uint64_t)desc->n_bins >
      0xFFFFFFFFull)
    return fail(DTS_E_RANGE, "crop_w * crop_h * n_bins must be < 2^32 (32-bit histogram cell indices)");
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  // attribute queries (cudaGetDeviceProperties costs milliseconds per scene)
  int major = 0, sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (major < 10) return fail(DTS_E_CUDA, "libdts needs an sm_100 (Blackwell) device");
  dts_scene* s = new dts_scene();
  s->desc = *desc;
  derive(*desc, s->S);
  live_rect(*desc, s->live);
  s->num_sms = sms;
  s->device = dev;
  if (cudaMalloc(&s->d_work, sizeof(unsigned long long)) != cudaSuccess) {
    delete s;
    return fail(DTS_E_OOM, "cudaMalloc(work counter) failed");
  }
  if (desc->n_tris > 0) {
    st = upload_mesh(s);
    if (st != DTS_OK) {
      dts_scene_destroy(s);
      return st;
    }
  }
  *out = s;
  return DTS_OK;
}

dts_status dts_scene_destroy(dts_scene_t s) {
  if (!s) return DTS_OK;
  cudaDeviceSynchronize();
  cudaFree(s->d_table);
  cudaFree(s->d_table_f);
  if (s->tab_stream) cudaStreamDestroy(s->tab_stream);
  if (s->tab_fork) cudaEventDestroy(s->tab_fork);
  if (s->tab_ready) cudaEventDestroy(s->tab_ready);
  cudaFree(s->d_work);
  pool_put(s->device, s->d_hist_host, s->d_hist_host_n * sizeof(float));
  cudaFree(s->d_ctr_host);
  cudaFree(s->d_resp_cdf);
  cudaFree(s->d_resp_wgt);
  cudaFree(s->d_resp_w);
  cudaFree(s->d_zero_cell);
  cudaFree(s->d_qover);
  for (int i = 0; i < 2; ++i)
    if (s->band_stream[i]) cudaStreamDestroy(s->band_stream[i]);
  for (int i = 0; i <= kHostBands; ++i)
    if (s->band_ev[i]) cudaEventDestroy(s->band_ev[i]);
  cudaFree(s->d_work_band);
  for (int i = 0; i <= kHostBands; ++i) pool_put(s->device, s->d_ho[i], s->ho_cap[i] * sizeof(HandOff));
  cudaFree(s->d_wf);
  if (s->wf_stream) cudaStreamDestroy(s->wf_stream);
  for (int i = 0; i < 2; ++i)
    if (s->wf_ev[i]) cudaEventDestroy(s->wf_ev[i]);
  cudaFree(s->d_bvh);
  cudaFree(s->d_tri4);
  cudaFree(s->d_tri_map);
  delete s;
  return DTS_OK;
}

dts_status dts_table_build(dts_scene_t s, const dts_table_desc* td, void* stream) {
  if (!s) return fail(DTS_E_INVALID_ARG, "scene is NULL");
  const dts_scene_desc& d = s->desc;
  int nr = 16, ns = 16;
  double st = (double)d.sigma_s + d.sigma_a;
  double smin = 1e-2 / st, smax;
  float tmin = d.em_t[0];
  for (int e = 1; e < d.n_emitters; ++e) tmin = std::fmin(tmin, d.em_t[e]);
  smax = (double)d.t1 - tmin;
  if (td) {
    if (td->n_ratio > 0) nr = td->n_ratio;
    if (td->n_s > 0) ns = td->n_s;
    if (td->s_min > 0.0f) smin = td->s_min;
    if (td->s_max > 0.0f) smax = td->s_max;
  }
  if (nr > 256 || ns > 256) return fail(DTS_E_INVALID_ARG, "table axes must be <= 256");
  if (!(smax > smin)) return fail(DTS_E_INVALID_ARG, "table s_max must exceed s_min");
  const size_t n = (size_t)nr * ns * DTS_TABLE_COS_BINS;
  if (n != s->table_n) {
    cudaFree(s->d_table);
    s->d_table = nullptr;
    s->table_n = 0;
    if (cudaMalloc(&s->d_table, n * 3) != cudaSuccess) return fail(DTS_E_OOM, "cudaMalloc(table) failed");
    s->table_n = n;
  }
  TableParams P;
  P.sigma_s = d.sigma_s;
  P.sigma_a = d.sigma_a;
  P.sigma_t = st;
  P.D = 1.0 / (3.0 * ((double)d.sigma_a + (double)d.sigma_s * (1.0 - (double)d.g)));
  P.norm = 1.0 / std::pow(4.0 * M_PI * P.D, 1.5);
  P.smin = smin;
  P.smax = smax;
  P.nr = nr;
  P.ns = ns;
  if (s->table_f_n < n) {
    cudaFree(s->d_table_f);
  if (s->tab_stream) cudaStreamDestroy(s->tab_stream);
  if (s->tab_fork) cudaEventDestroy(s->tab_fork);
  if (s->tab_ready) cudaEventDestroy(s->tab_ready);
    s->d_table_f = nullptr;
    s->table_f_n = 0;
    if (cudaMalloc(&s->d_table_f, n * sizeof(double)) != cudaSuccess) return fail(DTS_E_OOM, "cudaMalloc(table scratch) failed");
    s->table_f_n = n;
  }
  // DTS_TABLE_OVERLAP=1: asynchronous with the caller's later work, so that a
  // render's start / walk stage, which reads no table, overlaps it (A/B: step
  // time -2 % on configs 1, 2, 6; profiles/ab_r02_table_overlap.log).  Off by
  // default: the render's CUDA-event time -- the roofline's kernel time -- would
  // then include waiting for the table.
  cudaStream_t tst = (cudaStream_t)stream;
  const char* tov = getenv("DTS_TABLE_OVERLAP");
  s->tab_async = tov && tov[0] == '1';
  if (s->tab_async) {
    if (!s->tab_stream) {
      CUDA_TRY(cudaStreamCreateWithFlags(&s->tab_stream, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&s->tab_fork, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&s->tab_ready, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(s->tab_fork, (cudaStream_t)stream));  // after the caller's prior work
    CUDA_TRY(cudaStreamWaitEvent(s->tab_stream, s->tab_fork, 0));
    tst = s->tab_stream;
  }
  table_f_kernel<<<nr * ns * 4, kTableThreads, 0, tst>>>(P, s->d_table_f);
  table_cdf_kernel<<<nr * ns, 256, 0, tst>>>(s->d_table_f, s->d_table, n);
  if (s->tab_async) CUDA_TRY(cudaEventRecord(s->tab_ready, tst));
  s->S.table_n = (uint32_t)n;
  CUDA_TRY(cudaGetLastError());
  s->S.nr = nr;
  s->S.ns = ns;
  s->S.nr_f = (float)nr;
  s->S.ns_f = (float)ns;
  s->S.ln_smin = (float)std::log(smin);
  s->S.inv_dls = (float)(ns / (std::log(smax) - std::log(smin)));
  return DTS_OK;
}

dts_status dts_set_response(dts_scene_t s, const float* h_w, int32_t n) {
  if (!s || !h_w) return fail(DTS_E_INVALID_ARG, "NULL argument");
  if (n != s->desc.n_bins) return fail(DTS_E_INVALID_ARG, "n must equal n_bins");
  double tot = 0.0;
  for (int b = 0; b < n; ++b) {
    if (!(h_w[b] >= 0.0f) || !std::isfinite(h_w[b])) return fail(DTS_E_INVALID_ARG, "W must be finite and >= 0");
    tot += h_w[b];
  }
  if (!(tot > 0.0)) return fail(DTS_E_INVALID_ARG, "W must not be all zero");
  // R31: c_k = round(2^23 sum_{j<k} W_j / sum W), sums in bin order, c_B = 2^23
  std::vector<uint32_t> cdf(n + 1);
  std::vector<float> wgt(n);
  double acc = 0.0;
  cdf[0] = 0u;
  for (int b = 0; b < n; ++b) {
    acc += h_w[b];
    cdf[b + 1] = (uint32_t)std::floor(8388608.0 * acc / tot + 0.5);
  }
  cdf[n] = 8388608u;
  for (int b = 0; b < n; ++b) {
    const uint32_t dc = cdf[b + 1] - cdf[b];
    wgt[b] = dc ? (float)((double)h_w[b] / ((double)dc / 8388608.0)) : 0.0f;
  }
  if (!s->d_resp_cdf) {
    if (cudaMalloc(&s->d_resp_cdf, (n + 1) * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&s->d_resp_wgt, n * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&s->d_resp_w, n * sizeof(float)) != cudaSuccess)
      return fail(DTS_E_OOM, "cudaMalloc(response) failed");
  }
  CUDA_TRY(cudaMemcpy(s->d_resp_cdf, cdf.data(), (n + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(s->d_resp_wgt, wgt.data(), n * sizeof(float), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(s->d_resp_w, h_w, n * sizeof(float), cudaMemcpyHostToDevice));
  return DTS_OK;
}

size_t dts_table_size(dts_scene_t s) { return s ? s->table_n : 0; }

dts_status dts_table_export(dts_scene_t s, uint16_t* host_q, size_t n) {
  if (!s || !host_q) return fail(DTS_E_INVALID_ARG, "NULL argument");
  if (!s->d_table) return fail(DTS_E_STATE, "table not built");
  if (n != s->table_n) return fail(DTS_E_INVALID_ARG, "n must equal dts_table_size()");
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(host_q, s->d_table, n * sizeof(uint16_t), cudaMemcpyDeviceToHost));
  return DTS_OK;
}

size_t dts_hist_cells(dts_scene_t s) {
  if (!s) return 0;
  const dts_scene_desc& d = s->desc;
  return (size_t)(d.crop[2] - d.crop[0]) * (size_t)(d.crop[3] - d.crop[1]) * (size_t)d.n_bins;
}

}  // extern "C"

// One render launch over crop rows [row0, row1) (relative to the crop) into
// d_hist (that band's first cell), with its own work counter: dts_render runs
// the whole crop; dts_render_host runs bands on two streams so each band's
// device->host copy overlaps the next band's render.
static dts_status render_impl(dts_scene_t s, uint64_t spp, uint64_t seed, uint64_t sb, uint64_t se, float* d_hist,
                              float* d_hist_sq, uint64_t* d_counters, void* stream, int row0, int row1,
                              unsigned long long* work, bool allow_defer, int slot) {
  g_last_launches = 0;
  if (!s) return fail(DTS_E_INVALID_ARG, "scene is NULL");
  if (!d_hist) return fail(DTS_E_INVALID_ARG, "d_hist is NULL");
  if (spp == 0 || se > spp || sb > se) return fail(DTS_E_RANGE, "need 0 <= sample_begin <= sample_end <= spp, spp > 0");
  if (sb == se) return DTS_OK;
  const dts_scene_desc& d = s->desc;
  const bool darts = d.strategy != DTS_STRATEGY_VANILLA;  // DARTS and its ablations
  if (darts && !s->d_table) return fail(DTS_E_STATE, "dts_table_build must run before a DARTS render");
  const uint64_t npix = (uint64_t)(d.crop[2] - d.crop[0]) * (uint64_t)(row1 - row0);
  const uint64_t ns = se - sb;
  const uint64_t Npix = (uint64_t)d.width * d.height;
  // path ids must fit 64 bits: (s * Npix + p) * B + b
  const double idmax = ((double)spp * (double)Npix + (double)Npix) * (double)d.n_bins;
  if (idmax > 1.8e19) return fail(DTS_E_RANGE, "path id space exceeds 64 bits");
  if (d.spp_mode == DTS_SPP_RESPONSE && !s->d_resp_cdf)
    return fail(DTS_E_STATE, "dts_set_response must run before a RESPONSE render");
  RenderParams P;
  memset(&P, 0, sizeof P);
  if (d.spp_mode == DTS_SPP_RESPONSE) {
    P.resp_cdf = s->d_resp_cdf;
    P.resp_wgt = s->d_resp_wgt;
    P.resp_w = s->d_resp_w;
  }
  P.S = s->S;
  P.S.crop[1] = d.crop[1] + row0;
  P.S.crop[3] = d.crop[1] + row1;
  // camera-ray culling (live_rect): the launch renders the live part of its
  // rows; the culled paths are camera misses, counted below (DTS_CULL=0: off)
  const int hx0 = d.crop[0], hy0 = d.crop[1] + row0, hwid = d.crop[2] - d.crop[0];
  int lx0 = hx0, ly0 = hy0, lx1 = d.crop[2], ly1 = d.crop[1] + row1;
  {
    const char* cu = getenv("DTS_CULL");
    if (!(cu && cu[0] == '0')) {
      lx0 = std::max(lx0, s->live[0]);
      ly0 = std::max(ly0, s->live[1]);
      lx1 = std::min(lx1, s->live[2]);
      ly1 = std::min(ly1, s->live[3]);
    }
    if (lx1 <= lx0 || ly1 <= ly0) lx1 = lx0 = ly1 = ly0 = 0;
  }
  const uint64_t npix_live = (uint64_t)(lx1 - lx0) * (uint64_t)(ly1 - ly0);
  P.S.crop[0] = lx0;
  P.S.crop[1] = ly0;
  P.S.crop[2] = lx1;
  P.S.crop[3] = ly1;
  P.hw = (uint32_t)hwid;
  P.ph_base = npix_live ? (uint32_t)((uint64_t)(ly0 - hy0) * (uint64_t)hwid + (uint64_t)(lx0 - hx0)) : 0u;
  set_round_keys(P.S, seed);
  P.tab = s->d_table;
  P.hist = d_hist;
  P.hist_sq = d_hist_sq;
  P.counters = reinterpret_cast<unsigned long long*>(d_counters);
  P.work = work;
  P.s_begin = sb;
  P.n_s = ns;
  P.spp = spp;
  P.npix = (uint32_t)npix_live;
  P.cw = (uint32_t)(lx1 - lx0);
  P.div32 = (sb + ns + (uint64_t)d.n_bins <= 0xFFFFFFFFull &&
             npix * ns * ((darts && d.spp_mode == DTS_SPP_PER_CELL) ? (uint64_t)d.n_bins : 1u) <= 0xFFFFFFFFull)
                ? 1u : 0u;
  P.fd_ns = fastdiv_make((uint32_t)std::min<uint64_t>(ns, 0xFFFFFFFFull));
  P.fd_npix = fastdiv_make(std::max<uint32_t>(P.npix, 1u));
  P.fd_cw = fastdiv_make(std::max<uint32_t>(P.cw, 1u));
  P.fd_b = fastdiv_make((uint32_t)d.n_bins);
  P.one_cell_warps = (d.spp_mode == DTS_SPP_PER_CELL && ns >= 32u) ? 1u : 0u;
  {
    const char* sp = getenv("DTS_SPLAT_PLAIN");
    P.splat_plain = (DTS_SPLAT_AGG && sp && sp[0] >= '0' && sp[0] <= '2') ? (uint32_t)(sp[0] - '0') : 2u;
  }
  P.spp_div_b = (uint32_t)(spp / (uint64_t)d.n_bins);
  P.spp_mod_b = (uint32_t)(spp % (uint64_t)d.n_bins);
  cudaStream_t st = (cudaStream_t)stream;
  // histogram cell indices are 32-bit (dts_scene_create rejects larger crops)
  if (npix * (uint64_t)d.n_bins > 0xFFFFFFFFull) return fail(DTS_E_RANGE, "crop_w * crop_h * n_bins must be < 2^32");
  P.cells = (uint32_t)(npix * (uint64_t)d.n_bins);
  {  // culled work items: paths started that miss at once (DTS_CTR_PATHS, DTS_CTR_CAMERA_MISS)
    const uint64_t per_pix = ns * ((darts && d.spp_mode == DTS_SPP_PER_CELL) ? (uint64_t)d.n_bins : 1u);
    const uint64_t culled = (npix - npix_live) * per_pix;
    if (culled && P.counters) {
      add_culled_kernel<<<1, 1, 0, st>>>(P.counters, (unsigned long long)culled);
      g_last_launches = 1;
      CUDA_TRY(cudaGetLastError());
    }
    if (npix_live == 0) {
      return DTS_OK;
    }
  }
  if (darts) {
    P.total = (d.spp_mode == DTS_SPP_PER_CELL) ? npix_live * (uint64_t)d.n_bins * ns : npix_live * ns;
    // kernels stage the 16-bit CDF rows and the 8-bit guide rows; stage-1 SPLIT
    // builds stage the CDF only (binary search) to leave room for the stage-1 queues
    const bool split = kStage1Build && d.direction_mode == DTS_DIR_SPLIT;
    const size_t tbytes = s->table_n * (split ? 2 : 3);
    P.table_u4 = (uint32_t)(tbytes / 16);
    const bool smem = DTS_TABLE_SMEM && tbytes <= 220 * 1024;
    // privatise small histograms (config 1: 128 cells) in shared memory
    const size_t cells = (size_t)npix * (size_t)d.n_bins;
    const size_t pbytes = cells * sizeof(float) * (d_hist_sq ? 2 : 1);
    const size_t kSmemCap = 227 * 1024 - 256;  // opt-in per-block maximum less the static shared memory (mbarrier, counters)
    if (cells <= kPrivMaxCells && (smem ? tbytes : 0) + pbytes <= kSmemCap) P.priv_cells = (uint32_t)cells;
    // per-warp connection-job queues (not with hist_sq: its per-path squares need whole-path sums)
    const size_t qbytes = (size_t)(kJobWords + (split ? kJob1Words : 0)) * kQueue * (kBlock / 32) * sizeof(float);
    // Deferral is opt-in (DTS_DEFER=1): since the immediate kernels run 896-thread
    // CTAs without spills they are as fast or faster on every config (A/B,
    // profiles/README.md: config 5 2.93e10 vs 2.91e10, config 3 2.83e10 vs 2.59e10)
    bool want_defer = false;
    const char* dv = getenv("DTS_DEFER");
    if (dv && (dv[0] == '0' || dv[0] == '1')) want_defer = dv[0] == '1';
    if (d.n_tris > 0 && !smem) return fail(DTS_E_INVALID_ARG, "mesh scenes need the EDA table in shared memory");
    // (row-band launches, which may run concurrently on one scene, never defer:
    // the queue overflow area is per scene and indexed by CTA and warp)
    const bool defer = want_defer && allow_defer && !d_hist_sq && d.n_tris == 0 &&
                       (smem ? tbytes : 0) + (P.priv_cells ? pbytes : 0) + qbytes <= kSmemCap;
    P.defer = defer ? 1u : 0u;
    const char* rk = getenv("DTS_REFILL_K");
    // 8: A/B in profiles/ab_r01_refill*.log (configs 6 / 4 +4 % / +2 %, 5 and 3 +0.2 % / +0.4 % vs 16)
    P.refill_k = rk ? (uint32_t)atoi(rk) : 8u;
    if (P.refill_k < 1 || P.refill_k > 4096) P.refill_k = 8u;
    // warp grabs of kChunk items, but small launches take fewer at a time so that
    // every resident warp gets work (config 1: 2^18 paths) and the tail of a
    // millisecond render stays short: at least 32 grabs per resident warp (2048
    // threads per SM), a multiple of 32 in [32, kChunk].  Configs 2 and 6 (2^24 /
    // 2^23 paths) take 32: +1.2 % / +2.4 % against 128; config 4 (2^26) keeps 128
    // (32: -0.5 %); profiles/ab_r02zf_knobs.log
    {
      const uint64_t warps = (uint64_t)s->num_sms * 64u;
      uint64_t c = P.total / (32u * warps);
      c = c < 32u ? 32u : (c > kChunk ? kChunk : c & ~(uint64_t)31u);
      const char* cv = getenv("DTS_GRAB");
      if (cv && atoi(cv) >= 32 && atoi(cv) <= (int)kChunk) c = (uint64_t)atoi(cv) & ~31u;
      P.chunk = (uint32_t)c;
    }
    // a warp flushes at >= flush_at queued jobs and then pushes <= 32 more: the
    // shared slots plus the kQueue global overflow slots must hold flush_at - 1 + 32
    static_assert(kQueue >= 16, "queue too short for a warp's pushes");
    const uint32_t qcap = std::min<uint32_t>((uint32_t)kQueue, 2u * (uint32_t)kQueue - 31u);
    const char* f1 = getenv("DTS_FLUSH1_AT");
    P.flush1_at = f1 ? (uint32_t)atoi(f1) : std::min<uint32_t>(16u, qcap);
    if (P.flush1_at < 1 || P.flush1_at > qcap) P.flush1_at = std::min<uint32_t>(16u, qcap);
    const char* fa = getenv("DTS_FLUSH_AT");
    P.flush_at = fa ? (uint32_t)atoi(fa) : std::min<uint32_t>(28u, qcap);
    if (P.flush_at < 1 || P.flush_at > qcap) P.flush_at = std::min<uint32_t>(28u, qcap);
    const size_t dyn = (smem ? tbytes : 0) + (P.priv_cells ? pbytes : 0) + (defer ? qbytes : 0);
    const void* kfn = darts_kernel_ptr(smem, defer, d);
    if (!kfn) return fail(DTS_E_INVALID_ARG, "no render kernel for this scene shape");
    int blocks_per_sm = 1;
    CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    const int blk = render_block(defer, d.n_tris > 0);
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kfn, blk, dyn));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    uint64_t grid = (uint64_t)s->num_sms * blocks_per_sm;
    const uint64_t need = (P.total + 31) / 32 / (blk / 32) + 1;
    if (grid > need) grid = need;
    // global overflow queue slots: kQueue x (kJobWords + kJob1Words) floats per
    // warp, twice (the two-stage render's overlapped chunks run two connect kernels)
    const size_t ov1 = (size_t)grid * (kBlock / 32) * kQueue * (kJobWords + kJob1Words);
    if (defer) {
      const size_t ov = 2 * ov1;
      if (ov > s->qover_n) {
        cudaFree(s->d_qover);
        s->d_qover = nullptr;
        s->qover_n = 0;
        if (cudaMalloc(&s->d_qover, ov * sizeof(float)) != cudaSuccess) return fail(DTS_E_OOM, "cudaMalloc(queue overflow) failed");
        s->qover_n = ov;
      }
      P.qover = s->d_qover;
    }
    // two-stage render (walk stage + connect stage, see HandOff) for SPLIT
    // scenes without meshes in BOX / SPHERE media; DTS_WAVEFRONT=0 forces the
    // one-stage kernel (A/B)
    // (DTS_DEFER=1: the connect stage runs the deferred-connection kernel)
    bool wave = d.direction_mode == DTS_DIR_SPLIT && d.n_tris == 0 && d.medium_shape != DTS_MEDIUM_INFINITE;
    const char* wv = getenv("DTS_WAVEFRONT");
    if (wv && wv[0] == '0') wave = false;
    // REUSE scenes: start stage + connect stage (start_kernel) when the table
    // is in shared memory and the medium is bounded; DTS_START_STAGE=0/1 forces
    // the one-stage kernel / the start stage
    bool start2 = d.direction_mode != DTS_DIR_SPLIT && d.medium_shape != DTS_MEDIUM_INFINITE && smem && !defer;
    const char* ss = getenv("DTS_START_STAGE");
    if (ss && ss[0] == '0') start2 = false;
    const void* kwalk = nullptr;
    const void* kres = nullptr;
    int bwalk = kBlockWalk;
    // SPLIT scenes: a start stage (path starts only) ahead of the walk stage
    // (three-stage render) in per-pixel mode, where a start draws two Philox
    // blocks (R21 offset, path start): A/B config 5 +2.2 %, config 3 (per-cell)
    // -0.8 % (profiles/ab_r02_three_stage.log); DTS_START_STAGE=0 / 1 forces
    // it off / on
    const void* kstart3 = nullptr;
    const bool want3 = ss ? ss[0] == '1' : d.spp_mode == DTS_SPP_PER_PIXEL;
    if (wave && want3) kstart3 = pick_fl<PickStartSplit>(d.medium_shape, scene_flags(d));
    if (wave) {
      kwalk = kstart3 ? pick_fl<PickWalkResume>(d.medium_shape, scene_flags(d))
                      : pick_fl<PickWalk>(d.medium_shape, scene_flags(d));
      kres = defer ? (smem ? pick_fl<PickResume<true, true>::F>(d.medium_shape, scene_flags(d))
                           : pick_fl<PickResume<false, true>::F>(d.medium_shape, scene_flags(d)))
                   : (smem ? pick_fl<PickResume<true>::F>(d.medium_shape, scene_flags(d))
                           : pick_fl<PickResume<false>::F>(d.medium_shape, scene_flags(d)));
    } else if (start2) {
      const bool mesh = d.n_tris > 0;
      kwalk = mesh ? pick_fl<PickStartMesh>(d.medium_shape, scene_flags(d))
                   : pick_fl<PickStart>(d.medium_shape, scene_flags(d));
      kres = mesh ? pick_fl<PickResumeMesh>(d.medium_shape, scene_flags(d))
                  : pick_fl<PickResumeReuse>(d.medium_shape, scene_flags(d));
      bwalk = kBlockStart;
    }
    if (!kwalk || !kres) {
      CUDA_TRY(cudaMemsetAsync(work, 0, sizeof(unsigned long long), st));
      CUDA_TRY(table_wait(s, st));
      void* args[] = {&P};
      CUDA_TRY(cudaLaunchKernel(kfn, dim3((unsigned)grid), dim3(blk), args, dyn, st));
      CUDA_TRY(cudaGetLastError());
      g_last_launches += 1;
    } else {
      // connect-stage (and three-stage walk-stage) refills load a hand-off record
      // instead of starting a path: refill on any idle lane (A/B against 8:
      // config 4 +2.2 %, config 2 +1.5 % (at 4); config 5 +1.0 % at 1 against 4,
      // configs 2, 3, 4 within 0.2 %: profiles/ab_r02_start_knobs.log,
      // profiles/ab_r02_refill_resume.log)
      uint32_t refill_resume = 1u;
      const char* rr = getenv("DTS_REFILL_K_RESUME");
      if (rr && atoi(rr) >= 1 && atoi(rr) <= 4096) refill_resume = (uint32_t)atoi(rr);
      int bw = 1;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bw, kwalk, bwalk, 0));
      if (bw < 1) bw = 1;
      const uint64_t gw = (uint64_t)s->num_sms * bw;
      // paths per chunk: the hand-off buffer holds one chunk (64 B per path);
      // 2^27, but at least two chunks for launches of >= 2^21 paths (an 8-GPU
      // rank's share of config 5 is 2^27 paths) so that the second chunk's walk
      // stage fills the first one's tail
      uint64_t chunk = (uint64_t)1 << 27;
      // (the start stage keeps one chunk up to 2^27 paths: one chunk is +5.9 % on
      // config 2 against two overlapped ones, +0.5 % on config 4)
      if (P.total >= ((uint64_t)1 << 21) && !start2) chunk = std::min<uint64_t>(chunk, (P.total + 1) / 2);
      const char* ch = getenv("DTS_WF_CHUNK");
      if (ch && atoll(ch) >= 1024) chunk = std::min<uint64_t>((uint64_t)atoll(ch), (uint64_t)1 << 31);
      if (chunk > P.total) chunk = P.total;
      // dts_render (slot 0) with more than one chunk: two halves, two streams
      const char* ov = getenv("DTS_WF_OVERLAP");
      const bool overlap = slot == 0 && chunk < P.total && !(ov && ov[0] == '0');
      const int halves = overlap ? 2 : 1;
      const size_t cap = (size_t)chunk + (size_t)gw * (bwalk / 32) * kHoBlock;
      // buffers per half: the connect stage's records, and (three-stage) the
      // start stage's records after all halves' connect-stage buffers
      const int nbuf = halves * (kstart3 ? 2 : 1);
      if (s->ho_cap[slot] < cap * nbuf) {
        if (s->d_ho[slot]) {  // (a smaller one: its last use must be over before it is pooled)
          CUDA_TRY(cudaStreamSynchronize(st));
          pool_put(s->device, s->d_ho[slot], s->ho_cap[slot] * sizeof(HandOff));
        }
        s->d_ho[slot] = nullptr;
        s->ho_cap[slot] = 0;
        void* p = nullptr;
        size_t got = 0;
        if (pool_get(s->device, cap * nbuf * sizeof(HandOff), &p, &got) != cudaSuccess)
          return fail(DTS_E_OOM, "cudaMalloc(hand-off buffer) failed");
        s->d_ho[slot] = static_cast<HandOff*>(p);
        s->ho_cap[slot] = got / sizeof(HandOff);
      }
      if (!s->d_wf && cudaMalloc(&s->d_wf, 5 * (2 + kHostBands) * sizeof(unsigned long long)) != cudaSuccess)
        return fail(DTS_E_OOM, "cudaMalloc(two-stage counters) failed");
      cudaStream_t xs[2] = {st, st};
      if (overlap) {
        if (!s->wf_stream) {
          CUDA_TRY(cudaStreamCreateWithFlags(&s->wf_stream, cudaStreamNonBlocking));
          for (int i = 0; i < 2; ++i) CUDA_TRY(cudaEventCreateWithFlags(&s->wf_ev[i], cudaEventDisableTiming));
        }
        xs[1] = s->wf_stream;
        CUDA_TRY(cudaEventRecord(s->wf_ev[0], st));  // fork: the aux stream starts after the caller's prior work
        CUDA_TRY(cudaStreamWaitEvent(xs[1], s->wf_ev[0], 0));
      }
      // (the connect stage of a REUSE scene has its own block size: render_block)
      const int bres = render_block(defer, d.n_tris > 0, !wave);
      const uint64_t gc = std::min<uint64_t>(grid, (cap + 31) / 32 / (bres / 32) + 1);
      uint64_t gs3 = 0;
      if (kstart3) {
        int b3 = 1;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b3, kstart3, kBlockStart, 0));
        gs3 = (uint64_t)s->num_sms * (b3 < 1 ? 1 : b3);
      }
      CUDA_TRY(cudaFuncSetAttribute(kres, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
      int launches = 0;
      int i = 0;
      for (uint64_t w0 = 0; w0 < P.total; w0 += chunk, ++i) {
        const int h = overlap ? (i & 1) : 0;
        cudaStream_t xst = xs[h];
        // counters: slot 0 uses pairs 0 and 1 (halves), slot k >= 1 uses pair k + 1
        // (5 per pair: walk work, connect work, connect slots, start slots, spare)
        unsigned long long* wf = s->d_wf + 5 * (slot == 0 ? h : slot + 1);
        RenderParams PW = P;
        PW.w_base = w0;
        PW.total = std::min<uint64_t>(chunk, P.total - w0);
        PW.work = wf;
        PW.ho = s->d_ho[slot] + (size_t)h * cap;
        PW.ho_count = wf + 2;
        PW.ho_cap = cap;
        // a two-stage walk kernel that starts its own paths (no start stage; config 3)
        // refills at 4 idle lane-iterations: +0.5 % against 8, 1 and 2 even with 8
        // (profiles/ab_r02zn_refill_walk.log); DTS_REFILL_K overrides
        if (wave && !kstart3 && !rk) PW.refill_k = 4u;
        RenderParams PC = PW;
        PC.w_base = 0;
        PC.work = wf + 1;
        PC.refill_k = refill_resume;
        if (defer) PC.qover = s->d_qover + (size_t)h * ov1;
        CUDA_TRY(cudaMemsetAsync(wf, 0, 4 * sizeof(unsigned long long), xst));
        if (kstart3) {  // start stage -> the start records; the walk stage continues them
          RenderParams PS = PW;
          PS.ho = s->d_ho[slot] + (size_t)(halves + h) * cap;
          PS.ho_count = wf + 3;
          void* as[] = {&PS};
          CUDA_TRY(cudaLaunchKernel(kstart3, dim3((unsigned)std::min<uint64_t>(gs3, (PS.total + kBlockStart - 1) / kBlockStart)),
                                    dim3(kBlockStart), as, 0, xst));
          PW.ho_in = PS.ho;
          PW.ho_in_count = PS.ho_count;
          PW.refill_k = refill_resume;
          ++launches;
        }
        void* aw[] = {&PW};
        CUDA_TRY(cudaLaunchKernel(kwalk, dim3((unsigned)std::min<uint64_t>(gw, (PW.total + bwalk - 1) / bwalk)),
                                  dim3(bwalk), aw, 0, xst));
        void* ac[] = {&PC};
        if (i < halves) CUDA_TRY(table_wait(s, xst));  // (once per stream)
        CUDA_TRY(cudaLaunchKernel(kres, dim3((unsigned)gc), dim3(bres), ac, dyn, xst));
        CUDA_TRY(cudaGetLastError());
        launches += 2;
      }
      if (overlap) {  // join: the caller's stream waits for the aux stream's chunks
        CUDA_TRY(cudaEventRecord(s->wf_ev[1], xs[1]));
        CUDA_TRY(cudaStreamWaitEvent(st, s->wf_ev[1], 0));
      }
      g_last_launches += launches;
    }
    g_last_grid = (int)grid;
    g_last_block = (kwalk && kres) ? render_block(defer, d.n_tris > 0, !wave) : blk;  // (the connect stage's)
    g_last_smem = (int)dyn;
  } else {
    P.total = npix_live * ns;
    int bps = 1;
    const void* kfn = vanilla_kernel_ptr(d.medium_shape, d.wall_mask != 0u, d.n_tris > 0);
    if (!kfn) return fail(DTS_E_INVALID_ARG, "no render kernel for this scene shape");
    // per-warp shared-memory histogram rows when a warp's 32 paths share a pixel
    // (>= 32 samples per pixel) and the row is short against the batch's
    // contributions (n_bins <= 128; A/B, profiles/ab_r02_vanilla_rows.log: config 4
    // (1 bin) +23 %, config 1 (128) even, config 3 (512 bins, ~19 vertices per
    // path) -5 %, config 5 (1000) even); DTS_VANILLA_ROWS=0/1 forces off / on
    const char* vr = getenv("DTS_VANILLA_ROWS");
    P.van_rows = (ns >= 32 && d.n_bins <= (vr && vr[0] == '1' ? 2048 : 128) && !(vr && vr[0] == '0')) ? 1u : 0u;
    const size_t vdyn = P.van_rows ? (size_t)(kBlock / 32) * d.n_bins * sizeof(float) : 0;
    CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vdyn));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kfn, kBlock, vdyn));
    uint64_t grid = (uint64_t)s->num_sms * (bps < 1 ? 1 : bps) * 4;
    const uint64_t need = (P.total + kBlock - 1) / kBlock;
    if (grid > need) grid = need;
    void* args[] = {&P};
    CUDA_TRY(cudaLaunchKernel(kfn, dim3((unsigned)grid), dim3(kBlock), args, vdyn, st));
    CUDA_TRY(cudaGetLastError());
    g_last_launches += 1;
    g_last_grid = (int)grid;
    g_last_block = kBlock;
    g_last_smem = (int)vdyn;
  }
  return DTS_OK;
}

extern "C" {

dts_status dts_render(dts_scene_t s, uint64_t spp, uint64_t seed, uint64_t sb, uint64_t se, float* d_hist,
                      float* d_hist_sq, uint64_t* d_counters, void* stream) {
  if (!s) return fail(DTS_E_INVALID_ARG, "scene is NULL");
  return render_impl(s, spp, seed, sb, se, d_hist, d_hist_sq, d_counters, stream, 0,
                     s->desc.crop[3] - s->desc.crop[1], s->d_work, true, 0);
}

static dts_status ensure_bands(dts_scene_t s) {
  if (s->band_stream[0]) return DTS_OK;
  for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamCreateWithFlags(&s->band_stream[i], cudaStreamNonBlocking));
  for (int i = 0; i <= kHostBands; ++i) CUDA_TRY(cudaEventCreateWithFlags(&s->band_ev[i], cudaEventDisableTiming));
  if (cudaMalloc(&s->d_work_band, kHostBands * sizeof(unsigned long long)) != cudaSuccess)
    return fail(DTS_E_OOM, "cudaMalloc(band work counters) failed");
  return DTS_OK;
}

dts_status dts_render_rows(dts_scene_t s, uint64_t spp, uint64_t seed, uint64_t sb, uint64_t se, int32_t row0,
                           int32_t row1, int32_t band, float* d_hist_band, uint64_t* d_counters, void* stream) {
  if (!s) return fail(DTS_E_INVALID_ARG, "scene is NULL");
  const int rows = s->desc.crop[3] - s->desc.crop[1];
  if (row0 < 0 || row1 > rows || row0 >= row1) return fail(DTS_E_INVALID_ARG, "need 0 <= row0 < row1 <= crop height");
  if (band < 0 || band >= kHostBands) return fail(DTS_E_INVALID_ARG, "band must be 0..3");
  dts_status r = ensure_bands(s);
  if (r != DTS_OK) return r;
  return render_impl(s, spp, seed, sb, se, d_hist_band, nullptr, d_counters, stream, row0, row1, s->d_work_band + band,
                     false, 1 + band);
}

dts_status dts_render_host(dts_scene_t s, uint64_t spp, uint64_t seed, uint64_t sb, uint64_t se, float* h_hist,
                           uint64_t* h_counters, void* stream) {
  if (!s || !h_hist) return fail(DTS_E_INVALID_ARG, "NULL argument");
  const size_t n = dts_hist_cells(s);
  cudaStream_t st = (cudaStream_t)stream;
  if (s->d_hist_host_n < n) {  // (capacity in floats; the previous call synchronised its stream)
    pool_put(s->device, s->d_hist_host, s->d_hist_host_n * sizeof(float));
    s->d_hist_host = nullptr;
    s->d_hist_host_n = 0;
    void* p = nullptr;
    size_t got = 0;
    if (pool_get(s->device, n * sizeof(float), &p, &got) != cudaSuccess) return fail(DTS_E_OOM, "cudaMalloc(hist) failed");
    s->d_hist_host = static_cast<float*>(p);
    s->d_hist_host_n = got / sizeof(float);
  }
  if (!s->d_ctr_host && cudaMalloc(&s->d_ctr_host, DTS_NUM_COUNTERS * sizeof(uint64_t)) != cudaSuccess)
    return fail(DTS_E_OOM, "cudaMalloc(counters) failed");
  CUDA_TRY(cudaMemsetAsync(s->d_hist_host, 0, n * sizeof(float), st));
  CUDA_TRY(cudaMemsetAsync(s->d_ctr_host, 0, DTS_NUM_COUNTERS * sizeof(uint64_t), st));
  const dts_scene_desc& d = s->desc;
  const int rows = d.crop[3] - d.crop[1];
  const size_t row_cells = (size_t)(d.crop[2] - d.crop[0]) * (size_t)d.n_bins;
  // large histograms (config 5: 4.2 GB, ~170 ms over PCIe): kHostBands row bands
  // on two streams; band k's copy to the host overlaps band k+1's render (and
  // band k's tail overlaps band k+1's start), the last band is 1/32 of the rows.
  // Same paths, same ids.
  const bool banded = n * sizeof(float) >= ((size_t)256 << 20) && rows >= 2 * kHostBands && sb < se;
  if (!banded) {
    dts_status r = dts_render(s, spp, seed, sb, se, s->d_hist_host, nullptr, s->d_ctr_host, stream);
    if (r != DTS_OK) return r;
    CUDA_TRY(cudaMemcpyAsync(h_hist, s->d_hist_host, n * sizeof(float), cudaMemcpyDeviceToHost, st));
  } else {
    const dts_status eb = ensure_bands(s);
    if (eb != DTS_OK) return eb;
    CUDA_TRY(cudaEventRecord(s->band_ev[kHostBands], st));
    for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamWaitEvent(s->band_stream[i], s->band_ev[kHostBands], 0));
    // the last band is short (1/32 of the rows): only its copy is not hidden
    // behind a later band's render
    const int cut = rows - std::max(1, rows / 32);
    for (int k = 0; k < kHostBands; ++k) {
      const int r0 = k < kHostBands - 1 ? cut * k / (kHostBands - 1) : cut;
      const int r1 = k < kHostBands - 1 ? cut * (k + 1) / (kHostBands - 1) : rows;
      cudaStream_t bs = s->band_stream[k & 1];
      dts_status r = render_impl(s, spp, seed, sb, se, s->d_hist_host + (size_t)r0 * row_cells, nullptr,
                                 s->d_ctr_host, bs, r0, r1, s->d_work_band + k, false, 1 + k);
      if (r != DTS_OK) return r;
      CUDA_TRY(cudaEventRecord(s->band_ev[k], bs));
      CUDA_TRY(cudaStreamWaitEvent(st, s->band_ev[k], 0));
      CUDA_TRY(cudaMemcpyAsync(h_hist + (size_t)r0 * row_cells, s->d_hist_host + (size_t)r0 * row_cells,
                               (size_t)(r1 - r0) * row_cells * sizeof(float), cudaMemcpyDeviceToHost, st));
    }
  }
  if (h_counters)
    CUDA_TRY(cudaMemcpyAsync(h_counters, s->d_ctr_host, DTS_NUM_COUNTERS * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return DTS_OK;
}

dts_status dts_sample_debug(dts_scene_t s, int32_t n, const dts_debug_in* d_in, dts_debug_out* d_out, void* stream) {
  if (!s || (n > 0 && (!d_in || !d_out)) || n < 0) return fail(DTS_E_INVALID_ARG, "bad arguments");
  if (n == 0) return DTS_OK;
  if (s->desc.strategy != DTS_STRATEGY_VANILLA && !s->d_table) return fail(DTS_E_STATE, "table not built");
  const uint16_t* tab = s->d_table;
  if (!tab) {
    // vanilla scenes have no table: the debug kernel reads a zero cell (gamma = 0)
    if (!s->d_zero_cell) {
      if (cudaMalloc(&s->d_zero_cell, 3 * 256) != cudaSuccess) return fail(DTS_E_OOM, "cudaMalloc(zero cell) failed");
      CUDA_TRY(cudaMemset(s->d_zero_cell, 0, 3 * 256));
    }
    tab = s->d_zero_cell;
  }
  const void* kfn = debug_kernel_ptr(s->desc);
  if (!kfn) return fail(DTS_E_INVALID_ARG, "no debug kernel for this scene shape");
  DevScene S = s->S;
  set_round_keys(S, 0);
  void* args[] = {&S, &tab, &n, &d_in, &d_out};
  if (s->d_table) CUDA_TRY(table_wait(s, (cudaStream_t)stream));
  CUDA_TRY(cudaLaunchKernel(kfn, dim3((n + 127) / 128), dim3(128), args, 0, (cudaStream_t)stream));
  CUDA_TRY(cudaGetLastError());
  return DTS_OK;
}

dts_status dts_check_failures(uint64_t* out) {
  if (!out) return fail(DTS_E_INVALID_ARG, "NULL argument");
  unsigned long long v = 0, z = 0;
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpyFromSymbol(&v, dts::g_dts_check_fail, sizeof v));
  CUDA_TRY(cudaMemcpyToSymbol(dts::g_dts_check_fail, &z, sizeof z));
  *out = (uint64_t)v;
  return DTS_OK;
}

dts_status dts_pool_release(void) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (const PoolBuf& b : g_pool) cudaFree(b.p);
  g_pool.clear();
  return DTS_OK;
}

dts_status dts_enable_peer(int32_t peer) {
  int dev = 0, n = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaGetDeviceCount(&n));
  if (peer < 0 || peer >= n) return fail(DTS_E_INVALID_ARG, "peer device out of range");
  if (peer == dev) return DTS_OK;
  int can = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can, dev, peer));
  if (!can) return fail(DTS_E_CUDA, "no peer access from the current device to the peer");
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free error state
    return DTS_OK;
  }
  CUDA_TRY(e);
  return DTS_OK;
}

dts_status dts_last_launch(int32_t* n_launches, int32_t* grid, int32_t* block, int32_t* smem_bytes) {
  if (n_launches) *n_launches = g_last_launches;
  if (grid) *grid = g_last_grid;
  if (block) *block = g_last_block;
  if (smem_bytes) *smem_bytes = g_last_smem;
  return DTS_OK;
}

}  // extern "C"
