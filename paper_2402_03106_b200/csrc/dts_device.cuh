// dts_device.cuh -- device stages of the DARTS hot path (sm_100a, fp32).
//
// One DARTS vertex = direction (EDA (+) HG one-sample MIS),
// one analytic intersection reused by the connection and the walk
// (PAPER.md:287), elliptical connection (E20-E22) and DA-RIS
// free-path sampling (E9-E15).  The same functions serve the
// persistent render kernel and the dts_sample_debug kernel (template DBG).
// Readings R1..R29: DESIGN.md section 3.  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dts.h"

namespace dts {

// Device-side bounds checks of the check build (-DDTS_CHECKS=1, see
// dts_check_failures in dts.h): a failed check is counted, never trapped
// (compute-sanitizer is not available on the GPU pool).
#ifndef DTS_CHECKS
#define DTS_CHECKS 0
#endif
__device__ unsigned long long g_dts_check_fail;
#define DTS_CHECK(cond)                                              \
  do {                                                               \
    if (DTS_CHECKS && !(cond)) atomicAdd(&dts::g_dts_check_fail, 1ull); \
  } while (0)

constexpr float kPi = 3.14159265358979323846f;
constexpr float kInv4Pi = 0.0795774715459476679f;
constexpr float kLog2e = 1.44269504088896341f;
constexpr float kLn2 = 0.693147180559945309f;

enum { HIT_NONE = 0, HIT_OPEN = 1, HIT_WALL = 2, HIT_MISS = 3, HIT_SURF = 4 };
enum { KIND_CAMERA = 0, KIND_MEDIUM = 1, KIND_WALL = 2, KIND_SURF = 3 };
// compile-time scene variant flags of the render / debug kernels
enum { FL_WALLS = 1, FL_SPLIT = 2, FL_MULTI_E = 4, FL_MESH = 8 };
constexpr float kSurfEps = 1e-4f;  // R33: surface vertices sit this far off their triangle

// Launch-uniform scene constants, passed by value as a kernel parameter (lives
// in the constant bank: every lane reads the same address).
struct DevScene {
  float sigma_s, sigma_a, sigma_t, albedo, g, inv_sigma_t;
  float hg_k;        // (1 - g^2) / (4 pi)
  float hg_1pg2;     // 1 + g^2
  float hg_2g;       // 2 g
  float hg_1mg2;     // 1 - g^2
  float hg_1mg;      // 1 - g
  float hg_1pg;      // 1 + g
  float neg_inv4D_log2e;   // -log2(e) / (4 D)
  float neg_sa_log2e;      // -sigma_a log2(e)
  int32_t medium_shape;
  float center[3], radius2;
  float bmin[3], bmax[3];
  uint32_t wall_mask;
  float wall_albedo[6];
  int32_t n_emitters;
  float em_pos[DTS_MAX_EMITTERS][3];
  float em_t[DTS_MAX_EMITTERS];
  float em_k[DTS_MAX_EMITTERS];  // P_e / (4 pi) * N_e
  int32_t camera_kind;
  float cam_pos[3], fwd[3], right[3], upc[3];
  float tan_half, aspect;
  int32_t width, height;
  float det_radius;
  int32_t crop[4];
  double t0, dt;
  float dt_f;  // (float) dt
  int32_t n_bins, warped;
  int32_t strategy, direction_mode, spp_mode, max_bounces;
  int32_t conn_uniform;  // 1: P of S uniform (ablation of PAPER.md:295)
  float alpha;
  float r_excl, s_excess;
  float far_e;  // largest distance from an emitter to a point of the medium (+ margin; inf for INFINITE)
  // EDA table (R8-R10)
  int32_t nr, ns;
  float nr_f, ns_f;
  uint32_t table_n;        // CDF entries; an 8-bit guide table of the same length follows them
  float ln_smin, inv_dls;  // ns / (ln smax - ln smin)
  uint32_t seed_lo, seed_hi;
  uint32_t rk[20];  // Philox round keys (k0_r, k1_r), r = 0..9, of the launch's seed
  // triangle meshes (R32, R33): BVH nodes in depth-first order, 2 float4 each:
  // (lo.xyz, int a), (hi.xyz, int n): n > 0 leaf of triangles [a, a + n), n = 0
  // inner node with children node + 1 and a; triangles in leaf order, 3 float4
  // each: (v0.xyz, int material), (e1.xyz, -), (e2.xyz, -)
  const float4* bvh;
  const float4* tri4;
  const int32_t* tri_leaf;  // caller's triangle index -> leaf order (debug records)
  const int32_t* tri_orig;  // leaf order -> caller's triangle index (debug output)
  int32_t n_tris;
  // R32 per material: select ks, f = kd + kl pow(ca, n), p = pd cos + pl pow(ca, n), 1 / (n + 1)
  float mat_ks[DTS_MAX_MATERIALS], mat_kd[DTS_MAX_MATERIALS], mat_kl[DTS_MAX_MATERIALS];
  float mat_pd[DTS_MAX_MATERIALS], mat_pl[DTS_MAX_MATERIALS], mat_n[DTS_MAX_MATERIALS];
  float mat_inv_n1[DTS_MAX_MATERIALS];
};

// ----------------------------------------------------------------- vectors
struct f3 {
  float x, y, z;
};
__device__ __forceinline__ f3 mk(float x, float y, float z) { return f3{x, y, z}; }
__device__ __forceinline__ f3 operator+(f3 a, f3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ f3 operator-(f3 a, f3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ f3 operator*(f3 a, float s) { return mk(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float dot(f3 a, f3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ f3 fma3(f3 d, float t, f3 o) { return mk(fmaf(d.x, t, o.x), fmaf(d.y, t, o.y), fmaf(d.z, t, o.z)); }
__device__ __forceinline__ f3 ld3(const float* p) { return mk(p[0], p[1], p[2]); }
// double <-> float conversions as single F2F instructions (a C cast under
// --ftz adds a denormal test and a rescale; the values here are never denormal)
__device__ __forceinline__ float d2f(double x) {
  float r;
  asm("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double f2d(float x) {
  double r;
  asm("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(x));
  return r;
}

// ----------------------------------------------------------------- RNG (R24)
// Philox4x32-10 (Salmon et al. 2011); counter = (id_lo, id_hi, bounce, block).
// The key schedule depends only on the seed: the 10 round keys are computed
// once per launch on the host (DevScene::rk) and read from the constant bank,
// so a round is 2 IMAD.WIDE.U32 + 2 LOP3.
struct u4 {
  uint32_t a, b, c, d;
};
__device__ __forceinline__ u4 philox_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const uint32_t* rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;  // IMAD.WIDE.U32
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ rk[2 * r], n2 = hi0 ^ c3 ^ rk[2 * r + 1];
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return u4{c0, c1, c2, c3};
}
// R24: u = (r >> 9) 2^-23, built as a float in [1, 2) minus one (no int->float conversion)
__device__ __forceinline__ float mant01(uint32_t m23) { return __uint_as_float(0x3f800000u | m23) - 1.0f; }
__device__ __forceinline__ float unif(uint32_t r) { return mant01(r >> 9); }
// floor(n u) for u = unif(r), exactly: (n (r >> 9)) >> 23 (R20 emitter index,
// R21 bin offset).  Index work is integer work: an fp32 n * u rounds up across
// a slice boundary for ~2e-5 of the draws when n is not a power of two.
__device__ __forceinline__ uint32_t unif_index(uint32_t n, uint32_t r) {
  return (uint32_t)(((uint64_t)n * (uint64_t)(r >> 9)) >> 23);
}

// Small integer <-> float conversions on the FMA/ALU pipes instead of the XU
// pipe (I2F/F2I share it with MUFU, ~60 % busy in the DARTS vertex):
// u23f(x) = x exactly for x <= 2^23; f2u23(x) = floor(x) for 0 <= x < 2^23.
#ifndef DTS_MAGIC_CVT
#define DTS_MAGIC_CVT 0
#endif
__device__ __forceinline__ float u23f(uint32_t x) {
  if (DTS_MAGIC_CVT) return __uint_as_float(0x4B000000u + x) - 8388608.0f;
  return (float)x;
}
__device__ __forceinline__ uint32_t f2u23(float x) {
  if (DTS_MAGIC_CVT) return __float_as_uint(__fadd_rd(x, 8388608.0f)) - 0x4B000000u;
  return (uint32_t)x;
}

// ----------------------------------------------------------------- packed fp32 (sm_100 FADD2/FMUL2/FFMA2)
// Two independent IEEE fp32 operations per issue slot: the same round-to-
// nearest results as the scalar instructions, half the issue cost.  The path
// kernel is issue-bound, so the 8 RIS candidates are evaluated
// in pairs.  DTS_F32X2=0 builds the scalar form (A/B).
#ifndef DTS_F32X2
#define DTS_F32X2 1
#endif
__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ float2 f2s(float x) { return make_float2(x, x); }
#if DTS_F32X2
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
#else
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return f2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return f2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return f2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y)); }
#endif

// ----------------------------------------------------------------- accurate small-argument helpers
// -ln(1 - x) for x in [0, 1): series x + x^2/2 + x^3/3 below 1/64 (relative
// truncation error < x^3/4 < 1e-6), MUFU lg2 above (relative error < 1e-5).
__device__ __forceinline__ float neg_log1m(float x) {
  const float big = -__log2f(1.0f - x) * kLn2;
  const float ser = x * fmaf(x, fmaf(x, 0.33333334f, 0.5f), 1.0f);
  return x < 0.015625f ? ser : big;
}
// -ln(1 - x) with 1 - x supplied separately (omx, formed without cancellation
// by the caller: for x = u p with p = 1 - T, 1 - x = (1 - u) + u T stays
// accurate even when x -> 1).
__device__ __forceinline__ float neg_log1m2(float x, float omx) {
  const float big = -__log2f(omx) * kLn2;
  const float ser = x * fmaf(x, fmaf(x, 0.33333334f, 0.5f), 1.0f);
  return x < 0.015625f ? ser : big;
}
// 1 - exp(-y) for y >= 0
__device__ __forceinline__ float one_m_exp(float y) {
  const float big = 1.0f - exp2f(-y * kLog2e);
  const float ser = y * fmaf(-y, fmaf(-y, fmaf(-y, fmaf(-y, 1.0f / 120.0f, 1.0f / 24.0f), 1.0f / 6.0f), 0.5f), 1.0f);
  return y < 0.0625f ? ser : big;
}
__device__ __forceinline__ float fexp(float x) { return exp2f(x * kLog2e); }
// 1 - exp(-y) given T = fexp(-y) (the same value one_m_exp computes; one MUFU for both)
__device__ __forceinline__ float one_m_exp_T(float y, float T) {
  const float ser = y * fmaf(-y, fmaf(-y, fmaf(-y, fmaf(-y, 1.0f / 120.0f, 1.0f / 24.0f), 1.0f / 6.0f), 0.5f), 1.0f);
  return y < 0.0625f ? ser : 1.0f - T;
}

// ----------------------------------------------------------------- frames (R12)
// Direction at polar angle theta about n: cos theta and sin theta are built
// from opc = 1 + cos and omc = 1 - cos, each computed without cancellation by
// the caller, so directions near the pole (HG with g = 0.9) keep fp32 accuracy.
__device__ __forceinline__ f3 from_frame(f3 n, float opc, float omc, float phi) {
  // R12 tie-break: n_z >= -1e-6 takes the +z chart, so a structurally horizontal
  // normal (mesh facets) picks the same frame whatever the sign of its rounded n_z
  const float sign = n.z >= -1e-6f ? 1.0f : -1.0f;
  const float a = __fdividef(-1.0f, sign + n.z);  // sign + n.z in [1, 2]
  const float b = n.x * n.y * a;
  const f3 b1 = mk(1.0f + sign * n.x * n.x * a, sign * b, -sign * n.x);
  const f3 b2 = mk(b, sign + n.y * n.y * a, -n.y);
  const float cos_t = opc < omc ? opc - 1.0f : 1.0f - omc;
  const float sin_t = sqrtf(fmaxf(0.0f, opc * omc));
  float sp, cp;
  __sincosf(phi, &sp, &cp);
  const float cx = sin_t * cp, cy = sin_t * sp;
  return mk(b1.x * cx + b2.x * cy + n.x * cos_t, b1.y * cx + b2.y * cy + n.y * cos_t,
            b1.z * cx + b2.z * cy + n.z * cos_t);
}

// ----------------------------------------------------------------- HG
__device__ __forceinline__ float hg_eval(const DevScene& S, float mu) {
  const float den = fmaf(-S.hg_2g, mu, S.hg_1pg2);
  const float r = rsqrtf(den);
  return S.hg_k * r * r * r;
}
// HG inverse CDF (R25): returns 1 + cos and 1 - cos of the sampled angle.
// With den = 1 - g + 2 g u and sq = (1 - g^2) / den (the textbook form
// cos = (1 + g^2 - sq^2) / (2g)):
//   1 - cos = (1 - g)(1 - u)(sq + 1 - g) / den,  1 + cos = (1 + g) u (sq + 1 + g) / den.
__device__ __forceinline__ void hg_sample(const DevScene& S, float u, float& opc, float& omc) {
  if (S.g == 0.0f) {
    opc = 2.0f * (1.0f - u);
    omc = 2.0f * u;
    return;
  }
  const float den = fmaf(S.hg_2g, u, S.hg_1mg);
  const float inv = __fdividef(1.0f, den);
  const float sq = S.hg_1mg2 * inv;
  omc = S.hg_1mg * (1.0f - u) * (sq + S.hg_1mg) * inv;
  opc = S.hg_1pg * u * (sq + S.hg_1pg) * inv;
}

// ----------------------------------------------------------------- medium bounds (R15)
template <int SH, bool WALLS>
__device__ __forceinline__ int intersect(const DevScene& S, f3 o, f3 d, float& lo, float& hi, int& face) {
  face = -1;
  if (SH == DTS_MEDIUM_INFINITE) {
    lo = 0.0f;
    hi = __int_as_float(0x7f800000);
    return HIT_NONE;
  }
  if (SH == DTS_MEDIUM_SPHERE) {
    const f3 oc = o - ld3(S.center);
    const float b = dot(oc, d);
    const float c = dot(oc, oc) - S.radius2;
    const float disc = b * b - c;
    if (!(disc > 0.0f)) return HIT_MISS;
    const float s = sqrtf(disc);
    // roots without cancellation: tf = s - b, or -c / (b + s) when b > 0; tn tf = c
    const float tf = b > 0.0f ? -c * __fdividef(1.0f, b + s) : s - b;
    if (!(tf > 0.0f)) return HIT_MISS;
    const float tn = b > 0.0f ? -b - s : c * __fdividef(1.0f, tf);
    lo = fmaxf(tn, 0.0f);
    hi = tf;
    return HIT_OPEN;
  }
  // branchless slab test; 1/0 = inf and fminf/fmaxf drop the NaN of 0 * inf
  const float ix = __fdividef(1.0f, d.x), iy = __fdividef(1.0f, d.y), iz = __fdividef(1.0f, d.z);
  const float ax = (S.bmin[0] - o.x) * ix, bx = (S.bmax[0] - o.x) * ix;
  const float ay = (S.bmin[1] - o.y) * iy, by = (S.bmax[1] - o.y) * iy;
  const float az = (S.bmin[2] - o.z) * iz, bz = (S.bmax[2] - o.z) * iz;
  const float fx = fmaxf(ax, bx), fy = fmaxf(ay, by), fz = fmaxf(az, bz);
  const float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), 0.0f));
  const float tf = fminf(fminf(fx, fy), fz);
  if (!(tf > tn)) return HIT_MISS;
  // exit face: first axis attaining tf (ties -> lowest axis)
  const int axis = (fx == tf) ? 0 : ((fy == tf) ? 1 : 2);
  const float da = axis == 0 ? d.x : (axis == 1 ? d.y : d.z);
  const int ff = 2 * axis + (da > 0.0f ? 1 : 0);
  lo = tn;
  hi = tf;
  face = ff;
  return (WALLS && ((S.wall_mask >> ff) & 1u)) ? HIT_WALL : HIT_OPEN;
}

// Exit of a ray that starts inside the medium (medium and wall vertices,
// control vertices): lo = 0 and only the far root / the nearest exit plane is
// needed.  Same result as intersect() for an inside origin.
template <int SH, bool WALLS>
__device__ __forceinline__ int intersect_inside(const DevScene& S, f3 o, f3 d, float& lo, float& hi, int& face) {
  lo = 0.0f;
  face = -1;
  if (SH == DTS_MEDIUM_INFINITE) {
    hi = __int_as_float(0x7f800000);
    return HIT_NONE;
  }
  if (SH == DTS_MEDIUM_SPHERE) {
    const f3 oc = o - ld3(S.center);
    const float b = dot(oc, d);
    const float c = dot(oc, oc) - S.radius2;
    const float disc = b * b - c;
    if (!(disc > 0.0f)) return HIT_MISS;
    const float s = sqrtf(disc);
    const float tf = b > 0.0f ? -c * __fdividef(1.0f, b + s) : s - b;
    if (!(tf > 0.0f)) return HIT_MISS;
    hi = tf;
    return HIT_OPEN;
  }
  // the exit plane of each axis by the sign BIT of d: a +0 or -0 component then
  // gives (plane - o) * (1/d) = +inf (the ray never leaves through that axis);
  // a "d > 0" test would pick the wrong plane for +0 and return -inf
  const float tx = ((__float_as_int(d.x) >= 0 ? S.bmax[0] : S.bmin[0]) - o.x) * __fdividef(1.0f, d.x);
  const float ty = ((__float_as_int(d.y) >= 0 ? S.bmax[1] : S.bmin[1]) - o.y) * __fdividef(1.0f, d.y);
  const float tz = ((__float_as_int(d.z) >= 0 ? S.bmax[2] : S.bmin[2]) - o.z) * __fdividef(1.0f, d.z);
  const float tf = fminf(fminf(tx, ty), tz);  // NaN (0 * inf, an origin on a plane) is dropped
  if (!(tf > 0.0f)) return HIT_MISS;
  hi = tf;
  if (!WALLS) return HIT_OPEN;  // the exit face only matters when some face is a wall
  const int axis = (tx == tf) ? 0 : ((ty == tf) ? 1 : 2);
  const float da = axis == 0 ? d.x : (axis == 1 ? d.y : d.z);
  const int ff = 2 * axis + (da > 0.0f ? 1 : 0);
  face = ff;
  return ((S.wall_mask >> ff) & 1u) ? HIT_WALL : HIT_OPEN;
}

// ----------------------------------------------------------------- triangle meshes (R32, R33)
__device__ __forceinline__ f3 cross(f3 a, f3 b) {
  return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
// Nearest triangle hit with 0 < t < t_max over the BVH (ANY: the first hit
// found, for visibility); returns the triangle (leaf order) or -1.  Moller-
// Trumbore with inclusive edges, the test of the oracle in fp32.
// (Inlined by default, DTS_MESH_INLINE=0 builds it out of line; takes the two
// array pointers rather than the scene, whose address would force a local copy.)
#ifndef DTS_MESH_INLINE
#define DTS_MESH_INLINE 1
#endif
#if DTS_MESH_INLINE
#define DTS_MESH_FN __forceinline__
#else
#define DTS_MESH_FN __noinline__
#endif
template <bool ANY>
__device__ DTS_MESH_FN int mesh_trace_impl(const float4* __restrict__ bvh, const float4* __restrict__ tri4, f3 o, f3 d,
                                            float t_max, float& t_hit) {
  const f3 inv = mk(__fdividef(1.0f, d.x), __fdividef(1.0f, d.y), __fdividef(1.0f, d.z));
  int stack[40];
  int sp = 0, node = 0, best = -1;
  float tb = t_max;
  while (true) {
    const float4 a = __ldg(bvh + 2 * node), b = __ldg(bvh + 2 * node + 1);
    const float ax = (a.x - o.x) * inv.x, bx = (b.x - o.x) * inv.x;
    const float ay = (a.y - o.y) * inv.y, by = (b.y - o.y) * inv.y;
    const float az = (a.z - o.z) * inv.z, bz = (b.z - o.z) * inv.z;
    const float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), 0.0f));
    const float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fmaxf(az, bz));
    if (tn <= tf && tn < tb) {
      const int first = __float_as_int(a.w), cnt = __float_as_int(b.w);
      if (cnt == 0) {  // inner node: near side first is not needed for correctness
        stack[sp++] = first;
        ++node;
        continue;
      }
      for (int i = first; i < first + cnt; ++i) {
        const float4 t0 = __ldg(tri4 + 3 * i), t1 = __ldg(tri4 + 3 * i + 1), t2 = __ldg(tri4 + 3 * i + 2);
        const f3 e1 = mk(t1.x, t1.y, t1.z), e2 = mk(t2.x, t2.y, t2.z);
        const f3 pv = cross(d, e2);
        const float det = dot(e1, pv);
        const float idet = __fdividef(1.0f, det);
        const f3 sv = o - mk(t0.x, t0.y, t0.z);
        const float u = dot(sv, pv) * idet;
        const f3 qv = cross(sv, e1);
        const float v = dot(d, qv) * idet;
        const float t = dot(e2, qv) * idet;
        if (det != 0.0f && u >= 0.0f && v >= 0.0f && u + v <= 1.0f && t > 0.0f && t < tb) {
          tb = t;
          best = i;
          if (ANY) {
            t_hit = tb;
            return best;
          }
        }
      }
    }
    if (sp == 0) break;
    node = stack[--sp];
  }
  t_hit = tb;
  return best;
}
template <bool ANY>
__device__ __forceinline__ int mesh_trace(const DevScene& S, f3 o, f3 d, float t_max, float& t_hit) {
  return mesh_trace_impl<ANY>(S.bvh, S.tri4, o, d, t_max, t_hit);
}
// geometric normal of triangle tri turned to the side the direction w arrives from
__device__ __forceinline__ f3 tri_side_normal(const DevScene& S, int tri, f3 w, int& mat) {
  const float4 t0 = __ldg(S.tri4 + 3 * tri), t1 = __ldg(S.tri4 + 3 * tri + 1), t2 = __ldg(S.tri4 + 3 * tri + 2);
  f3 n = cross(mk(t1.x, t1.y, t1.z), mk(t2.x, t2.y, t2.z));
  n = n * rsqrtf(dot(n, n));
  mat = __float_as_int(t0.w);
  return dot(n, w) > 0.0f ? n * -1.0f : n;
}
// max(0, c)^n with 0^0 = 1 (pow of the oracle)
__device__ __forceinline__ float lobe_pow(float c, float n) {
  return c > 0.0f ? exp2f(n * __log2f(c)) : (n == 0.0f ? 1.0f : 0.0f);
}
// R32: f(w -> wo) = rho [(1 - ks) / pi + ks (n + 2) / (2 pi) max(0, wo . r)^n], r = mirror of w
__device__ __forceinline__ float bsdf_eval(const DevScene& S, int mat, f3 n, f3 w, f3 wo) {
  if (!(dot(wo, n) > 0.0f)) return 0.0f;
  const f3 r = w - n * (2.0f * dot(w, n));
  return fmaf(S.mat_kl[mat], lobe_pow(dot(wo, r), S.mat_n[mat]), S.mat_kd[mat]);
}

// R32 sampling at a surface vertex with normal n (incident side) and incident
// direction w: u_lobe < ks picks the lobe (cos alpha = u^{1/(n+1)} about the
// mirror direction), else the cosine hemisphere (cos theta = sqrt(1 - u));
// phi = 2 pi u_phi.  Writes wo; returns f cos / p_mix, 0 below the surface.
__device__ __forceinline__ float bsdf_sample(const DevScene& S, int mat, f3 n, f3 w, float u_lobe, float u,
                                             float u_phi, f3& wo) {
  const float phi = 2.0f * kPi * u_phi;
  const f3 rm = w - n * (2.0f * dot(w, n));
  if (u_lobe < S.mat_ks[mat]) {
    // 1 - cos alpha = 1 - u^{1/(n+1)} = 1 - e^{ln(u)/(n+1)} without cancellation
    // (a sharp lobe puts cos alpha within 1e-5 of 1)
    const float omc = one_m_exp(-__log2f(u) * (kLn2 * S.mat_inv_n1[mat]));
    wo = from_frame(rm, 2.0f - omc, omc, phi);
  } else {
    const float lz = sqrtf(1.0f - u);
    wo = from_frame(n, 1.0f + lz, __fdividef(u, 1.0f + lz), phi);
  }
  const float co = dot(wo, n);
  if (!(co > 0.0f)) return 0.0f;
  const float pw = lobe_pow(dot(wo, rm), S.mat_n[mat]);
  return fmaf(S.mat_kl[mat], pw, S.mat_kd[mat]) * co * __fdividef(1.0f, fmaf(S.mat_pd[mat], co, S.mat_pl[mat] * pw));
}

// medium length of the segment p -> xe (p inside the medium, dir its unit
// direction, r its length), or -1 if the segment is occluded
template <int SH, bool WALLS, bool MESH = false>
__device__ __forceinline__ float segment_len(const DevScene& S, f3 p, float r, f3 dir) {
  if (MESH) {  // R32: a triangle on the segment occludes it
    float tm;
    if (mesh_trace<true>(S, p, dir, r, tm) >= 0) return -1.0f;
  }
  if (SH == DTS_MEDIUM_INFINITE) return r;
  float lo, hi;
  int face;
  const int hit = intersect_inside<SH, WALLS>(S, p, dir, lo, hi, face);
  if (hit == HIT_MISS) return 0.0f;
  if (WALLS && hit == HIT_WALL && hi < r) return -1.0f;  // occluded by a wall (R15)
  return fmaxf(0.0f, fminf(hi, r) - lo);
}
// its transmittance (0 when occluded)
template <int SH, bool WALLS, bool MESH = false>
__device__ __forceinline__ float segment_tr(const DevScene& S, f3 p, f3 xe, float r, f3 dir) {
  const float len = segment_len<SH, WALLS, MESH>(S, p, r, dir);
  return len < 0.0f ? 0.0f : fexp(-S.sigma_t * len);
}

__device__ __forceinline__ f3 inward_normal(int face) {
  const float s = (face & 1) ? -1.0f : 1.0f;
  const int a = face >> 1;
  return mk(a == 0 ? s : 0.0f, a == 1 ? s : 0.0f, a == 2 ? s : 0.0f);
}

// ----------------------------------------------------------------- path state
struct PathState {
  f3 x, w;      // position, incoming direction (camera: primary direction)
  double resM;  // upper residual R_M - E = T_M - tau_e - elapsed (E5); R_m - E = resM - dt
  float beta;
  int kind, face;
  int e;        // emitter
};

// EDA table access (R10): 16-bit CDF rows of 256 per cell, followed by an
// 8-bit guide row per cell: guide[g] = largest j with q_j <= 256 g.
template <bool SMEM>
__device__ __forceinline__ uint32_t qload(const uint16_t* q, int i) {
  if (SMEM) return q[i];
  return __ldg(q + i);
}
template <bool SMEM>
__device__ __forceinline__ uint32_t gload(const uint8_t* g, int i) {
  if (SMEM) return g[i];
  return __ldg(g + i);
}

// R24: the SPLIT walk direction uses u8, u9, made of bits of the first Philox
// block that u0..u3 leave unused (u0, u2, u3: top 23 bits of r0, r2, r3; the
// Sobol row of u1: top 5 bits of r1): u8 = bits 0..22 of r1; u9 = bits 0..8 of
// r0 | bits 0..8 of r2 | bits 0..4 of r3.  So a walk-only vertex (two-stage
// render) needs one Philox call.
__device__ __forceinline__ float u8_split(const uint32_t (&r)[8]) { return mant01(r[1] & 0x7FFFFFu); }
__device__ __forceinline__ float u9_split(const uint32_t (&r)[8]) {
  return mant01(((r[0] & 0x1FFu) << 14) | ((r[2] & 0x1FFu) << 5) | (r[3] & 0x1Fu));
}

// ----------------------------------------------------------------- elliptical connection (E20-E22)
// Samples S on [C + dlo, C + dlo + width) from the truncated exponential of
// PAPER.md:295 and maps it to the polar distance t of E21; p_t is E22 with the
// Jacobian of R2.  cv = xe - x, C = |cv|, q = wc . cv.
struct EllSample {
  float t, pt, pSt, S;  // pSt = S - t (= r2 on the ellipse)
};
__device__ __forceinline__ EllSample ell_sample(const DevScene& S, f3 cv, float C, float q, f3 wc, float dlo,
                                                float width, float u7) {
  // truncated exponential on [S_lo, S_hi); e^{-st (S-S_lo)} = 1 - u7 span
  float L, pS;
  if (S.conn_uniform) {  // ablation: P uniform on [S_lo, S_hi)
    L = u7 * width;
    pS = __fdividef(1.0f, width);
  } else {
    const float span = one_m_exp(S.sigma_t * width);
    const float keep = fmaf(u7, fexp(-S.sigma_t * width), 1.0f - u7);  // 1 - u7 span
    L = neg_log1m2(u7 * span, keep) * S.inv_sigma_t;
    pS = S.sigma_t * keep * __fdividef(1.0f, span);
  }
  const float dSC = dlo + L;  // S - C
  const float Ssm = C + dSC;
  // S - q = (S - C) + (C - q), C - q = perp^2 / (C + q) for q > 0
  const f3 pv = cv - wc * q;
  const float perp2 = dot(pv, pv);
  const float Cmq = q > 0.0f ? perp2 * __fdividef(1.0f, C + q) : C - q;
  const float Smq = dSC + Cmq;
  const float inv2Smq = __fdividef(0.5f, Smq);
  EllSample e;
  e.S = Ssm;
  e.t = dSC * (Ssm + C) * inv2Smq;        // E21: (S^2 - C^2) / (2 (S - q))
  e.pSt = (Smq * Smq + perp2) * inv2Smq;  // S - t
  e.pt = pS * Smq * __fdividef(1.0f, e.pSt);  // E22 with the Jacobian of R2
  return e;
}

// Admissible S range of a connection along wc (case I, R14): S(t) = t +
// |x + wc t - xe| is non-decreasing, so the range is
// [max(Rm - E, S(clo)), min(RM - E, S(chi))).  Returned relative to C (S - C),
// formed without cancellation: S(t) - C = t + t (t - 2q) / (|x + wc t - xe| + C),
// (Rm - E) - C in double.  width = S_hi - S_lo, exact to rounding when both
// bounds are bin bounds.
struct SRange {
  float dlo, dhi, width;
};
__device__ __forceinline__ SRange conn_range(const DevScene& S, f3 x, f3 wc, f3 xe, float C, float q, float clo,
                                             float chi, double resM) {
  const f3 plo = fma3(wc, clo, x) - xe;
  const float lo_m_C = clo + clo * (clo - 2.0f * q) * __fdividef(1.0f, sqrtf(dot(plo, plo)) + C);
  float hi_m_C = __int_as_float(0x7f800000);
  if (isfinite(chi)) {
    const f3 phi_ = fma3(wc, chi, x) - xe;
    hi_m_C = chi + chi * (chi - 2.0f * q) * __fdividef(1.0f, sqrtf(dot(phi_, phi_)) + C);
  }
  const double dM_d = resM - f2d(C);
  const double dm_d = dM_d - S.dt;
  SRange r;
  r.dlo = d2f(dm_d);
  bool lo_bin = true;
  if (lo_m_C > r.dlo) { r.dlo = lo_m_C; lo_bin = false; }
  if (S.s_excess > 0.0f && S.s_excess > r.dlo) { r.dlo = S.s_excess; lo_bin = false; }
  const float dM_f = d2f(dM_d);
  const bool hi_bin = dM_f <= hi_m_C;
  r.dhi = hi_bin ? dM_f : hi_m_C;
  r.width = lo_bin && hi_bin ? S.dt_f : d2f((hi_bin ? dM_d : f2d(hi_m_C)) - (lo_bin ? dm_d : f2d(r.dlo)));
  return r;
}

// Contribution of the control vertex x_ell = x + wc t connected to the emitter
// (E2 throughput: sigma_s, transmittance of both legs, HG at x_ell, inverse
// square, pulse intensity), divided by p_t.  coef = beta (x the MIS/SPLIT
// connection weight, x 1/n_cell for a deferred splat).  pSt > 0: r2 = S - t.
template <int SH, bool WALLS, bool MESH = false>
__device__ __forceinline__ float conn_contrib(const DevScene& S, f3 x, f3 wc, f3 xe, float ek, float t, float pt,
                                              float pSt, float clo, float coef, f3* xell_out, float* r2_out) {
  const f3 xell = fma3(wc, t, x);
  const f3 de = xe - xell;
  float r2, r2sq;
  if (pSt > 0.0f) {  // on the ellipse r2 = S - t, formed without cancellation
    r2 = pSt;
    r2sq = pSt * pSt;
  } else {
    r2sq = dot(de, de);
    r2 = sqrtf(r2sq);
  }
  const f3 we = de * __fdividef(1.0f, r2);
  const float rho = hg_eval(S, dot(wc, we));
  // transmittance of both legs in one exponential
  const float len2 = segment_len<SH, WALLS, MESH>(S, xell, r2, we);
  const float tr = len2 < 0.0f ? 0.0f : fexp(-S.sigma_t * ((t - clo) + len2));
  float c = coef * S.sigma_s * tr * rho * ek * __fdividef(1.0f, r2sq * pt);
  if (S.r_excl > 0.0f && r2 < S.r_excl) c = 0.0f;
  if (xell_out) *xell_out = xell;
  if (r2_out) *r2_out = r2;
  return c;
}

// Runs a queued connection from an inside vertex (clo = 0) whose S range
// [C + dlo, C + dlo + width) is known and non-empty: S sample (E21-E22) and
// contribution (coef included).  m7e = u7's 23 bits | emitter << 23.
template <int SH, int FL>
__device__ __forceinline__ float conn_job_run(const DevScene& S, f3 x, f3 wc, float dlo, float width, float coef,
                                              uint32_t m7e) {
  constexpr bool WALLS = (FL & FL_WALLS) != 0, MESH = (FL & FL_MESH) != 0;
  const int e = (FL & FL_MULTI_E) ? (int)(m7e >> 23) : 0;
  const f3 xe = ld3(S.em_pos[e]);
  const f3 cv = xe - x;
  const float C = sqrtf(dot(cv, cv));
  const float q = dot(wc, cv);
  const EllSample es = ell_sample(S, cv, C, q, wc, dlo, width, mant01(m7e & 0x7FFFFFu));
  return conn_contrib<SH, WALLS, MESH>(S, x, wc, xe, S.em_k[e], es.t, es.pt, es.pSt, 0.0f, coef, nullptr, nullptr);
}

// Deferred connections (render kernel only): a medium or wall vertex whose
// connection S range is non-empty writes a job into its warp's shared-memory
// queue; the warp later runs up to 32 queued jobs at once, one per lane
// (conn_job_run), so the ~5-10 % of vertices that connect no longer run the
// S sample and contribution at a few active lanes.
constexpr int kJobWords = 11;  // x[3] w[3] dlo width coef m7e cell
#ifndef DTS_QUEUE
#define DTS_QUEUE 32
#endif
constexpr int kQueue = DTS_QUEUE;  // slots per warp
constexpr int kJob1Words = 14;  // stage-1 job: x[3] w_prev[3] resM(hi, lo) coef r4 r5 r6 m7e cell
// Stage-1 deferral (SPLIT: the whole connection stage queued) is a build
// option (-DDTS_STAGE1=1): it executes 8 % fewer instructions on config 5 but
// the alternation of two large code regions thrashes the instruction cache
// (ncu no_instruction stalls 0.25 -> 2.1 per issue) and it runs 12 % slower.
#ifndef DTS_STAGE1
#define DTS_STAGE1 0
#endif
constexpr bool kStage1Build = DTS_STAGE1 != 0;
struct Defer {
  float* q;           // this warp's queue: word f of slot j at q[f * qstride + j]
  float* q1;          // this warp's stage-1 queue (SPLIT: whole connection stages), same stride
  float* g;           // global overflow slots kQueue..2 kQueue-1 of q: word f of slot j at g[f * kQueue + j - kQueue]
  float* g1;          // the same for q1
  uint32_t qstride;   // words between fields (= kQueue * warps per CTA)
  uint32_t qn;        // jobs queued (warp-uniform)
  uint32_t qn1;       // stage-1 jobs queued (warp-uniform)
  unsigned act;       // lanes executing darts_vertex
  uint32_t lane_lt;   // lanes below this one
  uint32_t cell;      // the path's histogram cell
  float inv_n;        // 1 / paths of the cell
};

// Address of queue slot `slot` (< 2 kQueue): the first kQueue slots are in
// shared memory (stride qstride between fields), the next kQueue in the warp's
// global overflow area (stride kQueue), so a push never has to fall back to an
// inline connection.  *st receives the field stride.
__device__ __forceinline__ float* queue_slot(float* qs, uint32_t qstride, float* qg, uint32_t slot, uint32_t* st) {
  DTS_CHECK(slot < 2u * (uint32_t)kQueue);
  if (slot < (uint32_t)kQueue) {
    *st = qstride;
    return qs + slot;
  }
  *st = (uint32_t)kQueue;
  return qg + (slot - (uint32_t)kQueue);
}

// A medium event whose RIS distance is drawn later by the warp-collective
// sampler (RIS layout B); the vertex state is kept in PathState
// (x, w = the walk direction, resM, beta).
struct RisReq {
  bool need;
  float lo, T_m, counts;
};

// Applies a selected RIS candidate (E15): beta *= a mean(w) / w*, moves to
// x + w d and spends the counted time.
__device__ __forceinline__ void ris_apply(const DevScene& S, PathState& ps, float dsel, float W, float wsel,
                                          float counts) {
  const float beta_ris = S.albedo * (W * 0.125f) * __fdividef(1.0f, wsel);
  ps.beta *= beta_ris;
  ps.x = fma3(ps.w, dsel, ps.x);
  ps.resM -= f2d(counts * dsel);
  ps.kind = KIND_MEDIUM;
}

// End-of-vertex termination tests: early exit (no later
// connection can land before R_M) and non-finite throughput.
__device__ __forceinline__ bool vertex_tail(const PathState& ps, f3 xe, int& end_reason) {
  const f3 dn = ps.x - xe;
  const float Cn = sqrtf(dot(dn, dn));
  if (d2f(ps.resM) - Cn <= 0.0f) {
    end_reason = DTS_CTR_EARLY_EXIT;
    return false;
  }
  if (!isfinite(ps.beta)) {
    end_reason = DTS_CTR_NONFINITE;
    return false;
  }
  return true;
}

// Could a connection from x (inside the medium) reach the bin's lower residual
// resm = R_m - E at all?  S(t) = t + |x + w t - xe| over any chord from x is at
// most (farthest medium point from x) + (farthest medium point from any
// emitter, S.far_e): a larger resm means an empty S range for every direction.
template <int SH>
__device__ __forceinline__ bool may_connect_bound(const DevScene& S, f3 x, float resm) {
  if (SH == DTS_MEDIUM_BOX) {
    const float fx = fmaxf(x.x - S.bmin[0], S.bmax[0] - x.x);
    const float fy = fmaxf(x.y - S.bmin[1], S.bmax[1] - x.y);
    const float fz = fmaxf(x.z - S.bmin[2], S.bmax[2] - x.z);
    return resm <= sqrtf(fmaf(fx, fx, fmaf(fy, fy, fz * fz))) + S.far_e;
  }
  if (SH == DTS_MEDIUM_SPHERE) {
    const f3 d = x - ld3(S.center);
    return resm <= sqrtf(dot(d, d)) + sqrtf(S.radius2) + S.far_e;
  }
  return true;
}

// ----------------------------------------------------------------- direction mixture (E16-E19)
// One-sample MIS of the EDA table and HG at a medium vertex x with incoming
// direction w: gamma of E19 with the table cell of R10 at S = R_M - E (R11),
// technique by u4, cos(theta) by u5 (EDA: inverse transform of the cell's
// 16-bit CDF; HG about w), phi = pi (2 u6 - 1) (R12).  GUIDE: the CDF rows are
// followed by 8-bit guide rows (REUSE kernels stage both); without it the bin
// is found by an 8-step branchless binary search -- the same bin.
#ifndef DTS_EDA_PRED
#define DTS_EDA_PRED 0
#endif
struct MixDir {
  f3 om;
  float gamma, p_eda, p_hg, p_mix;
  bool eda;
};
template <bool SMEM, bool GUIDE>
__device__ __forceinline__ MixDir mix_direction(const DevScene& S, const uint16_t* __restrict__ tab, f3 x, f3 w,
                                                float resM, f3 xe, uint32_t r4, uint32_t r5, uint32_t r6) {
  const f3 cv = xe - x;
  const float C = sqrtf(dot(cv, cv));
  const float ratio = __fdividef(C, resM);
  const float ls = (__logf(resM) - S.ln_smin) * S.inv_dls;
  // DA_ONLY ablation: phase-function directions only (gamma = 0)
  const bool valid = (resM > 0.0f) && (ratio < 1.0f) && (ls >= 0.0f) && (ls < S.ns_f) &&
                     S.strategy != DTS_STRATEGY_DA_ONLY;
  MixDir m;
  m.gamma = valid ? __fdividef(ratio, ratio + S.alpha) : 0.0f;
  // (ir, is only address the table when valid: ratio in [0, 1), ls in [0, ns))
  const int ir = min((int)f2u23(ratio * S.nr_f), S.nr - 1);
  const int is = min((int)f2u23(ls), S.ns - 1);
  const uint16_t* qc = tab + (valid ? (size_t)(ir * S.ns + is) * DTS_TABLE_COS_BINS : 0);
  DTS_CHECK((size_t)(qc - tab) + DTS_TABLE_COS_BINS <= S.table_n);
  const f3 axis = cv * __fdividef(1.0f, C);
  const float u4 = unif(r4), u5 = unif(r5);
  const float phi = kPi * (2.0f * unif(r6) - 1.0f);
  m.eda = u4 < m.gamma;
  // Both techniques are evaluated by every lane and one is selected, so the
  // warp never splits into an EDA and an HG branch.
  // EDA: T = u5 * 65536 exactly; the bin is the largest j with q_j <= T, i.e.
  // q_j <= Ti = floor(T).
  const uint32_t Ti = r5 >> 16;
  int j;
  if (GUIDE) {  // guide entry of Ti's 1/256 slice, then bisect within the slice
    const uint8_t* gc = reinterpret_cast<const uint8_t*>(tab + S.table_n) + (qc - tab);
    const uint32_t gi = Ti >> 8;
    j = (int)gload<SMEM>(gc, gi);
    int jh = gi == 255u ? 255 : (int)gload<SMEM>(gc, gi + 1);
    DTS_CHECK(gi < 256u && j >= 0 && j < 256 && jh >= 0 && jh < 256);
#if DTS_EDA_PRED
    jh = m.eda ? jh : j;  // an HG lane's bin is unused (its p_eda bin is looked up below): it skips the bisection
#endif
    while (j < jh) {
      const int mid = (j + jh + 1) >> 1;
      DTS_CHECK(mid > 0 && mid < 256);
      if (qload<SMEM>(qc, mid) <= Ti) j = mid; else jh = mid - 1;
    }
  } else {  // q_0 = 0 <= Ti: binary search with steps 128 .. 1
    j = 0;
#pragma unroll
    for (int st = 128; st > 0; st >>= 1)
      if (qload<SMEM>(qc, j + st) <= Ti) j += st;
  }
  // T - q_j and q_{j+1} - T in units of 2^-7 are exact 23-bit integers
  const uint32_t T7 = r5 >> 9;  // 128 T
  uint32_t qa = qload<SMEM>(qc, j);
  uint32_t qb = j == 255 ? 65536u : qload<SMEM>(qc, j + 1);
  const float iq = __fdividef(1.0f / 128.0f, u23f(qb - qa));
  // HG about w_{k-1}
  float opc, omc;
  hg_sample(S, u5, opc, omc);
  {  // EDA: cos = -1 + (j + frac)/128: 1 + cos and 1 - cos from the integer parts (selected, not branched)
    const float fj = u23f((uint32_t)j);
    const float eo = (fj + u23f(T7 - (qa << 7)) * iq) * (1.0f / 128.0f);
    const float em = ((255.0f - fj) + u23f((qb << 7) - T7) * iq) * (1.0f / 128.0f);
    opc = m.eda ? eo : opc;
    omc = m.eda ? em : omc;
  }
  m.om = from_frame(m.eda ? axis : w, opc, omc, phi);
  if (!m.eda) {  // EDA pdf of the HG direction: bin of its cos to the emitter axis
    const int jb = (int)f2u23(fminf(fmaxf((dot(m.om, axis) + 1.0f) * 128.0f, 0.0f), 255.0f));
    DTS_CHECK(jb >= 0 && jb < 256);
    qa = qload<SMEM>(qc, jb);
    qb = jb == 255 ? 65536u : qload<SMEM>(qc, jb + 1);
  }
  m.p_eda = valid ? u23f(qb - qa) * (128.0f / 65536.0f / (2.0f * kPi)) : 0.0f;
  m.p_hg = hg_eval(S, dot(m.om, w));
  m.p_mix = m.gamma * m.p_eda + (1.0f - m.gamma) * m.p_hg;
  return m;
}

// ----------------------------------------------------------------- one DARTS vertex
// Returns true if the walk continues.  contrib receives the vertex's
// connection (+ wall NEE) contribution; end_reason the DTS_CTR_* of a stop.
// WALK (the walk stage of the two-stage render, SPLIT scenes): a vertex whose
// connection provably cannot land in its bin (conn_margin > 0) runs only the
// walk: the mixture direction, the connection's intersection and S range, and
// the wall NEE are skipped -- they would contribute exactly 0 -- and the walk's
// random numbers, directions and distances are the full vertex's, bit for bit.
// *walk_margin carries the margin in and its lower bound after the step out
// (margin - (1 + counts) d: see walk_kernel); while it stays positive the early
// exit test is skipped (R_M - E - C >= R_m - E - S_max > 0).
// NOCAM: the caller never passes a camera vertex (the connect stage of a REUSE
// scene's start-stage render: the start stage ran every camera vertex), so the
// camera branches (and R17) are compiled out.
template <bool DBG, bool SMEM, int SH, int FL, bool DEFER = false, bool WALK = false, bool NOCAM = false>
__device__ __forceinline__ bool darts_vertex(const DevScene& S, const uint16_t* __restrict__ tab, PathState& ps,
                                             const uint32_t (&r)[8], float& contrib, dts_debug_out* dbg,
                                             bool& conn_nonempty, bool& wall_nee, int& end_reason,
                                             const Defer* df = nullptr, bool* pushed = nullptr,
                                             RisReq* rq = nullptr, uint32_t* nsamp = nullptr,
                                             bool* pushed1 = nullptr, float* walk_margin = nullptr) {
  static_assert(!WALK || ((FL & FL_SPLIT) && !(FL & FL_MESH) && !DEFER && !DBG),
                "the walk stage serves SPLIT scenes without meshes");
  contrib = 0.0f;
  conn_nonempty = false;
  wall_nee = false;
  end_reason = 0;
  constexpr bool WALLS = (FL & FL_WALLS) != 0, SPLIT = (FL & FL_SPLIT) != 0, MESH = (FL & FL_MESH) != 0;
  static_assert(!(MESH && DEFER), "mesh scenes run the immediate render kernels only");
  const int e = (FL & FL_MULTI_E) ? ps.e : 0;  // one emitter: constant-bank operands
  const f3 xe = ld3(S.em_pos[e]);
  const float ek = S.em_k[e];
  f3 wc, ww;
  float wconn = 1.0f;
  const float resM = d2f(ps.resM);
  const bool cam = !NOCAM && ps.kind == KIND_CAMERA;  // (ps.kind changes only in step 1 below)

  // ---- SPLIT render kernel: queue this vertex's whole connection stage (stage 1) ----
  // A medium vertex whose connection can reach its bin at all (may_connect_bound)
  // writes x, w_{k-1}, R_M - E, beta / n_cell, u4..u7 and its cell into the
  // warp's stage-1 queue; the warp later runs up to 32 of them at once (mixture
  // direction, intersection, S range) and forwards the non-empty ones to the
  // sampling queue.  A lane that finds the queue full connects inline.
  bool skip_conn = WALK;
  if (SPLIT && DEFER && kStage1Build && !DBG) {
    const bool cand = ps.kind == KIND_MEDIUM && may_connect_bound<SH>(S, ps.x, d2f(ps.resM - S.dt));
    const unsigned m1 = __ballot_sync(df->act, cand);
    const uint32_t slot1 = df->qn1 + __popc(m1 & df->lane_lt);
    *pushed1 = cand;
    skip_conn = ps.kind == KIND_MEDIUM;  // queued, or unable to land in the bin
    if (cand) {
      uint32_t st;
      float* qq = queue_slot(df->q1, df->qstride, df->g1, slot1, &st);
      qq[0 * st] = ps.x.x; qq[1 * st] = ps.x.y; qq[2 * st] = ps.x.z;
      qq[3 * st] = ps.w.x; qq[4 * st] = ps.w.y; qq[5 * st] = ps.w.z;
      qq[6 * st] = __int_as_float(__double2hiint(ps.resM));
      qq[7 * st] = __int_as_float(__double2loint(ps.resM));
      qq[8 * st] = ps.beta * df->inv_n;
      qq[9 * st] = __uint_as_float(r[4]);
      qq[10 * st] = __uint_as_float(r[5]);
      qq[11 * st] = __uint_as_float(r[6]);
      qq[12 * st] = __uint_as_float((r[7] >> 9) | ((uint32_t)ps.e << 23));
      qq[13 * st] = __uint_as_float(df->cell);
    }
  }

  // ---- step 2: direction ----
  if (cam) {
    wc = ww = ps.w;
    if (DBG) {
      dbg->tech = 2;
      dbg->beta_dir = 1.0f;
    }
  } else if (WALLS && ps.kind == KIND_WALL) {
    const f3 n = inward_normal(ps.face);
    const float alb = S.wall_albedo[ps.face];
    const f3 cv = xe - ps.x;
    const float C = sqrtf(dot(cv, cv));
    const f3 we = cv * __fdividef(1.0f, C);
    const float cw = dot(n, we);
    const float resm = d2f(ps.resM - S.dt);
    float nee = 0.0f;
    if (!WALK && cw > 0.0f && resm - C <= 0.0f && resM - C > 0.0f) {  // E + C in [Rm, RM)
      // R14: time-checked direct NEE at a wall vertex
      nee = ps.beta * (alb * (1.0f / kPi)) * cw * ek * segment_tr<SH, WALLS, MESH>(S, ps.x, xe, C, we) *
            __fdividef(1.0f, C * C);
      if (S.r_excl > 0.0f && C < S.r_excl) nee = 0.0f;
      contrib += nee;
      wall_nee = nee > 0.0f;
      if (nsamp && nee != 0.0f) ++*nsamp;
    }
    if (DBG) dbg->nee = nee;
    // Lambertian: cosine hemisphere about n (1 - cos^2 = u5), beta *= albedo
    const float u5 = unif(r[5]);
    const float lz = sqrtf(1.0f - u5);  // cos theta; sin^2 theta = u5 = (1 + lz)(1 - lz)
    wc = ww = from_frame(n, 1.0f + lz, __fdividef(u5, 1.0f + lz), 2.0f * kPi * unif(r[6]));
    ps.beta *= alb;
    if (DBG) {
      dbg->tech = 3;
      dbg->beta_dir = alb;
    }
  } else if (MESH && ps.kind == KIND_SURF) {
    // R32: surface vertex on triangle ps.face: time-checked NEE as at walls
    // (R14) with the BSDF, then a BSDF-sampled direction for the connection and the walk
    int mat;
    const f3 n = tri_side_normal(S, ps.face, ps.w, mat);
    const f3 cv = xe - ps.x;
    const float C = sqrtf(dot(cv, cv));
    const f3 we = cv * __fdividef(1.0f, C);
    const float cw = dot(n, we);
    const float resm = d2f(ps.resM - S.dt);
    if (cw > 0.0f && resm - C <= 0.0f && resM - C > 0.0f) {  // E + C in [Rm, RM)
      float nee = ps.beta * bsdf_eval(S, mat, n, ps.w, we) * cw * ek *
                  segment_tr<SH, WALLS, MESH>(S, ps.x, xe, C, we) * __fdividef(1.0f, C * C);
      if (S.r_excl > 0.0f && C < S.r_excl) nee = 0.0f;
      contrib += nee;
      wall_nee = nee > 0.0f;
      if (nsamp && nee != 0.0f) ++*nsamp;
      if (DBG) dbg->nee = nee;
    }
    // lobe u4, direction u5, u6
    f3 wo;
    const float wgt = bsdf_sample(S, mat, n, ps.w, unif(r[4]), unif(r[5]), unif(r[6]), wo);
    if (DBG) {
      dbg->tech = 4;
      dbg->beta_dir = wgt;
    }
    if (!(wgt > 0.0f)) {  // below the surface: the path ends
      if (DBG) { dbg->event = 3; dbg->terminate = 1; dbg->beta_out = ps.beta; }
      end_reason = DTS_CTR_ESCAPES;
      return false;
    }
    ps.beta *= wgt;
    wc = ww = wo;
  } else {
    // medium vertex: one-sample MIS of EDA and HG
    if (SPLIT && skip_conn) {
      // R29 SPLIT, connection queued (or unreachable): only the walk's
      // independent HG direction is drawn here
      float o2, m2;
      hg_sample(S, u8_split(r), o2, m2);
      wc = ww = from_frame(ps.w, o2, m2, kPi * (2.0f * u9_split(r) - 1.0f));
    } else {
    const MixDir md = mix_direction<SMEM, !(SPLIT && kStage1Build)>(S, tab, ps.x, ps.w, resM, xe, r[4], r[5], r[6]);
    const f3 om = md.om;
    const bool eda = md.eda;
    const float gamma = md.gamma, p_eda = md.p_eda, p_hg = md.p_hg, p_mix = md.p_mix;
    const float ratio_w = __fdividef(p_hg, p_mix);
    wc = om;
    if (SPLIT) {
      // R29 SPLIT: MIS weight on the connection only; independent HG walk direction
      wconn = ratio_w;
      float o2, m2;
      hg_sample(S, u8_split(r), o2, m2);
      ww = from_frame(ps.w, o2, m2, kPi * (2.0f * u9_split(r) - 1.0f));
      if (DBG) dbg->beta_dir = 1.0f;
    } else {
      ww = om;
      ps.beta *= ratio_w;
      if (DBG) dbg->beta_dir = ratio_w;
    }
    if (DBG) {
      dbg->tech = eda ? 1 : 0;
      dbg->gamma = gamma;
      dbg->p_eda = p_eda;
      dbg->p_hg = p_hg;
      dbg->p_mix = p_mix;
    }
    }
  }
  if (DBG) {
    dbg->wc[0] = wc.x; dbg->wc[1] = wc.y; dbg->wc[2] = wc.z;
    dbg->ww[0] = ww.x; dbg->ww[1] = ww.y; dbg->ww[2] = ww.z;
    dbg->wconn = wconn;
  }

  // ---- intersection, reused by the connection and the walk ----
  float lo = 0.0f, hi = 0.0f;
  int face = -1;
  // one call site for every vertex kind: intersect() gives an inside origin
  // lo = 0 and the same exit as intersect_inside(), and a warp that mixes
  // camera and inside vertices then runs one intersection, not both (A/B:
  // config 4 +7 %, config 2 +1.6 %, config 5 even; profiles/ab_r02_isect1.log)
  int hit = intersect<SH, WALLS>(S, ps.x, ww, lo, hi, face);
  if (MESH && hit != HIT_MISS) {  // the interval ends at the nearest triangle (PAPER.md:301 case II)
    float tm;
    const int tri = mesh_trace<false>(S, ps.x, ww, hi, tm);
    if (tri >= 0) { hi = tm; hit = HIT_SURF; face = tri; }
  }
  // render kernel: non-empty connections of medium/wall vertices are queued (df)
  const bool defer = DEFER && !DBG && !cam;

  bool want_job = false;
  float job_dlo = 0.0f, job_width = 0.0f;
  float clo = lo, chi = hi;
  int hitc = WALK ? HIT_MISS : hit;
  if (SPLIT && ps.kind == KIND_MEDIUM) {
    if (skip_conn) {
      hitc = HIT_MISS;  // the connection stage runs from the stage-1 queue (or cannot land)
    } else {
      int fc;
      hitc = intersect_inside<SH, WALLS>(S, ps.x, wc, clo, chi, fc);
      if (MESH && hitc != HIT_MISS) {
        float tm;
        if (mesh_trace<false>(S, ps.x, wc, chi, tm) >= 0) { chi = tm; hitc = HIT_SURF; }
      }
    }
  }
  if (DBG) {
    dbg->t_lo = lo; dbg->t_hi = hi; dbg->hit = hit; dbg->face_hit = face;
    dbg->tc_lo = clo; dbg->tc_hi = chi;
  }

  // ---- step 3: elliptical connection (E20-E22; R13 every vertex, R17 unwarped camera) ----
  if (hitc != HIT_MISS) {
    const f3 cv = xe - ps.x;
    const float C2 = dot(cv, cv);
    const float C = sqrtf(C2);
    const float q = dot(wc, cv);
    const float u7 = unif(r[7]);
    float t = 0.0f, pt = 0.0f, Ssamp = 0.0f;
    float pSt = 0.0f;  // S - t (= r2 on the ellipse)
    bool ok = false;
    if (!(S.warped == 0 && cam)) {
      const SRange rg = conn_range(S, ps.x, wc, xe, C, q, clo, chi, ps.resM);
      if (DBG) { dbg->S_lo = C + rg.dlo; dbg->S_hi = C + rg.dhi; }
      if (rg.width > 0.0f && defer) {
        conn_nonempty = true;
        want_job = true;
        job_dlo = rg.dlo;
        job_width = rg.width;
      } else if (rg.width > 0.0f) {
        ok = true;
        const EllSample es = ell_sample(S, cv, C, q, wc, rg.dlo, rg.width, u7);
        Ssamp = es.S;
        t = es.t;
        pSt = es.pSt;
        pt = es.pt;
      }
    } else {
      // R17: unwarped camera vertex, shell |x(t) - xe| in [Rm, RM): <= 2 t-intervals
      const float resm = d2f(ps.resM - S.dt);
      float a_lo = clo;
      if (S.s_excess > 0.0f) {
        const float Se = C + S.s_excess;
        a_lo = fmaxf(a_lo, __fdividef((Se - C) * (Se + C), 2.0f * (Se - q)));
      }
      float ia0 = 0.f, ib0 = 0.f, ia1 = 0.f, ib1 = 0.f;
      int ni = 0;
      const float perp2 = C2 - q * q;
      const float radM = resM * resM - perp2;
      if (resM > 0.0f && radM > 0.0f) {
        const float hM = sqrtf(radM);
        const float radm = resm * resm - perp2;
        if (resm > 0.0f && radm > 0.0f) {
          const float hm = sqrtf(radm);
          ia0 = q - hM; ib0 = q - hm; ia1 = q + hm; ib1 = q + hM;
          ni = 2;
        } else {
          ia0 = q - hM; ib0 = q + hM;
          ni = 1;
        }
      }
      float m0 = 0.f, m1 = 0.f;
      if (ni >= 1) {
        ia0 = fmaxf(ia0, a_lo); ib0 = fminf(ib0, chi);
        if (ib0 > ia0) m0 = fexp(-S.sigma_t * (ia0 - clo)) * one_m_exp(S.sigma_t * (ib0 - ia0));
      }
      if (ni == 2) {
        ia1 = fmaxf(ia1, a_lo); ib1 = fminf(ib1, chi);
        if (ib1 > ia1) m1 = fexp(-S.sigma_t * (ia1 - clo)) * one_m_exp(S.sigma_t * (ib1 - ia1));
      }
      const float Z = m0 + m1;
      if (DBG) { dbg->S_lo = 0.0f; dbg->S_hi = Z; }
      if (Z > 0.0f) {
        ok = true;
        const float v = u7 * Z;
        const bool second = (m0 <= 0.0f) || (ni == 2 && !(v < m0));
        const float ia = second ? ia1 : ia0, ib = second ? ib1 : ib0;
        float up = second ? __fdividef(v - m0, m1) : __fdividef(v, m0);
        up = fminf(up, 0.99999994f);
        const float span = one_m_exp(S.sigma_t * (ib - ia));
        t = ia + neg_log1m2(up * span, fmaf(up, fexp(-S.sigma_t * (ib - ia)), 1.0f - up)) * S.inv_sigma_t;
        pt = __fdividef(S.sigma_t * fexp(-S.sigma_t * (t - clo)), Z);
      }
    }
    if (ok) {
      conn_nonempty = true;
      f3 xell;
      float r2;
      const float c = conn_contrib<SH, WALLS, MESH>(S, ps.x, wc, xe, ek, t, pt, pSt, clo, ps.beta * wconn, &xell, &r2);
      contrib += c;
      if (nsamp && c != 0.0f) ++*nsamp;
      if (DBG) {
        dbg->S = (S.warped == 0 && cam) ? t + r2 : Ssamp;
        dbg->t = t;
        dbg->x_ell[0] = xell.x; dbg->x_ell[1] = xell.y; dbg->x_ell[2] = xell.z;
        dbg->p_t = pt;
        dbg->contrib = c;
        dbg->conn_valid = 1;
      }
    }
  }
  if (DEFER && !DBG) {
    // queue the job (slots beyond the shared-memory queue are global overflow)
    const unsigned jm = __ballot_sync(df->act, want_job);
    const uint32_t slot = df->qn + __popc(jm & df->lane_lt);
    *pushed = want_job;
    if (want_job) {
      const float w8 = ps.beta * wconn * df->inv_n;
      const float w9 = __uint_as_float((r[7] >> 9) | ((uint32_t)ps.e << 23));
      const float w10 = __uint_as_float(df->cell);
      DTS_CHECK(slot < 2u * (uint32_t)kQueue);
      if (slot < (uint32_t)kQueue) {  // shared-memory slot (STS)
        float* qq = df->q + slot;
        const uint32_t st = df->qstride;
        qq[0 * st] = ps.x.x; qq[1 * st] = ps.x.y; qq[2 * st] = ps.x.z;
        qq[3 * st] = wc.x; qq[4 * st] = wc.y; qq[5 * st] = wc.z;
        qq[6 * st] = job_dlo; qq[7 * st] = job_width; qq[8 * st] = w8; qq[9 * st] = w9; qq[10 * st] = w10;
      } else {  // global overflow slot (STG)
        float* qq = df->g + (slot - (uint32_t)kQueue);
        constexpr uint32_t st = kQueue;
        qq[0 * st] = ps.x.x; qq[1 * st] = ps.x.y; qq[2 * st] = ps.x.z;
        qq[3 * st] = wc.x; qq[4 * st] = wc.y; qq[5 * st] = wc.z;
        qq[6 * st] = job_dlo; qq[7 * st] = job_width; qq[8 * st] = w8; qq[9 * st] = w9; qq[10 * st] = w10;
      }
    }
  }

  // ---- step 1 for the next vertex: DA distance sampling by RIS (E12-E15) ----
  if (hit == HIT_MISS) {
    if (DBG) { dbg->event = 0; dbg->terminate = 1; dbg->beta_out = ps.beta; }
    end_reason = DTS_CTR_ESCAPES;
    return false;
  }
  const float counts = (S.warped || !cam) ? 1.0f : 0.0f;
  const bool inf_hi = isinf(hi);
  const float y_m = S.sigma_t * (hi - lo);
  const float T_m = inf_hi ? 0.0f : fexp(-y_m);                        // 1 - p_m
  const float p_m = inf_hi ? 1.0f : one_m_exp_T(y_m, T_m);             // E12, R28
  const float u0 = unif(r[0]);
  if (DBG) dbg->p_m = p_m;
  if (rq) rq->need = false;
  if (u0 < p_m && S.strategy == DTS_STRATEGY_EDA_ONLY) {
    // EDA_ONLY ablation: one truncated-exponential distance (E13-E14, R1), eps = u2;
    // weight sigma_s e^{-st (d - lo)} / (p_cand p_m) = a
    const float u2 = unif(r[2]);
    const float d = fmaf(-__log2f(fmaf(u2, T_m, 1.0f - u2)), S.inv_sigma_t * kLn2, lo);
    ps.beta *= S.albedo;
    ps.x = fma3(ww, d, ps.x);
    ps.resM -= f2d(counts * d);
    if (WALK) *walk_margin -= (1.0f + counts) * d * 1.00001f;
    ps.kind = KIND_MEDIUM;
    ps.w = ww;
    if (DBG) { dbg->event = 1; dbg->istar = 0; dbg->d = d; dbg->beta_ris = S.albedo; }
  } else if (!DBG && rq && u0 < p_m) {
    // RIS layout B: the warp draws the distance after this call
    rq->need = true;
    rq->lo = lo;
    rq->T_m = T_m;
    rq->counts = counts;
    ps.w = ww;
    return true;
  } else if (u0 < p_m) {
    // candidates: Sobol row r = floor(32 u1) with Cranley-Patterson shift u2 (R6):
    // Q[r][i] = RI2(8r+i) = bitrev3(i)/8 + bitrev5(r)/256, shift and mod 1 done
    // exactly on 23-bit integers.
    const uint32_t br5 = __brev(r[1] >> 27) >> 27;
    const uint32_t m2 = r[2] >> 9;
    const f3 cv = xe - ps.x;
    const float qd = dot(ww, cv);
    const f3 perp = cv - ww * qd;
    const float perp2 = dot(perp, perp);
    // candidate i's 23-bit uniform: (m2 + bitrev3(i) 2^20 + bitrev5(row) 2^15) mod 2^23
    const uint32_t vbase = m2 + (br5 << 15);
    float e2[8], s3[8];
    float emax = -__int_as_float(0x7f800000);
    // pairs (2j, 2j + 1) of candidates in packed fp32; per candidate:
    //   E14 with the sign of R1: d = t_lo - ln(1 - p_m u) / sigma_t, with
    //   1 - p_m u = (1 - u) + u (1 - p_m), 1 - u = 2 - (1 + u) exact (MUFU lg2
    //   keeps the absolute error of d below ~1e-7 / sigma_t);
    //   Delta = R_M - E - d (R4); r^2 = |x + w d - x_e|^2 = (d - q)^2 + perp^2;
    //   s = Delta^{-1/2}; valid iff Delta > 0 and r <= Delta, tested as
    //   r^2 s^2 < Delta (for Delta <= 0, s = 1e10 makes it false);
    //   log2 of Phi' = Delta^{-3/2} exp(-r^2/(4 D Delta) - sigma_a Delta) (E9,
    //   constants dropped) = log2(s^3) + k1 r^2 s^2 + k2 Delta.
    const float2 Tm2 = f2s(T_m), lo2 = f2s(lo), negk = f2s(-S.inv_sigma_t * kLn2);
    const float2 negc = f2s(-counts), resM2 = f2s(resM), negqd = f2s(-qd), p2 = f2s(perp2);
    const float2 k1 = f2s(S.neg_inv4D_log2e), k2 = f2s(S.neg_sa_log2e);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t v0 = (vbase + ((__brev((uint32_t)(2 * j)) >> 29) << 20)) & 0x7FFFFFu;
      const uint32_t v1 = (vbase + ((__brev((uint32_t)(2 * j + 1)) >> 29) << 20)) & 0x7FFFFFu;
      const float2 M = f2(__uint_as_float(0x3f800000u | v0), __uint_as_float(0x3f800000u | v1));  // 1 + u
      const float2 u = add2(M, f2s(-1.0f));
      const float2 omu = fma2(M, f2s(-1.0f), f2s(2.0f));   // 1 - u, exact
      const float2 a = fma2(u, Tm2, omu);                   // 1 - p_m u
      const float2 d = fma2(f2(__log2f(a.x), __log2f(a.y)), negk, lo2);
      const float2 Delta = fma2(d, negc, resM2);
      const float2 dq = add2(d, negqd);
      const float2 r2 = fma2(dq, dq, p2);
      // (walk stage: every candidate is valid -- it lies on a chord from x, so
      // d + r <= S_max(x) < R_m - E by the positive connection margin (with its
      // 1e-3 safety), i.e. r < Delta with Delta >= 1e-3 -- so neither the clamp
      // nor the mask can change a value there and both are skipped)
      const float2 sv = WALK ? f2(rsqrtf(Delta.x), rsqrtf(Delta.y))
                             : f2(rsqrtf(fmaxf(Delta.x, 1e-20f)), rsqrtf(fmaxf(Delta.y, 1e-20f)));
      const float2 ss = mul2(sv, sv);
      const float2 q = mul2(r2, ss);                        // r^2 / Delta
      const float2 ex = fma2(q, k1, mul2(Delta, k2));
      const float2 cube = mul2(ss, sv);                     // s^3 (finite for invalid candidates)
      if (DBG) { dbg->cand_d[2 * j] = d.x; dbg->cand_d[2 * j + 1] = d.y; }
      e2[2 * j] = (WALK || q.x < Delta.x) ? ex.x : -__int_as_float(0x7f800000);
      e2[2 * j + 1] = (WALK || q.y < Delta.y) ? ex.y : -__int_as_float(0x7f800000);
      s3[2 * j] = cube.x;
      s3[2 * j + 1] = cube.y;
      emax = fmaxf(emax, fmaxf(e2[2 * j], e2[2 * j + 1]));
    }
    if (!WALK && emax == -__int_as_float(0x7f800000)) emax = 0.0f;  // all invalid: exp2(-inf) = 0, not NaN
    // R7: weights relative to the largest exponent, w_i = s_i^3 2^(e_i - emax)
    float2 W2 = f2s(0.0f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 x = add2(f2(e2[2 * j], e2[2 * j + 1]), f2s(-emax));
      const float2 w = mul2(f2(s3[2 * j], s3[2 * j + 1]), f2(exp2f(x.x), exp2f(x.y)));
      e2[2 * j] = w.x;
      e2[2 * j + 1] = w.y;
      W2 = add2(W2, w);
    }
    const float W = W2.x + W2.y;
    if (DBG) {
      for (int i = 0; i < 8; ++i) dbg->cand_wn[i] = W > 0.0f ? e2[i] / W : 0.0f;
    }
    if (!WALK && !(W > 0.0f)) {  // (walk stage: every candidate is valid, W > 0)
      if (DBG) { dbg->event = 4; dbg->terminate = 1; dbg->beta_out = ps.beta; }
      end_reason = DTS_CTR_RIS_INVALID;  // R5
      return false;
    }
    // resample: smallest i with sum_{j<=i} w_j > u3 W (CDF inversion in candidate order)
    const float thr = unif(r[3]) * W;
    // the partial sums are monotone: scanning them from the last to the first,
    // the last one found above thr is the first in candidate order
    float cum[7];
    cum[0] = e2[0];
#pragma unroll
    for (int i = 1; i < 7; ++i) cum[i] = cum[i - 1] + e2[i];
    float wsel = e2[7];
    uint32_t is = 7;
#pragma unroll
    for (int i = 6; i >= 0; --i) {
      const bool gt = cum[i] > thr;
      wsel = gt ? e2[i] : wsel;
      is = gt ? (uint32_t)i : is;
    }
    // regenerate the selected candidate's distance (cheaper than keeping all 8)
    const uint32_t brs = __brev(is) >> 29;
    const uint32_t vs = (m2 + ((brs * 32u + br5) << 15)) & 0x7FFFFFu;
    const float us = mant01(vs);
    const float dsel = fmaf(-__log2f(fmaf(us, T_m, 1.0f - us)), S.inv_sigma_t * kLn2, lo);
    const float beta_ris = S.albedo * (W * 0.125f) * __fdividef(1.0f, wsel);  // E15: a * mean(w) / w*
    ps.beta *= beta_ris;
    ps.x = fma3(ww, dsel, ps.x);
    ps.resM -= f2d(counts * dsel);
    ps.kind = KIND_MEDIUM;
    ps.w = ww;
    if (WALK) *walk_margin -= (1.0f + counts) * dsel * 1.00001f;
    if (DBG) { dbg->event = 1; dbg->istar = (int)is; dbg->d = dsel; dbg->beta_ris = beta_ris; }
  } else {
    if (WALLS && hit == HIT_WALL) {
      f3 xn = fma3(ww, hi, ps.x);
      const int a = face >> 1;
      const float pl = (face & 1) ? S.bmax[a] : S.bmin[a];
      xn.x = a == 0 ? pl : xn.x;  // snap onto the wall (selects, not branches)
      xn.y = a == 1 ? pl : xn.y;
      xn.z = a == 2 ? pl : xn.z;
      ps.x = xn;
      ps.resM -= f2d(counts * hi);
      ps.kind = KIND_WALL;
      if (WALK) *walk_margin -= (1.0f + counts) * hi * 1.00001f;
      ps.face = face;
      ps.w = ww;
      if (DBG) { dbg->event = 2; dbg->d = hi; dbg->beta_ris = 1.0f; }
    } else if (MESH && hit == HIT_SURF) {
      // R32/R33: the walk reaches the triangle; the vertex sits kSurfEps off it on the incident side
      int mat;
      const f3 n = tri_side_normal(S, face, ww, mat);
      ps.x = fma3(n, kSurfEps, fma3(ww, hi, ps.x));
      ps.resM -= f2d(counts * hi);
      ps.kind = KIND_SURF;
      ps.face = face;
      ps.w = ww;
      if (DBG) { dbg->event = 5; dbg->d = hi; dbg->beta_ris = 1.0f; }
    } else {
      if (DBG) { dbg->event = 3; dbg->terminate = 1; dbg->beta_out = ps.beta; }
      end_reason = DTS_CTR_ESCAPES;
      return false;
    }
  }
  if (DBG) {
    dbg->x_next[0] = ps.x.x; dbg->x_next[1] = ps.x.y; dbg->x_next[2] = ps.x.z;
    dbg->beta_out = ps.beta;
  }
  if (WALK && *walk_margin > 0.0f) {
    // walk stage: the connection margin still bounds R_M - E - C from below, so
    // the early exit provably does not fire; only the non-finite test remains
    if (!isfinite(ps.beta)) {
      end_reason = DTS_CTR_NONFINITE;
      return false;
    }
    return true;
  }
  const bool alive = vertex_tail(ps, xe, end_reason);
  if (DBG && !alive) dbg->terminate = 1;
  return alive;
}

// RIS layout B (SURVEY 8(a) "8-lane groups"): the warp draws the distances of
// every lane with a pending medium event (RisReq), four paths per round, one
// 8-lane group per path and one candidate per lane.  Per-path inputs are
// broadcast with shuffles; the group max-normalises the log weights (R7),
// scans them in candidate order (inclusive, 3 shuffles) and takes the first
// candidate whose partial sum exceeds u3 W -- CDF inversion in the candidate
// order of layout A / the oracle (E13-E15, R6).  All 32 lanes must call it.
// Returns, to each requesting lane, dsel, W and w*; W = 0 means all invalid (R5).
__device__ __forceinline__ void ris_warp(const DevScene& S, const PathState& ps, const RisReq& rq, f3 xe,
                                         uint32_t r1, uint32_t r2, uint32_t r3, int lane, float& dsel, float& W,
                                         float& wsel) {
  const unsigned FULL = 0xffffffffu;
  unsigned pend = __ballot_sync(FULL, rq.need);
  // per-path inputs, prepared by the owner lane
  float qd = 0.0f, perp2 = 0.0f;
  if (rq.need) {
    const f3 cv = xe - ps.x;
    qd = dot(ps.w, cv);
    const f3 perp = cv - ps.w * qd;
    perp2 = dot(perp, perp);
  }
  const float resM_o = d2f(ps.resM);
  const uint32_t m2_o = r2 >> 9, br5_o = __brev(r1 >> 27) >> 27;
  const float u3_o = unif(r3);
  const int g = lane >> 3, c = lane & 7;
  const uint32_t br3 = __brev((uint32_t)c) >> 29;
  dsel = 0.0f;
  W = 0.0f;
  wsel = 1.0f;
  while (pend) {
    // the (g+1)-th pending lane of this round is group g's path
    unsigned m = pend;
    for (int k = 0; k < g && m; ++k) m &= m - 1u;
    const int owner = m ? __ffs(m) - 1 : -1;
    const int src = owner >= 0 ? owner : lane;
    const float lo = __shfl_sync(FULL, rq.lo, src);
    const float T_m = __shfl_sync(FULL, rq.T_m, src);
    const float counts = __shfl_sync(FULL, rq.counts, src);
    const float resM = __shfl_sync(FULL, resM_o, src);
    const float q = __shfl_sync(FULL, qd, src);
    const float p2 = __shfl_sync(FULL, perp2, src);
    const uint32_t m2 = __shfl_sync(FULL, m2_o, src);
    const uint32_t br5 = __shfl_sync(FULL, br5_o, src);
    const float u3 = __shfl_sync(FULL, u3_o, src);
    // candidate c of the group's path (identical arithmetic to layout A)
    const uint32_t v = (m2 + ((br3 * 32u + br5) << 15)) & 0x7FFFFFu;
    const float ui = mant01(v);
    const float di = fmaf(-__log2f(fmaf(ui, T_m, 1.0f - ui)), S.inv_sigma_t * kLn2, lo);
    const float Delta = resM - counts * di;
    const float dq = di - q;
    const float r2i = fmaf(dq, dq, p2);
    const bool valid = owner >= 0 && r2i < Delta * fabsf(Delta);
    const float sr = rsqrtf(fmaxf(Delta, 1e-20f));
    const float ex = valid ? fmaf(S.neg_inv4D_log2e * r2i, sr * sr, S.neg_sa_log2e * Delta)
                           : -__int_as_float(0x7f800000);
    float emax = ex;
    emax = fmaxf(emax, __shfl_xor_sync(FULL, emax, 1));
    emax = fmaxf(emax, __shfl_xor_sync(FULL, emax, 2));
    emax = fmaxf(emax, __shfl_xor_sync(FULL, emax, 4));
    if (emax == -__int_as_float(0x7f800000)) emax = 0.0f;
    const float w = sr * sr * sr * exp2f(ex - emax);
    float cum = w;  // inclusive scan within the group
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const float t = __shfl_up_sync(FULL, cum, o, 8);
      if (c >= o) cum += t;
    }
    const float Wg = __shfl_sync(FULL, cum, 7, 8);
    const bool gt = cum > u3 * Wg;
    const unsigned gb = (__ballot_sync(FULL, gt) >> (8 * g)) & 0xFFu;
    const int is = gb ? __ffs(gb) - 1 : 7;
    const float ws = __shfl_sync(FULL, w, is, 8);
    const float ds = __shfl_sync(FULL, di, is, 8);
    // return to the owners: owner of group k reads lane 8k
    const unsigned here = pend;
    int k = -1;
    if (rq.need && ((here >> lane) & 1u)) {
      const int rank = __popc(here & ((1u << lane) - 1u));
      if (rank < 4) k = rank;
    }
    const int from = k >= 0 ? 8 * k : lane;
    const float Wr = __shfl_sync(FULL, Wg, from);
    const float wr = __shfl_sync(FULL, ws, from);
    const float dr = __shfl_sync(FULL, ds, from);
    if (k >= 0) {
      W = Wr;
      wsel = wr;
      dsel = dr;
    }
    // retire this round's (up to) four paths
    for (int j = 0; j < 4 && pend; ++j) pend &= pend - 1u;
  }
}

// Runs queued connection job (fields at q[f * st]).  Returns the contribution
// already scaled by 1 / n_cell, and its cell.
template <int SH, int FL>
__device__ __forceinline__ float conn_job_eval(const DevScene& S, const float* q, uint32_t st, uint32_t& cell) {
  const f3 x = mk(q[0 * st], q[1 * st], q[2 * st]);
  const f3 wc = mk(q[3 * st], q[4 * st], q[5 * st]);
  cell = __float_as_uint(q[10 * st]);
  return conn_job_run<SH, FL>(S, x, wc, q[6 * st], q[7 * st], q[8 * st], __float_as_uint(q[9 * st]));
}

}  // namespace dts
