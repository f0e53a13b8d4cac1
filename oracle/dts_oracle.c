/*
 * dts_oracle.c -- TEST INFRASTRUCTURE ONLY (see dts_oracle.h).
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the DARTS hot
 * path of "DARTS: Diffusion Approximated Residual Time Sampling for
 * Time-of-flight Rendering in Homogeneous Scattering Media" (arXiv 2402.03106).
 * Citations are PAPER.md line numbers (equations E1..E22 numbered in order of
 * appearance); the readings R1..R29 of ambiguous or
 * garbled passages are listed in DESIGN.md section 3 and are the same ones the
 * CUDA path implements.  Nothing here is blocked, fused or reordered beyond the
 * paper's own step order; the only libraries used are libm and pthreads.
 *
 * This file shares no code with paper_2402_03106_b200/csrc and must never be
 * linked into the product library.
 */
#include "dts_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_PI 3.14159265358979323846

/* ------------------------------------------------------------------------- */
/* Counter-based RNG: Philox4x32-10 (Salmon et al., SC'11).  R24: the paper
 * uses "a pre-computed table (32 by 8) of Sobol sequence" plus uniform random
 * offsets; the uniforms themselves come from this generator,
 * keyed by the seed and counted by (path id, bounce, block).                */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R24: uint32 -> [0,1) with the top 23 bits (an fp32 mantissa); never 1.0. */
double or_uniform(uint32_t r) { return (double)(r >> 9) * (1.0 / 8388608.0); }

static void draw4(uint64_t seed, uint64_t id, uint32_t bounce, uint32_t block, uint32_t out[4]) {
  uint32_t ctr[4] = {(uint32_t)id, (uint32_t)(id >> 32), bounce, block};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  or_philox4x32_10(ctr, key, out);
}

/* R6: Sobol dimension 0 (= van der Corput, base 2), points 0..255 row-major in
 * a 32 x 8 table. */
double or_sobol(int row, int col) {
  unsigned n = (unsigned)(8 * row + col);
  double v = 0.0, f = 0.5;
  while (n) {
    if (n & 1u) v += f;
    n >>= 1;
    f *= 0.5;
  }
  return v;
}

/* ------------------------------------------------------------------------- */
/* small vector helpers                                                       */
static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double norm3(const double a[3]) { return sqrt(dot3(a, a)); }
static void sub3(const double a[3], const double b[3], double o[3]) { o[0] = a[0] - b[0]; o[1] = a[1] - b[1]; o[2] = a[2] - b[2]; }
static void madd3(const double a[3], const double d[3], double t, double o[3]) {
  o[0] = a[0] + d[0] * t; o[1] = a[1] + d[1] * t; o[2] = a[2] + d[2] * t;
}
static void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
static void normalize3(double a[3]) { double n = norm3(a); a[0] /= n; a[1] /= n; a[2] /= n; }

/* R12: orthonormal frame about n (Duff et al. 2017); the chart is +z for
 * n_z >= -1e-6 (a tie-break: a horizontal normal whose n_z rounds to +-0 or
 * +-tiny picks one frame on both sides), else -z. */
static void onb(const double n[3], double b1[3], double b2[3]) {
  double sign = n[2] >= -1e-6 ? 1.0 : -1.0;
  double a = -1.0 / (sign + n[2]);
  double b = n[0] * n[1] * a;
  b1[0] = 1.0 + sign * n[0] * n[0] * a; b1[1] = sign * b; b1[2] = -sign * n[0];
  b2[0] = b; b2[1] = sign + n[1] * n[1] * a; b2[2] = -n[1];
}
static void from_frame(const double n[3], double cos_t, double phi, double out[3]) {
  double b1[3], b2[3];
  onb(n, b1, b2);
  double sin_t = sqrt(fmax(0.0, 1.0 - cos_t * cos_t));
  double cx = sin_t * cos(phi), cy = sin_t * sin(phi);
  for (int i = 0; i < 3; ++i) out[i] = b1[i] * cx + b2[i] * cy + n[i] * cos_t;
}

/* ------------------------------------------------------------------------- */
/* medium physics                                                             */
typedef struct {
  double sigma_t, albedo, D;
} derived;

static derived derive(const or_scene* sc) {
  derived d;
  d.sigma_t = sc->sigma_s + sc->sigma_a;
  d.albedo = sc->sigma_s / d.sigma_t;
  d.D = 1.0 / (3.0 * (sc->sigma_a + sc->sigma_s * (1.0 - sc->g))); /* E9 */
  return d;
}

/* E9 with c = 1: the transient DA fluence of a unit delta
 * pulse at distance sqrt(r2) after a delay dt; Heaviside: 0 for dt <= 0. */
double or_da_flux(const or_scene* sc, double r2, double dt) {
  if (!(dt > 0.0)) return 0.0;
  derived dv = derive(sc);
  double den = pow(4.0 * OR_PI * dv.D * dt, 1.5);
  return exp(-r2 / (4.0 * dv.D * dt) - sc->sigma_a * dt) / den;
}

/* Henyey-Greenstein phase function (standard form). */
double or_hg_eval(double g, double cos_theta) {
  double den = 1.0 + g * g - 2.0 * g * cos_theta;
  return (1.0 - g * g) / (4.0 * OR_PI * den * sqrt(den));
}

/* HG inverse CDF in cos(theta) measured from w_prev (R25). */
static double hg_sample_cos(double g, double u) {
  if (g == 0.0) return 1.0 - 2.0 * u;
  double sq = (1.0 - g * g) / (1.0 - g + 2.0 * g * u);
  return (1.0 + g * g - sq * sq) / (2.0 * g);
}

double or_hg_sample_cos(double g, double u) { return hg_sample_cos(g, u); }

/* E18: polar distance of the ellipse with foci distance C
 * and path-length sum S, in the direction at angle theta to the major axis. */
double or_polar_distance(double C, double S, double cos_theta) {
  return (S * S - C * C) / (2.0 * S - 2.0 * C * cos_theta);
}

/* ------------------------------------------------------------------------- */
/* analytic medium bounds (R15)                                  */
int or_intersect(const or_scene* sc, const double o[3], const double d[3], double* t_lo,
                 double* t_hi, int* face) {
  *face = -1;
  if (sc->medium_shape == OR_MEDIUM_INFINITE) {
    *t_lo = 0.0;
    *t_hi = INFINITY;
    return OR_HIT_NONE;
  }
  if (sc->medium_shape == OR_MEDIUM_SPHERE) {
    double oc[3];
    sub3(o, sc->center, oc);
    double b = dot3(oc, d);
    double c = dot3(oc, oc) - sc->radius * sc->radius;
    double disc = b * b - c;
    if (disc <= 0.0) return OR_HIT_MISS;
    double s = sqrt(disc);
    double tn = -b - s, tf = -b + s;
    if (tf <= 0.0) return OR_HIT_MISS;
    *t_lo = fmax(tn, 0.0);
    *t_hi = tf;
    return OR_HIT_OPEN;
  }
  /* box: slab test */
  double tn = -INFINITY, tf = INFINITY;
  int fface = -1;
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0) {
      if (o[a] < sc->bmin[a] || o[a] > sc->bmax[a]) return OR_HIT_MISS;
      continue;
    }
    double t1 = (sc->bmin[a] - o[a]) / d[a];
    double t2 = (sc->bmax[a] - o[a]) / d[a];
    double near = fmin(t1, t2), far = fmax(t1, t2);
    if (near > tn) tn = near;
    if (far < tf) {
      tf = far;
      fface = 2 * a + (d[a] > 0.0 ? 1 : 0);
    }
  }
  double lo = fmax(tn, 0.0);
  if (!(tf > lo)) return OR_HIT_MISS;
  *t_lo = lo;
  *t_hi = tf;
  *face = fface;
  return ((sc->wall_mask >> fface) & 1u) ? OR_HIT_WALL : OR_HIT_OPEN;
}

/* Medium length and visibility of the straight segment p -> xe (p inside the
 * medium).  R15: a segment leaving the medium through a wall is occluded. */
static void segment_medium(const or_scene* sc, const double p[3], const double xe[3], double* len,
                           double* vis) {
  double dvec[3];
  sub3(xe, p, dvec);
  double r = norm3(dvec);
  *vis = 1.0;
  if (sc->n_tris > 0) { /* R32: a triangle on the segment occludes it */
    double dir[3] = {dvec[0] / r, dvec[1] / r, dvec[2] / r}, tm;
    if (or_mesh_hit(sc, p, dir, r, &tm) >= 0) {
      *vis = 0.0;
      *len = r;
      return;
    }
  }
  if (sc->medium_shape == OR_MEDIUM_INFINITE) {
    *len = r;
    return;
  }
  double dir[3] = {dvec[0] / r, dvec[1] / r, dvec[2] / r};
  double lo, hi;
  int face;
  int hit = or_intersect(sc, p, dir, &lo, &hi, &face);
  if (hit == OR_HIT_MISS) {
    *len = 0.0;
    return;
  }
  *len = fmax(0.0, fmin(hi, r) - lo);
  if (hit == OR_HIT_WALL && hi < r) *vis = 0.0;
}

static void inward_normal(int face, double n[3]) {
  n[0] = n[1] = n[2] = 0.0;
  n[face / 2] = (face & 1) ? -1.0 : 1.0;
}

/* ------------------------------------------------------------------------- */
/* triangle meshes (R32, R33; opaque surfaces of PAPER.md:105, 221, 301)       */
/* Moller-Trumbore ray/triangle distance (edges inclusive), -1 for no hit */
static double tri_hit(const double* v, const double o[3], const double d[3]) {
  double e1[3], e2[3], s[3], p[3], qv[3];
  sub3(v + 3, v, e1);
  sub3(v + 6, v, e2);
  cross3(d, e2, p);
  double det = dot3(e1, p);
  if (det == 0.0) return -1.0;
  double inv = 1.0 / det;
  sub3(o, v, s);
  double u = dot3(s, p) * inv;
  if (u < 0.0 || u > 1.0) return -1.0;
  cross3(s, e1, qv);
  double vv = dot3(d, qv) * inv;
  if (vv < 0.0 || u + vv > 1.0) return -1.0;
  return dot3(e2, qv) * inv;
}

/* nearest hit over every triangle (no acceleration structure) */
int or_mesh_hit(const or_scene* sc, const double o[3], const double d[3], double t_max, double* t) {
  int best = -1;
  double tb = t_max;
  for (int i = 0; i < sc->n_tris; ++i) {
    double th = tri_hit(sc->tris + 9 * i, o, d);
    if (th > 0.0 && th < tb) {
      tb = th;
      best = i;
    }
  }
  if (best >= 0) *t = tb;
  return best;
}

/* geometric normal turned to the side the incident direction w comes from */
static void side_normal(const or_scene* sc, int tri, const double w[3], double n[3]) {
  const double* v = sc->tris + 9 * tri;
  double e1[3], e2[3];
  sub3(v + 3, v, e1);
  sub3(v + 6, v, e2);
  cross3(e1, e2, n);
  normalize3(n);
  if (dot3(n, w) > 0.0) { n[0] = -n[0]; n[1] = -n[1]; n[2] = -n[2]; }
}

/* R32: f = rho [(1 - ks) / pi + ks (n + 2) / (2 pi) max(0, wo . r)^n] on the
 * incident side, r = w - 2 (w . n_s) n_s the mirror direction (Lambertian for
 * ks = 0, normalised Phong lobe for ks = 1, "plastic" in between). */
double or_bsdf_eval(const or_scene* sc, int tri, const double w[3], const double wo[3]) {
  double n[3], r[3];
  side_normal(sc, tri, w, n);
  if (!(dot3(wo, n) > 0.0)) return 0.0;
  const double* m = sc->mats[sc->tri_mat[tri]];
  double wn = dot3(w, n);
  for (int i = 0; i < 3; ++i) r[i] = w[i] - 2.0 * wn * n[i];
  double ca = fmax(0.0, dot3(wo, r));
  return m[0] * ((1.0 - m[1]) / OR_PI + m[1] * (m[2] + 2.0) / (2.0 * OR_PI) * pow(ca, m[2]));
}

/* R32 sampling: u4 < ks picks the lobe (cos alpha = u5^{1/(n+1)} about r),
 * else the cosine hemisphere (cos theta = sqrt(1 - u5) about n_s); phi = 2 pi u6.
 * One-sample MIS over both: weight f cos / ((1 - ks) cos / pi + ks p_lobe). */
double or_bsdf_sample(const or_scene* sc, int tri, const double w[3], double u4, double u5, double u6,
                      double wo[3]) {
  double n[3], r[3];
  side_normal(sc, tri, w, n);
  const double* m = sc->mats[sc->tri_mat[tri]];
  double wn = dot3(w, n);
  for (int i = 0; i < 3; ++i) r[i] = w[i] - 2.0 * wn * n[i];
  if (u4 < m[1])
    from_frame(r, pow(u5, 1.0 / (m[2] + 1.0)), 2.0 * OR_PI * u6, wo);
  else
    from_frame(n, sqrt(fmax(0.0, 1.0 - u5)), 2.0 * OR_PI * u6, wo);
  double co = dot3(wo, n);
  if (!(co > 0.0)) return 0.0;
  double ca = fmax(0.0, dot3(wo, r));
  double p = (1.0 - m[1]) * co / OR_PI + m[1] * (m[2] + 1.0) / (2.0 * OR_PI) * pow(ca, m[2]);
  return or_bsdf_eval(sc, tri, w, wo) * co / p;
}

/* medium interval of a ray, cut at the nearest triangle (R32: case II of
 * PAPER.md:301, "the closest surface distance t_s") */
static int scene_intersect(const or_scene* sc, const double o[3], const double d[3], double* lo, double* hi,
                           int* face) {
  int hit = or_intersect(sc, o, d, lo, hi, face);
  if (hit == OR_HIT_MISS || sc->n_tris == 0) return hit;
  double tm;
  int tri = or_mesh_hit(sc, o, d, *hi, &tm);
  if (tri < 0) return hit;
  *hi = tm;
  *face = tri;
  return OR_HIT_SURF;
}

/* R33: surface vertex at x + d t, moved OR_SURF_EPS off the triangle on the side d arrives from */
static void surface_point(const or_scene* sc, int tri, const double x[3], const double d[3], double t,
                          double out[3]) {
  double n[3];
  side_normal(sc, tri, d, n);
  for (int i = 0; i < 3; ++i) out[i] = x[i] + d[i] * t + OR_SURF_EPS * n[i];
}

/* ------------------------------------------------------------------------- */
/* EDA table (E17-E18, R8-R10)                              */
static void legendre(int n, double z, double* pn, double* dpn) {
  double p0 = 1.0, p1 = z;
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  *pn = p1;
  *dpn = n * (z * p1 - p0) / (z * z - 1.0);
}

/* Gauss-Legendre nodes/weights on [-1, 1] by Newton iteration on P_n
 * (textbook; pinned against numpy.polynomial.legendre.leggauss in tests). */
static void gauss_legendre(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = cos(OR_PI * (i + 0.75) / (n + 0.5)), pn, dpn;
    for (int it = 0; it < 100; ++it) {
      legendre(n, z, &pn, &dpn);
      double dz = pn / dpn;
      z -= dz;
      if (fabs(dz) < 1e-15) break;
    }
    legendre(n, z, &pn, &dpn);
    x[i] = -z;
    w[i] = 2.0 / ((1.0 - z * z) * dpn * dpn);
  }
}

void or_gauss_legendre(int n, double* x, double* w) { gauss_legendre(n, x, w); }

/* E17: L_i(cos) = sigma_s * int_0^{t_M} exp(-sigma_t t) Phi(x_k + w t, S - t) dt,
 * emitter at the far focus at distance C, t_M from E18.  R9: the t-range is
 * cut at 40/sigma_t and split at the closest approach t = C cos; each part is
 * integrated by 4 panels of 8-point Gauss-Legendre. */
double or_table_integrand(const or_scene* sc, double C, double S, double cos_theta) {
  derived dv = derive(sc);
  double gx[8], gw[8];
  gauss_legendre(8, gx, gw);
  double tM = or_polar_distance(C, S, cos_theta);
  double tend = fmin(tM, 40.0 / dv.sigma_t);
  double tc = C * cos_theta;
  double cuts[3];
  int ncut = 0;
  cuts[ncut++] = 0.0;
  if (tc > 0.0 && tc < tend) cuts[ncut++] = tc;
  cuts[ncut++] = tend;
  double total = 0.0;
  for (int part = 0; part + 1 < ncut; ++part) {
    double a = cuts[part], b = cuts[part + 1];
    double h = (b - a) / 4.0;
    for (int panel = 0; panel < 4; ++panel) {
      double pa = a + panel * h;
      for (int i = 0; i < 8; ++i) {
        double t = pa + 0.5 * h * (1.0 + gx[i]);
        double r2 = t * t - 2.0 * t * C * cos_theta + C * C;
        double val = sc->sigma_s * exp(-dv.sigma_t * t) * or_da_flux(sc, r2, S - t);
        total += 0.5 * h * gw[i] * val;
      }
    }
  }
  return total;
}

typedef struct {
  const or_scene* sc;
  double* mass;
  uint16_t* q;
  int cell_begin, cell_end;
} table_job;

static void* table_worker(void* arg) {
  table_job* jb = (table_job*)arg;
  const or_scene* sc = jb->sc;
  double gxc[8], gwc[8];
  gauss_legendre(8, gxc, gwc);
  double F[256];
  for (int cell = jb->cell_begin; cell < jb->cell_end; ++cell) {
    int ir = cell / sc->table_ns, is = cell % sc->table_ns;
    double ratio = (ir + 0.5) / sc->table_nr;
    double S = sc->table_smin * pow(sc->table_smax / sc->table_smin, (is + 0.5) / sc->table_ns);
    double C = ratio * S;
    double dc = 2.0 / 256.0;
    double total = 0.0;
    for (int j = 0; j < 256; ++j) {
      double c0 = -1.0 + j * dc;
      double acc = 0.0;
      for (int n = 0; n < 8; ++n) {
        double cth = c0 + 0.5 * dc * (1.0 + gxc[n]);
        acc += 0.5 * dc * gwc[n] * or_table_integrand(sc, C, S, cth);
      }
      F[j] = acc;
      total += acc;
    }
    double cdf = 0.0;
    for (int j = 0; j < 256; ++j) {
      if (jb->mass) jb->mass[(size_t)cell * 256 + j] = F[j] / total;
      double qv = floor(65536.0 * cdf + 0.5);
      if (qv > 65535.0) qv = 65535.0;
      jb->q[(size_t)cell * 256 + j] = (uint16_t)qv;
      cdf += F[j] / total;
    }
  }
  return NULL;
}

int or_table_build(const or_scene* sc, double* mass, uint16_t* q, int nthreads) {
  int ncell = sc->table_nr * sc->table_ns;
  if (ncell <= 0 || !q) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > ncell) nthreads = ncell;
  pthread_t th[256];
  table_job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].sc = sc;
    jobs[t].mass = mass;
    jobs[t].q = q;
    jobs[t].cell_begin = (int)((long)ncell * t / nthreads);
    jobs[t].cell_end = (int)((long)ncell * (t + 1) / nthreads);
    pthread_create(&th[t], NULL, table_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* R10: nearest cell in (C/S, log S); invalid (gamma = 0) outside the S range. */
static int table_cell(const or_scene* sc, double C, double S, int* cell, double* margin) {
  *margin = INFINITY;
  if (!(S > 0.0)) return 0;
  double ratio = C / S;
  if (!(ratio < 1.0)) return 0;
  double fr = ratio * sc->table_nr;
  int ir = (int)floor(fr);
  double ls = (log(S) - log(sc->table_smin)) / (log(sc->table_smax) - log(sc->table_smin)) * sc->table_ns;
  if (!(ls >= 0.0) || !(ls < sc->table_ns)) return 0;
  int is = (int)floor(ls);
  if (ir >= sc->table_nr) ir = sc->table_nr - 1;
  double m1 = fmin(fr - floor(fr), ceil(fr) - fr);
  double m2 = fmin(ls - floor(ls), ceil(ls) - ls);
  *margin = fmin(m1, m2);
  *cell = ir * sc->table_ns + is;
  return 1;
}

static double q_at(const uint16_t* qc, int j) { return j >= 256 ? 65536.0 : (double)qc[j]; }

/* pdf (solid angle) of the EDA technique at cos(theta) to the emitter axis */
static double eda_pdf(const uint16_t* qc, double cos_theta, double* margin) {
  double pos = (cos_theta + 1.0) * 128.0;
  int j = (int)floor(pos);
  if (j < 0) j = 0;
  if (j > 255) j = 255;
  if (margin) *margin = fmin(pos - floor(pos), ceil(pos) - pos);
  double mass = (q_at(qc, j + 1) - q_at(qc, j)) / 65536.0;
  return mass * 128.0 / (2.0 * OR_PI);
}

/* ------------------------------------------------------------------------- */
/* one DARTS vertex           */
typedef struct {
  double x[3], w[3];
  double E, beta;
  int kind, face;
  /* per path */
  double Rm, RM, xe[3], Pe;
  int Ne;
  int bin; /* the path's time bin */
} pstate;

static double uu(const uint32_t r[12], int i) { return or_uniform(r[i]); }

/* R24, SPLIT walk direction: u8 and u9 are 23-bit integers made of bits of the
 * first Philox block that u0..u3 leave unused (u0, u2, u3 take the top 23 bits
 * of r0, r2, r3; the Sobol row of u1 only the top 5 bits of r1):
 *   u8: bits 0..22 of r1;
 *   u9: bits 0..8 of r0, then bits 0..8 of r2, then bits 0..4 of r3
 *       ((r0 & 0x1FF) << 14 | (r2 & 0x1FF) << 5 | (r3 & 0x1F)). */
static double u_split(const uint32_t r[12], int which) {
  uint32_t m = which == 0 ? (r[1] & 0x7FFFFFu)
                          : (((r[0] & 0x1FFu) << 14) | ((r[2] & 0x1FFu) << 5) | (r[3] & 0x1Fu));
  return (double)m * (1.0 / 8388608.0);
}

/* connection along wc from x, medium interval [lo, hi) of that ray.  Returns
 * the contribution (already multiplied by beta * wconn). */
static double connect(const or_scene* sc, const derived* dv, const pstate* ps, const double wc[3],
                      double wconn, double lo, double hi, int hitc, double u7, or_debug_out* dbg,
                      int* nonempty) {
  *nonempty = 0;
  if (dbg) { dbg->S_lo = dbg->S_hi = dbg->S = dbg->t = dbg->p_t = 0.0; dbg->contrib = 0.0; dbg->conn_valid = 0; dbg->m_conn = INFINITY; dbg->m_cond = INFINITY; }
  if (hitc == OR_HIT_MISS) return 0.0;
  double Cvec[3];
  sub3(ps->xe, ps->x, Cvec);
  double C = norm3(Cvec);
  double q = dot3(wc, Cvec); /* = C cos(theta) */
  double t, pt;
  const int unwarped_cam = (!sc->warped && ps->kind == OR_KIND_CAMERA);
  if (!unwarped_cam) {
    /* Case I elliptical sampling, E21, restricted to the
     * medium part [lo, hi) of the ray (case II reading R14). */
    double plo[3], phi_[3];
    madd3(ps->x, wc, lo, plo);
    double Slo_geo = lo + sqrt((ps->xe[0] - plo[0]) * (ps->xe[0] - plo[0]) + (ps->xe[1] - plo[1]) * (ps->xe[1] - plo[1]) + (ps->xe[2] - plo[2]) * (ps->xe[2] - plo[2]));
    double Shi_geo = INFINITY;
    if (isfinite(hi)) {
      madd3(ps->x, wc, hi, phi_);
      double dd[3];
      sub3(ps->xe, phi_, dd);
      Shi_geo = hi + norm3(dd);
    }
    double S_lo = fmax(ps->Rm - ps->E, Slo_geo);
    double S_hi = fmin(ps->RM - ps->E, Shi_geo);
    if (sc->parity_s_excess > 0.0) S_lo = fmax(S_lo, C + sc->parity_s_excess);
    if (dbg) { dbg->S_lo = S_lo; dbg->S_hi = S_hi; dbg->m_conn = fabs(S_hi - S_lo) / fmax(1.0, fabs(S_hi)); }
    if (!(S_hi > S_lo)) return 0.0;
    /* truncated exponential P on [S_m, S_M); or, as the
     * ablation of the same passage, P uniform ("will degrade to one of the
     * sampling method proposed by Jarabo et al.") */
    double S, pS;
    if (sc->conn_sampling == OR_CONN_UNIFORM_S) {
      S = S_lo + u7 * (S_hi - S_lo);
      pS = 1.0 / (S_hi - S_lo);
    } else if (isinf(S_hi)) {
      S = S_lo - log(1.0 - u7) / dv->sigma_t;
      pS = dv->sigma_t * exp(-dv->sigma_t * (S - S_lo));
    } else {
      double span = 1.0 - exp(-dv->sigma_t * (S_hi - S_lo));
      S = S_lo - log(1.0 - u7 * span) / dv->sigma_t;
      pS = dv->sigma_t * exp(-dv->sigma_t * (S - S_lo)) / span;
    }
    t = or_polar_distance(C, S, q / C); /* E21 */
    if (C == 0.0) t = 0.5 * S;
    pt = pS * (S - q) / (S - t); /* E22 with the Jacobian of R2 */
    if (dbg) {
      dbg->S = S;
      /* conditioning (not a decision): 1 / kappa with kappa the sum of the
       * amplification factors S/(S-q), S/(S_hi-S_lo) and (bin-bound) S/(S-C)
       * of the differences E21/E22 form; an fp32 evaluation of t and p_t is
       * accurate to ~1e-7 kappa */
      const int lo_bin = (ps->Rm - ps->E) >= Slo_geo && !(sc->parity_s_excess > 0.0 && C + sc->parity_s_excess > ps->Rm - ps->E);
      const int hi_bin = (ps->RM - ps->E) <= Shi_geo;
      double kappa = S / (S - q) + ((isinf(S_hi) || (lo_bin && hi_bin)) ? 0.0 : S / (S_hi - S_lo)) +
                     (lo_bin ? S / (S - C) : 0.0);
      dbg->m_cond = 1.0 / kappa;
    }
  } else {
    /* R17: unwarped camera vertex; the recorded time excludes the camera leg,
     * so the condition is on r2 = |x(t) - xe| in [Rm, RM): at most two
     * t-intervals on the ray, sampled by a truncated exponential. */
    double a_lo = lo;
    if (sc->parity_s_excess > 0.0) {
      double tmin = or_polar_distance(C, C + sc->parity_s_excess, q / C);
      a_lo = fmax(a_lo, tmin);
    }
    double ia[2], ib[2];
    int ni = 0;
    double radM = q * q - C * C + ps->RM * ps->RM;
    if (ps->RM > 0.0 && radM > 0.0) {
      double hM = sqrt(radM);
      double radm = q * q - C * C + ps->Rm * ps->Rm;
      if (ps->Rm > 0.0 && radm > 0.0) {
        double hm = sqrt(radm);
        ia[0] = q - hM; ib[0] = q - hm;
        ia[1] = q + hm; ib[1] = q + hM;
        ni = 2;
      } else {
        ia[0] = q - hM; ib[0] = q + hM;
        ni = 1;
      }
    }
    double ma[2] = {0, 0};
    double Z = 0.0;
    for (int i = 0; i < ni; ++i) {
      ia[i] = fmax(ia[i], a_lo);
      ib[i] = fmin(ib[i], hi);
      if (ib[i] > ia[i])
        ma[i] = exp(-dv->sigma_t * (ia[i] - lo)) - exp(-dv->sigma_t * (ib[i] - lo));
      Z += ma[i];
    }
    if (dbg) {
      dbg->S_lo = 0.0;
      dbg->S_hi = Z;
      dbg->m_conn = INFINITY; /* decision margin: distance of each interval from empty */
      for (int i = 0; i < ni; ++i) dbg->m_conn = fmin(dbg->m_conn, fabs(ib[i] - ia[i]) / fmax(1.0, fabs(ib[i])));
      /* conditioning of the R17 intervals (not a decision): the square roots of
       * q^2 - C^2 + R^2 and the interval widths against their positions */
      double kappa = 0.0;
      if (ni >= 1) kappa = fmax(kappa, C * C / radM);
      if (ni == 2) kappa = fmax(kappa, C * C / (q * q - C * C + ps->Rm * ps->Rm));
      for (int i = 0; i < ni; ++i)
        if (ib[i] > ia[i]) kappa += fabs(ib[i]) / (ib[i] - ia[i]);
      dbg->m_cond = kappa > 0.0 ? 1.0 / kappa : INFINITY;
    }
    if (!(Z > 0.0)) return 0.0;
    double v = u7 * Z;
    int k = (ni == 2 && !(v < ma[0])) ? 1 : 0;
    if (ma[0] <= 0.0) k = 1;
    double up = (k == 0) ? v / ma[0] : (v - ma[0]) / ma[1];
    if (up >= 1.0) up = nextafter(1.0, 0.0);
    double span = 1.0 - exp(-dv->sigma_t * (ib[k] - ia[k]));
    t = ia[k] - log(1.0 - up * span) / dv->sigma_t;
    pt = dv->sigma_t * exp(-dv->sigma_t * (t - lo)) / Z;
    if (dbg) dbg->S = t + 0.0;
  }
  *nonempty = 1;
  double xell[3];
  madd3(ps->x, wc, t, xell);
  double de[3];
  sub3(ps->xe, xell, de);
  double r2 = norm3(de);
  double we[3] = {de[0] / r2, de[1] / r2, de[2] / r2};
  double len2, vis;
  segment_medium(sc, xell, ps->xe, &len2, &vis);
  double Tr1 = exp(-dv->sigma_t * (t - lo));
  double Tr2 = exp(-dv->sigma_t * len2);
  double rho = or_hg_eval(sc->g, dot3(wc, we));
  double c = ps->beta * wconn * sc->sigma_s * Tr1 * rho * ps->Pe / (4.0 * OR_PI) * ps->Ne * vis * Tr2 /
             (r2 * r2 * pt);
  if (sc->parity_r_excl > 0.0 && r2 < sc->parity_r_excl) c = 0.0;
  if (dbg) {
    if (unwarped_cam) dbg->S = t + r2;
    dbg->t = t;
    dbg->x_ell[0] = xell[0]; dbg->x_ell[1] = xell[1]; dbg->x_ell[2] = xell[2];
    dbg->p_t = pt;
    dbg->contrib = c;
    dbg->conn_valid = 1;
  }
  return c;
}

/* Returns 1 if the walk continues.  *contrib receives this vertex's
 * connection (+ wall NEE) contribution. */
static int darts_vertex(const or_scene* sc, const derived* dv, const uint16_t* q, pstate* ps,
                        const uint32_t r[12], double* contrib, or_debug_out* dbg, or_stats* st) {
  *contrib = 0.0;
  double wc[3], ww[3];
  double wconn = 1.0;
  if (dbg) {
    memset(dbg, 0, sizeof(*dbg));
    dbg->m_event = dbg->m_select = dbg->m_tech = dbg->m_cell = dbg->m_hgbin = INFINITY;
    dbg->m_valid = dbg->m_conn = dbg->m_term = dbg->m_cond = INFINITY;
    dbg->istar = -1;
  }
  /* ---- step 2: direction ---- */
  if (ps->kind == OR_KIND_CAMERA) {
    memcpy(wc, ps->w, sizeof wc);
    memcpy(ww, ps->w, sizeof ww);
    if (dbg) { dbg->tech = 2; dbg->beta_dir = 1.0; }
  } else if (ps->kind == OR_KIND_WALL) {
    double n[3];
    inward_normal(ps->face, n);
    double alb = sc->wall_albedo[ps->face];
    /* R14: time-checked direct NEE from the wall vertex (wall-last paths) */
    double Cvec[3];
    sub3(ps->xe, ps->x, Cvec);
    double C = norm3(Cvec);
    double we[3] = {Cvec[0] / C, Cvec[1] / C, Cvec[2] / C};
    double cw = dot3(n, we);
    double arrive = ps->E + C;
    if (cw > 0.0 && arrive >= ps->Rm && arrive < ps->RM) {
      double len, vis;
      segment_medium(sc, ps->x, ps->xe, &len, &vis);
      double nee = ps->beta * (alb / OR_PI) * cw * ps->Pe / (4.0 * OR_PI) * ps->Ne * vis *
                   exp(-dv->sigma_t * len) / (C * C);
      if (sc->parity_r_excl > 0.0 && C < sc->parity_r_excl) nee = 0.0;
      *contrib += nee;
      if (st && nee != 0.0) {
        st->samples++;
        if (sc->spp_mode == OR_SPP_RESPONSE && sc->response[ps->bin] == 0.0) st->rejected++;
      }
      if (dbg) dbg->nee = nee;
      if (st && nee > 0.0) st->wall_nee++;
    }
    /* Lambertian: cosine-weighted hemisphere, beta *= albedo */
    double u5 = uu(r, 5), u6 = uu(r, 6);
    double rr = sqrt(u5), ph = 2.0 * OR_PI * u6;
    double lx = rr * cos(ph), ly = rr * sin(ph), lz = sqrt(fmax(0.0, 1.0 - u5));
    double b1[3], b2[3];
    onb(n, b1, b2);
    for (int i = 0; i < 3; ++i) wc[i] = ww[i] = b1[i] * lx + b2[i] * ly + n[i] * lz;
    ps->beta *= alb;
    if (dbg) { dbg->tech = 3; dbg->beta_dir = alb; }
  } else if (ps->kind == OR_KIND_SURF) {
    /* R32: surface vertex on triangle ps->face; time-checked NEE as at walls
     * (R14) with the BSDF, then a BSDF-sampled direction for the connection
     * and the walk */
    double n[3];
    side_normal(sc, ps->face, ps->w, n);
    double Cvec[3];
    sub3(ps->xe, ps->x, Cvec);
    double C = norm3(Cvec);
    double we[3] = {Cvec[0] / C, Cvec[1] / C, Cvec[2] / C};
    double cw = dot3(n, we);
    double arrive = ps->E + C;
    if (cw > 0.0 && arrive >= ps->Rm && arrive < ps->RM) {
      double len, vis;
      segment_medium(sc, ps->x, ps->xe, &len, &vis);
      double nee = ps->beta * or_bsdf_eval(sc, ps->face, ps->w, we) * cw * ps->Pe / (4.0 * OR_PI) * ps->Ne *
                   vis * exp(-dv->sigma_t * len) / (C * C);
      if (sc->parity_r_excl > 0.0 && C < sc->parity_r_excl) nee = 0.0;
      *contrib += nee;
      if (st && nee != 0.0) {
        st->samples++;
        if (sc->spp_mode == OR_SPP_RESPONSE && sc->response[ps->bin] == 0.0) st->rejected++;
      }
      if (dbg) dbg->nee = nee;
      if (st && nee > 0.0) st->wall_nee++;
    }
    double wo[3];
    double wgt = or_bsdf_sample(sc, ps->face, ps->w, uu(r, 4), uu(r, 5), uu(r, 6), wo);
    if (dbg) { dbg->tech = 4; dbg->beta_dir = wgt; }
    if (!(wgt > 0.0)) { /* sampled below the surface: the path ends */
      if (dbg) { dbg->event = 3; dbg->terminate = 1; dbg->beta_out = ps->beta; }
      if (st) st->escapes++;
      return 0;
    }
    memcpy(wc, wo, sizeof wc);
    memcpy(ww, wo, sizeof ww);
    ps->beta *= wgt;
  } else {
    /* medium vertex: one-sample MIS of EDA and HG */
    double Cvec[3];
    sub3(ps->xe, ps->x, Cvec);
    double C = norm3(Cvec);
    double S = ps->RM - ps->E; /* R11: upper residual */
    int cell = 0;
    double mcell;
    /* DA_ONLY ablation: phase-function directions only (gamma = 0) */
    int valid = sc->strategy == OR_STRATEGY_DA_ONLY ? 0 : table_cell(sc, C, S, &cell, &mcell);
    if (sc->strategy == OR_STRATEGY_DA_ONLY) mcell = INFINITY;
    double ratio = C / S;
    double gamma = valid ? ratio / (ratio + sc->alpha) : 0.0; /* E19 */
    double axis[3] = {0, 0, 1};
    if (C > 0.0) { axis[0] = Cvec[0] / C; axis[1] = Cvec[1] / C; axis[2] = Cvec[2] / C; }
    const uint16_t* qc = valid ? q + (size_t)cell * 256 : NULL;
    double u4 = uu(r, 4), u5 = uu(r, 5), u6 = uu(r, 6);
    double om[3];
    double p_eda = 0.0;
    int tech;
    double mh = INFINITY;
    if (u4 < gamma) {
      /* EDA: inverse transform of the cell's cos(theta) CDF */
      tech = 1;
      double T = (double)(r[5] >> 9) / 128.0; /* = u5 * 65536 */
      int j = 0;
      for (int jj = 0; jj < 256; ++jj)
        if ((double)qc[jj] <= T) j = jj;
      double qa = q_at(qc, j), qb = q_at(qc, j + 1);
      double frac = (T - qa) / (qb - qa);
      double cth = -1.0 + (j + frac) / 128.0;
      double phi = OR_PI * (2.0 * u6 - 1.0); /* R12: phi uniform in [-pi, pi) */
      from_frame(axis, cth, phi, om);
      p_eda = (qb - qa) / 65536.0 * 128.0 / (2.0 * OR_PI); /* the bin j is the sampled one: no decision */
    } else {
      tech = 0;
      double cth = hg_sample_cos(sc->g, u5);
      double phi = OR_PI * (2.0 * u6 - 1.0);
      from_frame(ps->w, cth, phi, om);
      if (valid) p_eda = eda_pdf(qc, dot3(om, axis), &mh);
    }
    double p_hg = or_hg_eval(sc->g, dot3(om, ps->w));
    double p_mix = gamma * p_eda + (1.0 - gamma) * p_hg;
    double ratio_w = p_hg / p_mix; /* rho_HG / p_mix, rho_HG = p_HG */
    memcpy(wc, om, sizeof wc);
    if (sc->direction_mode == OR_DIR_SPLIT) {
      /* R29 SPLIT: the MIS weight stays on the connection; the walk continues
       * with an independent HG direction. */
      wconn = ratio_w;
      double cth = hg_sample_cos(sc->g, u_split(r, 0));
      double phi = OR_PI * (2.0 * u_split(r, 1) - 1.0);
      from_frame(ps->w, cth, phi, ww);
      if (dbg) dbg->beta_dir = 1.0;
    } else {
      /* R29 REUSE (paper-literal) */
      memcpy(ww, om, sizeof ww);
      ps->beta *= ratio_w;
      if (dbg) dbg->beta_dir = ratio_w;
    }
    if (dbg) {
      dbg->tech = tech; dbg->gamma = gamma; dbg->p_eda = p_eda; dbg->p_hg = p_hg; dbg->p_mix = p_mix;
      dbg->m_tech = valid ? fabs(u4 - gamma) : INFINITY;
      dbg->m_cell = mcell;
      dbg->m_hgbin = mh;
    }
  }
  if (dbg) {
    memcpy(dbg->wc, wc, sizeof wc);
    memcpy(dbg->ww, ww, sizeof ww);
    dbg->wconn = wconn;
  }

  /* ---- intersection, reused by connection and walk ---- */
  double lo = 0, hi = 0;
  int face = -1;
  int hit = scene_intersect(sc, ps->x, ww, &lo, &hi, &face);
  double clo = lo, chi = hi;
  int hitc = hit, facec = face;
  if (sc->direction_mode == OR_DIR_SPLIT && ps->kind == OR_KIND_MEDIUM)
    hitc = scene_intersect(sc, ps->x, wc, &clo, &chi, &facec);
  if (dbg) { dbg->t_lo = lo; dbg->t_hi = hi; dbg->hit = hit; dbg->face_hit = face; dbg->tc_lo = clo; dbg->tc_hi = chi; }

  /* ---- step 3: elliptical connection ---- */
  int nonempty = 0;
  double c = connect(sc, dv, ps, wc, wconn, clo, chi, hitc, uu(r, 7), dbg, &nonempty);
  *contrib += c;
  if (st && nonempty) st->conn_nonempty++;
  /* every connection lands in the path's own bin (exact length control): a
   * path sample is rejected only if W is zero there */
  if (st && c != 0.0) {
    st->samples++;
    if (sc->spp_mode == OR_SPP_RESPONSE && sc->response[ps->bin] == 0.0) st->rejected++;
  }

  /* ---- step 1 (next vertex): DA distance sampling by RIS ---- */
  if (hit == OR_HIT_MISS) {
    if (dbg) { dbg->event = 0; dbg->terminate = 1; dbg->beta_out = ps->beta; }
    if (st) st->escapes++;
    return 0;
  }
  const double counts = (sc->warped || ps->kind != OR_KIND_CAMERA) ? 1.0 : 0.0;
  double p_m = isinf(hi) ? 1.0 : 1.0 - exp(-dv->sigma_t * (hi - lo)); /* E12, R28 */
  double u0 = uu(r, 0);
  if (dbg) { dbg->p_m = p_m; dbg->m_event = (p_m < 1.0) ? fabs(u0 - p_m) : INFINITY; }
  if (u0 < p_m && sc->strategy == OR_STRATEGY_EDA_ONLY) {
    /* EDA_ONLY ablation: one truncated-exponential distance (E13-E14, R1)
     * with epsilon = u2; weight sigma_s e^{-st(d-lo)} / (p_cand p_m) = sigma_s / sigma_t */
    double d = lo - log(1.0 - p_m * uu(r, 2)) / dv->sigma_t;
    madd3(ps->x, ww, d, ps->x);
    ps->beta *= sc->sigma_s / dv->sigma_t;
    ps->E += counts * d;
    ps->kind = OR_KIND_MEDIUM;
    memcpy(ps->w, ww, sizeof ps->w);
    if (dbg) { dbg->event = 1; dbg->istar = 0; dbg->d = d; dbg->beta_ris = sc->sigma_s / dv->sigma_t; dbg->m_select = INFINITY; dbg->m_valid = INFINITY; }
  } else if (u0 < p_m) {
    int N = sc->n_ris;
    int row = (int)floor(32.0 * uu(r, 1));
    double eps0 = uu(r, 2);
    double d[64], w[64], p_hat[64], pts[64][3];
    double W = 0.0, mval = INFINITY;
    for (int i = 0; i < N; ++i) {
      double ui = or_sobol(row, i % 8) + eps0; /* R6: Cranley-Patterson shift, mod 1 */
      ui -= floor(ui);
      d[i] = lo - log(1.0 - p_m * ui) / dv->sigma_t; /* E14 with the sign of R1 */
      madd3(ps->x, ww, d[i], pts[i]);
      double dd[3];
      sub3(pts[i], ps->xe, dd);
      double ri = norm3(dd);
      double Delta = ps->RM - ps->E - counts * d[i]; /* R4: upper residual */
      double p_cand = dv->sigma_t * exp(-dv->sigma_t * (d[i] - lo)) / p_m; /* E13 */
      p_hat[i] = 0.0;
      if (Delta > 0.0 && ri <= Delta) /* causal (Fig. 4) */
        p_hat[i] = dv->sigma_t * exp(-dv->sigma_t * (d[i] - lo)) * or_da_flux(sc, ri * ri, Delta); /* E10 */
      mval = fmin(mval, fabs(ri - Delta) / fmax(1.0, fabs(Delta)));
      w[i] = p_hat[i] / p_cand; /* E15: w = p_hat / p_candidate */
      W += w[i];
    }
    if (dbg) {
      dbg->m_valid = mval;
      for (int i = 0; i < N && i < 8; ++i) { dbg->cand_d[i] = d[i]; dbg->cand_wn[i] = W > 0 ? w[i] / W : 0.0; }
    }
    if (!(W > 0.0)) {
      /* R5: every candidate non-causal => the path cannot contribute */
      if (dbg) { dbg->event = 4; dbg->terminate = 1; dbg->beta_out = ps->beta; }
      if (st) st->ris_all_invalid++;
      return 0;
    }
    double u3 = uu(r, 3);
    int is = N - 1;
    double cum = 0.0, msel = INFINITY;
    int found = 0;
    for (int i = 0; i < N; ++i) {
      cum += w[i];
      if (i < N - 1) msel = fmin(msel, fabs(cum / W - u3));
      if (!found && cum > u3 * W) { is = i; found = 1; }
    }
    /* E15: unbiased contribution weight of the resampled candidate, then the
     * medium-event probability p_m of E12 and the throughput of E7 */
    double W_ris = (W / N) / p_hat[is];
    double beta_ris = sc->sigma_s * exp(-dv->sigma_t * (d[is] - lo)) * W_ris / p_m;
    ps->beta *= beta_ris;
    memcpy(ps->x, pts[is], sizeof ps->x);
    ps->E += counts * d[is];
    ps->kind = OR_KIND_MEDIUM;
    memcpy(ps->w, ww, sizeof ps->w);
    if (dbg) { dbg->event = 1; dbg->istar = is; dbg->d = d[is]; dbg->beta_ris = beta_ris; dbg->m_select = msel; }
  } else {
    if (hit == OR_HIT_WALL) {
      double xn[3];
      madd3(ps->x, ww, hi, xn);
      int a = face / 2;
      xn[a] = (face & 1) ? sc->bmax[a] : sc->bmin[a]; /* snap onto the wall plane */
      memcpy(ps->x, xn, sizeof xn);
      ps->E += counts * hi;
      ps->kind = OR_KIND_WALL;
      ps->face = face;
      memcpy(ps->w, ww, sizeof ps->w);
      if (dbg) { dbg->event = 2; dbg->d = hi; dbg->beta_ris = 1.0; }
    } else if (hit == OR_HIT_SURF) {
      /* R32/R33: the walk reaches the triangle (probability 1 - p_m) */
      double xn[3];
      surface_point(sc, face, ps->x, ww, hi, xn);
      memcpy(ps->x, xn, sizeof xn);
      ps->E += counts * hi;
      ps->kind = OR_KIND_SURF;
      ps->face = face;
      memcpy(ps->w, ww, sizeof ps->w);
      if (dbg) { dbg->event = 5; dbg->d = hi; dbg->beta_ris = 1.0; }
    } else {
      if (dbg) { dbg->event = 3; dbg->terminate = 1; dbg->beta_out = ps->beta; }
      if (st) st->escapes++;
      return 0;
    }
  }
  if (dbg) {
    memcpy(dbg->x_next, ps->x, sizeof ps->x);
    dbg->E_next = ps->E;
    dbg->beta_out = ps->beta;
  }
  /* early exit: no later connection can land before RM */
  double dd[3];
  sub3(ps->x, ps->xe, dd);
  double Cn = norm3(dd);
  if (dbg) dbg->m_term = fabs(ps->E + Cn - ps->RM) / fmax(1.0, ps->RM);
  if (ps->E + Cn >= ps->RM) {
    if (dbg) dbg->terminate = 1;
    if (st) st->early_exit++;
    return 0;
  }
  if (!isfinite(ps->beta)) {
    if (dbg) dbg->terminate = 1;
    return 0;
  }
  return 1;
}

void or_debug(const or_scene* sc, const uint16_t* q, int n, const or_debug_in* in, or_debug_out* out) {
  derived dv = derive(sc);
  double dt = (sc->t1 - sc->t0) / sc->n_bins;
  for (int i = 0; i < n; ++i) {
    pstate ps;
    memset(&ps, 0, sizeof ps);
    memcpy(ps.x, in[i].x, sizeof ps.x);
    memcpy(ps.w, in[i].w, sizeof ps.w);
    ps.E = in[i].E;
    ps.beta = in[i].beta;
    ps.kind = in[i].kind;
    ps.face = in[i].face;
    int e = in[i].emitter;
    ps.Rm = sc->t0 + in[i].bin * dt - sc->em_t[e];
    ps.RM = sc->t0 + (in[i].bin + 1) * dt - sc->em_t[e];
    memcpy(ps.xe, sc->em_pos[e], sizeof ps.xe);
    ps.Pe = sc->em_energy[e];
    ps.Ne = sc->n_emitters;
    ps.bin = in[i].bin;
    double c;
    darts_vertex(sc, &dv, q, &ps, in[i].r, &c, &out[i], NULL);
  }
}

/* ------------------------------------------------------------------------- */
/* path start: camera ray (R19) or detector point (R18), emitter (R20)        */
static int start_path(const or_scene* sc, uint64_t seed, uint64_t id, int px, int py, pstate* ps,
                      int* emitter) {
  uint32_t a[4], b[4], c[4];
  draw4(seed, id, 0xFFFFFFFFu, 0, a);
  draw4(seed, id, 0xFFFFFFFFu, 1, b);
  draw4(seed, id, 0xFFFFFFFFu, 2, c);
  /* R20: e = floor(N_e u) with u = m 2^-23, m the 23 high bits of a[2]: the
   * exact integer floor(N_e m / 2^23) (index work, bit-exact on both sides) */
  int e = or_uniform_index(sc->n_emitters, a[2]);
  *emitter = e;
  if (sc->camera_kind == OR_CAMERA_PINHOLE) {
    double fwd[3], right[3], upc[3];
    sub3(sc->look_at, sc->cam_pos, fwd);
    normalize3(fwd);
    cross3(fwd, sc->up, right);
    normalize3(right);
    cross3(right, fwd, upc);
    double h = tan(0.5 * sc->fov_y_deg * OR_PI / 180.0);
    double aspect = (double)sc->width / sc->height;
    double sx = (2.0 * (px + or_uniform(a[0])) / sc->width - 1.0) * h * aspect;
    double sy = (1.0 - 2.0 * (py + or_uniform(a[1])) / sc->height) * h;
    for (int i = 0; i < 3; ++i) ps->w[i] = fwd[i] + sx * right[i] + sy * upc[i];
    normalize3(ps->w);
    memcpy(ps->x, sc->cam_pos, sizeof ps->x);
    ps->beta = 1.0;
  } else {
    /* uniform point in the detector ball, uniform direction: fluence estimator */
    double rad = sc->det_radius * cbrt(or_uniform(b[0]));
    double z = 1.0 - 2.0 * or_uniform(b[1]);
    double s = sqrt(fmax(0.0, 1.0 - z * z));
    double ph = 2.0 * OR_PI * or_uniform(b[2]);
    ps->x[0] = sc->cam_pos[0] + rad * s * cos(ph);
    ps->x[1] = sc->cam_pos[1] + rad * s * sin(ph);
    ps->x[2] = sc->cam_pos[2] + rad * z;
    double z2 = 1.0 - 2.0 * or_uniform(b[3]);
    double s2 = sqrt(fmax(0.0, 1.0 - z2 * z2));
    double ph2 = 2.0 * OR_PI * or_uniform(c[0]);
    ps->w[0] = s2 * cos(ph2);
    ps->w[1] = s2 * sin(ph2);
    ps->w[2] = z2;
    ps->beta = 4.0 * OR_PI;
  }
  ps->E = 0.0;
  ps->kind = OR_KIND_CAMERA;
  ps->face = -1;
  return 0;
}

/* floor(n u) for u = (r >> 9) 2^-23 (R24), as the exact integer
 * (n (r >> 9)) >> 23: an index drawn from a uniform is index work and is taken
 * in integer arithmetic (no rounding), so that every implementation of R20 and
 * R21 picks the same index. */
int or_uniform_index(int n, uint32_t r) { return (int)(((uint64_t)(uint32_t)n * (uint64_t)(r >> 9)) >> 23); }

/* R21 per-pixel bin offset o_p for SPP_PER_PIXEL ("per-frame dedicated paths",
 * PAPER.md:373): o_p = floor(B u), u the first word of the pixel's Philox draw
 * at bounce 0xFFFFFFFE.  Sample s of pixel p goes to bin b = (s + o_p) mod B. */
int or_pixel_offset(const or_scene* sc, uint64_t seed, uint64_t p) {
  uint32_t a[4];
  draw4(seed, p, 0xFFFFFFFEu, 0, a);
  return or_uniform_index(sc->n_bins, a[0]);
}

/* n_pb: the number of samples s in [0, spp) of pixel p that land in bin b,
 * i.e. of s with s = (b - o_p) mod B (mod B): the cell's estimate is the mean
 * over these samples.  PER_CELL: spp. */
uint64_t or_cell_count(const or_scene* sc, uint64_t spp, int o_p, int b) {
  if (sc->spp_mode == OR_SPP_PER_CELL) return spp;
  uint64_t B = (uint64_t)sc->n_bins;
  uint64_t rel = (uint64_t)(((long)b - o_p) % (long)B + (long)B) % B;
  return spp / B + (rel < spp % B ? 1 : 0);
}

/* R31: the sensor response W (piecewise constant over the bins) is importance
 * sampled: a path's bin is b with probability pi_b = (c_{b+1} - c_b) / 2^23,
 * c_k = round(2^23 sum_{j<k} W_j / sum_j W_j) (sums in bin order), picked by the
 * 23-bit integer m of its start uniform as the b with c_b <= m < c_{b+1}; its
 * contribution is weighted by W_b / pi_b ("sample one time interval per path",
 * PAPER.md:258; rejection-free length control). */
static void response_cdf(const or_scene* sc, uint32_t* cdf) {
  double tot = 0.0;
  for (int b = 0; b < sc->n_bins; ++b) tot += sc->response[b];
  double acc = 0.0;
  cdf[0] = 0u;
  for (int b = 0; b < sc->n_bins; ++b) {
    acc += sc->response[b];
    cdf[b + 1] = (uint32_t)floor(8388608.0 * acc / tot + 0.5);
  }
  cdf[sc->n_bins] = 8388608u;
}

static int response_bin(const or_scene* sc, const uint32_t* cdf, uint32_t m, double* weight) {
  int b = 0;
  for (int k = 0; k < sc->n_bins; ++k)
    if (cdf[k] <= m) b = k;
  /* a bin with pi_b = 0 cannot be reached: c_b <= m < c_{b+1} needs c_{b+1} > c_b */
  double pi = (double)(cdf[b + 1] - cdf[b]) / 8388608.0;
  *weight = sc->response[b] / pi;
  return b;
}

/* Test-only trace of one path id to stderr (OR_TRACE_ID, read at first render). */
static uint64_t g_trace_id = ~0ull;
static FILE* g_trace_file = NULL;
static or_debug_out g_trace_out;

/* One DARTS path; returns acc (sum of its contributions). */
static double darts_path(const or_scene* sc, const derived* dv, const uint16_t* q, uint64_t seed,
                         uint64_t id, int px, int py, int b, double* order_acc, int n_orders,
                         or_stats* st, uint32_t* nvert) {
  pstate ps;
  memset(&ps, 0, sizeof ps);
  int e;
  start_path(sc, seed, id, px, py, &ps, &e);
  double dt = (sc->t1 - sc->t0) / sc->n_bins;
  ps.Rm = sc->t0 + b * dt - sc->em_t[e];
  ps.RM = sc->t0 + (b + 1) * dt - sc->em_t[e];
  memcpy(ps.xe, sc->em_pos[e], sizeof ps.xe);
  ps.Pe = sc->em_energy[e];
  ps.Ne = sc->n_emitters;
  ps.bin = b;
  if (st) st->paths++;
  if (nvert) *nvert = 0;
  /* camera ray must meet the medium */
  {
    double lo, hi;
    int f;
    if (or_intersect(sc, ps.x, ps.w, &lo, &hi, &f) == OR_HIT_MISS) {
      if (st) st->camera_miss++;
      return 0.0;
    }
  }
  if (sc->warped || sc->camera_kind == OR_CAMERA_SPHERE_DETECTOR) {
    double dd[3];
    sub3(ps.x, ps.xe, dd);
    if (norm3(dd) >= ps.RM) {
      if (st) st->early_exit++;
      return 0.0;
    }
  }
  double acc = 0.0;
  int k;
  int alive = 1;
  for (k = 0; k < sc->max_bounces && alive; ++k) {
    uint32_t r[12];
    draw4(seed, id, (uint32_t)k, 0, r);
    draw4(seed, id, (uint32_t)k, 1, r + 4);
    r[8] = r[9] = r[10] = r[11] = 0u; /* reserved */
    double c;
    if (g_trace_id == id && g_trace_file)
      fprintf(g_trace_file, "IN %d %d %d %.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g\n", k, ps.kind, ps.face,
              ps.x[0], ps.x[1], ps.x[2], ps.w[0], ps.w[1], ps.w[2], ps.E, ps.beta);
    alive = darts_vertex(sc, dv, q, &ps, r, &c, g_trace_id == id ? &g_trace_out : NULL, st);
    if (g_trace_id == id && g_trace_file)
      fprintf(g_trace_file, "OUT %d contrib %.9g event %d hit %d face_hit %d t_hi %.9g tc_hi %.9g S %.9g t %.9g p_t %.9g "
              "istar %d d %.9g beta_out %.9g m_event %.3g m_select %.3g m_tech %.3g m_cell %.3g m_valid %.3g m_conn %.3g\n",
              k, c, g_trace_out.event, g_trace_out.hit, g_trace_out.face_hit, g_trace_out.t_hi, g_trace_out.tc_hi,
              g_trace_out.S, g_trace_out.t, g_trace_out.p_t, g_trace_out.istar, g_trace_out.d, g_trace_out.beta_out,
              g_trace_out.m_event, g_trace_out.m_select, g_trace_out.m_tech, g_trace_out.m_cell, g_trace_out.m_valid,
              g_trace_out.m_conn);
    if (st) st->vertices++;
    if (nvert) (*nvert)++;
    acc += c;
    if (order_acc && k < n_orders) order_acc[k] += c;
  }
  if (alive && k >= sc->max_bounces && st) st->cap_hits++;
  if (!isfinite(acc)) {
    if (st) st->nonfinite++;
    if (order_acc) for (int i = 0; i < n_orders; ++i) order_acc[i] = 0.0;
    return 0.0;
  }
  return acc;
}

/* Vanilla baseline: exponential free flight, phase sampling and a
 * direct shadow connection at every vertex, splatted by its own arrival time. */
static void vanilla_path(const or_scene* sc, const derived* dv, uint64_t seed, uint64_t id, int px,
                         int py, double* hrow, double* hsq_row, double inv_spp, or_stats* st,
                         double* order_rows, int n_orders, size_t cells, size_t cell0) {
  pstate ps;
  memset(&ps, 0, sizeof ps);
  int e;
  start_path(sc, seed, id, px, py, &ps, &e);
  double te = sc->em_t[e];
  const double* xe = sc->em_pos[e];
  double Pe = sc->em_energy[e];
  int Ne = sc->n_emitters;
  double dt = (sc->t1 - sc->t0) / sc->n_bins;
  if (st) st->paths++;
  {
    double lo, hi;
    int f;
    if (or_intersect(sc, ps.x, ps.w, &lo, &hi, &f) == OR_HIT_MISS) {
      if (st) st->camera_miss++;
      return;
    }
  }
  double* path_bins = hsq_row ? (double*)calloc((size_t)sc->n_bins, sizeof(double)) : NULL;
  for (int k = 0; k < sc->max_bounces; ++k) {
    uint32_t r[4];
    draw4(seed, id, (uint32_t)k, 0, r);
    if (st) st->vertices++;
    if (ps.kind == OR_KIND_MEDIUM) {
      double cth = hg_sample_cos(sc->g, or_uniform(r[1]));
      double phi = OR_PI * (2.0 * or_uniform(r[2]) - 1.0);
      double nw[3];
      from_frame(ps.w, cth, phi, nw);
      memcpy(ps.w, nw, sizeof nw);
    } else if (ps.kind == OR_KIND_WALL) {
      double n[3], b1[3], b2[3];
      inward_normal(ps.face, n);
      onb(n, b1, b2);
      double u5 = or_uniform(r[1]), u6 = or_uniform(r[2]);
      double rr = sqrt(u5), ph = 2.0 * OR_PI * u6;
      double lx = rr * cos(ph), ly = rr * sin(ph), lz = sqrt(fmax(0.0, 1.0 - u5));
      for (int i = 0; i < 3; ++i) ps.w[i] = b1[i] * lx + b2[i] * ly + n[i] * lz;
      ps.beta *= sc->wall_albedo[ps.face];
    } else if (ps.kind == OR_KIND_SURF) {
      /* R32: lobe u3, direction u1, u2 */
      double wo[3];
      double wgt = or_bsdf_sample(sc, ps.face, ps.w, or_uniform(r[3]), or_uniform(r[1]), or_uniform(r[2]), wo);
      if (!(wgt > 0.0)) { if (st) st->escapes++; break; }
      memcpy(ps.w, wo, sizeof wo);
      ps.beta *= wgt;
    }
    double lo, hi;
    int face;
    int hit = scene_intersect(sc, ps.x, ps.w, &lo, &hi, &face);
    if (hit == OR_HIT_MISS) { if (st) st->escapes++; break; }
    double counts = (sc->warped || ps.kind != OR_KIND_CAMERA) ? 1.0 : 0.0;
    double dd0[3];
    sub3(ps.x, xe, dd0);
    double Cprev = norm3(dd0);
    double d = lo - log(1.0 - or_uniform(r[0])) / dv->sigma_t;
    if (d < hi) {
      madd3(ps.x, ps.w, d, ps.x);
      ps.E += counts * d;
      ps.beta *= dv->albedo;
      ps.kind = OR_KIND_MEDIUM;
    } else if (hit == OR_HIT_WALL) {
      d = hi;
      double xn[3];
      madd3(ps.x, ps.w, hi, xn);
      int a = face / 2;
      xn[a] = (face & 1) ? sc->bmax[a] : sc->bmin[a];
      memcpy(ps.x, xn, sizeof xn);
      ps.E += counts * hi;
      ps.kind = OR_KIND_WALL;
      ps.face = face;
    } else if (hit == OR_HIT_SURF) {
      d = hi;
      double xn[3];
      surface_point(sc, face, ps.x, ps.w, hi, xn);
      memcpy(ps.x, xn, sizeof xn);
      ps.E += counts * hi;
      ps.kind = OR_KIND_SURF;
      ps.face = face;
    } else {
      if (st) st->escapes++;
      break;
    }
    double Cvec[3];
    sub3(xe, ps.x, Cvec);
    double C = norm3(Cvec);
    double arrive = te + ps.E + C;
    if (arrive >= sc->t1) { if (st) st->early_exit++; break; }
    double we[3] = {Cvec[0] / C, Cvec[1] / C, Cvec[2] / C};
    double len, vis;
    segment_medium(sc, ps.x, xe, &len, &vis);
    double c;
    if (ps.kind == OR_KIND_MEDIUM) {
      c = ps.beta * or_hg_eval(sc->g, dot3(ps.w, we));
      if (sc->parity_s_excess > 0.0 && d + C - Cprev < sc->parity_s_excess) c = 0.0;
    } else if (ps.kind == OR_KIND_SURF) {
      double n[3];
      side_normal(sc, ps.face, ps.w, n);
      c = ps.beta * or_bsdf_eval(sc, ps.face, ps.w, we) * fmax(0.0, dot3(n, we));
    } else {
      double n[3];
      inward_normal(ps.face, n);
      c = ps.beta * (sc->wall_albedo[ps.face] / OR_PI) * fmax(0.0, dot3(n, we));
    }
    c *= exp(-dv->sigma_t * len) * vis * Pe / (4.0 * OR_PI) * Ne / (C * C);
    if (sc->parity_r_excl > 0.0 && C < sc->parity_r_excl) c = 0.0;
    if (c != 0.0 && isfinite(c)) {
      int bin = arrive >= sc->t0 ? (int)floor((arrive - sc->t0) / dt) : -1;
      double wgt = 1.0;
      if (bin >= 0 && bin < sc->n_bins && sc->spp_mode == OR_SPP_RESPONSE) wgt = sc->response[bin];
      if (st) {
        st->samples++;
        if (!(bin >= 0 && bin < sc->n_bins) || wgt == 0.0) st->rejected++; /* W = 0 at its time */
      }
      if (bin >= 0 && bin < sc->n_bins && wgt != 0.0) {
        hrow[bin] += wgt * c * inv_spp;
        if (path_bins) path_bins[bin] += wgt * c;
        if (order_rows && k < n_orders) order_rows[(size_t)k * cells + cell0 + bin] += wgt * c * inv_spp;
      }
    }
  }
  if (path_bins) {
    for (int b = 0; b < sc->n_bins; ++b) hsq_row[b] += path_bins[b] * path_bins[b] * inv_spp;
    free(path_bins);
  }
}

/* ------------------------------------------------------------------------- */
typedef struct {
  const or_scene* sc;
  const uint16_t* q;
  uint64_t spp, seed, s_begin, s_end;
  double *hist, *hist_sq, *order_hist;
  int n_orders;
  or_stats st;
  int tid, nthreads;
} render_job;

static int in_window(const or_scene* sc, int b) {
  return !(sc->bin_window[1] > sc->bin_window[0]) || (b >= sc->bin_window[0] && b < sc->bin_window[1]);
}

static void* render_worker(void* arg) {
  render_job* jb = (render_job*)arg;
  const or_scene* sc = jb->sc;
  derived dv = derive(sc);
  int cw = sc->crop[2] - sc->crop[0], ch = sc->crop[3] - sc->crop[1];
  uint64_t npix_local = (uint64_t)cw * ch;
  uint64_t B = (uint64_t)sc->n_bins;
  uint64_t Npix = (uint64_t)sc->width * sc->height;
  uint64_t ns = jb->s_end - jb->s_begin;
  size_t cells = (size_t)npix_local * B;
  double* oacc = jb->order_hist ? (double*)calloc((size_t)jb->n_orders, sizeof(double)) : NULL;
  if (sc->strategy == OR_STRATEGY_VANILLA) {
    uint64_t total = npix_local * ns;
    for (uint64_t i = (uint64_t)jb->tid; i < total; i += (uint64_t)jb->nthreads) {
      uint64_t pl = i % npix_local, s = jb->s_begin + i / npix_local;
      int px = sc->crop[0] + (int)(pl % cw), py = sc->crop[1] + (int)(pl / cw);
      uint64_t p = (uint64_t)py * sc->width + px;
      uint64_t id = s * Npix + p;
      vanilla_path(sc, &dv, jb->seed, id, px, py, jb->hist + pl * B, jb->hist_sq ? jb->hist_sq + pl * B : NULL,
                   1.0 / (double)jb->spp, &jb->st, jb->order_hist, jb->n_orders, cells, pl * B);
    }
  } else if (sc->spp_mode == OR_SPP_PER_CELL) {
    uint64_t total = npix_local * B * ns;
    for (uint64_t i = (uint64_t)jb->tid; i < total; i += (uint64_t)jb->nthreads) {
      uint64_t s = jb->s_begin + i % ns;
      uint64_t rest = i / ns;
      uint64_t pl = rest % npix_local;
      int b = (int)(rest / npix_local);
      if (!in_window(sc, b)) continue;
      int px = sc->crop[0] + (int)(pl % cw), py = sc->crop[1] + (int)(pl / cw);
      uint64_t p = (uint64_t)py * sc->width + px;
      uint64_t id = (s * Npix + p) * B + (uint64_t)b;
      if (oacc) memset(oacc, 0, sizeof(double) * jb->n_orders);
      double acc = darts_path(sc, &dv, jb->q, jb->seed, id, px, py, b, oacc, jb->n_orders, &jb->st, NULL);
      double inv_n = 1.0 / (double)jb->spp;
      jb->hist[pl * B + b] += acc * inv_n;
      if (jb->hist_sq) jb->hist_sq[pl * B + b] += acc * acc * inv_n;
      if (oacc)
        for (int k = 0; k < jb->n_orders; ++k) jb->order_hist[(size_t)k * cells + pl * B + b] += oacc[k] * inv_n;
    }
  } else {
    uint64_t total = npix_local * ns;
    uint32_t* cdf = NULL;
    if (sc->spp_mode == OR_SPP_RESPONSE) {
      cdf = (uint32_t*)malloc(sizeof(uint32_t) * (B + 1));
      response_cdf(sc, cdf);
    }
    for (uint64_t i = (uint64_t)jb->tid; i < total; i += (uint64_t)jb->nthreads) {
      uint64_t pl = i % npix_local, s = jb->s_begin + i / npix_local;
      int px = sc->crop[0] + (int)(pl % cw), py = sc->crop[1] + (int)(pl / cw);
      uint64_t p = (uint64_t)py * sc->width + px;
      uint64_t id = s * Npix + p;
      /* the cell's estimate is the mean over its n samples of X = scale * acc */
      int op = 0, b;
      double inv_n, scale = 1.0;
      if (cdf) {
        uint32_t a[4];
        draw4(jb->seed, id, 0xFFFFFFFFu, 0, a); /* R24: a[3] of the path-start draw */
        b = response_bin(sc, cdf, a[3] >> 9, &scale);
        inv_n = 1.0 / (double)jb->spp; /* every path of the pixel is a sample of every cell (X = 0 off its bin) */
      } else {
        op = or_pixel_offset(sc, jb->seed, p);
        b = (int)((s + (uint64_t)op) % B);
        if (!in_window(sc, b)) continue;
        inv_n = 1.0 / (double)or_cell_count(sc, jb->spp, op, b);
      }
      if (oacc) memset(oacc, 0, sizeof(double) * jb->n_orders);
      double acc = scale * darts_path(sc, &dv, jb->q, jb->seed, id, px, py, b, oacc, jb->n_orders, &jb->st, NULL);
      if (oacc)
        for (int k = 0; k < jb->n_orders; ++k) oacc[k] *= scale;
      jb->hist[pl * B + b] += acc * inv_n;
      if (jb->hist_sq) jb->hist_sq[pl * B + b] += acc * acc * inv_n;
      if (oacc)
        for (int k = 0; k < jb->n_orders; ++k) jb->order_hist[(size_t)k * cells + pl * B + b] += oacc[k] * inv_n;
    }
    free(cdf);
  }
  free(oacc);
  return NULL;
}

int or_render(const or_scene* sc, const uint16_t* q, uint64_t spp, uint64_t seed, uint64_t s_begin,
              uint64_t s_end, double* hist, double* hist_sq, double* order_hist, int n_orders,
              or_stats* stats, int nthreads) {
  if (!hist || s_end < s_begin) return -1;
  if ((sc->strategy == OR_STRATEGY_DARTS || sc->strategy == OR_STRATEGY_EDA_ONLY) && !q) return -2;
  if (sc->spp_mode == OR_SPP_RESPONSE && !sc->response) return -3;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  int cw = sc->crop[2] - sc->crop[0], ch = sc->crop[3] - sc->crop[1];
  size_t cells = (size_t)cw * ch * sc->n_bins;
  pthread_t th[256];
  render_job* jobs = (render_job*)calloc((size_t)nthreads, sizeof(render_job));
  for (int t = 0; t < nthreads; ++t) {
    render_job* jb = &jobs[t];
    jb->sc = sc; jb->q = q; jb->spp = spp; jb->seed = seed; jb->s_begin = s_begin; jb->s_end = s_end;
    jb->tid = t; jb->nthreads = nthreads; jb->n_orders = n_orders;
    jb->hist = (double*)calloc(cells, sizeof(double));
    jb->hist_sq = hist_sq ? (double*)calloc(cells, sizeof(double)) : NULL;
    jb->order_hist = order_hist ? (double*)calloc(cells * (size_t)n_orders, sizeof(double)) : NULL;
    pthread_create(&th[t], NULL, render_worker, jb);
  }
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    render_job* jb = &jobs[t];
    for (size_t i = 0; i < cells; ++i) hist[i] += jb->hist[i];
    if (hist_sq) for (size_t i = 0; i < cells; ++i) hist_sq[i] += jb->hist_sq[i];
    if (order_hist) for (size_t i = 0; i < cells * (size_t)n_orders; ++i) order_hist[i] += jb->order_hist[i];
    if (stats) {
      stats->paths += jb->st.paths; stats->camera_miss += jb->st.camera_miss;
      stats->vertices += jb->st.vertices; stats->conn_nonempty += jb->st.conn_nonempty;
      stats->ris_all_invalid += jb->st.ris_all_invalid; stats->early_exit += jb->st.early_exit;
      stats->escapes += jb->st.escapes; stats->cap_hits += jb->st.cap_hits;
      stats->nonfinite += jb->st.nonfinite; stats->wall_nee += jb->st.wall_nee;
      stats->samples += jb->st.samples; stats->rejected += jb->st.rejected;
    }
    free(jb->hist); free(jb->hist_sq); free(jb->order_hist);
  }
  free(jobs);
  return 0;
}

int or_render_ids(const or_scene* sc, const uint16_t* q, uint64_t spp, uint64_t seed, const uint64_t* ids,
                  int n, double* acc, uint32_t* nvert) {
  derived dv = derive(sc);
  uint64_t B = (uint64_t)sc->n_bins;
  uint64_t Npix = (uint64_t)sc->width * sc->height;
  (void)spp;
  const char* tr = getenv("OR_TRACE_ID");
  const char* tf = getenv("OR_TRACE_FILE");
  g_trace_id = (tr && tf) ? strtoull(tr, NULL, 10) : ~0ull;
  if (g_trace_file) fclose(g_trace_file);
  g_trace_file = (tr && tf) ? fopen(tf, "w") : NULL;
  for (int i = 0; i < n; ++i) {
    uint64_t id = ids[i];
    uint64_t p;
    int b;
    if (sc->spp_mode == OR_SPP_PER_CELL) {
      b = (int)(id % B);
      p = (id / B) % Npix;
    } else if (sc->spp_mode == OR_SPP_RESPONSE) {
      p = id % Npix;
      uint32_t cdf_local[4097], a[4];
      if (B > 4096) return -1;
      response_cdf(sc, cdf_local);
      draw4(seed, id, 0xFFFFFFFFu, 0, a);
      double wgt;
      b = response_bin(sc, cdf_local, a[3] >> 9, &wgt);
    } else {
      p = id % Npix;
      uint64_t s = id / Npix;
      b = (int)((s + (uint64_t)or_pixel_offset(sc, seed, p)) % B);
    }
    int px = (int)(p % (uint64_t)sc->width), py = (int)(p / (uint64_t)sc->width);
    acc[i] = darts_path(sc, &dv, q, seed, id, px, py, b, NULL, 0, NULL, nvert ? &nvert[i] : NULL);
  }
  if (g_trace_file) { fclose(g_trace_file); g_trace_file = NULL; }
  return 0;
}
