/*
 * dts_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU oracle for the DARTS hot path (arXiv 2402.03106,
 * reference text /root/reference/PAPER.md).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant generator with the CUDA library under
 * paper_2402_03106_b200/; this header is the oracle's own.
 *
 * Every length is a time (c = eta = 1, PAPER.md:106-110 E3 with eta/c = 1).
 * The readings R1..R29 referenced below are listed in DESIGN.md section 3.
 */
#ifndef DTS_ORACLE_H
#define DTS_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_MEDIUM_INFINITE = 0, OR_MEDIUM_SPHERE = 1, OR_MEDIUM_BOX = 2 };
enum { OR_CAMERA_PINHOLE = 0, OR_CAMERA_SPHERE_DETECTOR = 1 };
/* DA_ONLY: DA-RIS distances + phase-function directions; EDA_ONLY: exponential
 * distances + EDA/HG MIS directions; both keep the elliptical connection
 * (ablation). */
enum { OR_STRATEGY_DARTS = 0, OR_STRATEGY_VANILLA = 1, OR_STRATEGY_DA_ONLY = 2, OR_STRATEGY_EDA_ONLY = 3 };
/* distribution P of S in the elliptical sampling of E21 */
enum { OR_CONN_TRUNC_EXP = 0, OR_CONN_UNIFORM_S = 1 };
enum { OR_DIR_REUSE = 0, OR_DIR_SPLIT = 1 };
/* PER_CELL: spp paths per (pixel, bin) cell; PER_PIXEL: spp paths per pixel,
 * bin by a per-pixel offset (R21); RESPONSE: spp paths per pixel, bin drawn
 * with probability ~ the sensor response W (R31). */
enum { OR_SPP_PER_CELL = 0, OR_SPP_PER_PIXEL = 1, OR_SPP_RESPONSE = 2 };
enum { OR_KIND_CAMERA = 0, OR_KIND_MEDIUM = 1, OR_KIND_WALL = 2, OR_KIND_SURF = 3 };
enum { OR_HIT_NONE = 0, OR_HIT_OPEN = 1, OR_HIT_WALL = 2, OR_HIT_MISS = 3, OR_HIT_SURF = 4 };
/* R33: a surface vertex sits this far off its triangle, on the incident side */
#define OR_SURF_EPS 1e-4
#define OR_MAX_MATERIALS 8

typedef struct {
  double sigma_s, sigma_a, g;
  int32_t medium_shape;
  double center[3], radius, bmin[3], bmax[3];
  uint32_t wall_mask;
  double wall_albedo[6];
  int32_t n_emitters;
  double em_pos[8][3], em_t[8], em_energy[8];
  int32_t camera_kind;
  double cam_pos[3], look_at[3], up[3], fov_y_deg;
  int32_t width, height;
  double det_radius;
  int32_t crop[4]; /* x0, y0, x1, y1 (half-open); rendered pixels */
  double t0, t1;
  int32_t n_bins, warped;
  int32_t strategy, n_ris;
  double alpha;
  int32_t max_bounces, direction_mode, spp_mode;
  double parity_r_excl, parity_s_excess;
  int32_t table_nr, table_ns;
  double table_smin, table_smax;
  int32_t conn_sampling; /* OR_CONN_* */
  const double* response; /* RESPONSE: W per bin (n_bins values >= 0), else NULL */
  /* Triangle meshes (R32, R33; surfaces of PAPER.md:105, 221, 301): thin,
   * two-sided, opaque triangles inside the medium.  tris: n_tris x 9 (v0, v1,
   * v2); tri_mat: material per triangle; mats[m] = (rho, ks, n) of the BSDF
   * f = rho [(1 - ks) / pi + ks (n + 2) / (2 pi) max(0, wo . mirror(w))^n]. */
  int32_t n_tris;
  const double* tris;
  const int32_t* tri_mat;
  int32_t n_mats;
  double mats[OR_MAX_MATERIALS][3];
  /* Test-only work restriction: with bin_window[1] > bin_window[0], paths whose
   * bin lies outside [bin_window[0], bin_window[1]) are not traced (their cells
   * stay 0; every other cell, its sample count n_pb and its estimate are those
   * of the full render).  {0, 0}: every bin. */
  int32_t bin_window[2];
} or_scene;

/* 16-bit quantised per-cell CDF of the EDA direction table (R8-R10):
 * q[(ir*ns + is)*256 + j] = round(65536 * CDF_j), j = 0..255, CDF_0 = 0,
 * clamped to 65535; the terminal CDF_256 = 65536 is implicit. */

typedef struct {
  int32_t kind, face, bin, emitter;
  double x[3], w[3];
  double E, beta;
  uint32_t r[12]; /* raw Philox words: u_i = (r_i >> 9) * 2^-23; SPLIT u8/u9 from the low bits of r0..r3; r8..r11 reserved (R24) */
} or_debug_in;

typedef struct {
  /* direction stage */
  int32_t tech; /* 0 HG, 1 EDA, 2 camera (fixed), 3 wall cosine */
  double gamma, p_eda, p_hg, p_mix, wc[3], ww[3], beta_dir, wconn;
  /* intersection stage */
  double t_lo, t_hi, tc_lo, tc_hi;
  int32_t hit, face_hit;
  /* connection stage */
  double S_lo, S_hi, S, t, x_ell[3], p_t, contrib, nee;
  int32_t conn_valid;
  /* distance stage */
  double p_m;
  int32_t event; /* 0 none(miss), 1 medium, 2 wall, 3 escape, 4 RIS all-invalid */
  double cand_d[8], cand_wn[8];
  int32_t istar;
  double d, x_next[3], beta_ris, E_next, beta_out;
  int32_t terminate;
  /* decision margins (oracle only) */
  double m_event, m_select, m_tech, m_cell, m_hgbin, m_valid, m_conn, m_term, m_cond;
} or_debug_out;

typedef struct {
  uint64_t paths, camera_miss, vertices, conn_nonempty, ris_all_invalid,
      early_exit, escapes, cap_hits, nonfinite, wall_nee;
  /* path samples (non-zero connection contributions before W) and those
   * rejected because W is zero at their recorded time (Fig. 6) */
  uint64_t samples, rejected;
} or_stats;

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double or_uniform(uint32_t r);
double or_sobol(int row, int col);
double or_da_flux(const or_scene* sc, double r2, double dt); /* E9, full constants */
double or_hg_eval(double g, double cos_theta);
double or_polar_distance(double C, double S, double cos_theta); /* E18 */
double or_hg_sample_cos(double g, double u);
void or_gauss_legendre(int n, double* x, double* w);
int or_intersect(const or_scene* sc, const double o[3], const double d[3],
                 double* t_lo, double* t_hi, int* face);
/* nearest triangle hit with 0 < t < t_max (brute force); returns the triangle or -1 */
int or_mesh_hit(const or_scene* sc, const double o[3], const double d[3], double t_max, double* t);
/* BSDF of R32 at triangle tri for incident direction w (propagation) and outgoing wo */
double or_bsdf_eval(const or_scene* sc, int tri, const double w[3], const double wo[3]);
/* R32 sampling with u4 (lobe), u5, u6: writes wo, returns f cos / p (0: below the surface) */
double or_bsdf_sample(const or_scene* sc, int tri, const double w[3], double u4, double u5, double u6,
                      double wo[3]);

/* EDA table: the quadrature rule of R9, per-bin mass (double) and the
 * quantised CDF.  mass may be NULL.  Returns 0 on success. */
int or_table_build(const or_scene* sc, double* mass, uint16_t* q, int nthreads);
double or_table_integrand(const or_scene* sc, double C, double S, double cos_theta);

/* floor(n u) for the uniform u = (r >> 9) 2^-23 of R24, exactly: (n (r >> 9)) >> 23.
 * R20's emitter index (n = N_e) and R21's pixel offset (n = n_bins). */
int or_uniform_index(int n, uint32_t r);
/* R21: the per-pixel bin offset o_p of pixel p (row-major image index) */
int or_pixel_offset(const or_scene* sc, uint64_t seed, uint64_t p);
/* R21: n_pb, the number of samples s in [0, spp) with (s + o_p) mod B = b (PER_CELL: spp) */
uint64_t or_cell_count(const or_scene* sc, uint64_t spp, int o_p, int b);

void or_debug(const or_scene* sc, const uint16_t* q, int n, const or_debug_in* in,
              or_debug_out* out);

/* Render samples s in [s_begin, s_end) of every pixel in the crop and every bin.
 * hist/hist_sq: crop_w*crop_h*n_bins doubles, ACCUMULATED.  order_hist (nullable):
 * n_orders * cells, tallies contributions by connection index k (order k+1). */
int or_render(const or_scene* sc, const uint16_t* q, uint64_t spp, uint64_t seed,
              uint64_t s_begin, uint64_t s_end, double* hist, double* hist_sq,
              double* order_hist, int n_orders, or_stats* stats, int nthreads);

/* Per-path accumulated contribution for explicit path ids (DARTS only). */
int or_render_ids(const or_scene* sc, const uint16_t* q, uint64_t spp, uint64_t seed,
                  const uint64_t* ids, int n, double* acc, uint32_t* nvert);

#ifdef __cplusplus
}
#endif
#endif
