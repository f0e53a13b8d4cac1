/*
 * dts.h -- C ABI of the B200-native DARTS hot path (libdts.so).
 *
 * DARTS: "Diffusion Approximated Residual Time Sampling for Time-of-flight
 * Rendering in Homogeneous Scattering Media", arXiv 2402.03106.  Passages are
 * cited as PAPER.md:<line> (the paper text; equations E1..E22 numbered in order
 * of appearance) and readings R1..R33 of DESIGN.md section 3.
 *
 * One estimator is exposed: per-bin dedicated transient path tracing in a
 * homogeneous medium.  Every path vertex
 *   1. samples the free-path distance by RIS against transmittance x the
 *      transient diffusion fluence for the residual time (E9-E15),
 *   2. samples the direction from the EDA table mixed with Henyey-Greenstein
 *      by one-sample MIS (E16-E19),
 *   3. makes an elliptical connection to the pulse emitter that lands exactly
 *      in the path's time bin (E20-E22),
 *   4. splats into a pixel x time-bin histogram (camera-warped or unwarped,
 *      PAPER.md:50, 76).
 * A vanilla estimator (exponential flight, phase sampling, direct shadow
 * connection) runs through the same kernels, as do the
 * ablations of PAPER.md:426-435, a tabulated sensor response
 * and opaque triangle meshes with glossy / plastic BSDFs (
 * Table 1).
 *
 * Conventions (all calls):
 *  - lengths are times: c = eta = 1 (E3).
 *  - "device" pointers are CUDA global-memory pointers of the current device
 *    (d_hist may also be peer memory mapped into it, e.g. another GPU's
 *    histogram through CUDA IPC for a fused render + reduce);
 *    "host" pointers are ordinary (pageable or pinned) CPU memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device-side calls are asynchronous on that stream unless stated.
 *  - the library owns scene/table memory; the caller owns every buffer it
 *    passes in.  Errors never abort: a status is returned and a thread-local
 *    message is available from dts_last_error().  No call falls back to a CPU
 *    path: a missing/unsupported device returns DTS_E_CUDA.
 *  - one scene may be used by one stream at a time (dts_render_rows calls on
 *    distinct bands excepted: they may run concurrently).
 */
#ifndef DTS_H
#define DTS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DTS_ABI_VERSION 2
#define DTS_MAX_EMITTERS 8
#define DTS_MAX_MATERIALS 8
#define DTS_TABLE_COS_BINS 256 /* "[-1, 1] is uniformly subdivided into 256 bins" */

typedef struct dts_scene* dts_scene_t; /* opaque, library-owned */

typedef enum {
  DTS_OK = 0,
  DTS_E_INVALID_ARG = 1, /* bad pointer, size or scene parameter */
  DTS_E_STATE = 2,       /* e.g. dts_render(DARTS) before dts_table_build */
  DTS_E_CUDA = 3,        /* CUDA runtime error / no usable sm_100 device */
  DTS_E_OOM = 4,         /* device allocation failed */
  DTS_E_RANGE = 5        /* sample range or work count out of range */
} dts_status;

enum { DTS_MEDIUM_INFINITE = 0, DTS_MEDIUM_SPHERE = 1, DTS_MEDIUM_BOX = 2 };
enum { DTS_CAMERA_PINHOLE = 0, DTS_CAMERA_SPHERE_DETECTOR = 1 };
/* DARTS: full method.  VANILLA: exponential flight + phase sampling + direct
 * shadow connection.  Ablations of PAPER.md:426-435, both
 * with the elliptical connection: DA_ONLY = DA-RIS distances + phase-function
 * directions; EDA_ONLY = exponential distances + EDA/HG MIS directions. */
enum { DTS_STRATEGY_DARTS = 0, DTS_STRATEGY_VANILLA = 1, DTS_STRATEGY_DA_ONLY = 2, DTS_STRATEGY_EDA_ONLY = 3 };
/* Distribution P of S in the elliptical sampling E21: the
 * paper's truncated exponential, or uniform (the Jarabo et al. variant). */
enum { DTS_CONN_TRUNC_EXP = 0, DTS_CONN_UNIFORM_S = 1 };
enum { DTS_DIR_REUSE = 0, DTS_DIR_SPLIT = 1 };     /* R29 */
/* PER_CELL: spp paths per (pixel, bin) cell; PER_PIXEL: spp paths per pixel,
 * bin by a per-pixel Philox offset (R21); RESPONSE: spp paths per pixel, bin
 * drawn with probability ~ the sensor response W of dts_set_response and the
 * contribution weighted by W_b / pi_b, so cell (p, b) estimates W_b H[p, b]
 * and the sum over b the W-weighted image (R31). */
enum { DTS_SPP_PER_CELL = 0, DTS_SPP_PER_PIXEL = 1, DTS_SPP_RESPONSE = 2 };

/* Scene description.  Validation (dts_scene_create): sigma_s > 0, sigma_a >= 0,
 * -1 < g < 1; 1 <= n_emitters <= 8; width, height >= 1; crop
 * inside the image and non-empty; t1 > t0; n_bins >= 1; n_ris == 8;
 * alpha >= 0 (E19); 1 <= max_bounces <= 65536; box bmax > bmin; radius > 0;
 * strategy and conn_sampling one of their enums.  Every strategy but VANILLA
 * needs dts_table_build before dts_render (DA_ONLY does not read the table). */
typedef struct {
  float sigma_s, sigma_a, g; /* homogeneous medium, HG phase */
  int32_t medium_shape;      /* DTS_MEDIUM_*; the medium is index-matched, vacuum outside */
  float center[3], radius;   /* SPHERE */
  float bmin[3], bmax[3];    /* BOX */
  uint32_t wall_mask;        /* BOX faces that are Lambertian walls: bit f, f = 2*axis + (max side) */
  float wall_albedo[6];
  int32_t n_emitters;        /* isotropic point pulse emitters (Fig. 1) */
  float em_pos[DTS_MAX_EMITTERS][3];
  float em_t[DTS_MAX_EMITTERS];      /* emission start time tau_e */
  float em_energy[DTS_MAX_EMITTERS]; /* pulse energy P_e (intensity P_e / 4 pi) */
  int32_t camera_kind;               /* DTS_CAMERA_* (R18, R19) */
  float cam_pos[3], look_at[3], up[3], fov_y_deg;
  int32_t width, height;
  float det_radius;                  /* SPHERE_DETECTOR: ball radius, centred at cam_pos */
  int32_t crop[4];                   /* x0, y0, x1, y1 half-open: the rendered pixels */
  float t0, t1;                      /* bins [t0 + b dt, t0 + (b+1) dt), dt = (t1-t0)/n_bins (R27) */
  int32_t n_bins;
  int32_t warped;                    /* 1: camera-warped (scene-to-sensor time counted, R16) */
  int32_t strategy;                  /* DTS_STRATEGY_* */
  int32_t n_ris;                     /* RIS candidates, must be 8 */
  float alpha;                       /* E19 MIS preference, paper: 0.5 */
  int32_t max_bounces;               /* connection vertices per path (R22) */
  int32_t direction_mode;            /* DTS_DIR_* (R29) */
  int32_t spp_mode;                  /* DTS_SPP_* (R21) */
  float parity_r_excl;               /* TEST ONLY: drop contributions whose last segment < r (0 = off) */
  float parity_s_excess;             /* TEST ONLY: require S - C >= eps for medium-last paths (0 = off) */
  int32_t conn_sampling;             /* DTS_CONN_* (0 = paper) */
  /* Triangle meshes (the opaque surfaces of PAPER.md:105, 221,
   * 301, Table 1; readings R32, R33 in DESIGN.md): thin, two-sided, opaque
   * triangles strictly inside the medium (every vertex >= 1e-3 inside a BOX or
   * within a SPHERE's radius - 1e-3).  A ray's medium
   * interval ends at the nearest triangle (case II of PAPER.md:301); a surface
   * vertex sits 1e-4 off its triangle on the incident side (R33), does the
   * time-checked NEE of R14 with the BSDF, samples the BSDF and connects like a
   * wall vertex.  BSDF of material m (R32):
   *   f = rho [(1 - ks) / pi + ks (n + 2) / (2 pi) max(0, wo . mirror(w))^n]
   * (Lambertian for ks = 0, glossy Phong lobe for ks = 1, plastic between).
   * n_tris = 0: no mesh (tris, tri_mat ignored).  tris / tri_mat are HOST
   * arrays copied by dts_scene_create (a BVH is built over them); the caller
   * keeps ownership.  Rejected (DTS_E_INVALID_ARG): n_tris < 0, null arrays,
   * material index outside [0, n_mats), 1 > n_mats or n_mats > DTS_MAX_MATERIALS,
   * rho or ks outside [0, 1], n < 0, a vertex outside the medium margin,
   * degenerate (zero-area) triangles. */
  int32_t n_tris;
  const float* tris;                 /* HOST, n_tris x 9 floats: v0, v1, v2 */
  const int32_t* tri_mat;            /* HOST, n_tris material indices */
  int32_t n_mats;
  float mats[DTS_MAX_MATERIALS][3];  /* rho, ks, n */
} dts_scene_desc;

/* EDA table axes (R8): n_ratio uniform bins of C/S in [0,1), n_s log-spaced
 * bins of S in [s_min, s_max], 256 cos(theta) bins.  Zero fields take the
 * defaults 16, 16, 0.01/sigma_t, t1 - min(tau_e). */
typedef struct {
  int32_t n_ratio, n_s;
  float s_min, s_max;
} dts_table_desc;

/* Debug record: one DARTS vertex with caller-fixed state and raw Philox words.
 * kind: 0 camera/detector vertex (k = 0, direction fixed = w), 1 medium vertex
 * (w = incoming direction w_{k-1}), 2 wall vertex (face = wall index), 3 surface
 * vertex of a mesh scene (face = triangle index in the caller's order, x the
 * vertex position off the triangle, R33; a record whose index is out of range
 * is returned with terminate = 1 and nothing else set).
 * u_i = (r_i >> 9) * 2^-23 (R24): u0 event, u1 Sobol row, u2 CP shift, u3 RIS
 * select, u4 technique, u5 cos/bin, u6 phi, u7 connection; the SPLIT walk's
 * u8 = bits 0..22 of r1 and u9 = bits 0..8 of r0 | 0..8 of r2 | 0..4 of r3
 * (23-bit fractions); r8..r11 are reserved. */
typedef struct {
  int32_t kind, face, bin, emitter;
  float x[3], w[3];
  double E;    /* elapsed (counted) path time at the vertex */
  float beta;  /* throughput entering the vertex */
  float pad_;
  uint32_t r[12];
} dts_debug_in;

typedef struct {
  int32_t tech;   /* 0 HG, 1 EDA, 2 camera (fixed), 3 wall cosine, 4 surface BSDF (R32) */
  float gamma, p_eda, p_hg, p_mix;
  float wc[3], ww[3]; /* connection direction, walk direction */
  float beta_dir, wconn;
  float t_lo, t_hi, tc_lo, tc_hi; /* medium interval along ww / wc */
  int32_t hit, face_hit;          /* 0 none (infinite), 1 open boundary, 2 wall, 3 miss, 4 triangle (face_hit: caller's index) */
  float S_lo, S_hi, S, t, x_ell[3], p_t, contrib, nee;
  int32_t conn_valid;
  float p_m;
  int32_t event; /* 0 miss, 1 medium (RIS), 2 wall, 3 escape, 4 RIS all-invalid, 5 triangle */
  float cand_d[8], cand_wn[8];
  int32_t istar;
  float d, x_next[3], beta_ris;
  double E_next;
  float beta_out;
  int32_t terminate;
} dts_debug_out;

/* Counters accumulated by dts_render into a caller device array of
 * DTS_NUM_COUNTERS unsigned 64-bit integers. */
enum {
  DTS_CTR_PATHS = 0,       /* paths started (incl. camera misses) */
  DTS_CTR_CAMERA_MISS,     /* primary ray misses the medium */
  DTS_CTR_VERTICES,        /* vertex iterations (connection attempts) */
  DTS_CTR_CONN_NONEMPTY,   /* connections with a non-empty S range */
  DTS_CTR_RIS_INVALID,     /* walks ended by an all-invalid candidate set (R5) */
  DTS_CTR_EARLY_EXIT,      /* walks ended by the E + C >= R_M bound */
  DTS_CTR_ESCAPES,         /* walks that left the (convex) medium */
  DTS_CTR_CAP_HITS,        /* walks truncated at max_bounces */
  DTS_CTR_NONFINITE,       /* paths discarded for a non-finite contribution */
  DTS_CTR_WALL_NEE,        /* non-zero wall NEE contributions */
  DTS_CTR_SAMPLES,         /* path samples: non-zero connection / NEE contributions before W */
  DTS_CTR_REJECTED,        /* path samples whose recorded time has W = 0 (Fig. 6) */
  DTS_CTR_WALK_VERTICES,   /* of DTS_CTR_VERTICES: walk-only MEDIUM vertices of the two-stage render
                              (their connection provably could not reach the bin, so it was not sampled) */
  DTS_CTR_CAMERA_VERTICES, /* of DTS_CTR_VERTICES: camera / detector vertices (one per walk started) */
  DTS_CTR_WALL_VERTICES,   /* of DTS_CTR_VERTICES: wall and triangle-surface vertices (DARTS kernels) */
  DTS_NUM_COUNTERS
};

/* Creates a scene (validates, derives constants, allocates the table storage
 * on the current device).  Synchronous.  *out is NULL on failure.  Histogram
 * cell indices are 32-bit: crop_w * crop_h * n_bins >= 2^32 (e.g. a 2048 x 2048
 * crop with 1024 bins) is rejected with DTS_E_RANGE. */
dts_status dts_scene_create(const dts_scene_desc* desc, dts_scene_t* out);
/* Frees the scene; waits for its pending work.  NULL is a no-op. */
dts_status dts_scene_destroy(dts_scene_t scene);

/* Builds the EDA direction table of E17 on the device by the
 * deterministic quadrature of R9 in fp64, quantised to 16-bit per-cell CDFs
 * (R10).  desc may be NULL (defaults).  Asynchronous on stream.  (With
 * DTS_TABLE_OVERLAP=1 in the environment the build is ordered after the work
 * already enqueued on stream but runs on a scene-internal stream, so that
 * later work that reads no table -- a render's start / walk stage -- overlaps
 * it; every library call that reads the table (dts_render*, dts_sample_debug,
 * dts_table_export) then waits for it.) */
dts_status dts_table_build(dts_scene_t scene, const dts_table_desc* desc, void* stream);
/* Copies the quantised table (n_ratio*n_s*256 uint16, cell-major, cell =
 * ir*n_s + is) to host memory.  Synchronous.  n must equal the table size. */
dts_status dts_table_export(dts_scene_t scene, uint16_t* host_q, size_t n);
/* Number of table entries (0 before dts_table_build). */
size_t dts_table_size(dts_scene_t scene);

/* Sets the sensor response W(t) of DTS_SPP_RESPONSE scenes: h_w (host, n =
 * n_bins floats, finite, >= 0, not all zero) is W on each bin (piecewise
 * constant).  Copied; the bin CDF of R31 is built on the host in double
 * (c_k = round(2^23 sum_{j<k} W_j / sum W)).  Synchronous.  A RESPONSE render
 * without it fails with DTS_E_STATE.  VANILLA scenes weight each connection
 * by W at its arrival time. */
dts_status dts_set_response(dts_scene_t scene, const float* h_w, int32_t n);

/* Number of histogram cells: crop_w * crop_h * n_bins, layout [y][x][bin]
 * (bin fastest) over the crop. */
size_t dts_hist_cells(dts_scene_t scene);

/* Renders samples s in [sample_begin, sample_end) of every crop pixel and
 * every bin (SPP_PER_CELL: spp paths per (pixel, bin) cell; SPP_PER_PIXEL: spp
 * paths per pixel, bin by R21; VANILLA: spp paths per pixel splatting into all
 * bins).  Path identities -- and thus every random number -- depend only on
 * (seed, s, pixel, bin), so disjoint sample ranges shard a render exactly.
 * d_hist (device, dts_hist_cells floats) is ACCUMULATED (+=) with each path's
 * contribution / (paths of its cell); d_hist_sq (device, nullable) accumulates
 * contribution^2 / (paths of its cell); d_counters (device, nullable,
 * DTS_NUM_COUNTERS uint64) accumulates the counters.  Asynchronous.
 * Tuning knobs, read from the environment on every call (defaults are the
 * measured optima of profiles/README.md): DTS_DEFER=1 selects the kernels
 * with per-warp connection queues (default off: the immediate kernels are as
 * fast or faster on every config); DTS_FLUSH_AT (1..32, default 28) is the queue length
 * that triggers a batch; DTS_REFILL_K (default 8) is the idle
 * lane-iterations that trigger a lane refill; DTS_GRAB (32..128, a multiple of
 * 32; default 1/32 of the launch per resident warp within that range) is the
 * number of work items a warp takes from the global counter at a time.  None
 * changes any result beyond fp32 summation order.  Each path's contribution
 * reaches its histogram cell by one fp32 RED; builds with
 * -DDTS_SPLAT_AGG=1 can combine a warp's same-cell contributions first
 * (DTS_SPLAT_PLAIN=0).  DTS_DEFER applies to dts_render only: row-band
 * launches (dts_render_rows, dts_render_host's bands), which may run
 * concurrently on one scene, always take the immediate kernels.
 * SPLIT scenes (R29) without meshes in BOX or SPHERE media render in two stages
 * (DESIGN.md 5.2b): a walk kernel runs the vertices whose connection provably
 * cannot reach the bin, then hands each path to a connect kernel through a
 * library-owned HBM buffer of 64 bytes per path of a chunk (chunks of at most
 * 2^27 paths, and at least two for launches of >= 2^21 paths; DTS_WF_CHUNK
 * overrides; dts_render holds two chunks' worth -- 17 GB for config 5 -- and
 * overlaps consecutive chunks on an internal stream ordered after `stream`;
 * each row band holds one chunk's worth and runs its chunks in order).  In
 * per-pixel mode a start kernel decodes the paths ahead of the walk kernel
 * (three stages, a second buffer of the same size).  REUSE
 * scenes in BOX / SPHERE media with the table in shared memory render in two
 * stages too: a start kernel runs every path's start and camera vertex, a
 * connect kernel continues the survivors (one chunk up to 2^27 paths).  Pixels
 * whose every camera ray misses the medium are not launched (camera-ray
 * culling); they are counted as started paths that missed.
 * The paths, counters and histogram are those of the one-stage kernel
 * (DTS_WAVEFRONT=0, DTS_START_STAGE=0, DTS_CULL=0 select it); failing to
 * allocate a buffer is DTS_E_OOM. */
dts_status dts_render(dts_scene_t scene, uint64_t spp, uint64_t seed, uint64_t sample_begin,
                      uint64_t sample_end, float* d_hist, float* d_hist_sq, uint64_t* d_counters,
                      void* stream);

/* dts_render over crop rows [row0, row1) only (0 <= row0 < row1 <= crop
 * height), into d_hist_band = the band's first cell (row0 * crop width *
 * n_bins floats further than the crop's).  The same paths and ids as the
 * corresponding part of dts_render.  band (0..3) picks one of 4 library-owned
 * work counters: launches that may run concurrently need distinct bands.
 * Lets a caller pipeline a large histogram band by band (render / reduce /
 * copy).  Errors as dts_render; DTS_E_INVALID_ARG for a bad row range or band.
 * Asynchronous. */
dts_status dts_render_rows(dts_scene_t scene, uint64_t spp, uint64_t seed, uint64_t sample_begin,
                           uint64_t sample_end, int32_t row0, int32_t row1, int32_t band, float* d_hist_band,
                           uint64_t* d_counters, void* stream);

/* End-to-end variant with HOST buffers: zeroes a library-owned device
 * histogram, renders, and copies the result to h_hist (dts_hist_cells floats,
 * OVERWRITTEN) and the counters to h_counters (nullable).  Synchronous.  For
 * histograms >= 256 MB it renders 4 row bands of the crop on two library-owned
 * streams (ordered after `stream`) and copies each band while the next renders;
 * pinned h_hist lets the copies overlap.  The result is that of dts_render. */
dts_status dts_render_host(dts_scene_t scene, uint64_t spp, uint64_t seed, uint64_t sample_begin,
                           uint64_t sample_end, float* h_hist, uint64_t* h_counters, void* stream);

/* Runs one DARTS vertex per record with the SAME device functions the render
 * kernel uses (direction, intersection, connection, RIS distance).  d_in/d_out
 * are device arrays of n records.  Requires the table for medium vertices.
 * Asynchronous. */
dts_status dts_sample_debug(dts_scene_t scene, int32_t n, const dts_debug_in* d_in, dts_debug_out* d_out,
                            void* stream);

/* Number of failed device-side bounds checks (table, histogram, queue and
 * response-CDF indices) since the last call, then reset; always 0 unless the
 * library was built with -DDTS_CHECKS=1 (scripts/build_variants.sh).
 * Synchronizes the device. */
dts_status dts_check_failures(uint64_t* out);

/* The large library-owned buffers (the two-stage render's hand-off records,
 * dts_render_host's device histogram) go to a process-wide per-device pool when
 * their scene is destroyed (up to 96 GB per device) and are reused by later
 * scenes.  This frees every pooled buffer.  Thread-safe; synchronous. */
dts_status dts_pool_release(void);

/* Enables peer access from the current device to device `peer` (a no-op when
 * it is the current device or already enabled), so that a render kernel on
 * this device can accumulate into a histogram that lives on `peer` and was
 * mapped here through CUDA IPC (the fused render + reduce of shard.py).
 * DTS_E_INVALID_ARG for a device index out of range, DTS_E_CUDA when the pair
 * has no peer path.  Synchronous. */
dts_status dts_enable_peer(int32_t peer);

/* Kernel launches issued by the last dts_render on this thread (for the
 * bench's gpu_launches count) and the launch geometry. */
dts_status dts_last_launch(int32_t* n_launches, int32_t* grid, int32_t* block, int32_t* smem_bytes);

const char* dts_status_string(dts_status s);
const char* dts_last_error(void);
int32_t dts_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DTS_H */
