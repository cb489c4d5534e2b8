/*
 * pivgen_b200.h -- C ABI of the B200-native PIV image-pair generator.
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes, returns
 * an int status (0 = ok, nonzero = error; the message is available from
 * pgb_last_error(), thread-local) and never throws across the boundary.
 *
 * Two families:
 *   - *_dev : device pointers (caller-owned, e.g. torch tensors), an explicit
 *             cudaStream_t passed as `void*` (NULL = legacy default stream).
 *             Asynchronous with respect to the host.
 *   - host  : host pointers; the library stages through its own device
 *             workspace and returns when the result is back in host memory.
 *             These are the drop-in twins of the reference's native seam.
 *
 * Reference interfaces each entry replaces (paths relative to the reference
 * package root pkg/src/pivgen/):
 *   pgb_splat_accumulate      <- _native.pyx:14-17  splat_accumulate(...)
 *                                 (selected by backend.py:12-23)
 *   pgb_render_oracle_dev     <- raster.py:129-151 render_oracle() (untruncated, float64)
 *   pgb_render_pairs_dev      <- raster.py:108-126 splat() x 2 frames x B pairs
 *                                 (pipeline.py:300-313 render job fan-out)
 *   pgb_advect_dev            <- particles.py:129-136 advect()
 *   pgb_sample_flow_dev       <- flowfield.py:207-232 sample_flow()
 *   pgb_finalize_dev          <- raster.py:154-161 finalize()
 *   pgb_quantize_u16_dev      <- export.py:19-20 quantize_u16()
 *   pgb_match_histogram_dev   <- raster.py:164-187 match_histogram()
 *   pgb_sample_particles_splitmix_dev <- particles.py:61-147 with rng.py:33-106
 *                                 (reference RNG mode)
 *   pgb_finalize_splitmix_dev <- raster.py:154-161 finalize() with rng.py noise
 *   pgb_generate_batch_dev    <- pipeline.py:278-329 Sampler._render_batch()
 *   pgb_generate_batch        <- same, host buffers (end-to-end path)
 *   pgb_sample_particles_dev  <- particles.py:61-147 sample_particles /
 *                                 perturb_frame2 / advect / apply_hiding
 *   pgb_perturb_frame2_dev    <- particles.py:104-126 perturb_frame2()
 *   pgb_apply_hiding_dev      <- particles.py:139-147 apply_hiding()
 *   pgb_patch_side            <- raster.py:30-38 patch_side()
 */
#ifndef PIVGEN_B200_H
#define PIVGEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGB_ABI_VERSION 1

/* Point-spread function used by the renderer. */
enum pgb_psf {
  PGB_PSF_POINT = 0, /* Eq. (1) evaluated at pixel centres (reference semantics, _native.pyx:60-66) */
  PGB_PSF_ERF = 1    /* pixel-area mean of Eq. (1) (erf integration; extension) */
};

/* What the fused epilogue writes for each frame. */
enum pgb_out_mode {
  PGB_OUT_RAW = 0,      /* raw accumulation, float32, no clamp (raster.splat output)      */
  PGB_OUT_FINAL_F32 = 1,/* clip(raw + offset + noise, 0, 1), float32 (raster.finalize)   */
  PGB_OUT_FINAL_U16 = 2,/* quantize_u16(finalize(raw)), uint16 (export.quantize_u16)     */
  PGB_OUT_ACCUM = 3     /* out += raw (float32, in place; _native.splat_accumulate)       */
};

/* Generator configuration (mirror of config.py:83-108 plus extensions). */
typedef struct pgb_config {
  int32_t height, width;            /* image_height, image_width                      */
  int32_t n_capacity;               /* GeneratorConfig.particle_capacity() (config.py:139-146) */
  int32_t psf;                      /* enum pgb_psf                                    */
  uint64_t seed;
  double ppp_lo, ppp_hi;            /* seeding_density_range                           */
  double d_lo, d_hi;                /* diameter_range                                  */
  double i0_lo, i0_hi;              /* peak_intensity_range                            */
  double rho_lo, rho_hi;            /* rho_range                                       */
  double sigma_ratio;               /* diameter_sigma_ratio                            */
  double patch_multiplier;          /* patch_multiplier                                */
  double f2_sigma_std, f2_rho_std, f2_i0_std; /* frame2_*_std                          */
  double hide_probability;
  double bg_offset, noise_std;      /* noise.background_offset, noise.gaussian_std     */
  /* laser sheet (PAPER.md:286-290 Remark 1; off when laser_enabled == 0) */
  int32_t laser_enabled;
  int32_t reserved0;
  double laser_dz0, laser_shape, laser_q, laser_z_lo, laser_z_hi, laser_w;
} pgb_config;

/* One frame of an oracle-mode particle set, device pointers, `n` entries per pair. */
typedef struct pgb_particles {
  const double* pos;           /* (pairs, n, 2) float64 x,y                                */
  const float* i0;             /* (pairs, n)                                               */
  const float* sigma_x;
  const float* sigma_y;
  const float* rho;
  const unsigned char* mask;   /* (pairs, n) contribution mask (raster.contribution_mask)  */
} pgb_particles;

/* Per-pair statistics written by the generator (device arrays of length `pairs`). */
typedef struct pgb_pair_stats {
  double* seeding_density;     /* realized ppp                                             */
  int32_t* active_count;       /* M                                                        */
  int32_t* side;               /* patch side used for both frames                          */
  float* d_max;                /* max active diameter                                      */
} pgb_pair_stats;

int pgb_abi_version(void);
const char* pgb_last_error(void);

/* Smallest odd side >= ceil(round(multiplier * max_diameter + 1, 9)) (raster.py:30-38). */
int pgb_patch_side(double max_diameter, double multiplier);

/* ---- reference seam, host buffers ------------------------------------- */
/* Accumulates (+=) every masked particle's Gaussian patch into rows
 * [row_start, row_stop) of out (height x width, float32, C order).
 * Same contract as _native.splat_accumulate (_native.pyx:14-66). */
int pgb_splat_accumulate(const double* pos, const float* i0, const float* sigma_x,
                         const float* sigma_y, const float* rho, const unsigned char* mask,
                         int64_t n, int side, float* out, int height, int width,
                         int row_start, int row_stop);

/* ---- device-pointer entry points -------------------------------------- */
/* Untruncated full-image render of one frame (render_oracle, raster.py:129-151):
 * every masked particle at every pixel in float64, summed in index order,
 * rounded to float32 once. O(n * height * width): a test oracle, not a renderer. */
int pgb_render_oracle_dev(const double* pos, const float* i0, const float* sigma_x,
                          const float* sigma_y, const float* rho, const unsigned char* mask,
                          int64_t n, int height, int width, float* out, void* stream);

int pgb_splat_accumulate_dev(const double* pos, const float* i0, const float* sigma_x,
                             const float* sigma_y, const float* rho, const unsigned char* mask,
                             int64_t n, int side, float* out, int height, int width,
                             int row_start, int row_stop, int psf, void* stream);

/* Oracle-mode batch render: `pairs` pairs x 2 frames of injected particles.
 * side_per_pair: HOST array of `pairs` ints. out_mode: enum pgb_out_mode
 * (RAW or FINAL_*; noise keyed by (seed, batch, pair_base + p)).
 * bin_counts (optional, device, int32 [pairs][2][tiles]) receives the
 * per-tile exchange counts; tiles_out (optional, host) receives the tile count. */
int pgb_render_pairs_dev(const pgb_particles* frame1, const pgb_particles* frame2,
                         int64_t n_per_pair, int pairs, const int* side_per_pair,
                         int height, int width, int psf, int out_mode,
                         double bg_offset, double noise_std, uint64_t seed, uint64_t batch,
                         int64_t pair_base, void* out1, void* out2,
                         int32_t* bin_counts, int* tiles_out, void* stream);

/* Bilinear edge-clamped advection, float64, bit-exact with the reference. */
int pgb_advect_dev(const double* pos, int64_t n, const float* flow_uv, int height, int width,
                   double* out_pos, void* stream);

/* Bilinear (u, v) at positions (flowfield.py:207-232), float64 (n, 2) output. */
int pgb_sample_flow_dev(const double* pos, int64_t n, const float* flow_uv, int height, int width,
                        double* out_uv, void* stream);

int pgb_finalize_dev(const float* raw, int pairs, int height, int width, double bg_offset,
                     double noise_std, uint64_t seed, uint64_t batch, int64_t pair_base,
                     int frame, int out_mode, void* out, void* stream);

int pgb_quantize_u16_dev(const float* img, int64_t count, uint16_t* out, void* stream);

/* Histogram specification of `images` float32 images of `pixels` each (one
 * after another, in place allowed): levels rint(x*255) clipped to [0, 255],
 * midpoint-CDF source quantiles, searchsorted('left') into target_cdf
 * (device float64[256] = cumsum(hist) / sum(hist)), output mapping / 255.
 * Bit-identical to raster.py:164-187 match_histogram(). */
int pgb_match_histogram_dev(const float* img, float* out, int64_t images, int64_t pixels,
                            const double* target_cdf, void* stream);


/* Full generation of one batch shard: global pairs [pair_base, pair_base + pairs)
 * of batch `batch`. flows: device float32 [num_fields][height][width][2];
 * pair g (global, within the batch) uses field g / pairs_per_field.
 * out_mode: FINAL_F32 / FINAL_U16 / RAW. stats and bin_counts optional. */
int pgb_generate_batch_dev(const pgb_config* cfg, uint64_t batch, int64_t pair_base, int pairs,
                           const float* flows, int num_fields, int pairs_per_field,
                           int out_mode, void* img1, void* img2, const pgb_pair_stats* stats,
                           int32_t* bin_counts, void* stream);

/* Same with HOST buffers: flows host float32, img1/img2 host (pinned recommended).
 * stats (optional) are host arrays. Synchronous. */
int pgb_generate_batch(const pgb_config* cfg, uint64_t batch, int64_t pair_base, int pairs,
                       const float* flows, int num_fields, int pairs_per_field, int out_mode,
                       void* img1, void* img2, const pgb_pair_stats* stats);

/* Particle arrays of the generator (device outputs, each (pairs, n) or (pairs, n, 2)).
 * Any output pointer may be NULL. */
typedef struct pgb_particle_out {
  double* pos1; double* pos2;
  float* i0_1; float* sx_1; float* sy_1; float* rho_1;
  float* i0_2; float* sx_2; float* sy_2; float* rho_2;
  float* diameter; float* z1;
  unsigned char* active; unsigned char* visible1; unsigned char* visible2;
} pgb_particle_out;

int pgb_sample_particles_dev(const pgb_config* cfg, uint64_t batch, int64_t pair_base, int pairs,
                             const float* flows, int num_fields, int pairs_per_field,
                             const pgb_particle_out* out, const pgb_pair_stats* stats,
                             void* stream);

/* Reference-RNG mode: the reference's splitmix64 streams (rng.py:33-106) and
 * sample_particles / perturb_frame2 / apply_hiding / advect (particles.py:
 * 61-147) for global pairs [pair_base, pair_base + pairs) of `batch`. Fills
 * the arrays of `out` that are non-NULL ((pairs, n[, 2])); stats->active_count,
 * stats->side and stats->d_max are required. Uniform-derived values are
 * bit-identical to the reference; normals use normcdfinv for scipy's ndtri. */
int pgb_sample_particles_splitmix_dev(const pgb_config* cfg, uint64_t batch, int64_t pair_base, int pairs,
                                      const float* flows, int num_fields, int pairs_per_field,
                                      const pgb_particle_out* out, const pgb_pair_stats* stats, void* stream);

/* finalize() with the reference's noise stream (NOISE, lane = frame) for
 * `images` raw float32 images of `pixels` each (pairs pair_base + i). */
int pgb_finalize_splitmix_dev(const float* raw, float* out, int64_t pixels, int images, double bg_offset,
                              double noise_std, uint64_t seed, uint64_t batch, int64_t pair_base, int frame,
                              void* stream);

/* perturb_frame2 (particles.py:104-126) on caller arrays; same Philox draws as the
 * generator (stream "perturb", particle index). Output arrays may alias nothing. */
int pgb_perturb_frame2_dev(int64_t n, uint64_t seed, uint64_t batch, int64_t gpair,
                           double sd_sigma, double sd_i0, double sd_rho, const float* i0_1,
                           const float* sx_1, const float* sy_1, const float* rho_1, float* i0_2,
                           float* sx_2, float* sy_2, float* rho_2, void* stream);

/* apply_hiding (particles.py:139-147): visible_k = (U_k >= p_hide) & active. */
int pgb_apply_hiding_dev(int64_t n, uint64_t seed, uint64_t batch, int64_t gpair, double p_hide,
                         const unsigned char* active, unsigned char* visible1,
                         unsigned char* visible2, void* stream);

/* Tiling plan of the fused kernel for a config (for tests / tooling):
 * screen tiles (render work items), particle chunks (generate work items),
 * record capacity per (pair slot, frame, tile), shared memory per CTA. */
typedef struct pgb_plan_info {
  int tile_h, tile_w, tiles_y, tiles_x, chunks, chunk, capacity, halo, smem_bytes, threads;
} pgb_plan_info;
int pgb_plan(int height, int width, int64_t n_per_pair, double ppp_hi, int halo, int frames,
             pgb_plan_info* info);

/* Sum of device kernel launches issued by this library since load (for bench accounting). */
int64_t pgb_launch_count(void);

/* Particle-list overflow events on the current device since the last reset
 * (nonzero means some tile dropped particles: the batch is invalid). */
int pgb_overflow_count(void);
int pgb_overflow_reset(void);

/* ---- measurement probes ------------------------------------------------- */
/* `blocks` x 256 threads, each issuing 8 * iters dependent-free ex2.approx
 * (MUFU.EX2): the SFU issue-rate probe behind the splat's SFU roofline
 * (scripts/measure_peaks.py -> profiles/peaks.json). `sink` >= 256 floats. */
int pgb_probe_ex2_dev(int blocks, int iters, float* sink, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PIVGEN_B200_H */
