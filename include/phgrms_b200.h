/*
 * phgrms_b200.h -- C ABI of the B200-native P-HGRMS denoise path.
 *
 * The reference (arXiv 1306.5390 artifact, /root/reference/proj) has no FFI:
 * its boundary is the header-only C++ API in include/phgrms/denoise.hpp.
 * Every entry point below replaces one piece of that API; the C++ drop-in
 * headers in include/phgrms/ (same names and signatures as the reference)
 * are thin wrappers over these symbols, and INTEGRATION.md shows the
 * bindings a maintainer would add.
 *
 * Conventions
 *   - Images are uint8, row-major, index r*width+c, unpadded on the host
 *     side (reference: include/phgrms/image.hpp:16-51).
 *   - Every function returns PHG_OK (0) or a negative PHG_E* code; the
 *     message of the last failure on the calling thread is phg_last_error().
 *     PHG_EINVAL carries the reference's exact std::invalid_argument text.
 *   - Host-buffer functions are synchronous and blocking, like the
 *     reference; they run on the calling thread's current device (set with
 *     phg_set_device) on a library-owned stream.
 *   - Device functions (phg_dev_*) take device pointers and a cudaStream_t
 *     passed as void*; they enqueue work and return without synchronising.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point fails with PHG_ENODEV.
 */
#ifndef PHGRMS_B200_H
#define PHGRMS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHG_ABI_VERSION 1

enum {
    PHG_OK = 0,
    PHG_EINVAL = -1, /* std::invalid_argument in the reference            */
    PHG_ECUDA = -2,  /* CUDA runtime / driver failure                      */
    PHG_ENOMEM = -3, /* device or host allocation failure                  */
    PHG_ENODEV = -4  /* no usable CUDA device / kernel image               */
};

/* BorderMode, include/phgrms/denoise.hpp:27-30 */
enum { PHG_BORDER_FAITHFUL = 0, PHG_BORDER_INBOUNDS = 1 };

/* DenoiseParams, include/phgrms/denoise.hpp:34-52 (same field order). */
typedef struct phg_params {
    int32_t alpha;          /* |a-b| < alpha, alpha in [1,255]              */
    int32_t beta;           /* window radius >= 1                          */
    int32_t max_iterations; /* iteration cap k >= 1                        */
    int32_t card_threshold; /* flagged when cardinality < threshold, >= 1  */
    int32_t border;         /* PHG_BORDER_*                                */
} phg_params;

/* PassStats, include/phgrms/denoise.hpp:71-76 (same layout). */
typedef struct phg_pass_stats {
    int32_t iteration; /* 1-based */
    int32_t _pad;
    int64_t flagged;
    int64_t replaced;
    double elapsed_ms;
} phg_pass_stats;

/* ---------------------------------------------------------------- misc */
int phg_abi_version(void);
const char* phg_last_error(void);
/* DenoiseParams::validate (denoise.hpp:41-49): PHG_OK or PHG_EINVAL. */
int phg_validate_params(const phg_params* p);
int phg_device_count(int* count);
int phg_set_device(int device);
/* Kernel launches issued by this library on the calling thread since the
 * last reset (evidence for bench.py's gpu_launches). */
int64_t phg_launch_count(void);
void phg_reset_launch_count(void);

/* -------------------------------------------- reference API, host buffers */

/* compute_cardinality (denoise.hpp:227-241): counts[r*w+c] = number of
 * in-bounds window cells alpha-similar to (r,c), centre included. */
int phg_cardinality(const uint8_t* img, int width, int height, int alpha, int beta,
                    int32_t* counts);

/* denoise_pass (denoise.hpp:243-283) with a caller-supplied cardinality map
 * of card_width x card_height; writes a fresh image to `out` and one
 * PassStats (iteration = 1). */
int phg_denoise_pass(const uint8_t* img, int width, int height, const int32_t* card,
                     int card_width, int card_height, const phg_params* p, uint8_t* out,
                     phg_pass_stats* stats);

/* denoise (denoise.hpp:292-311): iterate up to p->max_iterations, stop
 * after the first iteration that replaced nothing.  `stats` has capacity
 * p->max_iterations; *iterations_run entries are filled.  `bands` is the
 * reference's Parallel engine worker count (row_blocks partition,
 * denoise.hpp:97-107); results are bit-identical for every band count, so on
 * one device any count runs the single-image pipeline.  With the environment
 * variable PHG_BAND_ENGINE=1, bands >= 2 runs the row-band engine instead
 * (halo exchange between bands on one device; a test hook for the band logic
 * the multi-device paths share). */
int phg_denoise(const uint8_t* img, int width, int height, const phg_params* p, int bands,
                uint8_t* out, phg_pass_stats* stats, int* iterations_run);

/* Denoise of a binary PGM file (P5, maxval <= 255) into a P5 file, with the
 * file I/O overlapped with the host<->device copies: the raster is read in
 * ~16 MB row chunks into pinned staging buffers while earlier chunks are
 * copied to the device, and the result is written while later chunks come
 * back.  Header parsing, error texts and the written
 * file are the reference's read_pgm / write_pgm (pgm.hpp:98-150); P2 input
 * returns PHG_EINVAL (the drop-in falls back to load_pgm). */
int phg_denoise_pgm_file(const char* in_path, const char* out_path, const phg_params* p,
                         phg_pass_stats* stats, int* iterations_run);

/* Batch of n independent images packed [n][height][width]; stats is
 * [n][max_iterations], iterations_run is [n]. */
int phg_denoise_batch(const uint8_t* imgs, int n, int width, int height, const phg_params* p,
                      uint8_t* out, phg_pass_stats* stats, int* iterations_run);

/* The Parallel engine (denoise.hpp:97-135) with GPUs as the workers, driven
 * from one process: devices[0..ndev) are the workers of row_blocks
 * (denoise.hpp:97-107).  n > 1 splits the batch into ndev image shards, one
 * host thread per distinct device, no exchange; n == 1 splits the image into
 * ndev row bands whose halo rows the fused kernels store straight into the
 * neighbours' buffers (peer stores, phg_halo_peer; bands thinner than the
 * halo copy them after each launch).  A device may appear more than once.  Same outputs
 * and stats layout as phg_denoise_batch, bit-identical to phg_denoise.
 * Errors: PHG_EINVAL "devices must list at least one GPU", "device D does
 * not exist". */
int phg_denoise_sharded(const uint8_t* imgs, int n, int width, int height, const phg_params* p,
                        const int* devices, int ndev, uint8_t* out, phg_pass_stats* stats,
                        int* iterations_run);

/* Input generators restated from the reference (out of the hot path; used
 * to build bench inputs without the oracle): synth_image(SmoothRandom=2,
 * Gradient=0, Checker=1), image.hpp:53-106; inject_sp_noise, noise.hpp:62-89
 * (mask may be NULL; returns corrupted count or PHG_EINVAL). */
int phg_synth_image(int width, int height, uint32_t seed, int kind, uint8_t* out);
int64_t phg_inject_sp_noise(const uint8_t* img, int width, int height, double density,
                            double salt_ratio, uint32_t seed, uint8_t* out, uint8_t* mask);

/* ------------------------------------- device-resident API (HBM inputs) */

/* A pitched device layout: image i, row r, column c lives at
 * data + i*image_stride + r*pitch + c.  pitch and image_stride must be
 * multiples of 16 (TMA), data 16-byte aligned. */
typedef struct phg_dev_image {
    uint8_t* data;
    int64_t pitch;
    int64_t image_stride;
    int32_t width;
    int32_t rows; /* rows held by the buffer (band rows incl. halo, or height) */
    int32_t n_images;
    int32_t _pad;
} phg_dev_image;

/* Largest number of iterations one fused launch can take for this beta
 * (temporal blocking depth; 0 if beta has no fused kernel). */
int phg_max_fused_iterations(int beta);

/* The launches phg_dev_denoise runs for these parameters on n_images images
 * of width x rows: fills iters_per_launch (capacity cap) with the iterations
 * of each fused launch and returns their number; negative on error.  E.g.
 * k = 5: {5} for beta = 1 (temporal blocking), {1,1,1,1,1} for beta = 2
 * (whose blocking does not pay) and for beta = 1 launches of >= 128 Mpx on
 * wide regions (single-buffer T = 1 tiles).  With iters_per_launch == NULL
 * only the count is returned. */
int phg_launch_plan(const phg_params* p, int width, int rows, int n_images, int* iters_per_launch, int cap);

/* Name of the kernel one fused launch of `iters` iterations runs for these
 * parameters (static string; "" if none).  For reports and profiles. */
const char* phg_fused_kernel_name(const phg_params* p, int iters);

/* One temporally blocked launch: `iters` (1..phg_max_fused_iterations)
 * fused cardinality+removal iterations, reading `src` and writing `dst`
 * (same geometry).  Buffer row y is global image row y + row_base of an
 * image with `height` rows; only global rows [own_lo, own_hi) are written
 * to dst and counted, and src must hold valid data for global rows
 * [own_lo - beta*iters, own_hi + beta*iters) clipped to [0, height).
 * counters (device, uint64 [n_images][kcap][2] = flagged, replaced) are
 * accumulated at iteration index it0 .. it0+iters-1. */
int phg_dev_fused_step(const phg_dev_image* src, const phg_dev_image* dst, int row_base,
                       int height, int own_lo, int own_hi, const phg_params* p, int it0,
                       int iters, uint64_t* counters, int kcap, void* stream);

/* A halo mirror (multi-GPU row bands): the owned rows [lo, hi) of a launch
 * are also stored to ptr + (row - row0) * pitch -- the next buffer of a
 * neighbouring band (same pitch), a peer or CUDA-IPC-mapped pointer, so
 * the halo exchange rides inside the launch (NVLink stores) instead of
 * following it. */
typedef struct phg_halo_peer {
    uint8_t* ptr;
    int32_t row0; /* global row of ptr's buffer row 0 */
    int32_t lo, hi;
    int32_t _pad;
} phg_halo_peer;

/* phg_dev_fused_step plus up to two halo mirrors (single-image bands).
 * The caller orders launches across bands: launch c of a band starts after
 * launch c-1 of both neighbours has finished. */
int phg_dev_fused_step_mirrored(const phg_dev_image* src, const phg_dev_image* dst, int row_base,
                                int height, int own_lo, int own_hi, const phg_params* p, int it0,
                                int iters, uint64_t* counters, int kcap, const phg_halo_peer* peers,
                                int npeers, void* stream);

/* CUDA IPC for one-process-per-GPU bands: export a device pointer as a
 * 64-byte handle + its offset inside the allocation; open it in another
 * process of the node (returns the mapped pointer incl. the offset); close. */
int phg_ipc_get_handle(const void* dev_ptr, uint8_t* handle, uint64_t* offset);
int phg_ipc_open_handle(const uint8_t* handle, uint64_t offset, void** dev_ptr);
int phg_ipc_close(void* dev_ptr, uint64_t offset);

/* Full k-iteration denoise of whole images resident on the device:
 * reads src, leaves the result in dst, uses tmp as the ping-pong partner
 * (src is never written, so the call is repeatable).  counters as above
 * with kcap = p->max_iterations, zeroed by the call. */
int phg_dev_denoise(const phg_dev_image* src, const phg_dev_image* dst,
                    const phg_dev_image* tmp, const phg_params* p, uint64_t* counters,
                    void* stream);

/* Standalone passes on device buffers (cardinality int32 pitched by
 * card_pitch elements). */
int phg_dev_cardinality(const phg_dev_image* src, int alpha, int beta, int32_t* card,
                        int64_t card_pitch, void* stream);
int phg_dev_removal(const phg_dev_image* src, const int32_t* card, int64_t card_pitch,
                    const phg_params* p, const phg_dev_image* dst, uint64_t* counters,
                    void* stream);

/* Metrics on either side of the denoise loop (metrics.hpp).
 * residual_noise_count (metrics.hpp:52-59): pixels whose cardinality C is
 * below card_threshold; beta = 1 runs the fp16 two-tile sweep without
 * writing the map.  sse: the exact uint64 numerator of mse
 * (metrics.hpp:25-35); mse = sse / (w*h), psnr from mse on the host.
 * Errors: "alpha must be in [1, 255]", "beta must be >= 1",
 * "card_threshold must be >= 1" (PHG_EINVAL). */
int phg_residual_noise_count(const uint8_t* img, int width, int height, int alpha, int beta,
                             int card_threshold, uint64_t* count);
int phg_sse(const uint8_t* a, const uint8_t* b, int width, int height, uint64_t* sse);
/* Device forms: counts[n_images] / sse[1] are device uint64 accumulated into
 * (zero them first); a and b share geometry. */
int phg_dev_residual_count(const phg_dev_image* img, int alpha, int beta, int card_threshold,
                           uint64_t* counts, void* stream);
int phg_dev_sse(const phg_dev_image* a, const phg_dev_image* b, uint64_t* sse, void* stream);

/* On-device, counter-based input generators for giga-pixel workloads
 * (kernel_gen.cuh).  The same structure as the
 * reference's SmoothRandom synth_image (white noise + clamped 3x3 mean) and
 * salt-and-pepper injection, but every pixel is a pure function of (seed,
 * image, row, column): NOT bit-equal to the mt19937 generators, and the noise
 * is Bernoulli(density) per pixel (expected, not exact, count).  The
 * buffer holds global rows [row_base, row_base + rows) of images `height`
 * rows tall (a row band; 0 and rows for whole images).  count (device
 * uint64, may be null) accumulates the corrupted pixels. */
int phg_dev_synth_smooth(const phg_dev_image* out, int row_base, int height, uint64_t seed, void* stream);
int phg_dev_inject_noise(const phg_dev_image* img, int row_base, int height, double density,
                         double salt_ratio, uint64_t seed, uint64_t* count, void* stream);

/* Diagnostic: out[S] = the fused kernels' device RMS replacement
 * round(sqrt(S/f)) (kernel_h2.cuh h2_rms, used by the beta = 1 and beta = 2
 * fused kernels) for every S in [0, n); f in {7, 8, 23, 24}, n <= 2^21.
 * The parity tests compare it with the reference's llround(sqrt(double(S)/f))
 * (denoise.hpp:163-169) exhaustively. */
int phg_debug_rms(int f, uint32_t n, uint32_t* out);

/* Turn device counters into reference PassStats: per image, truncate after
 * the first iteration with replaced == 0 (denoise.hpp:308). */
int phg_finalize_stats(const uint64_t* host_counters, int n_images, int kcap,
                       phg_pass_stats* stats, int* iterations_run);

#ifdef __cplusplus
}
#endif
#endif /* PHGRMS_B200_H */
