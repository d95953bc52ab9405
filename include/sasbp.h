/*
 * sasbp.h -- C ABI of libsasbp.so: B200-native time-domain backprojection (TDBP) for
 * synthetic aperture sonar, the data-parallel hot path of Gerg et al., "GPU Acceleration
 * for Synthetic Aperture Sonar Image Reconstruction" (arXiv 2101.05888).
 *
 * Citation key: P:n = PAPER.md line n; S:n = SPEC.md line n; R1..R21 = readings in DESIGN.md.
 *
 * The operation (DESIGN.md §1 "Definition"): for every pixel / voxel centre
 *   x = origin + ix*step_x + iy*step_y + iz*step_z                                   (R8)
 * the complex image is
 *   I(x) = sum_p sum_e  ehat_{p,e}((tau - t0_p) fs) * exp(+j 2 pi fc tau),
 *   tau  = (|x - tx_p| + |x - rx_{p,e}|) / c                       (Eq. 1 delay)
 * with ehat the linear interpolation of echoes[p][e][.] and echoes zero outside the
 * recorded window (R1, R2), weight 1, no beam gate, no normalisation (R6, R7, R10).
 * The inversion is the estimate of sigma(x) from e(t, x_RX) the paper poses.
 *
 * Conventions common to every call:
 *   - complex64 = two float32 (re, im) interleaved, little endian;
 *   - positions are fp64 NED metres; times in seconds; frequencies in Hz;
 *   - echoes are complex baseband, range compressed, sampled at fs, sample n taken
 *     t0_p + n/fs after ping p's transmit (R3, R4);
 *   - all entry points return a sas_status; on failure sas_last_error() gives a
 *     thread-local message.  No exception or abort crosses the ABI;
 *   - a handle lives on the CUDA device that was current at sas_bp_create and is not
 *     thread-safe; separate handles (e.g. one per device / rank) are independent;
 *   - SAS_E_CUDA is sticky: the handle must be destroyed;
 *   - NaN / Inf echoes are not scanned and propagate into the image.
 */
#ifndef SASBP_H
#define SASBP_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SASBP_API __attribute__((visibility("default")))
#else
#define SASBP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SAS_OK = 0,
  SAS_E_INVALID = -1,      /* bad argument: see each call                                   */
  SAS_E_STATE = -2,        /* call out of order (e.g. form before set_pings)                */
  SAS_E_NOMEM = -3,        /* device or pinned-host allocation failed                       */
  SAS_E_CUDA = -4,         /* CUDA runtime error (sticky for the handle)                    */
  SAS_E_UNSUPPORTED = -5   /* no usable sm_100 device, or an unsupported option             */
} sas_status;

/* Imaging grid.  Pixel (ix,iy,iz) is centred at
 * origin + ix*step_x + iy*step_y + iz*step_z.  Steps need not be axis aligned.
 * nz = 1 gives a 2D image; nz > 1 a voxel grid ("3D via 2D layers"). */
typedef struct {
  double origin[3];
  double step_x[3];
  double step_y[3];
  double step_z[3];
  int32_t nx, ny, nz;
} sas_grid;

typedef struct sas_bp_s* sas_bp_t;

/* Create a TDBP plan for `grid` on the current CUDA device and allocate its device image
 * and workspace once (the paper's slab allocator idea).
 *   fc        carrier frequency (> 0)        bandwidth  pulse bandwidth, 0 < bandwidth <= fs
 *   fs        complex sample rate (> 0)      c          sound speed (> 0), one constant (R9)
 * Errors: SAS_E_INVALID for non-finite / non-positive parameters, nx|ny|nz < 1, a zero or
 * non-finite step vector, degenerate (linearly dependent) steps when the axis has > 1
 * pixel, or more than 2^31 pixels; SAS_E_UNSUPPORTED when no sm_100 device is current;
 * SAS_E_NOMEM.  *out is NULL on failure. */
SASBP_API sas_status sas_bp_create(double fc, double bandwidth, double fs, double c, const sas_grid* grid,
                         sas_bp_t* out);

/* NULL-safe; frees every resource of the handle. */
SASBP_API void sas_bp_destroy(sas_bp_t h);

/* Copy a ping set to the device (host inputs; the caller may free them on return) and
 * replace any previous set.
 *   echoes  complex64 [P][E][Ns] host (pinned or pageable)
 *   tx      fp64 [P][3]     transmitter position per ping (stationary during transmit)
 *   rx      fp64 [P][E][3]  receiver phase centre per ping and element (stop-and-hop, R5)
 *   t0      fp64 [P] time of sample 0 after transmit, or NULL for all zero (R4)
 * Errors: SAS_E_INVALID for P|E|Ns < 1, NULL echoes/tx/rx, non-finite tx/rx/t0, P*E*Ns
 * overflow, or delays beyond 1e9 samples (sensor-to-grid distances and |t0| at fs; e.g. t0 in
 * the wrong unit); SAS_E_NOMEM; SAS_E_CUDA. Synchronous w.r.t. the host buffers. */
SASBP_API sas_status sas_bp_set_pings(sas_bp_t h, const float* echoes, int32_t P, int32_t E, int32_t Ns,
                            const double* tx, const double* rx, const double* t0);

/* As sas_bp_set_pings but `echoes_dev` is a DEVICE pointer (complex64 [P][E][Ns], 8-byte
 * aligned) that the handle BORROWS until work queued on `cuda_stream` by later form calls
 * completes; tx/rx/t0 are host arrays and are copied.  cuda_stream may be NULL (legacy
 * default stream). */
SASBP_API sas_status sas_bp_set_pings_device(sas_bp_t h, const void* echoes_dev, int32_t P, int32_t E,
                                   int32_t Ns, const double* tx, const double* rx, const double* t0,
                                   void* cuda_stream);

/* Form the image and copy it to the host: image_out complex64 [nz][ny][nx] (ix fastest).
 * Overwrites (never accumulates); may be called repeatedly.  Synchronous.
 * Errors: SAS_E_STATE before any set_pings; SAS_E_INVALID for NULL; SAS_E_CUDA. */
SASBP_API sas_status sas_bp_form(sas_bp_t h, float* image_out);

/* Form the image into DEVICE memory image_dev (complex64 [nz][ny][nx], 8-byte aligned),
 * asynchronously on cuda_stream (NULL = legacy default stream).
 * flags: 0 = overwrite, SAS_FORM_ACCUMULATE = add to the existing contents of image_dev
 * (ping-chunked / ping-sharded partial images: I(A u B) = I(A) + I(B)).
 * Ordering: the launch reads the handle's workspace (nav, owned echoes, beam axes, velocities)
 * after this call returns.  The handle records an event on cuda_stream, and every later call
 * that rewrites that workspace (sas_bp_set_pings[_device], sas_bp_form_streamed,
 * sas_bp_set_beam with axes, sas_bp_set_motion) first blocks the host until it has completed,
 * so a "set_pings(chunk); form_device(..., ACCUMULATE)" loop on any stream is race-free.  The
 * caller still owns the ordering of image_dev and of BORROWED echoes (set_pings_device) with
 * its own work on other streams. */
#define SAS_FORM_ACCUMULATE 1
SASBP_API sas_status sas_bp_form_device(sas_bp_t h, void* image_dev, void* cuda_stream, int32_t flags);

/* End-to-end formation from HOST echoes with the H2D copy overlapped with the backprojection:
 * the channels (ping x element rows) are split into `chunks` contiguous ranges (0 = automatic);
 * chunk c is copied on a copy stream while chunk c-1 is backprojected, each chunk accumulating
 * into the device image (I(A u B) = I(A) + I(B)), then the image is copied to image_out.
 * Arguments as sas_bp_set_pings + sas_bp_form (echoes should be pinned for the overlap to
 * happen; pageable memory works but serialises the copies).  Afterwards the handle holds the
 * ping set, so sas_bp_form / sas_bp_form_device may be called again.  Synchronous. */
SASBP_API sas_status sas_bp_form_streamed(sas_bp_t h, const float* echoes, int32_t P, int32_t E, int32_t Ns,
                                          const double* tx, const double* rx, const double* t0, float* image_out,
                                          int32_t chunks);

/* Algorithmic work counters of the current ping set (off the clock, for the metric):
 *   dense  = nx*ny*nz*P*E  pixel.ping.element terms;
 *   in_win = the terms whose interpolation support meets the record, u in (-1, Ns)
 *            (SURVEY §8(d) N_u), counted on the device in fp32 (K3); with a beam set
 *            (sas_bp_set_beam) only terms inside the cone(s) are counted.  Either may be NULL. */
SASBP_API sas_status sas_bp_count_terms(sas_bp_t h, uint64_t* dense, uint64_t* in_win);

/* The execution plan chosen for the current grid and ping set (diagnostics / tests):
 *   tile      pixels per CTA tile (x, y, z)
 *   window    samples staged per (tile, channel): cells of the interpolation window
 *   rx_mode   0 = 3-term series, 1 = 4-term series, 2 = exact receive-leg delay (chosen from
 *             the series truncation bound), 3 = refracted (sas_bp_set_medium)
 *   tma       1 = windows staged by TMA tensor loads, 0 = cp.async fallback (odd Ns, unaligned
 *             device echoes, or SASBP_NO_TMA=1 in the environment at set_pings time)
 *   batch     channels (ping x element) staged per pipeline step
 *   ctas_per_sm  resident CTAs per SM of the last form's kernel (0 before the first form)
 *   tail_split   2 when the last form split its last, at most half-full wave of tiles into two
 *                channel halves per tile (partial images added atomically into the zeroed image;
 *                never for SAS_FORM_ACCUMULATE), else 1 (0 before the first form)
 * Errors: SAS_E_INVALID for NULL; rx_mode / tma are -1 before the first set_pings. */
typedef struct {
  int32_t tile[3];
  int32_t window;
  int32_t rx_mode;
  int32_t tma;
  int32_t batch;
  int32_t ctas_per_sm;
  int32_t tail_split;
} sas_bp_plan;
SASBP_API sas_status sas_bp_get_plan(sas_bp_t h, sas_bp_plan* out);

/* Field-of-view gating and ray culling (P:160-162 ray culling, P:310/315
 * bistatic; reading R15).  With a beam set, form computes the GATED sum
 *   I_g(x) = sum_{p,e} [x in FOV(tx_p)] [bistatic -> x in FOV(rx_{p,e})] term_{p,e}(x)
 * with hard FWHM cones around per-ping axes a_p (along track) and b_p (boresight), NED unit
 * vectors: azimuth |v.a| <= |v| sin(az/2), elevation v.b > 0 and |v.(a x b)| <= (v.b) tan(el/2),
 * v = x - sensor.  Per-point decisions are taken in fp64 (identical to the oracle's); with cull = 1
 * the kernel skips (tile, channel) pairs whose tile provably misses a cone (exact sphere bound),
 * which never changes the result.
 *   beam  NULL -> back to the dense sum; az_fwhm in (0, inf) (>= pi disables the azimuth test),
 *         el_fwhm finite (<= 0 or >= pi disables the elevation test), bistatic / cull in {0, 1}
 *   axes  fp64 [P][2][3] = (a_p, b_p) per ping, orthonormal, copied; NULL = a = +x, b = +y
 *         for every ping (side-looking to starboard).  P must match the ping set at form time
 *         (else SAS_E_STATE).
 * Errors: SAS_E_INVALID for bad values or non-orthonormal axes; SAS_E_NOMEM; SAS_E_CUDA. */
typedef struct {
  double az_fwhm;
  double el_fwhm;
  int32_t bistatic;
  int32_t cull;
} sas_beam;
SASBP_API sas_status sas_bp_set_beam(sas_bp_t h, const sas_beam* beam, const double* axes, int32_t P);

/* Continuous receiver motion (the paper's motion model assumes continual
 * motion; reading R16): with velocities set, each ping's receivers move with the platform
 * velocity v_p during reception, the transmitter being stationary during the instantaneous
 * transmit, so the delay solves
 *   tau = ( |x - tx_p| + |x - rx_{p,e} - v_p tau| ) / c .
 * The kernel takes the exact reference solution per (tile, channel) in fp64 and the per-pixel
 * deviation to first order in the pixel offset (relative error ~ (|v|/c)(|d|/R)^2).
 *   vel  fp64 [P][3] NED m/s (|v| <= c/100), copied; NULL = stop-and-hop (R5).  P must match the
 *        ping set at form time (else SAS_E_STATE).
 * Errors: SAS_E_INVALID (non-finite or too fast), SAS_E_NOMEM, SAS_E_CUDA. */
SASBP_API sas_status sas_bp_set_motion(sas_bp_t h, const double* vel, int32_t P);

/* Tabled receiver trajectories (SURVEY §8(f) NEXT-2 "nav-time interpolation"; the paper keeps the
 * navigation in a position look-up table, and assumes continual motion; reading
 * R23): the position of receiver (p, e) during reception is given at K nodes t_k = k dt after
 * ping p's transmit and interpolated by the cubic Hermite spline with central-difference tangents
 * (second-order one-sided at the two ends; the end segments' cubics continue outside the table),
 * which reproduces any quadratic motion exactly -- lever arms turning with the platform's
 * attitude, sway / surge accelerations.  The transmitter stays at tx_p (instantaneous transmit,
 * P:92) and the delay solves
 *   tau = ( |x - tx_p| + |x - r_{p,e}(tau)| ) / c .
 * The kernel solves it exactly in fp64 at each (tile, channel) reference and follows the
 * trajectory's tangent line over the tile's delay spread (neglected: |r''| dtau^2 / 2, ~1e-7 m
 * for 1 m/s^2 over 0.5 ms).  The ping set's rx positions remain the ones the FOV gate uses
 * (reading R22).
 *   lut  fp64 [P][E][K][3] NED metres, copied; NULL = no table (back to fixed receivers).
 *        Replaces velocities set by sas_bp_set_motion (and vice versa: one motion model at a time).
 *        P and E must match the ping set at form time (else SAS_E_STATE).
 *   K    3..65536 nodes;  dt  node spacing in seconds (> 0).
 * Errors: SAS_E_INVALID (non-finite values, K or dt out of range, a node step faster than c/100),
 * SAS_E_NOMEM, SAS_E_CUDA.  Not combinable with sas_bp_set_medium or sas_bp_set_weighting
 * (form returns SAS_E_UNSUPPORTED). */
SASBP_API sas_status sas_bp_set_nav(sas_bp_t h, const double* lut, int32_t P, int32_t E, int32_t K, double dt);

/* Sediment-water refraction (reading R17): a flat interface
 * at z = zb (NED, z down) with sound speed c (create) above and c2 below; each leg's travel time
 * follows Fermat's principle (Snell's law), straight in the water for points above the
 * interface.  The kernel takes fp64 reference times per (tile, channel) and solves the
 * refraction point per term in fp32 (3 Newton steps; the time is stationary at the solution).
 *   c2 <= 0 -> back to isovelocity (R9).  Every sensor must be above the interface at form time
 *   (else SAS_E_INVALID); cannot be combined with sas_bp_set_motion (SAS_E_UNSUPPORTED).
 * Errors: SAS_E_INVALID for non-finite values; SAS_E_UNSUPPORTED if the window for a slow
 * sediment would not fit shared memory. */
SASBP_API sas_status sas_bp_set_medium(sas_bp_t h, double zb, double c2);

/* Spreading compensation (reading R18): with spreading = 1 every term is
 * multiplied by w = |x - tx_p| |x - rx_{p,e}|, the inverse of the spherical-spreading amplitude
 * 1/(|x_TX - x| |x_RX - x|) of Eq. (eqn:backprojection).  spreading = 0 (the
 * default) is the unweighted sum (R6).  Defined for stop-and-hop straight rays: form returns
 * SAS_E_UNSUPPORTED when combined with sas_bp_set_motion or sas_bp_set_medium.
 * Errors: SAS_E_INVALID for a NULL handle or spreading not in {0, 1}. */
SASBP_API sas_status sas_bp_set_weighting(sas_bp_t h, int32_t spreading);

/* Bytes of device memory the handle owns (image + workspace + owned ping copy). */
SASBP_API size_t sas_bp_workspace_bytes(sas_bp_t h);

/* Matched-filter range compression (row a1; the paper presumes compressed data; R14):
 *   out[ch][n] = sum_{m=0}^{Nr-1} raw[ch][n+m] * conj(replica[m]),  raw zero past Ns,
 * ch = 0..P*E-1, n = 0..Ns-1.  Host buffers, complex64; runs on the current device.
 * Errors: SAS_E_INVALID for P|E|Ns|Nr < 1 or NULL pointers; SAS_E_NOMEM; SAS_E_CUDA. */
SASBP_API sas_status sas_rangecompress(const float* raw, int32_t P, int32_t E, int32_t Ns,
                             const float* replica, int32_t Nr, float* out);

/* Device-pointer variant of sas_rangecompress, asynchronous on cuda_stream.  raw_dev and
 * out_dev must not overlap. */
SASBP_API sas_status sas_rangecompress_device(const void* raw_dev, int32_t P, int32_t E, int32_t Ns,
                                    const void* replica_dev, int32_t Nr, void* out_dev,
                                    void* cuda_stream);

/* Spectral whitening gain (Eq. (eqn:whitening); reading R21):
 *   P[k] = batch-mean M-point periodogram of raw (B = max(1, floor(Ns/M)) non-overlapping
 *          blocks per channel, zero past Ns, averaged over all nch channels and blocks)
 *   G[k] = h(1 / (gamma mean_k P + P[k])),  h = division by max_k (minimum attenuation 0 dB)
 * G is a power gain (gamma = 0 makes G P constant).  raw: complex64 [nch][Ns]; G: float [M] out,
 * HOST.  M must be 1 or even and <= 256; gamma >= 0 finite.
 * Errors: SAS_E_INVALID for bad sizes / gamma / NULL pointers or an all-zero batch (no spectrum);
 * SAS_E_NOMEM; SAS_E_CUDA. */
SASBP_API sas_status sas_whitening_gain(const float* raw, int32_t nch, int32_t Ns, int32_t M, double gamma, float* G);

/* Device variant: raw_dev and G_dev (float [M]) on the device, asynchronous on cuda_stream; an
 * all-zero batch writes NaN to every G_dev[k] instead of failing. */
SASBP_API sas_status sas_whitening_gain_device(const void* raw_dev, int32_t nch, int32_t Ns, int32_t M, double gamma,
                                               float* G_dev, void* cuda_stream);

/* Whitened range compression (R21 + R14): the data are filtered with the amplitude response
 * sqrt(G[k]) at f = k fs / M (the M-tap frequency-sampling FIR over one centred period,
 * w[i] = (1/M) sum_k sqrt(G[k]) exp(+j 2 pi k i / M), i = -M/2 .. M/2-1), then matched filtered:
 *   out[ch][n] = sum_m (w * raw_ch)[n + m] conj(replica[m]),  n = 0..Ns-1, raw zero outside 0..Ns-1.
 * Computed as ONE K1 pass with the composed filter conj(w) (x) replica (Nr + M - 1 taps, start lag
 * 1 - M/2).  G: float [M], HOST for this call (device for the _device variant), finite, >= 0.
 * Errors: SAS_E_INVALID (sizes, M not 1 or even <= 256, negative / non-finite G, NULL);
 * SAS_E_UNSUPPORTED if Nr + M - 1 > 8192; SAS_E_NOMEM; SAS_E_CUDA. */
SASBP_API sas_status sas_rangecompress_whitened(const float* raw, int32_t P, int32_t E, int32_t Ns,
                                                const float* replica, int32_t Nr, const float* G, int32_t M,
                                                float* out);

/* Device variant (raw_dev, replica_dev, G_dev, out_dev on the device; asynchronous). */
SASBP_API sas_status sas_rangecompress_whitened_device(const void* raw_dev, int32_t P, int32_t E, int32_t Ns,
                                                       const void* replica_dev, int32_t Nr, const float* G_dev,
                                                       int32_t M, void* out_dev, void* cuda_stream);

/* Band-limited xU upsampling by the 8-tap windowed sinc (SPEC S:396
 * "8-tap windowed-sinc on the upsampled (x4) compressed series"; reading R19):
 *   out[ch][U n + r] = sum_{m=-3}^{4} in[ch][n + m] L(r/U - m),  L(s) = sinc(s) sinc(s/4), |s| < 4,
 * in zero outside 0..Ns-1, ch = 0..nch-1, n = 0..Ns-1, r = 0..U-1.  The output is the same record
 * at rate U fs (same t0): feed it to sas_bp_create(..., U * fs, ...) for linear TDBP on the
 * upsampled series.  in: complex64 [nch][Ns]; out: complex64 [nch][U Ns] (caller-owned, must not
 * overlap in).  Host buffers; runs on the current device.
 * Errors: SAS_E_INVALID for nch|Ns < 1, U not in 1..16, NULL pointers or size overflow;
 * SAS_E_NOMEM; SAS_E_CUDA. */
SASBP_API sas_status sas_upsample(const float* in, int32_t nch, int32_t Ns, int32_t U, float* out);

/* Device-pointer variant of sas_upsample, asynchronous on cuda_stream (8-byte aligned). */
SASBP_API sas_status sas_upsample_device(const void* in_dev, int32_t nch, int32_t Ns, int32_t U, void* out_dev,
                                         void* cuda_stream);

/* Basebanding of real passband channels ("range compression +
 * basebanding"; reading R20): mix down by the carrier measured from each ping's transmit
 * instant (R3, R4), low-pass with the caller's FIR and keep every D-th sample:
 *   z[n] = x[n] exp(-j 2 pi fc (t0_p + n / fs_in)),             x zero outside 0..Nin-1
 *   out[ch][m] = sum_{k=0}^{Nh-1} h[k] z[m D + (Nh-1)/2 - k],    m = 0..Nout-1
 * channel ch = p E + e.  Output sample m is at t0_p + m D / fs_in: rate fs_in / D, same t0.
 *   x   float [P][E][Nin] real passband samples at fs_in
 *   t0  fp64 [P] seconds after transmit of sample 0, or NULL (= 0); host, copied
 *   h   float [Nh] FIR taps, Nh odd, 1..1023; host, copied (scale by 2 to keep the passband
 *       amplitude: a cos(2 pi f t + th) -> a exp(j ...) when sum(h) = 2)
 *   out complex64 [P][E][Nout]
 * Errors: SAS_E_INVALID for P|E|Nin|Nout|D < 1, even or out-of-range Nh, fs_in or fc not finite
 * and > 0, non-finite t0, NULL pointers; SAS_E_NOMEM; SAS_E_CUDA. */
SASBP_API sas_status sas_baseband(const float* x, int32_t P, int32_t E, int32_t Nin, double fs_in, double fc,
                                  const double* t0, const float* h, int32_t Nh, int32_t D, int32_t Nout,
                                  float* out);

/* Device variant of sas_baseband: x_dev, t0_dev (fp64 [P] or NULL), h_dev (float [Nh]) and out_dev
 * all on the device; fully asynchronous on cuda_stream (no host staging or allocation).  t0_dev and
 * h_dev values are not validated (non-finite values propagate to the output). */
SASBP_API sas_status sas_baseband_device(const void* x_dev, int32_t P, int32_t E, int32_t Nin, double fs_in,
                                         double fc, const double* t0_dev, const float* h_dev, int32_t Nh, int32_t D,
                                         int32_t Nout, void* out_dev, void* cuda_stream);

/* Thread-local message describing the last failure on this thread ("" if none). */
SASBP_API const char* sas_last_error(void);

/* Library version string, e.g. "sasbp 0.1.0 sm_100a". */
SASBP_API const char* sas_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SASBP_H */
