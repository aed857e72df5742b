/*
 * gsr.h -- C-ABI of libgsr.so: B200-native (sm_100a) differentiable scale-aware 2D Gaussian
 * rasterization of GSASR (arXiv 2501.06838).
 *
 * Operation (PAPER.md line numbers):
 *   Eq. 1  G_i(x,y) = alpha_i c_i f_i(x,y)
 *   Eq. 2  f_i(x,y) = (2 pi sx sy sqrt(1-rho^2))^-1 exp[-Q/2],
 *          Q = (dx^2/sx^2 - 2 rho dx dy/(sx sy) + dy^2/sy^2)/(1-rho^2)
 *   Eq. 4  I_SR(x,y;s) = sum_i G_i(x/s, y/s),  x in [0,sW-1], y in [0,sH-1]
 *   Alg. 1 only pairs inside the window ("rasterization ratio" r, default 0.1)
 * with the readings recorded in DESIGN.md ("Readings"):
 *   - output size  Hs = floor(s*H), Ws = floor(s*W)  (fp64)                          [R4]
 *   - sample point (x/s, y/s), no half-pixel offset                                  [R3]
 *   - window: x paired with W, y with H; pixel x is inside iff x0 <= x <= x1 with
 *       x0 = floor(s*(mu_x - r*W)) + 1,  x1 = ceil(s*(mu_x + r*W)) - 1
 *     (IEEE fp64, this operation order, no FMA; bounds clamped to +-2^30), y likewise
 *     with H; clipped to the image                                                    [R1,R2]
 *   - no clamping of parameters or output                                            [R8]
 *   - a Gaussian with a non-finite field, sigma_x <= 0, sigma_y <= 0 or |rho| >= 1 is
 *     invalid: it contributes 0 and receives 0 gradient                               [R20]
 *   - backward: gradient of the fixed pair set (window edges do not move)            [R11]
 *
 * Conventions shared by every entry point:
 *   - Parameters are float32 SoA device arrays (struct-of-arrays, C order):
 *       alpha[n]            opacity alpha
 *       mu[n][2]            centre (mu_x, mu_y) in LR pixels, mu = p + o
 *       sigma[n][2]         (sigma_x, sigma_y) in LR pixels
 *       rho[n]              correlation coefficient
 *       color[n][3]         (c_r, c_g, c_b)
 *   - Images are HWC float32: out[y][x][k], k = r,g,b (Alg. 1 l.1 "(sH, sW, 3)").
 *   - ratio r is passed as double (0.1 is not an fp32-exact value); 0 < r <= 1.
 *   - Ownership: the caller allocates every buffer (inputs, outputs, workspace). The library
 *     allocates nothing, keeps no state between calls (apart from the opt-in profiler and a
 *     launch counter, see gsr_profile_*) and never synchronises the stream.
 *   - Asynchrony: every compute entry point enqueues its kernels on `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream) and returns immediately.
 *   - Errors: GSR_EINVAL for host-checkable argument errors (nothing is launched);
 *     GSR_EWORKSPACE if workspace_bytes is smaller than the matching *_workspace_bytes();
 *     GSR_ECUDA if a launch failed (cudaGetLastError after the launches). Parameter-domain
 *     violations inside the arrays are NOT errors: such Gaussians are invalid (R20).
 *   - Limits: Hs, Ws <= 65535; n < 2^31 per call; up to GSR_MAX_IMAGES images per batched call.
 *   - Thread safety: concurrent calls are safe when they use different workspaces/outputs.
 */
#ifndef GSR_H
#define GSR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GSR_OK = 0,
    GSR_EINVAL = 1,
    GSR_EWORKSPACE = 2,
    GSR_ECUDA = 3
} gsr_status;

#define GSR_MAX_IMAGES 64

/* Scale vector (reading R22; "receives the predicted 2D Gaussians with an upsampling scale
 * vector"): an image may carry two scales, `scale` = s_x along x (W) and `scale_y` = s_y along y
 * (H). Every "s" of the readings above then applies per axis: Hs = floor(s_y H),
 * Ws = floor(s_x W), sample (x/s_x, y/s_y), window bounds along x with s_x and along y with s_y.
 * scale_y = 0 means s_y = s_x (the paper's isotropic case). The single-image entry points take
 * the scalar s only; the batched ones read scale_y from gsr_image.
 *
 * One image of a (ragged) batch. All images of a call share the parameter arrays: image k owns
 * Gaussians [g_off, g_off + g_cnt). Its output block starts at float offset out_off of `out`
 * (and of grad_out for the backward) and holds rows [row_begin, row_end) of the HR image:
 * (row_end - row_begin) * Ws * 3 floats, row-major HWC. row_begin = 0, row_end = -1 means the
 * whole image (Hs rows). Row bands are how the multi-GPU path shards an image. */
typedef struct gsr_image {
    int32_t lr_h;      /* H >= 1 */
    int32_t lr_w;      /* W >= 1 */
    double scale;      /* s (s_x when scale_y != 0) >= 1, finite */
    int64_t g_off;     /* first Gaussian of this image */
    int64_t g_cnt;     /* number of Gaussians of this image (may be 0) */
    int64_t out_off;   /* float offset of this image's output block */
    int32_t row_begin; /* first HR row of the band, 0 <= row_begin */
    int32_t row_end;   /* one past the last HR row (-1 = Hs); row_begin <= row_end <= Hs */
    double scale_y;    /* scale along y (H): 0 = `scale` (the paper's scalar s); else >= 1 */
} gsr_image;

/* Library version string (static storage). */
const char* gsr_version(void);

/* Hs = floor(s*H), Ws = floor(s*W) in fp64 (reading R4). GSR_EINVAL on bad arguments. */
gsr_status gsr_out_dims(int32_t lr_h, int32_t lr_w, double scale, int32_t* out_h, int32_t* out_w);

/* Scale-vector form (R22): Hs = floor(s_y H), Ws = floor(s_x W) in fp64 (scale_y = 0: s_y =
 * s_x); only these two are checked against the limits. GSR_EINVAL on bad arguments. */
gsr_status gsr_out_dims_v(int32_t lr_h, int32_t lr_w, double scale_x, double scale_y,
                          int32_t* out_h, int32_t* out_w);

/* Device workspace needed by the forward or backward of one batched call (bytes, 256-aligned
 * internally). Returns 0 if the arguments are invalid. The same size serves both passes. */
size_t gsr_workspace_bytes_batched(const gsr_image* imgs, int32_t n_imgs, int64_t n_total,
                                   double ratio);
/* Single-image convenience: n Gaussians, whole image. */
size_t gsr_workspace_bytes(int64_t n, int32_t lr_h, int32_t lr_w, double scale, double ratio);

/* Forward render (Alg. 1 / Eq. 4) of one image: out[Hs][Ws][3] is overwritten with
 * I_SR(x,y;s) = sum over valid Gaussians i whose window contains pixel (x,y) of
 * alpha_i c_i f_i(x/s, y/s). n = 0 gives an all-zero image. */
gsr_status gsr_render_fwd(const float* alpha, const float* mu, const float* sigma,
                          const float* rho, const float* color, int64_t n, int32_t lr_h,
                          int32_t lr_w, double scale, double ratio, float* out, void* workspace,
                          size_t workspace_bytes, void* stream);

/* Backward of the forward above for L with dL/dI_SR = grad_out[Hs][Ws][3]: writes
 * (overwrites) d_alpha[n], d_mu[n][2], d_sigma[n][2], d_rho[n], d_color[n][3] (float32,
 * same layouts as the inputs; d_mu is also dL/d(offset o) since mu = p + o). */
gsr_status gsr_render_bwd(const float* alpha, const float* mu, const float* sigma,
                          const float* rho, const float* color, int64_t n, int32_t lr_h,
                          int32_t lr_w, double scale, double ratio, const float* grad_out,
                          float* d_alpha, float* d_mu, float* d_sigma, float* d_rho,
                          float* d_color, void* workspace, size_t workspace_bytes, void* stream);

/* Batched/ragged forward: every image of imgs[0..n_imgs) (host array, read during the call
 * only) is rendered into its block of `out`. Blocks must not overlap. */
gsr_status gsr_render_fwd_batched(const float* alpha, const float* mu, const float* sigma,
                                  const float* rho, const float* color, int64_t n_total,
                                  const gsr_image* imgs, int32_t n_imgs, double ratio, float* out,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* Batched backward: grads for all n_total Gaussians (Gaussians not owned by any image get 0). */
gsr_status gsr_render_bwd_batched(const float* alpha, const float* mu, const float* sigma,
                                  const float* rho, const float* color, int64_t n_total,
                                  const gsr_image* imgs, int32_t n_imgs, double ratio,
                                  const float* grad_out, float* d_alpha, float* d_mu,
                                  float* d_sigma, float* d_rho, float* d_color, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* Backward split in two for row-band sharding:
 * gsr_render_bwd_moments_batched ACCUMULATES (+=) into moments[n_total][8] (float64, caller
 * zeroes it first) the per-Gaussian pair sums over the pixels of each image's row band. With
 * u = dx/sx, v = dy/sy, (dx, dy) = (x/s - mu_x, y/s - mu_y), D = 1 - rho^2, k = log2(e)/2,
 * wq = sqrt(k/D) (u - rho v), vq = sqrt(k) v, e = exp(-Q/2) = 2^-(wq^2 + vq^2),
 * g = dL/dI at the pixel, c' = alpha c K, K = (2 pi sx sy sqrt(D))^-1, w = e (g . c'):
 *   m[0..2] = sum e g_k,  m[3] = sum w wq,  m[4] = sum w vq,
 *   m[5] = sum w wq^2,    m[6] = sum w wq vq,  m[7] = sum w vq^2.
 * Sums of moments over bands (e.g. an all-reduce across ranks) are moments of the union.
 * gsr_finalize_grads turns moments into the gradients (closed forms in DESIGN.md). */
gsr_status gsr_render_bwd_moments_batched(const float* alpha, const float* mu, const float* sigma,
                                          const float* rho, const float* color, int64_t n_total,
                                          const gsr_image* imgs, int32_t n_imgs, double ratio,
                                          const float* grad_out, double* moments, void* workspace,
                                          size_t workspace_bytes, void* stream);
gsr_status gsr_finalize_grads(const float* alpha, const float* mu, const float* sigma,
                              const float* rho, const float* color, int64_t n_total,
                              const double* moments, float* d_alpha, float* d_mu, float* d_sigma,
                              float* d_rho, float* d_color, void* stream);

/* Variants of the two backward entry points with flags.
 * GSR_REUSE_BINNING: the workspace still holds the binning (sorted keys, permutation, cell
 * starts, records) computed by the immediately preceding call on the SAME parameter arrays,
 * images and ratio (typically this step's forward), enqueued on the same stream; the binning
 * stage (K1, radix sort, K1b) is skipped. Results are undefined if that precondition is false. */
#define GSR_REUSE_BINNING 0x1u
/* Data formats ("AMP in bfloat16"). Accepted by the _ex entry points
 * below (the finalize and pair count take GSR_PARAMS_BF16 only); the arithmetic is unchanged
 * (fp32 evaluation, fp64 rects/finalize), only what is read and written changes:
 *   GSR_OUT_BF16    the image arrays -- the forward's `out`, the backward's `grad_out` -- hold
 *                   bfloat16 elements (the forward rounds its fp32 sums to nearest-even on store);
 *                   gsr_image.out_off and the block sizes count elements.
 *   GSR_OUT_CHW     the image blocks are planar: element (k, y, x) of image block b at
 *                   b.out_off + k*rows*Ws + (y - row_begin)*Ws + x, rows = row_end - row_begin
 *                   (default: HWC, b.out_off + ((y - row_begin)*Ws + x)*3 + k).
 *   GSR_PARAMS_BF16 the five parameter arrays are bfloat16 (same SoA layouts); they are widened
 *                   exactly to fp32 where read. Gradients are always written as float32.
 * The backward's flags must describe the same formats as the forward's when
 * GSR_REUSE_BINNING is set. The single-image and non-_ex entry points use float32 HWC. */
#define GSR_OUT_BF16 0x4u
#define GSR_OUT_CHW 0x8u
#define GSR_PARAMS_BF16 0x10u
gsr_status gsr_render_fwd_batched_ex(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     void* out, void* workspace, size_t workspace_bytes,
                                     uint32_t flags, void* stream);
gsr_status gsr_render_bwd_batched_ex(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     const void* grad_out, float* d_alpha, float* d_mu,
                                     float* d_sigma, float* d_rho, float* d_color,
                                     void* workspace, size_t workspace_bytes, uint32_t flags,
                                     void* stream);
gsr_status gsr_render_bwd_moments_batched_ex(const void* alpha, const void* mu,
                                             const void* sigma, const void* rho,
                                             const void* color, int64_t n_total,
                                             const gsr_image* imgs, int32_t n_imgs, double ratio,
                                             const void* grad_out, double* moments,
                                             void* workspace, size_t workspace_bytes,
                                             uint32_t flags, void* stream);
gsr_status gsr_finalize_grads_ex(const void* alpha, const void* mu, const void* sigma,
                                 const void* rho, const void* color, int64_t n_total,
                                 const double* moments, float* d_alpha, float* d_mu,
                                 float* d_sigma, float* d_rho, float* d_color, uint32_t flags,
                                 void* stream);

/* ---- subset mode: one rank's halo of a row-band shard ------------------------
 * A rank that renders HR rows [b_r, b_{r+1}) of an image needs only the Gaussians whose support
 * rows meet them (its halo, gsr_band_span_*). The _subset entry points take that list instead
 * of scanning all n_total Gaussians: idx[0..m) (device int32, ascending, each inside its image's
 * [g_off, g_off + g_cnt); m <= n_total) selects the Gaussians that are binned and rendered; the
 * parameter arrays and gsr_image ranges stay those of the whole batch (global indices). Every
 * per-Gaussian OUTPUT is compact: entry t belongs to Gaussian idx[t]:
 *   gsr_render_bwd_moments_subset accumulates (+=) moments[t][8] (float64, [m][8], caller
 *     zeroes), with the layout of gsr_render_bwd_moments_batched;
 *   gsr_finalize_grads_subset writes d_alpha[t], d_mu[t][2], d_sigma[t][2], d_rho[t],
 *     d_color[t][3] (float32, compact [m] arrays) from moments[t] (same closed forms as
 *     gsr_finalize_grads).
 * A Gaussian left out of idx contributes nothing to the images (exactly what the render does
 * for a Gaussian whose support misses the band, R21). Workspace: gsr_workspace_bytes_subset
 * (sized by m). Flags and errors as for the _ex entry points; GSR_REUSE_BINNING requires the
 * preceding call to have used the same idx. */
size_t gsr_workspace_bytes_subset(const gsr_image* imgs, int32_t n_imgs, int64_t n_total,
                                  int64_t m, double ratio);
gsr_status gsr_render_fwd_subset(const void* alpha, const void* mu, const void* sigma,
                                 const void* rho, const void* color, int64_t n_total,
                                 const int32_t* idx, int64_t m, const gsr_image* imgs,
                                 int32_t n_imgs, double ratio, void* out, void* workspace,
                                 size_t workspace_bytes, uint32_t flags, void* stream);
gsr_status gsr_render_bwd_moments_subset(const void* alpha, const void* mu, const void* sigma,
                                         const void* rho, const void* color, int64_t n_total,
                                         const int32_t* idx, int64_t m, const gsr_image* imgs,
                                         int32_t n_imgs, double ratio, const void* grad_out,
                                         double* moments, void* workspace,
                                         size_t workspace_bytes, uint32_t flags, void* stream);
gsr_status gsr_finalize_grads_subset(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const int32_t* idx, int64_t m, const double* moments,
                                     float* d_alpha, float* d_mu, float* d_sigma, float* d_rho,
                                     float* d_color, uint32_t flags, void* stream);

/* ---- training-step adjacency ------------------------------------------
 * One fused training step of the rasterizer for the paper's L1 objective, from the RAW
 * outputs of the Gaussian Primary Head:
 *   alpha = sigmoid(raw_alpha), c = sigmoid(raw_color), sigma = sigmoid(raw_sigma),
 *   rho = rho_scale * tanh(raw_rho)  (paper: rho_scale = 1; SPEC's rho_eps: 1 - 1e-4),
 *   mu = ref + offset               (reference position p + predicted offset o)
 * then the forward render (as gsr_render_fwd_batched, written to `out`), the loss
 *   *loss = inv_numel * sum |out - gt|   (float64 device scalar, overwritten; gt has out's layout)
 * and the gradients of *loss with respect to every raw input (float32, input layouts,
 * overwritten; d_offset is also dL/d mu). The L1 subgradient is sign(out - gt) (0 at ties).
 * inv_numel <= 0 means 1 / (number of output elements of this call); pass the global value when
 * the batch is sharded. All arrays are device pointers; workspace from
 * gsr_train_workspace_bytes_batched. Errors as for the render entry points. */
size_t gsr_train_workspace_bytes_batched(const gsr_image* imgs, int32_t n_imgs, int64_t n_total,
                                         double ratio);
gsr_status gsr_train_step_l1_batched(const float* raw_alpha, const float* offset, const float* ref,
                                     const float* raw_sigma, const float* raw_rho,
                                     const float* raw_color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     float rho_scale, double inv_numel, const float* gt,
                                     float* out, double* loss, float* d_raw_alpha,
                                     float* d_offset, float* d_raw_sigma, float* d_raw_rho,
                                     float* d_raw_color, void* workspace, size_t workspace_bytes,
                                     void* stream);

/* Evaluation support (reading R21): a pair with Q >= 13.5^2 has exp(-Q/2) < 2^-131,
 * exactly 0 in the kernels' fp32 (flush-to-zero) exp, and every pixel outside the box
 * |x/s - mu_x| <= 13.5 sigma_x, |y/s - mu_y| <= 13.5 sigma_y is such a pair. The render kernels
 * evaluate each Gaussian over its SUPPORT RECT = window rect (R2) intersected with the integer box
 * [floor(s (mu - 13.5 sigma)), ceil(s (mu + 13.5 sigma))] (fp64, per axis); the results equal
 * those of an evaluation over the whole window. GSR_SUPPORT selects the support rect in the
 * introspection / counting calls below (default: the window rect of Alg. 1). */
#define GSR_SUPPORT 0x2u

/* Number of (Gaussian, pixel) pairs inside the windows, P = sum_i |rect_i| restricted to each
 * image's row band (the paper's work unit). Writes one int64 to *d_pairs (device
 * pointer). Uses the workspace. The _ex form with GSR_SUPPORT counts the pairs inside the
 * support rects instead (the pairs the kernels evaluate; the roofline's work unit); it also
 * accepts GSR_PARAMS_BF16. Other flag bits: GSR_EINVAL. */
gsr_status gsr_pair_count_batched(const float* alpha, const float* mu, const float* sigma,
                                  const float* rho, const float* color, int64_t n_total,
                                  const gsr_image* imgs, int32_t n_imgs, double ratio,
                                  int64_t* d_pairs, void* workspace, size_t workspace_bytes,
                                  void* stream);
gsr_status gsr_pair_count_batched_ex(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     uint32_t flags, int64_t* d_pairs, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* ---- K7: row-band planning for the multi-GPU path ---------------------------
 * The row-band shard gives rank r the HR rows [b_r, b_{r+1}) of every image; the boundaries
 * equalise the work (pairs) per rank, and the Gaussians whose support rows (R21) span a boundary
 * ("seam" Gaussians) have partial gradients on several ranks. Both need Alg. 1's window rect
 * (readings R1/R2) and the support box (R21) per Gaussian; these entry points compute
 * them with the render kernels' own code. Each comes as a device variant (params and outputs are
 * device pointers, enqueued on `stream`) and a host variant (_host: params and outputs are HOST
 * pointers, computed on the calling CPU thread, no CUDA call; the same arithmetic).
 *
 * gsr_row_pair_counts_*: rowpairs[roff_k + (y - row_begin_k)] for y in image k's band
 *   [row_begin_k, row_end_k), roff_k = sum_{j<k} (row_end_j - row_begin_j): the number of pairs
 *   of HR row y, sum_i [y0_i <= y <= y1_i] (x1_i - x0_i + 1) over the valid Gaussians of the
 *   image, with the window rect (flags 0; sums to gsr_pair_count_batched) or the support rect
 *   (GSR_SUPPORT; the pairs the kernels evaluate). int64, overwritten. Flags: GSR_SUPPORT,
 *   GSR_PARAMS_BF16.
 * gsr_band_span_*: bounds[k*(n_bands+1) + g] (HOST array, n_imgs x (n_bands+1), nondecreasing,
 *   inside image k's band) are the band boundaries of image k, 1 <= n_bands <= 64. For every
 *   Gaussian i: span[2i] = first and span[2i+1] = last band g whose rows [b_g, b_{g+1}) meet its
 *   clipped support rows widened by `margin` >= 0 rows ([y0 - margin, y1 + margin]); {-1, -1} if
 *   it is invalid (R20), not owned by an image, or its support rect is empty. Seam Gaussian:
 *   first < last. Halo of band r: first <= r <= last. int16, overwritten. Flags:
 *   GSR_PARAMS_BF16. */
gsr_status gsr_row_pair_counts_batched(const void* alpha, const void* mu, const void* sigma,
                                       const void* rho, const void* color, int64_t n_total,
                                       const gsr_image* imgs, int32_t n_imgs, double ratio,
                                       uint32_t flags, int64_t* rowpairs, void* stream);
gsr_status gsr_row_pair_counts_host(const void* alpha, const void* mu, const void* sigma,
                                    const void* rho, const void* color, int64_t n_total,
                                    const gsr_image* imgs, int32_t n_imgs, double ratio,
                                    uint32_t flags, int64_t* rowpairs);
gsr_status gsr_band_span_batched(const void* alpha, const void* mu, const void* sigma,
                                 const void* rho, const void* color, int64_t n_total,
                                 const gsr_image* imgs, int32_t n_imgs, double ratio,
                                 uint32_t flags, const int32_t* bounds, int32_t n_bands,
                                 int32_t margin, int16_t* span, void* stream);
gsr_status gsr_band_span_host(const void* alpha, const void* mu, const void* sigma,
                              const void* rho, const void* color, int64_t n_total,
                              const gsr_image* imgs, int32_t n_imgs, double ratio,
                              uint32_t flags, const int32_t* bounds, int32_t n_bands,
                              int32_t margin, int16_t* span);
/* gsr_rank_halo: rank `rank`'s share of the shard in one fused pass (the band spans above are
 * computed on the fly, nothing of size n is materialised but a byte per Gaussian of workspace):
 *   idx[0..m)        ascending indices of its halo (first <= rank <= last): the idx of the
 *                    gsr_*_subset calls;
 *   up[0..nu)        positions in idx of the Gaussians whose span is exactly [rank, rank+1] --
 *                    the seam rows swapped with rank + 1 (ascending Gaussian order, so both
 *                    neighbours list the same Gaussians in the same order);
 *   down[0..nd)      likewise [rank-1, rank], swapped with rank - 1;
 *   multi_pos/multi_slot[0..nm)  Gaussians of the halo spanning >= 3 bands: position in idx and
 *                    slot in the global list of all nM such Gaussians (every rank all-reduces a
 *                    [nM] buffer);
 *   totals[5]        {m, nu, nd, nm, nM} (device int64).
 * All output arrays are device int32 with capacity n_total; results are written asynchronously
 * on `stream`. Workspace: gsr_rank_halo_workspace_bytes(n_total). Bounds, n_bands and margin as
 * for gsr_band_span_*; 0 <= rank < n_bands. Flags: GSR_PARAMS_BF16. */
size_t gsr_rank_halo_workspace_bytes(int64_t n_total);
gsr_status gsr_rank_halo(const void* alpha, const void* mu, const void* sigma, const void* rho,
                         const void* color, int64_t n_total, const gsr_image* imgs,
                         int32_t n_imgs, double ratio, uint32_t flags, const int32_t* bounds,
                         int32_t n_bands, int32_t margin, int32_t rank, int32_t* idx,
                         int32_t* up, int32_t* down, int32_t* multi_pos, int32_t* multi_slot,
                         int64_t* totals, void* workspace, size_t workspace_bytes,
                         void* stream);

/* Parameter-domain check (R20): writes result[0] = number of Gaussians outside the
 * domain (a non-finite field, sigma_x <= 0, sigma_y <= 0 or |rho| >= 1) and result[1] = the
 * smallest such index (INT64 -1 = 0xffff...ffff when there is none); result is a DEVICE int64[2],
 * written asynchronously on `stream` (read it after a sync). Such Gaussians are not an error for
 * the render entry points (they contribute 0 and get zero gradient); this is the debugging aid
 * that reports them. Flags: GSR_PARAMS_BF16. */
gsr_status gsr_validate_params(const void* alpha, const void* mu, const void* sigma,
                               const void* rho, const void* color, int64_t n, uint32_t flags,
                               int64_t* result, void* stream);

/* ---- introspection for the parity tests (same kernels as the render path) ---------------- */

/* Per-Gaussian integer window rect as computed on the GPU (reading R2), clipped to the image:
 * rects[i] = {x0, x1, y0, y1}; an empty/invalid rect is {1, 0, 1, 0}. Single image. */
gsr_status gsr_debug_rects(const float* alpha, const float* mu, const float* sigma,
                           const float* rho, const float* color, int64_t n, int32_t lr_h,
                           int32_t lr_w, double scale, double ratio, int32_t* rects, void* stream);
/* The same with flags: GSR_SUPPORT returns the support rects (R21) the kernels evaluate. */
gsr_status gsr_debug_rects_ex(const float* alpha, const float* mu, const float* sigma,
                              const float* rho, const float* color, int64_t n, int32_t lr_h,
                              int32_t lr_w, double scale, double ratio, uint32_t flags,
                              int32_t* rects, void* stream);

/* Tile binning, materialised: for every backward render tile of the single image (tiles of
 * tile_w x tile_h HR px in row-major tile order, as reported by gsr_tile_shape), the exact list of
 * Gaussians whose support rect (R21) intersects the tile, in the order the backward kernel visits
 * them (cell order, ascending index within a cell). Two calls: first with ids == NULL to fill
 * counts[ntiles] (device int32); then with ids (device int32, sum(counts) entries, CSR by tile)
 * and cells (device int32, same length, the sort key = cell of each entry). */
gsr_status gsr_debug_tile_lists(const float* alpha, const float* mu, const float* sigma,
                                const float* rho, const float* color, int64_t n, int32_t lr_h,
                                int32_t lr_w, double scale, double ratio, int32_t* counts,
                                int32_t* ids, int32_t* cells, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Forward tile lists, materialised (test-only): for every forward render tile of the single
 * image (K4's tiles: ftile_w x ftile_h HR px in row-major order; the tile configuration is chosen
 * per call from the window width), the Gaussians K4 keeps -- its candidate stream (the tile's
 * cell rows, each trimmed by the cell reach on dense images) filtered by its support-rect test
 * (R21), in stream order -- and the evaluation path K4 assigns each (render_fwd.cu P_*). The
 * same device code as K4 (CandStream, fwd_classify). geom: host int32[3] <- {ftile_w, ftile_h,
 * number of forward tiles}. Two calls: offsets == NULL fills counts[ntiles] (device int32);
 * then offsets (device int32, exclusive prefix of counts) with ids (device int32, Gaussian
 * indices) and paths (device uint8), sum(counts) entries each, CSR by tile. */
gsr_status gsr_debug_fwd_tile_lists(const float* alpha, const float* mu, const float* sigma,
                                    const float* rho, const float* color, int64_t n,
                                    int32_t lr_h, int32_t lr_w, double scale, double ratio,
                                    int32_t* geom, const int32_t* offsets, int32_t* counts,
                                    int32_t* ids, uint8_t* paths, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* ---- measurement ------------------------------------------------------------------------ */

/* Phase timing for benchmarks (process-global, not thread-safe; off by default). While enabled,
 * every compute call records a pair of CUDA events on its stream around each phase:
 *   0 = binning (K1 keys + stable radix sort + cell starts + K1b records),
 *   1 = forward render kernel (K4), 2 = backward pair pass (K5), 3 = finalize (K6).
 * gsr_profile_collect synchronises the recorded events, returns the accumulated milliseconds
 * ms[4] and call counts calls[4] since the last reset, and the number of kernels libgsr
 * launched (*kernel_launches, counted whether or not profiling is enabled). reset != 0 clears
 * them. Any argument may be NULL. */
gsr_status gsr_profile_enable(int32_t on);
gsr_status gsr_profile_collect(double* ms, int64_t* calls, int64_t* kernel_launches,
                               int32_t reset);

/* Render-tile and cell geometry used by the kernels (compile-time constants). */
void gsr_tile_shape(int32_t* tile_w, int32_t* tile_h, int32_t* cell_w, int32_t* cell_h);

#ifdef __cplusplus
}
#endif

#endif /* GSR_H */
