// gsr_internal.cuh -- shared definitions of the sm_100a kernels behind include/gsr.h.
//
// Data layout in HBM:
//   params      float32 SoA from the caller (alpha, mu, sigma, rho, color), read by K1/K1b/K6.
//   keys/vals   uint32 cell key + int32 Gaussian index, radix-sorted (stable) -> perm.
//   cell_start  int32[total_cells+1]: first sorted position of each cell (CSR over cells).
//   rec         3 x float4 per sorted position (48 B record, see Rec below).
//   moments     float64[n][8], original Gaussian order (backward only).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

// GSR_BOUNDS_CHECK builds (tests only, tools/gpu_calls/gpu_r02_ci.sh): device asserts on the
// indices the kernels derive (compute-sanitizer is not available on the GPU pool); no-ops in the
// shipped build
#ifdef GSR_BOUNDS_CHECK
#include <cassert>
#define GSR_CHECK(c) assert(c)
#else
#define GSR_CHECK(c) ((void)0)
#endif

namespace gsr {

// ---- compile-time geometry -------------------------------------------------------------
constexpr int CELL = 16;       // cell edge (HR px): binning granularity (sort key)
#ifndef GSR_BWD_TILE_W
#define GSR_BWD_TILE_W 64
#endif
#ifndef GSR_BWD_TILE_H
#define GSR_BWD_TILE_H 8
#endif
constexpr int TILE_W = GSR_BWD_TILE_W;  // backward render tile (HR px, power of 2 >= 16);
constexpr int TILE_H = GSR_BWD_TILE_H;  // also the debug tile-list tile (TILE_H even)
// forward: a CTA renders one tile; each of its warps covers the whole tile (lane l owns a
// ROWS x STRIP block at column group l & 3, row group l >> 2) and takes its own share of the
// tile's Gaussians, so the warps' work is balanced by construction. Two configurations, chosen
// per call from the window size:
//   large (windows >= FWD_SMALL_WINDOW HR px): 2 x 8 px per lane -> 32 x 16 tiles
//   small (narrow windows, e.g. the x1..x4 training patches): 1 x 4 px per lane -> 16 x 8 tiles,
//         which wastes far fewer masked evaluations where a window covers only part of a tile
//         (GSR_FWD_SMALL_STRIP=8: 1 x 8 px per lane, 32 x 8 tiles evaluated per 16 x 8 column half;
//         measured 7% slower at C2)
// warps per forward CTA (each covers the whole tile for its share of the Gaussians): 2 for the
// large tiles (4 measured +2% at C5), 4 for the small ones (2: +35% at C2)
#ifndef GSR_FWD_WARPS_LARGE
#define GSR_FWD_WARPS_LARGE 2
#endif
#ifndef GSR_FWD_WARPS_SMALL
#define GSR_FWD_WARPS_SMALL 4
#endif
struct FwdCfgLarge { static constexpr int ROWS = 2, STRIP = 8, TW = 4 * STRIP, TH = 8 * ROWS, WARPS = GSR_FWD_WARPS_LARGE; };
#ifndef GSR_FWD_SMALL_STRIP
#define GSR_FWD_SMALL_STRIP 4
#endif
struct FwdCfgSmall { static constexpr int ROWS = 1, STRIP = GSR_FWD_SMALL_STRIP, TW = 4 * STRIP, TH = 8 * ROWS, WARPS = GSR_FWD_WARPS_SMALL; };
using FwdCfgWide = FwdCfgLarge;
constexpr int FWD_SMALL_WINDOW = 48;             // HR px: below this the small tiles are used
#ifndef GSR_FWD_REC
#define GSR_FWD_REC 1
#endif
constexpr float FWD_REC_DMAX = GSR_FWD_REC ? 1.0f : -1.0f;            // max a1/s for the forward's exp recurrence

#ifndef GSR_BWD_WARPS
#define GSR_BWD_WARPS 4
#endif
constexpr int BWD_WARPS = GSR_BWD_WARPS;
constexpr int BWD_THREADS = BWD_WARPS * 32;
constexpr int MAX_IMAGES = 64;
constexpr uint32_t KEY_SENTINEL_FLAG = 0xffffffffu;

// log2(e)/2: exp(-Q/2) = 2^(-HALF_LOG2E * Q)
constexpr double HALF_LOG2E = 0.72134752044448170368;
constexpr double TWO_PI = 6.28318530717958647693;

// Per-image constants, computed on the host in fp64, passed by value in ImgTable.
struct DevImg {
    double sx, sy;      // scale vector (R22): sx along x <-> W, sy along y <-> H (paper: sx = sy = s)
    double hx, hy;      // window half-extents r*W, r*H (LR px, fp64)
    long long g_off, g_cnt, out_off;
    float invsx, invsy; // fp32(1/sx), fp32(1/sy)
    int H, W, Hs, Ws;
    int row_begin, row_end;   // HR row band
    int offx, offy;           // cell-grid offsets (multiples of CELL, >= max rect extent)
    int ncx, ncy, cell_base;  // cells of this image: [cell_base, cell_base + ncx*ncy)
    int ntx, nty, tile_base;  // backward tiles (TILE_W x TILE_H) of this image
    int fntx, fnty, ftile_base;  // forward tiles (ImgTable::ftile_w x ftile_h)
    int stile_base, sftile_base;  // first backward / forward CTA tile in launch order (schedule)
    int wmax, hmax;           // upper bounds on the unclipped rect width/height
    int io;                   // image I/O format of out / grad_out (IO_BF16 | IO_CHW; 0 = fp32 HWC)
    int dense;                // >= 16 Gaussians per 16 x 16-px cell of the image (cell-reach trim)
};

constexpr int IO_BF16 = 1;    // GSR_OUT_BF16: image elements are bfloat16 (RNE on store)
constexpr int IO_CHW = 2;     // GSR_OUT_CHW: planar blocks, element (k, y, x) at k*rows*Ws + (y-rb)*Ws + x

struct ImgTable {
    int n_imgs;
    int total_cells;          // key of an unbinned Gaussian (sorts last)
    int total_tiles;          // backward tiles
    int total_ftiles;         // forward tiles
    int ftile_w, ftile_h;     // forward tile of this call (large or small configuration)
    int fwd_small;            // 1: FwdCfgSmall
    int params_bf16;          // GSR_PARAMS_BF16: the five parameter arrays are bfloat16
    // launch order of the images' tiles: densest images (most Gaussians per HR pixel, the
    // heaviest tiles) first, so the tail of the grid holds the light tiles
    int sched[MAX_IMAGES];
    DevImg img[MAX_IMAGES];
};

// K7 band planning (plan.cu): per-image row offsets of a row-count array, and band boundaries
constexpr int MAX_BANDS = 64;
struct RowOff { long long off[MAX_IMAGES + 1]; };
struct BandTable { int G, margin; int b[MAX_IMAGES][MAX_BANDS + 1]; };

// Sorted record (64 B = REC_F4 x float4), one per binned Gaussian, in cell order, in the form
// the render kernels consume (K1b, binning.cu):
//   r0 = {-ax, ay, dl_y, D}         anchor a = rint(s mu) (integer HR px, as float), fp32
//                                  residual dl = mu - a/s (LR px), D = a1/s (fp32 product)
//   r1 = {-a1 dl_x, b1, c1, c'_r}   factored exponent: q = -Q/2 log2 e = -(w^2 + v^2),
//                                  w = a1 dx + b1 dy, v = c1 dy; c' = alpha c K
//   r2 = {c'_g, c'_b, x0|x1<<16, y0|y1<<16}  clipped WINDOW rect (R2): the masks
//   r3 = {G1, G2, G3, rec}         G_t = 2^(-D^2 t^2) and rec = 1 if D <= FWD_REC_DMAX (forward
//                                  exponential recurrence), else all 0
// plus the class byte cls[p] (bit 0 = r3.w != 0: recurrence allowed), read by the forward's
// filter so that a Gaussian's evaluation path is decided before its record is loaded,
// plus the rect stream rects[p] = {support x0|x1<<16, support y0|y1<<16, window x, window y}:
// the support rect (R21) for tile filtering and loop bounds (pairs outside it are exactly 0
// in fp32), read by the forward producer and the backward scan without touching the records.
constexpr int REC_F4 = 4;

__host__ __device__ inline int find_image_by_tile(const ImgTable& t, int tile) {
    int lo = 0, hi = t.n_imgs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (t.img[mid].tile_base <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__host__ __device__ inline int find_image_by_ftile(const ImgTable& t, int tile) {
    int lo = 0, hi = t.n_imgs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (t.img[mid].ftile_base <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// image owning the render kernels' CTA tile `tile` (launch order, ImgTable::sched)
__host__ __device__ inline int find_image_by_stile(const ImgTable& t, int tile) {
    int lo = 0, hi = t.n_imgs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (t.img[t.sched[mid]].stile_base <= tile) lo = mid; else hi = mid - 1;
    }
    return t.sched[lo];
}
__host__ __device__ inline int find_image_by_sftile(const ImgTable& t, int tile) {
    int lo = 0, hi = t.n_imgs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (t.img[t.sched[mid]].sftile_base <= tile) lo = mid; else hi = mid - 1;
    }
    return t.sched[lo];
}

__host__ __device__ inline int find_image_by_gauss(const ImgTable& t, long long i) {
    // images sorted by g_off; returns -1 if i is not owned by any image
    int lo = 0, hi = t.n_imgs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (t.img[mid].g_off <= i) lo = mid; else hi = mid - 1;
    }
    if (t.n_imgs == 0) return -1;
    const DevImg& im = t.img[lo];
    if (i < im.g_off || i >= im.g_off + im.g_cnt) return -1;
    return lo;
}

// ---- the normative window rect (reading R2), fp64, fixed op order, no FMA ---------------
// Host and device share this code (the host planner K7 of plan.cu runs it on CPU arrays too):
// on the device the products/sums are the explicit round-to-nearest intrinsics (never fused);
// the host compiler gets -ffp-contract=off (build.py), so a*b and a-b are single IEEE ops there.
struct Rect { int x0u, y0u, x1u, y1u, x0, x1, y0, y1; bool nonempty; };

__host__ __device__ __forceinline__ double rn_mul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
__host__ __device__ __forceinline__ double rn_add(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
__host__ __device__ __forceinline__ double rn_sub(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}

__host__ __device__ __forceinline__ double clamp_bound(double v) {
    const double lim = 1073741824.0;  // 2^30
    return v < -lim ? -lim : (v > lim ? lim : v);
}

__host__ __device__ __forceinline__ Rect window_rect(float mux, float muy, const DevImg& im) {
    Rect r;
    double mx = (double)mux, my = (double)muy;
    double lx = rn_mul(im.sx, rn_sub(mx, im.hx));
    double ux = rn_mul(im.sx, rn_add(mx, im.hx));
    double ly = rn_mul(im.sy, rn_sub(my, im.hy));
    double uy = rn_mul(im.sy, rn_add(my, im.hy));
    long long ax0 = (long long)floor(clamp_bound(lx)) + 1;
    long long ax1 = (long long)ceil(clamp_bound(ux)) - 1;
    long long ay0 = (long long)floor(clamp_bound(ly)) + 1;
    long long ay1 = (long long)ceil(clamp_bound(uy)) - 1;
    r.x0u = (int)ax0;
    r.y0u = (int)ay0;
    r.x1u = (int)ax1;
    r.y1u = (int)ay1;
    long long cx0 = ax0 < 0 ? 0 : ax0;
    long long cx1 = ax1 > im.Ws - 1 ? im.Ws - 1 : ax1;
    long long cy0 = ay0 < im.row_begin ? im.row_begin : ay0;          // band clip
    long long cy1 = ay1 > im.row_end - 1 ? im.row_end - 1 : ay1;
    r.x0 = (int)cx0; r.x1 = (int)cx1; r.y0 = (int)cy0; r.y1 = (int)cy1;
    r.nonempty = (cx0 <= cx1) && (cy0 <= cy1) && !isnan(lx) && !isnan(ux) && !isnan(ly) &&
                 !isnan(uy);
    return r;
}

// Reading R21: the evaluation support. A pair with Q >= 13.5^2 has
// exp(-Q/2) = 2^(-kappa Q) < 2^-131, below the smallest fp32 normal: the kernels' ex2.approx.ftz
// returns exactly 0 for it, so it adds nothing to any sum. Q >= (dx/sx)^2 and Q >= (dy/sy)^2 for
// every rho, hence every pixel outside the box |x/s - mu_x| <= 13.5 sx, |y/s - mu_y| <= 13.5 sy
// is such a pair. The kernels evaluate the window rect (R2) intersected with the integer box
//   bx0 = floor(s (mu_x - 13.5 sx)),  bx1 = ceil(s (mu_x + 13.5 sx))   (fp64, this order)
// and produce the same fp32 results as an evaluation of the whole window.
constexpr double SUPPORT_SIGMAS = 13.5;

__host__ __device__ __forceinline__ Rect support_rect(float mux, float muy, float sxf, float syf,
                                                      const DevImg& im) {
    Rect r = window_rect(mux, muy, im);
    const double mx = (double)mux, my = (double)muy;
    const double tx = rn_mul(SUPPORT_SIGMAS, (double)sxf);
    const double ty = rn_mul(SUPPORT_SIGMAS, (double)syf);
    const double lx = rn_mul(im.sx, rn_sub(mx, tx));
    const double ux = rn_mul(im.sx, rn_add(mx, tx));
    const double ly = rn_mul(im.sy, rn_sub(my, ty));
    const double uy = rn_mul(im.sy, rn_add(my, ty));
    const int bx0 = (int)floor(clamp_bound(lx)), bx1 = (int)ceil(clamp_bound(ux));
    const int by0 = (int)floor(clamp_bound(ly)), by1 = (int)ceil(clamp_bound(uy));
    r.x0u = r.x0u > bx0 ? r.x0u : bx0;
    r.y0u = r.y0u > by0 ? r.y0u : by0;
    r.x1u = r.x1u < bx1 ? r.x1u : bx1;
    r.y1u = r.y1u < by1 ? r.y1u : by1;
    r.x0 = r.x0 > bx0 ? r.x0 : bx0;
    r.x1 = r.x1 < bx1 ? r.x1 : bx1;
    r.y0 = r.y0 > by0 ? r.y0 : by0;
    r.y1 = r.y1 < by1 ? r.y1 : by1;
    r.nonempty = r.nonempty && r.x0 <= r.x1 && r.y0 <= r.y1 && !isnan(lx) && !isnan(ux) &&
                 !isnan(ly) && !isnan(uy);
    return r;
}

// parameter element -> float (GSR_PARAMS_BF16: bfloat16 widened exactly)
__host__ __device__ __forceinline__ float ldf(float v) { return v; }
__host__ __device__ __forceinline__ float ldf(__nv_bfloat16 v) { return __bfloat162float(v); }

// ---- image I/O formats (NEXT-4): index and element access of out / grad_out ----------------
__device__ __forceinline__ long long img_index(const DevImg& im, int y, int x, int k) {
    const long long r = y - im.row_begin;
    return (im.io & IO_CHW) ? im.out_off + (long long)k * (im.row_end - im.row_begin) * im.Ws +
                                  r * im.Ws + x
                            : im.out_off + (r * im.Ws + x) * 3 + k;
}
__device__ __forceinline__ void img_store(void* out, const DevImg& im, long long off, float v) {
    if (im.io & IO_BF16) ((__nv_bfloat16*)out)[off] = __float2bfloat16_rn(v);
    else ((float*)out)[off] = v;
}
__device__ __forceinline__ float img_load(const void* p, const DevImg& im, long long off) {
    return (im.io & IO_BF16) ? __bfloat162float(((const __nv_bfloat16*)p)[off])
                             : ((const float*)p)[off];
}

__host__ __device__ __forceinline__ bool gaussian_valid(float a, float mx, float my, float sx, float sy,
                                               float rh, float cr, float cg, float cb) {
    bool fin = isfinite(a) && isfinite(mx) && isfinite(my) && isfinite(sx) && isfinite(sy) &&
               isfinite(rh) && isfinite(cr) && isfinite(cg) && isfinite(cb);
    return fin && sx > 0.f && sy > 0.f && fabsf(rh) < 1.f;
}

// validity (R20) of Gaussian i read from the parameter arrays (float32 or bfloat16)
template <class T>
__host__ __device__ __forceinline__ bool valid_at(const T* alpha, const T* mu, const T* sigma,
                                         const T* rho, const T* color, long long i) {
    return gaussian_valid(ldf(alpha[i]), ldf(mu[2 * i]), ldf(mu[2 * i + 1]), ldf(sigma[2 * i]),
                          ldf(sigma[2 * i + 1]), ldf(rho[i]), ldf(color[3 * i]),
                          ldf(color[3 * i + 1]), ldf(color[3 * i + 2]));
}

// ---- PTX helpers ------------------------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// adds `bytes` to the barrier's expected transaction count without arriving
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    // suspend-time hint (ns): the thread sleeps in hardware until the phase completes instead of
    // spinning and stealing issue slots from the compute warps of its SM sub-partition
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}

// non-blocking probe of a phase (no suspend)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 16-B asynchronous copy global (L2) -> shared, per thread; completion by commit/wait groups
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// split-K factor for small problems: keep >= ~4 CTAs per SM (148 SMs); 1, 2, 4 or 8
// Split factor KS in {1, 2, 4, 8} of a tile grid over `slots` co-resident CTAs (SMs x CTAs per
// SM): below 4 waves, minimises the wave-quantised time ceil(tiles KS / slots) (1/KS + o), o = a
// CTA's fixed cost relative to a whole tile's work, so that the last wave is not mostly idle
// (C2's backward: 656 tiles on 592 slots -> KS = 4, 0.77 -> 0.62 ms).
#ifndef GSR_SPLIT_OVERHEAD
#define GSR_SPLIT_OVERHEAD 0.05
#endif
inline int split_k_factor(long long tiles, long long slots) {
    if (slots <= 0) slots = 4 * 148;
    // >= 4 waves: the tail is small and the split's per-CTA costs (tile staging, shorter
    // sorted batches, the forward's DSMEM reduce) measured +11-12% at C3/C4
    if (tiles >= 4 * slots) return 1;
    int best = 1;
    double tbest = 1e300;
    for (int ks = 1; ks <= 8; ks *= 2) {
        const double waves = (double)((tiles * ks + slots - 1) / slots);
        const double t = waves * (1.0 / ks + GSR_SPLIT_OVERHEAD);
        if (t < tbest * (1.0 - 1e-9)) { tbest = t; best = ks; }
    }
    return best;
}
// co-resident CTAs of a kernel on this device (occupancy x SM count), cached by the caller
template <class K>
inline int resident_slots(K kernel, int threads, size_t smem) {
    int dev = 0, sms = 148, per = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess ||
        per <= 0)
        per = 4;
    return per * sms;
}

// ---- host-side launch accounting (gsr_profile_*) --------------------------------------------
void count_launches(long long k);          // kernels launched by libgsr (all phases)
int prof_begin(int phase, cudaStream_t st);  // returns a handle (-1 when profiling is off)
void prof_end(int handle, cudaStream_t st);

// ---- host-side launchers (defined in the .cu files) --------------------------------------
struct Workspace {
    uint32_t* keys_a; uint32_t* keys_b;
    int* vals_a; int* vals_b;
    int* hist;               // radix histograms [256 * nblocks]
    int* scan_tmp;           // block sums for the scan
    int* cell_start;         // [total_cells + 1]
    float4* rec;             // [REC_F4 * n] records (sorted order)
    int4* rects;             // [n] {support x, support y, window x, window y} (sorted order)
    uint8_t* cls;            // [n] record class bits (sorted order): bit 0 = forward recurrence ok
    double* moments;         // [8 * n] (backward)
    unsigned long long* counter;  // scratch counters
    int* tile_off;           // debug tile lists: [total_tiles + 1]
    int* ext;                // [2 * MAX_IMAGES]: per image max unclipped support-rect width,
                             // height over the binned Gaussians (tile candidate query, K1)
    int2* reach;             // [total_cells]: per cell the largest clipped support-rect right
                             // and bottom edge of its Gaussians ({-1, -1}: empty cell; K1b)
};

// Trims one cell row [cx_lo, cx_hi] of a tile's candidate query to the cells whose reach
// (Workspace::reach) meets the tile's first column X0 and row Y0: the cells outside
// [lo, hi] hold no Gaussian whose support rect reaches the tile, so only candidates the exact
// rect test would reject are skipped. Warp-collective (every lane, uniform arguments); returns
// false when no cell of the row can reach the tile.
__device__ __forceinline__ bool reach_trim(const int2* __restrict__ reach, int row, int cx_lo,
                                           int cx_hi, int X0, int Y0, int lane, int* lo,
                                           int* hi) {
    auto ok = [&](int c) {
        const int2 r = __ldg(reach + row + c);
        return r.x >= X0 && r.y >= Y0;
    };
    if (cx_hi - cx_lo < 32) {                                 // one load per lane
        const int c = cx_lo + lane;
        const unsigned m = __ballot_sync(0xffffffffu, c <= cx_hi && ok(c));
        if (m == 0u) return false;
        *lo = cx_lo + __ffs(m) - 1;
        *hi = cx_lo + 31 - __clz(m);
        return true;
    }
    int l = -1;
    for (int c0 = cx_lo; c0 <= cx_hi && l < 0; c0 += 32) {
        const unsigned m = __ballot_sync(0xffffffffu, c0 + lane <= cx_hi && ok(c0 + lane));
        if (m) l = c0 + __ffs(m) - 1;
    }
    if (l < 0) return false;
    int h = l;
    for (int c0 = cx_hi; c0 > l; c0 -= 32) {
        const unsigned m = __ballot_sync(0xffffffffu, c0 - lane > l && ok(c0 - lane));
        if (m) { h = c0 - (__ffs(m) - 1); break; }
    }
    *lo = l;
    *hi = h;
    return true;
}

// Candidate stream of a forward tile: the cell-row spans of up to 32 rows at a time (a chunk),
// each trimmed to the cells whose reach meets the tile (GSR_CELL_REACH), concatenated into one
// sequence of positions, so the kernel walks it in full batches of 32 across row ends (the
// backward's scan on the same stream measured +1.6% at C5). Warp 0 builds the chunk table (row starts + exclusive prefix of the row
// lengths) in shared memory for the CTA; every warp walks the same chunk sequence.
#ifndef GSR_CELL_REACH
#define GSR_CELL_REACH 1          // trim the tiles' cell rows by the cell reach (A/B)
#endif
struct CandChunk {
    int pre[33];             // exclusive prefix of the rows' lengths; pre[32] = total
    int st[32];              // first record of each row
    int cy_next;             // first cell row after the chunk
};
struct CandStream {
    int cy_hi, row0, row_stride, cx_lo, cx_hi, X0, Y0;
    bool trim;               // trim the rows by the cell reach (dense images, >= 6 cells per row:
                             // elsewhere the reach loads' latency at tile start cost more than
                             // the trim saved -- C2 +4%, C4 +2%; C5 -4%)
    const int* cs;
    const int2* reach;
    // warp 0: the chunk from cell row cy on with at least one candidate (or none left: total 0)
    __device__ __noinline__ void build(CandChunk& ch, int cy, int lane) const {
        while (true) {
            const int nrows = cy <= cy_hi ? min(32, cy_hi - cy + 1) : 0;
            int mylo = 0, myhi = -1;
            if (!GSR_CELL_REACH || !trim) {
                mylo = cx_lo;
                myhi = cx_hi;
            } else if (cx_hi - cx_lo < 32) {
                for (int i0 = 0; i0 < nrows; i0 += 4) {      // 4 rows' reach loads in flight
                    bool okv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int c = cx_lo + lane;
                        okv[u] = false;
                        if (i0 + u < nrows && c <= cx_hi) {
                            const int2 r = __ldg(reach + row0 + (cy + i0 + u) * row_stride + c);
                            okv[u] = r.x >= X0 && r.y >= Y0;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const unsigned m = __ballot_sync(0xffffffffu, okv[u]);
                        if (lane == i0 + u && m) {
                            mylo = cx_lo + __ffs(m) - 1;
                            myhi = cx_lo + 31 - __clz(m);
                        }
                    }
                }
            } else {
                for (int i = 0; i < nrows; ++i) {
                    int lo, hi;
                    const bool any = reach_trim(reach, row0 + (cy + i) * row_stride, cx_lo,
                                                cx_hi, X0, Y0, lane, &lo, &hi);
                    if (any && lane == i) { mylo = lo; myhi = hi; }
                }
            }
            int s0 = 0, len = 0;
            if (lane < nrows && myhi >= mylo) {
                const int row = row0 + (cy + lane) * row_stride;
                s0 = cs[row + mylo];
                len = cs[row + myhi + 1] - s0;
            }
            int inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            cy += nrows;
            const int total = __shfl_sync(0xffffffffu, inc, 31);
            if (total > 0 || nrows == 0) {
                ch.st[lane] = s0;
                ch.pre[lane + 1] = inc;
                if (lane == 0) {
                    ch.pre[0] = 0;
                    ch.cy_next = cy;
                }
                return;
            }
        }
    }
};

// position v of the chunk -> record index (r: a chunk row at or before v's row)
__device__ __forceinline__ int cand_index(const CandChunk& ch, int v, int r) {
    while (v >= ch.pre[r + 1]) ++r;
    GSR_CHECK(r >= 0 && r < 32 && v >= ch.pre[r]);
    return ch.st[r] + (v - ch.pre[r]);
}

// Tile candidate query over the cell grid (binning.cu): the Gaussians whose unclipped support
// origin lies in [T0 - ext + 1, T1]; ext >= 1 keeps the cell range non-empty and in bounds.
__device__ __forceinline__ int query_ext(const int* ext, int k, int axis) {
    return max(1, ext[2 * k + axis]);
}

// binning.cu
size_t binning_bytes(long long n, int total_cells, int total_tiles);
void carve_workspace(void* base, long long n, int total_cells, int total_tiles, Workspace* ws);
// Runs K1 (keys) + stable radix sort + cell starts + K1b (records). Returns sorted perm in
// *perm_out (points into ws).
// Parameter arrays are float32, or bfloat16 when tab.params_bf16 (GSR_PARAMS_BF16).
// gidx (subset mode): binned position t stands for Gaussian gidx[t] (n entries); nullptr = t.
cudaError_t bin_gaussians(const void* alpha, const void* mu, const void* sigma,
                          const void* rho, const void* color, long long n,
                          const ImgTable& tab, Workspace& ws, int** perm_out,
                          uint32_t** keys_sorted_out, cudaStream_t st,
                          const int* gidx = nullptr);
// Where a previous bin_gaussians() on the same table left perm / sorted keys in the workspace.
void binned_pointers(const ImgTable& tab, long long n, const Workspace& ws, int** perm,
                     uint32_t** keys_sorted);
cudaError_t launch_pair_count(const void* alpha, const void* mu, const void* sigma,
                              const void* rho, const void* color, long long n,
                              const ImgTable& tab, bool support, long long* d_pairs,
                              cudaStream_t st);
cudaError_t launch_validate(const void* alpha, const void* mu, const void* sigma,
                            const void* rho, const void* color, long long n, bool bf16,
                            unsigned long long* d_out, cudaStream_t st);
cudaError_t launch_debug_rects(const float* alpha, const float* mu, const float* sigma,
                               const float* rho, const float* color, long long n,
                               const ImgTable& tab, bool support, int* rects, cudaStream_t st);
cudaError_t launch_debug_tile_lists(const ImgTable& tab, const Workspace& ws, const int* perm,
                                    const uint32_t* keys_sorted, int* counts, int* ids,
                                    int* cells, cudaStream_t st);
cudaError_t exclusive_scan_i32(const int* in, int* out, long long n, int* tmp, cudaStream_t st);

// plan.cu (K7)
cudaError_t launch_row_pair_counts(const void* alpha, const void* mu, const void* sigma,
                                   const void* rho, const void* color, long long n,
                                   const ImgTable& tab, bool support, const RowOff& roff,
                                   long long* d_out, cudaStream_t st);
void row_pair_counts_host(const void* alpha, const void* mu, const void* sigma, const void* rho,
                          const void* color, long long n, const ImgTable& tab, bool support,
                          const RowOff& roff, long long* out);
cudaError_t launch_band_span(const void* alpha, const void* mu, const void* sigma,
                             const void* rho, const void* color, long long n, const ImgTable& tab,
                             const BandTable& bt, int16_t* d_span, cudaStream_t st);
void band_span_host(const void* alpha, const void* mu, const void* sigma, const void* rho,
                    const void* color, long long n, const ImgTable& tab, const BandTable& bt,
                    int16_t* span);

size_t rank_halo_bytes(long long n);
cudaError_t launch_rank_halo(const void* alpha, const void* mu, const void* sigma,
                             const void* rho, const void* color, long long n, const ImgTable& tab,
                             const BandTable& bt, int rank, void* ws, int* idx, int* up,
                             int* down, int* multi_pos, int* multi_slot, long long* totals,
                             cudaStream_t st);

// render_fwd.cu
cudaError_t launch_render_fwd(const ImgTable& tab, const Workspace& ws, float* out,
                              cudaStream_t st, const float* gt = nullptr,
                              double* loss_acc = nullptr);
// test-only: the forward tiles' kept candidates (offs == nullptr: counts[total_ftiles] only)
cudaError_t launch_debug_fwd_lists(const ImgTable& tab, const Workspace& ws, const int* perm,
                                   const int* offs, int* counts, int* ids, uint8_t* paths,
                                   cudaStream_t st);
// render_bwd.cu
// grad_out = dL/dI, or (img, gt != nullptr) the fused L1 gradient sign(img - gt) * inv_numel
cudaError_t launch_render_bwd_moments(const ImgTable& tab, const Workspace& ws, const int* perm,
                                      const float* grad_out, double* moments, cudaStream_t st,
                                      const float* img = nullptr, const float* gt = nullptr,
                                      float inv_numel = 0.f);
// Raw-parameter mode of the finalize (NEXT-1 activation layer): when raw != nullptr the
// gradients are chained through alpha = sigmoid, c = sigmoid, sigma = sigmoid,
// rho = rho_scale tanh, mu = p + o, using the raw inputs for the Jacobians.
struct RawParams {
    const float* raw_alpha; const float* raw_sigma; const float* raw_rho; const float* raw_color;
    float rho_scale;
};
// gidx (subset mode): entry t of moments / d_* belongs to Gaussian gidx[t] (n entries, compact)
cudaError_t launch_finalize(const void* alpha, const void* mu, const void* sigma,
                            const void* rho, const void* color, long long n,
                            const double* moments, float* d_alpha, float* d_mu, float* d_sigma,
                            float* d_rho, float* d_color, cudaStream_t st,
                            const RawParams* raw = nullptr, bool params_bf16 = false,
                            const int* gidx = nullptr);
// train.cu
cudaError_t launch_activate(const float* raw_alpha, const float* offset, const float* ref,
                            const float* raw_sigma, const float* raw_rho, const float* raw_color,
                            long long n, float rho_scale, float* alpha, float* mu, float* sigma,
                            float* rho, float* color, cudaStream_t st);
cudaError_t launch_scale_loss(double* loss, double scale, cudaStream_t st);

}  // namespace gsr
