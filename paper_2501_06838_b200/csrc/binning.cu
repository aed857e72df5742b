// binning.cu -- K1 (window rect + cell key), stable LSD radix sort, cell starts, K1b (records),
// pair count and the debug introspection kernels.
//
// Binning: every Gaussian's window has the same size (Alg. 1 window
// r*W x r*H in LR px, P:1385 / reading R1-R2), so a render tile's candidates are the Gaussians
// whose unclipped rect origin (x0u, y0u) lies in [Tx0 - wmax + 1, Tx1] x [Ty0 - hmax + 1, Ty1].
// Sorting Gaussians by the CELL x CELL cell of that origin turns each tile's candidate set into
// one contiguous record span per cell row -- no per-(Gaussian, tile) key duplication.
#include <utility>

#include "gsr_internal.cuh"

namespace gsr {

namespace {

constexpr int RS_WARPS = 8;
constexpr int RS_THREADS = RS_WARPS * 32;
constexpr int RS_SEG = 256;                      // items per warp segment
constexpr int RS_BLOCK = RS_WARPS * RS_SEG;      // 2048 items per block
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_BLOCK = SCAN_THREADS * SCAN_ITEMS;

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

long long rs_blocks(long long n) { return (n + RS_BLOCK - 1) / RS_BLOCK; }
long long scan_blocks(long long n) { return (n + SCAN_BLOCK - 1) / SCAN_BLOCK; }

// ---- K1: keys ----------------------------------------------------------------------------
// Binned positions t = 0..n-1 stand for Gaussian i = gidx[t] (subset mode: a rank's halo, see
// gsr_render_fwd_subset) or i = t (gidx == nullptr); vals/perm hold t, so every per-Gaussian
// output of the backward (moments, gradients) is indexed by t.
template <class T>
__global__ void k_keys(const T* __restrict__ alpha, const T* __restrict__ mu,
                       const T* __restrict__ sigma, const T* __restrict__ rho,
                       const T* __restrict__ color, long long n, ImgTable tab,
                       const int* __restrict__ gidx, uint32_t* __restrict__ keys,
                       int* __restrict__ vals, int* __restrict__ ext) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t key = (uint32_t)tab.total_cells;
    int k = -1, wx = 0, wy = 0;
    if (t < n) {
        const long long i = gidx ? (long long)gidx[t] : t;
        k = find_image_by_gauss(tab, i);
        if (k >= 0) {
            const DevImg& im = tab.img[k];
            float mx = ldf(mu[2 * i]), my = ldf(mu[2 * i + 1]);
            if (valid_at(alpha, mu, sigma, rho, color, i)) {
                Rect r = support_rect(mx, my, ldf(sigma[2 * i]), ldf(sigma[2 * i + 1]), im);
                if (r.nonempty) {
                    // key: cell of the unclipped support origin (>= the window origin, so
                    // inside the window-sized cell domain)
                    int cx = (r.x0u + im.offx) / CELL;
                    int cy = (r.y0u - im.row_begin + im.offy) / CELL;
                    key = (uint32_t)(im.cell_base + cy * im.ncx + cx);
                    wx = r.x1u - r.x0u + 1;
                    wy = r.y1u - r.y0u + 1;
                }
            }
        }
        keys[t] = key;
        vals[t] = (int)t;
    }
    // per-image max support extent: warp max over lanes of the same image (each group of lanes
    // with the same image reduces with its own group-uniform mask), then a block max in shared
    // memory, then one global atomic per (block, image) -- every warp of an image hitting the
    // same two global words serialised K1 on them (C5: ~86k warps per 4 images)
    __shared__ int bext[2 * MAX_IMAGES];
    for (int j = threadIdx.x; j < 2 * MAX_IMAGES; j += blockDim.x) bext[j] = 0;
    __syncthreads();
    const unsigned full = 0xffffffffu;
    const unsigned same = __match_any_sync(full, k);
    const int mwx = (int)__reduce_max_sync(same, (unsigned)wx);
    const int mwy = (int)__reduce_max_sync(same, (unsigned)wy);
    if (k >= 0 && (same & ((1u << (threadIdx.x & 31)) - 1u)) == 0 && (mwx | mwy)) {
        atomicMax(&bext[2 * k], mwx);
        atomicMax(&bext[2 * k + 1], mwy);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < 2 * MAX_IMAGES; j += blockDim.x)
        if (bext[j] > 0) atomicMax(&ext[j], bext[j]);
}

// ---- stable LSD radix sort, 8-bit digits -----------------------------------------------
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t* __restrict__ keys,
                                                        long long n, int shift,
                                                        int* __restrict__ hist, int nblocks) {
    __shared__ int cnt[256];
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) cnt[d] = 0;
    __syncthreads();
    const long long b0 = (long long)blockIdx.x * RS_BLOCK;
    constexpr int NI = RS_BLOCK / RS_THREADS;
    uint32_t k[NI];
#pragma unroll
    for (int c = 0; c < NI; ++c) {                  // loads together, then the counts
        const long long i = b0 + c * RS_THREADS + threadIdx.x;
        k[c] = i < n ? keys[i] : 0xffffffffu;
    }
#pragma unroll
    for (int c = 0; c < NI; ++c)
        if (b0 + c * RS_THREADS + threadIdx.x < n) atomicAdd(&cnt[(k[c] >> shift) & 255u], 1);
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RS_THREADS)
        hist[(long long)d * nblocks + blockIdx.x] = cnt[d];
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(
    const uint32_t* __restrict__ keys_in, const int* __restrict__ vals_in, long long n, int shift,
    const int* __restrict__ offs, int nblocks, uint32_t* __restrict__ keys_out,
    int* __restrict__ vals_out) {
    __shared__ int wcnt[RS_WARPS][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = threadIdx.x; d < RS_WARPS * 256; d += RS_THREADS) (&wcnt[0][0])[d] = 0;
    __syncthreads();
    const long long seg = (long long)blockIdx.x * RS_BLOCK + (long long)warp * RS_SEG;
    const unsigned lt = (1u << lane) - 1u;
    // the warp's RS_SEG keys and values, loaded together (one round of memory latency instead
    // of one per 32 items: small sorts are latency-bound, C1 has 18 blocks)
    constexpr int NI = RS_SEG / 32;
    uint32_t key[NI];
    int val[NI];
#pragma unroll
    for (int c = 0; c < NI; ++c) {
        const long long i = seg + 32 * c + lane;
        key[c] = i < n ? keys_in[i] : 0u;
        val[c] = i < n ? vals_in[i] : 0;
    }
    // pass 1: per-warp digit counts
#pragma unroll
    for (int c = 0; c < NI; ++c) {
        const bool valid = seg + 32 * c + lane < n;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (vm == 0) break;
        if (valid) {
            const unsigned d = (key[c] >> shift) & 255u;
            const unsigned peers = __match_any_sync(vm, d);
            if ((peers & lt) == 0) wcnt[warp][d] += __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps + global (digit, block) offset
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
        int run = offs[(long long)d * nblocks + blockIdx.x];
        for (int w = 0; w < RS_WARPS; ++w) {
            int t = wcnt[w][d];
            wcnt[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
    // pass 2: stable ranks and scatter
#pragma unroll
    for (int c = 0; c < NI; ++c) {
        const bool valid = seg + 32 * c + lane < n;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (vm == 0) break;
        unsigned d = 0, peers = 0;
        int pos = 0;
        if (valid) {
            d = (key[c] >> shift) & 255u;
            peers = __match_any_sync(vm, d);
            pos = wcnt[warp][d] + __popc(peers & lt);
        }
        __syncwarp();
        if (valid) {
            if ((peers & lt) == 0) wcnt[warp][d] += __popc(peers);
            GSR_CHECK(pos >= 0 && pos < n);
            keys_out[pos] = key[c];
            vals_out[pos] = val[c];
        }
        __syncwarp();
    }
}

// ---- exclusive scan (int32), reduce-then-scan ----------------------------------------------
__device__ __forceinline__ int block_incl_scan(int v, int* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        sh[lane] = w;
    }
    __syncthreads();
    int r = v + (warp > 0 ? sh[warp - 1] : 0);
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const int* __restrict__ in,
                                                              long long n,
                                                              int* __restrict__ sums) {
    __shared__ int sh[32];
    long long base = (long long)blockIdx.x * SCAN_BLOCK + (long long)threadIdx.x * SCAN_ITEMS;
    int v = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j)
        if (base + j < n) v += in[base + j];
    int incl = block_incl_scan(v, sh);
    if (threadIdx.x == SCAN_THREADS - 1) sums[blockIdx.x] = incl;
}

// single block: exclusive scan of the block sums in place (any count, sequential chunks)
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_sums(int* __restrict__ sums,
                                                            long long nb) {
    __shared__ int sh[32];
    __shared__ int last;
    int carry = 0;
    for (long long c = 0; c < nb; c += SCAN_THREADS) {
        long long i = c + threadIdx.x;
        int v = i < nb ? sums[i] : 0;
        int incl = block_incl_scan(v, sh);
        if (i < nb) sums[i] = carry + incl - v;
        if (threadIdx.x == SCAN_THREADS - 1) last = incl;
        __syncthreads();
        carry += last;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_down(const int* __restrict__ in,
                                                            long long n,
                                                            const int* __restrict__ sums,
                                                            int* __restrict__ out) {
    __shared__ int sh[32];
    long long base = (long long)blockIdx.x * SCAN_BLOCK + (long long)threadIdx.x * SCAN_ITEMS;
    int v[SCAN_ITEMS];
    int t = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        v[j] = (base + j < n) ? in[base + j] : 0;
        t += v[j];
    }
    int incl = block_incl_scan(t, sh);
    int run = sums[blockIdx.x] + incl - t;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        if (base + j < n) out[base + j] = run;
        run += v[j];
    }
}

// single block, whole array: sequential SCAN_BLOCK chunks with a carry (small scans: one
// launch instead of three)
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_single(const int* __restrict__ in,
                                                              long long n,
                                                              int* __restrict__ out) {
    __shared__ int sh[32];
    __shared__ int last;
    int carry = 0;
    for (long long c = 0; c < n; c += SCAN_BLOCK) {
        const long long base = c + (long long)threadIdx.x * SCAN_ITEMS;
        int v[SCAN_ITEMS];
        int t = 0;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            v[j] = (base + j < n) ? in[base + j] : 0;
            t += v[j];
        }
        const int incl = block_incl_scan(t, sh);
        int run = carry + incl - t;
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            if (base + j < n) out[base + j] = run;
            run += v[j];
        }
        if (threadIdx.x == SCAN_THREADS - 1) last = incl;
        __syncthreads();
        carry += last;
        __syncthreads();
    }
}

// ---- cell starts from sorted keys --------------------------------------------------------
// (and the empty reach of every cell, which K1b then raises for the non-empty ones)
__global__ void k_cell_start(const uint32_t* __restrict__ keys, long long n, int total_cells,
                             int* __restrict__ cell_start, int2* __restrict__ reach) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p > n) return;
    long long prev = p == 0 ? -1 : (long long)keys[p - 1];
    long long cur = p == n ? (long long)total_cells : (long long)keys[p];
    if (cur > total_cells) cur = total_cells;
    for (long long c = prev + 1; c <= cur; ++c) {
        cell_start[c] = (int)p;
        if (c < total_cells) reach[c] = make_int2(-1, -1);
    }
}

// ---- K1b: records in sorted order ---------------------------------------------------------
template <class T>
__global__ void k_records(const T* __restrict__ alpha, const T* __restrict__ mu,
                          const T* __restrict__ sigma, const T* __restrict__ rho,
                          const T* __restrict__ color, long long n, ImgTable tab,
                          const int* __restrict__ gidx, const uint32_t* __restrict__ keys,
                          const int* __restrict__ perm, float4* __restrict__ rec,
                          int4* __restrict__ rects, uint8_t* __restrict__ cls,
                          int2* __restrict__ reach) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // the key and the permutation are independent loads; the Gaussian's nine parameters are
    // then gathered together (one round of memory latency each instead of a chain)
    const uint32_t key = p < n ? keys[p] : 0xffffffffu;
    const bool valid = key < (uint32_t)tab.total_cells;
    // cell reach (Workspace::reach): the warp's lanes of one cell (sorted keys: contiguous)
    // reduce their support rects' right / bottom edges, one atomic pair per cell and warp
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const int pi = perm[p];
    const long long i = gidx ? (long long)gidx[pi] : (long long)pi;
    const float mxf = ldf(mu[2 * i]), myf = ldf(mu[2 * i + 1]);
    const float sxf = ldf(sigma[2 * i]), syf = ldf(sigma[2 * i + 1]);
    const float rhf = ldf(rho[i]), alf = ldf(alpha[i]);
    const float c0f = ldf(color[3 * i]), c1f = ldf(color[3 * i + 1]), c2f = ldf(color[3 * i + 2]);
    int k = find_image_by_gauss(tab, i);
    const DevImg& im = tab.img[k];
    Rect r = window_rect(mxf, myf, im);
    Rect sr = support_rect(mxf, myf, sxf, syf, im);
    double mx = mxf, my = myf;
    double sx = sxf, sy = syf;
    double rh = rhf, al = alf;
    double D = (1.0 - rh) * (1.0 + rh);
    // exponent in factored form (no cancellation):
    //   q = -Q/2 log2 e = -(w'^2 + v'^2),  w' = a1 dx + b1 dy,  v' = c1 dy
    //   a1 = sqrt(k/D)/sx, b1 = -rho sqrt(k/D)/sy, c1 = sqrt(k)/sy,  k = log2(e)/2
    double kd = sqrt(HALF_LOG2E / D);
    double a1 = kd / sx, b1 = -rh * kd / sy, c1 = sqrt(HALF_LOG2E) / sy;
    double K = 1.0 / (TWO_PI * sx * sy * sqrt(D));
    double axd = rint(im.sx * mx), ayd = rint(im.sy * my);   // anchor: nearest HR pixel
    double dlx = mx - axd / im.sx, dly = my - ayd / im.sy;
    double w = al * K;
    // consumer form: r0 = {-ax, ay, dl_y, D}, r1 = {-a1 dl_x, b1, c1, c'_r}
    // with D = a1/s formed in fp32 (the recurrence constants below use the same D)
    const float a1f = (float)a1;
    const float Df = a1f * im.invsx, d2 = Df * Df;
    float4 r0 = make_float4((float)(-axd), (float)ayd, (float)dly, Df);
    float4 r1 = make_float4((float)(-a1 * dlx), (float)b1, (float)c1, (float)(w * c0f));
    unsigned xs = (unsigned)r.x0 | ((unsigned)r.x1 << 16);
    unsigned ys = (unsigned)r.y0 | ((unsigned)r.y1 << 16);
    float4 r2 = make_float4((float)(w * c1f), (float)(w * c2f), __uint_as_float(xs),
                            __uint_as_float(ys));
    // r3: the forward's exponential-recurrence constants G_t = 2^(-D^2 t^2), t = 1..3, and -2D
    // (exact in fp32), when the recurrence is allowed (D <= FWD_REC_DMAX, render_fwd.cu MODE 2)
    const bool rec_ok = Df <= FWD_REC_DMAX;
    float4 r3 = make_float4(rec_ok ? exp2f(-d2) : 0.f, rec_ok ? exp2f(-4.f * d2) : 0.f,
                            rec_ok ? exp2f(-9.f * d2) : 0.f, rec_ok ? -2.f * Df : 0.f);
    rec[REC_F4 * p + 0] = r0;
    rec[REC_F4 * p + 1] = r1;
    rec[REC_F4 * p + 2] = r2;
    rec[REC_F4 * p + 3] = r3;
    // the rect stream the render kernels filter with (16 B per binned Gaussian)
    unsigned sxs = (unsigned)sr.x0 | ((unsigned)sr.x1 << 16);
    unsigned sys = (unsigned)sr.y0 | ((unsigned)sr.y1 << 16);
    rects[p] = make_int4((int)sxs, (int)sys, (int)xs, (int)ys);
    cls[p] = rec_ok ? 1 : 0;
    const unsigned grp = __match_any_sync(vm, key);
    const int mx1 = (int)__reduce_max_sync(grp, (unsigned)sr.x1);
    const int my1 = (int)__reduce_max_sync(grp, (unsigned)sr.y1);
    if ((threadIdx.x & 31) == __ffs(grp) - 1) {
        GSR_CHECK(key < (uint32_t)tab.total_cells && mx1 >= 0 && my1 >= 0);
        atomicMax(&reach[key].x, mx1);
        atomicMax(&reach[key].y, my1);
    }
}

// ---- pair count ---------------------------------------------------------------------------
template <class T>
__global__ void k_pair_count(const T* __restrict__ alpha, const T* __restrict__ mu,
                             const T* __restrict__ sigma, const T* __restrict__ rho,
                             const T* __restrict__ color, long long n, ImgTable tab,
                             bool support, unsigned long long* __restrict__ out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long v = 0;
    if (i < n) {
        int k = find_image_by_gauss(tab, i);
        if (k >= 0) {
            const DevImg& im = tab.img[k];
            float mx = ldf(mu[2 * i]), my = ldf(mu[2 * i + 1]);
            if (valid_at(alpha, mu, sigma, rho, color, i)) {
                Rect r = support ? support_rect(mx, my, ldf(sigma[2 * i]), ldf(sigma[2 * i + 1]),
                                                im)
                                 : window_rect(mx, my, im);
                if (r.nonempty)
                    v = (unsigned long long)(r.x1 - r.x0 + 1) * (unsigned long long)(r.y1 - r.y0 + 1);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

// R20 parameter-domain check (gsr_validate_params): count of invalid Gaussians and the smallest
// invalid index (atomicMin), per call
template <class T>
__global__ void k_validate(const T* __restrict__ alpha, const T* __restrict__ mu,
                           const T* __restrict__ sigma, const T* __restrict__ rho,
                           const T* __restrict__ color, long long n,
                           unsigned long long* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool bad = i < n && !valid_at(alpha, mu, sigma, rho, color, i);
    const unsigned m = __ballot_sync(0xffffffffu, bad);
    if (m && (threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], (unsigned long long)__popc(m));
        atomicMin(&out[1], (unsigned long long)(i + __ffs(m) - 1));
    }
}

__global__ void k_debug_rects(const float* __restrict__ alpha, const float* __restrict__ mu,
                              const float* __restrict__ sigma, const float* __restrict__ rho,
                              const float* __restrict__ color, long long n, ImgTable tab,
                              bool support, int4* __restrict__ rects) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int4 o = make_int4(1, 0, 1, 0);
    int k = find_image_by_gauss(tab, i);
    if (k >= 0) {
        const DevImg& im = tab.img[k];
        float mx = ldf(mu[2 * i]), my = ldf(mu[2 * i + 1]);
        if (valid_at(alpha, mu, sigma, rho, color, i)) {
            Rect r = support ? support_rect(mx, my, ldf(sigma[2 * i]), ldf(sigma[2 * i + 1]), im)
                             : window_rect(mx, my, im);
            if (r.nonempty) o = make_int4(r.x0, r.x1, r.y0, r.y1);
        }
    }
    rects[i] = o;
}

// Materialised per-tile candidate lists of the backward's tiles, walking the same cell spans as
// K5 (untrimmed cell rows) and keeping the candidates whose rect intersects the tile. One thread
// per tile (test-only; the forward's walk is materialised by k_debug_fwd_lists).
__global__ void k_debug_tile_lists(ImgTable tab, const int* __restrict__ ext,
                                   const int* __restrict__ cell_start,
                                   const int4* __restrict__ rects, const int* __restrict__ perm,
                                   const uint32_t* __restrict__ keys,
                                   const int* __restrict__ tile_off, int* __restrict__ counts,
                                   int* __restrict__ ids, int* __restrict__ cells) {
    int tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= tab.total_tiles) return;
    const int kimg = find_image_by_tile(tab, tile);
    const DevImg& im = tab.img[kimg];
    int t = tile - im.tile_base;
    int Tx0 = (t % im.ntx) * TILE_W, Ty0 = im.row_begin + (t / im.ntx) * TILE_H;
    int Tx1 = min(Tx0 + TILE_W - 1, im.Ws - 1), Ty1 = min(Ty0 + TILE_H - 1, im.row_end - 1);
    int cx_lo = (Tx0 - query_ext(ext, kimg, 0) + 1 + im.offx) / CELL;
    int cx_hi = min(im.ncx - 1, (Tx1 + im.offx) / CELL);
    int cy_lo = (Ty0 - im.row_begin - query_ext(ext, kimg, 1) + 1 + im.offy) / CELL;
    int cy_hi = min(im.ncy - 1, (Ty1 - im.row_begin + im.offy) / CELL);
    int c = 0;
    int base = ids ? tile_off[tile] : 0;
    for (int cy = cy_lo; cy <= cy_hi; ++cy) {
        int row = im.cell_base + cy * im.ncx;
        for (int p = cell_start[row + cx_lo]; p < cell_start[row + cx_hi + 1]; ++p) {
            const int4 rc = rects[p];
            unsigned xs = (unsigned)rc.x, ys = (unsigned)rc.y;
            int x0 = xs & 0xffff, x1 = xs >> 16, y0 = ys & 0xffff, y1 = ys >> 16;
            if (x1 < Tx0 || x0 > Tx1 || y1 < Ty0 || y0 > Ty1) continue;
            if (ids) {
                ids[base + c] = perm[p];
                cells[base + c] = (int)keys[p];
            }
            ++c;
        }
    }
    if (!ids) counts[tile] = c;
}

inline unsigned grid1d(long long n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

size_t binning_bytes(long long n, int total_cells, int total_tiles) {
    size_t b = 0;
    long long nb = rs_blocks(n);
    long long hist = 256 * nb;
    long long scan_src = hist > (long long)total_tiles + 1 ? hist : (long long)total_tiles + 1;
    b += 2 * align256(sizeof(uint32_t) * (size_t)n);            // keys a/b
    b += 2 * align256(sizeof(int) * (size_t)n);                 // vals a/b
    b += align256(sizeof(int) * (size_t)(hist + 1));            // hist
    b += align256(sizeof(int) * (size_t)(scan_blocks(scan_src) + 1));  // scan tmp
    b += align256(sizeof(int) * (size_t)(total_cells + 1));     // cell_start
    b += align256(sizeof(int2) * (size_t)(total_cells + 1));    // cell reach
    b += align256(sizeof(float4) * REC_F4 * (size_t)n);         // records
    b += align256(sizeof(int4) * (size_t)n);                    // rect stream
    b += align256((size_t)n);                                   // record classes
    b += align256(sizeof(double) * 8 * (size_t)n);              // moments
    b += align256(sizeof(unsigned long long) * 4);              // counters
    b += align256(sizeof(int) * (size_t)(total_tiles + 1));     // debug tile offsets
    b += align256(sizeof(int) * 2 * MAX_IMAGES);                // support extents
    return b + 256;
}

void carve_workspace(void* base, long long n, int total_cells, int total_tiles, Workspace* ws) {
    char* p = (char*)(((uintptr_t)base + 255) & ~uintptr_t(255));
    auto take = [&](size_t bytes) { char* r = p; p += align256(bytes); return (void*)r; };
    long long nb = rs_blocks(n);
    long long hist = 256 * nb;
    long long scan_src = hist > (long long)total_tiles + 1 ? hist : (long long)total_tiles + 1;
    ws->keys_a = (uint32_t*)take(sizeof(uint32_t) * (size_t)n);
    ws->keys_b = (uint32_t*)take(sizeof(uint32_t) * (size_t)n);
    ws->vals_a = (int*)take(sizeof(int) * (size_t)n);
    ws->vals_b = (int*)take(sizeof(int) * (size_t)n);
    ws->hist = (int*)take(sizeof(int) * (size_t)(hist + 1));
    ws->scan_tmp = (int*)take(sizeof(int) * (size_t)(scan_blocks(scan_src) + 1));
    ws->cell_start = (int*)take(sizeof(int) * (size_t)(total_cells + 1));
    ws->reach = (int2*)take(sizeof(int2) * (size_t)(total_cells + 1));
    ws->rec = (float4*)take(sizeof(float4) * REC_F4 * (size_t)n);
    ws->rects = (int4*)take(sizeof(int4) * (size_t)n);
    ws->cls = (uint8_t*)take((size_t)n);
    ws->moments = (double*)take(sizeof(double) * 8 * (size_t)n);
    ws->counter = (unsigned long long*)take(sizeof(unsigned long long) * 4);
    ws->tile_off = (int*)take(sizeof(int) * (size_t)(total_tiles + 1));
    ws->ext = (int*)take(sizeof(int) * 2 * MAX_IMAGES);
}

cudaError_t exclusive_scan_i32(const int* in, int* out, long long n, int* tmp, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    long long nb = scan_blocks(n);
    if (nb <= 4) {                                 // in-place safe: each chunk reads before it writes
        count_launches(1);
        k_scan_single<<<1, SCAN_THREADS, 0, st>>>(in, n, out);
        return cudaGetLastError();
    }
    count_launches(3);
    k_scan_reduce<<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, n, tmp);
    k_scan_sums<<<1, SCAN_THREADS, 0, st>>>(tmp, nb);
    k_scan_down<<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, n, tmp, out);
    return cudaGetLastError();
}

template <class T>
cudaError_t bin_gaussians_t(const T* alpha, const T* mu, const T* sigma, const T* rho,
                            const T* color, long long n, const int* gidx,
                          const ImgTable& tab, Workspace& ws, int** perm_out,
                          uint32_t** keys_sorted_out, cudaStream_t st) {
    cudaMemsetAsync(ws.ext, 0, sizeof(int) * 2 * MAX_IMAGES, st);
    if (n > 0) {
        count_launches(1);
        k_keys<<<grid1d(n, 256), 256, 0, st>>>(alpha, mu, sigma, rho, color, n, tab, gidx,
                                               ws.keys_a, ws.vals_a, ws.ext);
        int bits = 32 - __builtin_clz((unsigned)tab.total_cells | 1u);
        int passes = (bits + 7) / 8;
        long long nb = rs_blocks(n);
        uint32_t* kin = ws.keys_a; uint32_t* kout = ws.keys_b;
        int* vin = ws.vals_a; int* vout = ws.vals_b;
        for (int ps = 0; ps < passes; ++ps) {
            int shift = 8 * ps;
            count_launches(2);
            k_rs_hist<<<(unsigned)nb, RS_THREADS, 0, st>>>(kin, n, shift, ws.hist, (int)nb);
            cudaError_t e = exclusive_scan_i32(ws.hist, ws.hist, 256 * nb, ws.scan_tmp, st);
            if (e != cudaSuccess) return e;
            k_rs_scatter<<<(unsigned)nb, RS_THREADS, 0, st>>>(kin, vin, n, shift, ws.hist,
                                                             (int)nb, kout, vout);
            std::swap(kin, kout);
            std::swap(vin, vout);
        }
        count_launches(2);
        k_cell_start<<<grid1d(n + 1, 256), 256, 0, st>>>(kin, n, tab.total_cells,
                                                         ws.cell_start, ws.reach);
        k_records<<<grid1d(n, 256), 256, 0, st>>>(alpha, mu, sigma, rho, color, n, tab, gidx,
                                                   kin, vin,
                                                   ws.rec, ws.rects, ws.cls, ws.reach);
        *perm_out = vin;
        *keys_sorted_out = kin;
    } else {
        // no Gaussians: every cell is empty
        cudaMemsetAsync(ws.cell_start, 0, sizeof(int) * (size_t)(tab.total_cells + 1), st);
        cudaMemsetAsync(ws.reach, 0xff, sizeof(int2) * (size_t)(tab.total_cells + 1), st);
        *perm_out = ws.vals_a;
        *keys_sorted_out = ws.keys_a;
    }
    return cudaGetLastError();
}

void binned_pointers(const ImgTable& tab, long long n, const Workspace& ws, int** perm,
                     uint32_t** keys_sorted) {
    if (n <= 0) { *perm = ws.vals_a; *keys_sorted = ws.keys_a; return; }
    int bits = 32 - __builtin_clz((unsigned)tab.total_cells | 1u);
    int passes = (bits + 7) / 8;
    bool odd = passes & 1;
    *perm = odd ? ws.vals_b : ws.vals_a;
    *keys_sorted = odd ? ws.keys_b : ws.keys_a;
}

cudaError_t bin_gaussians(const void* alpha, const void* mu, const void* sigma, const void* rho,
                          const void* color, long long n, const ImgTable& tab, Workspace& ws,
                          int** perm_out, uint32_t** keys_sorted_out, cudaStream_t st,
                          const int* gidx) {
    if (tab.params_bf16) {
        using B = __nv_bfloat16;
        return bin_gaussians_t((const B*)alpha, (const B*)mu, (const B*)sigma, (const B*)rho,
                               (const B*)color, n, gidx, tab, ws, perm_out, keys_sorted_out, st);
    }
    return bin_gaussians_t((const float*)alpha, (const float*)mu, (const float*)sigma,
                           (const float*)rho, (const float*)color, n, gidx, tab, ws, perm_out,
                           keys_sorted_out, st);
}

cudaError_t launch_pair_count(const void* alpha, const void* mu, const void* sigma,
                              const void* rho, const void* color, long long n,
                              const ImgTable& tab, bool support, long long* d_pairs,
                              cudaStream_t st) {
    cudaMemsetAsync(d_pairs, 0, sizeof(long long), st);
    if (n > 0) {
        count_launches(1);
        if (tab.params_bf16) {
            using B = __nv_bfloat16;
            k_pair_count<B><<<grid1d(n, 256), 256, 0, st>>>(
                (const B*)alpha, (const B*)mu, (const B*)sigma, (const B*)rho, (const B*)color, n,
                tab, support, (unsigned long long*)d_pairs);
        } else {
            k_pair_count<float><<<grid1d(n, 256), 256, 0, st>>>(
                (const float*)alpha, (const float*)mu, (const float*)sigma, (const float*)rho,
                (const float*)color, n, tab, support, (unsigned long long*)d_pairs);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_validate(const void* alpha, const void* mu, const void* sigma,
                            const void* rho, const void* color, long long n, bool bf16,
                            unsigned long long* d_out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    count_launches(1);
    if (bf16) {
        using B = __nv_bfloat16;
        k_validate<B><<<grid1d(n, 256), 256, 0, st>>>((const B*)alpha, (const B*)mu,
                                                      (const B*)sigma, (const B*)rho,
                                                      (const B*)color, n, d_out);
    } else {
        k_validate<float><<<grid1d(n, 256), 256, 0, st>>>(
            (const float*)alpha, (const float*)mu, (const float*)sigma, (const float*)rho,
            (const float*)color, n, d_out);
    }
    return cudaGetLastError();
}

cudaError_t launch_debug_rects(const float* alpha, const float* mu, const float* sigma,
                               const float* rho, const float* color, long long n,
                               const ImgTable& tab, bool support, int* rects,
                               cudaStream_t st) {
    if (n > 0)
        k_debug_rects<<<grid1d(n, 256), 256, 0, st>>>(alpha, mu, sigma, rho, color, n, tab,
                                                      support, (int4*)rects);
    return cudaGetLastError();
}

cudaError_t launch_debug_tile_lists(const ImgTable& tab, const Workspace& ws, const int* perm,
                                    const uint32_t* keys_sorted, int* counts, int* ids,
                                    int* cells, cudaStream_t st) {
    int nt = tab.total_tiles;
    if (nt <= 0) return cudaSuccess;
    if (!ids) {
        k_debug_tile_lists<<<grid1d(nt, 64), 64, 0, st>>>(tab, ws.ext, ws.cell_start, ws.rects, perm,
                                                          keys_sorted, nullptr, counts, nullptr,
                                                          nullptr);
    } else {
        k_debug_tile_lists<<<grid1d(nt, 64), 64, 0, st>>>(tab, ws.ext, ws.cell_start, ws.rects, perm,
                                                          keys_sorted, nullptr, ws.tile_off,
                                                          nullptr, nullptr);
        cudaError_t e = exclusive_scan_i32(ws.tile_off, ws.tile_off, nt, ws.scan_tmp, st);
        if (e != cudaSuccess) return e;
        k_debug_tile_lists<<<grid1d(nt, 64), 64, 0, st>>>(tab, ws.ext, ws.cell_start, ws.rects, perm,
                                                          keys_sorted, ws.tile_off, counts, ids,
                                                          cells);
    }
    return cudaGetLastError();
}

}  // namespace gsr
