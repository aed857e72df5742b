// plan.cu -- K7: row-band planning for the multi-GPU path, on the device and on
// the host, with the same window / support rect code as the render kernels (gsr_internal.cuh).
//
//   row pair counts  rowpairs[y] = sum_i [y0_i <= y <= y1_i] (x1_i - x0_i + 1) over the rows
//                    of each image's band: the work per HR row, from which the band boundaries
//                    are chosen (equal pair counts per rank). Rect = window rect of Alg. 1
//                    (readings R1/R2) or, with GSR_SUPPORT, the support rect (R21) --
//                    the pairs the kernels evaluate.
//   band span        for boundaries b_0 <= ... <= b_G of an image, the first and last band that
//                    Gaussian i's support rows [y0 - margin, y1 + margin] meet ({-1, -1} when
//                    its support rect is empty or it is invalid, R20). A Gaussian is a SEAM
//                    Gaussian (its gradient is summed over ranks) iff first < last, and belongs
//                    to rank r's halo iff first <= r <= last.
#include "gsr_internal.cuh"

namespace gsr {

namespace {

template <class T>
__host__ __device__ __forceinline__ bool plan_rect(const T* alpha, const T* mu, const T* sigma,
                                                   const T* rho, const T* color, long long i,
                                                   const DevImg& im, bool support, Rect* r) {
    if (!valid_at(alpha, mu, sigma, rho, color, i)) return false;
    const float mx = ldf(mu[2 * i]), my = ldf(mu[2 * i + 1]);
    *r = support ? support_rect(mx, my, ldf(sigma[2 * i]), ldf(sigma[2 * i + 1]), im)
                 : window_rect(mx, my, im);
    return r->nonempty;
}

// first index g in [0, G) with b[g] <= y < b[g+1]; y below b[0] -> 0, at/after b[G] -> G - 1
__host__ __device__ __forceinline__ int band_of(const int* b, int G, int y) {
    int lo = 0, hi = G - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b[mid] <= y) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <class T>
__host__ __device__ __forceinline__ void span_fl(const T* alpha, const T* mu, const T* sigma,
                                                 const T* rho, const T* color, long long i,
                                                 const ImgTable& tab, const BandTable& bt,
                                                 int* first, int* last) {
    int f = -1, l = -1;
    const int k = find_image_by_gauss(tab, i);
    Rect r;
    if (k >= 0 && plan_rect(alpha, mu, sigma, rho, color, i, tab.img[k], true, &r)) {
        const int* b = bt.b[k];
        const int G = bt.G;
        const int ya = r.y0 - bt.margin, yb = r.y1 + bt.margin;
        if (yb >= b[0] && ya < b[G]) {
            f = band_of(b, G, ya < b[0] ? b[0] : ya);
            l = band_of(b, G, yb >= b[G] ? b[G] - 1 : yb);
        }
    }
    *first = f;
    *last = l;
}

template <class T>
__host__ __device__ __forceinline__ void span_one(const T* alpha, const T* mu, const T* sigma,
                                                  const T* rho, const T* color, long long i,
                                                  const ImgTable& tab, const BandTable& bt,
                                                  int16_t* span) {
    int f, l;
    span_fl(alpha, mu, sigma, rho, color, i, tab, bt, &f, &l);
    span[2 * i] = (int16_t)f;
    span[2 * i + 1] = (int16_t)l;
}

template <class T>
__global__ void k_row_diff(const T* __restrict__ alpha, const T* __restrict__ mu,
                           const T* __restrict__ sigma, const T* __restrict__ rho,
                           const T* __restrict__ color, long long n, ImgTable tab, bool support,
                           RowOff roff, long long* __restrict__ diff) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long a0 = -1, a1 = -1, w = 0;
    if (i < n) {
        const int k = find_image_by_gauss(tab, i);
        Rect r;
        if (k >= 0 && plan_rect(alpha, mu, sigma, rho, color, i, tab.img[k], support, &r)) {
            const DevImg& im = tab.img[k];
            w = (long long)(r.x1 - r.x0 + 1);
            a0 = roff.off[k] + (r.y0 - im.row_begin);
            if (r.y1 + 1 < im.row_end) a1 = roff.off[k] + (r.y1 + 1 - im.row_begin);
        }
    }
    // warp-aggregated atomics: consecutive Gaussians share LR rows, hence start/end rows. Each
    // group of lanes with the same address reduces with its own (group-uniform) mask.
    const unsigned full = 0xffffffffu, lt = (1u << (threadIdx.x & 31)) - 1u;
    {
        const unsigned peers = __match_any_sync(full, a0);
        const unsigned s = __reduce_add_sync(peers, (unsigned)w);       // widths < 2^16
        if (a0 >= 0 && (peers & lt) == 0) atomicAdd((unsigned long long*)&diff[a0],
                                                    (unsigned long long)s);
    }
    {
        const unsigned peers = __match_any_sync(full, a1);
        const unsigned s = __reduce_add_sync(peers, (unsigned)w);
        if (a1 >= 0 && (peers & lt) == 0) atomicAdd((unsigned long long*)&diff[a1],
                                                    (unsigned long long)(-(long long)s));
    }
}

// in-place inclusive scan of each image's rows (one CTA per image, sequential 1024-row chunks)
__global__ void __launch_bounds__(1024) k_row_scan(RowOff roff, long long* __restrict__ v) {
    __shared__ long long sh[32];
    __shared__ long long carry_sh;
    const int k = blockIdx.x;
    const long long b0 = roff.off[k], b1 = roff.off[k + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long carry = 0;
    for (long long c = b0; c < b1; c += 1024) {
        const long long i = c + threadIdx.x;
        long long x = i < b1 ? v[i] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        if (lane == 31) sh[warp] = x;
        __syncthreads();
        if (warp == 0) {
            long long y = sh[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += t;
            }
            sh[lane] = y;
        }
        __syncthreads();
        x += (warp > 0 ? sh[warp - 1] : 0) + carry;
        if (i < b1) v[i] = x;
        if (threadIdx.x == 1023) carry_sh = x;
        __syncthreads();
        carry = carry_sh;
        __syncthreads();
    }
}

template <class T>
__global__ void k_band_span(const T* __restrict__ alpha, const T* __restrict__ mu,
                            const T* __restrict__ sigma, const T* __restrict__ rho,
                            const T* __restrict__ color, long long n, ImgTable tab, BandTable bt,
                            int16_t* __restrict__ span) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) span_one(alpha, mu, sigma, rho, color, i, tab, bt, span);
}

template <class T>
void row_counts_host_t(const T* alpha, const T* mu, const T* sigma, const T* rho, const T* color,
                       long long n, const ImgTable& tab, bool support, const RowOff& ro,
                       long long* out) {
    const long long* roff = ro.off;
    for (long long j = 0; j < roff[tab.n_imgs]; ++j) out[j] = 0;
    for (long long i = 0; i < n; ++i) {
        const int k = find_image_by_gauss(tab, i);
        Rect r;
        if (k < 0 || !plan_rect(alpha, mu, sigma, rho, color, i, tab.img[k], support, &r)) continue;
        const DevImg& im = tab.img[k];
        const long long w = r.x1 - r.x0 + 1;
        out[roff[k] + (r.y0 - im.row_begin)] += w;
        if (r.y1 + 1 < im.row_end) out[roff[k] + (r.y1 + 1 - im.row_begin)] -= w;
    }
    for (int k = 0; k < tab.n_imgs; ++k)
        for (long long j = roff[k] + 1; j < roff[k + 1]; ++j) out[j] += out[j - 1];
}

inline unsigned grid1d(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// ---- rank halo (gsr_rank_halo): one rank's halo and seam sets from the band spans ----------
// categories: 0 halo (first <= r <= last), 1 up (span exactly [r, r+1]), 2 down ([r-1, r]),
// 3 multi in halo (last - first >= 2, in halo), 4 multi anywhere (last - first >= 2)
constexpr int HALO_T = 256, HALO_ITEMS = 4, HALO_BLOCK = HALO_T * HALO_ITEMS, NCAT = 5;

template <class T>
__global__ void __launch_bounds__(HALO_T) k_halo_count(
    const T* __restrict__ alpha, const T* __restrict__ mu, const T* __restrict__ sigma,
    const T* __restrict__ rho, const T* __restrict__ color, long long n, ImgTable tab,
    BandTable bt, int rank, uint8_t* __restrict__ flags, int* __restrict__ counts, int nb) {
    __shared__ int sh[NCAT][HALO_T / 32];
    const long long base = (long long)blockIdx.x * HALO_BLOCK + (long long)threadIdx.x * HALO_ITEMS;
    int c[NCAT] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < HALO_ITEMS; ++j) {
        const long long i = base + j;
        if (i >= n) break;
        int f, l;
        span_fl(alpha, mu, sigma, rho, color, i, tab, bt, &f, &l);
        const bool h = f >= 0 && f <= rank && l >= rank;
        const bool u = f == rank && l == rank + 1;
        const bool d = f == rank - 1 && l == rank && f >= 0;
        const bool ma = f >= 0 && l - f >= 2;
        const bool ml = ma && h;
        const uint8_t fl = (uint8_t)(h | (u << 1) | (d << 2) | (ml << 3) | (ma << 4));
        flags[i] = fl;
#pragma unroll
        for (int k = 0; k < NCAT; ++k) c[k] += (fl >> k) & 1;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NCAT; ++k) {
        int v = c[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sh[k][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < NCAT) {
        int v = 0;
        for (int w = 0; w < HALO_T / 32; ++w) v += sh[threadIdx.x][w];
        counts[(long long)threadIdx.x * nb + blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(HALO_T) k_halo_write(
    long long n, const uint8_t* __restrict__ flags, const int* __restrict__ offs, int nb,
    int* __restrict__ idx, int* __restrict__ up, int* __restrict__ down,
    int* __restrict__ multi_pos, int* __restrict__ multi_slot) {
    __shared__ int sh[NCAT][HALO_T / 32];
    const long long base = (long long)blockIdx.x * HALO_BLOCK + (long long)threadIdx.x * HALO_ITEMS;
    uint8_t fl[HALO_ITEMS];
    int c[NCAT] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < HALO_ITEMS; ++j) {
        fl[j] = base + j < n ? flags[base + j] : 0;
#pragma unroll
        for (int k = 0; k < NCAT; ++k) c[k] += (fl[j] >> k) & 1;
    }
    // block-exclusive prefix of the per-thread counts, per category
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int pre[NCAT];
#pragma unroll
    for (int k = 0; k < NCAT; ++k) {
        int v = c[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) sh[k][warp] = v;
        pre[k] = v - c[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NCAT; ++k) {
        int w0 = 0;
        for (int w = 0; w < warp; ++w) w0 += sh[k][w];
        pre[k] += w0 + offs[(long long)k * nb + blockIdx.x];
    }
#pragma unroll
    for (int j = 0; j < HALO_ITEMS; ++j) {
        const long long i = base + j;
        const uint8_t f = fl[j];
        const int hpos = pre[0];
        if (f & 1) idx[pre[0]++] = (int)i;
        if (f & 2) up[pre[1]++] = hpos;
        if (f & 4) down[pre[2]++] = hpos;
        if (f & 8) { multi_pos[pre[3]] = hpos; multi_slot[pre[3]++] = pre[4]; }
        if (f & 16) pre[4]++;
    }
}

// offs[k*nb + b] -= offs[k*nb] (the exclusive scan ran over all categories back to back)
__global__ void k_halo_rebase(int* __restrict__ offs, int nb) {
    const long long b0 = (long long)blockIdx.x * nb;
    const int first = offs[b0];
    __syncthreads();
    for (long long b = threadIdx.x; b < nb; b += blockDim.x) offs[b0 + b] -= first;
}

__global__ void k_halo_totals(const int* __restrict__ cnt, const int* __restrict__ offs, int nb,
                              long long* __restrict__ totals) {
    const int k = threadIdx.x;
    if (k < NCAT)
        totals[k] = nb > 0 ? (long long)offs[(long long)k * nb + nb - 1] +
                                 cnt[(long long)k * nb + nb - 1] : 0;
}

}  // namespace

size_t rank_halo_bytes(long long n) {
    const long long nb = (n + HALO_BLOCK - 1) / HALO_BLOCK;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    return al((size_t)n) + 2 * al(sizeof(int) * (size_t)(NCAT * nb + 1)) +
           al(sizeof(int) * (size_t)((NCAT * nb + 4095) / 4096 + 2)) + 256;
}

cudaError_t launch_rank_halo(const void* alpha, const void* mu, const void* sigma,
                             const void* rho, const void* color, long long n, const ImgTable& tab,
                             const BandTable& bt, int rank, void* ws, int* idx, int* up,
                             int* down, int* multi_pos, int* multi_slot, long long* totals,
                             cudaStream_t st) {
    const long long nb = (n + HALO_BLOCK - 1) / HALO_BLOCK;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    char* p = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    uint8_t* flags = (uint8_t*)p; p += al((size_t)n);
    int* cnt = (int*)p; p += al(sizeof(int) * (size_t)(NCAT * nb + 1));
    int* offs = (int*)p; p += al(sizeof(int) * (size_t)(NCAT * nb + 1));
    int* tmp = (int*)p;
    if (nb == 0) {
        cudaMemsetAsync(totals, 0, sizeof(long long) * NCAT, st);
        return cudaGetLastError();
    }
    count_launches(3);
    if (tab.params_bf16) {
        using B = __nv_bfloat16;
        k_halo_count<B><<<(unsigned)nb, HALO_T, 0, st>>>((const B*)alpha, (const B*)mu,
                                                         (const B*)sigma, (const B*)rho,
                                                         (const B*)color, n, tab, bt, rank, flags,
                                                         cnt, (int)nb);
    } else {
        k_halo_count<float><<<(unsigned)nb, HALO_T, 0, st>>>(
            (const float*)alpha, (const float*)mu, (const float*)sigma, (const float*)rho,
            (const float*)color, n, tab, bt, rank, flags, cnt, (int)nb);
    }
    // one exclusive scan over the 5 category-major count arrays, then per-category offsets are
    // the scan minus the category's base (categories are independent)
    cudaError_t e = exclusive_scan_i32(cnt, offs, NCAT * nb, tmp, st);
    if (e != cudaSuccess) return e;
    k_halo_rebase<<<NCAT, 256, 0, st>>>(offs, (int)nb);
    k_halo_write<<<(unsigned)nb, HALO_T, 0, st>>>(n, flags, offs, (int)nb, idx, up, down,
                                                  multi_pos, multi_slot);
    k_halo_totals<<<1, 32, 0, st>>>(cnt, offs, (int)nb, totals);
    return cudaGetLastError();
}

cudaError_t launch_row_pair_counts(const void* alpha, const void* mu, const void* sigma,
                                   const void* rho, const void* color, long long n,
                                   const ImgTable& tab, bool support, const RowOff& roff,
                                   long long* d_out, cudaStream_t st) {
    cudaMemsetAsync(d_out, 0, sizeof(long long) * (size_t)roff.off[tab.n_imgs], st);
    if (n > 0) {
        count_launches(1);
        if (tab.params_bf16) {
            using B = __nv_bfloat16;
            k_row_diff<B><<<grid1d(n, 256), 256, 0, st>>>((const B*)alpha, (const B*)mu,
                                                          (const B*)sigma, (const B*)rho,
                                                          (const B*)color, n, tab, support,
                                                          roff, d_out);
        } else {
            k_row_diff<float><<<grid1d(n, 256), 256, 0, st>>>(
                (const float*)alpha, (const float*)mu, (const float*)sigma, (const float*)rho,
                (const float*)color, n, tab, support, roff, d_out);
        }
    }
    count_launches(1);
    k_row_scan<<<tab.n_imgs, 1024, 0, st>>>(roff, d_out);
    return cudaGetLastError();
}

void row_pair_counts_host(const void* alpha, const void* mu, const void* sigma, const void* rho,
                          const void* color, long long n, const ImgTable& tab, bool support,
                          const RowOff& roff, long long* out) {
    if (tab.params_bf16) {
        using B = __nv_bfloat16;
        row_counts_host_t((const B*)alpha, (const B*)mu, (const B*)sigma, (const B*)rho,
                          (const B*)color, n, tab, support, roff, out);
    } else {
        row_counts_host_t((const float*)alpha, (const float*)mu, (const float*)sigma,
                          (const float*)rho, (const float*)color, n, tab, support, roff, out);
    }
}

cudaError_t launch_band_span(const void* alpha, const void* mu, const void* sigma,
                             const void* rho, const void* color, long long n, const ImgTable& tab,
                             const BandTable& bt, int16_t* d_span, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    count_launches(1);
    if (tab.params_bf16) {
        using B = __nv_bfloat16;
        k_band_span<B><<<grid1d(n, 256), 256, 0, st>>>((const B*)alpha, (const B*)mu,
                                                       (const B*)sigma, (const B*)rho,
                                                       (const B*)color, n, tab, bt, d_span);
    } else {
        k_band_span<float><<<grid1d(n, 256), 256, 0, st>>>(
            (const float*)alpha, (const float*)mu, (const float*)sigma, (const float*)rho,
            (const float*)color, n, tab, bt, d_span);
    }
    return cudaGetLastError();
}

void band_span_host(const void* alpha, const void* mu, const void* sigma, const void* rho,
                    const void* color, long long n, const ImgTable& tab, const BandTable& bt,
                    int16_t* span) {
    for (long long i = 0; i < n; ++i) {
        if (tab.params_bf16) {
            using B = __nv_bfloat16;
            span_one((const B*)alpha, (const B*)mu, (const B*)sigma, (const B*)rho,
                     (const B*)color, i, tab, bt, span);
        } else {
            span_one((const float*)alpha, (const float*)mu, (const float*)sigma,
                     (const float*)rho, (const float*)color, i, tab, bt, span);
        }
    }
}

}  // namespace gsr
